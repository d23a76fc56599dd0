#!/bin/bash
# interleaved A/B of an environment setting: ENV_B (e.g. "AC_PV_SPLITK=1") vs default, bench --config $C
C=${C:-gpt}
mkdir -p gpurun_out
: > gpurun_out/env_ab.txt
for rep in 1 2 3; do
for v in A B; do
  if [ $v = B ]; then E="$ENV_B"; else E=""; fi
  env $E timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu --no-e2e --no-unchunked > gpurun_out/env_$v.json 2>/dev/null
  python - <<PY >> gpurun_out/env_ab.txt
import json
d=json.loads(open("gpurun_out/env_$v.json").read())
st={k:v["ms_per_step"] for k,v in d["stages"].items() if isinstance(v,dict)}
print("$C $rep $v [$E]", d["ms_per_step"], {k:st[k] for k in list(st)[:3]})
PY
done; done
cat gpurun_out/env_ab.txt
