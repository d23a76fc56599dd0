#!/bin/bash
# A/B two library builds (scratch_libs/lib_old.so, lib_new.so) on one box, interleaved:
# bench.py --config $1 (default gpt), 4 rounds.  Prints ms/step and the first stages.
C=${1:-gpt}
mkdir -p gpurun_out
: > gpurun_out/ab_libs.txt
for rep in 1 2 3 4; do
for v in old new; do
  AC_LIB_PATH=scratch_libs/lib_$v.so timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu --no-e2e --no-unchunked > gpurun_out/ab_$v.json 2>/dev/null
  python - <<PY >> gpurun_out/ab_libs.txt
import json
d=json.loads(open("gpurun_out/ab_$v.json").read())
st={k:v["ms_per_step"] for k,v in d["stages"].items() if isinstance(v,dict)}
print("$rep $v", d["ms_per_step"], {k:st[k] for k in list(st)[:3]})
PY
done; done
cat gpurun_out/ab_libs.txt
