#!/bin/bash
# every (N_res, plan) case of dbg_af.py in its own process under a 60 s timeout
mkdir -p gpurun_out
for n in 64 192; do for i in 0 1 2 3 4; do
  timeout 60 python scripts/dbg_af.py $n $i >> gpurun_out/dbg_af.txt 2>&1 || echo "nres=$n plan=$i rc=$?" >> gpurun_out/dbg_af.txt
done; done
