#!/bin/bash
# ncu --set full of AlphaFold pair-stack kernels: the triangle scores (128-row kernel) and
# the triangle PV of the same chunk (row attention, chunk 2)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 23 -c 2 \
    -o gpurun_out/r3_full_af python scripts/node_run.py af > gpurun_out/r3_af_cap.log 2>&1
echo "rc=$?" >> gpurun_out/r3_af_cap.log
