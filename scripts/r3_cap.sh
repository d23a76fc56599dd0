#!/bin/bash
# ncu --set full of the GPT f2 scores + PV of chunk 5 with source correlation (per-line stalls)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 13 -c 2 \
    -o gpurun_out/r3_full_gpt_attn python scripts/node_run.py gpt > gpurun_out/r3_cap.log 2>&1
echo "rc=$?" >> gpurun_out/r3_cap.log
ls -la gpurun_out
