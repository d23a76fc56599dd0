#!/bin/bash
# ncu --set full on chosen GEMM launches of one GPT bench step. Usage: profile_gemm.sh TAG SKIP COUNT
TAG=$1; SKIP=${2:-20}; CNT=${3:-2}
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s $SKIP -c $CNT \
    -o gpurun_out/profg_${TAG} python bench.py --profile --steps 1 --warmup 1 > gpurun_out/profg_${TAG}.log 2>&1
