#!/bin/bash
# parity of the f2 chains, then interleaved A/B of scratch_libs/lib_old.so vs lib_new.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x -k "${PARITY_K:-gpt or f2 or tiny or unet or af or fused or evo}" > gpurun_out/r3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r3_parity.log
tail -3 gpurun_out/r3_parity.log
for C in ${AB_CONFIGS:-gpt}; do bash scripts/ab_libs.sh $C; cp gpurun_out/ab_libs.txt gpurun_out/r3_ab_$C.txt; done
