#!/bin/bash
# per-unit timeline of the fused PV (UNet chunk), split-K off / on
mkdir -p gpurun_out/tr0 gpurun_out/tr1
AC_PV_SPLITK=0 AC_TRACE=gpurun_out/tr0 timeout 300 python bench.py --config unet --steps 1 --warmup 1 --no-e2e --no-unchunked > /dev/null 2>&1
AC_PV_SPLITK=1 AC_TRACE=gpurun_out/tr1 timeout 300 python bench.py --config unet --steps 1 --warmup 1 --no-e2e --no-unchunked > /dev/null 2>&1
ls gpurun_out/tr0 | wc -l; ls gpurun_out/tr1 | wc -l
