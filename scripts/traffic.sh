#!/bin/bash
# DRAM bytes per launch of every gemm / combine launch of one bench step (for roofline.traffic)
for C in gpt unet; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"gemm_tc|stats_combine" --csv --log-file gpurun_out/traffic_${C}.csv \
      python bench.py --profile --config $C --steps 1 --warmup 0 > gpurun_out/traffic_${C}.log 2>&1
done
