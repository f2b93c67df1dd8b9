#!/bin/bash
set -x
O=gpurun_out/fc; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:"fc_gemm|fc_bias|gap|ce_kernel|loss_mean" -c 12 --csv --log-file $O/fc.csv \
  python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
