#!/bin/bash
# ncu full captures of the HBM-bound BN kernels in the RevNet-50 step
O=gpurun_out/nbn; mkdir -p $O
for k in bn_bwd_reduce_kernel bn_apply_fixed_kernel bn_bwd_dz_fixed_kernel; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 3 \
  -o $O/$k python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/$k.log 2>&1
done
ls -la $O
