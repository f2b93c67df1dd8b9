#!/bin/bash
# ncu full captures of the R50 conv_tc kernel (BN=256, bf16 out) and the halo wgrad
O=gpurun_out/ntc; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel" -s 30 -c 4 \
  -o $O/tc python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wgrad_halo_kernel" -s 4 -c 2 \
  -o $O/wh python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/wh.log 2>&1
ls -la $O
