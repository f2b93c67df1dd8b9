#!/bin/bash
set -x
O=gpurun_out/nh; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"conv_halo_kernel<.int.64" -s 8 -c 2 \
  -o $O/halo64 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"conv_tc_kernel<.int.64" -s 8 -c 2 \
  -o $O/tc64 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu2.log 2>&1
ls -la $O
