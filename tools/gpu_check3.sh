#!/bin/bash
# gpu_check2 + ncu full captures of the C=64 conv kernels
set -x
TAG=${1:-chk}
bash tools/gpu_check2.sh $TAG
O=gpurun_out/$TAG
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"conv_halo_kernel<.int.64" -s 8 -c 2 \
  -o $O/halo64 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu1.log 2>&1
