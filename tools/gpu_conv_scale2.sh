#!/bin/bash
set -x
O=gpurun_out/cs2; mkdir -p $O
M="--metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --kernel-name-base demangled -c 3 --csv"
for B in 32 64 128; do
  timeout 120 ncu $M -k regex:"conv_tc_kernel" python tools/conv_one.py 0 1 $B 32 32 64 64 3 1 1 > $O/tc_B${B}.csv 2>/dev/null
  PETRA_HALO_RESIDENT=0 timeout 120 ncu $M -k regex:"conv_halo" python tools/conv_one.py 0 2 $B 32 32 64 64 3 1 1 > $O/stream_B${B}.csv 2>/dev/null
  timeout 120 ncu $M -k regex:"conv_halo" python tools/conv_one.py 0 2 $B 32 32 64 64 3 1 1 > $O/res_B${B}.csv 2>/dev/null
  timeout 120 ncu $M -k regex:"conv_tc_kernel" python tools/conv_one.py 0 1 $B 32 32 64 256 1 1 1 > $O/tc1x1_B${B}.csv 2>/dev/null
done
ls $O
