#!/bin/bash
# per-launch device time of the R18 layer-1 3x3 conv (halo, resident weights) vs batch and grid cap
set -x
O=gpurun_out/cs; mkdir -p $O
for cap in 148 96 48; do
 for B in 8 16 32 64 128; do
  PETRA_CONV_CTAS=$cap timeout 120 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --kernel-name-base demangled -k regex:"conv_halo" -c 3 --csv \
    python tools/conv_one.py 0 2 $B 32 32 64 64 3 1 1 > $O/cap${cap}_B${B}.csv 2>/dev/null
 done
done
for cap in 148 96; do
 for B in 16 64; do
  PETRA_CONV_CTAS=$cap timeout 120 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --kernel-name-base demangled -k regex:"conv_halo" -c 3 --csv \
    python tools/conv_one.py 0 2 $B 16 16 128 128 3 1 1 > $O/l2cap${cap}_B${B}.csv 2>/dev/null
 done
done
ls $O
