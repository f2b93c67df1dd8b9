#!/bin/bash
O=gpurun_out/dbg3; mkdir -p $O
M="--metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --kernel-name-base demangled -c 3 --csv"
for d in 0 1 2 3 4; do
 for B in 64 128; do
  PETRA_CONV_CTAS=148 PETRA_DBG_HALO=$d timeout 120 ncu $M -k regex:"conv_halo" python tools/conv_one.py 0 2 $B 32 32 64 64 3 1 1 > $O/d${d}_B${B}.csv 2>/dev/null
 done
done
