#!/bin/bash
O=gpurun_out/dbg2; mkdir -p $O
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > $O/kt.log 2>&1
M="--metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --kernel-name-base demangled -c 3 --csv"
for d in 0 1; do
 for B in 64 128; do
  PETRA_CONV_CTAS=148 PETRA_DBG_HALO=$d timeout 120 ncu $M -k regex:"conv_halo" python tools/conv_one.py 0 2 $B 32 32 64 64 3 1 1 > $O/d${d}_B${B}.csv 2>/dev/null
 done
done
PETRA_CONV_CTAS=148 timeout 120 ncu $M -k regex:"conv_halo" python tools/conv_one.py 0 2 64 16 16 128 128 3 1 1 > $O/l2_B64.csv 2>/dev/null
PETRA_CONV_CTAS=148 timeout 120 ncu $M -k regex:"conv_halo" python tools/conv_one.py 0 2 64 56 56 64 64 3 1 1 > $O/r50l1_B64.csv 2>/dev/null
