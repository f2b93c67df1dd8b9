#!/bin/bash
# ncu full captures of the R18 small convs (conv_tc BN=64 fwd and dgrad)
O=gpurun_out/n18; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel" -s 40 -c 6 \
  -o $O/tc64 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/tc.log 2>&1
ls -la $O
