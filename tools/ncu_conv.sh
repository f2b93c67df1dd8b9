#!/bin/bash
# ncu --set full capture of ONE convolution pass (tools/conv_one.py) under gpurun.
# usage: bash tools/ncu_conv.sh TAG KERNEL_REGEX mode engine B H W Ci Co k s [flags]
TAG=${1:?tag}; K=${2:?kernel regex}; shift 2
O=gpurun_out/$TAG; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
  -o $O/full python tools/conv_one.py "$@" > $O/ncu.log 2>&1
ls -la $O
