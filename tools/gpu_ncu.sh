#!/bin/bash
# ncu captures of one kernel of the bench step (run under gpurun, one GPU).
# usage: bash tools/gpu_ncu.sh TAG KERNEL_REGEX [bench.py args...]
#   e.g. bash tools/gpu_ncu.sh r50tc conv_tc_kernel --model revnet50 --stages 8
# writes gpurun_out/TAG/{launches.csv,full.ncu-rep,*.log}
TAG=${1:?tag}; K=${2:?kernel regex}; shift 2
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 20 -c 3 \
  -o $O/full python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/full.log 2>&1
ls -la $O
