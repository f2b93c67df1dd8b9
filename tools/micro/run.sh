#!/bin/bash
# Build (sm_100a) and run the tcgen05 MMA-issue-rate microbenchmark ("MMA issue").
# usage (on a B200, e.g. under gpurun): bash tools/micro/run.sh
set -e
cd $(dirname $0)
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/umma_rate umma_rate.cu -lcuda
for cfg in "64 0 1" "64 1 1" "64 2 1" "64 2 2" "64 2 4" "64 2 1 3" "128 2 1" "128 2 2" "256 2 1" "256 2 2"; do
  timeout 20 /tmp/umma_rate $cfg || echo "cfg $cfg: timeout/fail"
done
