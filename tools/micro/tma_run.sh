#!/bin/bash
# Build and run the TMA fill-rate microbenchmark (tma_rate.cu) over copy shapes and ring depths.
cd $(dirname $0)
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_rate tma_rate.cu -lcuda || exit 1
for cfg in "0 64 6" "0 128 6" "0 256 3" "0 128 12" "1 64 6" "1 128 6" "1 256 4" "1 128 12" "2 128 6" "2 128 12" \
           "3 256 4" "3 512 3" "0 128 6 96" "1 128 6 96" "0 128 6 32" "1 128 6 32" "0 128 6 1" "1 128 6 1" "2 128 6 1"; do
  timeout 20 /tmp/tma_rate $cfg || echo "cfg $cfg: timeout/fail"
done
