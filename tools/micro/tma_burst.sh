#!/bin/bash
# Build and run the TMA burst microbenchmark (tma_burst.cu): do N back-to-back copies overlap?
cd $(dirname $0)
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_burst tma_burst.cu -lcuda || exit 1
for g in 1 148; do
for k in 0 1; do
  for R in 64 128 256; do
    for N in 1 2 4 8; do
      [ $((R * 128 * N)) -gt 200000 ] && continue
      timeout 20 /tmp/tma_burst $k $R $N 0 $g || echo "fail"
    done
  done
done
timeout 20 /tmp/tma_burst 0 128 8 1 $g
timeout 20 /tmp/tma_burst 1 128 8 1 $g
done
