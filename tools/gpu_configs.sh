#!/bin/bash
# BASELINE configs on one GPU: R34 / ImageNet32 b256 J=8, and the R50 stage-count sweep J = 1..16
set -x
O=gpurun_out/cfg; mkdir -p $O
timeout 900 python bench.py --model revnet34 --batch 256 --stages 8 --no-cpu-baseline --steps 20 > $O/r34_b256_j8.json 2> $O/r34.err
for J in 1 2 4 8 16; do
  timeout 900 python bench.py --model revnet50 --stages $J --no-cpu-baseline --steps 10 > $O/r50_j$J.json 2> $O/r50_j$J.err
done
timeout 900 python bench.py --model revnet18 --stages 8 --no-cpu-baseline --steps 20 > $O/r18_j8.json 2> $O/r18_j8.err
ls -la $O
