#!/bin/bash
# partition sweep (R18 J=4, R50 J=8) on 1 GPU
set -x
O=gpurun_out/part; mkdir -p $O
for p in "" 5,4,5,4 5,5,4,4 4,5,5,4 6,4,4,4 5,5,5,3; do
  timeout 600 python bench.py --no-cpu-baseline --steps 20 ${p:+--partition $p} > $O/r18_${p:-flop}.json 2>/dev/null
done
for p in "" 2,2,2,2,2,3,3,2 2,2,2,2,3,3,2,2 3,2,2,2,2,2,3,2 2,3,2,2,2,3,2,2; do
  timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline --steps 20 ${p:+--partition $p} > $O/r50_${p:-flop}.json 2>/dev/null
done
ls $O
