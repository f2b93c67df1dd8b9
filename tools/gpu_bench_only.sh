#!/bin/bash
# R18 + R50 bench lines only (tag in $1)
O=gpurun_out/${1:-bo}; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline > $O/bench_r18.json 2> $O/bench_r18.err
timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline > $O/bench_r50.json 2> $O/bench_r50.err
python tools/benchsum.py $O/bench_r18.json $O/bench_r50.json
