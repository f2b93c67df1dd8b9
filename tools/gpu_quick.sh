#!/bin/bash
# GPU tests + R18/R50 bench (tag in $1)
O=gpurun_out/${1:-quick}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_r18.json 2> $O/bench_r18.err
timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline > $O/bench_r50.json 2> $O/bench_r50.err
python tools/benchsum.py $O/bench_r18.json $O/bench_r50.json
