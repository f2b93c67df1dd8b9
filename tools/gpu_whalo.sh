#!/bin/bash
# halo wgrad: kernel parity first (bounded), then stage parity, then benches on/off
set -x
O=gpurun_out/whalo; mkdir -p $O
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "padded" > $O/pad.log 2>&1 || { tail -30 $O/pad.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for m in "revnet18 4" "revnet50 8"; do set -- $m
  timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline > $O/bench_$1.json 2> $O/bench_$1.err
  PETRA_WGRAD_HALO=0 timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline > $O/bench_$1_off.json 2> $O/bench_$1_off.err
done
python tools/benchsum.py $O/bench_*.json
