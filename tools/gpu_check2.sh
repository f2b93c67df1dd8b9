#!/bin/bash
# correctness + bench pass: smoke, GPU tests, conv sweep, R18/R50 benches
set -x
TAG=${1:-chk}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python tools/conv_fwd_sweep.py > $O/conv_fwd_sweep.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench_r18.json 2> $O/bench_r18.err
timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline > $O/bench_r50.json 2> $O/bench_r50.err
ls -la $O
