#!/bin/bash
# Quick GPU pass: build, GPU tests, one bench (R18 + the R50 sub-record), optional extra command.
# usage: bash tools/gpu_quick.sh TAG [extra shell command]
TAG=${1:?tag}; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
if [ $# -gt 0 ]; then bash -c "$*" > $O/extra.log 2>&1; fi
tail -3 $O/pytest_gpu.log
