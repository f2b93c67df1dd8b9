#!/bin/bash
# One gpurun pass: GPU tests, benches, launch list, ncu full capture of the top kernel.
# usage: bash tools/gpu_round.sh [tag]
set -x
TAG=${1:-run}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_r18.json 2> $O/bench_r18.err
PETRA_HALO=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_r18_halo.json 2> $O/bench_r18_halo.err
timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline > $O/bench_r50.json 2> $O/bench_r50.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r18.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 200 -c 3 \
   -o $O/prof_conv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
ls -la $O
