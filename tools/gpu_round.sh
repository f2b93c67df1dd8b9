#!/bin/bash
# One evidence pass on a B200 (under gpurun): build + smoke, the GPU tests, the default bench
# (R18 J=4 + the R50 J=8 sub-record) and the reference arm, the R50 bench line, the R18 ncu
# launch list (durations, grids, DRAM bytes) and ncu --set full captures of the conv kernels.
# usage: bash tools/gpu_round.sh [tag]
set -x
TAG=${1:-run}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench_r18.json 2> $O/bench_r18.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline > $O/bench_r50.json 2> $O/bench_r50.err
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file $O/launches_r18.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-north-star > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_halo_kernel -s 100 -c 2 \
   -o $O/prof_halo python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > $O/ncu_full_halo.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 200 -c 2 \
   -o $O/prof_conv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > $O/ncu_full_conv.log 2>&1
ls -la $O
