#!/bin/bash
# GPU tests + R50 bench + one-tick ncu launch list (time, DRAM bytes, tensor %) of R50 J=8
set -x
TAG=${1:-p}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench_r18.json 2> $O/bench_r18.err
timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline > $O/bench_r50.json 2> $O/bench_r50.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
  --clock-control none -s 31000 -c 1400 --csv --log-file $O/launches_r50.csv \
  python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_r50.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
  --clock-control none -s 6000 -c 700 --csv --log-file $O/launches_r18.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_r18.log 2>&1
ls -la $O
