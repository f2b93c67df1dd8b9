#!/bin/bash
# R50 profiling pass + smoke + new parity tests
set -x
TAG=${1:-r50}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "accumulation or mlp_config1" > $O/pytest_k.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none --csv --log-file $O/launches_r50.csv \
   python bench.py --model revnet50 --stages 8 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
ls -la $O
