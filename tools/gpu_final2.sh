#!/bin/bash
# round evidence: smoke, GPU tests, default bench (with cpu_baseline), R50 bench, launch list, ncu --set full of the top kernel
set -x
TAG=${1:-f3}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_r18.json 2> $O/bench_r18.err
timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline > $O/bench_r50.json 2> $O/bench_r50.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
  --clock-control none -s 6000 -c 700 --csv --log-file $O/launches_r18.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_r18.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"conv_halo_kernel<.int.64" -s 8 -c 2 \
  -o $O/prof_halo python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
ls -la $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"conv_tc_kernel<.int.256" -s 20 -c 2 \
  -o $O/prof_tc256 python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
  --clock-control none -s 31000 -c 1400 --csv --log-file $O/launches_r50.csv \
  python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_r50.log 2>&1
timeout 300 ./tools/micro/run.sh > $O/umma_rate.txt 2>&1
ls -la $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"wgrad_halo_kernel" -s 4 -c 2 \
  -o $O/prof_whalo python bench.py --model revnet50 --stages 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full3.log 2>&1
ls -la $O
