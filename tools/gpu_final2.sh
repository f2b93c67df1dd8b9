O=gpurun_out/r2final2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_r18.json 2> $O/bench_r18.err; python tools/benchsum.py $O/bench_r18.json 2>/dev/null | head -1
bash tools/configs.sh r2final2 > $O/configs_summary.txt 2>&1; cat $O/configs_summary.txt
