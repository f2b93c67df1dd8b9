O=gpurun_out/gsweep; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/conv_fwd_sweep.py > $O/sweep_graph.txt 2>&1
for cfg in "PETRA_CONV_PAIR=1" "PETRA_CONV_CS=1" "PETRA_CONV_CTAS=148"; do env $cfg timeout 300 python tools/conv_fwd_sweep.py > "$O/sweep_$cfg.txt" 2>&1; done
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "tc_conv" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for f in $O/sweep_*.txt; do echo "== $f"; cut -c1-75 "$f" | head -17; done
