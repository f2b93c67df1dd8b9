O=gpurun_out/pair2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "tc_conv_vs_simt" > $O/pytest_k.log 2>&1
echo "kernels rc=$?"; tail -5 $O/pytest_k.log
timeout 300 python -m pytest tests/test_bn_stats_gpu.py -x -q > $O/pytest_s.log 2>&1
echo "stats rc=$?"; tail -3 $O/pytest_s.log
for cfg in "PETRA_CONV_PAIR=0" "PETRA_CONV_PAIR=1"; do env $cfg timeout 300 python tools/conv_fwd_sweep.py > $O/sweep_$cfg.txt 2>&1; done
paste -d"\n" "$O/sweep_PETRA_CONV_PAIR=0.txt" "$O/sweep_PETRA_CONV_PAIR=1.txt" | head -34
