O=gpurun_out/cs1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_bn_stats_gpu.py -x -q > $O/pytest_k.log 2>&1
tail -3 $O/pytest_k.log
bash tools/ab.sh cs1ab "PETRA_CONV_CS=0" "PETRA_CONV_CS=1" "PETRA_CONV_CS=0" "PETRA_CONV_CS=1"
