O=gpurun_out/ab2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
bash tools/ab.sh ab2 "PETRA_FINALIZE_WARPS=8" "PETRA_FINALIZE_WARPS=32" "PETRA_CONV_CS=1 PETRA_CONV_CS_BN=128" "PETRA_CONV_CS=1 PETRA_CONV_CS_BN=64" "PETRA_FINALIZE_WARPS=8" "PETRA_FINALIZE_WARPS=32" "PETRA_CONV_CS=1 PETRA_CONV_CS_BN=128"
