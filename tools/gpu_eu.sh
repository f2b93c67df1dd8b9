O=gpurun_out/eu1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
bash tools/ab.sh eu1ab "PETRA_EARLY_UPDATE=0" "PETRA_EARLY_UPDATE=1" "PETRA_EARLY_UPDATE=0" "PETRA_EARLY_UPDATE=1"
