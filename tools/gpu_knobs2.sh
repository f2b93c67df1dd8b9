#!/bin/bash
# tests + bench sweep over grid-size knobs (R18 J=4, R50 J=8)
set -x
TAG=${1:-k}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
for cfg in "base:" "c112:PETRA_CONV_CTAS=112" "c96:PETRA_CONV_CTAS=96" "c74:PETRA_CONV_CTAS=74" "wg48:PETRA_WGRAD_CTAS=48" "wg37:PETRA_WGRAD_CTAS=37" "c96wg48:PETRA_CONV_CTAS=96 PETRA_WGRAD_CTAS=48"; do
  n=${cfg%%:*}; e=${cfg#*:}
  env $e timeout 600 python bench.py --no-cpu-baseline --steps 20 > $O/r18_$n.json 2>/dev/null
  env $e timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline --steps 20 > $O/r50_$n.json 2>/dev/null
done
ls -la $O
