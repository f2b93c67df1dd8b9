#!/bin/bash
# tests + bench sweep over tuning knobs (R18 J=4, R50 J=8)
set -x
TAG=${1:-k}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
for cfg in "base:" "split1:PETRA_SPLITK_MAX=1" "split4:PETRA_SPLITK_MAX=4" "wg74:PETRA_WGRAD_CTAS=74" "wg296:PETRA_WGRAD_CTAS=296" "split1wg74:PETRA_SPLITK_MAX=1 PETRA_WGRAD_CTAS=74"; do
  n=${cfg%%:*}; e=${cfg#*:}
  env $e timeout 600 python bench.py --no-cpu-baseline --steps 20 > $O/r18_$n.json 2>/dev/null
  env $e timeout 900 python bench.py --model revnet50 --stages 8 --no-cpu-baseline --steps 20 > $O/r50_$n.json 2>/dev/null
done
ls -la $O
