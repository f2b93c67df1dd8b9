#!/bin/bash
# conv / wgrad grid caps after the 128-register cap (co-residency changed)
O=gpurun_out/ctas2; mkdir -p $O
for c in 96 112 128; do for wc in 48 72; do for m in "revnet18 4" "revnet50 8"; do set -- $m
  PETRA_CONV_CTAS=$c PETRA_WGRAD_CTAS=$wc PETRA_WGRAD_HALO_CTAS=$wc timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline --steps 30 > $O/b_$1_c${c}_w$wc.json 2> /dev/null
done; done; done
for f in $O/b_*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["clocks"]["sm_mhz"])
PY
done
