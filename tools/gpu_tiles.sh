#!/bin/bash
# conv N-tile target sweep (PETRA_CONV_TILES) on R18 / R50
O=gpurun_out/tiles; mkdir -p $O
for c in 148 96 48 1; do for m in "revnet18 4" "revnet50 8"; do set -- $m
  PETRA_CONV_TILES=$c timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline --steps 30 > $O/b_$1_t$c.json 2> /dev/null
done; done
for c in 148 96 48 1; do for m in revnet18 revnet50; do python - $O/b_${m}_t$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k={x["name"]:x["ms_per_step"] for x in d["kernels"]}
print(sys.argv[1], d["value"], "fwd", k.get("conv_fwd_tc"), "dgrad", k.get("conv_dgrad_tc"), d["clocks"]["sm_mhz"])
PY
done; done
