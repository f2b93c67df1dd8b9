#!/bin/bash
# halo eligibility sweep: minimum work items x maximum zero-border overhead
O=gpurun_out/hsw; mkdir -p $O
for mw in 111 48 1; do for pad in 135 170 230; do for m in "revnet18 4" "revnet50 8"; do set -- $m
  PETRA_HALO_MIN_WORK=$mw PETRA_HALO_MAX_PAD=$pad timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline --steps 30 > $O/b_$1_w${mw}_p$pad.json 2> $O/b_$1_w${mw}_p$pad.err
done; done; done
for f in $O/b_*.json; do python - $f <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
  print(sys.argv[1], "FAILED"); sys.exit()
k={x["name"]:x["ms_per_step"] for x in d["kernels"]}
print(sys.argv[1], d["value"], "fwd", k.get("conv_fwd_tc"), "dgrad", k.get("conv_dgrad_tc"), "wgrad", k.get("conv_wgrad_tc"), d["clocks"]["sm_mhz"])
PY
done
