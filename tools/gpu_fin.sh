#!/bin/bash
# in-kernel BN finalize (PETRA_CONV_FINALIZE) and halo-wgrad CTA cap, R18 / R50
O=gpurun_out/fin; mkdir -p $O
for f in 0 1; do for wc in 24 48; do for m in "revnet18 4" "revnet50 8"; do set -- $m
  PETRA_CONV_FINALIZE=$f PETRA_WGRAD_HALO_CTAS=$wc timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline --steps 30 > $O/b_$1_f${f}_w$wc.json 2> /dev/null
done; done; done
for f in $O/b_*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k={x["name"]:x["ms_per_step"] for x in d["kernels"]}
print(sys.argv[1], d["value"], d["clocks"]["sm_mhz"], "merge", k.get("bn_stats_merge"), "wgrad", k.get("conv_wgrad_tc"), "fwd", k.get("conv_fwd_tc"))
PY
done
