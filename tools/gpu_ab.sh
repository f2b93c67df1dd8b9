#!/bin/bash
# A/B of an environment knob: $1 = variable, values 0 / 1, two repetitions, R18 and R50
V=${1:-PETRA_BN_BULK}; O=gpurun_out/ab_$V; mkdir -p $O
for rep in 1 2; do for v in 0 1; do for m in "revnet18 4" "revnet50 8"; do set -- $m
  env $V=$v timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline --steps 30 > $O/b_$1_v${v}_r$rep.json 2> /dev/null
done; done; done
for f in $O/b_*.json; do python - $f <<'PY'
import json,sys,os
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k={x["name"]:x["ms_per_step"] for x in d["kernels"]}
print(f'{os.path.basename(sys.argv[1]):26s} {d["value"]:>9} samples/s sm {d["clocks"]["sm_mhz"]} MHz; apply {k.get("bn_apply")} bwd_dz {k.get("bn_bwd_dz")} bwd_reduce {k.get("bn_bwd_reduce")} ms/step')
PY
done
