#!/bin/bash
# bulk-staged BN apply: chunk bytes x blocks per SM
O=gpurun_out/bulksw; mkdir -p $O
for ch in 12288 24576 49152; do for b in 2 4 8; do for m in "revnet18 4" "revnet50 8"; do set -- $m
  PETRA_BN_BULK_CHUNK=$ch PETRA_BN_BULK_BPS=$b timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline --steps 30 > $O/b_$1_c${ch}_b$b.json 2> /dev/null
done; done; done
for f in $O/b_*.json; do python - $f <<'PY'
import json,sys,os
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k={x["name"]:x["ms_per_step"] for x in d["kernels"]}
print(f'{os.path.basename(sys.argv[1]):28s} {d["value"]:>9} samples/s sm {d["clocks"]["sm_mhz"]} MHz; apply {k.get("bn_apply")} ms/step')
PY
done
