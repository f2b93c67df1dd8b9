#!/bin/bash
# bulk-staged BN passes: channel limit for the apply (A) and dz (D) variants, R50 J=8, two reps
O=gpurun_out/bulkc; mkdir -p $O
for rep in 1 2; do for cfg in "4096 2048" "4096 512" "512 512" "1024 1024"; do set -- $cfg
  PETRA_BN_BULK_MAXC=$1 PETRA_BN_BULK_DZ_MAXC=$2 timeout 600 python bench.py --model revnet50 --stages 8 --no-cpu-baseline --steps 30 > $O/b_A$1_D$2_r$rep.json 2> /dev/null
done; done
for f in $O/b_*.json; do python - $f <<'PY'
import json,sys,os
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k={x["name"]:x["ms_per_step"] for x in d["kernels"]}
print(f'{os.path.basename(sys.argv[1]):26s} {d["value"]:>9} samples/s sm {d["clocks"]["sm_mhz"]} MHz; apply {k.get("bn_apply")} bwd_dz {k.get("bn_bwd_dz")} ms/step')
PY
done
