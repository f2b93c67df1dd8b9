#!/bin/bash
# A/B of the bf16 inner-activation gradient (PETRA_INNER_DY16) on R50 J=8
O=gpurun_out/dy16ab; mkdir -p $O
for rep in 1 2; do for v in 0 1; do
  PETRA_INNER_DY16=$v timeout 600 python bench.py --model revnet50 --stages 8 --no-cpu-baseline --steps 30 > $O/b_v${v}_r$rep.json 2> /dev/null
done; done
for f in $O/b_*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k={x["name"]:x["ms_per_step"] for x in d["kernels"]}
print(sys.argv[1], d["value"], d["clocks"]["sm_mhz"], "dgrad", k.get("conv_dgrad_tc"), "reduce", k.get("bn_bwd_reduce"), "dz", k.get("bn_bwd_dz"))
PY
done
