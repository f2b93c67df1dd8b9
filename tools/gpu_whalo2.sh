#!/bin/bash
# halo wgrad sweep: pixels per block x CTA cap
O=gpurun_out/whalo2; mkdir -p $O
PETRA_WGRAD_HALO_PB=128 timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "padded" > $O/pad128.log 2>&1 || { tail -30 $O/pad128.log; exit 1; }
for pb in 64 128; do for c in 48 96 148; do for m in "revnet18 4" "revnet50 8"; do set -- $m
  PETRA_WGRAD_HALO_PB=$pb PETRA_WGRAD_HALO_CTAS=$c timeout 600 python bench.py --model $1 --stages $2 --no-cpu-baseline --steps 20 > $O/b_$1_pb${pb}_c$c.json 2> /dev/null
done; done; done
for f in $O/b_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
w=[k for k in d["kernels"] if k["name"]=="conv_wgrad_tc"][0]
print(sys.argv[1], d["value"], "wgrad ms/step", w["ms_per_step"], w["tflops"], d["clocks"]["sm_mhz"])
PY
done
