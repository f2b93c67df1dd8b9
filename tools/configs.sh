#!/bin/bash
# The other BASELINE.json configs on one B200 (bench lines, no CPU baseline):
#   configs[2] RevNet-34 / ImageNet32 shape, batch 256, J = 8
#   configs[4] RevNet-50 / ImageNet shape, batch 64, stage-count sweep J = 1, 2, 4, 8, 16
#   plus RevNet-18 J = 8.
# usage: bash tools/configs.sh TAG
TAG=${1:?tag}; O=gpurun_out/$TAG/configs; mkdir -p $O
timeout 900 python bench.py --model revnet34 --batch 256 --stages 8 --no-cpu-baseline --no-north-star > $O/r34_b256_j8.json 2> $O/r34.err
timeout 900 python bench.py --model revnet18 --stages 8 --no-cpu-baseline --no-north-star > $O/r18_j8.json 2> $O/r18_j8.err
for J in 1 2 4 8 16; do
  timeout 900 python bench.py --model revnet50 --stages $J --no-cpu-baseline > $O/r50_j$J.json 2> $O/r50_j$J.err
done
python - $O <<'PY'
import glob, json, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{os.path.basename(f):18s} {d['value']:10.1f} samples/s  {d['ms_per_step']:8.3f} ms/step  "
              f"{d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']}  partition {d['config']['partition_units']}")
    except Exception as e:
        print(os.path.basename(f), "FAILED", e)
PY
