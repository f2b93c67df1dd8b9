#!/bin/bash
# A/B of environment knobs on the default bench (R18 J=4 + the R50 J=8 sub-record), one B200.
# usage: bash tools/ab.sh TAG "ENV1=a ENV2=b" "ENV1=c" ...   (each argument: one configuration)
TAG=${1:?tag}; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $cfg timeout 600 python bench.py --no-cpu-baseline > $O/ab_$i.json 2> $O/ab_$i.err
  python - "$O/ab_$i.json" "$cfg" >> $O/ab_summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    n = d.get("north_star_r50", {})
    print(f"{sys.argv[2]:45s} R18 {d['value']:9.1f} ({d['clocks']['sm_mhz']} MHz)  R50 {n.get('value', 0):8.1f} "
          f"({n.get('clocks', {}).get('sm_mhz')} MHz {n.get('clocks', {}).get('reasons')})  conv_fwd serial "
          f"{d['kernels'][0]['ms_per_step'] if d['kernels'][0]['name']=='conv_fwd_tc' else '-'}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
cat $O/ab_summary.txt
