# conv / wgrad grid caps at low stage counts (R50 J=1, J=2; R18 J=4 reference)
O=gpurun_out/jcap; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for J in 1 2; do for c in "40 32" "64 40" "96 48" "148 48"; do set -- $c
  PETRA_CONV_CTAS=$1 PETRA_WGRAD_CTAS=$2 PETRA_WGRAD_HALO_CTAS=$2 timeout 600 python bench.py --model revnet50 --stages $J --no-cpu-baseline > $O/r50_j${J}_$1.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/r50_j${J}_$1.json').read().strip().splitlines()[-1]); print('R50 J=$J conv $1 wgrad $2', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
