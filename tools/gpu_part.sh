# partitions under PETRA_TAIL_PRIO=1 (R18 J=4); then R50 J=8 partitions
O=gpurun_out/${1:-part1}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for p in "" 5,4,3,6 5,3,4,6 4,4,4,6 5,4,5,4 6,4,4,4; do
  PETRA_TAIL_PRIO=1 timeout 600 python bench.py --no-cpu-baseline --no-north-star ${p:+--partition $p} > $O/r18_$p.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/r18_$p.json').read().strip().splitlines()[-1]); print('R18 part', d['config']['partition_units'], round(d['value'],1), d.get('stage_ms_per_tick'))"
done
for p in "" 2,2,2,2,2,3,3,2 2,2,2,2,3,3,2,2 2,2,2,3,2,2,2,3; do
  PETRA_TAIL_PRIO=1 timeout 600 python bench.py --no-cpu-baseline --model revnet50 --stages 8 ${p:+--partition $p} > $O/r50_$p.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/r50_$p.json').read().strip().splitlines()[-1]); print('R50 part', d['config']['partition_units'], round(d['value'],1), d['clocks']['sm_mhz'], d.get('stage_ms_per_tick'))"
done
