# R18 J=4 unit partitions, two passes (usage: bash tools/gpu_partitions.sh)
O=gpurun_out/part2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rep in 1 2; do for p in "" 5,4,3,6 4,4,4,6 5,3,4,6 4,4,5,5; do
  timeout 600 python bench.py --no-cpu-baseline --no-north-star ${p:+--partition $p} > $O/r18_${p}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/r18_${p}_$rep.json').read().strip().splitlines()[-1]); print('R18 part', d['config']['partition_units'], round(d['value'],1), d.get('stage_ms_per_tick'))"
done; done
