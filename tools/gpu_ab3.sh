bash tools/ab.sh ${1:-ab3} "PETRA_TAIL_PRIO=0" "PETRA_TAIL_PRIO=1" "PETRA_TAIL_PRIO=0" "PETRA_TAIL_PRIO=1" "PETRA_TAIL_PRIO=1 PETRA_STREAM_PRIO=0"
for f in gpurun_out/${1:-ab3}/ab_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('stage_ms_per_tick'), d.get('north_star_r50',{}).get('stage_ms_per_tick'))"; done
