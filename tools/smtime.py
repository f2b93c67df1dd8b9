"""Per-kernel device time and SM-time share of an ncu launch list with launch__grid_size
(tools/gpu_ncu.sh-style capture; serialised, cold cache).  SM-time of a launch is
approximated as duration x min(1, grid / 148): a grid of at most one wave holds that many
SMs for its duration; larger grids are taken to fill the GPU.  Under the tick's stream
concurrency, SM-time -- not serial time -- is what the stages compete for.
    python tools/smtime.py launches.csv [skip_launches]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[hdr]
ID, KN, MN, MU, MV = (h.index(x) for x in ('ID', 'Kernel Name', 'Metric Name', 'Metric Unit', 'Metric Value'))
S = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}
L = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= MV:
        continue
    d = L.setdefault(r[ID], {'n': r[KN].split('(')[0].replace('void ', '').replace('petra::<unnamed>::', '')})
    v = float(r[MV].replace(',', ''))
    if r[MN] == 'gpu__time_duration.sum':
        d['us'] = v * S.get(r[MU], 1)
    elif r[MN] == 'launch__grid_size':
        d['grid'] = v
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, d in enumerate(L.values()):
    if i < skip or 'us' not in d:
        continue
    a = agg[d['n']]
    a[0] += 1
    a[1] += d['us']
    a[2] += d['us'] * min(1.0, d.get('grid', 148) / 148.0)
tot_t = sum(a[1] for a in agg.values())
tot_s = sum(a[2] for a in agg.values())
print(f"serial {tot_t / 1e3:.3f} ms, SM-time {tot_s / 1e3:.3f} full-GPU ms over {sum(a[0] for a in agg.values())} launches")
print(f"{'SM-time':>8} {'serial':>7} {'launches':>8}  kernel")
for n, a in sorted(agg.items(), key=lambda kv: -kv[1][2])[:30]:
    print(f"{100 * a[2] / tot_s:7.1f}% {100 * a[1] / tot_t:6.1f}% {a[0]:8d}  {n[:90]}")
