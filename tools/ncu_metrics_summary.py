"""Summarise an ncu --metrics launch list with several metrics (time, DRAM bytes,
tensor-pipe %): per kernel name -> launches, share of device time, avg us, achieved
DRAM GB/s and mean tensor-pipe utilisation.
    python tools/ncu_metrics_summary.py launches.csv [skip_launches]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[hdr]
ID, KN, MN, MU, MV = (h.index(x) for x in ('ID', 'Kernel Name', 'Metric Name', 'Metric Unit', 'Metric Value'))
TS = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'second': 1e6, 's': 1e6}
BS = {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'B': 1.0, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
launch = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= MV:
        continue
    d = launch.setdefault(r[ID], {'name': r[KN].split('(')[0].replace('void ', '').replace('petra::<unnamed>::', '')})
    v = float(r[MV].replace(',', ''))
    m, u = r[MN], r[MU]
    if m == 'gpu__time_duration.sum':
        d['us'] = v * TS[u]
    elif m.startswith('dram__bytes'):
        d['bytes'] = d.get('bytes', 0.0) + v * BS[u]
    elif 'tensor' in m:
        d['tensor'] = v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, d in enumerate(launch.values()):
    if i < skip or 'us' not in d:
        continue
    a = agg[d['name']]
    a[0] += 1
    a[1] += d['us']
    a[2] += d.get('bytes', 0.0)
    a[3] += d.get('tensor', 0.0) * d['us']
tot = sum(a[1] for a in agg.values())
print(f"total device time {tot / 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches")
print(" share   avg_us  launches   GB/s  tensor%  kernel")
for k, (n, us, b, tw) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us / tot * 100:5.1f}% {us / n:8.2f} {n:8d} {b / us / 1e3 if us else 0:7.0f} {tw / us if us else 0:7.1f}  {k[:80]}")
