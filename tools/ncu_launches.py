"""Per-launch rows of a multi-metric ncu launch list for kernels matching a prefix:
time us, DRAM MB read/written, GB/s, tensor %, grid; grouped by identical shape.
    python tools/ncu_launches.py launches.csv <kernel prefix> [skip]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[hdr]
ID, KN, MN, MU, MV = (h.index(x) for x in ('ID', 'Kernel Name', 'Metric Name', 'Metric Unit', 'Metric Value'))
S = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3, 'byte': 1e-6, 'B': 1e-6,
     'Kbyte': 1e-3, 'KB': 1e-3, 'Mbyte': 1, 'MB': 1, 'Gbyte': 1e3, 'GB': 1e3, '%': 1, '': 1}
L = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= MV:
        continue
    d = L.setdefault(r[ID], {'n': r[KN].split('(')[0].replace('void ', '').replace('petra::<unnamed>::', '')})
    d[r[MN]] = float(r[MV].replace(',', '')) * S.get(r[MU], 1)
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g = collections.defaultdict(list)
for i, d in enumerate(L.values()):
    if i < skip or not d['n'].startswith(sys.argv[2]):
        continue
    key = (d['n'][:40], int(d.get('launch__grid_size', 0)), round(d.get('dram__bytes_read.sum', 0), 1),
           round(d.get('dram__bytes_write.sum', 0), 1))
    g[key].append((d['gpu__time_duration.sum'], d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0)))
print("count  avg_us  MB_rd  MB_wr   GB/s  tensor%  grid  kernel")
for k, v in sorted(g.items(), key=lambda x: -sum(t for t, _ in x[1])):
    us = sum(t for t, _ in v) / len(v)
    ten = sum(t for _, t in v) / len(v)
    print(f"{len(v):5d} {us:7.1f} {k[2]:6.1f} {k[3]:6.1f} {(k[2] + k[3]) / us * 1e3:6.0f} {ten:7.1f} {k[1]:5d}  {k[0]}")
