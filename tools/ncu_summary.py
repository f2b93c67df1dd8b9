"""Summarise an ncu --metrics gpu__time_duration.sum launch list: share, avg, count per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[hdr]; data = rows[hdr + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
mi = h.index('Metric Name')
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'second': 1e6, 's': 1e6}
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # drop the first N launches (setup)
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data[skip:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':  # other metrics of a multi-metric list
        continue
    name = r[ki].split('(')[0].replace('void ', '')
    name = name.replace('petra::<unnamed>::', '')
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', '')) * scale[r[ui]]
tot = sum(v for _, v in agg.values())
print(f"total device time {tot/1e3:.3f} ms over {sum(n for n, _ in agg.values())} launches")
print("share   avg_us   launches  kernel")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v/tot*100:5.1f}% {v/n:9.2f} {n:7d}  {k[:90]}")
