"""DRAM traffic per logical kernel launch from a multi-metric ncu launch list
(dram__bytes_read.sum + dram__bytes_write.sum, cold cache: ncu flushes caches
before each profiled kernel), grouped into the categories bench.py reports.
A logical launch = one launch of the category's main kernel (a split-K reduction
or phase fill launched with it is added to its bytes).  Writes JSON:
    python tools/traffic.py launches.csv out.json"""
import collections
import csv
import json
import re
import sys

MAIN = {  # category -> (main-kernel regex, helper-kernel regex)
    # third template argument = OUT16 (conv_tc_kernel<BN, STAGES, OUT16, KG, PAIR>, conv_halo_kernel<BN, T, OUT16>)
    "conv_fwd_tc": (r"(conv_tc_kernel|conv_halo_kernel)<\d+, \d+, 1[,>]", r"splitk_out_kernel<1>"),
    "conv_dgrad_tc": (r"(conv_tc_kernel|conv_halo_kernel)<\d+, \d+, 0[,>]", r"splitk_out_kernel<0>|phase_fill"),
    "conv_wgrad_tc": (r"wgrad_tc_kernel|wgrad_halo_kernel", r"splitk_sum4?_kernel"),
    "conv_fwd_stem_tc": (r"stem_fwd_kernel", None),
    "bn_apply": (r"bn_apply(_fixed|_tma)?_kernel", None),
    "bn_bwd_reduce": (r"bn_bwd_reduce(_tma)?_kernel", None),
    "bn_bwd_dz": (r"bn_bwd_dz(_fixed|_tma)?_kernel", None),
    "bn_stats_merge": (r"stats_finalize_kernel", None),
    "sgd_update": (r"sgd_kernel", None),
    "cvt_bf16": (r"f32_to_bf16|image_to_bf16x4", None),
}
S = {'byte': 1, 'B': 1, 'Kbyte': 1e3, 'KB': 1e3, 'Mbyte': 1e6, 'MB': 1e6, 'Gbyte': 1e9, 'GB': 1e9}
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[hdr]
ID, KN, MN, MU, MV = (h.index(x) for x in ('ID', 'Kernel Name', 'Metric Name', 'Metric Unit', 'Metric Value'))
L = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= MV:
        continue
    d = L.setdefault(r[ID], {'n': r[KN], 'b': 0.0})
    if r[MN].startswith('dram__bytes'):
        d['b'] += float(r[MV].replace(',', '')) * S[r[MU]]
out = {}
for cat, (main, helper) in MAIN.items():
    n = sum(1 for d in L.values() if re.search(main, d['n']))
    b = sum(d['b'] for d in L.values() if re.search(main, d['n']) or (helper and re.search(helper, d['n'])))
    if n:
        out[cat] = {"bytes_per_launch": b / n, "launches": n}
json.dump({"source": sys.argv[1], "cache": "cold (ncu --cache-control all)", "categories": out},
          open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
