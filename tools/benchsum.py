"""Print the headline numbers and kernel table of bench.py JSON lines."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline", {})
    print(f"{f}: {d.get('value')} {d.get('unit')} ms/step {d.get('ms_per_step')} e2e {d.get('e2e', {}).get('value')} "
          f"roof {r.get('kernel')} {r.get('achieved')} {r.get('unit')} frac {r.get('frac')} launches {d.get('gpu_launches')} clocks {d.get('clocks')}")
    for k in d.get("kernels", [])[:14]:
        print("    ", k)
