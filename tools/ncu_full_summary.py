"""Key metrics of an ncu --set full report (one block per profiled launch):
    python tools/ncu_full_summary.py report.ncu-rep "title" > summary.txt"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__cycles_active.avg", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "sm__memory_throughput.avg.pct_of_peak_sustained_elapsed"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
print(f"ncu --set full --clock-control none ({sys.argv[1]}): {sys.argv[2] if len(sys.argv) > 2 else ''}")
for r in rows[2:]:
    print("---")
    print("  Kernel Name =", r[h.index("Kernel Name")][:110])
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k} = {r[i]} {units[i]}")
    st = sorted(((float(r[i] or 0), n[len(STALLS):]) for i, n in enumerate(h)
                 if n.startswith(STALLS) and not n.endswith("not_issued")), reverse=True)
    tot = sum(v for v, _ in st) or 1.0
    print("  stall samples (top):", ", ".join(f"{n} {v / tot:.0%}" for v, n in st[:6]))
