"""Summaries of ncu outputs for profiles/: a --set full report (key metrics + top source lines) or
a --metrics gpu__time_duration.sum launch list (per-kernel totals and shares).

usage: python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
       python tools/ncu_summary.py launches.csv  > profiles/<name>.txt
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:70s} {r[i]:>20s} {units[i]}")
    print()
    print("top source lines by warp-stall samples:")
    src = subprocess.run([sys.executable, "tools/ncu_lines.py", path, "25"], capture_output=True, text=True).stdout
    print(src)


def launches(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(lines)
    h = next(rd)
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    for r in rd:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}.get(unit, 1.0)
        name = r[ki].split("(")[0]
        tot[name] += v * scale
        cnt[name] += 1
    T = sum(tot.values())
    print(f"total device time of listed launches: {T:.1f} ms over {sum(cnt.values())} launches")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"  {100 * tot[k] / T:6.2f}%  {tot[k]:12.2f} ms  {cnt[k]:6d} launches  {k}")


if __name__ == "__main__":
    p = sys.argv[1]
    report(p) if p.endswith(".ncu-rep") else launches(p)
