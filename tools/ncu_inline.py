"""Per-SASS-instruction metric of an ncu report mapped to its CUDA source line WITH the inline call
chain (nvdisasm --print-line-info-inline of the built library), aggregated per call chain.
usage: python tools/ncu_inline.py report.ncu-rep lib.so kernel_substring [metric] [N]
metric: 'Warp Stall Sampling (All Samples)' (default) or e.g. 'L2 Theoretical Sectors Local'."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
metric = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
N = int(sys.argv[5]) if len(sys.argv) > 5 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
im, ia = h.index(metric), h.index("Address")
addrs = [int(r[ia], 16) for r in rows[2:] if len(r) > ia and r[ia].startswith("0x")]
base = min(addrs)
vals = []
for r in rows[2:]:
    try:
        v = float(r[im] or 0)
    except (ValueError, IndexError):
        continue
    if v > 0:
        vals.append((v, int(r[ia], 16) - base))
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.startswith("hcov.") and f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "--print-line-info-inline", os.path.join(d, cub)], capture_output=True,
                      text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if kname in l and ".text." in l and "section" in l)
end = next(i for i in range(start + 1, len(sass)) if sass[i].strip().startswith(".section"))
amap, cur, last = {}, [], []
for l in sass[start:end]:
    s = l.strip()
    if s.startswith("//##"):
        cur.append(s)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        if cur:
            last = cur
        amap[int(m.group(1), 16)] = last
        cur = []


def chain(info):
    parts = []
    for x in info[:1]:
        for seg in re.findall(r'"[^"]*/([^"/]+)", line (\d+)', x):
            parts.append(f"{seg[0]}:{seg[1]}")
    return " <- ".join(parts)


agg = collections.Counter()
for v, a in vals:
    agg[chain(amap.get(a, []))] += v
tot = sum(agg.values())
print(f"{metric}: total {tot:.0f}")
for k, v in agg.most_common(N):
    print(f"{100 * v / tot:5.1f}%  {k}")
