"""Top source lines of an ncu report by warp-stall samples: python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
tot = 0
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        try:
            smp = int(r[4]); ins = int(r[7])
        except ValueError:
            continue
        rows.append((smp, ins, fname, int(r[0]), r[1].strip()[:90]))
        tot += smp
rows.sort(reverse=True)
print(f"total samples {tot}")
for smp, ins, f, ln, src in rows[:N]:
    print(f"{100.0*smp/max(tot,1):5.1f}% {smp:8d} inst {ins:14d}  {f}:{ln}  {src}")
