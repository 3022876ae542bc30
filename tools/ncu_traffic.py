"""Record k_engine's DRAM traffic per launch from an `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_engine --csv` log into
profiles/r2_engine_traffic.json (read by bench.py for roofline.traffic).

usage: python tools/ncu_traffic.py <ncu.csv> <workload label> <n> [profiles/r2_engine_traffic.json]
"""
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def parse(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[h]
    kn, mn, mu, mv = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    out = {}
    for r in rows[h + 1:]:
        if len(r) <= mv or "k_engine" not in r[kn]:
            continue
        out[r[mn]] = float(r[mv].replace(",", "")) * SCALE.get(r[mu], 1.0)
    return out


def main():
    path, wl, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
    dst = sys.argv[4] if len(sys.argv) > 4 else "profiles/r2_engine_traffic.json"
    m = parse(path)
    e = {"workload": wl, "n": n, "dram_bytes": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
         "dram_read": m["dram__bytes_read.sum"], "dram_write": m["dram__bytes_write.sum"],
         "duration_s_under_ncu": m.get("gpu__time_duration.sum"), "source": os.path.basename(path)}
    db = {"entries": []}
    if os.path.exists(dst):
        db = json.load(open(dst))
    db["entries"] = [x for x in db["entries"] if not (x["workload"] == wl and int(x["n"]) == n)] + [e]
    json.dump(db, open(dst, "w"), indent=1)
    print(json.dumps(e))


if __name__ == "__main__":
    main()
