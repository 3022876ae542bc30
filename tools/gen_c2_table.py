"""Write tests/golden/c2_eps_oracle.json: for each of C2's 64 ell values (R16) the exact
dense oracle L (Eq. (1)) and the eps-oracle L at eps in {1e-4, 1e-8}, computed
ONLY by ``oracle/`` from the seeded inputs of ``synth/`` (no CUDA-path value is involved).

Resumable: rows already present in the output are kept.  Usage:
    python tools/gen_c2_table.py [--out tests/golden/c2_eps_oracle.json] [--only i,j,...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle.eps_oracle import loglik_eps  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c2_eps_oracle.json"))
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS["C2"]
    s = synth.points(cfg)
    Z = oracle.sample_dense(s, synth.xi(cfg.n, cfg.seed_xi), cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    table = {"config": "C2", "n": cfg.n, "nu": cfg.nu, "sigma2": cfg.sigma2, "nugget": cfg.nugget,
             "ell_true": cfg.ell, "eps": list(cfg.eps), "source": "tools/gen_c2_table.py (oracle/ only)",
             "rows": {}}
    if os.path.exists(a.out):
        table = json.load(open(a.out))
    idx = [int(x) for x in a.only.split(",")] if a.only else range(len(cfg.ell_grid))
    for i in idx:
        if str(i) in table["rows"]:
            continue
        ell = cfg.ell_grid[i]
        t0 = time.time()
        r = loglik_eps(s, Z, cfg.sigma2, ell, cfg.nu, cfg.nugget, cfg.eps)
        row = {"ell": ell, "exact": list(r["exact"])}
        for e in cfg.eps:
            row[repr(e)] = r[e] if isinstance(r[e], str) else list(r[e])
            row["info " + repr(e)] = r[("info", e)]
        table["rows"][str(i)] = row
        json.dump(table, open(a.out + ".tmp", "w"), indent=1)
        os.replace(a.out + ".tmp", a.out)
        print(f"[{i}] ell={ell:.5f} exact={r['exact'][0]:.6f} "
              + " ".join(f"eps={e}: {row[repr(e)] if isinstance(row[repr(e)], str) else row[repr(e)][0]}"
                         for e in cfg.eps) + f"  ({time.time() - t0:.0f}s)", flush=True)


if __name__ == "__main__":
    main()
