"""Replicate MLE study (Fig. "BoxPlot").

The paper generates one large field Z0 = L~ xi at theta* from an H-Cholesky factor (n0 = 2e6
locations), draws M replicate data sets of n locations by random subsampling of Z0, runs the MLE
on each and shows boxplots of the estimates per n; the spread shrinks as n grows.

Here (R29): the master field is C4's data field (n0 = 524,288 uniform points,
theta* = (nu 0.5, ell 0.1, sigma2 1), tau^2 = 1e-6, Z0 from the eps_gen = 1e-10 uncapped factor;
the same Z the C4 MLE uses); replicate r of size n takes the seeded random subset
rng(6000 + 97 r + n).choice(n0, n, replace=False) of the master points with Z0 restricted to it;
each MLE is the theta-batched Nelder-Mead + grid driver (mle.py, R17: 64 candidates x 20
iterations from x0 = 1.5 theta*) with L~ from hcov_mle_batch at eps = 1e-6, k <= 20.

Results are appended one line per (n, r) to --out (resumable: done pairs are skipped), then
summarised by --summary into boxplot statistics per n.
  python tools/replicates.py --sizes 2000,4000,8000 --reps 10 --budget-s 1500
  python tools/replicates.py --summary gpurun_out/replicates.jsonl > profiles/r2_replicates.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def subset(n0: int, n: int, r: int) -> np.ndarray:
    return np.sort(np.random.default_rng(6000 + 97 * r + n).choice(n0, n, replace=False))


def summary(path: str) -> dict:
    rows = [json.loads(x) for x in open(path) if x.strip()]
    out = {"source": os.path.basename(path), "truth": {"nu": 0.5, "ell": 0.1, "sigma2": 1.0}, "per_n": {}}
    for n in sorted({r["n"] for r in rows}):
        rs = [r for r in rows if r["n"] == n]
        d = {"replicates": len(rs)}
        for k in ("nu", "ell", "sigma2", "microergodic"):
            v = np.array([r["theta_hat"][k] for r in rs])
            q = np.percentile(v, [0, 25, 50, 75, 100])
            d[k] = {"min": q[0], "q1": q[1], "median": q[2], "q3": q[3], "max": q[4], "mean": float(v.mean()),
                    "std": float(v.std(ddof=1)) if len(v) > 1 else 0.0}
        d["seconds_per_mle_mean"] = float(np.mean([r["seconds"] for r in rs]))
        out["per_n"][str(n)] = d
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2000,4000,8000")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/replicates.jsonl")
    ap.add_argument("--seed-out", default="profiles/r2_replicates.jsonl",
                    help="results of earlier calls (copied to --out first when --out does not exist)")
    ap.add_argument("--budget-s", type=float, default=1e9, help="stop starting new replicates after this")
    ap.add_argument("--summary", default="")
    a = ap.parse_args()
    if a.summary:
        print(json.dumps(summary(a.summary), indent=1))
        return

    import shutil
    import torch
    import paper_1709_08625_b200 as H
    from paper_1709_08625_b200 import mle

    t_start = time.time()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    if not os.path.exists(a.out) and os.path.exists(a.seed_out):
        shutil.copy(a.seed_out, a.out)
    done = set()
    if os.path.exists(a.out):
        for x in open(a.out):
            if x.strip():
                r = json.loads(x)
                done.add((r["n"], r["rep"]))
    cfg = synth.CONFIGS["C4"]
    s0 = synth.points(cfg)
    n0 = s0.shape[0]
    dev = torch.device("cuda", 0)
    T0 = H.Tree(torch.from_numpy(s0).to(dev))
    g = H.HMatrix(T0, (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget), synth.EPS_GEN["C4"], 0)
    g.cholesky()
    Z0 = g.sample(torch.from_numpy(synth.xi(n0, cfg.seed_xi)).to(dev)).cpu().numpy()
    del g, T0
    torch.cuda.empty_cache()
    truth = np.array([cfg.nu, cfg.ell, cfg.sigma2])
    for n in [int(x) for x in a.sizes.split(",")]:
        for r in range(a.reps):
            if (n, r) in done:
                continue
            if time.time() - t_start > a.budget_s:
                print(json.dumps({"stopped": "budget", "elapsed_s": time.time() - t_start}), flush=True)
                return
            idx = subset(n0, n, r)
            T = H.Tree(torch.from_numpy(np.ascontiguousarray(s0[idx])).to(dev))
            Z = torch.from_numpy(np.ascontiguousarray(Z0[idx])).to(dev)
            ev = mle.gpu_evaluator(T, Z, cfg.eps[0], cfg.kmax, cfg.nugget)
            t0 = time.time()
            S = mle.run_mle(ev, tuple(1.5 * truth), iters=a.iters)
            dt = time.time() - t0
            nu, ell, s2 = S.X[0]
            rec = {"n": n, "rep": r, "theta_hat": {"nu": nu, "ell": ell, "sigma2": s2,
                                                   "microergodic": s2 / ell ** (2 * nu)},
                   "negloglik": float(S.F[0]), "iters": a.iters, "seconds": dt,
                   "eps": cfg.eps[0], "kmax": cfg.kmax}
            with open(a.out, "a") as fh:
                fh.write(json.dumps(rec) + "\n")
            print(json.dumps(rec), flush=True)
            del T, Z


if __name__ == "__main__":
    main()
