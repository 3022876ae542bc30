"""C4 maximum-likelihood estimation on the GPU.

n = 524,288 uniform points, truth theta* = (nu 0.5, ell 0.1, sigma2 1), tau^2 = 1e-6; data
Z = L~ xi from a tight H-Cholesky factor (eps_gen = 1e-10, no rank cap; row 15); the objective is
L~(theta) at eps = 1e-6, k <= 20 through hcov_mle_batch; 64 candidates per iteration (mle.py,
reading R17) for 20 iterations from x0 = 1.5 x truth.

A run can be split over several processes: the simplex is checkpointed after every iteration
(--state; a resumed run is bitwise the same as one run, tests/test_mle_driver.py).  When all
iterations are done the estimate is checked against row 18:
  |nu^ - 0.5| <= 0.05;  ell^, sigma2^ within 25 %;  sigma2^/ell^(2 nu^) within 10 % of 10;
  L~(theta^) >= L~(theta*) - 2.

  python tools/mle_run.py --state gpurun_out/mle_c4_state.json --iters-now 5 [--config C4] [--n N]
Multi-GPU: under torchrun the candidates are sharded round-robin and all-gathered over NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=0, help="use the first n points (debug)")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--iters-now", type=int, default=20, help="iterations to run in this process")
    ap.add_argument("--state", default="gpurun_out/mle_c4_state.json")
    ap.add_argument("--seed-state", default="profiles/r2_mle_c4_state.json",
                    help="checkpoint to start from when --state does not exist yet")
    ap.add_argument("--trace", default="gpurun_out/mle_c4_trace.jsonl")
    ap.add_argument("--out", default="gpurun_out/mle_c4_result.json")
    ap.add_argument("--eps-gen", type=float, default=0.0)
    a = ap.parse_args()

    import torch
    import paper_1709_08625_b200 as H
    from paper_1709_08625_b200 import mle

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS[a.config]
    eps, kmax = cfg.eps[0], cfg.kmax
    s = synth.points(cfg)
    n = a.n or cfg.n
    s = s[:n]
    truth = (cfg.nu, cfg.ell, cfg.sigma2)
    t0 = time.time()
    tree = H.Tree(torch.from_numpy(s).to(dev))
    # data: Z = L~_gen xi at theta*, eps_gen = 1e-10 and no cap (row 15); deterministic, so every
    # process of a split run regenerates bitwise the same Z
    eg = a.eps_gen or synth.EPS_GEN.get(cfg.name, 1e-10)
    g = H.HMatrix(tree, (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget), eg, 0)
    g.cholesky()
    Z = g.sample(torch.from_numpy(synth.xi(n, cfg.seed_xi)).to(dev))
    del g
    t_gen = time.time() - t0
    if a.state and not os.path.exists(a.state) and a.seed_state and os.path.exists(a.seed_state):
        os.makedirs(os.path.dirname(a.state) or ".", exist_ok=True)
        shutil.copy(a.seed_state, a.state)
    os.makedirs(os.path.dirname(a.trace) or ".", exist_ok=True)
    ev = mle.gpu_evaluator(tree, Z, eps, kmax, cfg.nugget)
    n_ev = [0]

    def counted(xs):
        n_ev[0] += len(xs)
        return ev(xs)
    x0 = tuple(1.5 * np.array(truth))
    t1 = time.time()
    S = mle.run_mle(counted, x0, iters=a.iters, rank=rank, world=world, device=dev, trace=a.trace,
                    state=a.state, max_new_iters=a.iters_now)
    t_mle = time.time() - t1
    rec = {"config": cfg.name, "n": n, "eps": eps, "kmax": kmax, "eps_gen": eg, "world": world,
           "iters_done": S.iters_done, "iters": a.iters, "evals_this_call": n_ev[0],
           "mle_s_this_call": t_mle, "gen_s": t_gen,
           "evals_per_s_this_call": n_ev[0] / t_mle if t_mle > 0 else None,
           "best": S.X[0].tolist(), "negloglik_best": float(S.F[0])}
    if S.iters_done >= a.iters:
        nu, ell, s2 = S.X[0]
        L_hat = -float(S.F[0])
        L_true = float(H.eval_loglik(tree, (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget), Z, eps, kmax)["loglik"])
        micro = s2 / ell ** (2 * nu)
        micro_true = cfg.sigma2 / cfg.ell ** (2 * cfg.nu)
        checks = {"nu_abs_err<=0.05": abs(nu - cfg.nu) <= 0.05,
                  "ell_rel_err<=0.25": abs(ell - cfg.ell) <= 0.25 * cfg.ell,
                  "sigma2_rel_err<=0.25": abs(s2 - cfg.sigma2) <= 0.25 * cfg.sigma2,
                  "microergodic_rel_err<=0.10": abs(micro - micro_true) <= 0.10 * micro_true,
                  "L_hat>=L_true-2": L_hat >= L_true - 2.0}
        rec.update({"theta_hat": {"nu": nu, "ell": ell, "sigma2": s2}, "theta_true": dict(zip(("nu", "ell", "sigma2"), truth)),
                    "microergodic_hat": micro, "microergodic_true": micro_true,
                    "L_hat": L_hat, "L_true": L_true, "checks": checks, "all_ok": all(checks.values())})
    if rank == 0:
        print(json.dumps(rec), flush=True)
        with open(a.out, "w") as fh:
            json.dump(rec, fh, indent=1)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
