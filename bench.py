#!/usr/bin/env python
"""bench.py — log-likelihood evaluations per second of the H-matrix hot path on B200.

One step = one full evaluation of L~(theta) (Eq. (2)): H-assembly (A3-A6),
H-Cholesky (A7), log det + forward H-solve (A8-A10), i.e. BASELINE.json's metric
"log-likelihood evals/s (H-assemble+H-Cholesky+solve) at n=2M".  The cluster/block tree
(A1-A2) is theta-independent and built once before the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl hcov|reference]

Multi-GPU (torchrun, one rank per GPU): the theta candidates are sharded across ranks (each
rank owns whole factorizations), the per-step likelihood values are
all-gathered over NCCL, timing is the max over ranks; scaling is weak (fixed work per rank).
--impl reference times the CPU oracle (oracle/, dense fp64 Cholesky) on a bounded sample of the
same workload, extrapolated to the metric's n by the dense O(n^3) cost.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "log-likelihood evals/s (H-assemble+H-Cholesky+solve) at n=2M"


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="C5")
    p.add_argument("--theta", default="feasible", choices=["feasible", "config"],
                   help="feasible: C5's n / points / k with C4's kernel and eps = 1e-6 (DESIGN.md R24: C5's "
                        "own theta is not SPD under the method at n >= 65,536); config: the config as written")
    p.add_argument("--impl", default="hcov", choices=["hcov", "reference"])
    p.add_argument("--n", type=int, default=0, help="override n (debug only; not a bench line)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=0, help="oracle sample size (default: auto)")
    p.add_argument("--eps", type=float, default=0.0, help="override eps (0 = the workload's)")
    p.add_argument("--kmax", type=int, default=-1, help="override the rank cap (-1 = the workload's)")
    p.add_argument("--acc-cols", type=int, default=64, help="sampled columns for ||C - C~||_F / ||C||_F")
    p.add_argument("--out", default="", help="also write the JSON line to this file")
    p.add_argument("--factor-trunc", action="store_true",
                   help="SPD-preserving H-Cholesky order (hcov_tree_opts.factor_trunc, DESIGN.md R27)")
    p.add_argument("--kcap", type=int, default=0, help="rank capacity of the low-rank pools (0 = kmax)")
    p.add_argument("--cands-per-rank", type=int, default=1,
                   help="theta candidates per rank and step (> 1: hcov_mle_batch runs them in shared engine "
                        "launches); the batch is the config's theta with ell log-spaced in ell*[0.8, 1.25]")
    return p.parse_args()


# --------------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks line")
# --------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.count(",") >= 8]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, nm in enumerate(names):
                if "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# --------------------------------------------------------------------------------------------
def _theta_for(cfg, j: int, m: int):
    """Candidate j of m: the config's theta for m == 1; else ell log-spaced in ell*[0.8, 1.25]
    (SURVEY.md Sec. 8(d), C5's 8-GPU theta batch)."""
    if m == 1:
        return (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    f = 0.8 * (1.25 / 0.8) ** (j / (m - 1))
    return (cfg.sigma2, cfg.ell * f, cfg.nu, cfg.nugget)


def _oracle_cpu(cfg, n_s: int, th, reps: int = 1):
    """The oracle as it stands (dense Matern fill + LAPACK Cholesky + solve) on the first n_s
    points of the config at theta th, on every host core; returns (seconds per evaluation, threads)."""
    os.environ.setdefault("HCOV_ORACLE_THREADS", str(os.cpu_count() or 1))
    import oracle
    s = synth.points(cfg)[:n_s]
    Z = synth.xi(n_s, cfg.seed_xi)
    oracle.loglik_dense(s[:256], Z[:256], *th)      # build/load the C checker outside the clock
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.loglik_dense(s, Z, *th)
        ts.append(time.perf_counter() - t0)
    return min(ts), oracle.THREADS


def _cpu_sample_size(cfg, th, budget_s: float = 15.0) -> int:
    n_s = 2048
    t, _ = _oracle_cpu(cfg, n_s, th)
    # grow until one evaluation costs ~budget/4 (dense O(n^3))
    while n_s < cfg.n and t * 8 < budget_s / 2 and n_s * 2 <= 32768:
        n_s *= 2
        t, _ = _oracle_cpu(cfg, n_s, th)
    return n_s


def run_reference(args, cfg, rank: int, world: int):
    if rank != 0:
        return
    n = cfg.n
    th, eps, kmax, note, wl = bench_params(args, cfg)
    n_s = args.cpu_sample or _cpu_sample_size(cfg, th, budget_s=8.0)
    for _ in range(args.warmup):
        _oracle_cpu(cfg, min(n_s, 2048), th)
    ts = []
    for _ in range(args.steps):
        t, thr = _oracle_cpu(cfg, n_s, th)
        ts.append(t)
    t_step = float(np.mean(ts))
    t_full = t_step * (n / n_s) ** 3              # dense O(n^3) extrapolation to the metric's n
    v = 1.0 / t_full
    out = {"metric": METRIC, "value": v, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": wl, "n": n, "nu": th[2], "ell": th[1], "sigma2": th[0],
                      "nugget": th[3], "eps": eps, "kmax": kmax, "theta_note": note},
           "cpu_baseline": {"value": v, "unit": "evals/s", "cores": thr, "nproc": os.cpu_count(), "kind": "oracle",
                            "sample": f"dense oracle L(theta) on the first {n_s} of the {n} points, "
                                      f"{t_step:.2f} s/eval, extrapolated x(n/{n_s})^3"},
           "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def bench_params(args, cfg):
    """(theta, eps, kmax, note, workload label) of the benchmarked evaluation (R24)."""
    eps = args.eps if args.eps > 0 else None
    kmax = args.kmax if args.kmax >= 0 else cfg.kmax
    if args.theta == "config" or cfg.name != "C5":
        return ((cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget), eps or cfg.eps[0], kmax,
                "config theta as written" + ("" if eps is None else f" with eps={eps}"), cfg.name)
    c4 = synth.CONFIGS["C4"]
    return ((c4.sigma2, c4.ell, c4.nu, c4.nugget), eps or 1e-6, kmax,
            "C5's points, n and k with C4's kernel (nu=0.5, ell=0.1, sigma2=1, tau2=1e-6) and eps=1e-6: "
            "C5's own theta (nu=1, ell=0.05) is not SPD under the method at eps=1e-5 (DESIGN.md R24)",
            "C5-points/C4-kernel")


def _peaks():
    peaks, fp64 = {}, {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    try:
        fp64 = json.load(open(os.path.join(ROOT, "profiles", "r1_fp64_peak.json")))
    except OSError:
        pass
    return peaks, fp64


def _traffic(workload: str, n: int):
    """ncu dram bytes per launch of k_engine for this workload, from the committed capture summary
    (profiles/r2_engine_traffic.json, written by tools/ncu_traffic.py from an `ncu --set full` run)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r2_engine_traffic.json")))
    except OSError:
        return None, None
    for e in t.get("entries", []):
        if e.get("workload") == workload and int(e.get("n", -1)) == n:
            return float(e["dram_bytes"]), e.get("source")
    return None, None


def run_hcov(args, cfg, rank: int, world: int):
    import torch
    import paper_1709_08625_b200 as H

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    n = args.n or cfg.n
    s = synth.points(cfg)[:n] if args.n else synth.points(cfg)
    th0, eps, kmax, note, wl = bench_params(args, cfg)
    if args.n:
        wl = f"{wl}[n={n}]"
    stream = torch.cuda.current_stream()
    s_dev = torch.from_numpy(s).to(dev)
    tree = H.Tree(s_dev, factor_trunc=args.factor_trunc)   # A1-A2 (device kernels): theta-independent, untimed
    kcap = args.kcap
    if args.factor_trunc:
        wl = f"{wl}[SPD-preserving order, kcap={kcap}]"
    info = tree.info()
    # data: Z = L~_gen xi from a TIGHTER H-Cholesky factor than the one
    # evaluated (eps_gen = 1e-8, same rank cap), so v = L~^{-1} Z is not xi by construction
    # (row 15: 1e-8, "if memory forbids, 1e-7"; the first of these that fits the device is used)
    xi = torch.from_numpy(synth.xi(n, cfg.seed_xi)).to(dev)
    Z, gen, gen_mem = None, None, []
    e_row15 = synth.EPS_GEN.get(cfg.name, 1e-8)
    # tightest first; a pool overflow aborts the engine at once (HCOV_ERR_OUT_OF_MEMORY); the last
    # entry is a different (looser-capped) factor than the evaluated one, so v != xi in every case
    tries = [(min(e_row15, eps), kmax), (min(1e-7, eps), kmax), (min(3e-7, eps), kmax),
             (eps, max(1, kmax - 4) if kmax else 0)]
    for eg, kg in tries:
        try:
            hgen = H.HMatrix(tree, th0, eg, kg, kcap)
            try:
                hgen.cholesky()
                Z = hgen.sample(xi)
                gen = {"eps_gen": eg, "kmax_gen": kg}
            finally:
                gen_mem.append({"eps_gen": eg, "kmax_gen": kg, **hgen.mem_info()})
                del hgen
            break
        except H.HcovError as e:
            if e.code != 4:      # only "out of device memory" moves to the next eps_gen
                raise
    if Z is None:
        raise RuntimeError(f"could not generate Z: {gen_mem}")
    eps_gen = gen
    # theta candidates of one step: m_total = world x cands-per-rank, candidate j on rank j mod world
    # (SURVEY 8(e)); a single candidate is the config's theta
    cpr = max(1, args.cands_per_rank)
    m_total = world * cpr
    all_thetas = [_theta_for(type("T", (), {"sigma2": th0[0], "ell": th0[1], "nu": th0[2], "nugget": th0[3]}), j, m_total)
                  for j in range(m_total)]
    my_thetas = all_thetas[rank::world]
    my_theta = my_thetas[0]

    # accuracy of the evaluated C~ (north_star: ||C - C~||_F / ||C||_F <= 10 eps on sampled columns),
    # both sides on the device: C~ e_j from the assembled H-matrix, C e_j by direct Eq. (3) evaluation
    acc = None
    if args.acc_cols > 0:
        hacc = H.HMatrix(tree, my_theta, eps, kmax, kcap)
        cols = np.random.default_rng(7000 + rank).choice(n, args.acc_cols, replace=False)
        ct = hacc.columns(cols)
        ce = H.cov_columns(tree, my_theta, cols)
        fro = float(torch.linalg.norm(ct - ce) / torch.linalg.norm(ce))
        st_c = hacc.storage()
        del hacc, ct, ce
        acc = {"fro_rel_sampled": fro, "columns": int(args.acc_cols), "bar_10eps": 10 * eps, "ok": fro <= 10 * eps,
               "C_tilde_kB_per_dof": (st_c["dense_bytes"] + st_c["lowrank_bytes"]) / n / 1024.0,
               "C_tilde_max_rank": st_c["max_rank"]}

    def step():
        if cpr == 1:
            r = H.eval_loglik(tree, my_theta, Z, eps, kmax, kcap)
            return r, [r["loglik"]]
        ll, st = H.mle_batch(tree, Z, my_thetas, eps, kmax, kcap)
        if any(int(x) != 0 for x in st):
            raise RuntimeError(f"candidate rejected: {list(st)}")
        return None, list(ll)

    for _ in range(max(3, args.warmup)):
        r, lls = step()
    if cpr > 1:   # the first candidate once more on its own: result fields and the work model below
        r = H.eval_loglik(tree, my_theta, Z, eps, kmax, kcap)
    if r["status"] != 0:
        raise RuntimeError(f"evaluation failed: {r}")
    # ---- timed region -----------------------------------------------------------------------
    clocks = Clocks(dev.index)
    H.prof_control(enable_events=True, reset=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        _, lls = step()
        if dist:   # every rank receives all m_total values (the MLE update input)
            t = torch.tensor(lls, dtype=torch.float64, device=dev)
            g = torch.empty(world * cpr, dtype=torch.float64, device=dev)
            dist.all_gather_into_tensor(g, t)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    prof = H.prof_read()
    H.prof_control(enable_events=False, reset=True)
    clk = clocks.stop()
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = m_total * args.steps / (ms * 1e-3)
    if cpr > 1:
        H.eval_loglik(tree, my_theta, Z, eps, kmax, kcap)   # (outside the clock) the handle of the work model
    last = H.last_eval(tree)
    model = last.model_flops()
    st_l = last.storage()

    # ---- e2e: host Z (pinned) -> device inside the timed region, result back to host -----------
    Zh = Z.cpu().pin_memory()
    Zd = torch.empty_like(Z)
    k_e = max(1, min(args.steps, 2))
    if dist:
        dist.barrier()
    if cpr == 1:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(k_e):
            Zd.copy_(Zh, non_blocking=True)
            H.eval_loglik(tree, my_theta, Zd, eps, kmax, kcap)    # returns host scalars (D2H inside)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
    else:   # e2e of the batch: host Z copied in, the m values read back
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(k_e):
            Zd.copy_(Zh, non_blocking=True)
            H.mle_batch(tree, Zd, my_thetas, eps, kmax, kcap)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
    e2e = {"value": m_total * k_e / (ms_e2e * 1e-3), "unit": "evals/s", "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 3 * 8 if cpr == 1 else 12 * cpr}

    # ---- roofline of the dominant kernel (k_engine, one launch per step) ---------------------
    # achieved = SURVEY Sec. 8(d)'s method-work model at the measured ranks (hcov_model_flops) per
    # launch / the engine's CUDA-event time per launch; peak = measured fp64 FMA rate
    peaks, fp64 = _peaks()
    eng_ms = prof["ms"].get("engine", 0.0) / args.steps
    impl_fl = sum(v for k, v in prof["flop"].items() if k != "assembly_evals") / args.steps
    peak = float(fp64.get("dfma_tflops", 36.85))
    ach = model["total"] / (eng_ms * 1e-3) / 1e12 if eng_ms > 0 else 0.0
    traffic, tsrc = _traffic(wl, n)
    roof = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "traffic": traffic, "traffic_source": tsrc,
            "kernel": "k_engine (persistent DAG engine, 1 launch/step)",
            "model_flop_per_launch": model["total"], "model_breakdown": model,
            "impl_flop_per_launch": impl_fl, "impl_frac": impl_fl / (eng_ms * 1e-3) / 1e12 / peak if eng_ms else 0.0,
            "ms_per_launch": eng_ms,
            # C~ written once, L~ rewritten in place, L~ read by the solve: ~3 x bytes of L~
            "algorithmic_bytes_per_launch": 3.0 * (st_l["dense_bytes"] + st_l["lowrank_bytes"]),
            "peak_source": "profiles/r1_fp64_peak.json: measured DFMA loop on this pool's B200 (fp64 is not in "
                           "MEASURED_PEAKS.json; nominal 148 SM x 64 DFMA x 2 x 1.965 GHz = 37.2 TF/s)"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    out = {"metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": wl, "n": n, "nu": my_theta[2], "ell": my_theta[1], "sigma2": my_theta[0],
                      "nugget": my_theta[3], "eps": eps, "kmax": kmax, "kcap": kcap or kmax,
                      "factor_trunc": bool(args.factor_trunc), "Z_from_factor": eps_gen,
                      "theta_note": note, "config_as_written": {"name": cfg.name, "nu": cfg.nu, "ell": cfg.ell,
                                                                "eps": cfg.eps[0], "kmax": cfg.kmax},
                      "leaf": 32, "eta": 2.0, "parallelism": f"theta-batch dp{world}",
                      "candidates_per_step": m_total, "candidates_per_rank": cpr,
                      "l2": "inputs larger than L2 (H-matrix >> 126 MB)",
                      "tree": {k: info[k] for k in ("depth", "n_dense_tiles", "n_lowrank", "n_tasks", "n_waves")}},
           "loglik": r["loglik"], "logdet": r["logdet"], "quad": r["quad"], "max_rank": r["max_rank"],
           "cap_binds": r["cap_binds"], "acc_loss": r["acc_loss"], "interm_cuts": r["interm_cuts"],
           "min_pivot": r["min_pivot"], "z_generation": gen_mem,
           "memory_bytes": last.mem_info(),
           "accuracy": acc,
           "storage": {"L_tilde_kB_per_dof": (st_l["dense_bytes"] + st_l["lowrank_bytes"]) / n / 1024.0,
                       "C_tilde_kB_per_dof": acc["C_tilde_kB_per_dof"] if acc else None,
                       "paper_table4_C_tilde_kB_per_dof_at_2M": 7.4},
           "gpu_launches": int(prof["launches"] // max(1, args.steps)),
           "e2e": e2e, "roofline": roof, "clocks": clk,
           "stages_ms_per_step": {k: v / args.steps for k, v in prof["ms"].items()},
           "task_busy_cta_ms_per_step": {k: round(v / args.steps, 1) for k, v in prof["task_busy_ms"].items() if v},
           "status": r["status"]}
    if world == 1 and not args.no_cpu_baseline:
        n_s = args.cpu_sample or _cpu_sample_size(cfg, th0)
        t, thr = _oracle_cpu(cfg, n_s, th0)
        t_full = t * (n / n_s) ** 3
        out["cpu_baseline"] = {"value": 1.0 / t_full, "unit": "evals/s", "cores": thr, "nproc": os.cpu_count(),
                               "kind": "oracle",
                               "sample": f"dense oracle L(theta) on the first {n_s} of the {n} points: "
                                         f"{t:.2f} s, extrapolated x(n/{n_s})^3 = {t_full:.3g} s/eval"}
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")
    if dist:
        dist.destroy_process_group()


def _spawn(args) -> int:
    """--gpus N > 1 without torchrun: re-launch this script under torch.distributed.run (one rank per
    GPU, rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = _args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_hcov(args, cfg, rank, world)


if __name__ == "__main__":
    main()
