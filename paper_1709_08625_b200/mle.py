"""theta-batched maximum-likelihood driver (reading R17).

The paper maximises L~ with GSL's Nelder-Mead simplex over x = (nu, ell, sigma^2) from steps
(0.02, 0.04, 0.01) (listing).  On B200s each iteration evaluates a *batch* of 64
candidates instead of one or two points:

  * the 7 speculative Nelder-Mead points of the current simplex (reflection, expansion, outside and
    inside contraction, 3 shrink points), and
  * 57 grid points around the best vertex (3x3x3 - 1 offsets at +-h and at +-h/3, h = per-axis
    spread of the simplex; 5 points on the best-minus-centroid line at alpha in {-1, -1/2, 1/2,
    3/2, 2}).

The Nelder-Mead step is then resolved exactly as the sequential algorithm would (coefficients
1, 2, 1/2, 1/2) from the speculative values, and the best grid point replaces the worst vertex if
it beats the best one.  Candidates are sharded round-robin over the ranks (candidate j -> rank
j mod world); each rank owns whole factorizations (no collective inside an evaluation); the 64
values are all-gathered (NCCL over NVLink on GPUs, gloo in the CPU tests) and every rank applies
the identical deterministic update.  Outside the box nu in [0.05, 5], ell in [1e-3, 10],
sigma^2 in [1e-3, 1e3] the objective is +inf (not evaluated).

`evaluate(thetas) -> loglik` is the per-rank evaluator: `hcov_mle_batch` on the GPU
(`gpu_evaluator`), any function in tests.  Rejected candidates (not SPD) come back as -inf.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

LO = np.array([0.05, 1e-3, 1e-3])
HI = np.array([5.0, 10.0, 1e3])
ALPHAS = (-1.0, -0.5, 0.5, 1.5, 2.0)


def in_box(x: np.ndarray) -> bool:
    return bool(np.all(x >= LO) and np.all(x <= HI))


def grid_offsets() -> np.ndarray:
    o = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1) if (a, b, c) != (0, 0, 0)]
    o = np.array(o, dtype=np.float64)
    return np.concatenate([o, o / 3.0])   # 52 x 3


@dataclass
class Simplex:
    X: np.ndarray          # 4 x 3 vertices (nu, ell, sigma2)
    F: np.ndarray          # 4 objective values (-L)
    history: List[dict] = field(default_factory=list)

    def order(self):
        idx = np.lexsort((np.arange(len(self.F)), self.F))   # ascending F, ties -> lower index
        self.X, self.F = self.X[idx], self.F[idx]


def candidates(S: Simplex) -> np.ndarray:
    """The 64 candidates of one iteration (rows: nu, ell, sigma2)."""
    S.order()
    xb, xw = S.X[0], S.X[-1]
    c = S.X[:-1].mean(axis=0)
    r = c + (c - xw)
    e = c + 2.0 * (c - xw)
    oc = c + 0.5 * (r - c)
    ic = c - 0.5 * (c - xw)
    shrink = [xb + 0.5 * (S.X[i] - xb) for i in (1, 2, 3)]
    h = S.X.max(axis=0) - S.X.min(axis=0)
    grid = xb + grid_offsets() * h
    line = [xb + a * (xb - c) for a in ALPHAS]
    return np.vstack([r, e, oc, ic] + shrink + [grid] + line)   # 4 + 3 + 52 + 5 = 64


def resolve(S: Simplex, C: np.ndarray, f: np.ndarray) -> None:
    """Apply one sequential Nelder-Mead step from the speculative values, then the grid step."""
    S.order()
    fr, fe, foc, fic = f[0], f[1], f[2], f[3]
    n = len(S.F) - 1
    shrink = False
    if fr < S.F[0]:
        S.X[-1], S.F[-1] = (C[1], fe) if fe < fr else (C[0], fr)
    elif fr < S.F[n - 1]:
        S.X[-1], S.F[-1] = C[0], fr
    elif fr < S.F[-1]:
        if foc <= fr:
            S.X[-1], S.F[-1] = C[2], foc
        else:
            shrink = True
    else:
        if fic < S.F[-1]:
            S.X[-1], S.F[-1] = C[3], fic
        else:
            shrink = True
    if shrink:
        for k, i in enumerate((1, 2, 3)):
            S.X[i], S.F[i] = C[4 + k], f[4 + k]
    S.order()
    g = 7 + int(np.lexsort((np.arange(57), f[7:]))[0])
    if f[g] < S.F[0]:
        S.X[-1], S.F[-1] = C[g], f[g]
        S.order()


def shard(m: int, rank: int, world: int) -> List[int]:
    return list(range(rank, m, world))


def evaluate_all(C: np.ndarray, evaluate: Callable[[Sequence[Sequence[float]]], Sequence[float]],
                 rank: int = 0, world: int = 1, group=None, device=None) -> np.ndarray:
    """-L for every candidate: own shard evaluated locally, all-gathered across ranks."""
    import torch
    m = C.shape[0]
    mine = shard(m, rank, world)
    f = np.full(m, np.inf)
    todo = [j for j in mine if in_box(C[j])]
    if todo:
        ll = np.asarray(evaluate([tuple(C[j]) for j in todo]), dtype=np.float64)
        for j, v in zip(todo, ll):
            f[j] = -v if np.isfinite(v) else np.inf
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor(f, dtype=torch.float64, device=device)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        g = torch.stack(parts).cpu().numpy()           # world x m; rank r owns j = r mod world
        f = np.array([g[j % world, j] for j in range(m)])
    return f


def _save_state(path: str, S: Simplex, it_done: int) -> None:
    # exact round trip: float.hex of every vertex coordinate and value
    st = {"iters_done": it_done, "X": [[float(v).hex() for v in row] for row in S.X],
          "F": [float(v).hex() for v in S.F], "history": S.history}
    tmp = path + ".tmp"
    with open(tmp, "w") as fh:
        json.dump(st, fh)
    import os
    os.replace(tmp, path)


def _load_state(path: str):
    with open(path) as fh:
        st = json.load(fh)
    X = np.array([[float.fromhex(v) for v in row] for row in st["X"]])
    F = np.array([float.fromhex(v) for v in st["F"]])
    return Simplex(X, F, list(st["history"])), int(st["iters_done"])


def run_mle(evaluate, x0: Sequence[float], iters: int = 20, rank: int = 0, world: int = 1, group=None,
            device=None, trace: Optional[str] = None, state: Optional[str] = None,
            max_new_iters: Optional[int] = None) -> Simplex:
    """theta-batched Nelder-Mead + grid MLE from x0 = (nu, ell, sigma2); steps 20% of x0 (R17).

    state: checkpoint file (rank 0 writes it after every iteration; every rank reads it on entry),
    so a long MLE can run over several processes; a resumed run is bitwise the same as one run.
    max_new_iters: stop after this many iterations in this call (the checkpoint holds the rest)."""
    import os
    x0 = np.asarray(x0, dtype=np.float64)
    if state and os.path.exists(state):
        S, it0 = _load_state(state)
    else:
        X = np.vstack([x0] + [x0 + np.eye(3)[k] * 0.2 * x0[k] for k in range(3)])
        F = evaluate_all(X, evaluate, rank, world, group, device)
        S, it0 = Simplex(X, F), 0
        if state and rank == 0:
            _save_state(state, S, 0)
    stop = iters if max_new_iters is None else min(iters, it0 + max_new_iters)
    for it in range(it0, stop):
        C = candidates(S)
        f = evaluate_all(C, evaluate, rank, world, group, device)
        resolve(S, C, f)
        rec = {"iter": it, "best": S.X[0].tolist(), "negloglik": float(S.F[0]),
               "size": float(np.max(S.X.max(0) - S.X.min(0))),
               "rejected": int(np.sum(~np.isfinite(f)))}
        S.history.append(rec)
        if trace and rank == 0:
            with open(trace, "a") as fh:
                fh.write(json.dumps(rec) + "\n")
        if state and rank == 0:
            _save_state(state, S, it + 1)
    S.iters_done = stop
    return S


def gpu_evaluator(tree, Z, eps: float, kmax: int, nugget: float):
    """hcov_mle_batch on the current device: x = (nu, ell, sigma2) -> L~."""
    from . import mle_batch

    def ev(xs):
        thetas = [(x[2], x[1], x[0], nugget) for x in xs]
        ll, _ = mle_batch(tree, Z, thetas, eps, kmax)
        return ll
    return ev
