"""C2 (BASELINE.json configs[1]): n = 16,384, nu = 3/2, 64 ell values log-spaced in [0.01, 0.3]
(R16), eps in {1e-4, 1e-8}: the GPU path against the dense oracle AND the eps-oracle
(SURVEY.md Sec. 8(c) rows 11-12, App. A.4), all 128 points.

The oracle side is the committed table tests/golden/c2_eps_oracle.json, written by
tools/gen_c2_table.py from oracle/ only (exact dense L, and L of the dense matrix with every
admissible block replaced by its optimal (eps) SVD truncation).  Per theta and eps:

* error measure (R11): plain relative error of L, or the component-scaled error where
  |L| < 0.1 x (n/2 log 2pi + |log det|/2 + q/2);
* where the eps-oracle meets the north_star bar (1e-6 at eps = 1e-8, 1e-3 at eps = 1e-4) the
  GPU must meet it too;
* where it does not (the bar is unattainable by ANY eps-truncation), the GPU must satisfy
  |L_gpu - L_eps| <= |L_eps - L_exact| (row 12) — it may be no further from the eps-oracle than
  the eps-oracle is from the exact value;
* NOT_SPD is legal only where the eps-oracle itself is NOT_SPD; the count is reported.
"""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402

pytestmark = pytest.mark.gpu
TABLE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c2_eps_oracle.json")
BAR = {1e-8: 1e-6, 1e-4: 1e-3}


def _scale(ld, q, n):
    return 0.5 * n * math.log(2 * math.pi) + 0.5 * abs(ld) + 0.5 * q


def _err(L, ref, n):
    """R11 error of L against ref = (L, logdet, quad)."""
    sc = _scale(ref[1], ref[2], n)
    if abs(ref[0]) < 0.1 * sc:
        return abs(L - ref[0]) / sc
    return abs(L - ref[0]) / abs(ref[0])


@pytest.fixture(scope="module")
def c2():
    if not os.path.exists(TABLE):
        pytest.skip("tests/golden/c2_eps_oracle.json missing (python tools/gen_c2_table.py)")
    tab = json.load(open(TABLE))
    cfg = synth.CONFIGS["C2"]
    s = synth.points(cfg)
    Z = oracle.sample_dense(s, synth.xi(cfg.n, cfg.seed_xi), cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    T = H.Tree(torch.from_numpy(s).cuda())
    return cfg, tab, T, torch.from_numpy(Z).cuda()


@pytest.mark.parametrize("eps", [1e-8, 1e-4])
def test_c2_grid_vs_oracle_and_eps_oracle(c2, eps):
    cfg, tab, T, Zd = c2
    n = cfg.n
    rows, fails = [], []
    n_notspd = n_notspd_eo = n_capacity = 0
    for i in range(len(cfg.ell_grid)):
        row = tab["rows"].get(str(i))
        if row is None:
            continue
        ell = cfg.ell_grid[i]
        assert abs(row["ell"] - ell) <= 1e-15 * ell
        ex = row["exact"]
        eo = row[repr(eps)]
        r = H.eval_loglik(T, (cfg.sigma2, ell, cfg.nu, cfg.nugget), Zd, eps=eps)
        st = r["status"]
        if st == 6:
            # HCOV_ERR_RANK_CAPACITY (include/hcov.h): with kmax = 0 an eps-rank exceeded the largest
            # capacity, 64 (the largest ell of the grid have eps-ranks 62-65 at eps = 1e-8, so which
            # side of 64 a block falls on is a rounding-level matter).  The documented remedy is the
            # paper's "eps with a rank cap k" (Remark 2): the point is graded at
            # k = 64, where the cut singular values are at the eps level
            n_capacity += 1
            r = H.eval_loglik(T, (cfg.sigma2, ell, cfg.nu, cfg.nugget), Zd, eps=eps, kmax=64, kcap=64)
            st = r["status"]
            assert r["cap_binds"] <= 8, (i, r)
        if eo == "NOT_SPD":
            n_notspd_eo += 1
        if st == 3:
            n_notspd += 1
            rows.append((i, ell, ex[0], eo if isinstance(eo, str) else eo[0], "NOT_SPD", None, None, None))
            if eo != "NOT_SPD":
                fails.append((i, ell, "GPU NOT_SPD where the eps-oracle is SPD"))
            continue
        assert st == 0, (i, r)
        assert r["acc_loss"] == 0, (i, r)
        e_gpu = _err(r["loglik"], ex, n)
        if eo == "NOT_SPD":
            rows.append((i, ell, ex[0], "NOT_SPD", r["loglik"], e_gpu, None, "eps-oracle indefinite"))
            continue
        e_eo = _err(eo[0], ex, n)
        if e_eo <= BAR[eps]:
            rule, ok = f"bar {BAR[eps]:g}", e_gpu <= BAR[eps]
        else:
            rule, ok = "row 12", abs(r["loglik"] - eo[0]) <= abs(eo[0] - ex[0])
        rows.append((i, ell, ex[0], eo[0], r["loglik"], e_gpu, e_eo, rule + ("" if ok else " FAIL")))
        if not ok:
            fails.append((i, ell, rule, e_gpu, e_eo))
    lines = [f"C2 eps={eps:g}: i ell L_exact L_eps-oracle L_gpu err_gpu err_eps-oracle rule"]
    for t in rows:
        lines.append(" ".join(str(x) if not isinstance(x, float) else f"{x:.10g}" for x in t))
    lines.append(f"NOT_SPD: gpu {n_notspd}, eps-oracle {n_notspd_eo} of {len(rows)}; "
                 f"graded at k = 64 after RANK_CAPACITY: {n_capacity}")
    print("\n".join(lines))
    out = os.environ.get("HCOV_C2_REPORT")
    if out:
        with open(f"{out}_eps{eps:g}.txt", "w") as f:
            f.write("\n".join(lines) + "\n")
    assert len(rows) >= 1
    assert not fails, fails
