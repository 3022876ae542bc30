"""Debug: where does the H-Cholesky factor L~ leave the exact factor?  (R25 defect, near-full-rank.)

For small n, extract every column of L~ through hcov_sample (xi = e_j) and compare it, leaf block by
leaf block (internal order), with the exact dense Cholesky factor of C (oracle).  Prints the error
map per (eps, kcap) and the first leaf block (column-major elimination order) whose error exceeds
a threshold.  usage: python tools/dbg_factor.py [n]
"""
import os, sys, math
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
import paper_1709_08625_b200 as H

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
mode = sys.argv[2] if len(sys.argv) > 2 else "base"
th = (1.0, 0.1, 0.5, 1e-6)
s = synth.uniform_points(n, 11)
Z = oracle.sample_dense(s, synth.xi(n, 12), *th)
ref = oracle.loglik_dense(s, Z, *th)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
T = H.Tree(dev(s))
Tdb = {db: H.Tree(dev(s), dense_below=db) for db in (64, 128, 256)}
perm = T.perm_i2e()
real = np.nonzero(perm >= 0)[0]            # internal positions of real points
pr = perm[real]
C = oracle.cov_dense(s, *th)
Lx = oracle.cholesky(C[np.ix_(pr, pr)])      # exact factor in internal order (real rows only)
Cint = C[np.ix_(pr, pr)]
print(f"n={n} n_pad={perm.size} exact L={ref[0]:.12f}", flush=True)
from oracle import eps_oracle as EO
eo = EO.loglik_eps(s, Z, *th, eps_list=(1e-13, 1e-11, 1e-9), with_exact=False)
for e in (1e-13, 1e-11, 1e-9):
    v = eo[e]
    print(f"eps-oracle eps={e:g}: " + (v if isinstance(v, str) else f"L rel {abs(v[0]-ref[0])/abs(ref[0]):.2e} "
          f"logdet rel {abs(v[1]-ref[1])/abs(ref[1]):.2e} quad rel {abs(v[2]-ref[2])/abs(ref[2]):.2e}")
          + f" max_rank {eo[('info', e)]['max_rank']}", flush=True)

if mode == "base":
    cases = [(1e-13, 64, 32), (1e-13, 24, 32), (1e-11, 64, 32), (1e-11, 24, 32), (1e-9, 64, 32), (1e-9, 24, 32), (1e-9, 21, 32)]
else:   # bisection of the eps <= 1e-12 defect
    cases = [(1e-12, 64, 32), (3e-13, 64, 32), (1e-13, 64, 64), (1e-13, 64, 128), (1e-13, 64, 256),
             (1e-13, 80, 32), (1e-13, 96, 32), (1e-12, 96, 32), (3e-12, 64, 32)]
for eps, kcap, db in cases:
    hm = H.HMatrix(T if db == 32 else Tdb[db], th, eps=eps, kcap=kcap)
    # assembled C~ columns (external order) vs exact
    cols = hm.columns(list(range(n)))
    Ct = cols.cpu().numpy()
    ea = float(np.abs(Ct - C).max())
    try:
        st = hm.cholesky()
    except H.HcovError as e:
        print(f"eps={eps:g} kcap={kcap} dense_below={db}: cholesky error {e}", flush=True)
        continue
    r = hm.loglik(dev(Z))
    Lt = np.zeros((real.size, real.size))
    for k, j in enumerate(real):
        xi = np.zeros(n); xi[perm[j]] = 1.0
        z = hm.sample(dev(xi)).cpu().numpy()
        Lt[:, k] = z[pr]
    E = np.abs(Lt - Lx)
    # leaf-block error map (blocks of 32 internal positions of the padded order)
    leaf = real // 32
    nl = int(leaf.max()) + 1
    M = np.zeros((nl, nl))
    np.maximum.at(M, (leaf[:, None].repeat(real.size, 1), leaf[None, :].repeat(real.size, 0)), E)
    first = None
    for J in range(nl):
        for I in range(J, nl):
            if M[I, J] > 1e-9:
                first = (I, J, M[I, J]); break
        if first: break
    rec = np.abs(Lt @ Lt.T - Cint).max()
    print(f"eps={eps:g} kcap={kcap} dense_below={db}: L rel {abs(r['loglik']-ref[0])/abs(ref[0]):.2e} max_rank {r['max_rank']} "
          f"acc_loss {r['acc_loss']} | max|C~-C| {ea:.2e} | max|L~-L| {E.max():.2e} | max|L~L~^T - C| {rec:.2e} "
          f"| first bad leaf block {first}", flush=True)
    colerr = M.max(axis=0)
    print("   per leaf column max err: " + " ".join(f"{v:.0e}" for v in colerr), flush=True)
