"""Debug: is the eps = 1e-13 defect deterministic?  Repeated evaluations of the same case; bitwise
comparison of L, log det and q; the result counters.  usage: python tools/dbg_race.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
import paper_1709_08625_b200 as H

n = 1200
th = (1.0, 0.1, 0.5, 1e-6)
s = synth.uniform_points(n, 11)
Z = oracle.sample_dense(s, synth.xi(n, 12), *th)
ref = oracle.loglik_dense(s, Z, *th)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
T = H.Tree(dev(s))
for eps in (1e-13, 2e-13, 3e-13):
    vals = []
    for rep in range(4):
        r = H.eval_loglik(T, th, dev(Z), eps=eps, kcap=64)
        vals.append((r["loglik"], r["logdet"], r["quad"]))
    r.pop("n", None)
    same = all(v == vals[0] for v in vals)
    print(f"eps={eps:g}: rel {abs(vals[0][0]-ref[0])/abs(ref[0]):.2e} bitwise-repeatable={same} "
          f"L={[v[0] for v in vals]} result={r}", flush=True)
