"""The bench step for an ncu k_engine capture in under 300 s: C5's points (first n), the bench's
kernel (C4's theta, eps 1e-6, k 20), Z from a tighter factor as in bench.py, then two evaluations
(the second one is the profiled launch with -s <launches before it>).
  python tools/dram_probe.py [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2097152
cfg = synth.CONFIGS["C5"]
s = synth.points(cfg)[:n]
th = (1.0, 0.1, 0.5, 1e-6)
T = H.Tree(torch.from_numpy(s).cuda())
xi = torch.from_numpy(synth.xi(n, cfg.seed_xi)).cuda()
Z = None
for eg in (1e-7, 3e-7, 1e-6):
    g = H.HMatrix(T, th, eg, 20)
    try:
        g.cholesky()
        Z = g.sample(xi)
        break
    except H.HcovError as e:
        if e.code != 4:
            raise
    finally:
        del g
assert Z is not None
for _ in range(2):
    r = H.eval_loglik(T, th, Z, 1e-6, 20)
torch.cuda.synchronize()
print(r)
