"""GPU probe: per-stage wall times of the hot path for one config-like case (no oracle).

usage: python tools/probe.py n nu ell eps kmax [reps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402


def main():
    n, nu, ell, eps, kmax = int(sys.argv[1]), float(sys.argv[2]), float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
    reps = int(sys.argv[6]) if len(sys.argv) > 6 else 2
    s = synth.uniform_points(n, 1005)
    t0 = time.time()
    T = H.Tree(s)
    tb = time.time() - t0
    info = T.info()
    print(f"n={n} tree {tb:.2f}s info={info}", flush=True)
    Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
    th = (1.0, ell, nu, 1e-6)
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.time()
        h = H.HMatrix(T, th, eps, kmax)
        torch.cuda.synchronize()
        t1 = time.time()
        fl = h.cholesky()
        t2 = time.time()
        res = h.loglik(Z)
        t3 = time.time()
        st = h.storage()
        print(f"rep {r}: assemble {t1-t0:.3f}s chol {t2-t1:.3f}s loglik {t3-t2:.3f}s total {t3-t0:.3f}s "
              f"L={res['loglik']:.6f} ld={res['logdet']:.4f} q={res['quad']:.4f} maxr={res['max_rank']} "
              f"cap={res['cap_binds']} minpiv={res['min_pivot']:.3e} storage={st}", flush=True)
        del h


if __name__ == "__main__":
    main()
