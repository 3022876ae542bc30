"""Round-2 diagnostics (GPU): near-full-rank accuracy vs eps, C3 tight-factor SPD, bench eps_gen."""
import math, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
import paper_1709_08625_b200 as H

def dev(a): return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()

which = sys.argv[1:] or ["nfr", "c3"]
if "nfr" in which:
    n = 1200
    s = synth.uniform_points(n, 11)
    th = (1.0, 0.1, 0.5, 1e-6)
    Z = oracle.sample_dense(s, synth.xi(n, 12), *th)
    ref = oracle.loglik_dense(s, Z, *th)
    for db in (32, 4096):
        T = H.Tree(dev(s), dense_below=db)
        for interm in ("1e-2", "1e-6"):
            os.environ["HCOV_INTERM_REL"] = interm
            for eps in (1e-9, 1e-10, 1e-11, 1e-12, 1e-13, 1e-14):
                r = H.eval_loglik(T, th, dev(Z), eps=eps, kcap=64)
                print(f"nfr db={db} interm={interm} eps={eps:g}: st={r['status']} rel={abs(r['loglik']-ref[0])/abs(ref[0]):.2e} "
                      f"ld={abs(r['logdet']-ref[1])/abs(ref[1]):.2e} q={abs(r['quad']-ref[2])/abs(ref[2]):.2e} "
                      f"maxr={r['max_rank']} acc={r['acc_loss']} minpiv={r['min_pivot']:.3e}", flush=True)
    os.environ["HCOV_INTERM_REL"] = "1e-2"
if "c3" in which:
    cfg = synth.CONFIGS["C3"]
    s = synth.points(cfg)
    th = (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    T = H.Tree(dev(s))
    xi = dev(synth.xi(cfg.n, cfg.seed_xi))
    for eps, kmax, kcap in ((1e-10, 0, 64), (1e-9, 0, 64), (1e-8, 0, 64), (1e-10, 48, 48), (1e-6, 16, 16)):
        for interm in ("1e-2", "1e-6"):
            os.environ["HCOV_INTERM_REL"] = interm
            t0 = time.time()
            r = H.eval_loglik(T, th, xi, eps=eps, kmax=kmax, kcap=kcap)
            print(f"c3 eps={eps:g} kmax={kmax} kcap={kcap} interm={interm}: st={r['status']} L={r['loglik']:.6f} "
                  f"maxr={r['max_rank']} acc={r['acc_loss']} fail={r['fail_leaf']} minpiv={r['min_pivot']:.3e} "
                  f"cb={r['cap_binds']} ({time.time()-t0:.1f}s)", flush=True)
    os.environ["HCOV_INTERM_REL"] = "1e-2"
if "gen2m" in which:
    c5, c4 = synth.CONFIGS["C5"], synth.CONFIGS["C4"]
    s = synth.points(c5)
    th = (c4.sigma2, c4.ell, c4.nu, c4.nugget)
    T = H.Tree(dev(s))
    xi = dev(synth.xi(c5.n, c5.seed_xi))
    for eps in (1e-8, 1e-7, 3e-7):
        t0 = time.time()
        try:
            h = H.HMatrix(T, th, eps, 20)
            fl = h.cholesky()
            print(f"gen2m eps={eps:g}: ok fail={fl} {h.storage()} ({time.time()-t0:.1f}s)", flush=True)
            del h
        except H.HcovError as e:
            print(f"gen2m eps={eps:g}: {e} ({time.time()-t0:.1f}s)", flush=True)
