"""Round-2 diagnostics (GPU): where the accuracy of very tight eps is lost (near-full-rank n = 1200,
C3 eps_gen 1e-10), and the memory of the 2M tight generating factor."""
import math, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
import paper_1709_08625_b200 as H


def dev(a): return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


which = sys.argv[1:] or ["nfr", "c3", "gen2m"]
if "nfr" in which:
    n = 1200
    s = synth.uniform_points(n, 11)
    th = (1.0, 0.1, 0.5, 1e-6)
    C = oracle.cov_dense(s, *th)
    Z = oracle.sample_dense(s, synth.xi(n, 12), *th)
    ref = oracle.loglik_dense(s, Z, *th)
    T = H.Tree(dev(s))
    for eps in (1e-11, 1e-12, 1e-13, 1e-14):
        for kc in (48, 64):
            h = H.HMatrix(T, th, eps, 0, kc)
            Ct = h.columns(np.arange(n)).cpu().numpy()
            fro = np.linalg.norm(Ct - C) / np.linalg.norm(C)
            two = np.linalg.norm(Ct - C, 2) / np.linalg.norm(C, 2)
            st = h.storage()
            try:
                h.cholesky()
                r = h.loglik(dev(Z))
                msg = (f"rel={abs(r['loglik']-ref[0])/abs(ref[0]):.2e} ld={abs(r['logdet']-ref[1])/abs(ref[1]):.2e} "
                       f"acc={r['acc_loss']} cuts={r['interm_cuts']} maxrL={r['max_rank']}")
            except H.HcovError as e:
                msg = str(e)
            # eps-oracle-like: the dense Cholesky of the assembled C~ itself
            try:
                Lt = np.linalg.cholesky(0.5 * (Ct + Ct.T))
                ldt = 2 * np.log(np.diag(Lt)).sum()
                msg2 = f"logdet(C~ assembled) rel {abs(ldt-ref[1])/abs(ref[1]):.2e}"
            except np.linalg.LinAlgError:
                msg2 = "C~ assembled not SPD"
            print(f"nfr eps={eps:g} kcap={kc}: asm fro={fro:.2e} 2norm={two:.2e} maxrC={st['max_rank']} | {msg} | {msg2}",
                  flush=True)
            del h
if "c3" in which:
    cfg = synth.CONFIGS["C3"]
    s = synth.points(cfg)
    th = (cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
    T = H.Tree(dev(s))
    cols = np.random.default_rng(5).choice(cfg.n, 64, replace=False)
    ce = H.cov_columns(T, th, cols)
    for eps in (1e-8, 1e-9, 1e-10, 1e-11):
        h = H.HMatrix(T, th, eps, 0, 64)
        ct = h.columns(cols)
        fro = float(torch.linalg.norm(ct - ce) / torch.linalg.norm(ce))
        st = h.storage()
        try:
            h.cholesky()
            r = "factored ok"
        except H.HcovError as e:
            r = str(e)
        print(f"c3 eps={eps:g}: asm fro={fro:.2e} maxrC={st['max_rank']} | {r} | mem {h.mem_info()}", flush=True)
        del h
if "gen2m" in which:
    c5, c4 = synth.CONFIGS["C5"], synth.CONFIGS["C4"]
    s = synth.points(c5)
    th = (c4.sigma2, c4.ell, c4.nu, c4.nugget)
    T = H.Tree(dev(s))
    for eps, k in ((1e-6, 20), (1e-7, 20), (1e-8, 20)):
        t0 = time.time()
        h = H.HMatrix(T, th, eps, k)
        try:
            fl = h.cholesky()
            msg = f"ok {h.storage()}"
        except H.HcovError as e:
            msg = str(e)
        print(f"gen2m eps={eps:g} k={k}: {msg} ({time.time()-t0:.1f}s) mem {h.mem_info()}", flush=True)
        del h
    print("cuda mem", torch.cuda.mem_get_info(), flush=True)
