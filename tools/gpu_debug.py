"""Progressive GPU smoke/debug run: prints parity vs the oracle for growing cases."""
import sys, time, math
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle, synth
import paper_1709_08625_b200 as H

def run(n, eta, eps, nu=0.5, ell=0.1, kmax=0, seed=1, nug=1e-6, geom='u', dense_below=32):
    s = synth.uniform_points(n, seed) if geom == 'u' else synth.collinear_points(n, seed)
    xi = synth.xi(n, seed + 1)
    Z = oracle.sample_dense(s, xi, 1.0, ell, nu, nug) if n <= 20000 else xi
    t0 = time.time(); ref = oracle.loglik_dense(s, Z, 1.0, ell, nu, nug) if n <= 20000 else (float('nan'),)*3; to = time.time()-t0
    T = H.Tree(torch.from_numpy(s).cuda(), eta=eta, dense_below=dense_below)
    Zd = torch.from_numpy(Z).cuda()
    r = H.eval_loglik(T, (1.0, ell, nu, nug), Zd, eps, kmax)
    torch.cuda.synchronize(); t0 = time.time()
    r = H.eval_loglik(T, (1.0, ell, nu, nug), Zd, eps, kmax)
    torch.cuda.synchronize(); tg = time.time()-t0
    rel = abs(r['loglik']-ref[0])/abs(ref[0])
    print(f"n={n} eta={eta} eps={eps} nu={nu} ell={ell}: gpu L={r['loglik']:.10f} ld={r['logdet']:.6f} q={r['quad']:.6f} st={r['status']} maxr={r['max_rank']} | oracle L={ref[0]:.10f} ld={ref[1]:.6f} q={ref[2]:.6f} | rel={rel:.3e} gpu {tg*1e3:.1f} ms oracle {to:.2f}s info={T.info()['n_waves']} waves", flush=True)
    return rel

if __name__ == '__main__':
    stage = sys.argv[1] if len(sys.argv) > 1 else 'all'
    run(100, 0.0, 1e-8)
    run(2000, 0.0, 1e-8)
    run(33, 2.0, 1e-8)
    run(2000, 2.0, 1e-8)
    run(2000, 2.0, 1e-4)
    run(4096, 2.0, 1e-8, nu=1.0, ell=0.05)
    run(16384, 2.0, 1e-8, nu=1.5, ell=0.05)
    run(16384, 2.0, 1e-4, nu=1.5, ell=0.01)
