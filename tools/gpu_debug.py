"""Progressive GPU debug run: parity vs the oracle for growing cases (prints, no asserts)."""
import sys, time, math
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle, synth
import paper_1709_08625_b200 as H


def run(n, eta, eps, nu=0.5, ell=0.1, kmax=0, seed=1, nug=1e-6, geom='u', staged=False):
    s = synth.uniform_points(n, seed) if geom == 'u' else synth.collinear_points(n, seed)
    xi = synth.xi(n, seed + 1)
    Z = oracle.sample_dense(s, xi, 1.0, ell, nu, nug) if n <= 20000 else xi
    t0 = time.time()
    ref = oracle.loglik_dense(s, Z, 1.0, ell, nu, nug) if n <= 20000 else (float('nan'),) * 3
    to = time.time() - t0
    T = H.Tree(torch.from_numpy(s).cuda(), eta=eta)
    Zd = torch.from_numpy(Z).cuda()
    if staged:
        h = H.HMatrix(T, (1.0, ell, nu, nug), eps, kmax)
        h.cholesky()
        r = h.loglik(Zd)
        r['status'] = 0
    r = H.eval_loglik(T, (1.0, ell, nu, nug), Zd, eps, kmax)
    torch.cuda.synchronize(); t0 = time.time()
    H.prof_control(True, True)
    r = H.eval_loglik(T, (1.0, ell, nu, nug), Zd, eps, kmax)
    torch.cuda.synchronize(); tg = time.time() - t0
    p = H.prof_read()
    rel = abs(r['loglik'] - ref[0]) / abs(ref[0])
    info = T.info()
    print(f"n={n} eta={eta} eps={eps} nu={nu} ell={ell}: gpu L={r['loglik']:.10f} ld={r['logdet']:.6f} q={r['quad']:.6f} "
          f"st={r['status']} maxr={r['max_rank']} | oracle L={ref[0]:.10f} | rel={rel:.3e} gpu {tg*1e3:.1f} ms "
          f"oracle {to:.2f}s tasks={info['n_tasks']} crit={info['n_waves']}", flush=True)
    busy = {k: round(v, 2) for k, v in p['task_busy_ms'].items() if v}
    print("   busy ms:", busy, "engine ms:", round(p['ms']['engine'], 2), flush=True)
    print("   phases ms:", {k: round(v, 1) for k, v in p['phase_ms'].items()}, flush=True)
    return rel


if __name__ == '__main__':
    which = sys.argv[1] if len(sys.argv) > 1 else 'small'
    if which == 'small':
        run(100, 0.0, 1e-8)
        run(2000, 0.0, 1e-8)
        run(33, 2.0, 1e-8)
        run(2000, 2.0, 1e-8, staged=True)
        run(2000, 2.0, 1e-4)
        run(4096, 2.0, 1e-8, nu=1.0, ell=0.05)
    else:
        run(16384, 2.0, 1e-8, nu=1.5, ell=0.05)
        run(16384, 2.0, 1e-4, nu=1.5, ell=0.01)
        run(65536, 2.0, 1e-6, nu=0.5, ell=0.1, kmax=20)
