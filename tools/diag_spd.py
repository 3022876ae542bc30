"""Which C5-like configurations factor (SPD) at which n.  usage: python tools/diag_spd.py"""
import sys, time
import torch
sys.path.insert(0, '.')
import synth
import paper_1709_08625_b200 as H

cases = [(32768, 1.0, 0.05, 1e-5, 20, 0), (65536, 1.0, 0.05, 1e-5, 20, 0), (65536, 1.0, 0.05, 1e-5, 0, 64),
         (65536, 1.0, 0.05, 1e-6, 0, 64), (65536, 0.5, 0.1, 1e-6, 20, 0), (65536, 1.0, 0.05, 1e-7, 0, 64)]
for n, nu, ell, eps, kmax, kcap in cases:
    s = synth.uniform_points(n, 1005)
    T = H.Tree(torch.from_numpy(s).cuda())
    Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
    t0 = time.time()
    r = H.eval_loglik(T, (1.0, ell, nu, 1e-6), Z, eps, kmax, kcap)
    torch.cuda.synchronize()
    print(f"n={n} nu={nu} ell={ell} eps={eps} kmax={kmax} kcap={kcap}: status={r['status']} L={r['loglik']:.6f} "
          f"maxr={r['max_rank']} capbinds={r['cap_binds']} minpiv={r['min_pivot']:.3e} fail={r['fail_leaf']} "
          f"{time.time()-t0:.1f}s", flush=True)
