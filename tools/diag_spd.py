"""Which C5-like configurations factor (SPD) at which n.  usage: python tools/diag_spd.py [quick]"""
import sys, time
import torch
sys.path.insert(0, '.')
import synth
import paper_1709_08625_b200 as H

cases = [(65536, 1.0, 0.05, 1e-5, 20, 0), (65536, 1.0, 0.05, 1e-5, 0, 64), (65536, 1.0, 0.05, 1e-6, 0, 64),
         (131072, 1.0, 0.05, 1e-5, 20, 0), (131072, 1.0, 0.05, 1e-6, 20, 0), (131072, 1.0, 0.05, 1e-6, 0, 64),
         (524288, 1.0, 0.05, 1e-5, 20, 0), (524288, 1.0, 0.05, 1e-6, 20, 0), (524288, 1.0, 0.05, 1e-7, 32, 0),
         (2097152, 1.0, 0.05, 1e-5, 20, 0)]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    cases = cases[:6]
trees = {}
for n, nu, ell, eps, kmax, kcap in cases:
    if n not in trees:
        trees.clear()
        s = synth.uniform_points(n, 1005)
        trees[n] = H.Tree(torch.from_numpy(s).cuda())
    T = trees[n]
    Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
    t0 = time.time()
    try:
        r = H.eval_loglik(T, (1.0, ell, nu, 1e-6), Z, eps, kmax, kcap)
    except Exception as e:
        print(f"n={n} nu={nu} ell={ell} eps={eps} kmax={kmax} kcap={kcap}: {e}", flush=True)
        continue
    torch.cuda.synchronize()
    print(f"n={n} nu={nu} ell={ell} eps={eps} kmax={kmax} kcap={kcap}: status={r['status']} L={r['loglik']:.6f} "
          f"maxr={r['max_rank']} capbinds={r['cap_binds']} minpiv={r['min_pivot']:.3e} fail={r['fail_leaf']} "
          f"acc_loss={r['acc_loss']} interm_cuts={r['interm_cuts']} {time.time()-t0:.1f}s", flush=True)
