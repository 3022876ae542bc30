"""SPD-preserving mode at C5 scale: capacity vs memory vs SPD.  usage: python tools/diag_spd3.py"""
import sys, time
import torch
sys.path.insert(0, '.')
import synth
import paper_1709_08625_b200 as H

th = (1.0, 0.05, 1.0, 1e-6)
for n, cases in ((524288, ((1e-5, 20, 20), (1e-5, 20, 28), (1e-5, 20, 40))),
                 (2097152, ((1e-5, 20, 20), (1e-5, 20, 24), (1e-5, 20, 28)))):
    s = synth.uniform_points(n, 1005)
    Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
    T = H.Tree(torch.from_numpy(s).cuda(), factor_trunc=True)
    for eps, kmax, kcap in cases:
        t0 = time.time()
        try:
            r = H.eval_loglik(T, th, Z, eps, kmax, kcap)
            torch.cuda.synchronize()
            hm = H.last_eval(T)
            mi = hm.mem_info()
            print(f"n={n} spd eps={eps} kmax={kmax} kcap={kcap}: status={r['status']} L={r['loglik']:.6f} maxr={r['max_rank']} "
                  f"capbinds={r['cap_binds']} minpiv={r['min_pivot']:.3e} fail={r['fail_leaf']} acc_loss={r['acc_loss']} "
                  f"interm_cuts={r['interm_cuts']} {time.time()-t0:.1f}s mem={ {k: round(v/1e9, 2) for k, v in mi.items()} }", flush=True)
            del hm
        except Exception as e:
            print(f"n={n} spd eps={eps} kmax={kmax} kcap={kcap}: {e} {time.time()-t0:.1f}s", flush=True)
    del T
