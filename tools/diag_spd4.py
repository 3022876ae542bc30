"""One C5-kernel evaluation at n (default 2M), standard or SPD-preserving order.
usage: python tools/diag_spd4.py n spd eps kmax kcap"""
import sys, time
import torch
sys.path.insert(0, '.')
import synth
import paper_1709_08625_b200 as H
n, spd, eps, kmax, kcap = int(sys.argv[1]), sys.argv[2] == "1", float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
th = (1.0, 0.05, 1.0, 1e-6)
s = synth.uniform_points(n, 1005)
Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
T = H.Tree(torch.from_numpy(s).cuda(), factor_trunc=spd)
for rep in range(2):
    t0 = time.time()
    try:
        r = H.eval_loglik(T, th, Z, eps, kmax, kcap)
        torch.cuda.synchronize()
        mi = H.last_eval(T).mem_info()
        print(f"n={n} spd={spd} eps={eps} kmax={kmax} kcap={kcap}: status={r['status']} L={r['loglik']:.6f} maxr={r['max_rank']} "
              f"capbinds={r['cap_binds']} minpiv={r['min_pivot']:.3e} fail={r['fail_leaf']} acc_loss={r['acc_loss']} "
              f"interm_cuts={r['interm_cuts']} {time.time()-t0:.1f}s mem={ {k: round(v/1e9, 2) for k, v in mi.items()} }", flush=True)
    except Exception as e:
        print(f"n={n} spd={spd} eps={eps} kmax={kmax} kcap={kcap}: {e} {time.time()-t0:.1f}s", flush=True)
