"""SPD-preserving mode (factor_trunc, R27) on C5's kernel: does it factor where the paper's
order does not, and how close is it to the exact L where the oracle can tell.
usage: python tools/diag_spd2.py"""
import sys, time, math
import numpy as np
import torch
sys.path.insert(0, '.')
import synth, oracle
import paper_1709_08625_b200 as H

th = (1.0, 0.05, 1.0, 1e-6)
def run(T, Z, eps, kmax, kcap, tag):
    t0 = time.time()
    try:
        r = H.eval_loglik(T, th, Z, eps, kmax, kcap)
    except Exception as e:
        print(f"  {tag}: {e}", flush=True); return None
    torch.cuda.synchronize()
    print(f"  {tag} eps={eps} kmax={kmax} kcap={kcap}: status={r['status']} L={r['loglik']:.8f} ld={r['logdet']:.6f} "
          f"q={r['quad']:.6f} maxr={r['max_rank']} capbinds={r['cap_binds']} minpiv={r['min_pivot']:.3e} "
          f"acc_loss={r['acc_loss']} interm_cuts={r['interm_cuts']} {time.time()-t0:.2f}s", flush=True)
    return r

for n in (8192, 16384):
    s = synth.uniform_points(n, 1005)
    Zh = oracle.sample_dense(s, synth.xi(n, 2005), *th)
    ref = oracle.loglik_dense(s, Zh, *th)
    print(f"n={n} exact L={ref[0]:.8f} ld={ref[1]:.6f} q={ref[2]:.6f}", flush=True)
    Z = torch.from_numpy(Zh).cuda()
    for ft in (False, True):
        T = H.Tree(torch.from_numpy(s).cuda(), factor_trunc=ft)
        for eps, kmax, kcap in ((1e-5, 20, 64), (1e-6, 20, 64), (1e-8, 0, 64)):
            r = run(T, Z, eps, kmax, kcap, "spd" if ft else "std")
            if r and r["status"] == 0:
                sc = 0.5 * n * math.log(2 * math.pi) + 0.5 * abs(ref[1]) + 0.5 * ref[2]
                print(f"     rel {abs(r['loglik']-ref[0])/abs(ref[0]):.2e} scaled {abs(r['loglik']-ref[0])/sc:.2e}", flush=True)
for n in (65536, 131072, 524288, 2097152):
    s = synth.uniform_points(n, 1005)
    Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
    print(f"n={n}", flush=True)
    T = H.Tree(torch.from_numpy(s).cuda(), factor_trunc=True)
    for eps, kmax, kcap in ((1e-5, 20, 64), (1e-5, 20, 40)):
        run(T, Z, eps, kmax, kcap, "spd")
    del T
