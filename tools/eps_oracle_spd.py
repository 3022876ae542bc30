"""Is C5's kernel SPD under the METHOD's best possible approximation?  (last bullet.)

Runs the eps-oracle (oracle/eps_oracle.py: dense C, every admissible block replaced by its optimal
(eps, k) SVD truncation) on C5's kernel (sigma2 1, ell 0.05, nu 1, tau^2 1e-6) at
n = 32,768 uniform points (seed 1005), for several (eps, k), and reports whether the truncated matrix
admits a Cholesky factorisation, plus the exact L.  CPU only; calls only oracle/.
usage: python tools/eps_oracle_spd.py [n] > profiles/r2_eps_oracle_c5_32k.txt
"""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import oracle
from oracle import eps_oracle as EO

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
th = (1.0, 0.05, 1.0, 1e-6)
s = synth.uniform_points(n, 1005)
Z = synth.xi(n, 2005)
t0 = time.time()
C = oracle.cov_dense(s, *th)
print(f"n={n} theta={th} fill {time.time()-t0:.1f}s threads={oracle.THREADS}", flush=True)
t0 = time.time()
try:
    ex = oracle.loglik_from_factor(oracle.cholesky(C), Z)
    print(f"exact: L={ex[0]:.10f} logdet={ex[1]:.6f} quad={ex[2]:.6f} ({time.time()-t0:.1f}s)", flush=True)
except oracle.NotSPD as e:
    print(f"exact: NOT_SPD ({e})", flush=True)
t0 = time.time()
spectra = EO.truncation_spectra(s, C)
print(f"spectra of {len(spectra)} admissible blocks {time.time()-t0:.1f}s", flush=True)
rows = []
for eps, kmax in ((1e-5, 20), (1e-5, 0), (1e-6, 20), (1e-6, 0), (1e-7, 0), (1e-8, 0)):
    Ce, info = EO.eps_matrix(C, spectra, eps, kmax)
    t0 = time.time()
    try:
        r = oracle.loglik_from_factor(oracle.cholesky(Ce), Z)
        res = {"L": r[0], "logdet": r[1], "quad": r[2]}
    except oracle.NotSPD as e:
        res = {"status": "NOT_SPD", "detail": str(e)}
    del Ce
    row = {"n": n, "eps": eps, "kmax": kmax, **info, **res, "sec": round(time.time() - t0, 1)}
    rows.append(row)
    print(json.dumps(row), flush=True)
