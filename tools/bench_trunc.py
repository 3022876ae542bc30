"""Time the truncation kernel (one CTA, hcov_test_truncate) per QR path:
python tools/bench_trunc.py [m R reps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1709_08625_b200 as H

m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
R = int(sys.argv[2]) if len(sys.argv) > 2 else 92
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rng = np.random.default_rng(1)
A = np.linalg.qr(rng.standard_normal((m, R)))[0] * 10.0 ** (-np.arange(R) / 8.0)
B = rng.standard_normal((m, R))
X, Y = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
for path in (0, 1, 2):
    H.test_truncate(X, Y, 1e-10, rlim=R, path=path)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        U, V, r, cb, of = H.test_truncate(X, Y, 1e-10, rlim=R, path=path)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    S = A @ B.T
    err = np.linalg.norm(S - U.cpu().numpy() @ V.cpu().numpy().T, 2) / np.linalg.norm(S, 2)
    print(f"m={m} R={R} path={path}: {dt*1e3:.3f} ms/call (incl. malloc+copy), rank {r}, rel err {err:.2e}")
