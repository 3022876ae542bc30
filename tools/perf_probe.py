"""Engine timing probe for build variants (HCOV_LIB=<in-tree .so>): one warm-up and `reps` timed
evaluations of L~ at n points of C5's set, with the engine's phase / task-busy breakdown.
  python tools/perf_probe.py [n] [nu] [ell] [eps] [kmax] [reps]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402

a = sys.argv[1:] + [None] * 6
n = int(a[0] or 524288)
nu, ell = float(a[1] or 0.5), float(a[2] or 0.1)
eps, kmax, reps = float(a[3] or 1e-6), int(a[4] or 20), int(a[5] or 2)
s = synth.uniform_points(n, 1005)
T = H.Tree(torch.from_numpy(s).cuda())
Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
th = (1.0, ell, nu, 1e-6)
r = H.eval_loglik(T, th, Z, eps, kmax)
H.prof_control(enable_events=True, reset=True)
t0 = time.time()
for _ in range(reps):
    r = H.eval_loglik(T, th, Z, eps, kmax)
torch.cuda.synchronize()
wall = (time.time() - t0) / reps
p = H.prof_read()
H.prof_control(enable_events=False, reset=True)
out = {"lib": os.environ.get("HCOV_LIB", "libhcov.so"), "n": n, "theta": th, "eps": eps, "kmax": kmax,
       "engine_ms": p["ms"].get("engine", 0) / reps, "wall_s": wall, "loglik": r["loglik"], "status": r["status"],
       "max_rank": r["max_rank"],
       "task_busy_cta_s": {k: round(v / reps / 1e3, 2) for k, v in p["task_busy_ms"].items() if v},
       "phase_cta_s": {k: round(v / reps / 1e3, 2) for k, v in p["phase_ms"].items() if v},
       "phase_cls_cta_s": {k: round(v / reps / 1e3, 2) for k, v in p["phase_cls_ms"].items() if v > 1}}
print(json.dumps(out), flush=True)
