"""C2 grid tail (largest ell) at eps = 1e-8 under the A/B switches (HCOV_TERM_MIN / HCOV_DENSE_DMMA are
read at every evaluation): status, capacity counters and L for the last grid points."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1709_08625_b200 as H  # noqa: E402

cfg = synth.CONFIGS["C2"]
s = synth.points(cfg)
Z = oracle.sample_dense(s, synth.xi(cfg.n, cfg.seed_xi), cfg.sigma2, cfg.ell, cfg.nu, cfg.nugget)
T = H.Tree(torch.from_numpy(s).cuda())
Zd = torch.from_numpy(Z).cuda()
tab = json.load(open("tests/golden/c2_eps_oracle.json"))
for tm, dm in (("1", "1"), ("0", "1"), ("1", "0"), ("0", "0")):
    os.environ["HCOV_TERM_MIN"] = tm
    os.environ["HCOV_DENSE_DMMA"] = dm
    for i in (56, 60, 61, 62, 63):
        ell = cfg.ell_grid[i]
        r = H.eval_loglik(T, (cfg.sigma2, ell, cfg.nu, cfg.nugget), Zd, eps=1e-8)
        ex = tab["rows"][str(i)]["exact"][0]
        print(json.dumps({"term_min": tm, "dmma": dm, "i": i, "ell": ell, "status": r["status"], "L": r["loglik"],
                          "logdet": r["logdet"], "quad": r["quad"], "exact": ex, "max_rank": r["max_rank"],
                          "acc_loss": r.get("acc_loss"), "interm_cuts": r.get("interm_cuts"),
                          "cap_binds": r.get("cap_binds")}), flush=True)
