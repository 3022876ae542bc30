"""One warm-up + one measured evaluation (for ncu): python tools/prof_engine.py n nu ell eps kmax"""
import sys
import torch
sys.path.insert(0, ".")
import synth
import paper_1709_08625_b200 as H

n, nu, ell, eps, kmax = int(sys.argv[1]), float(sys.argv[2]), float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
s = synth.uniform_points(n, 1005)
T = H.Tree(torch.from_numpy(s).cuda())
Z = torch.from_numpy(synth.xi(n, 2005)).cuda()
for _ in range(2):
    r = H.eval_loglik(T, (1.0, ell, nu, 1e-6), Z, eps, kmax)
torch.cuda.synchronize()
print(r)
