import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn
c = synth.config("C3")
p = torch.from_numpy(c["points"]).cuda(); n = len(p)
t = wn.wn_build_tree(p)
mu = torch.from_numpy((c["normals"] * (4 * np.pi / n)).astype(np.float32)).cuda()
for pdeg in (2, 4, 4, 3, 4):
    for k in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        wn.wn_eval_fmm(t, mu, 0.002, op=0, p=pdeg, theta_f=0.5, leaf=32)
        torch.cuda.synchronize(); print(pdeg, k, round((time.perf_counter() - t0) * 1e3, 2), "ms")
