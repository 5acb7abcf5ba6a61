"""Microbenchmark of the traversal kernels on C3 (realistic μ after a few iterations)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
t = wn.wn_build_tree(p)
mu = torch.zeros(len(p), 3, device="cuda")
wn.wnnc_iterate(t, mu, iters=10, total_iters=40)
s = (torch.rand(len(p), device="cuda") - 0.5) * 1e-3
w = 0.0096
for _ in range(3):
    wn.wn_eval(t, mu, w); wn.wn_eval_grad(t, mu, w); wn.wn_eval_adjoint(t, s, w)
torch.cuda.synchronize()
wn.wn_prof_enable(True)
for _ in range(reps):
    wn.wn_eval(t, mu, w); wn.wn_eval_grad(t, mu, w); wn.wn_eval_adjoint(t, s, w)
pr = wn.wn_prof_read()
wn.wn_prof_enable(False)
out = {k: v[0] / max(v[1], 1) for k, v in pr.items() if v[1]}
print("ms per launch:", {k: round(v, 4) for k, v in out.items()})
