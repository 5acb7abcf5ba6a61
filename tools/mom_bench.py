"""Moment-build microbenchmark: wn_moments (vector and scalar attributes) on a prebuilt tree."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
t = wn.wn_build_tree(p)
g = torch.Generator(device="cuda").manual_seed(1)
nu = torch.randn(len(p), 3, device="cuda", generator=g)
s = torch.randn(len(p), device="cuda", generator=g)
for x in (nu, s):
    wn.wn_moments(t, x)
    torch.cuda.synchronize()
    wn.wn_prof_enable(True)
    for _ in range(reps):
        wn.wn_moments(t, x)
    pr = wn.wn_prof_read()
    wn.wn_prof_enable(False)
    print("dim", x.dim(), "moments us/build", round(1000 * pr["moments"][0] / reps, 1))
