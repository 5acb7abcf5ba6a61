"""Short workload for ncu: C3 tree + `iters` WNNC iterations (all hot kernels appear)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
t = wn.wn_build_tree(p)
mu = torch.zeros(len(p), 3, device="cuda")
wn.wnnc_iterate(t, mu, iters=iters, total_iters=40)
torch.cuda.synchronize()
print("ok", t.num_nodes, t.depth_used)
