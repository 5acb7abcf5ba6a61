"""Time wnnc_iterate(40 iterations, CUDA graph) on a prebuilt tree + per-class breakdown (no graph)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
nmax = int(sys.argv[2]) if len(sys.argv) > 2 else None  # optional: the first nmax points (a random subset)
p = torch.from_numpy(synth.config(cfg)["points"][:nmax]).cuda()
t = wn.wn_build_tree(p)
mu = torch.zeros(len(p), 3, device="cuda")
wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(3):
    mu.zero_()
    ev[0].record(); wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH); ev[1].record()
    torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]))
wn.wn_prof_enable(True)
mu.zero_(); wn.wnnc_iterate(t, mu, iters=40)
pr = wn.wn_prof_read(); wn.wn_prof_enable(False)
print(f"iterate40 ms {min(ts):.2f}", {k: round(v[0], 2) for k, v in pr.items() if v[1]})
