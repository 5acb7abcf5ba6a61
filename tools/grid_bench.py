"""Off-surface evaluation: F on a regular grid around the C3 cloud."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
c = synth.config("C3")
p = torch.from_numpy(c["points"]).cuda()
n = len(p)
mu = torch.from_numpy((c["normals"] * (4 * np.pi / n)).astype(np.float32)).cuda()
t = wn.wn_build_tree(p)
g = torch.linspace(-1.4, 1.4, res, device="cuda")
q = torch.stack(torch.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3).contiguous()
for m in (q[:10000], q):
    wn.wn_eval(t, mu, 0.002, q=m)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(3):
        F = wn.wn_eval(t, mu, 0.002, q=m)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 3
    print(f"{len(m)} queries: {ms:.2f} ms ({len(m) / ms / 1e3:.1f} M queries/s); inside fraction {(F > 0.5).float().mean().item():.3f}")
