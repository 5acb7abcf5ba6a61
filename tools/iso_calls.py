"""Per-call wall times of wn_iso_cells (C3, finest level 512^3) over consecutive calls in one process."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

c = synth.config("C3")
pts = torch.from_numpy(c["points"]).cuda()
t = wn.wn_build_tree(pts)
mu = torch.zeros(len(pts), 3, device="cuda")
wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_MU_ZERO)
w = float(np.float32(0.002))
for lmax in (9, 9, 9, 9, 9, 9, 10, 10, 10, 10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cells, vals, ev = wn.wn_iso_cells(t, mu, w, base_level=5, max_level=lmax, band=0.1, capacity=1 << 23)
    torch.cuda.synchronize()
    print(lmax, round((time.perf_counter() - t0) * 1e3, 2), "ms")
