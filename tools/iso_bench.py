"""Row f1: adaptive octree sampling of F around ½ (wn_iso_cells) on the solved C3 cloud — cells crossed, F
evaluations and time per call for several finest levels, against the dense lattice of the same level."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
c = synth.config(cfg)
pts = torch.from_numpy(c["points"]).cuda()
n = len(pts)
t = wn.wn_build_tree(pts)
mu = torch.zeros(n, 3, device="cuda")
wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
w = float(np.float32(0.002))
for base, lmax, band in ((5, 8, 0.1), (5, 9, 0.1), (5, 10, 0.1), (6, 10, 0.05)):
    wn.wn_iso_cells(t, mu, w, base_level=base, max_level=lmax, band=band)  # warm-up (and capacity)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        cells, vals, evals = wn.wn_iso_cells(t, mu, w, base_level=base, max_level=lmax, band=band, capacity=1 << 23)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    dense = ((1 << lmax) + 1) ** 3
    print(f"{cfg} iso cells base {base} max {lmax} ({1 << lmax}^3) band {band}: {len(cells)} cells crossed, "
          f"{evals} F evaluations ({evals / dense:.4f} of the {dense} lattice points), {ms:.2f} ms per call "
          f"(wall clock, synchronizing)")
