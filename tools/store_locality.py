"""How scattered are the epilogue's peer stores?  Under the query schedule a warp's 32 queries write their
rows at their Morton-sorted indices; count the 128-byte lines (float4 rows) and 32-byte sectors a warp's
stores touch, against 4 lines / 16 sectors for 32 contiguous rows."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

for cfg in sys.argv[1:] or ["C3", "C4", "C5"]:
    p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
    t = wn.wn_build_tree(p)
    q = wn.wn_tree_schedule(t).cpu().numpy().astype(np.int64)
    kind, _ = wn.wn_tree_schedule_stats(t)
    n = len(q) // 32 * 32
    w = q[:n].reshape(-1, 32)
    for rb, name in ((16, "float4 rows"), (4, "float rows")):
        lines = np.array([len(np.unique(r * rb // 128)) for r in w])
        sect = np.array([len(np.unique(r * rb // 32)) for r in w])
        print(f"{cfg} ({kind}) {name}: 128-B lines per warp mean {lines.mean():.2f} (ideal {32 * rb // 128}), "
              f"32-B sectors mean {sect.mean():.2f} (ideal {32 * rb // 32})")
