"""Per-rank work of the query shards (multi-GPU): equal counts (wn_shard_range) vs the
work-weighted plan (wn_shard_plan), using the actual per-query node tests + live terms of an A traversal
with the configuration's normals (wn_query_work), in schedule order (wn_tree_schedule)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

for cfg in sys.argv[1:] or ("C3", "C4", "C5"):
    c = synth.config(cfg)
    p = torch.from_numpy(c["points"]).cuda()
    n = len(p)
    t = wn.wn_build_tree(p)
    mu = torch.from_numpy((synth.random_signs(c["normals"], 7) * (4 * np.pi / n)).astype(np.float32)).cuda()
    cnt = wn.wn_query_work(t, mu, 0.004, op=0).cpu().numpy().astype(np.int64)  # caller order
    perm = wn.wn_tree_export(t)["perm"].cpu().numpy()                             # sorted → caller
    sched = wn.wn_tree_schedule(t).cpu().numpy()                                 # position → sorted
    work = (cnt[:, 0] * 13 + cnt[:, 3] * 10)[perm[sched]]                         # per schedule position
    for W in (2, 4, 8):
        eq = [wn.wn_shard_range(n, r, W) for r in range(W)]
        pl = wn.wn_shard_plan(t, W)
        we = np.array([work[b:e].sum() for b, e in eq])
        wp = np.array([work[pl[r]:pl[r + 1]].sum() for r in range(W)])
        print(f"{cfg} W={W}: max/mean work — equal counts {we.max() / we.mean():.3f}, plan {wp.max() / wp.mean():.3f}")
