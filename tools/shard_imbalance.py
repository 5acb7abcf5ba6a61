import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn
for cfg in ("C3", "C5", "C4"):
    c = synth.config(cfg); p = torch.from_numpy(c["points"]).cuda(); n = len(p)
    t = wn.wn_build_tree(p)
    mu = torch.from_numpy((c["normals"] * (4*np.pi/n)).astype(np.float32)).cuda()
    cnt = wn.wn_query_work(t, mu, 0.004, op=0).cpu().numpy().astype(np.int64)   # per query (caller order)
    e = wn.wn_tree_export(t)
    perm = e["perm"].cpu().numpy()
    # schedule order: qorder (Hilbert) of sorted points — not exported; approximate with sorted (Morton) order
    work = cnt[perm, 0] * 40 + cnt[perm, 3] * 10
    for W in (2, 4, 8):
        rs = [wn.wn_shard_range(n, r, W) for r in range(W)]
        tot = np.array([work[b:e_].sum() for b, e_ in rs])
        print(cfg, W, "imbalance max/mean %.3f" % (tot.max() / tot.mean()))
