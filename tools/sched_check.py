"""Per config: tree build time (incl. the schedule choice), chosen query schedule and its estimate, and the
40-iteration solve (CUDA graph)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
    bt = []
    wn.wn_prof_enable(True)
    t = wn.wn_build_tree(p)
    pr = wn.wn_prof_read()
    wn.wn_prof_enable(False)
    print(cfg, "build breakdown ms", {k: round(v[0], 2) for k, v in pr.items() if v[1]})
    for _ in range(3):
        torch.cuda.synchronize()
        ev[0].record()
        t = wn.wn_build_tree(p)
        ev[1].record()
        torch.cuda.synchronize()
        bt.append(ev[0].elapsed_time(ev[1]))
    kind, st = wn.wn_tree_schedule_stats(t)
    ts = []
    for _ in range(3):
        mu = torch.zeros(len(p), 3, device="cuda")
        ev[0].record()
        wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    print(f"{cfg} n={len(p)} build ms {min(bt):.2f} schedule {kind} {st} iterate40 ms {min(ts[1:]):.2f}", flush=True)
