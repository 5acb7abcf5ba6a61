"""Experiment (WN_EXP_SETSCHED variant): time the 40-iteration solve under query schedules read from files
(int32 sorted-point indices in schedule order), e.g. written by a host-side simulation of the traversal."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1]
p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
t = wn.wn_build_tree(p)
n = len(p)
wn._L.wn_exp_set_schedule.restype = ctypes.c_int
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for f in sys.argv[2:]:
    order = torch.from_numpy(np.fromfile(f, np.int32)).cuda()
    assert order.numel() == n
    assert wn._L.wn_exp_set_schedule(t.handle, ctypes.c_void_p(order.data_ptr()), None) == 0
    ts = []
    for _ in range(4):
        mu = torch.zeros(n, 3, device="cuda")
        ev[0].record()
        wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    print(cfg, f.split("/")[-1], f"iterate40 ms {min(ts[1:]):.2f}", flush=True)
