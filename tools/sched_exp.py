"""Experiment (variant build with WN_EXP_SETSCHED): the 40-iteration solve with the tree's Hilbert query
schedule vs a k-d schedule computed here (recursive median splits along the longest box axis at multiples
of 32 queries) — is grouping the warps' queries by k-d boxes worth building on the GPU?"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

sys.setrecursionlimit(100000)
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
t = wn.wn_build_tree(p)
xn = wn.wn_tree_export(t)["xn"].cpu().numpy().astype(np.float64)
n = len(xn)


def axis_bbox(q):
    return int(np.argmax(q.max(0) - q.min(0)))


def axis_sample(q, S=16, trim=2):  # extent of a 16-point sample without its 2 extremes per side
    s = np.sort(q[(np.arange(S) * len(q)) // S], 0)
    return int(np.argmax(s[S - 1 - trim] - s[trim]))


def kd(idx, out, axf):
    m = len(idx)
    if m <= 32:
        out.append(idx)
        return
    q = xn[idx]
    ax = axf(q)
    o = idx[np.argsort(q[:, ax], kind="stable")]
    left = (((m + 31) // 32) // 2) * 32
    kd(o[:left], out, axf)
    kd(o[left:], out, axf)


orders = {}
for name, axf in (("kd_bbox", axis_bbox), ("kd_sample", axis_sample)):
    out = []
    kd(np.arange(n), out, axf)
    orders[name] = np.concatenate(out).astype(np.int32)
hil = torch.empty(n, dtype=torch.int32, device="cuda")
wn._L.wn_tree_schedule(t.handle, ctypes.c_void_p(hil.data_ptr()), None)
orders["hilbert"] = hil.cpu().numpy()
wn._L.wn_exp_set_schedule.restype = ctypes.c_int
mu = torch.zeros(n, 3, device="cuda")
wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
perm = wn.wn_tree_export(t)["perm"].cpu().numpy()
cnt = wn.wn_query_work(t, mu, 0.004).cpu().numpy().astype(np.int64)
work_sorted = np.empty(n, np.int64)
work_sorted[np.arange(n)] = (cnt[:, 0] + cnt[:, 2])[perm]  # tests + leaf terms of sorted point k


def lpt(order, B=128):  # blocks of B schedule positions, heaviest block first
    nb = (n + B - 1) // B
    w = np.array([work_sorted[order[b * B:(b + 1) * B]].sum() for b in range(nb)])
    full = nb if n % B == 0 else nb - 1  # keep a ragged last block last
    ob = list(np.argsort(-w[:full], kind="stable")) + list(range(full, nb))
    return np.concatenate([order[b * B:(b + 1) * B] for b in ob]).astype(np.int32)


for k in list(orders):
    orders[k + "+lpt"] = lpt(orders[k])
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
res = {}
for name in ("hilbert", "hilbert+lpt", "kd_bbox", "kd_bbox+lpt", "kd_sample", "kd_sample+lpt", "hilbert"):
    order = torch.from_numpy(orders[name]).cuda()
    st = wn._L.wn_exp_set_schedule(t.handle, ctypes.c_void_p(order.data_ptr()), None)
    assert st == 0
    torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        mu = torch.zeros(n, 3, device="cuda")
        ev[0].record()
        wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    res[name] = mu.cpu().numpy()
    wn.wn_prof_enable(True)
    mu = torch.zeros(n, 3, device="cuda")
    wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_MU_ZERO)
    pr = wn.wn_prof_read()
    wn.wn_prof_enable(False)
    print(cfg, name, f"iterate40 ms {min(ts[1:]):.2f}", {k: round(v[0], 2) for k, v in pr.items() if v[1]}, flush=True)
a, b = res["hilbert"], res["kd_sample"]
print("orientation agreement", float(np.mean(np.sum(a * b, 1) > 0)), "max rel diff",
      float(np.max(np.linalg.norm(a - b, axis=1)) / np.max(np.linalg.norm(a, axis=1))))
