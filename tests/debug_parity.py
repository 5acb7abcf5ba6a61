"""Debug helper: compare tree / per-query decisions / values of the GPU path and the oracle on one case."""
import sys
import numpy as np
import torch
import oracle
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = synth.config(name)
p = cfg["points"]
n = len(p)
rng = np.random.default_rng(16)
mu = (synth.random_signs(cfg["normals"], 1005) * (4 * np.pi / n)).astype(np.float32)
w = float(np.float32(0.002))
t = wn.wn_build_tree(torch.from_numpy(p).cuda())
e = {k: v.cpu().numpy() for k, v in wn.wn_tree_export(t).items()}
xn, xf = oracle.normalize(p)
ot = oracle.Tree(xn)
o = ot.export()
print("nodes gpu/ora", t.num_nodes, ot.num_nodes, "depth", t.depth_used, ot.max_depth)
for k in ("perm", "depth", "pb", "pe", "child_begin", "child_count"):
    print(k, "equal" if np.array_equal(e[k], o[k]) else f"DIFF at {np.nonzero(e[k] != o[k])[0][:5]}")
mu_d = torch.from_numpy(mu).cuda()
F = wn.wn_eval(t, mu_d, w).cpu().numpy().astype(np.float64)
cnt = wn.wn_query_work(t, mu_d, w, 2.0).cpu().numpy()
cl = oracle.Cloud(p)
idx = rng.choice(n, 3000, replace=False)
Fo, co = cl.F(mu, w, qidx=idx, counters=True)
S = cl.abs_scale(oracle.OP_A, mu, w, qidx=idx)
err = np.abs(F[idx] - Fo)
rel = err / np.maximum(1e-4 * np.abs(Fo), 2e-6 * S)
bad = np.where(rel > 1)[0]
print(f"nbad={len(bad)} max rel={rel.max():.3e}")
c = cnt[idx]
print("different test counts:", int(np.sum(c[:, 0] != co[:, 0])), " term counts:", int(np.sum(c[:, 1] + c[:, 2] != co[:, 1] + co[:, 2])))
for i in bad[:8]:
    print(f"  q{idx[i]}: gpu {F[idx[i]]:.8e} ora {Fo[i]:.8e} S {S[i]:.3e} gpu cnt {c[i]} ora cnt {co[i]}")
# moments at this size
rep, attr, W = [x.cpu().numpy() for x in wn.wn_moments(t, mu_d)]
orep, oattr, oW = ot.moments(mu.astype(np.float64))
edge = 2.0 ** (1 - o["depth"].astype(np.float64))
dr = np.abs(rep - orep).max(1) / edge
print("max rep err / edge", dr.max(), "at depth", o["depth"][np.argmax(dr)], "max attr err", np.abs(attr - oattr).max(), np.abs(oattr).max())
