"""Small workload touching every kernel path (tree, moments, A/G/Aᵀ at sources and queries, graph iteration,
transpose adjoint, order 1, world-1 communicator, emulated ranks) — run it against the WN_DEBUG build
(WN_LIB=paper_2405_16634_b200/exp/debug/libwn.so) to exercise the device-side bounds checks."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

p = torch.from_numpy(synth.config("C1")["points"]).cuda()
n = len(p)
rng = np.random.default_rng(0)
mu = torch.from_numpy((rng.standard_normal((n, 3)) * 4 * np.pi / n).astype(np.float32)).cuda()
s = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
q = torch.from_numpy(rng.uniform(-1.5, 1.5, (300, 3)).astype(np.float32)).cuda()
t = wn.wn_build_tree(p)
wn.wn_moments(t, mu)
wn.wn_eval(t, mu, 0.01)
wn.wn_eval_grad(t, mu, 0.01, q=q)
wn.wn_eval_adjoint(t, s, 0.01)
wn.wn_eval_adjoint(t, s, 0.01, mode=wn.WN_ADJ_TRANSPOSE, mu_geom=mu)
wn.wn_query_work(t, mu, 0.01)
m = torch.zeros(n, 3, device="cuda")
wn.wnnc_iterate(t, m, iters=3, total_iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
m = torch.zeros(n, 3, device="cuda")
wn.wnnc_iterate(t, m, iters=2, total_iters=40, adjoint_mode=wn.WN_ADJ_TRANSPOSE)
wn.wn_tree_set_far_order(t, 1)
wn.wn_eval(t, mu, 0.01)
m = torch.zeros(n, 3, device="cuda")
wn.wnnc_iterate(t, m, iters=2, total_iters=40)
wn.wn_tree_set_far_order(t, 0)
comm = wn.wn_comm_init(0, 1, wn.wn_comm_unique_id())
m = torch.zeros(n, 3, device="cuda")
wn.wnnc_iterate(t, m, comm=comm, iters=2, total_iters=40)
comm.close()
m = torch.zeros(n, 3, device="cuda")
wn.wnnc_iterate_emulated(t, m, 3, iters=2, total_iters=40)
t2 = wn.wn_build_tree(torch.from_numpy(synth.config("C2")["points"][:6000]).cuda())   # several moment tiles
m = torch.zeros(6000, 3, device="cuda")
wn.wnnc_iterate(t2, m, iters=2, total_iters=40)
torch.cuda.synchronize()
print("workload ok")
