"""Row f4: the GPU FMM (wn_eval_fmm) against the Alg. 4 treecode (wn_eval / _grad / _adjoint) on one cloud —
time per operator application (CUDA events), interaction counts, and the relative L2 difference between
the two (≈ the treecode's own error at c = 2, the FMM at p = 4 being ~1e-5 from the dense sum)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
c = synth.config(cfg)
p = torch.from_numpy(c["points"]).cuda()
n = len(p)
t = wn.wn_build_tree(p)
mu = torch.from_numpy((c["normals"] * (4 * np.pi / n)).astype(np.float32)).cuda()
s = torch.from_numpy(np.random.default_rng(3).uniform(-0.5, 0.5, n).astype(np.float32)).cuda()
w = 0.002


def timed(f, reps=5):
    f()  # (builds the FMM plan for new parameters)
    f()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        out = f()
    ev[1].record()
    torch.cuda.synchronize()
    return out, ev[0].elapsed_time(ev[1]) / reps


tree_ops = {0: lambda: wn.wn_eval(t, mu, w), 1: lambda: wn.wn_eval_adjoint(t, s, w), 2: lambda: wn.wn_eval_grad(t, mu, w)}
for op, name in ((0, "F (A)"), (1, "A^T"), (2, "gradF (G)")):
    ref, tms = timed(tree_ops[op])
    for pdeg, th, leaf in ((2, 0.5, 32), (4, 0.5, 32), (4, 0.7, 32), (2, 0.7, 16), (3, 0.8, 16), (2, 0.9, 8)):
        attr = s if op == 1 else mu
        (out, cnt), fms = timed(lambda: wn.wn_eval_fmm(t, attr, w, op=op, p=pdeg, theta_f=th, leaf=leaf, counts=True))
        d = (torch.linalg.norm(out - ref) / torch.linalg.norm(ref)).item()
        print(f"{cfg} {name:10s} treecode {tms:7.2f} ms | FMM p={pdeg} theta={th} leaf={leaf}: {fms:7.2f} ms, M2L {cnt[0]}, "
              f"P2P leaf pairs {cnt[1]}, rel. L2 difference to the treecode {d:.2e}")
