"""One FMM application on a config (for ncu launch lists): python tools/fmm_one.py C3 p theta leaf"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
p, th, leaf = int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
c = synth.config(cfg)
pts = torch.from_numpy(c["points"]).cuda()
t = wn.wn_build_tree(pts)
mu = torch.from_numpy((c["normals"] * (4 * np.pi / len(pts))).astype(np.float32)).cuda()
out, cnt = wn.wn_eval_fmm(t, mu, 0.002, op=0, p=p, theta_f=th, leaf=leaf, counts=True)
torch.cuda.synchronize()
print("ok", cnt)
