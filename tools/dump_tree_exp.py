"""Experiment: dump a GPU tree (export, the solved mu's representatives, the Hilbert schedule) for tools-side simulation."""
import sys, numpy as np, torch, ctypes
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn
for cfg in sys.argv[1:]:
    p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
    t = wn.wn_build_tree(p)
    mu = torch.zeros(len(p), 3, device="cuda")
    wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
    e = {k: v.cpu().numpy() for k, v in wn.wn_tree_export(t).items()}
    rep, attr, W = wn.wn_moments(t, mu)
    hil = torch.empty(len(p), dtype=torch.int32, device="cuda")
    wn._L.wn_tree_schedule(t.handle, ctypes.c_void_p(hil.data_ptr()), None)
    np.savez(f"gpurun_out/tree_{cfg}.npz", hil=hil.cpu().numpy(), rep=rep.cpu().numpy(), **e)
    print(cfg, "ok", {k: v.shape for k, v in e.items()})
