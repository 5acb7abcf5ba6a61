import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2405_16634_b200 import synth
import paper_2405_16634_b200.wn as wn
cfg, f = sys.argv[1], sys.argv[2]
p = torch.from_numpy(synth.config(cfg)["points"]).cuda()
t = wn.wn_build_tree(p)
order = torch.from_numpy(np.fromfile(f, np.int32)).cuda()
wn._L.wn_exp_set_schedule.restype = ctypes.c_int
assert wn._L.wn_exp_set_schedule(t.handle, ctypes.c_void_p(order.data_ptr()), None) == 0
mu = torch.zeros(len(p), 3, device="cuda")
wn.wnnc_iterate(t, mu, iters=2, total_iters=40, flags=wn.WN_FLAG_MU_ZERO)
torch.cuda.synchronize(); print("ok")
