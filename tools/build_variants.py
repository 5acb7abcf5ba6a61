"""Build experimental libwn variants (macros) into paper_2405_16634_b200/exp/<name>/libwn.so."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_16634_b200 import build as b
VARIANTS = {
    "base": [],
    "debug": ["WN_DEBUG"],  # device-side bounds checks (trap on violation)
    "setsched": ["WN_EXP_SETSCHED"],  # wn_exp_set_schedule hook for tools/sched_exp.py
    "tb64": ["WN_EXP_TRAVBLOCK=64"],  # 64-query traversal blocks
    "tb256": ["WN_EXP_TRAVBLOCK=256"],
    "lb5": ["WN_EXP_LBMIN=5"],  # resident 256-thread-equivalents per SM of the one-warp traversal
    "mt512": ["WN_EXP_MOMTILE=512"],  # moment-build tiles of 512 / 2048 points (default 1024)
    "mt2048": ["WN_EXP_MOMTILE=2048"],
    "mt1152": ["WN_EXP_MOMTILE=1152"],  # C3: 435 tiles ≤ 148 SMs × 3 resident tiles (one wave)
    "mt1280": ["WN_EXP_MOMTILE=1280"],
    "mt256": ["WN_EXP_MOMTILE=256"],
    "mt384": ["WN_EXP_MOMTILE=384"],
    "mt768": ["WN_EXP_MOMTILE=768"],
    "mw64": ["WN_EXP_MOMWARP=64"],  # moment build: nodes of >= 64 / 128 points summed by a warp (default 32)
    "mw128": ["WN_EXP_MOMWARP=128"],
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    d = os.path.join(b.HERE, "exp", n)
    b.build(lib=os.path.join(d, "libwn.so"), obj=os.path.join(d, "obj"), defines=VARIANTS[n])
    print(n, "ok")
