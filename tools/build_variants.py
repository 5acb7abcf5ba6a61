"""Build experimental libwn variants (macros) into paper_2405_16634_b200/exp/<name>/libwn.so."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_16634_b200 import build as b
VARIANTS = {
    "base": [],
    "debug": ["WN_DEBUG"],
    "setsched": ["WN_EXP_SETSCHED"],
    "tb64": ["WN_EXP_TRAVBLOCK=64"],  # 64-query traversal blocks
    "tb256": ["WN_EXP_TRAVBLOCK=256"],
    "lb5": ["WN_EXP_LBMIN=5"],
    "few4k": ["WN_EXP_FEWTILES=4096"],  # moments: prefix blocks sum the earlier tile totals up to 4096 tiles  # resident 256-thread-equivalents per SM of the one-warp traversal
    "kdlpt": ["WN_EXP_KDLPT"],  # k-d schedule with the heaviest blocks first  # wn_exp_set_schedule hook for tools/sched_exp.py  # device-side bounds checks (trap on violation)
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    d = os.path.join(b.HERE, "exp", n)
    b.build(lib=os.path.join(d, "libwn.so"), obj=os.path.join(d, "obj"), defines=VARIANTS[n])
    print(n, "ok")
