"""Build libwn.so from the committed sources (git HEAD) into paper_2405_16634_b200/exp/head/, next to the
working-tree build — an A/B baseline for tools/run_variants_cfg.sh."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_16634_b200 import build as b
d = os.path.join(b.HERE, "exp", "head")
src = os.path.join(b.ROOT, ".exp_head", "csrc")  # two levels below the root: the sources' relative includes hold
os.makedirs(src, exist_ok=True)
for f in os.listdir(b.CSRC):
    if f.endswith((".cu", ".cuh")):
        rel = os.path.relpath(os.path.join(b.CSRC, f), b.ROOT)
        with open(os.path.join(src, f), "wb") as fh:
            fh.write(subprocess.check_output(["git", "show", f"HEAD:{rel}"], cwd=b.ROOT))
b.CSRC = src
b.build(lib=os.path.join(d, "libwn.so"), obj=os.path.join(d, "obj"))
print("head ok")
