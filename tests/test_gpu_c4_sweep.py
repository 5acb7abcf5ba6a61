"""C4 robustness sweep: smoothing widths (w1, w2) × opening parameter c on the stress
cloud (thin plate + thin torus + 1 % outliers, N = 200,000), GPU against the oracle.

PAPER.md:L808-L813 (§5.2.5) presets larger widths for noisier inputs; PAPER.md:L385 (Alg. 4) is the
far-field criterion |x − x_B| > c·width(B).  For every setting: the 40-iteration solve on the bench path
(CUDA graph, μ⁰ = 0), its time, the algorithmic work per query and operator (counting pass, same decisions),
the orientation agreement with the oracle's solve and P_co of both against the analytic normals (outliers
excluded).  Gated by WN_SWEEP=1 (≈ 5 min of oracle time on 16 cores); rows go to $WN_SWEEP_OUT (JSON).
"""
import json
import os
import time

import numpy as np
import pytest

import oracle
from paper_2405_16634_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(os.environ.get("WN_SWEEP") != "1", reason="sweep: set WN_SWEEP=1")]

WIDTHS = [(0.002, 0.016), (0.01, 0.04), (0.02, 0.08)]
THETAS = [1.0, 2.0, 4.0]
ROWS = []


@pytest.fixture(scope="module")
def c4():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    cfg = synth.config("C4")
    yield wn, cfg, oracle.Cloud(cfg["points"])
    out = os.environ.get("WN_SWEEP_OUT")
    if out and ROWS:
        with open(out, "w") as f:
            json.dump(ROWS, f, indent=1)


@pytest.mark.parametrize("theta", THETAS)
@pytest.mark.parametrize("widths", WIDTHS)
def test_c4_sweep(c4, widths, theta):
    wn, cfg, cl = c4
    p, nr, inl = cfg["points"], cfg["normals"], cfg["inlier"]
    w1, w2 = (float(np.float32(x)) for x in widths)
    pts = torch.from_numpy(p).cuda()
    prm = dict(w_min=w1, w_max=w2, theta=theta, iters=40, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
    tree = wn.wn_build_tree(pts)
    mu = torch.zeros(tree.n, 3, device="cuda")
    wn.wnnc_iterate(tree, mu, **prm)  # (captures the graph)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    mu.zero_()
    ev[0].record()
    wn.wnnc_iterate(tree, mu, **prm)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    m = mu.cpu().numpy()
    wn.wn_work_count_enable(True)
    mu2 = torch.zeros_like(mu)
    wn.wnnc_iterate(tree, mu2, **{**prm, "flags": wn.WN_FLAG_MU_ZERO})
    work = wn.wn_work_count_read()
    wn.wn_work_count_enable(False)
    kind, _ = wn.wn_tree_schedule_stats(tree)
    t0 = time.perf_counter()
    mo, _ = cl.solve(iters=40, w1=w1, w2=w2, theta=theta)
    t_oracle = time.perf_counter() - t0
    agree = float(np.mean(np.sum(m * mo, axis=1) > 0))
    pg, po = oracle.p_co(m[inl], nr[inl]), oracle.p_co(mo[inl], nr[inl])
    n = tree.n
    napp = {"A": 79, "AT": 40, "G": 40}  # traversals per solve (iteration 1's A(0) is skipped: μ⁰ = 0)
    ROWS.append(dict(w1=w1, w2=w2, theta=theta, ms_40_iters=ms, schedule=kind,
                     tests_per_query={k: work[k]["tests"] / (napp[k] * n) for k in napp},
                     far_per_query={k: work[k]["far"] / (napp[k] * n) for k in napp},
                     near_per_query={k: work[k]["near"] / (napp[k] * n) for k in napp},
                     agreement_vs_oracle=agree, p_co_gpu=pg, p_co_oracle=po, oracle_s=t_oracle,
                     oracle_threads=oracle.num_threads()))
    assert agree > 0.999, agree
    assert abs(pg - po) <= 1e-3, (pg, po)
