"""GPU ↔ oracle parity of the path bench.py times, at the BASELINE configs' full sizes (needs a B200).

bench.py runs `wnnc_iterate` with WN_FLAG_GRAPH | WN_FLAG_MU_ZERO on clouds far above the small-cloud
threshold: the one-warp `trav_kernel` with its fused epilogues (s = ½ − Aμ, r = Aᵀs, Σ(Ar)², rescale), the
query schedule the tree chose (k-d on C3, Hilbert heaviest-first on C4) and the captured CUDA graph.  These
tests compare exactly that path with the fp64 oracle (oracle/), element by element from identical inputs
(one iteration ≤ 1e-3 relative per point for ≥ 99.9 % of the points, E to 1e-6,
α to 1e-3) and after the whole 40-iteration solve (orientation agreement with the oracle > 99.9 %, BASELINE
north_star; P_co against the analytic normals, §5.1.4).
"""
import numpy as np
import pytest

import oracle
from paper_2405_16634_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

W1, W2 = float(np.float32(0.002)), float(np.float32(0.016))
BENCH_FLAGS = None  # set from the binding (WN_FLAG_GRAPH | WN_FLAG_MU_ZERO)


@pytest.fixture(scope="module")
def wn():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    global BENCH_FLAGS
    BENCH_FLAGS = wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO
    return wn


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


_CACHE = {}


def _c3(wn):
    """The headline cloud, its GPU tree (the bench's launch configuration) and its oracle."""
    if "C3" not in _CACHE:
        cfg = synth.config("C3")
        _CACHE["C3"] = (cfg, wn.wn_build_tree(_cuda(cfg["points"])), oracle.Cloud(cfg["points"]))
    return _CACHE["C3"]


def _per_point(m_gpu, m_ora, name):
    err = np.linalg.norm(m_gpu - m_ora, axis=1) / np.maximum(np.linalg.norm(m_ora, axis=1), 1e-300)
    frac = float(np.mean(err < 1e-3))
    assert frac >= 0.999, f"{name}: {frac:.5f} of points within 1e-3 (percentiles 50/99/100: " \
                          f"{np.percentile(err, [50, 99, 100])})"
    return frac


def test_c3_bench_path_is_the_one_warp_kd_path(wn):
    cfg, t, _ = _c3(wn)
    kind, _ = wn.wn_tree_schedule_stats(t)
    assert kind == "kd", "C3 must take the k-d query schedule (the configuration bench.py times)"
    assert t.n > 60000  # above the small-cloud threshold: trav_kernel, not trav_split_kernel


def test_c3_first_iteration_bench_flags(wn):
    # iteration 1 of 40 from μ = 0 (w = w2): r = Aᵀ(½) (EPI_R), Σ(Ar)² (EPI_SQ), α, μ' = α r, rescale
    cfg, t, cl = _c3(wn)
    mu = torch.zeros(t.n, 3, device="cuda")
    st = wn.wnnc_iterate(t, mu, stats=True, iters=1, total_iters=40, flags=BENCH_FLAGS)
    mo, so = cl.solve(iters=1, total_iters=40, w1=W1, w2=W2)
    _per_point(mu.cpu().numpy(), mo, "C3 iteration 1")
    assert st[0]["E"] == pytest.approx(so[0, 0], rel=1e-6)
    assert st[0]["alpha"] == pytest.approx(so[0, 1], rel=1e-3)
    assert st[0]["width"] == so[0, 4]
    _CACHE["C3_mu1"] = mo


def test_c3_second_iteration_from_oracle_state(wn):
    # iteration 2 from the oracle's μ¹ (rounded to fp32 on both sides): every fused epilogue of the bench
    # path from identical inputs — s = ½ − Aμ (EPI_S), r, Σ(Ar)², μ' and the rescale (EPI_RESCALE)
    cfg, t, cl = _c3(wn)
    mo1 = _CACHE.get("C3_mu1")
    if mo1 is None:
        mo1, _ = cl.solve(iters=1, total_iters=40, w1=W1, w2=W2)
    mu1 = mo1.astype(np.float32)
    mu = _cuda(mu1)
    st = wn.wnnc_iterate(t, mu, stats=True, iters=1, first_iter=2, total_iters=40, flags=wn.WN_FLAG_GRAPH)
    mo2, so = cl.solve(mu0=mu1.astype(np.float64) * cl.scale ** 2, iters=1, first_iter=2, total_iters=40,
                       w1=W1, w2=W2)
    _per_point(mu.cpu().numpy(), mo2, "C3 iteration 2")
    assert st[0]["E"] == pytest.approx(so[0, 0], rel=1e-6)
    assert st[0]["alpha"] == pytest.approx(so[0, 1], rel=1e-3)
    assert st[0]["rr"] == pytest.approx(so[0, 2], rel=1e-4)


def test_c3_forty_iterations_orientation(wn):
    cfg, t, cl = _c3(wn)
    mu = torch.zeros(t.n, 3, device="cuda")
    wn.wnnc_iterate(t, mu, iters=40, flags=BENCH_FLAGS)
    m = mu.cpu().numpy()
    mo, _ = cl.solve(iters=40, w1=W1, w2=W2)
    agree = float(np.mean(np.sum(m * mo, axis=1) > 0))
    assert agree > 0.999, agree
    pg, po = oracle.p_co(m, cfg["normals"]), oracle.p_co(mo, cfg["normals"])
    assert pg >= 0.999 and abs(pg - po) <= 1e-3, (pg, po)


def test_c4_forty_iterations_orientation(wn):
    # thin features + 1 % outliers (the stress config; Hilbert schedule, heaviest blocks first)
    cfg = synth.config("C4")
    p, nr, inl = cfg["points"], cfg["normals"], cfg["inlier"]
    t = wn.wn_build_tree(_cuda(p))
    kind, _ = wn.wn_tree_schedule_stats(t)
    assert kind == "hilbert", "C4 keeps the Hilbert schedule (DESIGN.md §Query schedule)"
    mu = torch.zeros(t.n, 3, device="cuda")
    wn.wnnc_iterate(t, mu, iters=40, flags=BENCH_FLAGS)
    m = mu.cpu().numpy()
    mo, _ = oracle.Cloud(p).solve(iters=40, w1=W1, w2=W2)
    agree = float(np.mean(np.sum(m * mo, axis=1) > 0))
    assert agree > 0.999, agree
    pg, po = oracle.p_co(m[inl], nr[inl]), oracle.p_co(mo[inl], nr[inl])
    assert pg >= 0.999 and abs(pg - po) <= 1e-3, (pg, po)


def test_transpose_adjoint_kd_path(wn):
    # exact-transpose Aᵀ above the k-d threshold (4096 points): scatter in the k-d query order
    cfg = synth.config("C2", n=20000)
    p, nr = cfg["points"], cfg["normals"]
    rng = np.random.default_rng(21)
    mu = (nr * (4 * np.pi / len(p)) * (1 + 0.2 * rng.standard_normal((len(p), 1)))).astype(np.float32)
    s = rng.standard_normal(len(p)).astype(np.float32)
    t = wn.wn_build_tree(_cuda(p))
    kind, _ = wn.wn_tree_schedule_stats(t)
    assert kind == "kd"
    w = float(np.float32(0.005))
    g = wn.wn_eval_adjoint(t, _cuda(s), w, 2.0, mode=wn.WN_ADJ_TRANSPOSE, mu_geom=_cuda(mu)).cpu().numpy()
    ref = oracle.Cloud(p).AT_transpose(s, mu, w)
    err = np.linalg.norm(g - ref, axis=1)
    mag = np.linalg.norm(ref, axis=1)
    rms = np.sqrt(np.mean(mag ** 2))
    assert np.all(err <= np.maximum(1e-4 * mag, 1e-4 * 1e-3 * rms)), np.max(err / np.maximum(mag, 1e-3 * rms))


def test_transpose_solve_kd_graph(wn):
    # 40 transpose-mode iterations (k-d scatter path, CUDA graph replayed twice) vs the oracle's
    cfg = synth.config("C2")
    p = cfg["points"]
    t = wn.wn_build_tree(_cuda(p))
    outs = []
    for _ in range(2):
        mu = torch.zeros(t.n, 3, device="cuda")
        wn.wnnc_iterate(t, mu, iters=40, adjoint_mode=wn.WN_ADJ_TRANSPOSE, flags=BENCH_FLAGS)
        outs.append(mu.cpu().numpy())
    # graph replay reproduces the trajectory up to the fp64 atomics' order (transpose.cu): same orientations
    assert np.mean(np.sum(outs[0] * outs[1], axis=1) > 0) > 0.9999
    mo, _ = oracle.Cloud(p).solve(iters=40, w1=W1, w2=W2, mode="transpose")
    agree = float(np.mean(np.sum(outs[0] * mo, axis=1) > 0))
    assert agree > 0.999, agree


def test_grid_field_full_size_sampled(wn):
    # row f1 at scale: F and ∇F on a 128³ grid around the C3 cloud (2.1 M arbitrary queries: the one-warp
    # kernel in the queries' Hilbert order), oracle on 3000 sampled grid points
    cfg, t, cl = _c3(wn)
    n = t.n
    mu = (cfg["normals"] * (4 * np.pi / n)).astype(np.float32)
    lo, hi = cfg["points"].min(0), cfg["points"].max(0)
    c, h = (lo + hi) / 2, (hi - lo) / 2 * 1.1
    ax = [np.linspace(c[k] - h[k], c[k] + h[k], 128, dtype=np.float32) for k in range(3)]
    q = np.stack(np.meshgrid(*ax, indexing="ij"), -1).reshape(-1, 3)
    w = W1
    F = wn.wn_eval(t, _cuda(mu), w, 2.0, q=_cuda(q)).cpu().numpy()
    idx = np.random.default_rng(22).choice(len(q), 3000, replace=False)
    Fo, cnt = cl.F(mu, w, 2.0, queries=q[idx], counters=True)
    S = cl.abs_scale(oracle.OP_A, mu, w, queries=q[idx])
    err = np.abs(F[idx] - Fo)
    assert np.all(err <= np.maximum(1e-4 * np.abs(Fo), 2e-6 * S)), np.max(err / np.maximum(np.abs(Fo), 1e-30))
    G = wn.wn_eval_grad(t, _cuda(mu), w, 2.0, q=_cuda(q)).cpu().numpy()[idx]
    Go = cl.gradF(mu, w, 2.0, queries=q[idx])
    SG = cl.abs_scale(oracle.OP_G, mu, w, queries=q[idx])
    eg = np.linalg.norm(G - Go, axis=1)
    assert np.all(eg <= np.maximum(1e-4 * np.linalg.norm(Go, axis=1), 2e-6 * SG))
