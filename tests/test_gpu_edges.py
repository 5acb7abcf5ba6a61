"""Edge cases of the GPU path against the oracle (through the C ABI): the degenerate and tiny clouds,
the largest and the hardest BASELINE configurations, the ABI's maximum size and the node-count limit."""
import numpy as np
import pytest

import oracle
from paper_2405_16634_b200 import synth
from test_gpu_parity import W1, W2, _check_decisions, _check_queries, _cuda

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wn():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    return wn


def test_single_point_is_degenerate(wn):
    # one point has zero extent: the §5.1.1 normalization (longest half-extent → 10/11) is undefined,
    # so both sides refuse it (reading R-degenerate)
    p = np.array([[0.3, -0.2, 0.1]], np.float32)
    with pytest.raises(wn.WnError, match="DEGENERATE"):
        wn.wn_build_tree(_cuda(p))
    with pytest.raises(Exception):
        oracle.Cloud(p)


@pytest.mark.parametrize("n", [2, 3, 5])
def test_tiny_clouds(wn, n):
    # the smallest trees: two and three points (root split into one-point leaves), five points.
    # Operators at the sources and off the cloud, and 40 iterations.
    rng = np.random.default_rng(30 + n)
    p = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    mu = rng.standard_normal((n, 3)).astype(np.float32)
    s = rng.standard_normal(n).astype(np.float32)
    q = rng.uniform(-2, 2, (50, 3)).astype(np.float32)
    w = float(np.float32(0.01))
    t = wn.wn_build_tree(_cuda(p))
    cl = oracle.Cloud(p)
    assert t.num_nodes == cl.t.num_nodes
    for theta in (2.0, float("inf")):
        _check_queries(wn.wn_eval(t, _cuda(mu), w, theta).cpu().numpy(), cl.F(mu, w, theta), None,
                       cl.abs_scale(oracle.OP_A, mu, w, theta), name=f"F n={n}")
        _check_queries(wn.wn_eval(t, _cuda(mu), w, theta, q=_cuda(q)).cpu().numpy(), cl.F(mu, w, theta, queries=q),
                       None, cl.abs_scale(oracle.OP_A, mu, w, theta, queries=q), name=f"F(q) n={n}")
        _check_queries(wn.wn_eval_grad(t, _cuda(mu), w, theta, q=_cuda(q)).cpu().numpy(),
                       cl.gradF(mu, w, theta, queries=q), None,
                       cl.abs_scale(oracle.OP_G, mu, w, theta, queries=q), name=f"gradF(q) n={n}")
        _check_queries(wn.wn_eval_adjoint(t, _cuda(s), w, theta).cpu().numpy(), cl.AT(s, w, theta), None,
                       cl.abs_scale(oracle.OP_AT, s, w, theta), name=f"AT n={n}")
    m = torch.zeros(n, 3, device="cuda")
    wn.wnnc_iterate(t, m, iters=40, flags=wn.WN_FLAG_GRAPH)
    mo, _ = cl.solve(iters=40, w1=W1, w2=W2)
    m = m.cpu().numpy()
    zero = np.linalg.norm(mo, axis=1) == 0  # no neighbour outside the cutoff: the solve stays at μ = 0
    assert np.array_equal(np.linalg.norm(m, axis=1) == 0, zero)
    if not zero.all():
        assert np.all(np.sum(m[~zero] * mo[~zero], axis=1) > 0)


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_hard_and_largest_configs_sampled(wn, cfg):
    # C4: thin plate + thin torus + 1 % outliers (200k); C5: 4M-point multi-shape scene (the largest
    # BASELINE configuration) — every operator at 2000 sampled sources against the oracle treecode
    c = synth.config(cfg)
    p = c["points"]
    n = len(p)
    rng = np.random.default_rng(40)
    mu = (synth.random_signs(c["normals"], 1006) * (4 * np.pi / n)).astype(np.float32)
    s = (0.5 - rng.uniform(0, 1, n)).astype(np.float32)
    t = wn.wn_build_tree(_cuda(p))
    cl = oracle.Cloud(p)
    idx = rng.choice(n, 2000, replace=False)
    w = float(np.float32(0.004))
    F = wn.wn_eval(t, _cuda(mu), w).cpu().numpy()
    Fo, cnt = cl.F(mu, w, qidx=idx, counters=True)
    _check_queries(F[idx], Fo, cnt, cl.abs_scale(oracle.OP_A, mu, w, qidx=idx), name=f"F {cfg}")
    _check_decisions(wn.wn_query_work(t, _cuda(mu), w, op=0).cpu().numpy()[idx], cnt, name=f"F {cfg}")
    G = wn.wn_eval_grad(t, _cuda(mu), w).cpu().numpy()
    Go, cnt = cl.gradF(mu, w, qidx=idx, counters=True)
    _check_queries(G[idx], Go, cnt, cl.abs_scale(oracle.OP_G, mu, w, qidx=idx), name=f"gradF {cfg}")
    R = wn.wn_eval_adjoint(t, _cuda(s), w).cpu().numpy()
    Ro, cnt = cl.AT(s, w, qidx=idx, counters=True)
    _check_queries(R[idx], Ro, cnt, cl.abs_scale(oracle.OP_AT, s, w, qidx=idx), name=f"AT {cfg}")


def test_maximum_size(wn):
    # the ABI's limit, N = 2^25 points on a unit sphere with outward area-weighted normals:
    # (1) Theorem 1 at c = 2 — F ≈ 1 inside, ≈ 0 outside (the far field of a 33M-point tree);
    # (2) c = ∞ at 32 near-surface queries against the oracle's dense sum, exact up to fp32 (every
    #     point, every leaf of the full-size tree);  (3) one point more is refused.
    n = 1 << 25
    p, nrm = synth.sphere(n, seed=41)
    mu = (nrm * (4 * np.pi / n)).astype(np.float32)
    t = wn.wn_build_tree(_cuda(p))
    rng = np.random.default_rng(42)
    d = rng.standard_normal((64, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = np.concatenate([rng.uniform(0.2, 0.9, 32), rng.uniform(1.1, 1.8, 32)])
    q = (d * r[:, None]).astype(np.float32)
    w = float(np.float32(1e-3))
    F = wn.wn_eval(t, _cuda(mu), w, 2.0, q=_cuda(q)).cpu().numpy()
    assert np.all(np.abs(F[:32] - 1) < 0.02) and np.all(np.abs(F[32:]) < 0.02), F
    qs = (d[:32] * rng.uniform(0.97, 1.03, 32)[:, None]).astype(np.float32)
    Fi = wn.wn_eval(t, _cuda(mu), w, float("inf"), q=_cuda(qs)).cpu().numpy()
    xn, xf = oracle.normalize(p)
    ot = oracle.Tree(xn, 1)  # the dense sum reads only the normalized points
    sc = xf[3]
    ref = ot.dense(oracle.OP_A, mu.astype(np.float64) * sc * sc, w, oracle.normalize_apply(xf, qs))
    S = ot.dense(oracle.OP_A | oracle.ABS, mu.astype(np.float64) * sc * sc, w, oracle.normalize_apply(xf, qs))
    _check_queries(Fi, ref, None, S, name="F c=inf, N=2^25")
    del t
    torch.cuda.empty_cache()
    with pytest.raises(wn.WnError, match="ARG"):
        wn.wn_build_tree(torch.zeros(n + 1, 3, device="cuda"))


def test_node_count_limit(wn):
    # 2^23 coincident pairs at D = 21: every pair is a chain of ≈ 13 nodes down to depth 21, > 2^26
    # nodes in all — beyond the traversal's 32-bit record offsets, so the build must refuse, not wrap
    rng = np.random.default_rng(43)
    c = rng.uniform(-1, 1, (1 << 23, 3)).astype(np.float32)
    p = np.repeat(c, 2, axis=0)
    with pytest.raises(wn.WnError, match="ARG"):
        wn.wn_build_tree(_cuda(p), 21)


def test_split_and_single_warp_kernels_agree(wn):
    # a 70k cloud's own points take the one-warp-per-32-queries kernel; 50k of them passed as arbitrary
    # queries take the split kernel (several warps per query group, below 60k queries): the same
    # quantities, identical per-query work counts, values within the parity tolerance of each other
    p = synth.config("C3")["points"][:70000]
    n = len(p)
    rng = np.random.default_rng(44)
    mu = (rng.standard_normal((n, 3)) * 4 * np.pi / n).astype(np.float32)
    t = wn.wn_build_tree(_cuda(p))
    idx = rng.choice(n, 50000, replace=False)
    w = float(np.float32(0.004))
    for op, ev in ((0, wn.wn_eval), (2, wn.wn_eval_grad)):
        full = ev(t, _cuda(mu), w).cpu().numpy()[idx]
        part = ev(t, _cuda(mu), w, q=_cuda(p[idx])).cpu().numpy()
        cf = wn.wn_query_work(t, _cuda(mu), w, op=op).cpu().numpy()[idx]
        cp = wn.wn_query_work(t, _cuda(mu), w, op=op, q=_cuda(p[idx])).cpu().numpy()
        np.testing.assert_array_equal(cp, cf)
        ref = full.reshape(len(idx), -1)
        err = np.linalg.norm(part.reshape(len(idx), -1) - ref, axis=1)
        assert np.all(err <= 1e-5 * np.linalg.norm(ref, axis=1) + 1e-6 * np.sqrt(np.mean(ref ** 2))), err.max()


@pytest.mark.parametrize("shape", ["planar", "collinear"])
def test_flat_clouds(wn, shape):
    # zero extent along one (planar) or two (collinear) axes: the normalization uses the longest half-extent
    # (§5.1.1), the tree degenerates to quadtree / binary splits — structure bit-exact, operators at parity
    rng = np.random.default_rng(45)
    n = 3000
    p = np.zeros((n, 3), np.float32)
    if shape == "planar":
        p[:, :2] = rng.uniform(-1, 1, (n, 2))
    else:
        p[:, 0] = rng.uniform(-1, 1, n)
    p += np.float32(0.25)
    mu = (rng.standard_normal((n, 3)) * 4 * np.pi / n).astype(np.float32)
    t = wn.wn_build_tree(_cuda(p))
    e = {k: v.cpu().numpy() for k, v in wn.wn_tree_export(t).items()}
    cl = oracle.Cloud(p)
    o = cl.t.export()
    for k in ("perm", "depth", "pb", "pe", "child_begin", "child_count"):
        np.testing.assert_array_equal(e[k], o[k], err_msg=k)
    w = float(np.float32(0.01))
    F = wn.wn_eval(t, _cuda(mu), w).cpu().numpy()
    Fo, cnt = cl.F(mu, w, counters=True)
    _check_queries(F, Fo, cnt, cl.abs_scale(oracle.OP_A, mu, w), name=f"F {shape}")
    G = wn.wn_eval_grad(t, _cuda(mu), w).cpu().numpy()
    Go, cnt = cl.gradF(mu, w, counters=True)
    _check_queries(G, Go, cnt, cl.abs_scale(oracle.OP_G, mu, w), name=f"gradF {shape}")
    m = torch.zeros(n, 3, device="cuda")
    wn.wnnc_iterate(t, m, iters=3, total_iters=40)
    assert np.isfinite(m.cpu().numpy()).all()
