"""First-order far field on the GPU (`wn_tree_set_far_order(t, 1)`) against the
oracle's order-1 treecode (tests/test_oracle_order1.py pins it), through the C ABI.  Same protocol as
tests/test_gpu_parity.py: per-query |gpu − oracle| ≤ max(1e-4·|ref|, 2e-6·S), identical opening
decisions (the order does not change them), 40-iteration orientation agreement ≥ 99.9 %."""
import numpy as np
import pytest

import oracle
from paper_2405_16634_b200 import synth
from test_gpu_parity import CLOUDS, W1, W2, _check_decisions, _check_queries, _cuda

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wn():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    return wn


@pytest.mark.parametrize("name", ["sphere2k", "torus50k", "clustered"])
@pytest.mark.parametrize("op,w", [("F", 0.016), ("gradF", 0.002), ("AT", 0.009)])
@pytest.mark.parametrize("theta", [2.0, 1.0])
def test_order1_operators_at_sources(wn, name, op, w, theta):
    p = CLOUDS[name]()
    n = len(p)
    rng = np.random.default_rng(22)
    mu = rng.standard_normal((n, 3)).astype(np.float32) * np.float32(4 * np.pi / n)
    a = rng.uniform(0.5, 2, n).astype(np.float32)
    s = (0.5 - rng.uniform(0, 1, n)).astype(np.float32)
    w = float(np.float32(w))
    t = wn.wn_build_tree(_cuda(p))
    wn.wn_tree_set_far_order(t, 1)
    cl = oracle.Cloud(p)
    if op == "F":
        g = wn.wn_eval(t, _cuda(mu), w, theta, a=_cuda(a)).cpu().numpy()
        ref, cnt = cl.F(mu, w, theta, a=a, counters=True, order=1)
        S = cl.abs_scale(oracle.OP_A, mu, w, theta, a=a, order=1)
        _check_decisions(wn.wn_query_work(t, _cuda(mu * a[:, None]), w, theta, op=0).cpu().numpy(), cnt)
    elif op == "gradF":
        g = wn.wn_eval_grad(t, _cuda(mu), w, theta).cpu().numpy()
        ref, cnt = cl.gradF(mu, w, theta, counters=True, order=1)
        S = cl.abs_scale(oracle.OP_G, mu, w, theta, order=1)
    else:
        g = wn.wn_eval_adjoint(t, _cuda(s), w, theta).cpu().numpy()
        ref, cnt = cl.AT(s, w, theta, counters=True, order=1)
        S = cl.abs_scale(oracle.OP_AT, s, w, theta, order=1)
    _check_queries(g, ref, cnt, S, name=f"{name}/{op}/order1")


def test_order1_at_arbitrary_queries(wn):
    p, n_ = synth.fibonacci_sphere(20000)
    mu = (n_ * (4 * np.pi / 20000)).astype(np.float32)
    g = np.linspace(-1.6, 1.6, 19, dtype=np.float32)
    q = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3).astype(np.float32)
    t = wn.wn_build_tree(_cuda(p))
    wn.wn_tree_set_far_order(t, 1)
    cl = oracle.Cloud(p)
    w = float(np.float32(0.002))
    F = wn.wn_eval(t, _cuda(mu), w, 2.0, q=_cuda(q)).cpu().numpy()
    Fo, cnt = cl.F(mu, w, 2.0, queries=q, counters=True, order=1)
    _check_queries(F, Fo, cnt, cl.abs_scale(oracle.OP_A, mu, w, queries=q, order=1), name="F(q)/order1")
    G = wn.wn_eval_grad(t, _cuda(mu), w, 2.0, q=_cuda(q)).cpu().numpy()
    Go, cnt = cl.gradF(mu, w, 2.0, queries=q, counters=True, order=1)
    _check_queries(G, Go, cnt, cl.abs_scale(oracle.OP_G, mu, w, queries=q, order=1), name="gradF(q)/order1")


def test_order1_reduces_far_field_error(wn):
    # the GPU's order-1 error against the dense sum (oracle definition) is well below its order-0 error
    p = CLOUDS["torus50k"]()[:12000]
    rng = np.random.default_rng(3)
    n = len(p)
    mu = (rng.standard_normal((n, 3)) * 4 * np.pi / n).astype(np.float32)
    cl = oracle.Cloud(p)
    w = 1e-5
    ref = cl.F(mu, w, dense=True)
    t = wn.wn_build_tree(_cuda(p))
    e = []
    for order in (0, 1):
        wn.wn_tree_set_far_order(t, order)
        g = wn.wn_eval(t, _cuda(mu), w, 2.0).cpu().numpy()
        e.append(np.sqrt(np.mean((g - ref) ** 2) / np.mean(ref ** 2)))
    assert e[1] < 0.5 * e[0], e


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_order1_forty_iterations_orientation(wn, cfg):
    c = synth.config(cfg)
    p = c["points"]
    t = wn.wn_build_tree(_cuda(p))
    wn.wn_tree_set_far_order(t, 1)
    mu = torch.zeros(len(p), 3, device="cuda")
    wn.wnnc_iterate(t, mu, iters=40, flags=wn.WN_FLAG_GRAPH)
    m = mu.cpu().numpy()
    mo, _ = oracle.Cloud(p).solve(iters=40, w1=W1, w2=W2, order=1)
    assert np.mean(np.sum(m * mo, axis=1) > 0) >= 0.999
    if cfg == "C1":
        assert oracle.p_co(m, c["normals"]) >= 0.999


def test_order_switch_and_graph_cache(wn):
    # the cached iteration graph is keyed on the order: 0 → 1 → 0 reproduces the order-0 trajectory
    p = CLOUDS["sphere2k"]()
    t = wn.wn_build_tree(_cuda(p))
    out = []
    for order in (0, 1, 0):
        wn.wn_tree_set_far_order(t, order)
        mu = torch.zeros(len(p), 3, device="cuda")
        wn.wnnc_iterate(t, mu, iters=3, total_iters=40, flags=wn.WN_FLAG_GRAPH)
        out.append(mu.cpu().numpy())
    np.testing.assert_array_equal(out[0], out[2])
    assert not np.array_equal(out[0], out[1])


def test_order1_errors(wn):
    p = CLOUDS["sphere2k"]()
    t = wn.wn_build_tree(_cuda(p))
    with pytest.raises(wn.WnError, match="ARG"):
        wn.wn_tree_set_far_order(t, 2)
    wn.wn_tree_set_far_order(t, 1)
    mu = torch.zeros(len(p), 3, device="cuda")
    with pytest.raises(wn.WnError, match="ARG"):
        wn.wnnc_iterate(t, mu, iters=1, adjoint_mode=wn.WN_ADJ_TRANSPOSE)
    with pytest.raises(wn.WnError, match="ARG"):
        wn.wn_eval_adjoint(t, torch.zeros(len(p), device="cuda"), 0.01, mode=wn.WN_ADJ_TRANSPOSE, mu_geom=mu)
