"""Pins of the oracle's kernels and dense / treecode operators against what the paper and the
mathematics fix (no GPU).  Each test names the passage it pins."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import OP_A, OP_AT, OP_G
from paper_2405_16634_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
FOUR_PI = 4 * np.pi


def _two_point_tree(src, qry):
    """Tree over the single source `src` (normalized frame); dense queries at `qry`."""
    t = oracle.Tree(np.array([src], np.float32))
    return t, np.array(qry, np.float32).reshape(-1, 3)


def test_grad_phi_closed_form():
    # PAPER.md:L213 ∇Φ(y) = −y/(4π|y|^3); SPEC.md:L100 example y=(1,0,0) → (−1/(4π),0,0)
    t, q = _two_point_tree([-0.5, 0, 0], [0.5, 0, 0])
    g = [t.dense(OP_A, np.eye(3)[k][None], 1e-3, q)[0] for k in range(3)]
    np.testing.assert_allclose(g, GOLD["grad_phi_unit_x"]["value"], rtol=1e-15, atol=1e-18)
    # magnitude law |∇Φ(y)| = 1/(4π|y|^2) at |y| = 2
    t, q = _two_point_tree([-1.0, 0, 0], [1.0, 0, 0])
    g = [t.dense(OP_A, np.eye(3)[k][None], 1e-3, q)[0] for k in range(3)]
    np.testing.assert_allclose(g, GOLD["grad_phi_2x"]["value"], rtol=1e-15, atol=1e-18)


def test_hess_phi_closed_form_and_trace():
    # PAPER.md:L270 HΦ(1,0,0) = diag(2,−1,−1)/(4π);  G = −HΦ·μ
    t, q = _two_point_tree([-0.5, 0, 0], [0.5, 0, 0])
    H = -np.stack([t.dense(OP_G, np.eye(3)[k][None], 1e-3, q)[0] for k in range(3)], axis=1)
    np.testing.assert_allclose(H * FOUR_PI, np.diag(GOLD["hess_phi_unit_x"]["diag_times_4pi"]), atol=1e-14)
    rng = np.random.default_rng(0)
    for _ in range(20):
        y = rng.uniform(-0.45, 0.45, 3).astype(np.float32)
        t, q = _two_point_tree([0, 0, 0], y)
        H = -np.stack([t.dense(OP_G, np.eye(3)[k][None], 1e-4, q)[0] for k in range(3)], axis=1)
        np.testing.assert_allclose(H, H.T, rtol=0, atol=1e-12 * np.abs(H).max())       # symmetric
        assert abs(np.trace(H)) <= 1e-12 * np.abs(H).max()                            # harmonic


def test_kernel_symmetry():
    # ∇Φ odd, HΦ even: swap source and query
    rng = np.random.default_rng(1)
    for _ in range(20):
        a = rng.uniform(-0.9, 0.9, 3).astype(np.float32)
        b = rng.uniform(-0.9, 0.9, 3).astype(np.float32)
        mu = rng.standard_normal(3)
        t1, q1 = _two_point_tree(a, b)
        t2, q2 = _two_point_tree(b, a)
        assert np.isclose(t1.dense(OP_A, mu[None], 1e-4, q1)[0], -t2.dense(OP_A, mu[None], 1e-4, q2)[0], rtol=1e-14)
        np.testing.assert_allclose(t1.dense(OP_G, mu[None], 1e-4, q1), t2.dense(OP_G, mu[None], 1e-4, q2), rtol=1e-13)


def test_gradient_is_derivative_of_field():
    # ∇F(y;μ) = Σ HΦ(y−x_j)μ_j: G must be −(finite difference of F).
    rng = np.random.default_rng(2)
    src = rng.uniform(-0.8, 0.8, (64, 3)).astype(np.float32)
    mu = rng.standard_normal((64, 3))
    t = oracle.Tree(src)
    h = 2.0 ** -16
    for q0 in ([0.9375, 0.125, -0.25], [-0.5, 0.96875, 0.5]):
        q0 = np.array(q0, np.float32)
        G = t.dense(OP_G, mu, 1e-3, q0[None])[0]
        fd = []
        for k in range(3):
            e = np.zeros(3, np.float32)
            e[k] = h
            Fp = t.dense(OP_A, mu, 1e-3, (q0 + e)[None])[0]
            Fm = t.dense(OP_A, mu, 1e-3, (q0 - e)[None])[0]
            fd.append((Fp - Fm) / (2 * h))
        np.testing.assert_allclose(-G, fd, rtol=2e-6, atol=1e-9 * np.abs(G).max())


def test_smoothing_cutoff():
    # §4.4: kernels are 0 if ‖x_i − x_j‖ < w, live at ≥ w
    t, q = _two_point_tree([0, 0, 0], [0.25, 0, 0])
    mu = np.array([[1.0, 0, 0]])
    assert t.dense(OP_A, mu, 0.2500001, q)[0] == 0.0
    assert t.dense(OP_A, mu, 0.25, q)[0] != 0.0
    assert np.all(t.dense(OP_G, mu, 0.3, q) == 0.0)


def test_winding_number_indicator():
    # Theorem 1: F = 1 inside, 0 outside, with μ = σ n (Eq. L222)
    N = 20000
    p, n = synth.fibonacci_sphere(N)
    c = oracle.Cloud(p)
    mu = n * (FOUR_PI / N)
    q = np.array([[0, 0, 0], [0.3, 0.2, -0.1], [3, 0, 0], [0, -2.5, 1]], np.float32)
    F = c.F(mu, 1e-3, queries=q, dense=True)
    np.testing.assert_allclose(F[:2], 1.0, atol=1e-5)
    np.testing.assert_allclose(F[2:], 0.0, atol=1e-5)
    # off-surface ∇F → 0 (indicator is piecewise constant)
    g = c.gradF(mu, 1e-3, queries=q, dense=True)
    assert np.abs(g).max() < 1e-4


@pytest.fixture(scope="module")
def fib20k():
    N = 20000
    p, n = synth.fibonacci_sphere(N)
    c = oracle.Cloud(p)
    R = c.scale * 1.0                     # sphere radius in the normalized frame
    sig_n = FOUR_PI * R * R / N           # σ in the normalized frame
    idx = np.arange(0, N, 97)
    return c, n, R, sig_n, idx


def test_sphere_smoothed_A_closed_form(fib20k):
    # on-surface value of the smoothed field: A(σn)_i → ½ − w/(4R)  (derived from
    # PAPER.md:L222 + §4.4: dS = 2πρdρ, (x−y)·n = ρ²/(2R) over the cut-out cap)
    c, n, R, sig, idx = fib20k
    w = 0.15
    A = c.t.dense(OP_A, n * sig, w, c.xn[idx])
    # the continuum limit; the discrete cut-out cap adds ±1-point noise (~4e-4 per query)
    assert abs(A.mean() / (0.5 - w / (4 * R)) - 1) < 1e-3
    np.testing.assert_allclose(A, 0.5 - w / (4 * R), rtol=3e-3)


def test_sphere_smoothed_G_closed_form(fib20k):
    # −∇F at surface points: G(σn)_i → (1/(2w) − w/(8R²)) n_i, tangential part → 0
    c, n, R, sig, idx = fib20k
    w = 0.15
    G = c.t.dense(OP_G, n * sig, w, c.xn[idx])
    nn = n[idx]
    gn = np.sum(G * nn, axis=1)
    assert abs(gn.mean() / (1 / (2 * w) - w / (8 * R * R)) - 1) < 1e-2
    np.testing.assert_allclose(gn, 1 / (2 * w) - w / (8 * R * R), rtol=3e-2)
    tang = np.linalg.norm(G - gn[:, None] * nn, axis=1)
    assert tang.mean() < 1e-3 * gn.mean() and tang.max() < 3e-3 * gn.min()


def test_sphere_smoothed_AT_closed_form(fib20k):
    # Aᵀ(1)_j = Σ_i ∇Φ(x_i − x_j) → (N/(4πR²))·(2R − w)/(4R)·n_j
    c, n, R, sig, idx = fib20k
    w = 0.15
    N = len(n)
    AT = c.t.dense(OP_AT, np.ones(N), w)[idx]
    expect = N / (FOUR_PI * R * R) * (2 * R - w) / (4 * R)
    atn = np.sum(AT * n[idx], axis=1)
    assert abs(atn.mean() / expect - 1) < 1e-3
    np.testing.assert_allclose(atn, expect, rtol=1e-2)


def test_dense_adjoint_and_symmetry():
    # ⟨Aμ, s⟩ = ⟨μ, Aᵀs⟩ and ⟨Gμ, ν⟩ = ⟨μ, Gν⟩
    rng = np.random.default_rng(3)
    for trial in range(5):
        p = rng.uniform(-1, 1, (500, 3)).astype(np.float32)
        c = oracle.Cloud(p)
        mu, nu = rng.standard_normal((500, 3)), rng.standard_normal((500, 3))
        s = rng.standard_normal(500)
        w = 0.05
        lhs = np.dot(c.t.dense(OP_A, mu, w), s)
        rhs = np.sum(mu * c.t.dense(OP_AT, s, w))
        assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1)
        g1 = np.sum(c.t.dense(OP_G, mu, w) * nu)
        g2 = np.sum(mu * c.t.dense(OP_G, nu, w))
        assert abs(g1 - g2) <= 1e-12 * max(abs(g1), 1)


def _relL2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_treecode_infinite_c_is_dense():
    # c = ∞ ⇒ Alg. 4 never takes a representative ⇒ the dense sum
    rng = np.random.default_rng(4)
    p = rng.uniform(-1, 1, (2000, 3)).astype(np.float32)
    c = oracle.Cloud(p)
    mu, s = rng.standard_normal((2000, 3)), rng.standard_normal(2000)
    w = 0.002
    for op, nu in ((OP_A, mu), (OP_G, mu), (OP_AT, s)):
        d = c.t.dense(op, nu, w)
        t = c.t.tree(op, nu, w, theta=np.inf)
        assert _relL2(t, d) <= 1e-12


def test_treecode_converges_in_c():
    # SPEC volume instance: error falls as c grows; at c=2 within the literal
    # treecode's own accuracy (A 2.5e-2, Aᵀ 2.7e-2, G 3.5e-3)
    rng = np.random.default_rng(5)
    p = rng.uniform(-1, 1, (5000, 3)).astype(np.float32)
    c = oracle.Cloud(p)
    mu = rng.standard_normal((5000, 3))
    mu /= np.linalg.norm(mu, axis=1, keepdims=True)
    s = rng.standard_normal(5000)
    w = 0.002
    bound = {OP_A: 5e-2, OP_AT: 5e-2, OP_G: 2e-2}
    for op, nu in ((OP_A, mu), (OP_G, mu), (OP_AT, s)):
        d = c.t.dense(op, nu, w)
        errs = [_relL2(c.t.tree(op, nu, w, theta=th), d) for th in (1, 2, 4, 8)]
        assert all(errs[i + 1] < errs[i] for i in range(3)), errs
        assert errs[1] <= bound[op], errs
        assert errs[3] < errs[1] / 8


def test_single_point_node_far_equals_near():
    # a one-point node: rep = the point, ν_B = ν_j ⇒ far and leaf branches give the same term
    # (SURVEY a-notes).  Checked by varying c on an instance where only one-point leaves change branch.
    p = np.array([[0.9, 0.9, 0.9], [-0.9, -0.9, -0.9], [0.9, -0.9, 0.0]], np.float32)
    t = oracle.Tree(p)
    mu = np.array([[1.0, 2, 3], [0.5, -1, 2], [-1, 0.25, 1]])
    vals, fars = [], []
    for th in (1.6, 2.2, 3.0, np.inf):
        v, cnt = t.tree(OP_A, mu, 1e-3, theta=th, counters=True)
        assert np.all(cnt[:, 0] == 4)           # root opened, 3 one-point children tested
        vals.append(v)
        fars.append(cnt[:, 1].sum())
    assert fars[0] > 0 and fars[-1] == 0        # the one-point leaves did switch branch
    for v in vals[1:]:
        np.testing.assert_allclose(v, vals[0], rtol=1e-14)


def test_transpose_mode_exact_adjoint():
    # north-star adjoint: exact transpose of treecode A at frozen geometry g(μ)
    rng = np.random.default_rng(6)
    p, n = synth.sphere(3000, seed=7)
    c = oracle.Cloud(p)
    mu = n * 0.004 * (1 + 0.3 * rng.standard_normal((3000, 1)))
    v = rng.standard_normal((3000, 3))
    s = rng.standard_normal(3000)
    w = 0.004
    Tv = c.t.A_frozen(mu, v, w)
    TTs = c.t.AT_transpose(mu, s, w)
    lhs, rhs = np.dot(Tv, s), np.sum(v * TTs)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    # frozen-geometry A applied to μ itself is the ordinary treecode A(μ)
    np.testing.assert_allclose(c.t.A_frozen(mu, mu, w), c.t.tree(OP_A, mu, w), rtol=1e-12, atol=1e-15)
