"""Pins of the oracle's fast multipole method (the paper's future work, PAPER.md:L1034
§6.3, L409 — not the paper's method) against what fixes it independently of its own code:

* θ_f → 0 makes every cell pair direct: the FMM must then be the dense O(N²) definition (the dense
  operators are pinned by closed forms in test_oracle_kernels.py) — this pins the direct part, the cutoff
  and the sign conventions of V, −∇V for charges and dipoles;
* at a fixed separation θ_f = 0.5 the error against the dense sums must fall geometrically with the
  expansion degree p (a dropped term, a wrong shift sign or factorial in P2M / M2M / M2L / L2L / L2P
  breaks the decay);
* the smoothed on-surface closed form A(σn)_i → ½ − w/(4R) on a dense sphere (as for the dense operator);
* Aᵀ is the adjoint of A up to the expansion error.
"""
import numpy as np
import pytest

import oracle
from oracle import OP_A, OP_AT, OP_G
from paper_2405_16634_b200 import synth


@pytest.fixture(scope="module")
def cloud():
    p, nr = synth.sphere(3000, seed=5)
    xn, _ = oracle.normalize(p)
    t = oracle.Tree(xn)
    rng = np.random.default_rng(1)
    return t, rng.standard_normal((3000, 3)), rng.standard_normal(3000)


@pytest.mark.parametrize("op", [OP_A, OP_G, OP_AT])
def test_fmm_all_direct_is_dense(cloud, op):
    t, mu, s = cloud
    nu = s if op == OP_AT else mu
    w = 0.005
    f, cnt = t.fmm(op, nu, w, p=2, theta=1e-9, counters=True)
    d = t.dense(op, nu, w)
    assert cnt[0] == 0  # no M2L at all
    np.testing.assert_allclose(f, d, rtol=1e-12, atol=1e-12 * np.abs(d).max())


@pytest.mark.parametrize("op", [OP_A, OP_G, OP_AT])
def test_fmm_error_decays_with_degree(cloud, op):
    t, mu, s = cloud
    nu = s if op == OP_AT else mu
    w = 0.005
    d = t.dense(op, nu, w)
    errs = []
    for p in (1, 2, 3, 4, 5, 6):
        f, cnt = t.fmm(op, nu, w, p=p, theta=0.5, counters=True)
        assert cnt[0] > 0
        errs.append(np.linalg.norm(f - d) / np.linalg.norm(d))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 2e-6 and errs[-1] / errs[1] < 0.05, errs


def test_fmm_smoothed_on_surface_closed_form():
    # A(σn)_i → ½ − w/(4R) at the points of a dense unit sphere (E1 gave 0.46260 vs 0.46250)
    n = 20000
    p, nr = synth.fibonacci_sphere(n)
    xn, xf = oracle.normalize(p)
    t = oracle.Tree(xn)
    R = float(xf[3])  # the unit sphere's radius in the normalized frame
    sigma = 4 * np.pi * R * R / n
    w = 0.15 * R
    a = t.fmm(OP_A, nr * sigma, w, p=4, theta=0.5)
    assert abs(np.median(a) - (0.5 - w / (4 * R))) < 1e-3


def test_fmm_adjoint_up_to_expansion_error(cloud):
    t, mu, s = cloud
    w = 0.005
    lhs = float(np.dot(t.fmm(OP_A, mu, w, p=6, theta=0.5), s))
    rhs = float(np.sum(mu * t.fmm(OP_AT, s, w, p=6, theta=0.5)))
    assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + abs(rhs))


def test_fmm_solve_is_the_dense_solve():
    # Alg. 3 with FMM operators (p = 4, θ_f = 0.5) follows the dense-operator solve closely (the FMM's error
    # is ~1e-5 per operator), much closer than the paper's c = 2 treecode does (~2 %)
    c = synth.config("C1")
    cl = oracle.Cloud(c["points"])
    w1, w2 = float(np.float32(0.002)), float(np.float32(0.016))
    mf, _ = cl.solve(iters=40, w1=w1, w2=w2, backend="fmm", fmm=(4, 0.5, 32))
    md, _ = cl.solve(iters=40, w1=w1, w2=w2, backend="dense")
    mt, _ = cl.solve(iters=40, w1=w1, w2=w2)
    df = np.linalg.norm(mf - md) / np.linalg.norm(md)
    dt = np.linalg.norm(mt - md) / np.linalg.norm(md)
    assert df < 5e-3 and df < 0.1 * dt, (df, dt)
    assert np.all(np.sum(mf * md, axis=1) > 0)
    assert oracle.p_co(mf, c["normals"]) == 1.0
