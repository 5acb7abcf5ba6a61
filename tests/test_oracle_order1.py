"""Pins of the oracle's first-order far field (the paper itself uses the order-0
representative term of Alg. 4, and points to expansions via Barill et al., L409).

A far node B with sources x_j = x_B + d_j contributes Σ_j f(x_j) (f = op's kernel times ν_j); the
first-order far field adds Σ_j ∇f(x_B)·d_j to the order-0 term f(x_B)·ν_B.  What fixes it without
retyping the formula:
  * Taylor's theorem: with sources at distance R, the order-0 error falls like R^-(k+1) and the
    order-1 error like R^-(k+2) (k = 2 for A and Aᵀ, 3 for G) — a dropped term, a wrong sign or a
    wrong factor leaves the order-1 error at the order-0 rate;
  * a one-point node has d_j = 0, so when only one-point nodes are far both orders agree exactly;
  * c = ∞ uses no far node at all (= the dense sum);
  * on a real cloud with a random attribute, the first-order term removes most of the far-field error.
"""
import numpy as np
import pytest

import oracle
from oracle import OP_A, OP_AT, OP_G
from paper_2405_16634_b200 import synth

KDEC = {OP_A: 2, OP_AT: 2, OP_G: 3}


def _slope(R, e):
    return np.polyfit(np.log(R), np.log(e), 1)[0]


@pytest.mark.parametrize("op", [OP_A, OP_AT, OP_G])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_far_field_decay_rates(op, seed):
    rng = np.random.default_rng(seed)
    xn = (rng.uniform(-0.4, 0.4, (5, 3))).astype(np.float32)
    t = oracle.Tree(xn)
    if op == OP_AT:
        nu = rng.standard_normal(5)
        nu[:2] = np.abs(nu[:2])
        nu[2:4] = -np.abs(nu[2:4])  # mixed signs: Σ s_j d_j ≠ 0 about the |s|-weighted rep
    else:
        nu = rng.standard_normal((5, 3))
    dirn = rng.standard_normal(3)
    dirn /= np.linalg.norm(dirn)
    R = np.array([8.0, 16.0, 32.0, 64.0])
    e0, e1 = [], []
    for r in R:
        q = (r * dirn)[None].astype(np.float32)
        ref = t.dense(op, nu, 1e-9, queries=q)
        e0.append(np.abs(t.tree(op, nu, 1e-9, 1.0, queries=q, order=0) - ref).max())
        e1.append(np.abs(t.tree(op, nu, 1e-9, 1.0, queries=q, order=1) - ref).max())
    k = KDEC[op]
    assert abs(_slope(R, e0) + (k + 1)) < 0.3, (_slope(R, e0), k)
    assert abs(_slope(R, e1) + (k + 2)) < 0.3, (_slope(R, e1), k)
    assert e1[-1] < 0.1 * e0[-1]


@pytest.mark.parametrize("op", [OP_A, OP_AT, OP_G])
def test_one_point_nodes_have_no_first_order_term(op):
    # two points in different root children; queries at distances where the root is opened but
    # both one-point children are far: the two orders must agree to the last bit
    xn = np.array([[-0.5, -0.5, -0.5], [0.5, 0.5, 0.5]], np.float32)
    t = oracle.Tree(xn)
    rng = np.random.default_rng(4)
    nu = rng.standard_normal(2) if op == OP_AT else rng.standard_normal((2, 3))
    q = np.array([[2.6, -0.5, -0.5], [-0.5, 2.6, 0.5]], np.float32)  # < c·2 = 4 from the root rep, > 2 from each point
    o0, c0 = t.tree(op, nu, 1e-9, 2.0, queries=q, counters=True, order=0)
    o1 = t.tree(op, nu, 1e-9, 2.0, queries=q, order=1)
    assert np.all(c0[:, 0] == 3) and np.all(c0[:, 1] == 2)  # root opened, both children far
    np.testing.assert_array_equal(o0, o1)


@pytest.mark.parametrize("op", [OP_A, OP_AT, OP_G])
def test_infinite_c_is_dense(op):
    xn, _ = oracle.normalize(synth.sphere(400, seed=5)[0])
    t = oracle.Tree(xn)
    rng = np.random.default_rng(6)
    nu = rng.standard_normal(400) if op == OP_AT else rng.standard_normal((400, 3))
    np.testing.assert_allclose(t.tree(op, nu, 0.01, np.inf, order=1), t.dense(op, nu, 0.01), rtol=1e-12,
                               atol=1e-12)


@pytest.mark.parametrize("op", [OP_A, OP_AT, OP_G])
def test_first_order_reduces_far_field_error(op):
    # a random attribute on a real cloud (C2 torus, 12k points), cutoff far below the node sizes:
    # the order-1 error is well below the order-0 error at the same c (measured ≈ 4×)
    cl = oracle.Cloud(synth.config("C2")["points"][:12000])
    rng = np.random.default_rng(3)
    n = cl.t.n
    nu = rng.standard_normal(n) if op == OP_AT else rng.standard_normal((n, 3)) * 4 * np.pi / n
    ref = cl.t.dense(op, nu, 1e-6)
    sc = np.sqrt(np.mean(ref ** 2))
    e0 = np.sqrt(np.mean((cl.t.tree(op, nu, 1e-6, 2.0, order=0) - ref) ** 2)) / sc
    e1 = np.sqrt(np.mean((cl.t.tree(op, nu, 1e-6, 2.0, order=1) - ref) ** 2)) / sc
    assert e1 < 0.5 * e0, (e0, e1)
