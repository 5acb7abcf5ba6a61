"""Pins of the oracle's normalization, Morton keys, octree and representatives (no GPU)."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2405_16634_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_normalize_spec_example():
    # PAPER.md:L419 "fit into the cube [−1,1]^3 with a margin of 1/11"
    g = GOLD["normalize_two_points"]
    xn, xf = oracle.normalize(np.array(g["raw"], np.float32))
    np.testing.assert_allclose(xn, np.array(g["xn"], np.float32), rtol=0, atol=0)
    assert abs(xf[3] - g["scale"]) < 1e-15            # input → normalized multiplier 20/121
    # idempotence: normalizing a normalized cloud is (almost) the identity
    p, _ = synth.sphere(1000, seed=3, R=5, center=(100, 100, 100))
    xn, xf = oracle.normalize(p)
    assert np.abs(xn).max() <= 10 / 11 + 1e-6
    xn2, xf2 = oracle.normalize(xn)
    assert abs(xf2[3] - 1) < 1e-6 and np.abs(xf2[:3]).max() < 1e-6
    # round trip to the input frame within fp32 rounding of the normalized coords
    back = xn.astype(np.float64) / xf[3] + xf[:3]
    assert np.abs(back - p).max() < 5 * 2 ** -24 * 5 * 11 / 10 + 1e-4


def test_normalize_errors():
    with pytest.raises(oracle.OracleError, match="empty"):
        oracle.normalize(np.zeros((0, 3), np.float32))
    with pytest.raises(oracle.OracleError, match="non-finite"):
        oracle.normalize(np.array([[0, 0, 0], [np.nan, 0, 0]], np.float32))
    with pytest.raises(oracle.OracleError, match="degenerate"):
        oracle.normalize(np.ones((5, 3), np.float32))


def _cell_of_prefix(key, D, level):
    """Decode the level-`level` prefix of a Morton key into integer cell coordinates."""
    ix = iy = iz = 0
    for l in range(1, level + 1):
        d = (int(key) >> (3 * (D - l))) & 7
        ix, iy, iz = 2 * ix + (d >> 2), 2 * iy + ((d >> 1) & 1), 2 * iz + (d & 1)
    return ix, iy, iz


def test_keys_locate_cells():
    # the level-l prefix of a point's key names the depth-l cell of [−1,1]^3 that contains it
    rng = np.random.default_rng(0)
    xn = rng.uniform(-10 / 11, 10 / 11, (300, 3)).astype(np.float32)
    D = 15
    k = oracle.keys(xn, D)
    for i in range(300):
        for level in (1, 4, 9, 15):
            cell = np.array(_cell_of_prefix(k[i], D, level))
            w = 2.0 / 2 ** level
            lo = -1 + cell * w
            assert np.all(lo <= xn[i]) and np.all(xn[i] < lo + w)


def _bruteforce_tree(keys, D):
    """Independent construction: BFS over groups of equal key prefixes (not recursive partition)."""
    order = np.lexsort((np.arange(len(keys)), keys))
    sk = keys[order]
    nodes = [(0, 0, len(keys))]            # (depth, pb, pe) in Morton positions
    out, head = [], 0
    kids = {}
    while head < len(nodes):
        d, pb, pe = nodes[head]
        out.append((d, pb, pe))
        ch = []
        if pe - pb > 1 and d < D:
            pref = [int(x) >> (3 * (D - d - 1)) for x in sk[pb:pe]]
            s = pb
            for i in range(pb + 1, pe + 1):
                if i == pe or pref[i - pb] != pref[s - pb]:
                    ch.append(len(nodes))
                    nodes.append((d + 1, s, i))
                    s = i
        kids[head] = ch
        head += 1
    cb = np.array([kids[i][0] if kids[i] else -1 for i in range(len(out))])
    cc = np.array([len(kids[i]) for i in range(len(out))])
    o = np.array(out)
    return order, o[:, 0], o[:, 1], o[:, 2], cb, cc


@pytest.mark.parametrize("case", ["uniform", "sphere", "clustered"])
def test_tree_matches_bruteforce(case):
    # stop at one point or depth D; BFS layout, children in octant-digit order
    rng = np.random.default_rng(1)
    if case == "uniform":
        p = rng.uniform(-1, 1, (3000, 3)).astype(np.float32)
    elif case == "sphere":
        p, _ = synth.sphere(3000, seed=2)
    else:
        base = rng.uniform(-1, 1, (50, 3))
        p = (base[rng.integers(0, 50, 3000)] + 1e-5 * rng.standard_normal((3000, 3))).astype(np.float32)
    xn, _ = oracle.normalize(p)
    for D in (4, 15):
        t = oracle.Tree(xn, D)
        e = t.export()
        order, depth, pb, pe, cb, cc = _bruteforce_tree(oracle.keys(xn, D), D)
        np.testing.assert_array_equal(e["perm"], order)
        np.testing.assert_array_equal(e["depth"], depth)
        np.testing.assert_array_equal(e["pb"], pb)
        np.testing.assert_array_equal(e["pe"], pe)
        np.testing.assert_array_equal(e["child_begin"], cb)
        np.testing.assert_array_equal(e["child_count"], cc)
        assert e["depth"].max() <= D


def test_tree_spec_examples():
    # SPEC.md:L173-L175
    t = oracle.Tree(np.array([[0.1, 0.2, 0.3]], np.float32))
    e = t.export()
    assert t.num_nodes == 1 and e["depth"][0] == 0 and e["child_count"][0] == 0
    octs = np.array([[sx, sy, sz] for sx in (-.5, .5) for sy in (-.5, .5) for sz in (-.5, .5)], np.float32)
    e = oracle.Tree(octs).export()
    assert len(e["depth"]) == 9 and e["child_count"][0] == 8 and np.all(e["depth"][1:] == 1)
    e = oracle.Tree(np.full((10, 3), 0.3, np.float32), 15).export()
    assert len(e["depth"]) == 16 and e["depth"][-1] == 15 and e["pe"][-1] - e["pb"][-1] == 10
    assert np.all(e["child_count"][:-1] == 1)


def test_representatives():
    # PAPER.md:L371-L378 Eqs node-rep-loc / node-rep-vec
    g = GOLD["rep_weighted_mean"]
    # put the two example points into the normalized frame with an identity-like transform:
    # points (0,0,0) and (1,0,0) scaled by 0.5 (still a convex combination test)
    xn = np.array(g["points"], np.float32) * 0.5
    t = oracle.Tree(xn)
    nu = np.array([[g["weights"][0], 0, 0], [0, 0, -g["weights"][1]]], np.float64)
    rep, attr, W = t.moments(nu)
    np.testing.assert_allclose(rep[0], np.array(g["rep"]) * 0.5, rtol=1e-15)
    np.testing.assert_allclose(attr[0], nu.sum(0), rtol=1e-15)
    assert W[0] == 4.0
    # conservation (parent = Σ children), convex combination, zero-weight centroid, one-point reps
    rng = np.random.default_rng(3)
    p, _ = synth.sphere(4000, seed=4)
    xn, _ = oracle.normalize(p)
    t = oracle.Tree(xn)
    e = t.export()
    nu = rng.standard_normal((4000, 3))
    nu[:500] = 0.0
    rep, attr, W = t.moments(nu)
    s = rng.standard_normal(4000)
    rep1, attr1, W1 = t.moments(s)
    srt = xn[e["perm"]].astype(np.float64)
    for k in range(t.num_nodes):
        if e["child_count"][k]:
            ch = slice(e["child_begin"][k], e["child_begin"][k] + e["child_count"][k])
            np.testing.assert_allclose(attr[k], attr[ch].sum(0), rtol=1e-10, atol=1e-12)
            assert np.isclose(attr1[k], attr1[ch].sum(), rtol=1e-10, atol=1e-12)
            assert np.isclose(W[k], W[ch].sum(), rtol=1e-12)
        pts = srt[e["pb"][k]:e["pe"][k]]
        if len(pts) == 1:
            assert np.all(rep[k] == pts[0])
        elif W[k] == 0:
            np.testing.assert_allclose(rep[k], pts.mean(0), rtol=1e-12, atol=1e-15)
        else:
            assert np.all(rep[k] >= pts.min(0) - 1e-12) and np.all(rep[k] <= pts.max(0) + 1e-12)


def test_icosphere_generator_matches_table5_mesh():
    # PAPER.md:L952-L957 Table 5 GT column: total area 12.566, mean 7.670e-5, max 9.253e-5 (Voronoi);
    # our barycentric vertex areas of the same level-7 icosphere reproduce total / mean / max.
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table5.json")))
    p, v, f = synth.icosphere(7)
    assert len(p) == gold["n_points"]
    tri = np.linalg.norm(np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]]), axis=1) / 2
    area = np.zeros(len(v))
    for k in range(3):
        np.add.at(area, f[:, k], tri / 3)
    g = gold["gt_voronoi_area"]
    assert abs(area.sum() / g["total"] - 1) < 1e-4
    assert abs(area.mean() / g["mean"] - 1) < 1e-3
    assert abs(area.max() / g["max"] - 1) < 1e-3
