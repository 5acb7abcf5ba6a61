"""Adaptive octree sampling of the winding-number field around F = ½ (the WNF
reconstruction hand-off) through the C ABI (`wn_iso_cells`).

Pinned against the oracle's F on the full lattice of the finest level: the refinement rule (a cell stays
active while its corners come within `band` of ½; the finest cells the level set crosses are returned) is
replayed on that dense lattice in numpy, once with every threshold tightened and once loosened by the
parity tolerance of F — the GPU's cells must lie between the two sets, and its corner values must equal the
oracle's lattice values within the tolerance.  With a band that keeps every cell active the result must be
exactly the dense crossing set.
"""
import numpy as np
import pytest

import oracle
from paper_2405_16634_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-3  # |F_gpu − F_oracle| at c = 2 (per-query parity: max(1e-4·|F|, 2e-6·Σ|terms|) ≪ 1e-3 here)


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    n = 3000
    pts, nrm = synth.sphere(n, seed=12)
    r = np.linalg.norm(pts, axis=1).mean()
    mu = (nrm * (4 * np.pi * r * r / n)).astype(np.float32)  # area-weighted outward normals: F ≈ 1 inside
    t = wn.wn_build_tree(torch.from_numpy(pts).cuda())
    c0, c1, c2, sc = t.xform
    box = (c0 - 1.0 / sc, c1 - 1.0 / sc, c2 - 1.0 / sc, c0 + 1.0 / sc, c1 + 1.0 / sc, c2 + 1.0 / sc)
    w = float(np.float32(0.01))
    lmax = 6
    side = (1 << lmax) + 1
    ii = np.arange(side) / (1 << lmax)
    lo, hi = np.array(box[:3]), np.array(box[3:])
    # the lattice points exactly as the kernel forms them: float(lo + (hi − lo)·idx / 2^level) per axis
    ax = [(lo[a] + (hi[a] - lo[a]) * ii).astype(np.float32) for a in range(3)]
    X, Y, Z = np.meshgrid(ax[0], ax[1], ax[2], indexing="ij")
    q = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    Fd = np.asarray(oracle.Cloud(pts).F(mu, w, queries=q)).reshape(side, side, side)
    return wn, t, torch.from_numpy(mu).cuda(), box, w, lmax, Fd


def _replay(Fd, lmax, l0, iso, band, tol):
    """the refinement rule on the dense lattice; tol > 0 loosens every threshold, tol < 0 tightens it"""
    n0 = 1 << l0
    I, J, K = np.meshgrid(np.arange(n0), np.arange(n0), np.arange(n0), indexing="ij")
    cells = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1)
    for level in range(l0, lmax + 1):
        f = 1 << (lmax - level)
        v = np.stack([Fd[(cells[:, 0] + (b & 1)) * f, (cells[:, 1] + (b >> 1 & 1)) * f, (cells[:, 2] + (b >> 2 & 1)) * f]
                      for b in range(8)], axis=1)
        lo, hi = v.min(1), v.max(1)
        if level == lmax:
            keep = (lo < iso + tol) & (hi >= iso - tol)
            return cells[keep]
        keep = (lo <= iso + band + tol) & (hi >= iso - band - tol)
        kc = cells[keep]
        ch = np.array([[b & 1, b >> 1 & 1, b >> 2 & 1] for b in range(8)])
        cells = (2 * kc[:, None, :] + ch[None, :, :]).reshape(-1, 3)


def _set(c):
    return set(map(tuple, np.asarray(c).tolist()))


@pytest.mark.parametrize("l0,band", [(2, 0.1), (3, 0.25), (4, 0.05)])
def test_iso_cells_match_dense_oracle(setup, l0, band):
    wn, t, mu, box, w, lmax, Fd = setup
    cells, vals, evals = wn.wn_iso_cells(t, mu, w, box=box, base_level=l0, max_level=lmax, band=band, capacity=64)
    cells, vals = cells.cpu().numpy(), vals.cpu().numpy()
    got = _set(cells)
    strict, loose = _set(_replay(Fd, lmax, l0, 0.5, band, -TOL)), _set(_replay(Fd, lmax, l0, 0.5, band, TOL))
    assert len(strict) > 1000  # the sphere's level set crosses many cells at 64³
    assert strict <= got <= loose, (len(strict - got), len(got - loose))
    assert len(got) == len(cells)  # no duplicates
    ref = np.stack([Fd[cells[:, 0] + (b & 1), cells[:, 1] + (b >> 1 & 1), cells[:, 2] + (b >> 2 & 1)] for b in range(8)], 1)
    np.testing.assert_allclose(vals, ref, rtol=0, atol=TOL)
    assert evals < 0.5 * Fd.size  # adaptive: far fewer evaluations than the dense lattice


def test_iso_cells_without_pruning_is_the_dense_set(setup):
    # band ≥ the field's range keeps every cell active: the finest level is the full lattice
    wn, t, mu, box, w, lmax, Fd = setup
    cells, _, evals = wn.wn_iso_cells(t, mu, w, box=box, base_level=3, max_level=lmax, band=10.0)
    got = _set(cells.cpu().numpy())
    strict, loose = _set(_replay(Fd, lmax, 3, 0.5, 10.0, -TOL)), _set(_replay(Fd, lmax, 3, 0.5, 10.0, TOL))
    assert strict <= got <= loose
    assert evals >= Fd.size  # every lattice point of the finest level (plus the coarser levels')


def test_iso_cells_errors(setup):
    wn, t, mu, box, w, lmax, Fd = setup
    for kw in (dict(base_level=8), dict(base_level=5, max_level=4), dict(max_level=21), dict(band=-1.0),
               dict(box=(0, 0, 0, 0, 1, 1))):
        args = dict(box=box, base_level=3, max_level=5)
        args.update(kw)
        with pytest.raises(wn.WnError, match="ARG"):
            wn.wn_iso_cells(t, mu, w, **args)


def test_iso_cells_single_level(setup):
    # base_level = max_level: no refinement, the crossing cells of the 2^l lattice itself
    wn, t, mu, box, w, lmax, Fd = setup
    cells, vals, evals = wn.wn_iso_cells(t, mu, w, box=box, base_level=4, max_level=4, band=0.1)
    f = 1 << (lmax - 4)
    Fl = Fd[::f, ::f, ::f]  # the level-4 lattice is every 4th point of the level-6 one
    got = _set(cells.cpu().numpy())
    strict, loose = _set(_replay(Fl, 4, 4, 0.5, 0.1, -TOL)), _set(_replay(Fl, 4, 4, 0.5, 0.1, TOL))
    assert strict <= got <= loose and len(got) > 0
    assert evals == 17 ** 3
