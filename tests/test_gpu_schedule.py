"""The query schedule (tree_build.cu:kd_schedule, capi.cu:choose_schedule) against a numpy model of the same
k-d construction: recursive splits of the current order into runs of multiples of 32 queries, along the
axis of the largest robust extent of a 16-point sample, global levels on 16-bit quantized coordinates
(stable), the last levels (segments ≤ 2048) on the exact coordinates (ties: previous order). The schedule
only groups queries into warps — every result is independent of it — so the GPU tests check it exactly."""
import numpy as np
import pytest

from paper_2405_16634_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LOCAL = 2048


@pytest.fixture(scope="module")
def wn():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_16634_b200.wn as wn

    return wn


def _left(m):
    return (((m + 31) // 32) // 2) * 32 if m > 32 else m


def _axis(c):  # c: the segment's coordinates in current order (float32)
    m = len(c)
    v = np.sort(c[(np.arange(16) * m) // 16], axis=0)
    e = v[13] - v[2]
    return int(np.argmax(e))


def kd_model(xn):
    xn = np.asarray(xn, np.float32)
    n = len(xn)
    order = np.arange(n)
    segs = [(0, n)]
    q16 = lambda x: np.clip(np.floor((x.astype(np.float64) + 1.0) * 2.0 ** 15), 0, 2 ** 16 - 1)
    while max(e - b for b, e in segs) > LOCAL:  # global levels
        nxt = []
        for b, e in segs:
            m = e - b
            if m > 32:
                seg = order[b:e]
                ax = _axis(xn[seg])
                order[b:e] = seg[np.argsort(q16(xn[seg, ax]), kind="stable")]
            lf = _left(m)
            nxt += [(b, b + lf), (b + lf, e)]
        segs = nxt
    for b0, e0 in segs:  # local levels inside each segment
        sub = [(b0, e0)]
        while max(e - b for b, e in sub) > 32:
            nxt = []
            for b, e in sub:
                m = e - b
                if m > 32:
                    seg = order[b:e]
                    ax = _axis(xn[seg])
                    order[b:e] = seg[np.argsort(xn[seg, ax], kind="stable")]
                lf = _left(m)
                nxt += [(b, b + lf), (b + lf, e)]
            sub = nxt
    return order


@pytest.mark.parametrize("cfg,nmax", [("C2", 20000), ("C3", 70001), ("C2", 4133), ("C5", 300000)])
def test_kd_schedule_matches_model(wn, cfg, nmax):
    rng = np.random.default_rng(7)
    p = synth.config(cfg)["points"]
    p = p[np.sort(rng.choice(len(p), nmax, replace=False))] if nmax < len(p) else p
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    kind, st = wn.wn_tree_schedule_stats(t)
    if nmax in (20000, 70001):
        assert kind == "kd", (kind, st)  # compact surfaces: fewer visits, no heavier warp
    elif kind != "kd":
        pytest.skip(f"Hilbert chosen for this cloud: {st}")
    assert st["kd_total"] < st["hilbert_total"] and st["kd_max"] <= st["hilbert_max"]
    xn = wn.wn_tree_export(t)["xn"].cpu().numpy()
    got = wn.wn_tree_schedule(t).cpu().numpy()
    np.testing.assert_array_equal(np.sort(got), np.arange(len(p)))
    np.testing.assert_array_equal(got, kd_model(xn))


def test_outlier_cloud_keeps_hilbert(wn):
    # C4 (thin plate + torus + 1 % outliers): k-d puts the outliers' queries together into warps with
    # mutually distant queries — the heaviest warp exceeds Hilbert's, so the Hilbert schedule is kept
    p = synth.config("C4")["points"]
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    kind, st = wn.wn_tree_schedule_stats(t)
    assert kind == "hilbert" and st["kd_max"] > st["hilbert_max"], st


def test_small_cloud_no_choice(wn):
    p = synth.config("C1")["points"]
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    kind, st = wn.wn_tree_schedule_stats(t)
    assert kind == "hilbert" and all(v == 0 for v in st.values())
