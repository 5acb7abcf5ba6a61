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


def _hilbert_keys(xn, b=10):  # tree_build.cu:hilbert_keys (Skilling's transform, 10 bits per axis)
    q = np.clip(np.floor((xn.astype(np.float64) + 1.0) * 2.0 ** (b - 1)), 0, 2 ** b - 1).astype(np.int64)
    X = [q[:, 0].copy(), q[:, 1].copy(), q[:, 2].copy()]
    Q = 1 << (b - 1)
    while Q > 1:
        P = Q - 1
        for i in range(3):
            hit = (X[i] & Q) != 0
            tt = (X[0] ^ X[i]) & P
            x0 = np.where(hit, X[0] ^ P, X[0] ^ tt)
            if i:
                X[i] = np.where(hit, X[i], X[i] ^ tt)
            X[0] = x0
        Q >>= 1
    for i in (1, 2):
        X[i] ^= X[i - 1]
    t = np.zeros_like(X[0])
    Q = 1 << (b - 1)
    while Q > 1:
        t = np.where((X[2] & Q) != 0, t ^ (Q - 1), t)
        Q >>= 1
    for i in range(3):
        X[i] ^= t
    key = np.zeros(len(xn), np.int64)
    for bit in range(b - 1, -1, -1):
        for i in range(3):
            key = (key << 1) | ((X[i] >> bit) & 1)
    return key


def test_hilbert_schedule_blocks_heaviest_first(wn):
    # when Hilbert is kept (C4), the schedule is the Hilbert order with its 128-query blocks permuted
    # (heaviest first by the visit estimate); the ragged last block stays last
    p = synth.config("C4")["points"]
    t = wn.wn_build_tree(torch.from_numpy(p).cuda())
    kind, _ = wn.wn_tree_schedule_stats(t)
    assert kind == "hilbert"
    xn = wn.wn_tree_export(t)["xn"].cpu().numpy()
    ref = np.argsort(_hilbert_keys(xn), kind="stable")
    got = wn.wn_tree_schedule(t).cpu().numpy()
    n, B = len(p), 128
    full = n // B
    np.testing.assert_array_equal(got[full * B:], ref[full * B:])
    gb = got[:full * B].reshape(full, B)
    rb = ref[:full * B].reshape(full, B)
    key = {tuple(r): k for k, r in enumerate(rb)}
    idx = [key.get(tuple(g), -1) for g in gb]
    assert min(idx) >= 0 and sorted(idx) == list(range(full))
    assert idx != list(range(full))  # (the estimate does reorder the blocks)
