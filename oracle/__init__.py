"""oracle — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes front end of the plain fp64 C oracle in ``wn_oracle.c`` (see its header for what it
computes and what pins it).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  It never imports the
product package ``paper_2405_16634_b200`` (only the product's seeded input generators are shared,
and those hold none of the method's arithmetic).

Frames (§5.1.1 normalization, DESIGN.md R-frame): the C oracle works in the
normalized frame.  Here μ (an area element) maps as μ_norm = scale²·μ, F is frame invariant,
∇F_in = scale·∇F_norm and Aᵀ_in = scale²·Aᵀ_norm.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wn_oracle.c")
_LIB = os.path.join(_HERE, "libwn_oracle.so")

OP_A, OP_G, OP_AT, ABS, ORDER1 = 0, 1, 2, 8, 16


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, OpenMP, no fp contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "wn_oracle.h"))
    ):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.wo_normalize.argtypes = [P, I64, P, P]
        L.wo_normalize.restype = I32
        L.wo_normalize_apply.argtypes = [P, P, I64, P]
        L.wo_keys.argtypes = [P, I64, I32, P]
        L.wo_tree_build.argtypes = [P, I64, I32]
        L.wo_tree_build.restype = P
        L.wo_tree_free.argtypes = [P]
        L.wo_tree_num_nodes.argtypes = [P]
        L.wo_tree_num_nodes.restype = I64
        L.wo_tree_max_depth.argtypes = [P]
        L.wo_tree_export.argtypes = [P] + [P] * 6
        L.wo_moments.argtypes = [P, P, I32, P, P, P]
        L.wo_dense_op.argtypes = [P, I32, P, I32, P, I64, D, P]
        L.wo_tree_op.argtypes = [P, I32, P, I32, P, P, I64, D, D, P, P]
        L.wo_tree_A_frozen.argtypes = [P, P, P, D, D, P]
        L.wo_tree_AT_transpose.argtypes = [P, P, P, D, D, P]
        L.wo_solve.argtypes = [P, P, D, D, I32, I32, I32, D, I32, I32, I32, I32, P]
        L.wo_solve.restype = I32
        L.wo_num_threads.restype = I32
        L.wo_rescale.argtypes = [I64, P, P, P]
        L.wo_fmm_op.argtypes = [P, I32, P, I32, D, I32, D, I32, P, P]
        L.wo_fmm_config.argtypes = [I32, D, I32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(lib().wo_num_threads())


class OracleError(RuntimeError):
    pass


def normalize(raw):
    """returns (xn fp32 n×3, xf = [cx, cy, cz, scale])."""
    raw = _f32(raw).reshape(-1, 3)
    xn = np.empty_like(raw)
    xf = np.zeros(4, np.float64)
    rc = lib().wo_normalize(_p(raw), raw.shape[0], _p(xn), _p(xf))
    if rc:
        raise OracleError({1: "empty", 2: "non-finite", 3: "degenerate"}[rc])
    return xn, xf


def normalize_apply(xf, raw):
    raw = _f32(raw).reshape(-1, 3)
    xn = np.empty_like(raw)
    xf = _f64(xf)
    lib().wo_normalize_apply(_p(xf), _p(raw), raw.shape[0], _p(xn))
    return xn


def keys(xn, D=15):
    xn = _f32(xn).reshape(-1, 3)
    k = np.empty(xn.shape[0], np.uint64)
    lib().wo_keys(_p(xn), xn.shape[0], D, _p(k))
    return k


class Tree:
    """Recursive octree over normalized fp32 points."""

    def __init__(self, xn, D=15):
        self.xn = _f32(xn).reshape(-1, 3)
        self.n = self.xn.shape[0]
        self.D = D
        self._h = lib().wo_tree_build(_p(self.xn), self.n, D)
        if not self._h:
            raise OracleError("tree build failed")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().wo_tree_free(self._h)
            self._h = None

    @property
    def num_nodes(self) -> int:
        return int(lib().wo_tree_num_nodes(self._h))

    @property
    def max_depth(self) -> int:
        return int(lib().wo_tree_max_depth(self._h))

    def export(self):
        nn = self.num_nodes
        perm = np.empty(self.n, np.int32)
        arrs = [np.empty(nn, np.int32) for _ in range(5)]
        lib().wo_tree_export(self._h, _p(perm), *[_p(a) for a in arrs])
        depth, pb, pe, cb, cc = arrs
        return dict(perm=perm, depth=depth, pb=pb, pe=pe, child_begin=cb, child_count=cc)

    def moments(self, nu):
        nu = _f64(nu)
        dim = 1 if nu.ndim == 1 else 3
        nn = self.num_nodes
        rep = np.empty((nn, 3))
        attr = np.empty((nn, dim))
        W = np.empty(nn)
        lib().wo_moments(self._h, _p(nu), dim, _p(rep), _p(attr), _p(W))
        return rep, (attr[:, 0] if dim == 1 else attr), W

    # --- operators, normalized frame -------------------------------------------------------
    def dense(self, op, nu, w, queries=None):
        nu = _f64(nu)
        dim = 1 if nu.ndim == 1 else 3
        q = None if queries is None else _f32(queries).reshape(-1, 3)
        m = self.n if q is None else q.shape[0]
        od = 1 if (op == OP_A or op & ABS) else 3
        out = np.empty((m, od))
        lib().wo_dense_op(self._h, op, _p(nu), dim, None if q is None else _p(q), m, float(w), _p(out))
        return out[:, 0] if od == 1 else out

    def tree(self, op, nu, w, theta=2.0, queries=None, qidx=None, counters=False, order=0):
        """Alg. 4 treecode; order=1: first-order far field (not the paper's)."""
        if order == 1:
            op |= ORDER1
        nu = _f64(nu)
        dim = 1 if nu.ndim == 1 else 3
        q = None if queries is None else _f32(queries).reshape(-1, 3)
        qi = None if qidx is None else np.ascontiguousarray(qidx, dtype=np.int64)
        m = q.shape[0] if q is not None else (qi.shape[0] if qi is not None else self.n)
        od = 1 if ((op & ~ORDER1) == OP_A or op & ABS) else 3
        out = np.empty((m, od))
        cnt = np.empty((m, 4), np.int64) if counters else None
        lib().wo_tree_op(self._h, op, _p(nu), dim, None if q is None else _p(q),
                         None if qi is None else _p(qi), m, float(w), float(theta), _p(out),
                         None if cnt is None else _p(cnt))
        out = out[:, 0] if od == 1 else out
        return (out, cnt) if counters else out

    def fmm(self, op, nu, w, p=4, theta=0.5, leaf=32, counters=False):
        """FMM: A (op OP_A, ν n×3) / G (OP_G, ν n×3) / Aᵀ (OP_AT, s n) at the sources."""
        nu = _f64(nu)
        dim = 1 if nu.ndim == 1 else 3
        od = 1 if op == OP_A else 3
        out = np.empty((self.n, od))
        cnt = np.zeros(2, np.int64)
        lib().wo_fmm_op(self._h, op, _p(nu), dim, float(w), int(p), float(theta), int(leaf), _p(out), _p(cnt))
        out = out[:, 0] if od == 1 else out
        return (out, cnt) if counters else out

    def A_frozen(self, mu_geom, nu, w, theta=2.0):
        out = np.empty(self.n)
        lib().wo_tree_A_frozen(self._h, _p(_f64(mu_geom)), _p(_f64(nu)), float(w), float(theta), _p(out))
        return out

    def AT_transpose(self, mu_geom, s, w, theta=2.0):
        out = np.empty((self.n, 3))
        lib().wo_tree_AT_transpose(self._h, _p(_f64(mu_geom)), _p(_f64(s)), float(w), float(theta), _p(out))
        return out

    def solve(self, mu0=None, w1=0.002, w2=0.016, iters=40, theta=2.0, backend="tree", mode="gather",
              wnnc=True, first_iter=1, total_iters=None, order=0, fmm=(4, 0.5, 32)):
        """Alg. 3 in the normalized frame; returns (mu_norm n×3, stats iters×5).  backend "tree" (Alg. 4),
        "dense" or "fmm" (row f4: fmm = (p, θ_f, leaf), separation width w2)."""
        mu = np.zeros((self.n, 3)) if mu0 is None else _f64(mu0).copy()
        stats = np.empty((iters, 5))
        total = iters if total_iters is None else total_iters
        if backend == "fmm":
            lib().wo_fmm_config(int(fmm[0]), float(fmm[1]), int(fmm[2]))
        lib().wo_solve(self._h, _p(mu), float(w1), float(w2), int(iters), int(first_iter), int(total),
                       float(theta), {"tree": 0, "dense": 1, "fmm": 2}[backend], 0 if mode == "gather" else 1,
                       1 if wnnc else 0, int(order), _p(stats))
        return mu, stats


def rescale(mu_prev, mu_hat):
    """WNNC rescale (Alg. 3): μ̂_i |μ'_i| / |μ̂_i|, μ'_i kept where |μ̂_i| = 0."""
    mp = _f64(mu_prev).reshape(-1, 3)
    mh = _f64(mu_hat).reshape(-1, 3)
    out = np.empty_like(mp)
    lib().wo_rescale(mp.shape[0], _p(mp), _p(mh), _p(out))
    return out


def width_schedule(k: int, n: int, w1: float, w2: float) -> float:
    """Alg. 3, PAPER.md:L335 (n = 1 ⇒ w1)."""
    if n == 1:
        return w1
    return w2 * (n - k) / (n - 1) + w1 * (k - 1) / (n - 1)


# --- input-frame wrappers (the C-ABI's frame, DESIGN.md R-frame) ------------------------------
class Cloud:
    """Caller-frame point cloud: normalization + tree, operators with input-frame μ / outputs."""

    def __init__(self, raw, D=15):
        self.raw = _f32(raw).reshape(-1, 3)
        self.xn, self.xf = normalize(self.raw)
        self.scale = float(self.xf[3])
        self.t = Tree(self.xn, D)

    def _mu_norm(self, mu, a=None):
        mu = _f64(mu).reshape(-1, 3)
        if a is not None:
            mu = mu * _f64(a)[:, None]
        return mu * self.scale ** 2

    def _q(self, queries):
        return None if queries is None else normalize_apply(self.xf, queries)

    def F(self, mu, w, theta=2.0, a=None, queries=None, dense=False, qidx=None, counters=False, order=0):
        if dense:
            return self.t.dense(OP_A, self._mu_norm(mu, a), w, self._q(queries))
        return self.t.tree(OP_A, self._mu_norm(mu, a), w, theta, self._q(queries), qidx, counters, order)

    def gradF(self, mu, w, theta=2.0, a=None, queries=None, dense=False, qidx=None, counters=False, order=0):
        """∇F in the input frame (= −G scaled by `scale`)."""
        if dense:
            g = self.t.dense(OP_G, self._mu_norm(mu, a), w, self._q(queries))
            return -g * self.scale
        r = self.t.tree(OP_G, self._mu_norm(mu, a), w, theta, self._q(queries), qidx, counters, order)
        if counters:
            return -r[0] * self.scale, r[1]
        return -r * self.scale

    def AT(self, s, w, theta=2.0, dense=False, qidx=None, counters=False, order=0):
        if dense:
            return self.t.dense(OP_AT, _f64(s), w) * self.scale ** 2
        r = self.t.tree(OP_AT, _f64(s), w, theta, None, qidx, counters, order)
        if counters:
            return r[0] * self.scale ** 2, r[1]
        return r * self.scale ** 2

    def abs_scale(self, op, nu_in, w, theta=2.0, a=None, queries=None, qidx=None, order=0):
        """S_i = Σ_j |term_ij| of the treecode sum at query i, in the output's frame (the conditioning
        scale of a cancelling sum; used for the parity error floor)."""
        if op == OP_AT:
            return self.t.tree(OP_AT | ABS, _f64(nu_in), w, theta, None, qidx, order=order) * self.scale ** 2
        S = self.t.tree(op | ABS, self._mu_norm(nu_in, a), w, theta, self._q(queries), qidx, order=order)
        return S * (self.scale if op == OP_G else 1.0)

    def fmm(self, op, nu_in, w, p=4, theta_f=0.5, leaf=32, counters=False):
        """FMM (row f4) in the input frame: op OP_A → F (ν = μ), OP_G → ∇F (μ), OP_AT → Aᵀ (ν = s)."""
        if op == OP_AT:
            r = self.t.fmm(OP_AT, _f64(nu_in), w, p, theta_f, leaf, counters)
            sc = self.scale ** 2
        else:
            r = self.t.fmm(op, self._mu_norm(nu_in), w, p, theta_f, leaf, counters)
            sc = 1.0 if op == OP_A else -self.scale
        return (r[0] * sc, r[1]) if counters else r * sc

    def AT_transpose(self, s, mu_geom, w, theta=2.0):
        return self.t.AT_transpose(self._mu_norm(mu_geom), _f64(s), w, theta) * self.scale ** 2

    def solve(self, **kw):
        mu, stats = self.t.solve(**kw)
        return mu / self.scale ** 2, stats


# --- metrics: PAPER.md:L514-L521 ---------------------------------------------------------------
def unit(v):
    v = _f64(v)
    n = np.linalg.norm(v, axis=1, keepdims=True)
    return np.where(n > 0, v / np.where(n > 0, n, 1), 0.0)


def p_co(n_est, n_gt):
    """P_co = #{n·n_gt > 0}/N (strict)."""
    return float(np.mean(np.sum(unit(n_est) * unit(n_gt), axis=1) > 0))


def ae_pcd(n_est, n_gt):
    """AE_pcd = mean (1 − n_gt·n)/2."""
    return float(np.mean((1 - np.sum(unit(n_est) * unit(n_gt), axis=1)) / 2))
