"""Thin ctypes binding of libwn (include/wn.h).  Argument marshalling only: every step of the hot path
runs in the CUDA kernels behind the C ABI.  Functions carry the C names; tensors are torch CUDA
tensors (fp32, contiguous) and the current torch stream is passed as the CUDA stream.

Importing this module loads ``libwn.so`` and fails loudly if it is missing — there is no CPU
fallback (build it with ``python -m paper_2405_16634_b200.build`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_LIB_PATH = os.environ.get("WN_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwn.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libwn.so not built ({_LIB_PATH}); run paper_2405_16634_b200.build.build()")
_L = C.CDLL(_LIB_PATH)

WN_OK, WN_ERR_ARG, WN_ERR_EMPTY, WN_ERR_NONFINITE, WN_ERR_DEGENERATE, WN_ERR_CUDA, WN_ERR_OOM, WN_ERR_NCCL = range(8)
WN_ADJ_GATHER, WN_ADJ_TRANSPOSE = 0, 1
WN_FLAG_GRAPH = 1
WN_FLAG_COMM_NCCL = 2
WN_FLAG_MU_ZERO = 4
WN_FLAG_HOST_WAIT = 8
PROF_CLASSES = ("trav_A", "trav_AT", "trav_G", "moments", "tree", "other")
STATUS_NAMES = {0: "WN_OK", 1: "WN_ERR_ARG", 2: "WN_ERR_EMPTY", 3: "WN_ERR_NONFINITE", 4: "WN_ERR_DEGENERATE",
                5: "WN_ERR_CUDA", 6: "WN_ERR_OOM", 7: "WN_ERR_NCCL"}
EXPORTED = ("wn_last_error", "wn_version", "wn_launch_count", "wn_prof_enable", "wn_prof_read", "wn_build_tree",
            "wn_tree_destroy", "wn_tree_info", "wn_tree_export", "wn_moments", "wn_eval", "wn_eval_grad",
            "wn_eval_adjoint", "wnnc_iterate", "wnnc_solve_host", "wn_comm_unique_id", "wn_comm_init",
            "wn_comm_destroy", "wn_shard_range", "wn_work_count_enable", "wn_work_count_read", "wn_query_work",
            "wn_tree_set_far_order", "wnnc_iterate_emulated", "wn_shard_plan", "wn_tree_schedule",
            "wn_tree_schedule_stats", "wn_comm_init_local", "wn_comm_arena_export", "wn_comm_arena_import", "wn_eval_fmm", "wn_tree_set_fmm",
            "wn_iso_cells")


class wnnc_params(C.Structure):
    _fields_ = [("w_min", C.c_float), ("w_max", C.c_float), ("theta", C.c_float), ("iters", C.c_int32),
                ("first_iter", C.c_int32), ("total_iters", C.c_int32), ("adjoint_mode", C.c_int32),
                ("flags", C.c_int32)]


class wnnc_iter_stats(C.Structure):
    _fields_ = [("E", C.c_double), ("alpha", C.c_double), ("rr", C.c_double), ("qq", C.c_double),
                ("width", C.c_double), ("ms", C.c_double), ("tests", C.c_int64), ("far_terms", C.c_int64),
                ("near_terms", C.c_int64), ("live_terms", C.c_int64)]


P, I32, I64, F32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
_sig = {
    "wn_last_error": ([], C.c_char_p), "wn_version": ([], C.c_char_p), "wn_launch_count": ([], C.c_uint64),
    "wn_prof_enable": ([I32], I32), "wn_prof_read": ([P, P], I32),
    "wn_build_tree": ([P, I64, I32, P, P], I32), "wn_tree_destroy": ([P], I32),
    "wn_tree_info": ([P, P, P, P, P], I32), "wn_tree_export": ([P] * 10, I32),
    "wn_moments": ([P, P, I32, P, P, P, P, P], I32),
    "wn_eval": ([P, P, P, P, I64, F32, F32, P, P], I32), "wn_eval_grad": ([P, P, P, P, I64, F32, F32, P, P], I32),
    "wn_eval_adjoint": ([P, P, F32, F32, I32, P, P, P], I32),
    "wnnc_iterate": ([P, P, P, P, P, P], I32), "wnnc_solve_host": ([P, I64, I32, P, P, P, P, P], I32),
    "wn_comm_unique_id": ([P], I32), "wn_comm_init": ([I32, I32, P, P], I32), "wn_comm_destroy": ([P], I32),
    "wn_shard_range": ([I64, I32, I32, P, P], I32),
    "wn_work_count_enable": ([I32], I32), "wn_work_count_read": ([P], I32),
    "wn_query_work": ([P, I32, P, P, I64, F32, F32, P, P], I32),
    "wn_tree_set_far_order": ([P, I32, P], I32),
    "wnnc_iterate_emulated": ([P, P, P, I32, P, P], I32),
    "wn_shard_plan": ([P, I32, P, P], I32),
    "wn_tree_schedule": ([P, P, P], I32),
    "wn_tree_schedule_stats": ([P, P, P], I32),
    "wn_comm_init_local": ([I32, I32, P], I32),
    "wn_comm_arena_export": ([P, I64, P, P], I32),
    "wn_comm_arena_import": ([P, P], I32),
    "wn_eval_fmm": ([P, I32, P, F32, I32, F32, I32, P, P, P], I32),
    "wn_tree_set_fmm": ([P, I32, F32, I32], I32),
    "wn_iso_cells": ([P, P, F32, F32, P, I32, I32, F32, F32, I64, P, P, P, P, P], I32),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_L, _name)
    _f.argtypes = _args
    _f.restype = _res


class WnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(st):
    if st != WN_OK:
        raise WnError(st, _L.wn_last_error().decode(errors="replace"))


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _dev_f32(t, shape_last=None):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError("expected a contiguous float32 CUDA tensor")
    if shape_last is not None and t.shape[-1] != shape_last:
        raise ValueError(f"expected last dimension {shape_last}")
    return t


def wn_version() -> str:
    return _L.wn_version().decode()


def wn_launch_count() -> int:
    return int(_L.wn_launch_count())


def wn_prof_enable(enable: bool = True):
    _check(_L.wn_prof_enable(1 if enable else 0))


def wn_prof_read():
    ms = (C.c_double * 6)()
    n = (C.c_int64 * 6)()
    _check(_L.wn_prof_read(ms, n))
    return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(PROF_CLASSES)}


def wn_work_count_enable(enable: bool = True):
    _check(_L.wn_work_count_enable(1 if enable else 0))


def wn_work_count_read():
    c = (C.c_int64 * 12)()
    _check(_L.wn_work_count_read(c))
    return {k: dict(tests=int(c[4 * i]), far=int(c[4 * i + 1]), near=int(c[4 * i + 2]), live=int(c[4 * i + 3]))
            for i, k in enumerate(("A", "AT", "G"))}


def wn_eval_fmm(tree: Tree, attr: torch.Tensor, width: float, op: int = 0, p: int = 4, theta_f: float = 0.5,
                leaf: int = 32, counts: bool = False):
    """FMM at the sources: op 0 F (attr μ N×3), 2 ∇F (μ), 1 Aᵀ (attr s, N)."""
    if op == 1:
        _dev_f32(attr)
    else:
        _dev_f32(attr, 3)
    out = torch.empty((tree.n,) if op == 0 else (tree.n, 3), dtype=torch.float32, device=attr.device)
    c = (C.c_int64 * 2)()
    _check(_L.wn_eval_fmm(tree.handle, int(op), _ptr(attr), float(width), int(p), float(theta_f), int(leaf),
                          _ptr(out), c, _stream()))
    return (out, (int(c[0]), int(c[1]))) if counts else out


def wn_tree_set_fmm(tree: Tree, p: int, theta_f: float = 0.5, leaf: int = 32):
    """wnnc_iterate's operators: p = 0 the paper's treecode (default), 1..6 the FMM."""
    _check(_L.wn_tree_set_fmm(tree.handle, int(p), float(theta_f), int(leaf)))


def wn_iso_cells(tree: Tree, mu: torch.Tensor, width: float, theta: float = 2.0, box=None, base_level: int = 4,
                 max_level: int = 8, iso: float = 0.5, band: float = 0.1, capacity: int = 1 << 20):
    """Adaptive octree sampling of F around its iso level (the WNF hand-off): the max_level
    cells the level set crosses as (cells int32 [k, 3], corner values [k, 8], F evaluations).  box defaults to
    the tree's normalization cube (input frame)."""
    _dev_f32(mu, 3)
    if box is None:
        c0, c1, c2, sc = tree.xform
        box = (c0 - 1.0 / sc, c1 - 1.0 / sc, c2 - 1.0 / sc, c0 + 1.0 / sc, c1 + 1.0 / sc, c2 + 1.0 / sc)
    bx = (C.c_float * 6)(*[float(v) for v in box])
    cnt, ev = C.c_int64(0), C.c_int64(0)
    while True:
        cells = torch.empty(max(capacity, 1), 3, dtype=torch.int32, device=mu.device)
        vals = torch.empty(max(capacity, 1), 8, dtype=torch.float32, device=mu.device)
        _check(_L.wn_iso_cells(tree.handle, _ptr(mu), float(width), float(theta), bx, int(base_level), int(max_level),
                               float(iso), float(band), int(capacity), _ptr(cells), _ptr(vals), C.byref(cnt),
                               C.byref(ev), _stream()))
        if cnt.value <= capacity:
            return cells[:cnt.value], vals[:cnt.value], int(ev.value)
        capacity = int(cnt.value)


def wn_query_work(tree, mu, width, theta=2.0, op=0, q=None):
    """Per-query (tests, far terms, leaf-point terms, live terms) of wn_eval (op 0) / wn_eval_grad (op 2)."""
    _dev_f32(mu, 3)
    m = tree.n if q is None else _dev_f32(q, 3).shape[0]
    c = torch.empty(m, 4, dtype=torch.int32, device=tree.device)
    _check(_L.wn_query_work(tree.handle, int(op), _ptr(mu), _ptr(q), m, float(width), float(theta), _ptr(c),
                            _stream()))
    return c


class Tree:
    """Owns a wn_tree handle (octree over the caller's points)."""

    def __init__(self, handle, device):
        self._h = handle
        self.device = device
        n, nn, d = C.c_int64(), C.c_int64(), C.c_int32()
        xf = (C.c_double * 4)()
        _check(_L.wn_tree_info(self._h, C.byref(n), C.byref(nn), C.byref(d), xf))
        self.n, self.num_nodes, self.depth_used = n.value, nn.value, d.value
        self.xform = tuple(xf)

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            _L.wn_tree_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def wn_build_tree(pts: torch.Tensor, max_depth: int = 15) -> Tree:
    _dev_f32(pts, 3)
    h = C.c_void_p()
    _check(_L.wn_build_tree(_ptr(pts), pts.shape[0], int(max_depth), _stream(), C.byref(h)))
    return Tree(h, pts.device)


def wn_tree_destroy(tree: Tree):
    tree.close()


def wn_tree_set_far_order(tree: Tree, order: int):
    """0: the paper's representative far term (Alg. 4); 1: first-order far field."""
    _check(_L.wn_tree_set_far_order(tree.handle, int(order), _stream()))


def wn_tree_export(tree: Tree):
    dev = tree.device
    n, nn = tree.n, tree.num_nodes
    out = dict(keys=torch.empty(n, dtype=torch.int64, device=dev), perm=torch.empty(n, dtype=torch.int32, device=dev),
               xn=torch.empty(n, 3, dtype=torch.float32, device=dev))
    for k in ("depth", "pb", "pe", "child_begin", "child_count"):
        out[k] = torch.empty(nn, dtype=torch.int32, device=dev)
    _check(_L.wn_tree_export(tree.handle, *[_ptr(out[k]) for k in ("keys", "perm", "xn", "depth", "pb", "pe",
                                                                   "child_begin", "child_count")], _stream()))
    return out


def wn_moments(tree: Tree, nu: torch.Tensor, a: torch.Tensor | None = None):
    _dev_f32(nu)
    dim = 1 if nu.dim() == 1 else 3
    nn = tree.num_nodes
    rep = torch.empty(nn, 3, dtype=torch.float32, device=tree.device)
    attr = torch.empty(nn, dim, dtype=torch.float32, device=tree.device)
    W = torch.empty(nn, dtype=torch.float64, device=tree.device)
    _check(_L.wn_moments(tree.handle, _ptr(nu), dim, _ptr(_dev_f32(a)), _ptr(rep), _ptr(attr), _ptr(W), _stream()))
    return rep, (attr[:, 0] if dim == 1 else attr), W


def wn_eval(tree: Tree, mu, width, theta=2.0, a=None, q=None):
    """F at q (input frame) or at the sources (q = None)."""
    _dev_f32(mu, 3)
    m = tree.n if q is None else _dev_f32(q, 3).shape[0]
    F = torch.empty(m, dtype=torch.float32, device=tree.device)
    _check(_L.wn_eval(tree.handle, _ptr(mu), _ptr(_dev_f32(a)), _ptr(q), m, float(width), float(theta), _ptr(F),
                      _stream()))
    return F


def wn_eval_grad(tree: Tree, mu, width, theta=2.0, a=None, q=None):
    """∇F (input frame); at the sources this is −G(μ)."""
    _dev_f32(mu, 3)
    m = tree.n if q is None else _dev_f32(q, 3).shape[0]
    g = torch.empty(m, 3, dtype=torch.float32, device=tree.device)
    _check(_L.wn_eval_grad(tree.handle, _ptr(mu), _ptr(_dev_f32(a)), _ptr(q), m, float(width), float(theta), _ptr(g),
                           _stream()))
    return g


def wn_eval_adjoint(tree: Tree, s, width, theta=2.0, mode=WN_ADJ_GATHER, mu_geom=None):
    _dev_f32(s)
    out = torch.empty(tree.n, 3, dtype=torch.float32, device=tree.device)
    _check(_L.wn_eval_adjoint(tree.handle, _ptr(s), float(width), float(theta), int(mode), _ptr(_dev_f32(mu_geom)),
                              _ptr(out), _stream()))
    return out


def make_params(w_min=0.002, w_max=0.016, theta=2.0, iters=40, first_iter=1, total_iters=0,
                adjoint_mode=WN_ADJ_GATHER, flags=0) -> wnnc_params:
    return wnnc_params(w_min, w_max, theta, iters, first_iter, total_iters, adjoint_mode, flags)


def _stats_dict(s):
    return {k: getattr(s, k) for k, _ in wnnc_iter_stats._fields_}


def wnnc_iterate(tree: Tree, mu: torch.Tensor, comm=None, stats: bool = False, **params):
    """In-place Alg. 3 on mu (N×3, input frame).  Returns per-iteration stats (list of dicts) if asked."""
    _dev_f32(mu, 3)
    p = make_params(**params)
    st = (wnnc_iter_stats * p.iters)() if stats else None
    _check(_L.wnnc_iterate(tree.handle, _ptr(mu), C.byref(p), comm.handle if comm else None, st, _stream()))
    if stats:
        return [_stats_dict(s) for s in st]
    return None


def wnnc_solve_host(pts_host: torch.Tensor, max_depth=15, return_mu=False, stats=False, **params):
    """End-to-end: host points in, unit normals out (host tensors; pinned memory recommended)."""
    if pts_host.is_cuda or pts_host.dtype != torch.float32 or not pts_host.is_contiguous():
        raise ValueError("pts_host must be a contiguous float32 CPU tensor")
    n = pts_host.shape[0]
    pin = pts_host.is_pinned()
    normals = torch.empty(n, 3, dtype=torch.float32, pin_memory=pin)
    mu = torch.empty(n, 3, dtype=torch.float32, pin_memory=pin) if return_mu else None
    p = make_params(**params)
    st = (wnnc_iter_stats * p.iters)() if stats else None
    _check(_L.wnnc_solve_host(_ptr(pts_host), n, int(max_depth), C.byref(p), _ptr(normals), _ptr(mu), st, _stream()))
    out = [normals]
    if return_mu:
        out.append(mu)
    if stats:
        out.append([_stats_dict(s) for s in st])
    return out[0] if len(out) == 1 else tuple(out)


def wn_shard_range(n: int, rank: int, world: int):
    b, e = C.c_int64(), C.c_int64()
    _check(_L.wn_shard_range(int(n), int(rank), int(world), C.byref(b), C.byref(e)))
    return b.value, e.value


class Comm:
    def __init__(self, handle, rank, world):
        self._h, self.rank, self.world = handle, rank, world

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            _L.wn_comm_destroy(self._h)
            self._h = None


def wn_comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_L.wn_comm_unique_id(buf))
    return bytes(buf)


def wnnc_iterate_emulated(tree: Tree, mu: torch.Tensor, world: int, **params):
    """Diagnostic: `world` ranks of the peer-memory exchange emulated on this GPU; returns every rank's μ."""
    _dev_f32(mu, 3)
    p = make_params(**params)
    reps = torch.empty(world, tree.n, 3, dtype=torch.float32, device=tree.device)
    _check(_L.wnnc_iterate_emulated(tree.handle, _ptr(mu), C.byref(p), int(world), _ptr(reps), _stream()))
    return reps


def wn_tree_schedule(tree: Tree) -> torch.Tensor:
    """Sorted-point index at each position of the query schedule (k-d boxes or Hilbert runs)."""
    out = torch.empty(tree.n, dtype=torch.int32, device=tree.device)
    _check(_L.wn_tree_schedule(tree.handle, _ptr(out), _stream()))
    return out


def wn_tree_schedule_stats(tree: Tree):
    """("kd" | "hilbert", {hilbert_total, hilbert_max, kd_total, kd_max}) — the estimate behind the choice."""
    kind = C.c_int32(0)
    st = (C.c_int64 * 4)()
    _check(_L.wn_tree_schedule_stats(tree.handle, C.byref(kind), st))
    keys = ("hilbert_total", "hilbert_max", "kd_total", "kd_max")
    return ("kd" if kind.value == 1 else "hilbert"), dict(zip(keys, list(st)))


def wn_shard_plan(tree: Tree, world: int):
    """The work-weighted query shards of a `world`-rank solve: list of world + 1 schedule positions."""
    b = (C.c_int64 * (world + 1))()
    _check(_L.wn_shard_plan(tree.handle, int(world), b, _stream()))
    return list(b)


def wn_comm_init(rank: int, world: int, uid: bytes) -> Comm:
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    h = C.c_void_p()
    _check(_L.wn_comm_init(int(rank), int(world), buf, C.byref(h)))
    return Comm(h, rank, world)


def wn_comm_init_local(rank: int, world: int) -> Comm:
    """Communicator without NCCL: the caller exchanges the arena handles (wn_comm_arena_export/_import)."""
    h = C.c_void_p()
    _check(_L.wn_comm_init_local(int(rank), int(world), C.byref(h)))
    return Comm(h, rank, world)


def wn_comm_arena_export(comm: Comm, n: int) -> bytes:
    buf = (C.c_uint8 * 64)()
    _check(_L.wn_comm_arena_export(comm.handle, int(n), buf, _stream()))
    return bytes(buf)


def wn_comm_arena_import(comm: Comm, handles):
    """handles: every rank's 64-byte handle, in rank order."""
    blob = b"".join(handles)
    buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
    _check(_L.wn_comm_arena_import(comm.handle, buf))


def wn_comm_destroy(comm: Comm):
    comm.close()
