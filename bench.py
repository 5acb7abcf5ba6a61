"""bench.py — WNNC hot-path benchmark (BASELINE.json metric: WNNC iterations/s and source-query
interactions/s at N = 500k, 1/2/4/8 B200).

One *step* = one pass of the whole hot path (SURVEY §8(a) rows a1–a9) over the synthetic workload:
wn_build_tree (normalize, Morton sort, octree) + wnnc_iterate (40 iterations of Alg. 3: 4 moment
builds + 4 treecode traversals + α per iteration).  Inputs are resident in HBM when a step starts.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

N > 1 is launched with torchrun (one process per GPU, NCCL); queries are sharded in Morton order and
the ranks exchange s, r, μ and the Σ partials every iteration (strong scaling of the 500k problem).
--impl reference times the fp64 CPU oracle (the only reference this paper-only task has) on the host.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2405_16634_b200 import synth  # noqa: E402

ITERS = 40
CONFIG_TEXT = {
    "C1": "C1: unit sphere, N=2,000 uniform, 40 WNNC iterations, theta=2, D=15, w 0.016->0.002",
    "C2": "C2: torus R=1 r=0.3, N=50,000, 0.5% Gaussian noise, 40 WNNC iterations, theta=2, D=15, w 0.016->0.002",
    "C3": "C3: bumpy sphere r=1+0.15 sin(5t) sin(4p), N=500,000, nonuniform density 10:1, 40 WNNC iterations, "
          "theta=2, D=15, w 0.016->0.002",
    "C4": "C4: thin plate + thin torus + 1% outliers, N=200,000, 40 WNNC iterations, theta=2, D=15",
    "C5": "C5: 8-shape scene, N=4,000,000, 0.25% noise, 40 WNNC iterations, theta=2, D=15",
}
# Algorithmic FP32 operations per unit of work (FMA = 2 flops, rsqrt = 1):
#   opening test: d = (hi − x_q) + lo (3 sub + 3 add, DESIGN.md R-prec) + d² (1 mul + 2 fma = 5)
#                 + far compare (1) + cutoff compare (1)                                      = 13
#   live kernel evaluation, on top of its d²:
#     A : rsqrt 1 + r⁻³ 2 + d·ν 5 + accumulate 2                                           = 10
#     Aᵀ: rsqrt 1 + r⁻³ 2 + s·r⁻³ 1 + accumulate 6                                         = 10
#     G : rsqrt 1 + r⁻², r⁻³ 2 + d·ν 5 + 3(d·ν)r⁻² 2 + ν − t d 6 + accumulate 6            = 22
FLOPS_TEST = 13
FLOPS_TERM = {"A": 10, "AT": 10, "G": 22}
# first-order far field (--order 1): the order-0 term plus M e / eᵀMe / D·e (traverse.cu term1)
FLOPS_TERM1 = {"A": 34, "AT": 23, "G": 55}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self._p:
            time.sleep(0.25)
            self._p.terminate()
            self._p.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _oracle_sample(points, iters, threads_note=""):
    """The fp64 C oracle (test infrastructure, as it stands) on the host: tree + `iters` iterations of
    the 40-iteration schedule.  Returns (seconds for the iterations, cores)."""
    import oracle

    cl = oracle.Cloud(points)
    t0 = time.perf_counter()
    cl.t.solve(iters=iters, total_iters=ITERS, w1=float(np.float32(0.002)), w2=float(np.float32(0.016)))
    return time.perf_counter() - t0, oracle.num_threads()


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    cfg = synth.config(args.config)
    pts = cfg["points"]
    per_step = max(1, args.ref_iters)
    for _ in range(args.warmup):
        _oracle_sample(pts, per_step)
    times = []
    cores = 1
    for _ in range(args.steps):
        dt, cores = _oracle_sample(pts, per_step)
        times.append(dt)
    T = float(np.sum(times))
    value = args.steps * per_step / T
    sample = f"{per_step} of the {ITERS} iterations (schedule iterations 1..{per_step}) per step on the full " \
             f"N={len(pts)} cloud, fp64 oracle treecode, tree build excluded"
    line = {"impl": "reference", "metric": "WNNC iterations/s", "value": value, "unit": "iterations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": CONFIG_TEXT[args.config], "n_points": len(pts)},
            "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2405_16634_b200.wn as wn

    comm = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(wn.wn_comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = wn.wn_comm_init(rank, world, bytes(uid.cpu().numpy().tobytes()))

    cfg = synth.config(args.config)
    pts_h = cfg["points"]
    n = len(pts_h)
    pts = torch.from_numpy(pts_h).to(dev)
    params = dict(iters=ITERS, theta=args.theta, adjoint_mode=wn.WN_ADJ_TRANSPOSE if args.transpose else 0,
                  flags=(wn.WN_FLAG_GRAPH if args.graph else 0) | (wn.WN_FLAG_COMM_NCCL if args.comm == "nccl" else 0)
                  | wn.WN_FLAG_MU_ZERO)  # every step starts from the paper's μ = 0: iteration 1 takes A(0) = 0
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def step(**over):
        tree = wn.wn_build_tree(pts)
        if args.order:
            wn.wn_tree_set_far_order(tree, args.order)
        if args.fmm:
            wn.wn_tree_set_fmm(tree, args.fmm, args.fmm_theta, args.fmm_leaf)
        mu = torch.zeros(n, 3, dtype=torch.float32, device=dev)
        wn.wnnc_iterate(tree, mu, comm=comm, **{**params, **over})
        return tree, mu

    exchange_note = None
    for wi in range(args.warmup):
        try:
            step()
        except wn.WnError as e:  # peer-memory setup fails on every rank alike (collective agreement)
            if comm is None or args.comm != "peer" or wi > 0:
                raise
            params["flags"] |= wn.WN_FLAG_COMM_NCCL
            exchange_note = f"NCCL broadcasts (peer-memory setup failed: {e})"
            step()
    torch.cuda.synchronize()

    # ---- algorithmic work of one step (counting variant, same decisions; untimed) ----
    wn.wn_work_count_enable(True)
    tree, mu = step(flags=params["flags"] & ~wn.WN_FLAG_GRAPH)
    work = wn.wn_work_count_read()
    wn.wn_work_count_enable(False)
    depth_used, num_nodes = tree.depth_used, tree.num_nodes
    sched_kind, _ = wn.wn_tree_schedule_stats(tree)  # k-d boxes or Hilbert runs (chosen per tree)
    del tree

    # ---- per-kernel-class device time (CUDA events around every launch group; untimed pass, no graph) ----
    wn.wn_prof_enable(True)
    for _ in range(args.prof_steps):
        flush.zero_()
        step(flags=params["flags"] & ~wn.WN_FLAG_GRAPH)
    prof = wn.wn_prof_read()
    wn.wn_prof_enable(False)

    # ---- timed region: K steps, per-step CUDA events, L2 flushed between steps (outside the events) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = wn.wn_launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = wn.wn_launch_count() - l0
    ms =float(sum(a.elapsed_time(b) for a, b in ev)) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = ITERS / (ms / 1e3)

    # ---- end to end through the C ABI with HOST buffers (H2D points, D2H normals inside the region) ----
    e2e = None
    if world == 1:
        pts_pin = torch.from_numpy(pts_h).pin_memory()
        wn.wnnc_solve_host(pts_pin, **params)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            wn.wnnc_solve_host(pts_pin, **params)
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / args.steps
        e2e = {"value": ITERS / te, "unit": "iterations/s", "h2d_bytes_per_step": int(n * 12),
               "d2h_bytes_per_step": int(n * 12), "ms_per_step": 1e3 * te}
    else:  # N ranks through the public API: every rank H2D-copies the points (replicated sources), builds
        # the tree and runs the sharded solve; rank 0 reads the result back; time = max over ranks
        pts_pin = torch.from_numpy(pts_h).pin_memory()
        mu_host = torch.empty(n, 3, dtype=torch.float32).pin_memory()
        pts_dev = torch.empty(n, 3, dtype=torch.float32, device=dev)
        tes = []
        for _ in range(args.steps + 1):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pts_dev.copy_(pts_pin, non_blocking=True)
            tree = wn.wn_build_tree(pts_dev)
            mu = torch.zeros(n, 3, dtype=torch.float32, device=dev)
            wn.wnnc_iterate(tree, mu, comm=comm, **params)
            if rank == 0:
                mu_host.copy_(mu, non_blocking=True)
            torch.cuda.synchronize()
            tes.append(time.perf_counter() - t0)
            del tree
        t = torch.tensor([sum(tes[1:]) / args.steps], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        te = float(t.item())
        e2e = {"value": ITERS / te, "unit": "iterations/s", "h2d_bytes_per_step": int(world * n * 12),
               "d2h_bytes_per_step": int(n * 12), "ms_per_step": 1e3 * te,
               "note": "every rank copies the points (replicated sources); rank 0 reads mu back"}
    # ---- exchange check (N > 1, untimed): the peer-memory solve must equal the NCCL solve bit for bit on
    # every rank, and all ranks must hold the same result (both equal the single-GPU trajectory) ----
    exchange_check = None
    if world > 1:
        outs = []
        for extra in (0, wn.WN_FLAG_COMM_NCCL):
            tree = wn.wn_build_tree(pts)
            mu = torch.zeros(n, 3, dtype=torch.float32, device=dev)
            wn.wnnc_iterate(tree, mu, comm=comm, **{**params, "flags": params["flags"] | extra})
            outs.append(mu)
            del tree
        same = int(torch.equal(outs[0], outs[1]))
        h = outs[0].view(torch.int32).to(torch.int64).sum().reshape(1)
        hs = [torch.zeros_like(h) for _ in range(world)]
        torch.distributed.all_gather(hs, h)
        ok = torch.tensor([same], device=dev)
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
        exchange_check = {"peer_equals_nccl_on_all_ranks": bool(ok.item()),
                          "ranks_identical": bool(all(int(x.item()) == int(hs[0].item()) for x in hs))}

    if rank != 0:
        return 0
    # ---- roofline of the dominant kernel class (the treecode traversals) ----
    trav_ms = sum(prof[k][0] for k in ("trav_A", "trav_AT", "trav_G")) / args.prof_steps
    trav_launches = sum(prof[k][1] for k in ("trav_A", "trav_AT", "trav_G")) / args.prof_steps
    fterm = FLOPS_TERM1 if args.order == 1 else FLOPS_TERM
    flops = sum(FLOPS_TEST * work[c]["tests"] + fterm[c] * work[c]["live"] for c in ("A", "AT", "G"))
    achieved = flops / (trav_ms / 1e3) / 1e12
    props = torch.cuda.get_device_properties(dev)
    sm_count = props.multi_processor_count
    clocks = clk.summary()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    fmax = float(peaks.get("sm_max_mhz", clocks.get("sm_max_mhz") or 1965.0))
    peak = sm_count * 128 * 2 * fmax * 1e6 / 1e12
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[args.config]["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    interactions = sum(work[c]["live"] for c in ("A", "AT", "G"))
    # the same traversals on SURVEY §8(d) d.4's FP32 lane-instruction basis (7 per node test; 7 / 7 / 15 per far
    # term of A / Aᵀ / G; a near term 6 more) against the FP32 issue rate of 128 lanes per SM per cycle
    per_term = {"A": 7, "AT": 7, "G": 15}
    lane_instr = sum(7 * work[c]["tests"] + per_term[c] * work[c]["far"] + (per_term[c] + 6) * work[c]["near"]
                     for c in ("A", "AT", "G"))
    issue_peak = sm_count * 128 * fmax * 1e6
    issue_basis = {"achieved": lane_instr / (trav_ms / 1e3), "peak": issue_peak, "unit": "FP32 lane-instructions/s",
                   "frac": lane_instr / (trav_ms / 1e3) / issue_peak,
                   "per_unit": "SURVEY 8(d) d.4: 7 per node test, 7/7/15 per far term (A/AT/G), +6 per near term"}
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "issue_basis": issue_basis,
                "kernel": "treecode traversals (trav_kernel A/AT/G), %.0f launches/step, %.3f ms/step"
                          % (trav_launches, trav_ms),
                "peak_note": f"FP32 FMA pipe: {sm_count} SMs x 128 lanes x 2 flop x {fmax:.0f} MHz "
                             "(sm_max_mhz of MEASURED_PEAKS.json; derived, DESIGN.md §Roofline)",
                "bound_note": "the traversals are instruction-issue bound, not FP32-throughput bound: "
                              "ncu shows 72-81 % issue-slot utilization with ~37 instructions per "
                              "warp-level node visit, of which 13 flops are the algorithmic node test "
                              "(profiles/r02_ncu_trav_v4.txt: 76.0 % issue active, FMA pipe 29 %, ALU 35 %; "
                              "DESIGN.md §6)",
                "work": work}
    if args.fmm:  # FMM operators: the M2L contraction (fp64) of every application over the FMM runs' time
        tree = wn.wn_build_tree(pts)
        mu1 = torch.zeros(n, 3, dtype=torch.float32, device=dev)
        _, (nm2l, np2p) = wn.wn_eval_fmm(tree, mu1, float(np.float32(0.016)), op=0, p=args.fmm,
                                         theta_f=args.fmm_theta, leaf=args.fmm_leaf, counts=True)
        del tree
        ncoef = (args.fmm + 1) * (args.fmm + 2) * (args.fmm + 3) // 6
        apps = 4 * ITERS - 1  # (iteration 1's A(0) is skipped)
        flops = apps * nm2l * 2.0 * ncoef * ncoef
        achieved = flops / (trav_ms / 1e3) / 1e12
        peak64 = sm_count * 64 * 2 * fmax * 1e6 / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak64, "unit": "TFLOP/s (fp64)",
                    "frac": achieved / peak64, "traffic": None,
                    "kernel": f"FMM runs (P2M/M2M/M2L/L2L/L2P+P2P), {apps} per step, {trav_ms:.1f} ms/step; "
                              f"{nm2l} M2L cell pairs and {np2p} P2P leaf pairs per application",
                    "peak_note": f"FP64: {sm_count} SMs x 64 lanes x 2 flop x {fmax:.0f} MHz (derived)",
                    "bound_note": "achieved counts only the M2L contractions (2 np^2 fp64 flops per cell pair): "
                                  "a lower bound on the FMM's arithmetic rate"}
    line = {
        "metric": "WNNC iterations/s", "value": value, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": CONFIG_TEXT[args.config], "n_points": n, "iters_per_step": ITERS,
                   "theta": args.theta, "far_order": args.order, "max_depth": 15, "depth_used": depth_used,
                   "operators": (f"FMM p={args.fmm} theta_f={args.fmm_theta} leaf={args.fmm_leaf} (row f4)"
                                 if args.fmm else "treecode (Alg. 4)"),
                   "num_nodes": num_nodes, "query_schedule": sched_kind,
                   "adjoint": "transpose" if args.transpose else "gather",
                   "launch": "CUDA graph per solve" if args.graph else "stream launches (one solve per tree)",
                   "l2": "flushed between steps (256 MiB write outside the per-step events)",
                   "parallelism": f"query-sharded x{world}" if world > 1 else "1 GPU",
                   "exchange": (exchange_note or ("peer-memory stores in the traversal epilogues"
                                                  if args.comm == "peer" else "NCCL broadcasts"))
                               if world > 1 else None,
                   "step": "wn_build_tree + 40 x (4 moment builds + 4 traversals + alpha)"},
        "interactions_per_s": {"counted": interactions * 1e3 / ms, "effective_dense": 4.0 * n * n * ITERS * 1e3 / ms,
                               "unit": "source-query interactions/s",
                               "note": "counted = live kernel evaluations (far + leaf) of the traversals; "
                                       "effective_dense = 4 N^2 per iteration (the O(N^2) sums replaced)"},
        "breakdown_ms_per_step": {k: v[0] / args.prof_steps for k, v in prof.items()},
        **({"exchange_check": exchange_check} if exchange_check else {}),
        "roofline": roofline,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks,
        "e2e": e2e,
        "paper_context": {"rtx3090_40iter_500k_s": 31.63, "rtx3090_40iter_50k_s": 1.25,
                          "source": "PAPER.md:L89-L96 teaser (other hardware: context only)"},
    }
    if world == 1 and not args.no_cpu_baseline:
        dt, cores = _oracle_sample(pts_h, args.ref_iters)
        line["cpu_baseline"] = {"value": args.ref_iters / dt, "unit": "iterations/s", "cores": cores,
                                "kind": "oracle",
                                "sample": f"iterations 1..{args.ref_iters} of the 40-iteration schedule on the "
                                          f"full N={n} cloud (fp64 oracle treecode, tree build excluded)"}
    print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    return 0


def run_grid(args):
    """Row f1: the winding-number field F(q) = Σ_j ∇Φ_w(q − x_j)·μ_j (the WNF
    reconstruction of §6.1.4) at the R³ points of a grid around the cloud, with μ the solved
    WNNC normals (one untimed 40-iteration solve).  A step = one wn_eval over the whole grid (queries
    resident in HBM; normalization, Hilbert query schedule, moment build, traversal)."""
    import torch

    world, rank, local = _dist()
    if world > 1 and rank != 0:
        return 0  # (grid evaluation is a one-GPU line)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2405_16634_b200.wn as wn

    cfg = synth.config(args.config)
    pts_h = cfg["points"]
    n = len(pts_h)
    pts = torch.from_numpy(pts_h).to(dev)
    tree = wn.wn_build_tree(pts)
    mu = torch.zeros(n, 3, device=dev)
    wn.wnnc_iterate(tree, mu, iters=ITERS, theta=args.theta, flags=wn.WN_FLAG_GRAPH | wn.WN_FLAG_MU_ZERO)
    R = args.grid
    lo, hi = pts_h.min(0), pts_h.max(0)
    c, h = (lo + hi) / 2, (hi - lo) / 2 * 1.1
    axes = [torch.linspace(float(c[k] - h[k]), float(c[k] + h[k]), R, device=dev) for k in range(3)]
    q = torch.stack(torch.meshgrid(*axes, indexing="ij"), -1).reshape(-1, 3).contiguous()
    m = q.shape[0]
    w = float(np.float32(0.002))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        F = wn.wn_eval(tree, mu, w, args.theta, q=q)
    torch.cuda.synchronize()
    # algorithmic work (counting variant, same decisions; untimed)
    wn.wn_work_count_enable(True)
    wn.wn_eval(tree, mu, w, args.theta, q=q)
    work = wn.wn_work_count_read()["A"]
    wn.wn_work_count_enable(False)
    wn.wn_prof_enable(True)
    wn.wn_eval(tree, mu, w, args.theta, q=q)
    prof = wn.wn_prof_read()
    wn.wn_prof_enable(False)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = wn.wn_launch_count()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            F = wn.wn_eval(tree, mu, w, args.theta, q=q)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    launches = wn.wn_launch_count() - l0
    ms = float(sum(a.elapsed_time(b) for a, b in ev)) / args.steps
    inside = float((F > 0.5).float().mean().item())
    # end to end: host grid in (pinned), F back to the host, through the same public call
    q_pin, F_pin = q.cpu().pin_memory(), torch.empty(m, dtype=torch.float32).pin_memory()
    q_dev = torch.empty_like(q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        q_dev.copy_(q_pin, non_blocking=True)
        F_pin.copy_(wn.wn_eval(tree, mu, w, args.theta, q=q_dev), non_blocking=True)
    torch.cuda.synchronize()
    te = (time.perf_counter() - t0) / args.steps
    trav_ms = prof["trav_A"][0]
    flops = FLOPS_TEST * work["tests"] + FLOPS_TERM["A"] * work["live"]
    props = torch.cuda.get_device_properties(dev)
    fmax = 1965.0
    try:
        fmax = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", fmax))
    except OSError:
        pass
    peak = props.multi_processor_count * 128 * 2 * fmax * 1e6 / 1e12
    achieved = flops / (trav_ms / 1e3) / 1e12
    line = {"metric": "off-surface winding-number field F(q) queries/s", "value": m / (ms / 1e3),
            "unit": "queries/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"F on a {R}^3 grid (1.1 x bbox) around {CONFIG_TEXT[args.config]}; "
                                   f"mu = the solved WNNC normals; w = 0.002, theta = {args.theta}",
                       "n_points": n, "queries": m, "query_schedule": "hilbert (per call)",
                       "l2": "flushed between steps (256 MiB write outside the per-step events)",
                       "step": "wn_eval: normalize + Hilbert schedule of the queries + moment build + traversal",
                       "inside_fraction": inside},
            "breakdown_ms_per_step": {k: v[0] for k, v in prof.items() if v[1]},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": f"treecode traversal trav_kernel<A> over {m} queries, {trav_ms:.3f} ms",
                         "work": work},
            "gpu_launches": int(launches), "clocks": clk.summary(),
            "e2e": {"value": m / te, "unit": "queries/s", "h2d_bytes_per_step": int(m * 12),
                    "d2h_bytes_per_step": int(m * 4), "ms_per_step": 1e3 * te}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 5; 64 with --grid)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--theta", type=float, default=2.0)
    ap.add_argument("--transpose", action="store_true", help="north-star exact-transpose adjoint")
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                    help="multi-GPU exchange: peer-memory stores fused into the traversals (default) or NCCL")
    ap.add_argument("--order", type=int, default=0, choices=[0, 1],
                    help="far-field order: 0 = the paper's Alg. 4 (headline), 1 = first-order (SURVEY §8 row f2)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-iters", type=int, default=3, help="oracle iterations per sample / reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prof-steps", type=int, default=2, help="untimed steps with per-kernel CUDA events")
    ap.add_argument("--graph", action="store_true",
                    help="capture each solve's 40 iterations as a CUDA graph (a step builds a new tree, so the graph "
                         "is captured and launched once: 110.2 vs 109.3 ms per C3 step — off by default)")
    ap.add_argument("--no-graph", action="store_true", help=argparse.SUPPRESS)  # (the default; kept for scripts)
    ap.add_argument("--fmm", type=int, default=0,
                    help="row f4: run the solve's operators by FMM of this degree (1..6) instead of the treecode")
    ap.add_argument("--fmm-theta", type=float, default=0.7, help="FMM separation parameter theta_f")
    ap.add_argument("--fmm-leaf", type=int, default=32, help="FMM leaf size (<= 32 points)")
    ap.add_argument("--grid", type=int, default=0,
                    help="row f1: time F(q) on a GRID^3 grid around the cloud (queries/s) instead of the solve")
    args = ap.parse_args()
    if args.steps is None:  # a grid step takes ~8 ms: enough of them to span the clock sampler's 100 ms period
        args.steps = 64 if args.grid else 5
    if args.impl == "reference":
        return run_reference(args)
    if args.grid:
        return run_grid(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
