/* include/wn.h — C ABI of libwn, the B200-native (sm_100a) WNNC hot path.
 *
 * WNNC = "Fast and Globally Consistent Normal Orientation based on the Winding Number Normal
 * Consistency" (Lin, Shi, Liu; arXiv 2405.16634).  "PAPER.md:Lnnn" cites a line of the paper's
 * LaTeX source and the section / equation / algorithm it falls in.
 *
 * What the library computes (all of it in hand-written CUDA kernels for sm_100a):
 *   - the octree of Alg. 4 (§4.5): normalization into [−1,1]^3 with a 1/11 margin
 *     (§5.1.1), Morton keys, a device radix sort and level-wise node emission;
 *   - per application, the |ν|-weighted representatives (Eqs node-rep-loc/vec);
 *   - treecode traversals (Alg. 4) of the three operators
 *       A(μ)_i  = Σ_j ∇Φ_w(x_i − x_j)·μ_j                      (Eq wnf-discretization)
 *       Aᵀ(s)_j = Σ_i s_i ∇Φ_w(x_i − x_j)                      (Alg. 2)
 *       G(μ)_i  = −Σ_j HΦ_w(x_i − x_j) μ_j = −∇F(x_i; μ)       (L264-L272)
 *     with ∇Φ(y) = −y/(4π|y|^3), HΦ(y) = −I/(4π|y|^3) + 3yyᵀ/(4π|y|^5), both set to 0 when
 *     |y| < w (smoothing width, §4.4);
 *   - the WNNC iteration, Alg. 3 with the grad step of Alg. 2 (L297-L342).
 *
 * Conventions:
 *   - Every array argument is a DEVICE pointer unless marked (host).  Arrays are dense, row-major,
 *     fp32 unless stated; "N×3" means n rows of (x, y, z).  The caller owns every buffer it passes;
 *     the library never frees or retains them past the call.
 *   - Inputs and outputs are in the CALLER's frame and point order.  Internally the library
 *     normalizes and sorts in Morton order.  `width` and `theta` are in the
 *     normalized frame, as in the paper (defaults w ∈ [0.002, 0.016], c = 2, L419).
 *     μ is an oriented area element: μ_norm = scale²·μ, F is frame invariant,
 *     ∇F_in = scale·∇F_norm, Aᵀ_in = scale²·Aᵀ_norm (scale = wn_tree_info xform[3]).
 *   - `stream` is a cudaStream_t (0 = legacy default stream).  Calls are stream-ordered and return
 *     without synchronizing unless stated.  Calls on one tree must be serialized (one stream):
 *     per-tree scratch is reused.  Different trees are independent.
 *   - Errors: every call returns a wn_status; nothing throws across the ABI.  On a status ≠ WN_OK
 *     no caller output buffer has been written, and wn_last_error() (thread-local) describes it.
 *     The library never falls back to a CPU path: without a usable sm_100 device every compute
 *     call returns WN_ERR_CUDA.
 */
#ifndef WN_H
#define WN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wn_tree_s* wn_tree; /* opaque: Morton-ordered points, octree, per-tree scratch */
typedef struct wn_comm_s* wn_comm; /* opaque: NCCL communicator for query-sharded iteration  */

typedef enum {
  WN_OK = 0,
  WN_ERR_ARG = 1,        /* bad argument (width ≤ 0, theta ≤ 0, depth ∉ [1,21], iters < 1, …) */
  WN_ERR_EMPTY = 2,      /* n < 1 */
  WN_ERR_NONFINITE = 3,  /* NaN / Inf coordinate */
  WN_ERR_DEGENERATE = 4, /* all points identical (zero extent, PAPER.md:L419 normalization undefined) */
  WN_ERR_CUDA = 5,       /* CUDA runtime error or no usable device */
  WN_ERR_OOM = 6,        /* device allocation failed */
  WN_ERR_NCCL = 7        /* NCCL unavailable or failed */
} wn_status;

enum { WN_ADJ_GATHER = 0,    /* Aᵀ by its own traversal with |s|-weighted reps */
       WN_ADJ_TRANSPOSE = 1  /* exact transpose of treecode A at frozen geometry g(μ): scatter into node
                                accumulators, then push down the tree (BASELINE north star)           */ };

enum {
  WN_FLAG_GRAPH = 1,      /* wnnc_params.flags: capture the iteration loop in a CUDA graph */
  WN_FLAG_COMM_NCCL = 2,  /* multi-GPU: exchange with NCCL broadcasts instead of the default peer-memory
                             stores fused into the traversal epilogues (see wnnc_iterate) */
  WN_FLAG_MU_ZERO = 4,    /* the caller's mu is all zeros (the paper's initialization) and
                             first_iter = 1: iteration 1 takes A(0) = 0, i.e. s = ½ exactly, without a
                             moment build and traversal (bit-identical to computing it) */
  WN_FLAG_HOST_WAIT = 8   /* peer-memory exchange: after each exchanging traversal the HOST waits for every
                             rank's signal (stream synchronize + polling), instead of a device-side wait
                             kernel — no kernel ever waits on another process, so ranks may share a GPU
                             (the multi-process tests); not with WN_FLAG_GRAPH (WN_ERR_ARG) */
};

typedef struct {
  float w_min;          /* w1, final smoothing width (PAPER.md:L419 default 0.002)             */
  float w_max;          /* w2, initial smoothing width (default 0.016); w_min ≤ w_max            */
  float theta;          /* opening constant c of Alg. 4: far iff |x − x_B| > c·edge(B) (default 2) */
  int32_t iters;        /* iterations to run in this call (default 40)                          */
  int32_t first_iter;   /* 1-based index of the first iteration within the schedule (default 1) */
  int32_t total_iters;  /* n of Alg. 3's schedule w = w2 (n−i)/(n−1) + w1 (i−1)/(n−1); 0 ⇒ iters */
  int32_t adjoint_mode; /* WN_ADJ_GATHER (default) or WN_ADJ_TRANSPOSE                             */
  int32_t flags;        /* WN_FLAG_* */
} wnnc_params;

/* Per-iteration diagnostics written by wnnc_iterate (host array of iters records). */
typedef struct {
  double E;      /* E = ‖b − A_w μ‖² before the grad step (Eq value-energy) */
  double alpha;  /* α = rᵀr / ‖A_w r‖² (Alg. 2), 0 if ‖A_w r‖ = 0                              */
  double rr;     /* rᵀr                                                                        */
  double qq;     /* ‖A_w r‖²                                                                   */
  double width;  /* w used in this iteration                                                   */
  double ms;     /* device time of the iteration: the GPU's global timer read by a one-thread kernel
                    at every iteration boundary (inside the CUDA graph too; only in calls that ask
                    for stats, which get their own cached graph)                                 */
  /* algorithmic work of the iteration's traversals (summed over A, Aᵀ, G), only while
     wn_work_count_enable(1) is on, else −1: opening tests, representative (far) terms,
     leaf-point (near) terms, terms past the cutoff (r ≥ w)                                      */
  int64_t tests, far_terms, near_terms, live_terms;
} wnnc_iter_stats;

/* ---- library --------------------------------------------------------------------------------- */
const char* wn_last_error(void);             /* (host) message of the last non-OK status, this thread */
const char* wn_version(void);                /* (host) build string */
/* (host) number of CUDA kernels this library has launched in this process (graph replays count
   each kernel node); used by bench.py to report gpu_launches. */
uint64_t wn_launch_count(void);
/* (host) per-kernel-class device-time accounting with CUDA events on the launching stream.
   enable = 1 starts (and zeroes) it; wn_prof_read synchronizes the device and returns, for each of
   the WN_PROF_* classes, the summed milliseconds and the number of launches. */
enum { WN_PROF_TRAV_A = 0, WN_PROF_TRAV_AT = 1, WN_PROF_TRAV_G = 2, WN_PROF_MOMENTS = 3,
       WN_PROF_TREE = 4, WN_PROF_OTHER = 5, WN_PROF_NCLASS = 6 };
wn_status wn_prof_enable(int32_t enable);
wn_status wn_prof_read(double ms[WN_PROF_NCLASS] /*host*/, int64_t launches[WN_PROF_NCLASS] /*host*/);
/* (host) algorithmic-work accounting: while enabled, traversals run their counting variant (the same
   decisions) and accumulate, per class (A, Aᵀ, G): node opening tests, representative (far) terms,
   leaf-point terms, and live terms (far + leaf terms with r ≥ w, i.e. the kernel evaluations actually
   needed).  enable = 1 zeroes the counters.  wn_work_count_read synchronizes the device;
   counts[4·class + {0,1,2,3}]. */
wn_status wn_work_count_enable(int32_t enable);
wn_status wn_work_count_read(int64_t counts[12] /*host*/);

/* ---- tree (§4.5; normalization L419) ------------------------------------------ */
/* Build the octree of n caller-frame points pts (N×3).  Root cell = [−1,1]^3 of the normalized frame;
   a node is a leaf iff it holds one point or has depth max_depth (D, 1..21, paper default 15).
   Synchronizes `stream` (reads the bounding box and node counts).  *out is owned by the caller and
   released with wn_tree_destroy. */
wn_status wn_build_tree(const float* pts, int64_t n, int32_t max_depth, void* stream, wn_tree* out /*host*/);
wn_status wn_tree_destroy(wn_tree t);
/* (host outputs) sizes and the similarity transform: xn = (x − xform[0:3]) · xform[3]. */
wn_status wn_tree_info(wn_tree t, int64_t* num_points, int64_t* num_nodes, int32_t* depth_used,
                       double xform[4]);
/* Far-field order used by every later wn_eval / wn_eval_grad / wn_query_work / wn_eval_adjoint
   (gather) / wnnc_iterate call on t.  0 (default): the paper's Alg. 4 — a far node B contributes its
   representative term K(x_i − x_B)·ν_B.  1: first-order far field (SURVEY §8
   row f2, an extension; the paper points to expansions via Barill et al., L409): the far term also
   includes Σ_{j∈B} ∇_x K(x_i − x)|_{x_B}·(x_j − x_B) ν_j, from per-node first moments (symmetric
   M = Σ_j ν_j (x_j − x_B)ᵀ for vector ν, D = Σ_j s_j (x_j − x_B) for scalar s).  Opening decisions
   and near-field terms are unchanged.  Order 1 is not defined for the transpose-mode adjoint
   (WN_ADJ_TRANSPOSE ⇒ WN_ERR_ARG).  The first call with order 1 allocates its scratch (stream-ordered
   on `stream`; ≈ 200 B per point).  WN_ERR_ARG for order ∉ {0, 1}. */
wn_status wn_tree_set_far_order(wn_tree t, int32_t order, void* stream);
/* Export the structure (device outputs, any may be NULL): keys[N] uint64 Morton keys in sorted order
   (3·D bits, level-1 octant digit most significant, digit = 4·x + 2·y + z); perm[N] caller index of
   the k-th sorted point; xn[N×3] normalized coordinates in sorted order; per node in BFS order
   (children contiguous, ascending digit): depth, pb, pe (sorted-point range), child_begin (−1 for a
   leaf), child_count. */
wn_status wn_tree_export(wn_tree t, uint64_t* keys, int32_t* perm, float* xn, int32_t* depth, int32_t* pb,
                         int32_t* pe, int32_t* child_begin, int32_t* child_count, void* stream);
/* Representatives of attribute nu (caller order; dim 3 ⇒ N×3 vector, dim 1 ⇒ N scalar) optionally
   multiplied per point by a[N] (NULL ⇒ 1): rep[Nn×3] = x_{B,ν} (normalized frame),
   attr[Nn×dim] = ν_B, W[Nn] (double) = Σ|ν| — BFS node order.  Diagnostic / parity entry point. */
wn_status wn_moments(wn_tree t, const float* nu, int32_t dim, const float* a, float* rep, float* attr,
                     double* W, void* stream);

/* ---- operators (Alg. 4 treecode) -------------------------------------------------------------- */
/* F(q) = Σ_j ∇Φ_w(q − x_j)·(a_j μ_j)  (the winding-number field; A(μ) when q = NULL).
   mu[N×3] caller order, input frame; a[N] or NULL; q[M×3] input-frame queries or NULL (⇒ the N source
   points, m ignored); width w > 0; theta c > 0 (+inf ⇒ exact sum).  F[M] (or F[N]). */
wn_status wn_eval(wn_tree t, const float* mu, const float* a, const float* q, int64_t m, float width,
                  float theta, float* F, void* stream);
/* ∇F(q) (input frame; = −G(μ) at the points).  gradF[M×3]. */
wn_status wn_eval_grad(wn_tree t, const float* mu, const float* a, const float* q, int64_t m, float width,
                       float theta, float* gradF, void* stream);
/* Per-query work of wn_eval (op 0) / wn_eval_grad (op 2) with the same arguments, without computing
   the field: counts[M×4] (int32, query order) = node tests, far terms, leaf-point terms, live terms.
   A one-point node always takes the representative branch here (its far and leaf terms coincide), so
   far + leaf-point terms equals Alg. 4's far + near count.  Diagnostic / parity entry point. */
wn_status wn_query_work(wn_tree t, int32_t op, const float* mu, const float* q, int64_t m, float width, float theta,
                        int32_t* counts, void* stream);
/* Adaptive octree sampling of F around its iso level (the WNF reconstruction hand-off,
   PAPER.md:L1005-L1008).  box = {lo_x, lo_y, lo_z, hi_x, hi_y, hi_z} (input frame) is cut into 2^base_level
   cells per axis (base_level 0..7); per level F is evaluated once at every distinct corner of the active
   cells (wn_eval's Alg. 4 traversal, width, theta), a cell stays active while min ≤ iso + band and
   max ≥ iso − band over its corners (band ≥ 0) and is split in eight, down to max_level (≤ 20).  Output:
   the max_level cells the level set crosses (min < iso ≤ max): cells[k×3] (int32 lattice coordinates
   i, j, k of the cell's low corner; its extent is (hi − lo)/2^max_level), values[k×8] (corner F, corner
   b at (i + (b&1), j + (b>>1&1), k + (b>>2&1))), at most `capacity` of them (device buffers; may be NULL
   when capacity = 0); *count (host) = the number of crossed cells (may exceed capacity: call again with
   more room); *evals (host, may be NULL) = F evaluations over all levels.  Synchronizes `stream`.
   WN_ERR_ARG for bad levels, band, box or buffers, or more than 2^26 active cells in a level. */
wn_status wn_iso_cells(wn_tree t, const float* mu, float width, float theta, const float box[6], int32_t base_level,
                       int32_t max_level, float iso, float band, int64_t capacity, int32_t* cells, float* values,
                       int64_t* count, int64_t* evals, void* stream);
/* out[N×3] = (Aᵀ s)_j = Σ_i s_i ∇Φ_w(x_i − x_j)  (input frame), s[N] caller order.
   mode WN_ADJ_GATHER: own traversal with |s|-weighted representatives.
   mode WN_ADJ_TRANSPOSE: exact transpose of wn_eval's treecode at the geometry of mu_geom[N×3]
   (required in this mode, else WN_ERR_ARG). */
wn_status wn_eval_adjoint(wn_tree t, const float* s, float width, float theta, int32_t mode,
                          const float* mu_geom, float* out, void* stream);

/* ---- solver (Alg. 3 + Alg. 2) ----------------------------------------------- */
/* Run p->iters iterations of: w = schedule(i); s = ½ − A_w μ; r = A_wᵀ s; α = rᵀr/‖A_w r‖²;
   μ' = μ + α r; μ̂ = G_w(μ'); μ_i = μ̂_i |μ'_i| / |μ̂_i| (μ'_i kept if |μ̂_i| = 0).
   mu[N×3] caller order, input frame, in/out; zeros ⇒ the paper's initialization (L301).
   comm NULL ⇒ one GPU; otherwise queries are sharded over the communicator's ranks (every rank passes
   the full mu and receives the full, rank-identical result).  Exchange (multi-GPU): by default each
   traversal's epilogue stores its owned rows and Σ partials straight into every rank's replica through
   CUDA IPC peer mappings (NVLink / NVSwitch), the last block of the launch signals every rank and a
   device-side wait orders the next step — no separate collective; the first call per communicator (and
   any call with a larger N) sets up the per-rank arena collectively (≈ 150 B per point: the exchanged
   rows, partials and the transpose-mode accumulators; synchronizes `stream`).  WN_FLAG_COMM_NCCL selects
   grouped ncclBroadcasts instead.  Both give the single-GPU trajectory bit for bit.  Transpose-mode
   adjoint (WN_ADJ_TRANSPOSE) across ranks — the north star's "scatters into node moments and is then pushed
   down the tree": every rank scatters its shard into its own node / point accumulators; peer mode: a
   signal and wait, then every rank adds all ranks' accumulators in rank order (IPC reads) and pushes down
   for all points; NCCL mode: an all-reduce of the accumulators, then the same push-down.  The replicas
   stay identical bit for bit; against one GPU the result differs by the rounding of the scatter's fp64
   atomics (as two single-GPU transpose runs do).  Trees with more than 3 nodes per point are refused
   across ranks (WN_ERR_ARG).  At most 8 ranks in peer mode (WN_ERR_ARG beyond).  stats (host, p->iters
   records) may be NULL; when given the call synchronizes `stream` before returning. */
wn_status wnnc_iterate(wn_tree t, float* mu, const wnnc_params* p, wn_comm comm, wnnc_iter_stats* stats,
                       void* stream);
/* Diagnostic: the peer-memory exchange of `world` (1..8) ranks emulated on this one GPU, serialized on
   `stream` — every rank's traversal over its shard reads its own replica and stores into all replicas,
   every wait is issued after all signals (none ever spins).  mu as in wnnc_iterate (rank 0's result);
   replicas (device, world×N×3, may be NULL) receives every rank's final μ.  No CUDA graph; synchronizes
   `stream`; both adjoint modes. */
wn_status wnnc_iterate_emulated(wn_tree t, float* mu, const wnnc_params* p, int32_t world, float* replicas,
                                void* stream);
/* End-to-end convenience for HOST buffers: copies pts_host (N×3) to the device, builds the tree,
   runs wnnc_iterate from μ = 0, copies the unit-normalized result (zero rows stay zero) to
   normals_host (N×3, host) and, if mu_host ≠ NULL, the raw μ (input frame).  Synchronizes `stream`.
   Pinned host buffers give the fastest copies. */
wn_status wnnc_solve_host(const float* pts_host, int64_t n, int32_t max_depth, const wnnc_params* p,
                          float* normals_host, float* mu_host, wnnc_iter_stats* stats, void* stream);

/* Fast multipole evaluation at the n sources (the paper's future work, PAPER.md:L1034 —
   an alternative to Alg. 4's treecode, not the paper's method).  op 0: F = Σ_j ∇Φ_w(x_i − x_j)·μ_j (attr =
   μ, N×3, input frame, out N) as wn_eval; op 2: ∇F (attr μ, out N×3) as wn_eval_grad; op 1: Aᵀ(s) (attr
   = s, N, out N×3) as wn_eval_adjoint's gather mode — the same sums, evaluated by Cartesian Taylor
   multipole / local expansions of total degree p (1..6) between well-separated cells (|c_t − c_s|·θ_f >
   r_t + r_s and every point pair beyond the cutoff w) and directly between the remaining FMM leaves
   (octree nodes with at most `leaf` ≤ 32 points or no children).  counts (host, 2, may be NULL): M2L cell
   pairs and P2P leaf pairs.  Synchronizes `stream`; the interaction lists (built level by level on the
   first call) are cached on the tree for the same (p, θ_f, leaf, width). */
wn_status wn_eval_fmm(wn_tree t, int32_t op, const float* attr, float width, int32_t p, float theta_f, int32_t leaf,
                      float* out, int64_t* counts, void* stream);
/* Select the operators of later wnnc_iterate calls on this tree: p = 0 (default) the paper's Alg. 4 treecode,
   p = 1..6 the FMM of wn_eval_fmm (single GPU, gather-mode adjoint; one plan per solve, built with the
   schedule's largest width w_max as separation width, so every iteration's expanded pairs are beyond its
   cutoff).  The FMM plan is built on the first call (host-synchronizing) and cached on the tree. */
wn_status wn_tree_set_fmm(wn_tree t, int32_t p, float theta_f, int32_t leaf);

/* ---- multi-GPU (NCCL over NVLink / NVSwitch) ---------------------------------------------------- */
wn_status wn_comm_unique_id(uint8_t id[128] /*host*/);
/* Collective over `world` processes, one GPU each (the current device of the calling thread). */
wn_status wn_comm_init(int32_t rank, int32_t world, const uint8_t id[128] /*host*/, wn_comm* out /*host*/);
wn_status wn_comm_destroy(wn_comm c);
/* Communicator without NCCL (bootstrap over the caller's own channel, e.g. torch.distributed gloo): the
   peer-memory arena is set up by wn_comm_arena_export on every rank (allocates this rank's block for n
   points, writes its 64-byte CUDA IPC handle to `handle`, host) and wn_comm_arena_import with all ranks'
   handles in rank order (world × 64 bytes, host; opens the peers' blocks).  Work-weighted shards are then
   computed by every rank alone (identical: the plan is deterministic).  The NCCL exchange
   (WN_FLAG_COMM_NCCL) is unavailable on such a communicator (WN_ERR_ARG). */
wn_status wn_comm_init_local(int32_t rank, int32_t world, wn_comm* out /*host*/);
wn_status wn_comm_arena_export(wn_comm c, int64_t n, uint8_t handle[64] /*host*/, void* stream);
wn_status wn_comm_arena_import(wn_comm c, const uint8_t* handles /*host, world × 64*/);
/* (host) Query shard of `rank`: sorted-point range [*begin, *end) of n points split over `world`
   ranks in contiguous Morton ranges aligned to WN_SHARD_ALIGN queries (so per-block reduction
   partials are identical for every world size).  Pure host arithmetic. */
enum { WN_SHARD_ALIGN = 256 };
wn_status wn_shard_range(int64_t n, int32_t rank, int32_t world, int64_t* begin, int64_t* end);
/* The query schedule (diagnostic): qorder[N] (device) = sorted-point index at each schedule position —
   the order the traversals (32 consecutive positions per warp) and the multi-GPU shards follow. */
wn_status wn_tree_schedule(wn_tree t, int32_t* qorder, void* stream);
/* Which schedule wn_build_tree chose (host outputs, either may be NULL): *kind = 0 Hilbert-curve runs
   (its 128-query blocks ordered heaviest first by the estimate below; N ≥ 4096), 1 k-d boxes of 32
   queries (recursive median splits); stats = warp-level visits of the A traversal over
   the unit-weight geometry, counted on every 4th warp of each schedule, used for the choice: {Hilbert
   total, Hilbert heaviest warp, k-d total, k-d heaviest warp} (all 0 when no choice was made:
   N < 4096).  The schedule never changes a result. */
wn_status wn_tree_schedule_stats(wn_tree t, int32_t* kind, int64_t stats[4]);
/* The shards wnnc_iterate actually uses for `world` ranks (1..64) on this tree: bounds[world + 1] (host),
   rank r owns schedule positions [bounds[r], bounds[r+1]), multiples of WN_SHARD_ALIGN, split by
   estimated work (the node tests of the A traversal over the unit-weight geometry) so that non-uniform
   clouds load the ranks evenly; wn_shard_range is the equal-count split.  Synchronizes `stream`. */
wn_status wn_shard_plan(wn_tree t, int32_t world, int64_t* bounds, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WN_H */
