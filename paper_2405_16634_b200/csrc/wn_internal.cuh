// wn_internal.cuh — shared declarations of the libwn CUDA sources (sm_100a).
// Not part of the ABI; see include/wn.h for the public contract.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/wn.h"

namespace wn {

// WN_DEBUG builds (tools/build_variants.py "debug") trap on any out-of-range index the kernels compute —
// the bounds checks stand in for compute-sanitizer, which this GPU pool does not allow
#ifdef WN_DEBUG
#define WN_DCHECK(cond, what)                                                                   \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("libwn WN_DEBUG check failed: %s (%s:%d)\n", what, __FILE__, __LINE__);           \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define WN_DCHECK(cond, what) \
  do {                        \
  } while (0)
#endif

constexpr int kMaxDepth = 21;
constexpr float kInv4Pi = 0.0795774715459476679f;  // 1/(4π)

// Kinds of attribute a moment build aggregates.
enum AttrKind { ATTR_VEC = 0, ATTR_SCALAR = 1, ATTR_UNIT = 2 };

// One moment build's output: a 64-byte record per node (BFS order), rec[4·i + {0,1,2,3}]:
//   R = (x_B, y_B, z_B, thr)   thr = (c·edge)² in fp32, or −1 for a one-point node (always "far":
//                               rep = the point, ν_B = ν_j, so far and leaf terms coincide)
//   V = (ν_B.x, ν_B.y, ν_B.z, topo) for vector ν, (s_B, 0, 0, topo) for scalar ν
//   L = (x_B − hi, y_B − hi, z_B − hi, 0): the fp32 remainder of the fp64 representative; decisions and the
//       far term use d = (hi − x_q) + lo (error ~1e-7·|d| instead of ulp(x_B)/|d|), DESIGN.md R-prec.
//   X = unused (pads the record to one aligned 64-byte half line)
// topo (int bits): leaf = 0; internal = (child_begin << 4) | (count − 1); L.w = one-point-leaf child mask
constexpr int kRec = 4;  // float4 per record
struct NodeSet {
  float4* rec = nullptr;
  // order-1 far field, 2 float4 per node: vector ν: (Mxx, Myy, Mzz, tr M), (Mxy, Mxz,
  // Myz, 0) with M = sym Σ_j ν_j (x_j − x_B)ᵀ; scalar s: (D, 0), D = Σ_j s_j (x_j − x_B); null for order 0
  float4* ext = nullptr;
};

struct IterScratch {
  int64_t n = 0;
  float4* mu = nullptr;      // μ, normalized frame, sorted order
  float4* mup = nullptr;     // μ' = μ + α r
  float4* r = nullptr;       // r = Aᵀ s
  float* s = nullptr;        // s = ½ − A μ
  double* part = nullptr;    // per-group partials: [3][nblk] (Σs², Σ|r|², Σq²), nblk = part_slots(n)
  double* dstats = nullptr;  // per-iteration (E, α, rr, qq, w) — device
  int64_t* dcounts = nullptr;  // (iters + 1) × 12 snapshots of the work counters (counting runs only)
  int64_t stats_cap = 0;
  unsigned long long* dstamp = nullptr;  // iters + 1 device timestamps (ns): iteration i runs between [i] and [i + 1]
  double* alpha = nullptr;   // current α (device) + the α reduction's block sums and ticket (alpha_words())
  float* tmp = nullptr;      // generic N×4 scratch
  int nblk = 0;
};
// Tile plan of the per-iteration moment builds (moments.cu): the sorted points are cut into tiles of
// kMomTile; a node whose points lie in one tile is summed from that tile's per-point terms in shared memory
// (one thread per node below kMomWarpNode points, one warp above), a node across tiles from the partial
// sums at its two ends (the "endpoints") and the totals of the tiles in between.
#ifndef WN_EXP_MOMTILE
#define WN_EXP_MOMTILE 1024
#endif
constexpr int kMomTile = WN_EXP_MOMTILE;  // the default tile; choose_mom_tile adapts it per cloud size
constexpr int kMomTileMax = 1280;
// points per moment-build tile for n points on `sms` SMs (moments.cu:choose_mom_tile)
int choose_mom_tile(int64_t n, int sms);
#ifndef WN_EXP_MOMWARP
#define WN_EXP_MOMWARP 32
#endif
constexpr int kMomWarpNode = WN_EXP_MOMWARP;  // nodes with this many points or more are summed by a warp
constexpr int kMomNC = 13;        // sums per node of the widest layout (vector attribute, first order)
struct MomPlan {
  bool ready = false;
  int64_t nsmall = 0, nlarge = 0, ncross = 0;
  // one-tile nodes with ≥ 2 points, ascending first point (hence grouped by tile), as descriptors
  // {node, pb − tile start | (pe − tile start) << 16, topo, smask | tdepth << 16}; small: < kMomWarpNode points
  int4* small = nullptr;
  int4* large = nullptr;
  int32_t* tile_soff = nullptr;  // ntiles + 1: tile k's small nodes are small[tile_soff[k], tile_soff[k + 1])
  int32_t* tile_loff = nullptr;  // likewise for the large ones
  int2* onept = nullptr;         // per sorted point: {its one-point node, topo} if that node is built, else {−1, ·}
  int32_t* cross = nullptr;      // nodes over more than one tile
  uint64_t* ep_key = nullptr;    // 2·ncross, ascending: tile·(kMomTile + 1) + local index
  int32_t* ep_slot = nullptr;    // its slot: 2c ↔ Σ from pb to its tile's end, 2c + 1 ↔ Σ from pe's tile start to pe
  int32_t* tile_eoff = nullptr;  // ntiles + 1 offsets into ep_key
  double* epval = nullptr;       // 2·ncross × kMomNC endpoint sums
};
// Fast-multipole plan of a tree (fmm.cu): cell geometry, node lists, the sorted interaction
// lists for (p, θ_f, leaf, separation width wsep), and the expansion scratch
struct FmmPlan {
  bool ready = false;
  int p = 0, leaf = 0;
  double theta = 0.0;
  float wsep = 0.f;
  double *ctr = nullptr, *rad = nullptr, *M = nullptr, *L = nullptr;
  uint8_t* leaf_flag = nullptr;
  int32_t* leaves = nullptr;
  int64_t nleaves = 0;
  std::vector<int32_t*> inner, kids;  // per level: internal active nodes / active non-root nodes
  std::vector<int64_t> ninner, nkids;
  uint64_t *m2l = nullptr, *p2p = nullptr;  // sorted (target << 32 | source)
  int64_t nm2l = 0, np2p = 0;
  int32_t *om = nullptr, *op2 = nullptr;    // CSR offsets per target node
  // M2L pairs grouped by their translation vector c_t − c_s (equal vectors ⇒ one derivative tensor):
  // gidx = the m2l positions in group order, ginv its inverse, chunks of ≤ 128 (p ≥ 5: 64) pairs of one
  // group, Lp = the per-pair local expansions in group order (nm2l × np)
  int32_t *gidx = nullptr, *ginv = nullptr;
  int4 *chunks = nullptr, *chunks_small = nullptr;  // {first pair, pairs, group}: full and small chunks
  int64_t nchunk_small = 0;
  double* Tg = nullptr;  // per group: the derivative tensor T_δ, |δ| ≤ 2p (graded order)
  int64_t nchunk = 0, ngroups = 0;
  double* Lp = nullptr;
  int32_t* m2lt = nullptr;  // the target cells with a non-empty M2L list
  int64_t nm2lt = 0;
  double4* VG = nullptr;  // per sorted point: the far field (V, ∇V) from L2P
  // P2P work items {leaf index, list range, item of its leaf}, per leaf {T, items, partial base}, the
  // leaves of several items (combined from partial sums)
  int4 *items = nullptr, *linfo = nullptr;
  int64_t nitems = 0, nmleaves = 0;
  int32_t* mleaves = nullptr;
  double4* part = nullptr;
  std::vector<void*> owned;
};
// Query shards of a multi-GPU solve: schedule positions [b[r], b[r+1]) for rank r, multiples of
// WN_SHARD_ALIGN, split by estimated work (capi.cu:plan_shards); world = 0 ⇒ equal counts (wn_shard_range)
constexpr int kMaxShardRanks = 64;
struct ShardPlan {
  int world = 0;
  int64_t b[kMaxShardRanks + 1] = {};
};

}  // namespace wn

struct wn_tree_s {
  int64_t n = 0, nn = 0, nleaves = 0;
  int D = 15, depth_used = 0;
  double xf[4] = {0, 0, 0, 1};
  int device = 0;
  float4* pts = nullptr;        // N normalized points, Morton order (w unused)
  int32_t* perm = nullptr;      // sorted position → caller index
  uint64_t* keys = nullptr;     // sorted keys
  int32_t* qorder = nullptr;    // query schedule: sorted point indices in k-d or Hilbert order (or null)
  int sched_kind = 0;           // 0: Hilbert runs, 1: k-d boxes (capi.cu:choose_schedule)
  long long sched_stats[4] = {};  // warp-level visits of the estimate: Hilbert total, max; k-d total, max
  int32_t* depth = nullptr;     // per node (BFS)
  int32_t* pb = nullptr;
  int32_t* pe = nullptr;
  int32_t* cb = nullptr;        // first child (BFS), −1 for leaves
  int32_t* cc = nullptr;        // child count
  int32_t* parent = nullptr;    // −1 for the root
  int32_t* leaf_of = nullptr;   // sorted point → its leaf node
  int32_t* topo = nullptr;      // per node traversal code (see NodeSet)
  int32_t* smask = nullptr;     // per node: bit k set iff child k is a one-point leaf; bits 8..12: chain length
  int32_t* tdepth = nullptr;    // per node: depth whose (c·edge)² is its threshold (its chain's bottom)
  int32_t* mom_live = nullptr;  // the nodes a traversal can visit (root + the child groups of internal codes)
  int64_t mom_nlive = 0;
  float4* centroid = nullptr;   // unweighted centroid per node (Σ|ν| = 0 fallback)
  double* sums = nullptr;       // Nn × 8 fp64 node sums of the running build
  int mom_cut = 0;              // moment builds: levels < mom_cut run in one block
  int64_t* mom_loff = nullptr;  //   level offsets on the device
  wn::MomPlan mplan[2];          // per-iteration moment builds: [0] the visitable nodes, [1] every node (export)
  double* mom_ttot = nullptr;    // per-tile totals of the running build (ntiles × kMomNC)
  wn::ShardPlan shard;           // work-weighted query shards for the last world size used
  int64_t mom_ntiles = 0;
  int mom_tile = 0;              // points per tile of the moment builds (choose_mom_tile, per tree)
  bool mom_order1_ready = false;  // prefix scratch + set[0].ext sized for the first-order far field
  int far_order = 0;              // wn_tree_set_far_order: 0 (the paper's Alg. 4) or 1 (row f2)
  int fmm_p = 0, fmm_leaf = 32;   // wn_tree_set_fmm: wnnc_iterate's operators by FMM of degree fmm_p (0: treecode)
  float fmm_theta = 0.5f;
  wn::FmmPlan fmm;
  wn::NodeSet set[2];           // [0] = current attribute, [1] = frozen geometry (transpose mode)
  std::vector<int64_t> level_off;  // host: BFS offset of each level, size depth_used + 2
  wn::IterScratch it;
  float4* qbuf = nullptr;       // normalized arbitrary queries
  int32_t* qbuf_order = nullptr;  // their Hilbert schedule
  int64_t qcap = 0;
  // transpose-mode accumulators
  double* tvb = nullptr;        // node accumulators V_B (Nn×3, fp64)
  double* tu = nullptr;         // point accumulators U_j (N×3, fp64)
  // CUDA graph of the iteration loop (WN_FLAG_GRAPH), cached per parameter set
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  uint64_t graph_launches = 0;  // kernel nodes in the graph
  std::vector<uint8_t> graph_key;
  // recorded on the caller's stream at the end of every call on the tree: destruction waits for it, so
  // no buffer returns to the pool while queued work (on any stream, blocking or not) may still read it
  cudaEvent_t done_ev = nullptr;
};

namespace wn {

// ---- error plumbing (capi.cu) ----
wn_status set_error(wn_status st, const std::string& msg);
wn_status cuda_status(cudaError_t e, const char* what);
#define WN_TRY(x)                 \
  do {                            \
    wn_status st_ = (x);          \
    if (st_ != WN_OK) return st_; \
  } while (0)
#define WN_CUDA(call)                                                      \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) return ::wn::cuda_status(e_, #call);            \
  } while (0)

// ---- launch accounting / profiling (capi.cu) ----
struct ProfScope {
  ProfScope(int cls, cudaStream_t s, int nlaunch = 1);
  ~ProfScope();
  int cls;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
};
void count_launches(int n);
int64_t* work_counters(int cls);  // device counters of a traversal class, or null when counting is off

// drop the cached CUDA graph of the iteration loop (a buffer it references is about to be freed)
void invalidate_graph(wn_tree_s* t);

// ---- tree build (tree_build.cu) ----
wn_status build_tree(const float* pts, int64_t n, int D, cudaStream_t s, wn_tree_s* t);
void free_tree(wn_tree_s* t);
// order[k] = index of the k-th of n points along a 3-D Hilbert curve of [−1,1]^3 (query schedule)
wn_status hilbert_schedule(const float4* pts, int64_t n, int32_t* order, cudaStream_t s);
wn_status kd_schedule(const float4* pts, int64_t n, int32_t* order, cudaStream_t s);
// ascending stable sort of n 64-bit keys on their low `bits` bits into out (device)
wn_status sort_keys_u64(const uint64_t* keys, int64_t n, int bits, uint64_t* out, cudaStream_t s);
// exclusive scan of m uint32 flags (tree_build.cu), *total = the sum (device)
wn_status scan_u32(const uint32_t* in, uint32_t* out, int64_t m, uint32_t* total, cudaStream_t s);
// F at m input-frame queries q[m×3] given in a spatially coherent order (wn_eval's path — moments of mu,
// traversal — without the per-call Hilbert schedule), F[m]
wn_status eval_field(wn_tree_s* t, const float* mu, const float* q, int64_t m, float width, float theta, float* F,
                     cudaStream_t s);
wn_status sort_keys_u64_perm(const uint64_t* keys, int64_t n, int bits, uint64_t* out, int32_t* perm,
                             cudaStream_t s);

// ---- moments (moments.cu) ----
// Build node records for attribute `kind` into `out`.  vec: float4 ν (sorted order), scal: float s.
// a (optional, caller order) multiplies ν per point in fp64 before aggregation.
// If axpy_r != nullptr: ν = vec + α·axpy_r (α read on device from *alpha) and ν is written to axpy_out.
struct MomentArgs {
  int kind = ATTR_VEC;
  const float4* vec = nullptr;
  const float* scal = nullptr;
  const float* a_sorted = nullptr;  // per sorted point multiplier, or null
  const float4* axpy_r = nullptr;
  const double* alpha = nullptr;
  float4* axpy_out = nullptr;
  float theta = 2.0f;
  NodeSet out;
  float4* centroid_out = nullptr;   // ATTR_UNIT: writes the centroid table
  int32_t* leaf_of_out = nullptr;   // ATTR_UNIT: writes the leaf node of every sorted point
  bool write_W = false;             // also store each node's Σ|ν| in tree sums[8·i] (wn_moments export)
  bool order1 = false;              // also the first moments (out.ext), row f2
  bool all_nodes = false;           // every node (wn_moments export), not only the visitable ones
};
wn_status build_moments(wn_tree_s* t, const MomentArgs& m, cudaStream_t s);
wn_status plan_moments(wn_tree_s* t, cudaStream_t s);  // once per tree, after the topology
// tile plan over the visitable nodes (which = 0) or every node (1; wn_moments export) — tree_build.cu
wn_status plan_moment_tiles(wn_tree_s* t, int which, cudaStream_t s);
wn_status enable_order1(wn_tree_s* t, cudaStream_t s);  // first wn_tree_set_far_order(t, 1)

// ---- traversal (traverse.cu) ----
enum TravOp { OP_A = 0, OP_AT = 1, OP_G = 2 };
enum Epi {
  EPI_PLAIN = 0,     // out_f (A) or out_v (AT/G) = scale_out · Σ/(4π), G negated when `negate`
  EPI_S = 1,         // s = ½ − Σ/(4π); partial Σ s²
  EPI_SQ = 2,        // partial Σ (Σ/(4π))² only
  EPI_R = 3,         // r = Σ/(4π); partial Σ|r|²
  EPI_RESCALE = 4    // μ_out = μ̂ |μ'| / |μ̂| (μ̂ = Σ/(4π)); keep μ' if |μ̂| = 0
};
constexpr int kMaxPeers = 8;  // ranks of the peer-memory exchange (one NVLink / NVSwitch node)
struct TravArgs {
  int op = OP_A;
  int epi = EPI_PLAIN;
  NodeSet nodes;                 // decisions + representative positions + (by default) attributes
  const float4* attr = nullptr;  // optional override of the records supplying V (frozen geometry)
  const float4* pts = nullptr;   // sorted sources
  const float4* vec = nullptr;   // leaf-point vector attributes (sorted)
  const float* scal = nullptr;   // leaf-point scalar attributes (sorted)
  const int32_t* nrange_pb = nullptr;
  const int32_t* nrange_pe = nullptr;
  const float4* queries = nullptr;  // query points (normalized)
  int64_t q_begin = 0, q_end = 0;   // query index range (positions in the schedule)
  const int32_t* qorder = nullptr;  // schedule position → query index (null: identity)
  const int32_t* out_map = nullptr; // output index = out_map[q] (perm) or q
  float* out_f = nullptr;
  float4* out_v4 = nullptr;         // float4 output (internal vectors)
  float* out_v3 = nullptr;          // N×3 output (caller layout)
  float scale_out = 1.0f;
  const float4* mup = nullptr;      // EPI_RESCALE: μ'
  double* partial = nullptr;        // per-group partials (indexed by schedule position / kPartQ)
  float w2 = 0.0f;
  int stack_depth = 128;
  int root_single = 0;              // 1 iff the root is a one-point leaf (n = 1)
  int order1 = 0;                   // first-order far field (nodes.ext), row f2
  int split = 0;                    // small clouds: warps per query group (0: one-warp kernel; 4 or 8, traverse.cu)
  bool nowork = false;              // keep this launch out of the wn_work_count totals
  int prof_cls = -1;                // profiling class override (-1: by operator)
  int64_t nnodes = 0, npts = 0;     // sizes (WN_DEBUG bounds checks)
  int64_t* work = nullptr;          // set by traverse(): counting variant accumulates 4 totals
  int32_t* qcounts = nullptr;       // optional per-query (tests, far, leaf points, live terms), output order
  int32_t* wvisits = nullptr;       // optional (counting variant, one-warp kernel): per schedule warp, child visits + leaf points
  int wstride = 1;                  // traverse_visits: count every wstride-th warp of the schedule (wvisits compact)
  // peer-memory exchange (multi-GPU, fused): the epilogue stores its row / block partial into every rank's
  // replica and the last block signals every rank; world = 0 ⇒ local outputs only
  int world = 0;
  float* peer_f[kMaxPeers] = {};
  float4* peer_v4[kMaxPeers] = {};
  double* peer_part[kMaxPeers] = {};
  unsigned long long* peer_sig[kMaxPeers] = {};
  unsigned int* done = nullptr;
};
wn_status traverse(const TravArgs& a, cudaStream_t s);
wn_status traverse_visits(const TravArgs& a, cudaStream_t s);  // per-warp visits only (a.wvisits)

// ---- peer-memory exchange arena (comm.cu): every rank's replicas of the exchanged arrays ----
struct PeerArena {
  int world = 0, rank = 0;
  int64_t cap = 0, part_stride = 0;
  void* own = nullptr;                 // this rank's cudaMalloc block (IPC-exported)
  void* base[kMaxPeers] = {};          // every rank's block, mapped here (own or IPC-opened)
  bool opened[kMaxPeers] = {};
  float* s[kMaxPeers] = {};            // s = ½ − Aμ            (N)
  float4* r[kMaxPeers] = {};           // r = Aᵀ s              (N)
  float4* mu[2][kMaxPeers] = {};       // μ, ping-pong by iteration parity (N each)
  double* part[kMaxPeers] = {};        // Σ partials [3][blocks]
  double* vb[kMaxPeers] = {};          // transpose-mode adjoint: node accumulators V_B (node_cap × 3)
  double* u[kMaxPeers] = {};           //   and the near-field accumulators U_j (N × 3) of each rank's shard
  int64_t node_cap = 0;                // nodes the vb block holds (kArenaNodesPerPoint · N)
  unsigned long long* sig[kMaxPeers] = {};  // signal words (remote atomic adds)
  unsigned long long* expected = nullptr;   // local: next wait target (advanced by the wait kernel)
  int64_t pending_n = 0;                    // local communicators: exported for this N, not yet imported
  unsigned int* done = nullptr;             // local: finished blocks of the running traversal
};

// ---- fast multipole evaluation (fmm.cu) ----
// op OP_A: out (sorted or out_map order) = scale·V; OP_G: scale·(−∇V) for dipoles vec; OP_AT: scale·(−∇V)
// for charges scal; counts: M2L cell pairs, P2P leaf pairs
wn_status fmm_plan(wn_tree_s* t, int p, double theta, int leafsz, float wsep, cudaStream_t s);  // cached per tree
void fmm_plan_free(FmmPlan& F);
wn_status fmm_run(wn_tree_s* t, int op, const float4* vec, const float* scal, float w, const int32_t* out_map,
                  float* out, float4* out4, double scale, cudaStream_t s);
// the solver's elementwise steps around FMM operators (sorted order; Σ partials per 32 points)
void fmm_epi_s(int64_t n, const float* V, float* sv, double* part, cudaStream_t s);
void fmm_epi_sq(int64_t n, const float* V, double* part, cudaStream_t s);
void fmm_epi_r(int64_t n, const float4* r, double* part, cudaStream_t s);
void fmm_axpy(int64_t n, const float4* mu, const float4* r, const double* alpha, float4* mup, cudaStream_t s);
void fmm_epi_rescale(int64_t n, const float4* hat, const float4* mup, float4* mu, cudaStream_t s);

// ---- transpose-mode adjoint (transpose.cu) ----
// node / point accumulators, allocated once per tree — before any graph capture that uses them
wn_status ensure_transpose_scratch(wn_tree_s* t, cudaStream_t st);
wn_status adjoint_transpose(wn_tree_s* t, const NodeSet& geo, const float* s_sorted, float w2,
                            float4* r_out, double* partial, cudaStream_t st);
// multi-GPU form: (1) each rank scatters its shard [q0, q1) of the schedule into its own accumulators
// vb (nodes × 3) and u (N × 3); (2) after every rank has scattered, each rank adds all ranks' accumulators
// in rank order (identical sums on every rank) and pushes them down for every point, so r and its Σ|r|²
// partials are whole on every rank without a further exchange
wn_status adjoint_scatter_shard(wn_tree_s* t, const NodeSet& geo, const float* s_sorted, float w2, int64_t q0,
                                int64_t q1, double* vb, double* u, cudaStream_t st);
wn_status adjoint_reduce_pushdown(wn_tree_s* t, const double* const* vbs, const double* const* us, int world,
                                  float4* r_out, double* partial, cudaStream_t st);
constexpr int kArenaNodesPerPoint = 3;  // node capacity of a peer arena's transpose accumulators, per point

// ---- small utility kernels (iterate.cu) ----
#ifndef WN_EXP_TRAVBLOCK
#define WN_EXP_TRAVBLOCK 128
#endif
constexpr int kTravBlock = WN_EXP_TRAVBLOCK;  // queries per block (4 warps: the block tail holds an SM slot for less; 256: +0.8 %)
static_assert(WN_SHARD_ALIGN % kTravBlock == 0, "rank shards must hold whole traversal blocks (Σ partials)");
inline int trav_blocks(int64_t nq) { return (int)((nq + kTravBlock - 1) / kTravBlock); }
// Σ partials (s², |r|², (Ar)²) are kept per 32-query warp group of the query schedule: each warp writes its
// own slot (no block barrier in the epilogues), and α sums the slots in one fixed order
constexpr int kPartQ = 32;
constexpr int kAlphaBlocks = 32;  // blocks of the α reduction (ops.cu:k_alpha)
constexpr size_t alpha_words() { return 1 + 3 * kAlphaBlocks + 1; }
static_assert(WN_SHARD_ALIGN % kPartQ == 0, "rank shards must hold whole partial groups");
__host__ __device__ inline int64_t part_slots(int64_t nq) { return (nq + kPartQ - 1) / kPartQ; }

}  // namespace wn
