// capi.cu — the extern "C" surface of include/wn.h: argument checks, error reporting, launch accounting,
// and the host orchestration of the operators and of Alg. 3.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <algorithm>
#include <vector>

#include "wn_comm.cuh"
#include "wn_internal.cuh"
#include "wn_ops.cuh"

namespace wn {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

wn_status set_error(wn_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

wn_status cuda_status(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? WN_ERR_OOM : WN_ERR_CUDA;
}

static thread_local bool g_capturing = false;  // inside a CUDA-graph capture of the iteration loop

void count_launches(int n) {
  if (!g_capturing) g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed);
}

// ---- profiling: CUDA events on the launching stream ----
struct ProfRec {
  int cls;
  int nlaunch;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;

ProfScope::ProfScope(int c, cudaStream_t st, int nlaunch) : cls(c), s(st) {
  if (g_capturing) return;  // recorded into a graph: counted per graph launch instead
  count_launches(nlaunch);
  if (!g_prof_on) return;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof.push_back({c, nlaunch, a, b});
}
ProfScope::~ProfScope() {
  if (b) cudaEventRecord(b, s);
}

// ---- algorithmic-work counting (node tests, representative terms, leaf-point terms per class) ----
static bool g_count_on = false;
static int64_t* g_work = nullptr;

int64_t* work_counters(int cls) {
  if (!g_count_on || !g_work || cls < 0 || cls > 2) return nullptr;
  return g_work + 4 * cls;
}

void invalidate_graph(wn_tree_s* t) {
  if (t->graph_exec) cudaGraphExecDestroy(t->graph_exec);
  t->graph_exec = nullptr;
  t->graph_key.clear();
}

// marks the end of a call on a tree: free_tree waits for this point of the caller's stream
struct TreeUse {
  wn_tree_s* t;
  cudaStream_t s;
  TreeUse(wn_tree_s* tree, void* stream) : t(tree), s((cudaStream_t)stream) {}
  ~TreeUse() {
    if (t && t->done_ev) cudaEventRecord(t->done_ev, s);
  }
};

static wn_status check_device() {
  int dev = 0, n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return set_error(WN_ERR_CUDA, "no CUDA device available (libwn has no CPU path)");
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(WN_ERR_CUDA, "cudaGetDevice failed");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return set_error(WN_ERR_CUDA, "libwn is built for sm_100a (B200); device is not compute 10.x");
  // keep freed stream-ordered allocations cached in the device pool (tree builds reuse them)
  static bool pool_done[64] = {false};
  if (dev < 64 && !pool_done[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_done[dev] = true;
  }
  return WN_OK;
}

static wn_status ensure_scratch(wn_tree_s* t, cudaStream_t s) {
  IterScratch& it = t->it;
  if (it.mu) return WN_OK;
  const int64_t n = t->n;
  it.n = n;
  it.nblk = (int)part_slots(n);
  WN_CUDA(cudaMallocAsync((void**)&it.mu, n * sizeof(float4), s));
  WN_CUDA(cudaMallocAsync((void**)&it.mup, n * sizeof(float4), s));
  WN_CUDA(cudaMallocAsync((void**)&it.r, n * sizeof(float4), s));
  WN_CUDA(cudaMallocAsync((void**)&it.s, n * sizeof(float), s));
  WN_CUDA(cudaMallocAsync((void**)&it.tmp, n * sizeof(float4), s));
  WN_CUDA(cudaMallocAsync((void**)&it.part, 3 * (size_t)it.nblk * sizeof(double), s));
  WN_CUDA(cudaMallocAsync((void**)&it.alpha, alpha_words() * sizeof(double), s));
  WN_CUDA(cudaMemsetAsync(it.alpha, 0, alpha_words() * sizeof(double), s));  // (the reduction's ticket = 0)
  return WN_OK;
}

static int stack_depth(const wn_tree_s* t) { return 8 * (t->depth_used + 2); }

// per-iteration stats buffer (E, α, Σr², Σ(Ar)², w per iteration) of at least `iters` rows; growing it
// frees the old block, which a cached CUDA graph may still reference: the graph is dropped with it
static wn_status ensure_dstats(wn_tree_s* t, int iters, cudaStream_t s) {
  IterScratch& it = t->it;
  if (it.stats_cap >= iters) return WN_OK;
  invalidate_graph(t);
  if (it.dstats) cudaFreeAsync(it.dstats, s);
  if (it.dcounts) cudaFreeAsync(it.dcounts, s);
  it.dstats = nullptr;
  it.dcounts = nullptr;
  it.stats_cap = 0;
  WN_CUDA(cudaMallocAsync((void**)&it.dstats, 5 * sizeof(double) * (size_t)iters, s));
  WN_CUDA(cudaMallocAsync((void**)&it.dcounts, 12 * sizeof(int64_t) * (size_t)(iters + 1), s));
  if (it.dstamp) cudaFreeAsync(it.dstamp, s);
  it.dstamp = nullptr;
  WN_CUDA(cudaMallocAsync((void**)&it.dstamp, sizeof(unsigned long long) * (size_t)(iters + 1), s));
  it.stats_cap = iters;
  return WN_OK;
}

// per-iteration device time: the global nanosecond timer at each iteration boundary (a one-thread kernel;
// works inside the captured graph, where event timing is not available); only for calls that ask for stats
constexpr int kFlagStamps = 1 << 16;  // internal wnnc_params flag (part of the graph key)
__global__ void k_stamp(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}
static void stamp(wn_tree_s* t, const wnnc_params& p, int row, cudaStream_t s) {
  if (!(p.flags & kFlagStamps)) return;
  k_stamp<<<1, 1, 0, s>>>(t->it.dstamp + row);
  count_launches(1);
}

// per-iteration work counts (only while counting is on): snapshot of the class totals
static void snap_counts(wn_tree_s* t, int row, cudaStream_t s) {
  if (g_count_on && g_work) cudaMemcpyAsync(t->it.dcounts + 12 * row, g_work, 12 * sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
}

// several warps per query group below this many queries (too few query warps to fill the GPU otherwise);
// decided on the whole cloud, so every rank of a sharded run picks the same kernel
static int64_t split_max() {
  static int64_t v = [] {
    const char* e = getenv("WN_SPLIT_MAX");
    return e ? (int64_t)atoll(e) : (int64_t)60000;  // measured: C2 (50k) −25 %, a 65k subset of C3 +10 %
  }();
  return v;
}

// warps per 32-query group of the small-cloud kernel, from the whole query count (every rank the same):
// 8 up to 512 groups, else 4 (measured on C3 subsets and C1/C2: 5k / 12k points −14 % / −8 % with 8,
// 25k / 45k +27 % / +39 %)
static int split_factor(int64_t nq) { return (nq + 31) / 32 <= 512 ? 8 : 4; }

static TravArgs base_args(const wn_tree_s* t, float w2) {
  TravArgs a;
  a.pts = t->pts;
  a.nrange_pb = t->pb;
  a.nrange_pe = t->pe;
  a.queries = t->pts;
  a.q_begin = 0;
  a.q_end = t->n;
  a.w2 = w2;
  a.stack_depth = stack_depth(t);
  a.root_single = t->n == 1;
  a.qorder = t->qorder;
  a.nnodes = t->nn;
  a.npts = t->n;
  a.split = t->n <= split_max() ? split_factor(t->n) : 0;
  return a;
}

static bool bad_width(float w) { return !(w > 0.f) || std::isnan(w); }
static bool bad_theta(float c) { return !(c > 0.f) || std::isnan(c); }

// per WN_SHARD_ALIGN block of the query schedule: its queries' node tests (from a counting traversal)
__global__ void k_block_work(int64_t n, const int32_t* __restrict__ qorder, const int32_t* __restrict__ cnt,
                             int64_t b0, int64_t b1, int64_t* __restrict__ bw) {
  const int64_t b = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= b1) return;
  int64_t w = 0;
  const int64_t k1 = std::min<int64_t>(n, (b + 1) * WN_SHARD_ALIGN);
  for (int64_t k = b * WN_SHARD_ALIGN; k < k1; ++k) w += cnt[4 * (int64_t)(qorder ? qorder[k] : k)];
  bw[b] = w;
}

// Work-weighted query shards for `world` ranks: the per-block node tests of the A traversal
// over the fixed unit-weight geometry (decisions do not depend on the width; the representatives of later
// attributes move little) — counted by each rank over its equal-count share and summed over the ranks
// (comm), or all here (emulated ranks) — then rank r starts at the first block where the running work
// reaches r/world of the total.  Shards only decide which rank computes which blocks: every result is
// unchanged.  Cached on the tree per world size; computed outside any graph capture.
static wn_status plan_shards(wn_tree_s* t, int world, wn_comm comm, cudaStream_t s) {
  ShardPlan& P = t->shard;
  if (world <= 1 || world > kMaxShardRanks) {
    P.world = 0;
    return WN_OK;
  }
  if (P.world == world) return WN_OK;
  IterScratch& it = t->it;
  const int64_t n = t->n, nb = (n + WN_SHARD_ALIGN - 1) / WN_SHARD_ALIGN;
  int64_t q0 = 0, q1 = n;
  if (comm && !comm_has_nccl(comm)) comm = nullptr;  // a local communicator: every rank counts all blocks
  if (comm) wn_shard_range(n, comm_rank(comm), world, &q0, &q1);
  int64_t* bw = nullptr;
  WN_CUDA(cudaMallocAsync((void**)&bw, nb * sizeof(int64_t), s));
  WN_CUDA(cudaMemsetAsync(bw, 0, nb * sizeof(int64_t), s));
  TravArgs ca = base_args(t, 0.0f);
  ca.op = OP_A;
  ca.epi = EPI_PLAIN;
  ca.nodes = t->set[1];
  ca.vec = it.mu;  // (values unused: only the decisions are counted)
  ca.q_begin = q0;
  ca.q_end = q1;
  ca.out_map = nullptr;
  ca.qcounts = reinterpret_cast<int32_t*>(it.tmp);  // n × 4 int32, indexed by query
  ca.nowork = true;
  ca.prof_cls = WN_PROF_OTHER;
  wn_status st = traverse(ca, s);
  if (st == WN_OK && q1 > q0) {
    const int64_t b0 = q0 / WN_SHARD_ALIGN, b1 = (q1 + WN_SHARD_ALIGN - 1) / WN_SHARD_ALIGN;
    k_block_work<<<(unsigned)((b1 - b0 + 255) / 256), 256, 0, s>>>(n, t->qorder, ca.qcounts, b0, b1, bw);
    count_launches(1);
  }
  if (st == WN_OK && comm) st = comm_allreduce_i64(comm, bw, nb, s);
  std::vector<int64_t> h(nb);
  if (st == WN_OK) {
    cudaError_t e = cudaMemcpyAsync(h.data(), bw, nb * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_status(e, "shard plan");
  }
  cudaFreeAsync(bw, s);
  if (st != WN_OK) return st;
  int64_t total = 0;
  for (int64_t v : h) total += v + 1;  // + 1: a block costs something even when empty of tests
  P.b[0] = 0;
  int64_t run = 0, blk = 0;
  for (int r = 1; r < world; ++r) {
    const int64_t target = (total * r) / world;  // (exact integer arithmetic: identical on every rank)
    while (blk < nb && run + h[blk] + 1 <= target) run += h[blk++] + 1;
    P.b[r] = std::min<int64_t>(n, blk * WN_SHARD_ALIGN);
  }
  P.b[world] = n;
  P.world = world;
  return WN_OK;
}

// ---- query schedule: k-d boxes or Hilbert runs (tree_build.cu:kd_schedule / hilbert_schedule) ----
// Both are permutations of the same queries, so every result is unchanged; what differs is the work of
// each warp. k-d boxes are more compact (fewer visits in total) but put isolated queries (outliers)
// together, and a warp of mutually distant queries is a long serial chain that can outlast the rest of
// the launch (C4: the heaviest warp 1.4× Hilbert's, the A traversal 1.4× slower). The choice counts the
// warp-level visits of the A traversal over the unit-weight geometry (no cutoff: the shard planner's
// estimate) under both and keeps k-d only if it visits less in total and its heaviest warp is no heavier
// than Hilbert's (C4 with k-d: 5 % fewer visits, heaviest warp +7 %, solve +5 %). Deterministic (integer
// counts): every rank takes the same schedule.
#ifndef WN_EXP_QSCHED
#define WN_EXP_QSCHED 2  // 0: Hilbert, 1: k-d, 2: chosen per tree
#endif
constexpr int64_t kKdMinPoints = 4096;  // below: Hilbert (the choice would cost more than it saves)
constexpr int kSampleStride = 4;        // the choice counts every 4th warp of each schedule

__global__ void __launch_bounds__(1024) k_sum_max(const int32_t* __restrict__ v, int64_t m, long long* __restrict__ out) {
  __shared__ long long ss[32], sx[32];
  long long sm = 0, mx = 0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    sm += v[i];
    mx = max(mx, (long long)v[i]);
  }
  for (int o = 16; o; o >>= 1) {
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    ss[threadIdx.x >> 5] = sm;
    sx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      sm += ss[k];
      mx = max(mx, sx[k]);
    }
    out[0] = sm;
    out[1] = mx;
  }
}

static wn_status schedule_cost(wn_tree_s* t, const int32_t* order, int stride, int32_t* wv, long long* dev2,
                               cudaStream_t s) {
  TravArgs ca = base_args(t, 0.0f);
  ca.op = OP_A;
  ca.epi = EPI_PLAIN;
  ca.nodes = t->set[1];
  ca.vec = t->it.mu;  // (values unused: only the visits are counted)
  ca.qorder = order;
  ca.out_map = nullptr;
  ca.wvisits = wv;
  ca.wstride = stride;
  ca.nowork = true;
  ca.prof_cls = WN_PROF_OTHER;
  WN_TRY(traverse_visits(ca, s));
  k_sum_max<<<1, 1024, 0, s>>>(wv, ((t->n + 31) / 32 + stride - 1) / stride, dev2);
  count_launches(1);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

// new schedule = the old one with its kTravBlock-query chunks permuted (chunk j of the new = perm[j] of the old)
__global__ void k_permute_chunks(const int32_t* __restrict__ src, int32_t* __restrict__ dst, const int32_t* __restrict__ perm,
                                 int64_t n) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  dst[k] = src[(int64_t)perm[k / kTravBlock] * kTravBlock + k % kTravBlock];
}

static wn_status choose_schedule(wn_tree_s* t, cudaStream_t s) {
  t->sched_kind = 0;
  if (WN_EXP_QSCHED == 0 || t->n < kKdMinPoints) return WN_OK;
  WN_TRY(ensure_scratch(t, s));
  const int64_t n = t->n, nw = (n + 31) / 32, nb = (n + kTravBlock - 1) / kTravBlock;
  int32_t *kd = nullptr, *wv = nullptr, *perm = nullptr;
  long long* dev = nullptr;
  cudaError_t ae = cudaMallocAsync((void**)&kd, n * sizeof(int32_t), s);
  if (ae == cudaSuccess) ae = cudaMallocAsync((void**)&wv, 2 * nw * sizeof(int32_t), s);
  if (ae == cudaSuccess) ae = cudaMallocAsync((void**)&perm, nb * sizeof(int32_t), s);
  if (ae == cudaSuccess) ae = cudaMallocAsync((void**)&dev, 4 * sizeof(long long), s);
  // the choice compares every kSampleStride-th warp of both schedules (the sample total, its heaviest warp);
  // the heaviest-first Hilbert order below counts every warp
  wn_status st = ae == cudaSuccess ? kd_schedule(t->pts, n, kd, s) : cuda_status(ae, "schedule scratch");
  if (st == WN_OK) st = schedule_cost(t, t->qorder, kSampleStride, wv, dev, s);
  if (st == WN_OK) st = schedule_cost(t, kd, kSampleStride, wv + nw, dev + 2, s);
  long long h[4] = {};
  if (st == WN_OK) {
    cudaError_t e = cudaMemcpyAsync(h, dev, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_status(e, "schedule choice");
  }
  const bool use_kd = WN_EXP_QSCHED == 1 || (h[2] < h[0] && h[3] <= h[1]);
  std::vector<int32_t> hw(nw);
  if (st == WN_OK && !use_kd) {
    st = schedule_cost(t, t->qorder, 1, wv, dev, s);
    cudaError_t e = st == WN_OK ? cudaMemcpyAsync(hw.data(), wv, nw * sizeof(int32_t), cudaMemcpyDeviceToHost, s)
                                : cudaSuccess;
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_status(e, "schedule costs");
  }
  if (st == WN_OK) {
    for (int k = 0; k < 4; ++k) t->sched_stats[k] = h[k];
    cudaError_t e = cudaSuccess;
    if (use_kd) {  // (heaviest blocks first measured here too: +1 % at C2, C3, C5 — not done)
      e = cudaMemcpyAsync(t->qorder, kd, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
      t->sched_kind = 1;
    } else {
      // Hilbert: launch the heaviest blocks first (cost = the block's heaviest warp; a ragged last block
      // stays last) — the long chains then overlap the rest of the launch (C4: 75.0 → 69.1 ms per solve)
      std::vector<int64_t> cost(nb, 0);
      for (int64_t w = 0; w < nw; ++w) cost[w / (kTravBlock / 32)] = std::max<int64_t>(cost[w / (kTravBlock / 32)], hw[w]);
      std::vector<int32_t> hp(nb);
      for (int64_t b = 0; b < nb; ++b) hp[b] = (int32_t)b;
      const int64_t full = n % kTravBlock == 0 ? nb : nb - 1;
      std::stable_sort(hp.begin(), hp.begin() + full, [&](int32_t x, int32_t y) { return cost[x] > cost[y]; });
      e = cudaMemcpyAsync(perm, hp.data(), nb * sizeof(int32_t), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) {
        k_permute_chunks<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(t->qorder, kd, perm, n);
        count_launches(1);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaMemcpyAsync(t->qorder, kd, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // (hp is a host buffer of this frame)
    }
    if (e != cudaSuccess) st = cuda_status(e, "schedule copy");
  }
  for (void* p : {(void*)kd, (void*)wv, (void*)perm, (void*)dev})
    if (p) cudaFreeAsync(p, s);
  return st;
}

// route a traversal's outputs into every rank's replica (peer-memory exchange); none when P is null
static void peer_route(TravArgs& ta, const PeerArena* P, float* const* f, float4* const* v4, int part_slot) {
  if (!P) return;
  ta.world = P->world;
  for (int r = 0; r < P->world; ++r) {
    if (f) ta.peer_f[r] = f[r];
    if (v4) ta.peer_v4[r] = v4[r];
    ta.peer_part[r] = P->part[r] + part_slot * P->part_stride;
    ta.peer_sig[r] = P->sig[r];
  }
  ta.done = P->done;
}

// ---- Alg. 3 loop over a query range [q0, q1) of the sorted points (multi-GPU: this rank's shard) ----
// Exchanges (multi-GPU): with peer-memory arenas the traversal epilogues store into every rank's replica
// and a device-side wait follows each exchanging traversal; μ ping-pongs between the arena's two buffers
// (iteration i reads μ[i % 2], its G epilogue writes μ[(i + 1) % 2]).  `views` are the ranks this process
// drives: normally one (its own rank; moments, α and μ' from its replica); several when W ranks are
// emulated on one GPU (wnnc_iterate_emulated: each rank's traversal over its shard and its own replica,
// serialized on one stream, all waits after all signals).  No views but a comm: NCCL broadcasts.
static wn_status run_iterations(wn_tree_s* t, const wnnc_params& p, wn_comm comm, const PeerArena* const* views,
                                int nviews, cudaStream_t s) {
  IterScratch& it = t->it;
  const int total = p.total_iters > 0 ? p.total_iters : p.iters;
  const bool transpose = p.adjoint_mode == WN_ADJ_TRANSPOSE;
  const PeerArena* P = nviews > 0 ? views[0] : nullptr;
  int64_t q0 = 0, q1 = t->n;
  if (comm && !P) shard_of(&t->shard, t->n, comm_rank(comm), comm_world(comm), &q0, &q1);
  const bool nccl = comm && !P;
  const int me = P ? P->rank : 0;
  float* sb = P ? P->s[me] : it.s;
  float4* rb = P ? P->r[me] : it.r;
  double* part = P ? P->part[me] : it.part;
  const int64_t stride = P ? P->part_stride : it.nblk;
  // queries follow the Hilbert schedule; multi-GPU shards are schedule ranges (exchanged via staging)
  const int32_t* qord = t->qorder;
  float* stage = (float*)it.tmp;  // n × 4 floats
  // one exchanging traversal: every view's shard (inputs from its own replica), then every view's wait
  enum Rows { NONE, S, R, MU0, MU1 };
  auto run_traversal = [&](const TravArgs& ta, int slot, Rows in, Rows out) -> wn_status {
    if (!P) {
      TravArgs tv = ta;
      tv.q_begin = q0;
      tv.q_end = q1;
      return traverse(tv, s);
    }
    for (int v = 0; v < nviews; ++v) {
      const PeerArena& A = *views[v];
      TravArgs tv = ta;
      shard_of(&t->shard, t->n, A.rank, A.world, &tv.q_begin, &tv.q_end);
      if (in == S) tv.scal = A.s[A.rank];
      if (in == R) tv.vec = A.r[A.rank];
      if (in == MU0 || in == MU1) tv.vec = A.mu[in == MU1][A.rank];
      peer_route(tv, &A, out == S ? A.s : nullptr,
                 out == R ? A.r : (out == MU0 || out == MU1) ? A.mu[out == MU1] : nullptr, slot);
      WN_TRY(traverse(tv, s));
    }
    for (int v = 0; v < nviews; ++v) {
      if (p.flags & WN_FLAG_HOST_WAIT) WN_TRY(comm_peer_wait_host(*views[v], s));
      else comm_peer_wait(*views[v], s);
    }
    return WN_OK;
  };
  stamp(t, p, 0, s);
  snap_counts(t, 0, s);
  if (t->fmm_p > 0) {  // row f4: every operator by FMM (single GPU, gather semantics: each operator from its own attribute)
    for (int i = 0; i < p.iters; ++i) {
      const int k = p.first_iter + i;
      const float w = width_at(k, total, (double)p.w_min, (double)p.w_max);
      const int64_t n = t->n;
      float* V = reinterpret_cast<float*>(it.tmp);  // n floats of the n × 4 scratch
      if (i == 0 && k == 1 && (p.flags & WN_FLAG_MU_ZERO)) {
        s_half(n, it.s, it.part, s);
      } else {
        WN_TRY(fmm_run(t, OP_A, it.mu, nullptr, w, nullptr, V, nullptr, 1.0, s));
        fmm_epi_s(n, V, it.s, it.part, s);
      }
      WN_TRY(fmm_run(t, OP_AT, nullptr, it.s, w, nullptr, nullptr, it.r, 1.0, s));
      fmm_epi_r(n, it.r, it.part + it.nblk, s);
      WN_TRY(fmm_run(t, OP_A, it.r, nullptr, w, nullptr, V, nullptr, 1.0, s));
      fmm_epi_sq(n, V, it.part + 2 * (int64_t)it.nblk, s);
      alpha_step(it.part, (int)part_slots(n), it.nblk, (double)w, it.alpha, it.dstats + 5 * i, s);
      fmm_axpy(n, it.mu, it.r, it.alpha, it.mup, s);
      float4* hat = reinterpret_cast<float4*>(it.tmp);  // μ̂ = G(μ') (the n × 4 scratch; V is no longer needed)
      WN_TRY(fmm_run(t, OP_G, it.mup, nullptr, w, nullptr, nullptr, hat, 1.0, s));
      fmm_epi_rescale(n, hat, it.mup, it.mu, s);
      stamp(t, p, i + 1, s);
      snap_counts(t, i + 1, s);
    }
    return WN_OK;
  }
  for (int i = 0; i < p.iters; ++i) {
    const int k = p.first_iter + i;
    const float w = width_at(k, total, (double)p.w_min, (double)p.w_max);
    const float w2 = w * w;
    const int cur = i & 1;
    float4* mu_cur = P ? P->mu[cur][me] : it.mu;
    // (1) s = ½ − A_w μ  (+ Σ s² partials)
    if (i == 0 && k == 1 && (p.flags & WN_FLAG_MU_ZERO) && !transpose) {
      // μ⁰ = 0: A(0) = 0 term by term, s = ½ exactly — every rank fills its whole replica
      if (P)
        for (int v = 0; v < nviews; ++v) s_half(t->n, views[v]->s[views[v]->rank], views[v]->part[views[v]->rank], s);
      else
        s_half(t->n, sb, part, s);
    } else {
      MomentArgs m1;
      m1.kind = ATTR_VEC;
      m1.vec = mu_cur;
      m1.theta = p.theta;
      m1.out = transpose ? t->set[1] : t->set[0];
      m1.order1 = t->far_order == 1;
      WN_TRY(build_moments(t, m1, s));
      TravArgs a1 = base_args(t, w2);
      a1.qorder = qord;
      a1.op = OP_A;
      a1.epi = EPI_S;
      a1.nodes = m1.out;
      a1.vec = mu_cur;
      a1.out_f = sb;
      a1.partial = part;
      a1.order1 = t->far_order;
      WN_TRY(run_traversal(a1, 0, cur ? MU1 : MU0, S));
      if (nccl) WN_TRY(comm_allgather_f(comm, sb, 1, t->n, qord, stage, &t->shard, s));
    }
    // (2) r = A_wᵀ s  (+ Σ|r|² partials)
    if (transpose && !comm && !P) {
      WN_TRY(adjoint_transpose(t, t->set[1], sb, w2, rb, part + stride, s));
    } else if (transpose && P) {
      // multi-GPU transpose form: every view scatters its shard into its own replica's accumulators and
      // signals; after all signals each view adds every rank's accumulators (rank order) and pushes down
      // for all points into its own replica — r and the Σ|r|² partials are whole on every rank
      for (int v = 0; v < nviews; ++v) {
        const PeerArena& A = *views[v];
        int64_t b = 0, e = 0;
        shard_of(&t->shard, t->n, A.rank, A.world, &b, &e);
        WN_TRY(adjoint_scatter_shard(t, t->set[1], A.s[A.rank], w2, b, e, A.vb[A.rank], A.u[A.rank], s));
        comm_peer_signal(A, s);
      }
      for (int v = 0; v < nviews; ++v) {
        if (p.flags & WN_FLAG_HOST_WAIT) WN_TRY(comm_peer_wait_host(*views[v], s));
        else comm_peer_wait(*views[v], s);
      }
      for (int v = 0; v < nviews; ++v) {
        const PeerArena& A = *views[v];
        WN_TRY(adjoint_reduce_pushdown(t, A.vb, A.u, A.world, A.r[A.rank], A.part[A.rank] + stride, s));
      }
    } else if (transpose) {  // NCCL: all-reduce of the accumulators, then the same replicated push-down
      WN_TRY(ensure_transpose_scratch(t, s));
      WN_TRY(adjoint_scatter_shard(t, t->set[1], sb, w2, q0, q1, t->tvb, t->tu, s));
      WN_TRY(comm_allreduce_f64(comm, t->tvb, 3 * t->nn, s));
      WN_TRY(comm_allreduce_f64(comm, t->tu, 3 * t->n, s));
      const double* vb1[1] = {t->tvb};
      const double* u1[1] = {t->tu};
      WN_TRY(adjoint_reduce_pushdown(t, vb1, u1, 1, rb, part + stride, s));
    } else {
      MomentArgs m2;
      m2.kind = ATTR_SCALAR;
      m2.scal = sb;
      m2.theta = p.theta;
      m2.out = t->set[0];
      m2.order1 = t->far_order == 1;
      WN_TRY(build_moments(t, m2, s));
      TravArgs a2 = base_args(t, w2);
      a2.qorder = qord;
      a2.op = OP_AT;
      a2.epi = EPI_R;
      a2.nodes = t->set[0];
      a2.scal = sb;
      a2.out_v4 = rb;
      a2.partial = part + stride;
      a2.order1 = t->far_order;
      WN_TRY(run_traversal(a2, 1, S, R));
      if (nccl) WN_TRY(comm_allgather_f(comm, (float*)rb, 4, t->n, qord, stage, &t->shard, s));
    }
    // (3) Σ (A_w r)²  — gather: r's own representatives; transpose: μ's frozen geometry
    MomentArgs m3;
    m3.kind = ATTR_VEC;
    m3.vec = rb;
    m3.theta = p.theta;
    m3.out = t->set[0];
    m3.order1 = t->far_order == 1;
    WN_TRY(build_moments(t, m3, s));
    TravArgs a3 = base_args(t, w2);
    a3.qorder = qord;
    a3.op = OP_A;
    a3.epi = EPI_SQ;
    a3.nodes = transpose ? t->set[1] : t->set[0];
    a3.attr = transpose ? t->set[0].rec : nullptr;
    a3.vec = rb;
    a3.partial = part + 2 * stride;
    a3.order1 = t->far_order;
    WN_TRY(run_traversal(a3, 2, R, NONE));
    if (nccl) WN_TRY(comm_allgather_partials(comm, part, stride, t->n, &t->shard, s));
    // α = Σr² / Σ(Ar)²  (Alg. 2), fixed-order reduction of the partials
    // (the partial arrays' stride may exceed this cloud's block count: a peer arena sized for a larger N)
    alpha_step(part, (int)part_slots(t->n), stride, (double)w, it.alpha, it.dstats + 5 * i, s);
    // (4) μ' = μ + α r (fused into the moment build), μ̂ = G_w(μ'), μ = μ̂ |μ'|/|μ̂|
    MomentArgs m4;
    m4.kind = ATTR_VEC;
    m4.vec = mu_cur;
    m4.axpy_r = rb;
    m4.alpha = it.alpha;
    m4.axpy_out = it.mup;
    m4.theta = p.theta;
    m4.out = t->set[0];
    m4.order1 = t->far_order == 1;
    WN_TRY(build_moments(t, m4, s));
    TravArgs a4 = base_args(t, w2);
    a4.qorder = qord;
    a4.op = OP_G;
    a4.epi = EPI_RESCALE;
    a4.nodes = t->set[0];
    a4.vec = it.mup;
    a4.mup = it.mup;
    a4.out_v4 = it.mu;
    a4.order1 = t->far_order;
    WN_TRY(run_traversal(a4, 0, NONE, cur ? MU0 : MU1));
    if (nccl) WN_TRY(comm_allgather_f(comm, (float*)it.mu, 4, t->n, qord, stage, &t->shard, s));
    stamp(t, p, i + 1, s);
    snap_counts(t, i + 1, s);
  }
  return WN_OK;
}

}  // namespace wn

using namespace wn;

extern "C" {

const char* wn_last_error(void) { return g_last_error.c_str(); }
const char* wn_version(void) { return "libwn 0.1 (sm_100a, " __DATE__ ")"; }
uint64_t wn_launch_count(void) { return g_launches.load(); }

wn_status wn_prof_enable(int32_t enable) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  g_prof_on = enable != 0;
  return WN_OK;
}

wn_status wn_prof_read(double ms[WN_PROF_NCLASS], int64_t launches[WN_PROF_NCLASS]) {
  for (int c = 0; c < WN_PROF_NCLASS; ++c) {
    ms[c] = 0.0;
    launches[c] = 0;
  }
  WN_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& r : g_prof) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) ms[r.cls] += t;
    launches[r.cls] += r.nlaunch;
  }
  return WN_OK;
}

wn_status wn_work_count_enable(int32_t enable) {
  if (enable && !g_work) WN_CUDA(cudaMalloc((void**)&g_work, 12 * sizeof(int64_t)));
  if (enable) WN_CUDA(cudaMemset(g_work, 0, 12 * sizeof(int64_t)));
  g_count_on = enable != 0;
  return WN_OK;
}

wn_status wn_work_count_read(int64_t counts[12]) {
  for (int k = 0; k < 12; ++k) counts[k] = 0;
  if (!g_work) return WN_OK;
  WN_CUDA(cudaDeviceSynchronize());
  WN_CUDA(cudaMemcpy(counts, g_work, 12 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return WN_OK;
}

wn_status wn_build_tree(const float* pts, int64_t n, int32_t max_depth, void* stream, wn_tree* out) {
  if (!out) return set_error(WN_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n < 1) return set_error(WN_ERR_EMPTY, "empty point set (n < 1)");
  if (!pts) return set_error(WN_ERR_ARG, "pts is NULL");
  if (max_depth < 1 || max_depth > kMaxDepth) return set_error(WN_ERR_ARG, "max_depth must be in [1, 21]");
  // 32-bit node byte offsets in the traversal (64-B records) bound the node count: n ≤ 2^25 points
  if (n > (int64_t)1 << 25) return set_error(WN_ERR_ARG, "n > 2^25 points is not supported");
  WN_TRY(check_device());
  wn_tree_s* t = new (std::nothrow) wn_tree_s();
  if (!t) return set_error(WN_ERR_OOM, "host allocation failed");
  cudaGetDevice(&t->device);
  const cudaError_t ee = cudaEventCreateWithFlags(&t->done_ev, cudaEventDisableTiming);
  wn_status st = ee == cudaSuccess ? build_tree(pts, n, max_depth, (cudaStream_t)stream, t)
                                   : cuda_status(ee, "cudaEventCreate");
  if (st == WN_OK) st = choose_schedule(t, (cudaStream_t)stream);
  if (t->done_ev) cudaEventRecord(t->done_ev, (cudaStream_t)stream);
  if (st != WN_OK) {
    free_tree(t);
    delete t;
    return st;
  }
  *out = t;
  return WN_OK;
}

wn_status wn_tree_destroy(wn_tree t) {
  if (!t) return WN_OK;
  free_tree(t);
  delete t;
  return WN_OK;
}

wn_status wn_tree_set_far_order(wn_tree t, int32_t order, void* stream) {
  TreeUse use_(t, stream);
  if (!t) return set_error(WN_ERR_ARG, "tree is NULL");
  if (order != 0 && order != 1) return set_error(WN_ERR_ARG, "far-field order must be 0 or 1");
  if (order == 1) WN_TRY(enable_order1(t, (cudaStream_t)stream));
  t->far_order = order;
  return WN_OK;
}

wn_status wn_tree_set_fmm(wn_tree t, int32_t p, float theta_f, int32_t leaf) {
  if (!t) return set_error(WN_ERR_ARG, "tree is NULL");
  if (p < 0 || p > 6) return set_error(WN_ERR_ARG, "FMM degree must be 0 (treecode) or 1..6");
  if (p > 0 && (leaf < 1 || leaf > 32 || !(theta_f > 0.f)))
    return set_error(WN_ERR_ARG, "FMM leaf must be in 1..32 and theta_f > 0");
  invalidate_graph(t);
  t->fmm_p = p;
  t->fmm_theta = theta_f;
  t->fmm_leaf = leaf;
  return WN_OK;
}

wn_status wn_tree_info(wn_tree t, int64_t* num_points, int64_t* num_nodes, int32_t* depth_used, double xform[4]) {
  if (!t) return set_error(WN_ERR_ARG, "tree is NULL");
  if (num_points) *num_points = t->n;
  if (num_nodes) *num_nodes = t->nn;
  if (depth_used) *depth_used = t->depth_used;
  if (xform)
    for (int a = 0; a < 4; ++a) xform[a] = t->xf[a];
  return WN_OK;
}

wn_status wn_tree_export(wn_tree t, uint64_t* keys, int32_t* perm, float* xn, int32_t* depth, int32_t* pb,
                         int32_t* pe, int32_t* child_begin, int32_t* child_count, void* stream) {
  TreeUse use_(t, stream);
  if (!t) return set_error(WN_ERR_ARG, "tree is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t N = t->n, NN = t->nn;
  if (keys) WN_CUDA(cudaMemcpyAsync(keys, t->keys, N * 8, cudaMemcpyDeviceToDevice, s));
  if (perm) WN_CUDA(cudaMemcpyAsync(perm, t->perm, N * 4, cudaMemcpyDeviceToDevice, s));
  if (xn) WN_CUDA(cudaMemcpy2DAsync(xn, 12, t->pts, 16, 12, N, cudaMemcpyDeviceToDevice, s));
  if (depth) WN_CUDA(cudaMemcpyAsync(depth, t->depth, NN * 4, cudaMemcpyDeviceToDevice, s));
  if (pb) WN_CUDA(cudaMemcpyAsync(pb, t->pb, NN * 4, cudaMemcpyDeviceToDevice, s));
  if (pe) WN_CUDA(cudaMemcpyAsync(pe, t->pe, NN * 4, cudaMemcpyDeviceToDevice, s));
  if (child_begin) WN_CUDA(cudaMemcpyAsync(child_begin, t->cb, NN * 4, cudaMemcpyDeviceToDevice, s));
  if (child_count) WN_CUDA(cudaMemcpyAsync(child_count, t->cc, NN * 4, cudaMemcpyDeviceToDevice, s));
  return WN_OK;
}

wn_status wn_moments(wn_tree t, const float* nu, int32_t dim, const float* a, float* rep, float* attr, double* W,
                     void* stream) {
  TreeUse use_(t, stream);
  if (!t || !nu) return set_error(WN_ERR_ARG, "tree or nu is NULL");
  if (dim != 1 && dim != 3) return set_error(WN_ERR_ARG, "dim must be 1 or 3");
  cudaStream_t s = (cudaStream_t)stream;
  WN_TRY(ensure_scratch(t, s));
  IterScratch& it = t->it;
  MomentArgs m;
  m.theta = 2.0f;
  m.out = t->set[0];
  if (dim == 3) {
    gather_vec_a(t->n, t->perm, nu, a, it.mu, it.s, it.mup, s);
    m.kind = ATTR_VEC;
    m.vec = it.mu;
  } else {
    gather_scal(t->n, t->perm, nu, it.s, s);
    if (a) gather_scal(t->n, t->perm, a, (float*)it.tmp, s);
    m.kind = ATTR_SCALAR;
    m.scal = it.s;
  }
  if (a) m.a_sorted = dim == 3 ? it.s : (const float*)it.tmp;
  m.write_W = W != nullptr;
  m.all_nodes = true;  // diagnostic export: every node's representative
  WN_TRY(build_moments(t, m, s));
  const size_t NN = t->nn;
  const size_t pitch = kRec * sizeof(float4);
  if (rep) WN_CUDA(cudaMemcpy2DAsync(rep, 12, t->set[0].rec, pitch, 12, NN, cudaMemcpyDeviceToDevice, s));
  if (attr)
    WN_CUDA(cudaMemcpy2DAsync(attr, 4 * dim, t->set[0].rec + 1, pitch, 4 * dim, NN, cudaMemcpyDeviceToDevice, s));
  if (W) WN_CUDA(cudaMemcpy2DAsync(W, 8, t->sums, 64, 8, NN, cudaMemcpyDeviceToDevice, s));
  return WN_OK;
}

// presorted: the queries are already spatially coherent (wn_iso_cells: corners in Morton order), so the
// per-call Hilbert schedule is skipped and warps take consecutive queries
static wn_status eval_common(wn_tree t, int op, const float* mu, const float* a, const float* q, int64_t m,
                             float width, float theta, float* out, void* stream, int32_t* qcounts = nullptr,
                             bool presorted = false) {
  TreeUse use_(t, stream);
  if (!t || !mu || (!out && !qcounts)) return set_error(WN_ERR_ARG, "tree, mu or output is NULL");
  if (bad_width(width)) return set_error(WN_ERR_ARG, "width must be > 0");
  if (bad_theta(theta)) return set_error(WN_ERR_ARG, "theta must be > 0");
  if (q && m < 0) return set_error(WN_ERR_ARG, "m < 0");
  cudaStream_t s = (cudaStream_t)stream;
  WN_TRY(ensure_scratch(t, s));
  IterScratch& it = t->it;
  // ν = a·μ: moments use μ and a separately (exact fp64 products); leaf terms use fl(a·μ)
  gather_vec_a(t->n, t->perm, mu, a, it.mu, (float*)it.tmp, it.mup, s);
  MomentArgs mm;
  mm.kind = ATTR_VEC;
  mm.vec = it.mu;
  mm.a_sorted = a ? (const float*)it.tmp : nullptr;
  mm.theta = theta;
  mm.out = t->set[0];
  mm.order1 = t->far_order == 1;
  WN_TRY(build_moments(t, mm, s));
  TravArgs ta = base_args(t, width * width);
  ta.order1 = t->far_order;
  ta.op = op;
  ta.epi = EPI_PLAIN;
  ta.nodes = t->set[0];
  ta.vec = a ? it.mup : it.mu;
  const double sc = t->xf[3];
  // frame factors (include/wn.h): F_in = s²·Σ_n(ν), ∇F_in = −s³·G_n(ν)
  ta.scale_out = op == OP_A ? (float)(sc * sc) : (float)(-sc * sc * sc);
  if (q) {
    if (m == 0) return WN_OK;
    if (t->qcap < m) {
      if (t->qbuf) cudaFreeAsync(t->qbuf, s);
      if (t->qbuf_order) cudaFreeAsync(t->qbuf_order, s);
      t->qbuf = nullptr;
      t->qbuf_order = nullptr;
      t->qcap = 0;
      WN_CUDA(cudaMallocAsync((void**)&t->qbuf, m * sizeof(float4), s));
      WN_CUDA(cudaMallocAsync((void**)&t->qbuf_order, m * sizeof(int32_t), s));
      t->qcap = m;
    }
    normalize_queries(m, q, t->xf, t->qbuf, s);
    if (!presorted) WN_TRY(hilbert_schedule(t->qbuf, m, t->qbuf_order, s));  // coherent warps for arbitrary queries (f1)
    ta.queries = t->qbuf;
    ta.q_end = m;
    ta.split = m <= split_max() ? split_factor(m) : 0;
    ta.out_map = nullptr;
    ta.qorder = presorted ? nullptr : t->qbuf_order;
  } else {
    ta.out_map = t->perm;
  }
  if (op == OP_A) ta.out_f = out;
  else ta.out_v3 = out;
  if (qcounts) {  // counting run: per-query work only
    ta.qcounts = qcounts;
    ta.out_f = nullptr;
    ta.out_v3 = nullptr;
  }
  return traverse(ta, s);
}

wn_status wn_eval(wn_tree t, const float* mu, const float* a, const float* q, int64_t m, float width, float theta,
                  float* F, void* stream) {
  return eval_common(t, OP_A, mu, a, q, m, width, theta, F, stream);
}

wn_status wn_eval_grad(wn_tree t, const float* mu, const float* a, const float* q, int64_t m, float width,
                       float theta, float* gradF, void* stream) {
  return eval_common(t, OP_G, mu, a, q, m, width, theta, gradF, stream);
}

wn_status wn_query_work(wn_tree t, int32_t op, const float* attr, const float* q, int64_t m, float width,
                        float theta, int32_t* counts, void* stream) {
  if (op != 0 && op != 2) return set_error(WN_ERR_ARG, "op must be 0 (F) or 2 (gradF)");
  return eval_common(t, op == 0 ? OP_A : OP_G, attr, nullptr, q, m, width, theta, nullptr, stream, counts);
}

wn_status wn_eval_fmm(wn_tree t, int32_t op, const float* attr, float width, int32_t p, float theta_f, int32_t leaf,
                      float* out, int64_t* counts, void* stream) {
  TreeUse use_(t, stream);
  if (!t || !attr || !out) return set_error(WN_ERR_ARG, "tree, attribute or output is NULL");
  if (op < 0 || op > 2) return set_error(WN_ERR_ARG, "op must be 0 (F), 1 (A^T) or 2 (gradF)");
  if (bad_width(width)) return set_error(WN_ERR_ARG, "width must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  WN_TRY(ensure_scratch(t, s));
  IterScratch& it = t->it;
  const double sc = t->xf[3];
  WN_TRY(fmm_plan(t, p, theta_f, leaf, width, s));  // (cached: the same parameters reuse the lists)
  wn_status st;
  if (op == 1) {  // Aᵀ(s) = −∇ of the charges' potential;  Aᵀ_in = s²·Aᵀ_n
    gather_scal(t->n, t->perm, attr, it.s, s);
    st = fmm_run(t, OP_AT, nullptr, it.s, width, t->perm, out, nullptr, sc * sc, s);
  } else {  // dipoles μ: F = V (F_in = s²·V_n(μ_in)), ∇F = ∇V (∇F_in = −s³·G_n(μ_in), G = −∇V)
    gather_vec_a(t->n, t->perm, attr, nullptr, it.mu, nullptr, nullptr, s);
    st = fmm_run(t, op == 0 ? OP_A : OP_G, it.mu, nullptr, width, t->perm, out, nullptr,
                 op == 0 ? sc * sc : -sc * sc * sc, s);
  }
  if (st == WN_OK && counts) {
    counts[0] = t->fmm.nm2l;
    counts[1] = t->fmm.np2p;
  }
  if (st == WN_OK) WN_CUDA(cudaStreamSynchronize(s));
  return st;
}

wn_status wn_eval_adjoint(wn_tree t, const float* sv, float width, float theta, int32_t mode, const float* mu_geom,
                          float* out, void* stream) {
  TreeUse use_(t, stream);
  if (!t || !sv || !out) return set_error(WN_ERR_ARG, "tree, s or output is NULL");
  if (bad_width(width)) return set_error(WN_ERR_ARG, "width must be > 0");
  if (bad_theta(theta)) return set_error(WN_ERR_ARG, "theta must be > 0");
  if (mode != WN_ADJ_GATHER && mode != WN_ADJ_TRANSPOSE) return set_error(WN_ERR_ARG, "bad adjoint mode");
  if (mode == WN_ADJ_TRANSPOSE && !mu_geom) return set_error(WN_ERR_ARG, "transpose mode needs mu_geom");
  if (mode == WN_ADJ_TRANSPOSE && t->far_order != 0)
    return set_error(WN_ERR_ARG, "transpose-mode adjoint is defined for the order-0 far field only");
  cudaStream_t s = (cudaStream_t)stream;
  WN_TRY(ensure_scratch(t, s));
  IterScratch& it = t->it;
  const double sc2 = t->xf[3] * t->xf[3];   // Aᵀ_in = s²·Aᵀ_n
  gather_scal(t->n, t->perm, sv, it.s, s);
  const float w2 = width * width;
  if (mode == WN_ADJ_GATHER) {
    MomentArgs m;
    m.kind = ATTR_SCALAR;
    m.scal = it.s;
    m.theta = theta;
    m.out = t->set[0];
    m.order1 = t->far_order == 1;
    WN_TRY(build_moments(t, m, s));
    TravArgs ta = base_args(t, w2);
    ta.order1 = t->far_order;
    ta.op = OP_AT;
    ta.epi = EPI_PLAIN;
    ta.nodes = t->set[0];
    ta.scal = it.s;
    ta.out_map = t->perm;
    ta.out_v3 = out;
    ta.scale_out = (float)sc2;
      return traverse(ta, s);
  }
  gather_vec(t->n, t->perm, mu_geom, 1.0, it.mu, s);
  MomentArgs m;
  m.kind = ATTR_VEC;
  m.vec = it.mu;
  m.theta = theta;
  m.out = t->set[1];
  WN_TRY(build_moments(t, m, s));
  WN_TRY(adjoint_transpose(t, t->set[1], it.s, w2, it.r, nullptr, s));
  scatter_vec(t->n, t->perm, it.r, sc2, out, s);
  return WN_OK;
}

static wn_status check_params(const wnnc_params* p) {
  if (!p) return set_error(WN_ERR_ARG, "params is NULL");
  if (bad_width(p->w_min) || bad_width(p->w_max)) return set_error(WN_ERR_ARG, "widths must be > 0");
  if (p->w_min > p->w_max) return set_error(WN_ERR_ARG, "w_min > w_max");
  if (bad_theta(p->theta)) return set_error(WN_ERR_ARG, "theta must be > 0");
  if (p->iters < 1) return set_error(WN_ERR_ARG, "iters < 1");
  const int total = p->total_iters > 0 ? p->total_iters : p->iters;
  if (p->first_iter < 1 || p->first_iter + p->iters - 1 > total) return set_error(WN_ERR_ARG, "bad first_iter");
  if (p->adjoint_mode != WN_ADJ_GATHER && p->adjoint_mode != WN_ADJ_TRANSPOSE)
    return set_error(WN_ERR_ARG, "bad adjoint_mode");
  return WN_OK;
}

wn_status wnnc_iterate_emulated(wn_tree t, float* mu, const wnnc_params* p, int32_t world, float* replicas,
                                void* stream) {
  TreeUse use_(t, stream);
  if (!t || !mu) return set_error(WN_ERR_ARG, "tree or mu is NULL");
  WN_TRY(check_params(p));
  if (world < 1 || world > kMaxPeers) return set_error(WN_ERR_ARG, "world must be 1..8");
  if (p->adjoint_mode == WN_ADJ_TRANSPOSE && t->far_order != 0)
    return set_error(WN_ERR_ARG, "transpose-mode adjoint is defined for the order-0 far field only");
  if (p->adjoint_mode == WN_ADJ_TRANSPOSE && t->nn > kArenaNodesPerPoint * t->n)
    return set_error(WN_ERR_ARG, "transpose-mode adjoint across ranks: the tree has more than 3 nodes per point");
  cudaStream_t s = (cudaStream_t)stream;
  WN_TRY(ensure_scratch(t, s));
  IterScratch& it = t->it;
  WN_TRY(ensure_dstats(t, p->iters, s));
  WN_TRY(plan_shards(t, world, nullptr, s));
  PeerArena arenas[kMaxPeers];
  void* blocks[kMaxPeers] = {};
  wn_status st = emulated_arenas(world, t->n, arenas, blocks);
  const double sc2 = t->xf[3] * t->xf[3];
  if (st == WN_OK) {
    const PeerArena* views[kMaxPeers];
    for (int v = 0; v < world; ++v) {
      views[v] = &arenas[v];
      gather_vec(t->n, t->perm, mu, sc2, arenas[0].mu[0][v], s);  // every rank's replica of μ⁰
    }
    st = run_iterations(t, *p, nullptr, views, world, s);
  }
  if (st == WN_OK) {
    const int e = p->iters & 1;
    scatter_vec(t->n, t->perm, arenas[0].mu[e][0], 1.0 / sc2, mu, s);
    if (replicas)
      for (int v = 0; v < world; ++v) scatter_vec(t->n, t->perm, arenas[0].mu[e][v], 1.0 / sc2, replicas + 3 * t->n * v, s);
    cudaError_t ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) st = cuda_status(ce, "wnnc_iterate_emulated");
  } else {
    cudaStreamSynchronize(s);
  }
  for (int v = 0; v < world; ++v)
    if (blocks[v]) cudaFree(blocks[v]);
  return st;
}

wn_status wnnc_iterate(wn_tree t, float* mu, const wnnc_params* p_in, wn_comm comm, wnnc_iter_stats* stats,
                       void* stream) {
  TreeUse use_(t, stream);
  if (!t || !mu) return set_error(WN_ERR_ARG, "tree or mu is NULL");
  WN_TRY(check_params(p_in));
  wnnc_params pl = *p_in;
  pl.flags = (pl.flags & ~kFlagStamps) | (stats ? kFlagStamps : 0);
  const wnnc_params* p = &pl;
  if ((p->flags & WN_FLAG_HOST_WAIT) && (p->flags & WN_FLAG_GRAPH))
    return set_error(WN_ERR_ARG, "WN_FLAG_HOST_WAIT waits on the host: it cannot be captured in a CUDA graph");
  if (comm && !comm_has_nccl(comm) && (p->flags & WN_FLAG_COMM_NCCL))
    return set_error(WN_ERR_ARG, "a local communicator has no NCCL exchange");
  if (t->far_order != 0 && p->adjoint_mode == WN_ADJ_TRANSPOSE)
    return set_error(WN_ERR_ARG, "transpose-mode adjoint is defined for the order-0 far field only");
  cudaStream_t s = (cudaStream_t)stream;
  WN_TRY(ensure_scratch(t, s));
  IterScratch& it = t->it;
  WN_TRY(ensure_dstats(t, p->iters, s));
  const double sc2 = t->xf[3] * t->xf[3];
  // multi-GPU exchange: peer-memory stores fused into the traversal epilogues (default), or NCCL
  const PeerArena* P = nullptr;
  if (comm && !(p->flags & WN_FLAG_COMM_NCCL)) WN_TRY(comm_peer_arena(comm, t->n, s, &P));
  if (P && p->adjoint_mode == WN_ADJ_TRANSPOSE && t->nn > P->node_cap)
    return set_error(WN_ERR_ARG, "transpose-mode adjoint across ranks: the tree has more than 3 nodes per point");
  if (comm) WN_TRY(plan_shards(t, comm_world(comm), comm, s));
  if (p->adjoint_mode == WN_ADJ_TRANSPOSE) WN_TRY(ensure_transpose_scratch(t, s));  // before any capture
  if (t->fmm_p > 0) {  // FMM operators (row f4): one plan for the whole schedule (separation width w_max ≥ every w)
    if (comm || p->adjoint_mode != WN_ADJ_GATHER)
      return set_error(WN_ERR_ARG, "FMM operators: single GPU and gather-mode adjoint only");
    WN_TRY(fmm_plan(t, t->fmm_p, t->fmm_theta, t->fmm_leaf, p->w_max, s));
  }
  float4* mu0 = P ? P->mu[0][P->rank] : t->it.mu;
  gather_vec(t->n, t->perm, mu, sc2, mu0, s);             // μ_norm = scale²·μ
  if (p->flags & WN_FLAG_GRAPH) {
    // the whole iteration loop as one CUDA graph: captured on a private stream, cached per parameters
    const void* arena = P ? P->own : nullptr;
    std::vector<uint8_t> key(sizeof(wnnc_params) + sizeof(comm) + sizeof(int) + sizeof(arena) + sizeof(ShardPlan) + 1);
    key.back() = (g_count_on ? 1 : 0) | (t->fmm_p << 1);  // counting variants / FMM degree are baked into the graph
    uint8_t* kp = key.data();
    memcpy(kp, p, sizeof(wnnc_params));
    kp += sizeof(wnnc_params);
    memcpy(kp, &comm, sizeof(comm));
    kp += sizeof(comm);
    memcpy(kp, &t->far_order, sizeof(int));
    kp += sizeof(int);
    memcpy(kp, &arena, sizeof(arena));
    kp += sizeof(arena);
    memcpy(kp, &t->shard, sizeof(ShardPlan));
    if (!t->graph_exec || key != t->graph_key) {
      if (t->graph_exec) cudaGraphExecDestroy(t->graph_exec);
      t->graph_exec = nullptr;
      if (!t->cap_stream) WN_CUDA(cudaStreamCreateWithFlags(&t->cap_stream, cudaStreamNonBlocking));
      WN_CUDA(cudaStreamBeginCapture(t->cap_stream, cudaStreamCaptureModeThreadLocal));
      g_capturing = true;
      wn_status st = run_iterations(t, *p, comm, &P, P ? 1 : 0, t->cap_stream);
      g_capturing = false;
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(t->cap_stream, &graph);
      if (st != WN_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamEndCapture");
      size_t nnodes = 0;
      cudaGraphGetNodes(graph, nullptr, &nnodes);
      std::vector<cudaGraphNode_t> nodes(nnodes);
      cudaGraphGetNodes(graph, nodes.data(), &nnodes);
      t->graph_launches = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        cudaGraphNodeGetType(nd, &ty);
        t->graph_launches += ty == cudaGraphNodeTypeKernel;
      }
      e = cudaGraphInstantiate(&t->graph_exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_status(e, "cudaGraphInstantiate");
      t->graph_key = key;
    }
    ProfScope ps(WN_PROF_OTHER, s, 0);
    count_launches((int)t->graph_launches);
    WN_CUDA(cudaGraphLaunch(t->graph_exec, s));
  } else {
    WN_TRY(run_iterations(t, *p, comm, &P, P ? 1 : 0, s));
  }
  const float4* mu_end = P ? P->mu[p->iters & 1][P->rank] : t->it.mu;
  scatter_vec(t->n, t->perm, mu_end, 1.0 / sc2, mu, s);  // back to the input frame
  if (stats) {
    std::vector<double> h(5 * (size_t)p->iters);
    std::vector<int64_t> c(12 * (size_t)(p->iters + 1), 0);
    WN_CUDA(cudaMemcpyAsync(h.data(), t->it.dstats, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    std::vector<unsigned long long> ts(p->iters + 1, 0);
    if (g_count_on) WN_CUDA(cudaMemcpyAsync(c.data(), t->it.dcounts, c.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaMemcpyAsync(ts.data(), t->it.dstamp, ts.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < p->iters; ++i) {
      wnnc_iter_stats& o = stats[i];
      o.E = h[5 * i];
      o.alpha = h[5 * i + 1];
      o.rr = h[5 * i + 2];
      o.qq = h[5 * i + 3];
      o.width = h[5 * i + 4];
      o.ms = 1e-6 * (double)(ts[i + 1] - ts[i]);
      int64_t w[4] = {-1, -1, -1, -1};
      if (g_count_on)
        for (int k = 0; k < 4; ++k) {
          w[k] = 0;
          for (int cls = 0; cls < 3; ++cls) w[k] += c[12 * (i + 1) + 4 * cls + k] - c[12 * i + 4 * cls + k];
        }
      o.tests = w[0];
      o.far_terms = w[1];
      o.near_terms = w[2];
      o.live_terms = w[3];
    }
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

wn_status wnnc_solve_host(const float* pts_host, int64_t n, int32_t max_depth, const wnnc_params* p,
                          float* normals_host, float* mu_host, wnnc_iter_stats* stats, void* stream) {
  if (!pts_host || !normals_host) return set_error(WN_ERR_ARG, "host buffer is NULL");
  if (n < 1) return set_error(WN_ERR_EMPTY, "empty point set (n < 1)");
  WN_TRY(check_params(p));
  WN_TRY(check_device());
  cudaStream_t s = (cudaStream_t)stream;
  float *dp = nullptr, *dmu = nullptr, *dn = nullptr;
  const size_t bytes = (size_t)n * 3 * sizeof(float);
  WN_CUDA(cudaMallocAsync((void**)&dp, bytes, s));
  WN_CUDA(cudaMallocAsync((void**)&dmu, bytes, s));
  WN_CUDA(cudaMallocAsync((void**)&dn, bytes, s));
  WN_CUDA(cudaMemcpyAsync(dp, pts_host, bytes, cudaMemcpyHostToDevice, s));
  WN_CUDA(cudaMemsetAsync(dmu, 0, bytes, s));
  wn_tree t = nullptr;
  wn_status st = wn_build_tree(dp, n, max_depth, stream, &t);
  wnnc_params pz = *p;
  if (pz.first_iter == 1) pz.flags |= WN_FLAG_MU_ZERO;  // μ⁰ = 0 here by construction
  if (st == WN_OK) st = wnnc_iterate(t, dmu, &pz, nullptr, stats, stream);
  if (st == WN_OK) {
    unit_normals(n, dmu, dn, s);
    cudaMemcpyAsync(normals_host, dn, bytes, cudaMemcpyDeviceToHost, s);
    if (mu_host) cudaMemcpyAsync(mu_host, dmu, bytes, cudaMemcpyDeviceToHost, s);
  }
  cudaFreeAsync(dp, s);
  cudaFreeAsync(dmu, s);
  cudaFreeAsync(dn, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (t) wn_tree_destroy(t);
  if (st != WN_OK) return st;
  if (e != cudaSuccess) return cuda_status(e, "wnnc_solve_host");
  return WN_OK;
}

wn_status wn_tree_schedule(wn_tree t, int32_t* qorder, void* stream) {
  TreeUse use_(t, stream);
  if (!t || !qorder) return set_error(WN_ERR_ARG, "tree or output is NULL");
  WN_CUDA(cudaMemcpyAsync(qorder, t->qorder, t->n * sizeof(int32_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return WN_OK;
}

wn_status wn_tree_schedule_stats(wn_tree t, int32_t* kind, int64_t stats[4]) {
  if (!t) return set_error(WN_ERR_ARG, "tree is NULL");
  if (kind) *kind = t->sched_kind;
  if (stats)
    for (int k = 0; k < 4; ++k) stats[k] = t->sched_stats[k];
  return WN_OK;
}

wn_status wn_shard_plan(wn_tree t, int32_t world, int64_t* bounds, void* stream) {
  TreeUse use_(t, stream);
  if (!t || !bounds || world < 1 || world > kMaxShardRanks) return set_error(WN_ERR_ARG, "bad shard-plan arguments");
  cudaStream_t s = (cudaStream_t)stream;
  WN_TRY(ensure_scratch(t, s));
  WN_TRY(plan_shards(t, world, nullptr, s));
  for (int r = 0; r < world; ++r) {
    int64_t b = 0, e = 0;
    shard_of(&t->shard, t->n, r, world, &b, &e);
    bounds[r] = b;
  }
  bounds[world] = t->n;
  return WN_OK;
}

wn_status wn_shard_range(int64_t n, int32_t rank, int32_t world, int64_t* begin, int64_t* end) {
  if (world < 1 || rank < 0 || rank >= world || n < 0 || !begin || !end)
    return set_error(WN_ERR_ARG, "bad shard arguments");
  const int64_t blocks = (n + WN_SHARD_ALIGN - 1) / WN_SHARD_ALIGN;
  const int64_t b0 = blocks * rank / world, b1 = blocks * (rank + 1) / world;
  *begin = std::min<int64_t>(n, b0 * WN_SHARD_ALIGN);
  *end = std::min<int64_t>(n, b1 * WN_SHARD_ALIGN);
  return WN_OK;
}

}  // extern "C"

#ifdef WN_EXP_SETSCHED
// experiment hook (variant builds only): replace the tree's query schedule with qorder[N] (device)
extern "C" wn_status wn_exp_set_schedule(wn_tree t, const int32_t* qorder, void* stream) {
  if (!t || !qorder) return wn::set_error(WN_ERR_ARG, "tree or schedule is NULL");
  WN_CUDA(cudaMemcpyAsync(t->qorder, qorder, t->n * sizeof(int32_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return WN_OK;
}
#endif

namespace wn {
wn_status eval_field(wn_tree_s* t, const float* mu, const float* q, int64_t m, float width, float theta, float* F,
                     cudaStream_t s) {
  return eval_common(t, OP_A, mu, nullptr, q, m, width, theta, F, (void*)s, nullptr, true);
}
}  // namespace wn
