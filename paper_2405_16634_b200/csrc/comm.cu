// comm.cu — NCCL communicator for query-sharded iteration over NVLink 5 / NVSwitch.
//
// Sources, tree and node moments are replicated on every rank; each rank traverses a contiguous
// Morton range of queries (wn_shard_range, aligned to WN_SHARD_ALIGN so the per-block Σ partials are
// the same blocks for every world size).  After each traversal the owned rows are exchanged with a
// grouped ncclBroadcast per rank (an all-gather with uneven shards); the three Σ partial arrays are
// exchanged the same way before α, so every rank reduces identical partials in the same order and the
// trajectory is bit-identical to the single-GPU one.  NCCL is dlopen()ed (libnccl.so.2 — the copy
// torch already loaded, when present), so libwn has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>
#include <new>
#include <string>

#include "wn_comm.cuh"
#include "wn_internal.cuh"

struct wn_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  wn::PeerArena arena;  // peer-memory exchange (fused into the traversal epilogues), built on first use
};

namespace wn {
namespace {

struct Nccl {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
      return;
    }
#define SYM(f, name) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, name))
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Broadcast, "ncclBroadcast");
    SYM(AllGather, "ncclAllGather");
    SYM(AllReduce, "ncclAllReduce");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Broadcast && n.AllGather && n.AllReduce &&
           n.GroupStart && n.GroupEnd;
    if (!n.ok) n.err = "libnccl.so.2 lacks required symbols";
  });
  return n;
}

wn_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return WN_OK;
  const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
  return set_error(WN_ERR_NCCL, std::string(what) + ": " + m);
}

}  // namespace

wn_status comm_shard(wn_comm c, int64_t n, int64_t* q0, int64_t* q1) {
  return wn_shard_range(n, c->rank, c->world, q0, q1);
}

namespace {
// schedule-ordered staging: stage[k] = buf[qorder[k]] (pack the owned range) and the inverse (unpack)
__global__ void k_pack(const float* __restrict__ buf, const int32_t* __restrict__ qorder, int64_t b, int64_t e,
                       int comps, float* __restrict__ stage) {
  const int64_t k = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= e) return;
  const int64_t q = qorder[k];
  for (int c = 0; c < comps; ++c) stage[k * comps + c] = buf[q * comps + c];
}
__global__ void k_unpack(const float* __restrict__ stage, const int32_t* __restrict__ qorder, int64_t n, int comps,
                         float* __restrict__ buf) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t q = qorder[k];
  for (int c = 0; c < comps; ++c) buf[q * comps + c] = stage[k * comps + c];
}
}  // namespace

void shard_of(const ShardPlan* plan, int64_t n, int rank, int world, int64_t* b, int64_t* e) {
  if (plan && plan->world == world) {
    *b = plan->b[rank];
    *e = plan->b[rank + 1];
  } else {
    wn_shard_range(n, rank, world, b, e);
  }
}

wn_status comm_allgather_f(wn_comm c, float* buf, int comps, int64_t n, const int32_t* qorder, float* stage,
                           const ShardPlan* plan, cudaStream_t s) {
  Nccl& N = nccl();
  float* x = buf;
  if (qorder) {  // the owned rows are a schedule range: gather them into schedule order first
    int64_t b = 0, e = 0;
    shard_of(plan, n, c->rank, c->world, &b, &e);
    if (e > b) k_pack<<<(unsigned)((e - b + 255) / 256), 256, 0, s>>>(buf, qorder, b, e, comps, stage);
    count_launches(1);
    x = stage;
  }
  ncclResult_t r = N.GroupStart();
  for (int k = 0; k < c->world && r == ncclSuccess; ++k) {
    int64_t b = 0, e = 0;
    shard_of(plan, n, k, c->world, &b, &e);
    if (e > b) r = N.Broadcast(x + b * comps, x + b * comps, (size_t)(e - b) * comps, ncclFloat32, k, c->comm, s);
  }
  ncclResult_t r2 = N.GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r == ncclSuccess && qorder) {
    k_unpack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(stage, qorder, n, comps, buf);
    count_launches(1);
  }
  return nccl_status(r, "ncclBroadcast (all-gather)");
}

wn_status comm_allgather_partials(wn_comm c, double* part, int64_t stride, int64_t n, const ShardPlan* plan,
                                  cudaStream_t s) {
  Nccl& N = nccl();
  ncclResult_t r = N.GroupStart();
  for (int a = 0; a < 3 && r == ncclSuccess; ++a)
    for (int k = 0; k < c->world && r == ncclSuccess; ++k) {
      int64_t b = 0, e = 0;
      shard_of(plan, n, k, c->world, &b, &e);
      const int64_t b0 = b / kPartQ, b1 = (e + kPartQ - 1) / kPartQ;  // partials per 32-query group
      if (b1 > b0) {
        double* p = part + a * stride + b0;
        r = N.Broadcast(p, p, (size_t)(b1 - b0), ncclFloat64, k, c->comm, s);
      }
    }
  ncclResult_t r2 = N.GroupEnd();
  if (r == ncclSuccess) r = r2;

  return nccl_status(r, "ncclBroadcast (partials)");
}

wn_status comm_allreduce_i64(wn_comm c, int64_t* buf, int64_t count, cudaStream_t s) {
  return nccl_status(nccl().AllReduce(buf, buf, (size_t)count, ncclInt64, ncclSum, c->comm, s), "ncclAllReduce (work)");
}

wn_status comm_allreduce_f64(wn_comm c, double* buf, int64_t count, cudaStream_t s) {
  return nccl_status(nccl().AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, c->comm, s),
                     "ncclAllReduce (adjoint accumulators)");
}

int comm_rank(wn_comm c) { return c->rank; }
int comm_world(wn_comm c) { return c->world; }

// ---------------- peer-memory exchange (B200-native form of the per-traversal all-gather) ----------------
// Every rank allocates one IPC-capable block (cudaMalloc) holding the exchanged arrays — s (N fp32),
// r (N float4), μ (2 × N float4: ping-pong, so a fast rank's G epilogue never overwrites the μ a slow
// rank's axpy still reads), the Σ partials (3 × blocks fp64) — and a signal word.  The handles are
// all-gathered once (NCCL) and opened with cudaIpcOpenMemHandle, so every rank holds a device pointer
// to every replica; the traversal epilogues then store each owned row into all replicas over NVLink
// and the last block of each launch signals every rank (system-scope fence + remote atomic add).
// A one-thread wait kernel on each rank spins on its own signal word until all ranks have signalled
// that exchange — its target advances on the device, so a captured CUDA graph can be replayed.
namespace {
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// a rank that never signals (a crashed peer) must not hang the GPU: give up after 10 s and trap
constexpr unsigned long long kPeerWaitTimeoutNs = 10ull * 1000 * 1000 * 1000;

__global__ void k_peer_wait(unsigned long long* sig, unsigned long long* expected, int world) {
  const unsigned long long target = *expected + (unsigned long long)world;
  *expected = target;
  const unsigned long long t0 = globaltimer_ns();
  unsigned long long v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(sig) : "memory");
    if (v >= target) break;
    if (globaltimer_ns() - t0 > kPeerWaitTimeoutNs) {
      printf("libwn: peer-memory exchange timed out (signal %llu of %llu)\n", v, target);
      __trap();
    }
    __nanosleep(200);
  }
  __threadfence_system();
}
}  // namespace

static void arena_release(PeerArena& A) {
  for (int r = 0; r < A.world; ++r)
    if (A.opened[r] && A.base[r]) cudaIpcCloseMemHandle(A.base[r]);
  if (A.own) cudaFree(A.own);
  A = PeerArena();
}

// the arena's layout inside one block of `arena_bytes(n)` bytes
struct ArenaLayout {
  size_t o_s, o_r, o_mu0, o_mu1, o_part, o_vb, o_u, o_sig, bytes;
  int64_t nb, node_cap;
  explicit ArenaLayout(int64_t n) {
    nb = part_slots(n);
    node_cap = kArenaNodesPerPoint * n;
    o_s = 0;
    o_r = align256(o_s + n * sizeof(float));
    o_mu0 = align256(o_r + n * sizeof(float4));
    o_mu1 = align256(o_mu0 + n * sizeof(float4));
    o_part = align256(o_mu1 + n * sizeof(float4));
    o_vb = align256(o_part + 3 * nb * sizeof(double));
    o_u = align256(o_vb + 3 * node_cap * sizeof(double));
    o_sig = align256(o_u + 3 * n * sizeof(double));
    bytes = align256(o_sig + 4 * sizeof(uint64_t));
  }
};

// point A (rank `rank` of `world`) at every rank's block; blocks[r] mapped in this process
static void arena_bind(PeerArena& A, void* const* blocks, int world, int rank, int64_t n) {
  const ArenaLayout L(n);
  A.world = world;
  A.rank = rank;
  A.cap = n;
  A.part_stride = L.nb;
  A.node_cap = L.node_cap;
  for (int r = 0; r < world; ++r) {
    char* b = static_cast<char*>(blocks[r]);
    A.base[r] = blocks[r];
    A.s[r] = reinterpret_cast<float*>(b + L.o_s);
    A.r[r] = reinterpret_cast<float4*>(b + L.o_r);
    A.mu[0][r] = reinterpret_cast<float4*>(b + L.o_mu0);
    A.mu[1][r] = reinterpret_cast<float4*>(b + L.o_mu1);
    A.part[r] = reinterpret_cast<double*>(b + L.o_part);
    A.vb[r] = reinterpret_cast<double*>(b + L.o_vb);
    A.u[r] = reinterpret_cast<double*>(b + L.o_u);
    A.sig[r] = reinterpret_cast<unsigned long long*>(b + L.o_sig);
  }
  char* own = static_cast<char*>(blocks[rank]);
  A.expected = reinterpret_cast<unsigned long long*>(own + L.o_sig) + 1;  // local: next wait target
  A.done = reinterpret_cast<unsigned int*>(reinterpret_cast<unsigned long long*>(own + L.o_sig) + 2);
}

wn_status comm_peer_arena(wn_comm c, int64_t n, cudaStream_t s, const PeerArena** out) {
  PeerArena& A = c->arena;
  if (c->world > kMaxPeers) return set_error(WN_ERR_ARG, "peer-memory exchange supports at most 8 ranks");
  if (A.own && A.cap >= n) {
    *out = &A;
    return WN_OK;
  }
  if (!c->comm)  // a local communicator's arena comes from wn_comm_arena_export / _import
    return set_error(WN_ERR_ARG, "local communicator: call wn_comm_arena_export/_import for this N first");
  // (re)build, collectively: every rank reaches this point in the same wnnc_iterate call
  arena_release(A);
  const ArenaLayout L(n);
  WN_CUDA(cudaStreamSynchronize(s));
  void* own = nullptr;
  WN_CUDA(cudaMalloc(&own, L.bytes));
  WN_CUDA(cudaMemset(own, 0, L.bytes));
  cudaIpcMemHandle_t mine;
  WN_CUDA(cudaIpcGetMemHandle(&mine, own));
  cudaIpcMemHandle_t* dh = nullptr;
  WN_CUDA(cudaMalloc(&dh, sizeof(cudaIpcMemHandle_t) * c->world));
  WN_CUDA(cudaMemcpy(dh + c->rank, &mine, sizeof(mine), cudaMemcpyHostToDevice));
  Nccl& N = nccl();
  wn_status st = nccl_status(N.AllGather(dh + c->rank, dh, sizeof(mine), ncclUint8, c->comm, s),
                             "ncclAllGather (IPC handles)");
  cudaIpcMemHandle_t hs[kMaxPeers];
  if (st == WN_OK) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMemcpy(hs, dh, sizeof(mine) * c->world, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = cuda_status(e, "IPC handle exchange");
  }
  cudaFree(dh);
  if (st != WN_OK) {
    cudaFree(own);
    return st;
  }
  void* blocks[kMaxPeers] = {};
  bool opened[kMaxPeers] = {};
  cudaError_t oe = cudaSuccess;
  for (int r = 0; r < c->world && oe == cudaSuccess; ++r) {
    if (r == c->rank) {
      blocks[r] = own;
      continue;
    }
    oe = cudaIpcOpenMemHandle(&blocks[r], hs[r], cudaIpcMemLazyEnablePeerAccess);
    opened[r] = oe == cudaSuccess;
  }
  // every rank must agree before anyone stores into a peer: min over ranks of "all opens succeeded"
  int32_t* flag = nullptr;
  int32_t ok = oe == cudaSuccess ? 1 : 0, all_ok = 0;
  WN_CUDA(cudaMalloc(&flag, sizeof(int32_t)));
  WN_CUDA(cudaMemcpy(flag, &ok, sizeof(ok), cudaMemcpyHostToDevice));
  st = nccl_status(N.AllReduce(flag, flag, 1, ncclInt32, ncclMin, c->comm, s), "ncclAllReduce (peer arena)");
  if (st == WN_OK) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMemcpy(&all_ok, flag, sizeof(all_ok), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = cuda_status(e, "peer arena agreement");
  }
  cudaFree(flag);
  if (st == WN_OK && !all_ok)
    st = oe != cudaSuccess ? cuda_status(oe, "cudaIpcOpenMemHandle (peer arena)")
                           : set_error(WN_ERR_CUDA, "peer arena: another rank could not map the replicas");
  if (st != WN_OK) {
    for (int r = 0; r < c->world; ++r)
      if (opened[r]) cudaIpcCloseMemHandle(blocks[r]);
    cudaFree(own);
    return st;
  }
  arena_bind(A, blocks, c->world, c->rank, n);
  A.own = own;
  for (int r = 0; r < c->world; ++r) A.opened[r] = opened[r];
  *out = &A;
  return WN_OK;
}

// W ranks in this process on this GPU (wnnc_iterate_emulated): one plain block per rank
wn_status emulated_arenas(int world, int64_t n, PeerArena* arenas, void** blocks) {
  const ArenaLayout L(n);
  for (int r = 0; r < world; ++r) {
    WN_CUDA(cudaMalloc(&blocks[r], L.bytes));
    WN_CUDA(cudaMemset(blocks[r], 0, L.bytes));
  }
  for (int r = 0; r < world; ++r) arena_bind(arenas[r], blocks, world, r, n);
  return WN_OK;
}

void comm_peer_wait(const PeerArena& A, cudaStream_t s) {
  k_peer_wait<<<1, 1, 0, s>>>(A.sig[A.rank], A.expected, A.world);
  count_launches(1);
}

namespace {
__global__ void k_peer_signal_all(PeerArena A) {
  __threadfence_system();
  for (int r = 0; r < A.world; ++r) atomicAdd_system(A.sig[r], 1ull);
}
}  // namespace

void comm_peer_signal(const PeerArena& A, cudaStream_t s) {
  k_peer_signal_all<<<1, 1, 0, s>>>(A);
  count_launches(1);
}

wn_status comm_peer_wait_host(const PeerArena& A, cudaStream_t s) {
  WN_CUDA(cudaStreamSynchronize(s));  // this rank's signals and stores are issued and done
  unsigned long long cur = 0;         // the wait target lives on the device (device-side waits advance it too)
  WN_CUDA(cudaMemcpy(&cur, A.expected, sizeof(cur), cudaMemcpyDeviceToHost));
  const unsigned long long target = cur + (unsigned long long)A.world;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    unsigned long long v = 0;
    WN_CUDA(cudaMemcpy(&v, A.sig[A.rank], sizeof(v), cudaMemcpyDeviceToHost));
    if (v >= target) break;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
      return set_error(WN_ERR_CUDA, "peer-memory exchange: a rank did not signal within 120 s");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  WN_CUDA(cudaMemcpy(A.expected, &target, sizeof(target), cudaMemcpyHostToDevice));
  return WN_OK;
}

bool comm_has_nccl(wn_comm c) { return c && c->comm; }

}  // namespace wn

using namespace wn;

extern "C" {

wn_status wn_comm_unique_id(uint8_t id[128]) {
  Nccl& N = nccl();
  if (!N.ok) return set_error(WN_ERR_NCCL, N.err);
  ncclUniqueId u;
  {
    wn_status st = nccl_status(N.GetUniqueId(&u), "ncclGetUniqueId");
    if (st != WN_OK) return st;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::copy(u.internal, u.internal + 128, reinterpret_cast<char*>(id));
  return WN_OK;
}

wn_status wn_comm_init(int32_t rank, int32_t world, const uint8_t id[128], wn_comm* out) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world) return set_error(WN_ERR_ARG, "bad comm arguments");
  Nccl& N = nccl();
  if (!N.ok) return set_error(WN_ERR_NCCL, N.err);
  ncclUniqueId u;
  std::copy(id, id + 128, reinterpret_cast<uint8_t*>(u.internal));
  wn_comm_s* c = new (std::nothrow) wn_comm_s();
  if (!c) return set_error(WN_ERR_OOM, "host allocation failed");
  c->rank = rank;
  c->world = world;
  wn_status st = nccl_status(N.CommInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
  if (st != WN_OK) {
    delete c;
    return st;
  }
  *out = c;
  return WN_OK;
}

wn_status wn_comm_init_local(int32_t rank, int32_t world, wn_comm* out) {
  if (!out || world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    return set_error(WN_ERR_ARG, "bad local comm arguments (world 1..8)");
  wn_comm_s* c = new (std::nothrow) wn_comm_s();
  if (!c) return set_error(WN_ERR_OOM, "host allocation failed");
  c->rank = rank;
  c->world = world;
  *out = c;
  return WN_OK;
}

wn_status wn_comm_arena_export(wn_comm c, int64_t n, uint8_t handle[64], void* stream) {
  if (!c || !handle || n < 1) return set_error(WN_ERR_ARG, "bad arena export arguments");
  if (c->comm) return set_error(WN_ERR_ARG, "NCCL communicators set their arena up collectively");
  arena_release(c->arena);
  const ArenaLayout L(n);
  WN_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  void* own = nullptr;
  WN_CUDA(cudaMalloc(&own, L.bytes));
  cudaError_t e = cudaMemset(own, 0, L.bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, own);
  if (e != cudaSuccess) {
    cudaFree(own);
    return cuda_status(e, "wn_comm_arena_export");
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::copy(reinterpret_cast<const uint8_t*>(&h), reinterpret_cast<const uint8_t*>(&h) + 64, handle);
  c->arena.own = own;
  c->arena.cap = 0;  // not usable before the import
  c->arena.pending_n = n;
  return WN_OK;
}

wn_status wn_comm_arena_import(wn_comm c, const uint8_t* handles) {
  if (!c || !handles || !c->arena.own || c->arena.pending_n < 1)
    return set_error(WN_ERR_ARG, "wn_comm_arena_import: export this rank's arena first");
  PeerArena& A = c->arena;
  void* blocks[kMaxPeers] = {};
  bool opened[kMaxPeers] = {};
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < c->world && e == cudaSuccess; ++r) {
    if (r == c->rank) {
      blocks[r] = A.own;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::copy(handles + 64 * r, handles + 64 * (r + 1), reinterpret_cast<uint8_t*>(&h));
    e = cudaIpcOpenMemHandle(&blocks[r], h, cudaIpcMemLazyEnablePeerAccess);
    opened[r] = e == cudaSuccess;
  }
  if (e != cudaSuccess) {
    for (int r = 0; r < c->world; ++r)
      if (opened[r]) cudaIpcCloseMemHandle(blocks[r]);
    return cuda_status(e, "cudaIpcOpenMemHandle (wn_comm_arena_import)");
  }
  void* own = A.own;
  const int64_t n = A.pending_n;
  arena_bind(A, blocks, c->world, c->rank, n);
  A.own = own;
  for (int r = 0; r < c->world; ++r) A.opened[r] = opened[r];
  return WN_OK;
}

wn_status wn_comm_destroy(wn_comm c) {
  if (!c) return WN_OK;
  if (c->arena.own) {
    cudaDeviceSynchronize();
    arena_release(c->arena);
  }
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
  return WN_OK;
}

}  // extern "C"
