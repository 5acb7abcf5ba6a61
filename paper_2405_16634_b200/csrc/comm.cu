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
#include <mutex>
#include <new>
#include <string>

#include "wn_comm.cuh"
#include "wn_internal.cuh"

struct wn_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
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
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Broadcast && n.GroupStart && n.GroupEnd;
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

wn_status comm_allgather_f(wn_comm c, float* buf, int comps, int64_t n, const int32_t* qorder, float* stage,
                           cudaStream_t s) {
  Nccl& N = nccl();
  float* x = buf;
  if (qorder) {  // the owned rows are a schedule range: gather them into schedule order first
    int64_t b = 0, e = 0;
    wn_shard_range(n, c->rank, c->world, &b, &e);
    if (e > b) k_pack<<<(unsigned)((e - b + 255) / 256), 256, 0, s>>>(buf, qorder, b, e, comps, stage);
    count_launches(1);
    x = stage;
  }
  ncclResult_t r = N.GroupStart();
  for (int k = 0; k < c->world && r == ncclSuccess; ++k) {
    int64_t b = 0, e = 0;
    wn_shard_range(n, k, c->world, &b, &e);
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

wn_status comm_allgather_partials(wn_comm c, double* part, int64_t stride, int64_t n, cudaStream_t s) {
  Nccl& N = nccl();
  ncclResult_t r = N.GroupStart();
  for (int a = 0; a < 3 && r == ncclSuccess; ++a)
    for (int k = 0; k < c->world && r == ncclSuccess; ++k) {
      int64_t b = 0, e = 0;
      wn_shard_range(n, k, c->world, &b, &e);
      const int64_t b0 = b / kTravBlock, b1 = (e + kTravBlock - 1) / kTravBlock;  // partials per traversal block
      if (b1 > b0) {
        double* p = part + a * stride + b0;
        r = N.Broadcast(p, p, (size_t)(b1 - b0), ncclFloat64, k, c->comm, s);
      }
    }
  ncclResult_t r2 = N.GroupEnd();
  if (r == ncclSuccess) r = r2;

  return nccl_status(r, "ncclBroadcast (partials)");
}

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

wn_status wn_comm_destroy(wn_comm c) {
  if (!c) return WN_OK;
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
  return WN_OK;
}

}  // extern "C"
