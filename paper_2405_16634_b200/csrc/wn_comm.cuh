// wn_comm.cuh — query-sharded multi-GPU plumbing; NCCL is loaded at run time.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/wn.h"
#include "wn_internal.cuh"

namespace wn {
wn_status comm_shard(wn_comm c, int64_t n, int64_t* q0, int64_t* q1);
// Every rank owns the rows of schedule positions [q0, q1) of a sorted-order array of n rows × comps floats
// (row = qorder[k], or k when qorder is null); make it whole on all ranks.  stage: n × comps scratch.
wn_status comm_allgather_f(wn_comm c, float* buf, int comps, int64_t n, const int32_t* qorder, float* stage,
                           const ShardPlan* plan, cudaStream_t s);
// The three per-block partial arrays (stride entries each, blocks of kTravBlock queries).
wn_status comm_allgather_partials(wn_comm c, double* part, int64_t stride, int64_t n, const ShardPlan* plan,
                                  cudaStream_t s);
// rank r's query range [*b, *e): the plan's when it is for this world size, else equal counts
void shard_of(const ShardPlan* plan, int64_t n, int rank, int world, int64_t* b, int64_t* e);
wn_status comm_allreduce_i64(wn_comm c, int64_t* buf, int64_t count, cudaStream_t s);
wn_status comm_allreduce_f64(wn_comm c, double* buf, int64_t count, cudaStream_t s);
// this rank's signal to every rank (after a step that is not a traversal, e.g. the adjoint scatter)
void comm_peer_signal(const PeerArena& A, cudaStream_t s);
int comm_rank(wn_comm c);
int comm_world(wn_comm c);
// Peer-memory exchange: the communicator's arena (collective on first use or growth; synchronizes s),
// and the per-exchange device-side wait for every rank's signal.
wn_status comm_peer_arena(wn_comm c, int64_t n, cudaStream_t s, const PeerArena** out);
void comm_peer_wait(const PeerArena& A, cudaStream_t s);
// the same wait on the host: synchronize s, then poll this rank's signal word (WN_FLAG_HOST_WAIT)
wn_status comm_peer_wait_host(const PeerArena& A, cudaStream_t s);
bool comm_has_nccl(wn_comm c);  // false for wn_comm_init_local communicators
// W emulated ranks in one process (diagnostic): plain blocks[W] bound as each other's replicas
wn_status emulated_arenas(int world, int64_t n, PeerArena* arenas, void** blocks);
}  // namespace wn
