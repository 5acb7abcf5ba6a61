// transpose.cu — exact-transpose adjoint of the treecode (BASELINE north star:
// "the adjoint kernel, which scatters into node moments and is then pushed down the tree").
//
// Treecode A at frozen geometry g(μ) (reps and per-query decisions of A(μ), Alg. 4)
// is linear in the attribute ν:  (T_g ν)_i = Σ_{far B} ∇Φ_w(x_i − x_B)·Σ_{j∈B} ν_j + Σ_{near j} ∇Φ_w(x_i − x_j)·ν_j.
// Its exact transpose is  (T_gᵀ s)_j = U_j + Σ_{B ∋ j} V_B  with
//     V_B = Σ_{i: B far for i} s_i ∇Φ_w(x_i − x_B),   U_j = Σ_{i: j near for i} s_i ∇Φ_w(x_i − x_j).
// Kernel 1 runs the same warp-cooperative traversal as A (same fp32 decisions, Hilbert query schedule);
// the lanes' contributions to up to four nodes (or leaf points) at a time are summed with one warp
// reduce-scatter, after which different lanes issue the fp64 atomics (one per node and component).
// Kernel 2 pushes down: r_j = U_j + Σ over the ancestors of j's leaf, and emits Σ|r|² block partials.
#include <cuda_runtime.h>

#include "wn_internal.cuh"

namespace wn {
namespace {

constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ float dist2(float dx, float dy, float dz) {
  return __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));
}

__device__ __forceinline__ void warp_add3(float x, float y, float z, double* dst, int lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    x += __shfl_xor_sync(FULL, x, o);
    y += __shfl_xor_sync(FULL, y, o);
    z += __shfl_xor_sync(FULL, z, o);
  }
  if (lane == 0) {
    atomicAdd(dst + 0, (double)x);
    atomicAdd(dst + 1, (double)y);
    atomicAdd(dst + 2, (double)z);
  }
}

// Reduce-scatter of 16 per-lane values (four targets × (x, y, z, ·)) over the warp: 8 + 4 + 2 + 1 + 1
// shuffles; afterwards lane l holds the total of value 8·l₄ + 4·l₃ + 2·l₂ + l₁, i.e. target 2·l₄ + l₃,
// component 2·l₂ + l₁ (lanes l and l ^ 1 hold the same total).  A per-target butterfly would take 15.
__device__ __forceinline__ float reduce_scatter16(const float (&v)[16], int lane, int& target, int& comp) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  float w8[8], w4[4], w2v[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float send = b4 ? v[i] : v[8 + i];
    w8[i] = (b4 ? v[8 + i] : v[i]) + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b3 ? w8[i] : w8[4 + i];
    w4[i] = (b3 ? w8[4 + i] : w8[i]) + __shfl_xor_sync(FULL, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b2 ? w4[i] : w4[2 + i];
    w2v[i] = (b2 ? w4[2 + i] : w4[i]) + __shfl_xor_sync(FULL, send, 4);
  }
  const float send = b1 ? w2v[0] : w2v[1];
  float tot = (b1 ? w2v[1] : w2v[0]) + __shfl_xor_sync(FULL, send, 2);
  tot += __shfl_xor_sync(FULL, tot, 1);
  target = (b4 ? 2 : 0) + (b3 ? 1 : 0);
  comp = (b2 ? 2 : 0) + (b1 ? 1 : 0);
  return tot;
}

__global__ void __launch_bounds__(kTravBlock) scatter_kernel(
    const float4* __restrict__ G, const float4* __restrict__ pts,
    const int32_t* __restrict__ npb, const int32_t* __restrict__ npe, const float* __restrict__ s_sorted,
    int64_t q_begin, int64_t q_end, float w2, int stack_depth, double* __restrict__ VB, double* __restrict__ U,
    const int32_t* __restrict__ qorder) {
  extern __shared__ int2 stk_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int2* stk = stk_all + warp * stack_depth;
  const int64_t kq = q_begin + (int64_t)blockIdx.x * kTravBlock + threadIdx.x;  // schedule position
  const bool valid = kq < q_end;
  const int64_t q = (valid && qorder) ? (int64_t)qorder[kq] : kq;
  const float4 xq = valid ? pts[q] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float sq = valid ? s_sorted[q] * kInv4Pi : 0.f;
  const uint32_t active = __ballot_sync(FULL, valid);
  if (!active) return;
  int sp = 0;
  if (lane == 0) stk[0] = make_int2(0, (int)active);
  sp = 1;
  __syncwarp();
  while (sp > 0) {
    --sp;
    const int2 e = stk[sp];
    __syncwarp();
    // lane 0's copies of words every lane read alike: warp-uniform loop control and branches (traverse.cu)
    const int code = __shfl_sync(FULL, e.x, 0);
    const int cb = code >> 4, ncc = (code & 7) + 1;
    const bool mine = ((uint32_t)e.y >> lane) & 1u;
    for (int k0 = 0; k0 < ncc; k0 += 4) {
      // up to four children: each lane's contributions v[4·kk + (x, y, z, ·)], then one reduce-scatter
      float v[16];
      bool anylive = false;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = k0 + kk;
        float cx = 0.f, cy = 0.f, cz = 0.f;
        if (k < ncc) {
          const int node = cb + k;
          const float4 R = __ldg(G + kRec * (int64_t)node);
          const float4 Lo = __ldg(G + kRec * (int64_t)node + 2);
          // d = (hi − x_q) + lo: the decisions of the frozen-geometry A traversal (R-prec)
          const float ex = __fadd_rn(__fsub_rn(R.x, xq.x), Lo.x), ey = __fadd_rn(__fsub_rn(R.y, xq.y), Lo.y),
                      ez = __fadd_rn(__fsub_rn(R.z, xq.z), Lo.z);
          const float d2 = dist2(ex, ey, ez);
          const bool far = d2 > R.w;
          // s_i ∇Φ(x_i − x_B) = s_i d / (4π r³), d = x_B − x_i
          const bool live = mine && far && !(d2 < w2);
          if (live) {
            const float inv = rsqrtf(d2);
            const float c = sq * inv * inv * inv;
            cx = c * ex; cy = c * ey; cz = c * ez;
          }
          anylive |= live;
          const uint32_t open = __ballot_sync(FULL, mine && !far);
          if (open) {
            const int topo = __shfl_sync(FULL, __float_as_int(__ldg(G + kRec * (int64_t)node + 1).w), 0);
            if (topo != 0) {
              if (lane == 0) stk[sp] = make_int2(topo, (int)open);
              ++sp;
            } else {  // leaf-coded node: its points, one butterfly per point into U (grouping: no gain)
              const bool lm = (open >> lane) & 1u;
              const int j0 = __shfl_sync(FULL, npb[node], 0), j1 = __shfl_sync(FULL, npe[node], 0);
              for (int j = j0; j < j1; ++j) {
                const float4 P = __ldg(pts + j);
                const float px = __fsub_rn(P.x, xq.x), py = __fsub_rn(P.y, xq.y), pz = __fsub_rn(P.z, xq.z);
                const float e2 = dist2(px, py, pz);
                float ux = 0.f, uy = 0.f, uz = 0.f;
                const bool lv = lm && !(e2 < w2);
                if (lv) {
                  const float inv = rsqrtf(e2);
                  const float c = sq * inv * inv * inv;
                  ux = c * px; uy = c * py; uz = c * pz;
                }
                if (__any_sync(FULL, lv)) warp_add3(ux, uy, uz, U + 3 * (int64_t)j, lane);
              }
            }
          }
        }
        v[4 * kk + 0] = cx;
        v[4 * kk + 1] = cy;
        v[4 * kk + 2] = cz;
        v[4 * kk + 3] = 0.f;
      }
      if (!__any_sync(FULL, anylive)) continue;
      int child, comp;
      const float tot = reduce_scatter16(v, lane, child, comp);
      if (!(lane & 1) && comp < 3 && k0 + child < ncc && tot != 0.f)
        atomicAdd(VB + 3 * (int64_t)(cb + k0 + child) + comp, (double)tot);
    }
    __syncwarp();
  }
}

// the ranks' accumulators added in rank order (every rank computes the same sums)
struct RankPtrs {
  const double* p[kMaxPeers];
};
__global__ void sum_ranks_kernel(int64_t m, RankPtrs src, int world, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  double acc = src.p[0][i];
  for (int r = 1; r < world; ++r) acc += src.p[r][i];
  out[i] = acc;
}

__global__ void pushdown_kernel(int64_t n, const int32_t* __restrict__ leaf_of, const int32_t* __restrict__ parent,
                                const double* __restrict__ VB, const double* __restrict__ U, float scale,
                                float4* __restrict__ r, double* __restrict__ partial) {
  const int64_t j = (int64_t)blockIdx.x * kTravBlock + threadIdx.x;
  double part = 0.0;
  if (j < n) {
    double x = U[3 * j], y = U[3 * j + 1], z = U[3 * j + 2];
    for (int b = leaf_of[j]; b >= 0; b = parent[b]) {
      x += VB[3 * (int64_t)b];
      y += VB[3 * (int64_t)b + 1];
      z += VB[3 * (int64_t)b + 2];
    }
    const float fx = (float)x * scale, fy = (float)y * scale, fz = (float)z * scale;
    r[j] = make_float4(fx, fy, fz, 0.f);
    part = (double)fx * fx + (double)fy * fy + (double)fz * fz;
  }
  if (partial) {  // one slot per 32 points (kPartQ), as the traversal epilogues
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    if ((threadIdx.x & 31) == 0 && j - (threadIdx.x & 31) < n) partial[j >> 5] = part;
  }
}

}  // namespace

wn_status ensure_transpose_scratch(wn_tree_s* t, cudaStream_t st) {
  if (t->tvb && t->tu) return WN_OK;
  WN_CUDA(cudaMallocAsync((void**)&t->tvb, 3 * sizeof(double) * (size_t)t->nn, st));
  WN_CUDA(cudaMallocAsync((void**)&t->tu, 3 * sizeof(double) * (size_t)t->n, st));
  return WN_OK;
}

wn_status adjoint_transpose(wn_tree_s* t, const NodeSet& geo, const float* s_sorted, float w2, float4* r_out,
                            double* partial, cudaStream_t st) {
  // (inside a graph capture the accumulators exist already: wnnc_iterate allocates them before capturing)
  WN_TRY(ensure_transpose_scratch(t, st));
  WN_CUDA(cudaMemsetAsync(t->tvb, 0, 3 * sizeof(double) * (size_t)t->nn, st));
  WN_CUDA(cudaMemsetAsync(t->tu, 0, 3 * sizeof(double) * (size_t)t->n, st));
  const int stack_depth = 8 * (t->depth_used + 2);
  const unsigned grid = (unsigned)trav_blocks(t->n);
  {
    ProfScope ps(WN_PROF_TRAV_AT, st, 2);
    scatter_kernel<<<grid, kTravBlock, (size_t)(kTravBlock / 32) * stack_depth * sizeof(int2), st>>>(
        geo.rec, t->pts, t->pb, t->pe, s_sorted, 0, t->n, w2, stack_depth, t->tvb, t->tu, t->qorder);
    pushdown_kernel<<<grid, kTravBlock, 0, st>>>(t->n, t->leaf_of, t->parent, t->tvb, t->tu, 1.0f, r_out, partial);
  }
  count_launches(2);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

wn_status adjoint_scatter_shard(wn_tree_s* t, const NodeSet& geo, const float* s_sorted, float w2, int64_t q0,
                                int64_t q1, double* vb, double* u, cudaStream_t st) {
  WN_CUDA(cudaMemsetAsync(vb, 0, 3 * sizeof(double) * (size_t)t->nn, st));
  WN_CUDA(cudaMemsetAsync(u, 0, 3 * sizeof(double) * (size_t)t->n, st));
  if (q1 <= q0) return WN_OK;
  const int stack_depth = 8 * (t->depth_used + 2);
  ProfScope ps(WN_PROF_TRAV_AT, st, 1);
  scatter_kernel<<<(unsigned)trav_blocks(q1 - q0), kTravBlock, (size_t)(kTravBlock / 32) * stack_depth * sizeof(int2),
                   st>>>(geo.rec, t->pts, t->pb, t->pe, s_sorted, q0, q1, w2, stack_depth, vb, u, t->qorder);
  count_launches(1);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

wn_status adjoint_reduce_pushdown(wn_tree_s* t, const double* const* vbs, const double* const* us, int world,
                                  float4* r_out, double* partial, cudaStream_t st) {
  WN_TRY(ensure_transpose_scratch(t, st));
  if (world < 1 || world > kMaxPeers) return set_error(WN_ERR_ARG, "internal: adjoint world size");
  RankPtrs pv{}, pu{};
  for (int r = 0; r < world; ++r) {
    pv.p[r] = vbs[r];
    pu.p[r] = us[r];
  }
  ProfScope ps(WN_PROF_TRAV_AT, st, 3);
  const int64_t mv = 3 * t->nn, mu = 3 * t->n;
  sum_ranks_kernel<<<(unsigned)((mv + 255) / 256), 256, 0, st>>>(mv, pv, world, t->tvb);
  sum_ranks_kernel<<<(unsigned)((mu + 255) / 256), 256, 0, st>>>(mu, pu, world, t->tu);
  pushdown_kernel<<<(unsigned)trav_blocks(t->n), kTravBlock, 0, st>>>(t->n, t->leaf_of, t->parent, t->tvb, t->tu,
                                                                       1.0f, r_out, partial);
  count_launches(3);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

}  // namespace wn
