// tree_build.cu — octree construction on the device.
//
// PAPER.md:L370 (§4.5): "we first build an octree T to spatially partition the input point set.
// The partitioning stops if the node contains only one point or if the user-specified maximum depth
// D is reached."  PAPER.md:L419 (§5.1.1): points are "normalized to fit into the cube [−1,1]^3 with
// a margin of 1/11".  Readings: root cell = [−1,1]^3, bbox-centred uniform scale with the
// longest half-extent at 10/11, children in ascending octant digit 4·x + 2·y + z, a coordinate on a
// split plane goes to the upper octant.
//
// B200 design: instead of the recursive partition the paper implies, the tree is emitted from sorted
// Morton keys.  For sorted keys k_0 ≤ … ≤ k_{N−1} let lcp(k) be the number of leading octal digits
// shared by keys k−1 and k (lcp(0) = lcp(N) = −1).  A node at level ℓ is a run of points sharing ℓ
// digits whose parent run holds ≥ 2 points; point k starts exactly the nodes of levels
//     lo_k = lcp(k) + 1  …  hi_k = min(D, max(lcp(k) + 1, lcp(k+1) + 1))
// and node (ℓ, k) is internal iff ℓ < hi_k (its first child is (ℓ+1, k)).  BFS order = (level, k).
// Kernels: bbox → normalize + keys → stable LSD radix sort (8-bit digits, match_any ranking) →
// gather → per-tile level counts → one flat scan → emission → parent / child-count → per-level pe.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "wn_internal.cuh"

namespace wn {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;                    // per thread → 2048 keys per tile
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kEmitThreads = 256;                // points per emission tile

struct BBox {
  float lo[3], hi[3];
  int nonfinite;
  int pad;
  double xf[4];
};

__global__ void bbox_partial(const float* __restrict__ p, int64_t n, float* __restrict__ part, int* bad) {
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  int nf = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float v = p[3 * i + a];
      if (!isfinite(v)) nf = 1;
      lo[a] = fminf(lo[a], v);
      hi[a] = fmaxf(hi[a], v);
    }
  }
  __shared__ float slo[3][32], shi[3][32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if (lane == 0) { slo[a][w] = lo[a]; shi[a][w] = hi[a]; }
  }
  if (__any_sync(0xffffffffu, nf) && lane == 0) atomicOr(bad, 1);
  __syncthreads();
  if (threadIdx.x < 3) {
    int a = threadIdx.x;
    float l = INFINITY, h = -INFINITY;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { l = fminf(l, slo[a][k]); h = fmaxf(h, shi[a][k]); }
    part[6 * blockIdx.x + a] = l;
    part[6 * blockIdx.x + 3 + a] = h;
  }
}

// xf = (c, scale): c = (lo + hi)/2, half = max_a (hi − lo)/2, scale = (10/11)/half  (fp64)
__global__ void __launch_bounds__(1024) bbox_final(const float* __restrict__ part, int nb, const int* bad, BBox* out) {
  __shared__ float slo[3][32], shi[3][32];
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    for (int a = 0; a < 3; ++a) {
      lo[a] = fminf(lo[a], part[6 * b + a]);
      hi[a] = fmaxf(hi[a], part[6 * b + 3 + a]);
    }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if (lane == 0) { slo[a][w] = lo[a]; shi[a][w] = hi[a]; }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { lo[a] = fminf(lo[a], slo[a][k]); hi[a] = fmaxf(hi[a], shi[a][k]); }
  double half = 0.0;
  for (int a = 0; a < 3; ++a) {
    out->lo[a] = lo[a];
    out->hi[a] = hi[a];
    out->xf[a] = ((double)lo[a] + (double)hi[a]) * 0.5;
    double h = ((double)hi[a] - (double)lo[a]) * 0.5;
    if (h > half) half = h;
  }
  out->xf[3] = half > 0.0 ? (10.0 / 11.0) / half : 0.0;
  out->nonfinite = *bad;
}

__device__ __forceinline__ uint64_t spread3(uint32_t v) {  // 21 bits → every third bit
  uint64_t x = v & 0x1fffffu;
  x = (x | (x << 32)) & 0x1f00000000ffffull;
  x = (x | (x << 16)) & 0x1f0000ff0000ffull;
  x = (x | (x << 8)) & 0x100f00f00f00f00full;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

__device__ __forceinline__ uint32_t quantize(float xn, int D) {
  double v = floor(((double)xn + 1.0) * ldexp(1.0, D - 1));
  double qmax = (double)((1u << D) - 1u);
  v = fmin(fmax(v, 0.0), qmax);
  return (uint32_t)v;
}

__global__ void normalize_keys(const float* __restrict__ p, int64_t n, const BBox* bb, int D,
                               float4* __restrict__ xn, uint64_t* __restrict__ keys, int32_t* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double c0 = bb->xf[0], c1 = bb->xf[1], c2 = bb->xf[2], sc = bb->xf[3];
  float x = (float)(__dsub_rn((double)p[3 * i + 0], c0) * sc);
  float y = (float)(__dsub_rn((double)p[3 * i + 1], c1) * sc);
  float z = (float)(__dsub_rn((double)p[3 * i + 2], c2) * sc);
  xn[i] = make_float4(x, y, z, 0.f);
  uint32_t qx = quantize(x, D), qy = quantize(y, D), qz = quantize(z, D);
  keys[i] = (spread3(qx) << 2) | (spread3(qy) << 1) | spread3(qz);
  idx[i] = (int32_t)i;
}

// ---- stable LSD radix sort of (key, idx) ------------------------------------------------------
__global__ void radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift, int ntiles,
                           uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int k = 0; k < kSortItems; ++k) {
    int64_t i = base + k * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void radix_scatter(const uint64_t* __restrict__ kin, const int32_t* __restrict__ vin,
                              uint64_t* __restrict__ kout, int32_t* __restrict__ vout, int64_t n, int shift,
                              int ntiles, const uint32_t* __restrict__ offs) {
  constexpr int W = kSortThreads / 32;
  __shared__ uint32_t wcnt[W][256];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < W * 256; d += kSortThreads) (&wcnt[0][0])[d] = 0;
  __syncthreads();
  // each warp owns a contiguous chunk of kSortItems*32 keys of the tile → tile order preserved
  int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)w * (kSortItems * 32);
  const uint32_t lt = (1u << lane) - 1u;
  for (int r = 0; r < kSortItems; ++r) {
    int64_t i = base + r * 32 + lane;
    uint32_t d = i < n ? (uint32_t)((kin[i] >> shift) & 255u) : 256u;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (d < 256u && lane == __ffs(peers) - 1) wcnt[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    int d = threadIdx.x;  // 256 threads ↔ 256 digits
    uint32_t run = offs[(int64_t)d * ntiles + blockIdx.x];
    for (int k = 0; k < W; ++k) {
      uint32_t c = wcnt[k][d];
      wcnt[k][d] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int r = 0; r < kSortItems; ++r) {
    int64_t i = base + r * 32 + lane;
    uint64_t key = i < n ? kin[i] : 0;
    uint32_t d = i < n ? (uint32_t)((key >> shift) & 255u) : 256u;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t pos = 0;
    if (d < 256u) pos = wcnt[w][d] + __popc(peers & lt);
    __syncwarp();
    if (d < 256u) {
      kout[pos] = key;
      vout[pos] = vin[i];
      if (lane == __ffs(peers) - 1) wcnt[w][d] += __popc(peers);
    }
    __syncwarp();
  }
}

// exclusive scan of m uint32 (exact integer sums: any association gives the same result), three launches:
// per-block totals (4096 elements per block), one-block scan of the totals, per-block scan + offset
constexpr int kScanT = 1024, kScanPer = 4, kScanBlk = kScanT * kScanPer;

__device__ __forceinline__ uint32_t block_exscan_u32(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[kScanT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    ws[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t r = (w ? ws[w - 1] : 0u) + x - v;
  if (total) *total = ws[kScanT / 32 - 1];
  __syncthreads();
  return r;
}

__device__ __forceinline__ void load4(const uint32_t* __restrict__ in, int64_t i, int64_t m, uint32_t v[4]) {
  if (i + 3 < m && ((reinterpret_cast<uintptr_t>(in + i) & 15) == 0)) {
    const uint4 q = *reinterpret_cast<const uint4*>(in + i);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i + k < m ? in[i + k] : 0u;
  }
}

__global__ void __launch_bounds__(kScanT) scan_blocks(const uint32_t* __restrict__ in, int64_t m,
                                                      uint32_t* __restrict__ bsum) {
  uint32_t v[4];
  load4(in, (int64_t)blockIdx.x * kScanBlk + kScanPer * threadIdx.x, m, v);
  uint32_t tot;
  block_exscan_u32(v[0] + v[1] + v[2] + v[3], &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanT) scan_top(uint32_t* __restrict__ bsum, int nb, uint32_t* total) {
  uint32_t run = 0;
  for (int b0 = 0; b0 < nb; b0 += kScanT) {  // nb ≤ a few thousand
    const int b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? bsum[b] : 0u;
    uint32_t tot;
    const uint32_t e = block_exscan_u32(v, &tot);
    if (b < nb) bsum[b] = run + e;
    run += tot;
  }
  if (threadIdx.x == 0 && total) *total = run;
}

__global__ void __launch_bounds__(kScanT) scan_apply(const uint32_t* in, uint32_t* out, int64_t m,
                                                     const uint32_t* __restrict__ boff) {
  const int64_t i = (int64_t)blockIdx.x * kScanBlk + kScanPer * threadIdx.x;
  uint32_t v[4];
  load4(in, i, m, v);
  uint32_t run = boff[blockIdx.x] + block_exscan_u32(v[0] + v[1] + v[2] + v[3], nullptr);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (i + k < m) {
      out[i + k] = run;
      run += v[k];
    }
}

__global__ void gather_sorted(const float4* __restrict__ xn, const int32_t* __restrict__ idx, int64_t n,
                              float4* __restrict__ pts, int32_t* __restrict__ perm) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t j = idx[k];
  pts[k] = xn[j];
  perm[k] = j;
}

// 3-D Hilbert index of a point (Skilling's transpose algorithm) on a 2^kHilbertBits grid of [−1,1]^3
#ifndef WN_EXP_HBITS
#define WN_EXP_HBITS 10
#endif
constexpr int kHilbertBits = WN_EXP_HBITS;
__global__ void hilbert_keys(const float4* __restrict__ pts, int64_t n, uint64_t* __restrict__ hk,
                             int32_t* __restrict__ hv) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const float4 p = pts[k];
  uint32_t X[3] = {quantize(p.x, kHilbertBits), quantize(p.y, kHilbertBits), quantize(p.z, kHilbertBits)};
  const uint32_t M = 1u << (kHilbertBits - 1);
  for (uint32_t Q = M; Q > 1; Q >>= 1) {  // inverse undo
    const uint32_t P = Q - 1;
    for (int i = 0; i < 3; ++i) {
      if (X[i] & Q) {
        X[0] ^= P;
      } else {
        const uint32_t t = (X[0] ^ X[i]) & P;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  for (int i = 1; i < 3; ++i) X[i] ^= X[i - 1];  // Gray encode
  uint32_t t = 0;
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  for (int i = 0; i < 3; ++i) X[i] ^= t;
  uint64_t h = 0;
  for (int b = kHilbertBits - 1; b >= 0; --b)
    h = (h << 3) | (((X[0] >> b) & 1u) << 2) | (((X[1] >> b) & 1u) << 1) | ((X[2] >> b) & 1u);
  hk[k] = h;
  hv[k] = (int32_t)k;
}

__device__ __forceinline__ int common_digits(uint64_t a, uint64_t b, int D) {
  if (a == b) return D;
  return (__clzll((long long)(a ^ b)) - (64 - 3 * D)) / 3;
}

// levels started by point k: [lo, hi] (lo > hi ⇒ none)
__device__ __forceinline__ void level_range(const uint64_t* keys, int64_t n, int D, int64_t k, int& lo, int& hi) {
  int l0 = k == 0 ? -1 : common_digits(keys[k - 1], keys[k], D);
  int l1 = k + 1 >= n ? -1 : common_digits(keys[k], keys[k + 1], D);
  lo = l0 + 1;
  hi = min(D, max(l0 + 1, l1 + 1));
}

__global__ void level_counts(const uint64_t* __restrict__ keys, int64_t n, int D, int ntiles,
                             uint32_t* __restrict__ cnt) {
  __shared__ uint32_t c[kMaxDepth + 1];
  if (threadIdx.x <= D) c[threadIdx.x] = 0;
  __syncthreads();
  int64_t k = blockIdx.x * (int64_t)kEmitThreads + threadIdx.x;
  int lo = 1, hi = 0;
  if (k < n) level_range(keys, n, D, k, lo, hi);
  int lane = threadIdx.x & 31;
  for (int l = 0; l <= D; ++l) {
    uint32_t b = __ballot_sync(0xffffffffu, lo <= l && l <= hi);
    if (lane == 0 && b) atomicAdd(&c[l], __popc(b));
  }
  __syncthreads();
  if (threadIdx.x <= D) cnt[(int64_t)threadIdx.x * ntiles + blockIdx.x] = c[threadIdx.x];
}

__global__ void emit_nodes(const uint64_t* __restrict__ keys, int64_t n, int D, int ntiles,
                           const uint32_t* __restrict__ offs, int32_t* __restrict__ depth, int32_t* __restrict__ pb,
                           int32_t* __restrict__ cb, int32_t* __restrict__ cc, int32_t* __restrict__ parent) {
  constexpr int W = kEmitThreads / 32;
  __shared__ uint32_t wtot[W][kMaxDepth + 1];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t k = blockIdx.x * (int64_t)kEmitThreads + threadIdx.x;
  int lo = 1, hi = 0;
  if (k < n) level_range(keys, n, D, k, lo, hi);
  for (int l = 0; l <= D; ++l) {
    uint32_t b = __ballot_sync(0xffffffffu, lo <= l && l <= hi);
    if (lane == 0) wtot[w][l] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x <= D) {  // exclusive scan over warps, per level
    uint32_t run = 0;
    for (int q = 0; q < W; ++q) {
      uint32_t v = wtot[q][threadIdx.x];
      wtot[q][threadIdx.x] = run;
      run += v;
    }
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  int32_t prev = -1;
  for (int l = 0; l <= D; ++l) {
    bool f = lo <= l && l <= hi;
    uint32_t b = __ballot_sync(0xffffffffu, f);
    if (!f) continue;
    int32_t idx = (int32_t)(offs[(int64_t)l * ntiles + blockIdx.x] + wtot[w][l] + __popc(b & lt));
    depth[idx] = l;
    pb[idx] = (int32_t)k;
    if (l < hi) {          // internal: first child is (l+1, k), count filled by child_counts
      cc[idx] = 0;
    } else {               // leaf
      cb[idx] = -1;
      cc[idx] = 0;
    }
    if (l > lo) {
      parent[idx] = prev;
      cb[prev] = idx;
    } else {
      parent[idx] = l == 0 ? -1 : -2;   // −2: parent starts at an earlier point → binary search
    }
    prev = idx;
  }
}

__global__ void find_parents(int64_t nn, const int32_t* __restrict__ depth, const int32_t* __restrict__ pb,
                             const int64_t* __restrict__ loff, int32_t* __restrict__ parent) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn || parent[i] != -2) return;
  int l = depth[i];
  int32_t key = pb[i];
  int64_t a = loff[l - 1], b = loff[l] - 1;   // largest j in [a, b] with pb[j] ≤ key
  while (a < b) {
    int64_t m = (a + b + 1) >> 1;
    if (pb[m] <= key) a = m; else b = m - 1;
  }
  parent[i] = (int32_t)a;
}

__global__ void child_counts(int64_t nn, const int32_t* __restrict__ depth, const int32_t* __restrict__ parent,
                             const int64_t* __restrict__ loff, const int32_t* __restrict__ cb,
                             int32_t* __restrict__ cc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < 1 || i >= nn) return;
  int32_t p = parent[i];
  bool last = (i + 1 == loff[depth[i] + 1]) || parent[i + 1] != p;
  if (last) cc[p] = (int32_t)(i - cb[p] + 1);
}

// Traversal code per node: leaf 0; internal (child_begin << 4) | (count − 1).  A chain of single-child
// nodes holds the same points at every level — the same representative and ν_B — while its threshold
// (c·edge)² shrinks by 4 per level, so a lane is far somewhere in the chain iff it is far at the chain's
// bottom, and the term is the same at every level: the chain's top takes the bottom's children, the
// bottom's one-point-child mask and the bottom's depth for its threshold (tdepth), and the chain length
// goes to smask bits 8..12 (the counting traversal re-derives Alg. 4's per-level tests from it).
// Nodes strictly inside a chain are never visited.
__global__ void topo_codes(int64_t nn, const int32_t* __restrict__ cb, const int32_t* __restrict__ cc,
                           const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                           const int32_t* __restrict__ depth, int32_t* __restrict__ topo, int32_t* __restrict__ smask,
                           int32_t* __restrict__ tdepth) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  int64_t b = i;  // chain bottom
  int len = 1;
#ifndef WN_EXP_NOCHAIN
  while (cc[b] == 1) {
    b = cb[b];
    ++len;
  }
#endif
  tdepth[i] = depth[b];
  const int nc = cc[b];
  if (nc == 0) {
    topo[i] = 0;
    smask[i] = len << 8;
    return;
  }
  const int c0 = cb[b];
  int single = 0;  // bit k: child k is a one-point leaf
  for (int c = c0; c < c0 + nc; ++c) single |= ((cc[c] == 0) && (pe[c] - pb[c] == 1)) << (c - c0);
#ifndef WN_EXP_NOPSEUDO
  if (single == (1 << nc) - 1) {
    // every child is a one-point leaf, whose term is exactly its point's direct term (rep = the point,
    // ν_B = ν_j, lo = 0): opening the node = a direct sum over its points, like a multi-point leaf —
    // no child group to push and pop.  Bit 13 tells the counting traversal to count one node test per
    // point, as Alg. 4 tests each child.
    topo[i] = 0;
    smask[i] = single | (len << 8) | (1 << 13);
    return;
  }
#endif
  topo[i] = (c0 << 4) | (nc - 1);
  smask[i] = single | (len << 8);
}

// the nodes a traversal can visit: the root and every child group referenced by an internal code
__global__ void mark_visited(int64_t nn, const int32_t* __restrict__ topo, uint32_t* __restrict__ vis) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  if (i == 0) vis[0] = 1;
  const int code = topo[i];
  if (code != 0) {
    const int c0 = code >> 4, nc = (code & 7) + 1;
    for (int c = c0; c < c0 + nc; ++c) vis[c] = 1;
  }
}
__global__ void compact_visited(int64_t nn, const uint32_t* __restrict__ vis, const uint32_t* __restrict__ pos,
                                int32_t* __restrict__ list) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nn && vis[i]) list[pos[i]] = (int32_t)i;
}

__global__ void level_pe(int64_t i0, int64_t i1, int64_t n, const int32_t* __restrict__ parent,
                         const int32_t* __restrict__ pb, int32_t* __restrict__ pe) {
  int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= i1) return;
  int32_t p = parent[i];
  if (p < 0) { pe[i] = (int32_t)n; return; }
  bool last = (i + 1 == i1) || parent[i + 1] != p;
  pe[i] = last ? pe[p] : pb[i + 1];
}

template <typename T>
wn_status dalloc(T** p, size_t count, cudaStream_t s) {
  cudaError_t e = cudaMallocAsync((void**)p, std::max<size_t>(count, 1) * sizeof(T), s);
  if (e == cudaErrorMemoryAllocation) return set_error(WN_ERR_OOM, "device allocation failed");
  if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync");
  return WN_OK;
}

// temporaries of one host routine: every block still held is freed (stream-ordered) when the routine
// returns, on the error paths too; keep() hands a block over to a longer-lived owner
struct TempSet {
  cudaStream_t s;
  std::vector<void*> held;
  explicit TempSet(cudaStream_t st) : s(st) {}
  ~TempSet() {
    for (void* p : held) cudaFreeAsync(p, s);
  }
  template <typename T>
  wn_status alloc(T** p, size_t count) {
    *p = nullptr;
    WN_TRY(dalloc(p, count, s));
    held.push_back((void*)*p);
    return WN_OK;
  }
  void keep(void* p) {
    for (auto& q : held)
      if (q == p) q = held.back(), held.pop_back();
  }
  void release(void* p) {
    keep(p);
    cudaFreeAsync(p, s);
  }
};

// exclusive scan (in may equal out); total (device) optional
wn_status scan_excl(const uint32_t* in, uint32_t* out, int64_t m, uint32_t* total, cudaStream_t s) {
  const int nb = (int)((m + kScanBlk - 1) / kScanBlk);
  uint32_t* bsum = nullptr;
  wn_status st = dalloc(&bsum, (size_t)nb, s);
  if (st != WN_OK) return st;
  scan_blocks<<<nb, kScanT, 0, s>>>(in, m, bsum);
  scan_top<<<1, kScanT, 0, s>>>(bsum, nb, total);
  scan_apply<<<nb, kScanT, 0, s>>>(in, out, m, bsum);
  cudaFreeAsync(bsum, s);
  return WN_OK;
}

}  // namespace

// stable LSD radix sort of (key, value) pairs on the low `bits` bits of the keys; ka / va are consumed,
// the values in key order are copied to out
static wn_status sort_pairs(uint64_t* ka, int32_t* va, int64_t n, int bits, int32_t* out, cudaStream_t s,
                            uint64_t* kout = nullptr) {
  const int ntiles = (int)((n + kSortTile - 1) / kSortTile);
  uint64_t* kb = nullptr;
  int32_t* vb = nullptr;
  uint32_t* hist = nullptr;
  TempSet tmp(s);  // kb, vb, hist: freed here whatever the parity of the passes (and on errors)
  WN_TRY(tmp.alloc(&kb, n));
  WN_TRY(tmp.alloc(&vb, n));
  WN_TRY(tmp.alloc(&hist, (size_t)256 * ntiles));
  const int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    radix_hist<<<ntiles, kSortThreads, 0, s>>>(ka, n, 8 * p, ntiles, hist);
    WN_TRY(scan_excl(hist, hist, (int64_t)256 * ntiles, nullptr, s));
    radix_scatter<<<ntiles, kSortThreads, 0, s>>>(ka, va, kb, vb, n, 8 * p, ntiles, hist);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  WN_CUDA(cudaMemcpyAsync(out, va, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if (kout) WN_CUDA(cudaMemcpyAsync(kout, ka, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  count_launches(5 * passes);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

wn_status fmm_scan(const uint32_t* in, uint32_t* out, int64_t m, uint32_t* total, cudaStream_t s) {
  return scan_excl(in, out, m, total, s);
}
wn_status scan_u32(const uint32_t* in, uint32_t* out, int64_t m, uint32_t* total, cudaStream_t s) {
  return scan_excl(in, out, m, total, s);
}

// ascending sort of n 64-bit keys on their low `bits` bits (stable LSD radix), out = the sorted keys
__global__ void k_iota(int64_t n, int32_t* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}
wn_status sort_keys_u64(const uint64_t* keys, int64_t n, int bits, uint64_t* out, cudaStream_t s) {
  if (n <= 0) return WN_OK;
  TempSet tmp(s);
  uint64_t* ka = nullptr;
  int32_t *va = nullptr, *vo = nullptr;
  WN_TRY(tmp.alloc(&ka, n));
  WN_TRY(tmp.alloc(&va, n));
  WN_TRY(tmp.alloc(&vo, n));
  WN_CUDA(cudaMemcpyAsync(ka, keys, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  k_iota<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, va);
  count_launches(1);
  return sort_pairs(ka, va, n, bits, vo, s, out);
}
// the same, also returning the permutation: perm[k] = the input position of the k-th sorted key
wn_status sort_keys_u64_perm(const uint64_t* keys, int64_t n, int bits, uint64_t* out, int32_t* perm,
                             cudaStream_t s) {
  if (n <= 0) return WN_OK;
  TempSet tmp(s);
  uint64_t* ka = nullptr;
  int32_t* va = nullptr;
  WN_TRY(tmp.alloc(&ka, n));
  WN_TRY(tmp.alloc(&va, n));
  WN_CUDA(cudaMemcpyAsync(ka, keys, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  k_iota<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, va);
  count_launches(1);
  return sort_pairs(ka, va, n, bits, perm, s, out);
}

wn_status hilbert_schedule(const float4* pts, int64_t n, int32_t* order, cudaStream_t s) {
  if (n <= 0) return WN_OK;
  uint64_t* ka = nullptr;
  int32_t* va = nullptr;
  TempSet tmp(s);
  WN_TRY(tmp.alloc(&ka, n));
  WN_TRY(tmp.alloc(&va, n));
  const int hbits = 3 * kHilbertBits;
  {
    ProfScope ps(WN_PROF_TREE, s, 0);
    hilbert_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pts, n, ka, va);
    count_launches(1);
    WN_TRY(sort_pairs(ka, va, n, hbits, order, s));
  }
  return WN_OK;
}

// ---- k-d query schedule -----------------------------------------------------------------------------
// A warp takes 32 consecutive schedule positions. Grouping them by recursive median splits — k-d boxes of
// 32 queries — instead of Hilbert-curve runs makes a warp's queries more compact, so fewer child groups
// are visited with a partial lane mask (C3: −9 % warp-level visits). Level-synchronous on the GPU: every
// segment of the current order holding more than 32 queries is stably sorted along the axis of its
// largest robust extent and split at a multiple of 32 (left part: ⌊⌈m/32⌉/2⌋·32 queries).
constexpr int kKdQBits = 16;  // coordinate quantization of the sort keys (ties keep the previous order)

__global__ void kd_iota(int64_t n, int32_t* __restrict__ order, int32_t* __restrict__ seg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  order[i] = (int32_t)i;
  seg[i] = 0;
}

// split axis of each segment: the extent of a 16-point sample (evenly spaced in the current order) without
// its two extremes per side — robust to the few far outliers that would otherwise select the normal axis
// of a thin surface patch; 3 = no split (≤ 32 queries)
__global__ void kd_axes(const float4* __restrict__ pts, const int32_t* __restrict__ order,
                        const int32_t* __restrict__ sb, const int32_t* __restrict__ se, int nseg,
                        uint8_t* __restrict__ axis) {
  const int sg = blockIdx.x * blockDim.x + threadIdx.x;
  if (sg >= nseg) return;
  const int b = sb[sg], m = se[sg] - b;
  if (m <= 32) {
    axis[sg] = 3;
    return;
  }
  float4 smp[16];  // the 16 sample points, loaded together
#pragma unroll
  for (int k = 0; k < 16; ++k) smp[k] = pts[order[b + (int)(((int64_t)k * m) / 16)]];
  float best = -1.f;
  int ax = 0;
  for (int c = 0; c < 3; ++c) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = c == 0 ? smp[k].x : (c == 1 ? smp[k].y : smp[k].z);
    for (int i = 1; i < 16; ++i) {  // insertion sort of the sample
      const float x = v[i];
      int j = i - 1;
      while (j >= 0 && v[j] > x) {
        v[j + 1] = v[j];
        --j;
      }
      v[j + 1] = x;
    }
    const float e = v[13] - v[2];
    if (e > best) {
      best = e;
      ax = c;
    }
  }
  axis[sg] = (uint8_t)ax;
}

__global__ void kd_keys(const float4* __restrict__ pts, const int32_t* __restrict__ order,
                        const int32_t* __restrict__ seg, const uint8_t* __restrict__ axis, int64_t n,
                        uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int sg = seg[i], ax = axis[sg];
  const int32_t q = order[i];
  uint32_t c = 0;
  if (ax < 3) {
    const float4 p = pts[q];
    c = quantize(ax == 0 ? p.x : (ax == 1 ? p.y : p.z), kKdQBits);
  }
  key[i] = ((uint64_t)sg << kKdQBits) | c;
  val[i] = q;
}

// after the sort: each query's half of its segment, and the children's ranges (segment 2s: left, 2s+1: right)
__global__ void kd_split(const uint64_t* __restrict__ skey, int64_t n, const int32_t* __restrict__ sb,
                         const int32_t* __restrict__ se, int32_t* __restrict__ seg, int32_t* __restrict__ sb2,
                         int32_t* __restrict__ se2) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int sg = (int)(skey[i] >> kKdQBits);
  const int b = sb[sg], e = se[sg], m = e - b;
  WN_DCHECK(b <= i && i < e, "k-d segment of a query");
  const int left = m > 32 ? (((m + 31) / 32) / 2) * 32 : m;
  seg[i] = 2 * sg + ((int)i - b >= left ? 1 : 0);
  if (i == b) {
    sb2[2 * sg] = b;
    se2[2 * sg] = b + left;
    sb2[2 * sg + 1] = b + left;
    se2[2 * sg + 1] = e;
  }
}

// the last levels of a segment of ≤ kKdLocal queries inside one block: the same splits, the sort a bitonic
// sort in shared memory on unique keys (sub-segment, coordinate, position): equal coordinates keep the
// previous order, as in the global levels
constexpr int kKdLocal = 2048;
__device__ __forceinline__ unsigned long long kd_fkey(float f) {  // order-preserving float → 32-bit key
  const uint32_t u = __float_as_uint(f);
  return (unsigned long long)((u & 0x80000000u) ? ~u : (u | 0x80000000u));
}

__global__ void __launch_bounds__(1024) kd_local(const float4* __restrict__ pts, int32_t* __restrict__ order,
                                                 const int32_t* __restrict__ sb, const int32_t* __restrict__ se) {
  __shared__ unsigned long long key[kKdLocal];
  __shared__ int32_t id[kKdLocal];  // (coordinates re-read from pts: L1/L2-resident)
  __shared__ uint8_t sid[kKdLocal];
  __shared__ int16_t ssb[128], sse[128], nsb[128], nse[128];
  __shared__ uint8_t sax[128];
  __shared__ int nsub, more;
  const int b = sb[blockIdx.x], m = se[blockIdx.x] - b, tid = threadIdx.x;
  WN_DCHECK(b >= 0 && m >= 0 && m <= kKdLocal, "k-d local segment");
  if (m <= 32) return;  // (uniform: one segment per block)
  for (int i = tid; i < m; i += 1024) {
    id[i] = order[b + i];
    sid[i] = 0;
  }
  if (tid == 0) {
    nsub = 1;
    ssb[0] = 0;
    sse[0] = (int16_t)m;
  }
  __syncthreads();
  int M = 32;
  while (M < m) M <<= 1;
  for (;;) {
    if (tid == 0) {
      int mo = 0;
      for (int k = 0; k < nsub; ++k) mo |= (sse[k] - ssb[k]) > 32;
      more = mo;
    }
    __syncthreads();
    if (!more) break;
    if (tid < nsub) {  // split axis (as kd_axes: robust extent of a 16-point sample)
      const int bb = ssb[tid], mm = sse[tid] - bb;
      int ax = 3;
      if (mm > 32) {
        float4 smp[16];  // the 16 sample points, loaded together
#pragma unroll
        for (int k = 0; k < 16; ++k) smp[k] = pts[id[bb + (k * mm) / 16]];
        float best = -1.f;
        for (int c = 0; c < 3; ++c) {
          float v[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = c == 0 ? smp[k].x : (c == 1 ? smp[k].y : smp[k].z);
          for (int i = 1; i < 16; ++i) {
            const float x = v[i];
            int j = i - 1;
            while (j >= 0 && v[j] > x) {
              v[j + 1] = v[j];
              --j;
            }
            v[j + 1] = x;
          }
          const float e = v[13] - v[2];
          if (e > best) {
            best = e;
            ax = c;
          }
        }
      }
      sax[tid] = (uint8_t)ax;
    }
    __syncthreads();
    for (int i = tid; i < M; i += 1024) {
      if (i < m) {
        const int g = sid[i], ax = sax[g];
        unsigned long long c = 0ull;
        if (ax < 3) {
          const float4 p = pts[id[i]];
          c = kd_fkey(ax == 0 ? p.x : (ax == 1 ? p.y : p.z));
        }
        key[i] = ((unsigned long long)g << 43) | (c << 11) | (unsigned long long)i;
      } else {
        key[i] = ~0ull;
      }
    }
    __syncthreads();
    for (int k = 2; k <= M; k <<= 1)  // bitonic sort, ascending
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < M; i += 1024) {
          const int l = i ^ j;
          if (l > i) {
            const unsigned long long x = key[i], y = key[l];
            if (((i & k) == 0) == (x > y)) {
              key[i] = y;
              key[l] = x;
            }
          }
        }
        __syncthreads();
      }
    // gather into the new order, then the children's ranges and each query's child
    int32_t rid[2];
    uint8_t rs[2];
    for (int r = 0; r < 2; ++r) {
      const int i = tid + r * 1024;
      if (i < m) {
        const int src = (int)(key[i] & 0x7FFull);
        rid[r] = id[src];
        rs[r] = (uint8_t)(key[i] >> 43);
      }
    }
    __syncthreads();
    for (int r = 0; r < 2; ++r) {
      const int i = tid + r * 1024;
      if (i < m) {
        id[i] = rid[r];
        const int g = rs[r], bb = ssb[g], mm = sse[g] - bb;
        const int left = mm > 32 ? (((mm + 31) / 32) / 2) * 32 : mm;
        sid[i] = (uint8_t)(2 * g + (i - bb >= left ? 1 : 0));
      }
    }
    if (tid < nsub) {
      const int bb = ssb[tid], mm = sse[tid] - bb;
      const int left = mm > 32 ? (((mm + 31) / 32) / 2) * 32 : mm;
      nsb[2 * tid] = (int16_t)bb;
      nse[2 * tid] = (int16_t)(bb + left);
      nsb[2 * tid + 1] = (int16_t)(bb + left);
      nse[2 * tid + 1] = (int16_t)(bb + mm);
    }
    __syncthreads();
    if (tid < 2 * nsub) {
      ssb[tid] = nsb[tid];
      sse[tid] = nse[tid];
    }
    __syncthreads();
    if (tid == 0) nsub *= 2;
    __syncthreads();
  }
  for (int i = tid; i < m; i += 1024) order[b + i] = id[i];
}

wn_status kd_levels(const float4* pts, int64_t n, int levels, int32_t* order, uint64_t* key, uint64_t* skey,
                    int32_t* val, int32_t* seg, int32_t* sb, int32_t* se, int32_t* sb2, int32_t* se2, uint8_t* axis,
                    cudaStream_t s);

wn_status kd_schedule(const float4* pts, int64_t n, int32_t* order, cudaStream_t s) {
  if (n <= 0) return WN_OK;
  int levels = 0;  // global splits until every segment holds ≤ kKdLocal queries (from the sizes alone)
  {
    std::vector<int64_t> sz{n};
    while (*std::max_element(sz.begin(), sz.end()) > kKdLocal) {
      std::vector<int64_t> nx;
      for (int64_t m : sz) {
        if (m <= 32) continue;
        const int64_t left = (((m + 31) / 32) / 2) * 32;
        nx.push_back(left);
        nx.push_back(m - left);
      }
      std::sort(nx.begin(), nx.end());
      nx.erase(std::unique(nx.begin(), nx.end()), nx.end());
      sz.swap(nx);
      ++levels;
    }
  }
  const int64_t maxseg = (int64_t)1 << levels;
  uint64_t *key = nullptr, *skey = nullptr;
  int32_t *val = nullptr, *seg = nullptr, *sb = nullptr, *se = nullptr, *sb2 = nullptr, *se2 = nullptr;
  uint8_t* axis = nullptr;
  wn_status st = dalloc(&key, n, s);
  if (st == WN_OK) st = dalloc(&skey, n, s);
  if (st == WN_OK) st = dalloc(&val, n, s);
  if (st == WN_OK) st = dalloc(&seg, n, s);
  if (st == WN_OK) st = dalloc(&sb, maxseg, s);
  if (st == WN_OK) st = dalloc(&se, maxseg, s);
  if (st == WN_OK) st = dalloc(&sb2, maxseg, s);
  if (st == WN_OK) st = dalloc(&se2, maxseg, s);
  if (st == WN_OK) st = dalloc(&axis, maxseg, s);
  if (st == WN_OK) st = kd_levels(pts, n, levels, order, key, skey, val, seg, sb, se, sb2, se2, axis, s);
  for (void* p : {(void*)key, (void*)skey, (void*)val, (void*)seg, (void*)sb, (void*)se, (void*)sb2, (void*)se2,
                  (void*)axis})
    if (p) cudaFreeAsync(p, s);
  return st;
}

wn_status kd_levels(const float4* pts, int64_t n, int levels, int32_t* order, uint64_t* key, uint64_t* skey,
                    int32_t* val, int32_t* seg, int32_t* sb, int32_t* se, int32_t* sb2, int32_t* se2, uint8_t* axis,
                    cudaStream_t s) {
  const unsigned g = (unsigned)((n + 255) / 256);
  {
    ProfScope ps(WN_PROF_TREE, s, 0);
    kd_iota<<<g, 256, 0, s>>>(n, order, seg);
    const int32_t init[2] = {0, (int32_t)n};
    WN_CUDA(cudaMemcpyAsync(sb, &init[0], sizeof(int32_t), cudaMemcpyHostToDevice, s));
    WN_CUDA(cudaMemcpyAsync(se, &init[1], sizeof(int32_t), cudaMemcpyHostToDevice, s));
    for (int L = 0; L < levels; ++L) {
      const int nseg = 1 << L;
      kd_axes<<<(nseg + 127) / 128, 128, 0, s>>>(pts, order, sb, se, nseg, axis);
      kd_keys<<<g, 256, 0, s>>>(pts, order, seg, axis, n, key, val);
      WN_TRY(sort_pairs(key, val, n, kKdQBits + L, order, s, skey));
      WN_CUDA(cudaMemsetAsync(sb2, 0, 2 * (size_t)nseg * sizeof(int32_t), s));
      WN_CUDA(cudaMemsetAsync(se2, 0, 2 * (size_t)nseg * sizeof(int32_t), s));
      kd_split<<<g, 256, 0, s>>>(skey, n, sb, se, seg, sb2, se2);
      std::swap(sb, sb2);
      std::swap(se, se2);
      count_launches(3);
    }
    kd_local<<<(unsigned)(1u << levels), 1024, 0, s>>>(pts, order, sb, se);
    count_launches(2);
    WN_CUDA(cudaGetLastError());
  }
  return WN_OK;
}

// keys of the visitable-node list: each node's first sorted point (the moment pass then reads the
// prefix entries in point order)
__global__ void live_keys(int64_t m, const int32_t* __restrict__ list, const int32_t* __restrict__ pb,
                          uint64_t* __restrict__ k, int32_t* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int32_t node = list[i];
  k[i] = (uint64_t)pb[node];
  v[i] = node;
}

// ---- tile plan of the per-iteration moment builds (moments.cu: mom_tiles / mom_cross) ----
__global__ void k_node_keys(int64_t m, const int32_t* __restrict__ list, const int32_t* __restrict__ pb,
                            uint64_t* __restrict__ k, int32_t* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int32_t node = list ? list[i] : (int32_t)i;
  k[i] = (uint64_t)pb[node];
  v[i] = node;
}

// class of a listed node: 0 one point, 1 small (one tile), 2 large (one tile), 3 across tiles
__device__ __forceinline__ int node_class(int32_t b, int32_t e, int T) {
  if (e - b == 1) return 0;
  if (b / T != (e - 1) / T) return 3;
  return e - b < kMomWarpNode ? 1 : 2;
}

__global__ void k_class_flag(int64_t m, const int32_t* __restrict__ list, const int32_t* __restrict__ pb,
                             const int32_t* __restrict__ pe, int cls, int T, uint32_t* __restrict__ flag) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int32_t i = list[k];
  flag[k] = node_class(pb[i], pe[i], T) == cls;
}

// compaction of one class in list order; one-tile classes as descriptors (local point range, code, one-point
// child mask, threshold depth: what the tile build needs in one load)
__global__ void k_class_put(int64_t m, const int32_t* __restrict__ list, const uint32_t* __restrict__ flag,
                            const uint32_t* __restrict__ pos, const int32_t* __restrict__ pb,
                            const int32_t* __restrict__ pe, const int32_t* __restrict__ topo,
                            const int32_t* __restrict__ smask, const int32_t* __restrict__ tdepth, int T,
                            int4* __restrict__ desc, int32_t* __restrict__ ids) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m || !flag[k]) return;
  const int32_t i = list[k];
  if (ids) {
    ids[pos[k]] = i;
  } else {
    const int32_t b0 = (pb[i] / T) * T;
    desc[pos[k]] = make_int4(i, (pb[i] - b0) | ((pe[i] - b0) << 16), topo[i], smask[i] | (tdepth[i] << 16));
  }
}

__global__ void k_onept(int64_t m, const int32_t* __restrict__ list, const int32_t* __restrict__ pb,
                        const int32_t* __restrict__ pe, const int32_t* __restrict__ topo, int2* __restrict__ onept) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int32_t i = list[k];
  if (pe[i] - pb[i] == 1) onept[pb[i]] = make_int2(i, topo[i]);  // (a point's one-point node is its leaf: unique)
}

// tile k's descriptors start at the first whose first point is ≥ k·T (lists sorted by first point)
__global__ void k_tile_off(int64_t ntiles, const int4* __restrict__ desc, int64_t nd, const int32_t* __restrict__ pb,
                           int T, int32_t* __restrict__ off) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k > ntiles) return;
  const int64_t target = k * (int64_t)T;
  int64_t lo = 0, hi = nd;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)pb[desc[mid].x] < target) lo = mid + 1;
    else hi = mid;
  }
  off[k] = (int32_t)lo;
}

// endpoints of the cross-tile nodes: Σ from pb to the end of pb's tile, Σ from the start of (pe − 1)'s tile to pe
__global__ void k_ep_keys(int64_t nc, const int32_t* __restrict__ cross, const int32_t* __restrict__ pb,
                          const int32_t* __restrict__ pe, int T, uint64_t* __restrict__ key,
                          int32_t* __restrict__ slot) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const int64_t b = pb[cross[c]], e = pe[cross[c]];
  const int64_t ta = b / T, tb = (e - 1) / T;
  key[2 * c] = (uint64_t)(ta * (T + 1) + (b - ta * T));
  key[2 * c + 1] = (uint64_t)(tb * (T + 1) + (e - tb * T));
  slot[2 * c] = (int32_t)(2 * c);
  slot[2 * c + 1] = (int32_t)(2 * c + 1);
}

__global__ void k_tile_eoff(int64_t ntiles, const uint64_t* __restrict__ key, int64_t ne, int T,
                            int32_t* __restrict__ off) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k > ntiles) return;
  const uint64_t target = (uint64_t)k * (T + 1);
  int64_t lo = 0, hi = ne;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  off[k] = (int32_t)lo;
}

static int key_bits(int64_t maxval) {
  int bits = 1;
  while (bits < 62 && ((int64_t)1 << bits) <= maxval) ++bits;
  return bits;
}

wn_status plan_moment_tiles(wn_tree_s* t, int which, cudaStream_t s) {
  MomPlan& P = t->mplan[which];
  if (P.ready) return WN_OK;
  TempSet tmp(s);
  if (t->mom_tile <= 0) return set_error(WN_ERR_ARG, "internal: moment tile size not chosen");
  const int T = t->mom_tile;
  const int64_t n = t->n, ntiles = (n + T - 1) / T;
  // the node list in ascending first point: the visitable nodes (already sorted) or all nodes (sorted here)
  const int32_t* list = t->mom_live;
  int64_t m = t->mom_nlive;
  if (which == 1) {
    m = t->nn;
    uint64_t* k = nullptr;
    int32_t *v = nullptr, *sorted = nullptr;
    WN_TRY(tmp.alloc(&k, m));
    WN_TRY(tmp.alloc(&v, m));
    WN_TRY(tmp.alloc(&sorted, m));
    k_node_keys<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, nullptr, t->pb, k, v);
    count_launches(1);
    WN_TRY(sort_pairs(k, v, m, key_bits(n), sorted, s));
    list = sorted;
  }
  uint32_t *flag = nullptr, *pos = nullptr;
  WN_TRY(tmp.alloc(&flag, m + 1));
  WN_TRY(tmp.alloc(&pos, m + 1));
  const unsigned g = (unsigned)((m + 255) / 256);
  int64_t cnt[4] = {0, 0, 0, 0};
  for (int cls = 1; cls <= 3; ++cls) {
    k_class_flag<<<g, 256, 0, s>>>(m, list, t->pb, t->pe, cls, T, flag);
    WN_TRY(scan_excl(flag, pos, m, pos + m, s));
    uint32_t c = 0;
    WN_CUDA(cudaMemcpyAsync(&c, pos + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    cnt[cls] = c;
    int4* desc = nullptr;
    int32_t* ids = nullptr;
    if (cls == 1) {
      WN_TRY(dalloc(&P.small, std::max<int64_t>(c, 1), s));
      desc = P.small;
    } else if (cls == 2) {
      WN_TRY(dalloc(&P.large, std::max<int64_t>(c, 1), s));
      desc = P.large;
    } else {
      WN_TRY(dalloc(&P.cross, std::max<int64_t>(c, 1), s));
      ids = P.cross;
    }
    k_class_put<<<g, 256, 0, s>>>(m, list, flag, pos, t->pb, t->pe, t->topo, t->smask, t->tdepth, T, desc, ids);
    count_launches(5);
  }
  P.nsmall = cnt[1];
  P.nlarge = cnt[2];
  P.ncross = cnt[3];
  WN_TRY(dalloc(&P.onept, n, s));
  WN_CUDA(cudaMemsetAsync(P.onept, 0xff, n * sizeof(int2), s));
  k_onept<<<g, 256, 0, s>>>(m, list, t->pb, t->pe, t->topo, P.onept);
  WN_TRY(dalloc(&P.tile_soff, ntiles + 1, s));
  WN_TRY(dalloc(&P.tile_loff, ntiles + 1, s));
  WN_TRY(dalloc(&P.tile_eoff, ntiles + 1, s));
  const unsigned gt = (unsigned)((ntiles + 256) / 256);
  k_tile_off<<<gt, 256, 0, s>>>(ntiles, P.small, P.nsmall, t->pb, T, P.tile_soff);
  k_tile_off<<<gt, 256, 0, s>>>(ntiles, P.large, P.nlarge, t->pb, T, P.tile_loff);
  count_launches(3);
  const int64_t ne = 2 * P.ncross;
  WN_TRY(dalloc(&P.ep_key, std::max<int64_t>(ne, 1), s));
  WN_TRY(dalloc(&P.ep_slot, std::max<int64_t>(ne, 1), s));
  WN_TRY(dalloc(&P.epval, (size_t)kMomNC * std::max<int64_t>(ne, 1), s));
  if (ne > 0) {
    uint64_t* k = nullptr;
    int32_t* v = nullptr;
    WN_TRY(tmp.alloc(&k, ne));
    WN_TRY(tmp.alloc(&v, ne));
    k_ep_keys<<<(unsigned)((P.ncross + 255) / 256), 256, 0, s>>>(P.ncross, P.cross, t->pb, t->pe, T, k, v);
    count_launches(1);
    WN_TRY(sort_pairs(k, v, ne, key_bits(ntiles * (int64_t)(T + 1)), P.ep_slot, s, P.ep_key));
  }
  k_tile_eoff<<<gt, 256, 0, s>>>(ntiles, P.ep_key, ne, T, P.tile_eoff);
  count_launches(1);
  if (!t->mom_ttot) WN_TRY(dalloc(&t->mom_ttot, (size_t)kMomNC * ntiles, s));
  WN_CUDA(cudaGetLastError());
  P.ready = true;
  return WN_OK;
}

wn_status build_tree(const float* pts, int64_t n, int D, cudaStream_t s, wn_tree_s* t) {
  t->n = n;
  t->D = D;
  TempSet tmp(s);  // temporaries: freed on every return path
  // --- bbox + transform (a1) ---
  int nb = (int)std::min<int64_t>((n + 255) / 256, 1184);
  float* part = nullptr;
  int* bad = nullptr;
  BBox* bb = nullptr;
  WN_TRY(tmp.alloc(&part, 6 * (size_t)nb));
  WN_TRY(tmp.alloc(&bad, 1));
  WN_TRY(tmp.alloc(&bb, 1));
  WN_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  {
    ProfScope ps(WN_PROF_TREE, s, 2);
    bbox_partial<<<nb, 256, 0, s>>>(pts, n, part, bad);
    bbox_final<<<1, 1024, 0, s>>>(part, nb, bad, bb);
  }
  BBox hb;
  WN_CUDA(cudaMemcpyAsync(&hb, bb, sizeof(BBox), cudaMemcpyDeviceToHost, s));
  WN_CUDA(cudaStreamSynchronize(s));
  if (hb.nonfinite) return set_error(WN_ERR_NONFINITE, "non-finite point coordinate");
  if (!(hb.xf[3] > 0.0)) return set_error(WN_ERR_DEGENERATE, "all points coincide (zero extent)");
  for (int a = 0; a < 4; ++a) t->xf[a] = hb.xf[a];

  // --- normalize, keys, sort (a1) ---
  float4* xn = nullptr;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  int32_t *v0 = nullptr, *v1 = nullptr;
  WN_TRY(tmp.alloc(&xn, n));
  WN_TRY(tmp.alloc(&k0, n));
  WN_TRY(tmp.alloc(&k1, n));
  WN_TRY(tmp.alloc(&v0, n));
  WN_TRY(tmp.alloc(&v1, n));
  int ntiles = (int)((n + kSortTile - 1) / kSortTile);
  uint32_t* hist = nullptr;
  WN_TRY(tmp.alloc(&hist, (size_t)256 * ntiles));
  int passes = (3 * D + 7) / 8;
  {
    ProfScope ps(WN_PROF_TREE, s, 1 + 5 * passes + 1);
    normalize_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pts, n, bb, D, xn, k0, v0);
    for (int p = 0; p < passes; ++p) {
      radix_hist<<<ntiles, kSortThreads, 0, s>>>(k0, n, 8 * p, ntiles, hist);
      WN_TRY(scan_excl(hist, hist, (int64_t)256 * ntiles, nullptr, s));
      radix_scatter<<<ntiles, kSortThreads, 0, s>>>(k0, v0, k1, v1, n, 8 * p, ntiles, hist);
      std::swap(k0, k1);
      std::swap(v0, v1);
    }
    WN_TRY(dalloc(&t->pts, n, s));
    WN_TRY(dalloc(&t->perm, n, s));
    gather_sorted<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(xn, v0, n, t->pts, t->perm);
  }
  t->keys = k0;
  tmp.keep(k0);  // owned by the tree from here
  // --- query schedule: the sorted points in Hilbert order (warps get spatially compact query sets;
  //     a Z-order jump between diagonal octants no longer splits a warp's 32 queries) ---
  if (!getenv("WN_EXP_NOHILBERT")) {
    WN_TRY(dalloc(&t->qorder, n, s));
    WN_TRY(hilbert_schedule(t->pts, n, t->qorder, s));
  }
  for (void* p : {(void*)k1, (void*)v0, (void*)v1, (void*)xn, (void*)hist, (void*)part, (void*)bad, (void*)bb})
    tmp.release(p);

  // --- node counts per level (a2) ---
  int etiles = (int)((n + kEmitThreads - 1) / kEmitThreads);
  int64_t m = (int64_t)(D + 1) * etiles;
  uint32_t *cnt = nullptr, *offs = nullptr;
  WN_TRY(tmp.alloc(&cnt, m + 1));
  WN_TRY(tmp.alloc(&offs, m + 1));
  {
    ProfScope ps(WN_PROF_TREE, s, 4);
    level_counts<<<etiles, kEmitThreads, 0, s>>>(t->keys, n, D, etiles, cnt);
    WN_TRY(scan_excl(cnt, offs, m, offs + m, s));
  }
  std::vector<uint32_t> hoffs(m + 1);
  WN_CUDA(cudaMemcpyAsync(hoffs.data(), offs, (m + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  WN_CUDA(cudaStreamSynchronize(s));
  t->nn = hoffs[m];
  if (t->nn + 1 > ((int64_t)1 << 26)) {  // the traversal addresses 64-byte records with 32-bit byte offsets
    return set_error(WN_ERR_ARG, "octree with more than 2^26 - 1 nodes (deep chains of close points)");
  }
  t->level_off.assign(D + 2, t->nn);
  int used = 0;
  for (int l = 0; l <= D; ++l) {
    t->level_off[l] = hoffs[(int64_t)l * etiles];
    if (t->level_off[l] < t->nn) used = l;
  }
  t->depth_used = used;
  t->level_off.resize(used + 2);
  t->level_off[used + 1] = t->nn;
  int64_t nn = t->nn;

  // --- emission ---
  WN_TRY(dalloc(&t->depth, nn, s));
  WN_TRY(dalloc(&t->pb, nn, s));
  WN_TRY(dalloc(&t->pe, nn, s));
  WN_TRY(dalloc(&t->cb, nn, s));
  WN_TRY(dalloc(&t->cc, nn, s));
  WN_TRY(dalloc(&t->parent, nn, s));
  WN_TRY(dalloc(&t->topo, nn, s));
  WN_TRY(dalloc(&t->smask, nn, s));
  WN_TRY(dalloc(&t->tdepth, nn, s));
  WN_TRY(dalloc(&t->centroid, nn, s));
  WN_TRY(dalloc(&t->leaf_of, n, s));
  WN_TRY(dalloc(&t->sums, 8 * (size_t)nn, s));
  for (int k = 0; k < 2; ++k) {
    WN_TRY(dalloc(&t->set[k].rec, (size_t)kRec * (nn + 1), s));  // +1: the traversal prefetches one past a group
    WN_CUDA(cudaMemsetAsync(t->set[k].rec, 0, sizeof(float4) * kRec * (nn + 1), s));
  }
  int64_t* loff = nullptr;
  WN_TRY(tmp.alloc(&loff, t->level_off.size()));
  WN_CUDA(cudaMemcpyAsync(loff, t->level_off.data(), t->level_off.size() * sizeof(int64_t),
                          cudaMemcpyHostToDevice, s));
  {
    unsigned g = (unsigned)((nn + 255) / 256);
    ProfScope ps(WN_PROF_TREE, s, 4 + used + 1);
    emit_nodes<<<etiles, kEmitThreads, 0, s>>>(t->keys, n, D, etiles, offs, t->depth, t->pb, t->cb, t->cc,
                                                t->parent);
    find_parents<<<g, 256, 0, s>>>(nn, t->depth, t->pb, loff, t->parent);
    child_counts<<<g, 256, 0, s>>>(nn, t->depth, t->parent, loff, t->cb, t->cc);
    for (int l = 0; l <= used; ++l) {
      int64_t i0 = t->level_off[l], i1 = t->level_off[l + 1];
      level_pe<<<(unsigned)((i1 - i0 + 255) / 256), 256, 0, s>>>(i0, i1, n, t->parent, t->pb, t->pe);
    }
    topo_codes<<<g, 256, 0, s>>>(nn, t->cb, t->cc, t->pb, t->pe, t->depth, t->topo, t->smask, t->tdepth);
  }
  {  // the visited nodes, compacted in BFS order (per-iteration moment builds skip the rest)
    uint32_t *vis = nullptr, *pos = nullptr;
    WN_TRY(tmp.alloc(&vis, nn + 1));
    WN_TRY(tmp.alloc(&pos, nn + 1));
    WN_CUDA(cudaMemsetAsync(vis, 0, (nn + 1) * sizeof(uint32_t), s));
    const unsigned g = (unsigned)((nn + 255) / 256);
    mark_visited<<<g, 256, 0, s>>>(nn, t->topo, vis);
    WN_TRY(scan_excl(vis, pos, nn, pos + nn, s));
    uint32_t nlive = 0;
    WN_CUDA(cudaMemcpyAsync(&nlive, pos + nn, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    t->mom_nlive = nlive;
    WN_TRY(dalloc(&t->mom_live, std::max<int64_t>(nlive, 1), s));
    compact_visited<<<g, 256, 0, s>>>(nn, vis, pos, t->mom_live);
    tmp.release(vis);
    tmp.release(pos);
    count_launches(5);
    if (nlive > 1) {  // in first-point order (the moment builds' tile plan relies on it)
      uint64_t* k = nullptr;
      int32_t* v = nullptr;
      WN_TRY(tmp.alloc(&k, nlive));
      WN_TRY(tmp.alloc(&v, nlive));
      live_keys<<<(unsigned)((nlive + 255) / 256), 256, 0, s>>>(nlive, t->mom_live, t->pb, k, v);
      count_launches(1);
      int bits = 1;
      while (bits < 62 && ((int64_t)1 << bits) <= n) ++bits;
      WN_TRY(sort_pairs(k, v, nlive, bits, t->mom_live, s));
      tmp.release(k);
      tmp.release(v);
    }
  }
  tmp.release(loff);
  tmp.release(cnt);
  tmp.release(offs);
  WN_CUDA(cudaGetLastError());

  // --- fixed node data: unweighted centroids (unit weights) ---
  WN_TRY(plan_moments(t, s));
  MomentArgs ma;
  ma.kind = ATTR_UNIT;
  ma.out = t->set[1];
  ma.centroid_out = t->centroid;
  ma.leaf_of_out = t->leaf_of;
  WN_TRY(build_moments(t, ma, s));
  // the per-iteration builds rewrite only V of one-point nodes: their R = (x_j, −1) and L are fixed here
  WN_CUDA(cudaMemcpyAsync(t->set[0].rec, t->set[1].rec, sizeof(float4) * kRec * (nn + 1), cudaMemcpyDeviceToDevice, s));
  return WN_OK;
}

void free_tree(wn_tree_s* t) {
  void* ptrs[] = {t->pts, t->perm, t->keys, t->qorder, t->depth, t->pb, t->pe, t->cb, t->cc, t->parent, t->leaf_of,
                  t->topo, t->smask, t->tdepth, t->mom_live, t->mom_loff, t->mom_ttot, t->centroid, t->sums, t->set[0].rec, t->set[1].rec, t->set[0].ext,
                  t->it.mu, t->it.mup, t->it.r, t->it.s, t->it.part, t->it.dstats, t->it.dcounts, t->it.dstamp, t->it.alpha, t->it.tmp,
                  t->qbuf, t->qbuf_order, t->tvb, t->tu};
  // the last call's work (on whatever stream it was queued) must finish before the memory returns to
  // the pool; then stream-ordered frees, no device-wide synchronization
  if (t->done_ev) {
    cudaEventSynchronize(t->done_ev);
    cudaEventDestroy(t->done_ev);
    t->done_ev = nullptr;
  }
  if (t->graph_exec) cudaGraphExecDestroy(t->graph_exec);
  t->graph_exec = nullptr;
  if (t->cap_stream) {
    cudaStreamSynchronize(t->cap_stream);
    cudaStreamDestroy(t->cap_stream);
    t->cap_stream = nullptr;
  }
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, 0);
  fmm_plan_free(t->fmm);
  for (MomPlan& P : t->mplan)
    for (void* p : {(void*)P.small, (void*)P.large, (void*)P.tile_soff, (void*)P.tile_loff, (void*)P.onept,
                    (void*)P.cross, (void*)P.ep_key, (void*)P.ep_slot, (void*)P.tile_eoff, (void*)P.epval})
      if (p) cudaFreeAsync(p, 0);

}

}  // namespace wn
