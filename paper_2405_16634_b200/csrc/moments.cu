// moments.cu — per-application representatives.
//
// PAPER.md:L371-L378 (§4.5, Eqs node-rep-loc / node-rep-vec): for attribute ν,
//     x_{B,ν} = Σ_{i∈B} |ν_i| x_i / Σ_{j∈B} |ν_j| ,   ν_B = Σ_{i∈B} ν_i .
// Readings: Σ|ν| = 0 ⇒ the node's unweighted centroid; a one-point node's rep is the
// point itself; |ν| is the Euclidean norm (vector) or |s| (scalar).
//
// B200 design: fp64 node sums (W, P, V) are built bottom-up: a leaf sums its points, an internal node
// sums its children IN CHILD ORDER (deterministic; child sums are loaded 4 at a time so their
// latencies overlap).  No fences, no atomics; kernel boundaries order the levels:
//   1. one launch for every leaf at or below the cut level (the first level with ≥ 1024 nodes);
//   2. one launch per pair of levels, deepest first, for the internal nodes at or below the cut (the
//      upper level of a pair forms its children's sums from the grandchildren in the same order);
//   3. one single-block launch for the few levels above the cut (__syncthreads() between levels).
// Each node writes its 64-byte traversal record (rep hi + lo, threshold, ν_B, topology code).
// Traffic O(N + Nn): ≈ 32 B/point + 64 B fp64 sums + 64 B record per node.
#include <cuda_runtime.h>

#include <algorithm>

#include "wn_internal.cuh"

namespace wn {
namespace {

constexpr int kMomThreads = 256;
constexpr int kTopThreads = 512;

struct Sums {
  double W, P[3], V[3];
};

struct TreeView {
  const float4* pts;
  const int32_t *pb, *pe, *cb, *cc, *depth, *topo, *smask;  // depth: the threshold depth (tdepth)
  double* sums;
  const float4* centroid;
};

__device__ __forceinline__ float thr_of(float theta, int depth) {
  // (c · edge)², edge = 2^{1−depth} of the root cube [−1,1]^3, in fp32 (exact power-of-two scaling)
  float cw = theta * __int_as_float((127 + 1 - depth) << 23);
  return __fmul_rn(cw, cw);
}

template <int KIND>
__device__ __forceinline__ void write_record(int64_t i, const Sums& S, int cnt, float4 p0, int depth, int topo,
                                             int smask, float theta, const float4* __restrict__ centroid,
                                             const MomentArgs& m) {
  float4 R, L = make_float4(0.f, 0.f, 0.f, 0.f);
  if (cnt == 1) {
    R = make_float4(p0.x, p0.y, p0.z, -1.0f);
  } else {
    float rx, ry, rz;
    if (S.W > 0.0) {
      const double x = S.P[0] / S.W, y = S.P[1] / S.W, z = S.P[2] / S.W;
      rx = (float)x;
      ry = (float)y;
      rz = (float)z;
      L = make_float4((float)(x - (double)rx), (float)(y - (double)ry), (float)(z - (double)rz), 0.f);
    } else {
      const float4 c = centroid[i];
      rx = c.x; ry = c.y; rz = c.z;
    }
    R = make_float4(rx, ry, rz, thr_of(theta, depth));
  }
  float4* rec = m.out.rec + kRec * i;
  rec[0] = R;
  if (KIND == ATTR_SCALAR)
    rec[1] = make_float4((float)S.V[0], 0.f, 0.f, __int_as_float(topo));
  else
    rec[1] = make_float4((float)S.V[0], (float)S.V[1], (float)S.V[2], __int_as_float(topo));
  L.w = __int_as_float(smask);  // which children are one-point leaves
  rec[2] = L;
  if (KIND == ATTR_UNIT) m.centroid_out[i] = make_float4(R.x, R.y, R.z, 0.f);
}

// one node per thread: a leaf sums its points, an internal node its children's fp64 sums in child order;
// the children's sums are loaded 4 at a time so their L2 latencies overlap
template <int KIND, bool DEEP = false>
__device__ __forceinline__ void process_node(int64_t i, int depth, const TreeView& tv, const MomentArgs& m,
                                             float alpha) {
  Sums S = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  const int nc = tv.cc[i];
  const int j0 = tv.pb[i], j1 = tv.pe[i];
  if (nc == 0) {
    for (int j = j0; j < j1; ++j) {
      const float4 x = tv.pts[j];
      double a, v0 = 0, v1 = 0, v2 = 0;
      if (KIND == ATTR_VEC) {
        float4 v = m.vec[j];
        if (m.axpy_r) {  // μ' = μ + α r (Alg. 2 line 3), fused: written once, read by the G traversal
          const float4 r = m.axpy_r[j];
          v = make_float4(fmaf(alpha, r.x, v.x), fmaf(alpha, r.y, v.y), fmaf(alpha, r.z, v.z), 0.f);
          m.axpy_out[j] = v;
        }
        v0 = v.x; v1 = v.y; v2 = v.z;
        if (m.a_sorted) {
          const double f = m.a_sorted[j];
          v0 *= f; v1 *= f; v2 *= f;
        }
        a = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
      } else if (KIND == ATTR_SCALAR) {
        v0 = m.scal[j];
        if (m.a_sorted) v0 *= (double)m.a_sorted[j];
        a = fabs(v0);
      } else {
        a = 1.0;
        v0 = 1.0;
        m.leaf_of_out[j] = (int32_t)i;
      }
      S.W += a;
      S.P[0] += a * (double)x.x;
      S.P[1] += a * (double)x.y;
      S.P[2] += a * (double)x.z;
      S.V[0] += v0;
      S.V[1] += v1;
      S.V[2] += v2;
    }
  } else if (DEEP) {
    // the children's sums are formed here from the grandchildren (same operations, same order as the
    // child's own thread), so two levels are finished per launch
    const int c0 = tv.cb[i];
    for (int c = c0; c < c0 + nc; ++c) {
      const int gn = tv.cc[c];
      Sums C = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
      const int g0 = gn ? tv.cb[c] : c;
      for (int g = g0; g < g0 + (gn ? gn : 1); ++g) {  // a leaf child contributes its stored sums
        const double2* q = reinterpret_cast<const double2*>(tv.sums + 8 * (int64_t)g);
        const double2 a = q[0], b = q[1], d = q[2], e = q[3];
        if (gn) {
          C.W += a.x; C.P[0] += a.y; C.P[1] += b.x; C.P[2] += b.y; C.V[0] += d.x; C.V[1] += d.y; C.V[2] += e.x;
        } else {
          C.W = a.x; C.P[0] = a.y; C.P[1] = b.x; C.P[2] = b.y; C.V[0] = d.x; C.V[1] = d.y; C.V[2] = e.x;
        }
      }
      S.W += C.W;
      for (int k = 0; k < 3; ++k) {
        S.P[k] += C.P[k];
        S.V[k] += C.V[k];
      }
    }
  } else {
    const double2* c = reinterpret_cast<const double2*>(tv.sums + 8 * (int64_t)tv.cb[i]);
#ifndef WN_EXP_MOM_BATCH
#define WN_EXP_MOM_BATCH 2
#endif
    constexpr int B = WN_EXP_MOM_BATCH;
    for (int k0 = 0; k0 < nc; k0 += B) {
      double2 q[B][4];
#pragma unroll
      for (int k = 0; k < B; ++k)
        if (k0 + k < nc)
#pragma unroll
          for (int u = 0; u < 4; ++u) q[k][u] = c[4 * (k0 + k) + u];
#pragma unroll
      for (int k = 0; k < B; ++k)
        if (k0 + k < nc) {
          S.W += q[k][0].x;
          S.P[0] += q[k][0].y;
          S.P[1] += q[k][1].x;
          S.P[2] += q[k][1].y;
          S.V[0] += q[k][2].x;
          S.V[1] += q[k][2].y;
          S.V[2] += q[k][3].x;
        }
    }
  }
  double2* o = reinterpret_cast<double2*>(tv.sums + 8 * i);
  o[0] = make_double2(S.W, S.P[0]);
  o[1] = make_double2(S.P[1], S.P[2]);
  o[2] = make_double2(S.V[0], S.V[1]);
  o[3] = make_double2(S.V[2], 0.0);
  const float4 p0 = (j1 - j0 == 1) ? tv.pts[j0] : make_float4(0.f, 0.f, 0.f, 0.f);
  write_record<KIND>(i, S, j1 - j0, p0, tv.depth[i], tv.topo[i], tv.smask[i], m.theta, tv.centroid, m);
}

template <int KIND>
__global__ void __launch_bounds__(kTopThreads) moments_top(TreeView tv, MomentArgs m, const int64_t* __restrict__ loff,
                                                           int cut) {
  const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
  for (int l = cut - 1; l >= 0; --l) {
    const int64_t i0 = loff[l], i1 = loff[l + 1];
    for (int64_t i = i0 + threadIdx.x; i < i1; i += kTopThreads) process_node<KIND>(i, l, tv, m, alpha);
    __syncthreads();
  }
}

// leaves (MODE 0: every leaf in [i0, i1), any level) or internal nodes of one level (MODE 1)
// MODE 0: every leaf in [i0, i1) (any level).  MODE 1: the internal nodes of levels `level` ([imid, i1))
// and `level − 1` ([i0, imid)) — the latter from their grandchildren.
template <int KIND, int MODE>
#ifndef WN_EXP_MOM_LB
#define WN_EXP_MOM_LB 4
#endif
__global__ void __launch_bounds__(kMomThreads, WN_EXP_MOM_LB) moments_range(TreeView tv, MomentArgs m, int64_t i0, int64_t imid,
                                                             int64_t i1, int level) {
  const int64_t i = i0 + blockIdx.x * (int64_t)kMomThreads + threadIdx.x;
  if (i >= i1) return;
  const bool leaf = tv.cc[i] == 0;
  if (leaf != (MODE == 0)) return;
  const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
  if (MODE == 0) process_node<KIND>(i, tv.depth[i], tv, m, alpha);
  else if (i >= imid) process_node<KIND>(i, level, tv, m, alpha);
  else process_node<KIND, true>(i, level - 1, tv, m, alpha);
}

// ---------------- tile builds (per-iteration attributes: ATTR_VEC, ATTR_SCALAR) ----------------
// Every octree node B covers a contiguous range [pb, pe) of the Morton-sorted points.  The sorted points
// are cut into tiles of wn_tree_s::mom_tile points (choose_mom_tile; tree_build.cu:plan_moment_tiles
// lists, per tile, the nodes whose points lie in it):
//   mom_tiles  (one block per tile) computes every point's terms (|ν|, |ν|x, ν, …) once into shared memory
//              (coalesced loads; μ' = μ + α r written here; a one-point node's V = ν_j written here), then
//              sums each node's range directly — one thread per node below kMomWarpNode points, one warp
//              per larger node (lane-strided, then a fixed butterfly) — and writes its record; the same
//              warps form the tile's total and, for the nodes across tiles, the partial sums at their ends;
//   mom_cross  (one warp per node across tiles) adds  the partial sum at pb + the totals of the tiles in
//              between (lane-strided, fixed butterfly) + the partial sum at pe.
// fp64 direct sums in a fixed order: the error of a node's sum is relative to its own terms (as the
// oracle's direct sums), Σ|ν| = 0 exactly iff every ν_j = 0 (a sum of non-negative terms), and the result
// is bit-deterministic.  One-point nodes take their point's own values (rep = the point).
// First-order far field (ORD = 1): the terms also carry sym(ν_j x_jᵀ) (vector ν, 6) or
// s_j x_j (scalar, 3), and each node stores its first moment about the representative,
// sym M = sym(Σ ν_j x_jᵀ) − sym(ν_B x_Bᵀ) or D = Σ s_j x_j − s_B x_B, in NodeSet::ext.  DESIGN.md §Moments.

// components of a point's terms: 0: |ν|, 1-3: |ν|x, 4..: ν (3 or 1), then the first-order sums (6 or 3)
template <int KIND, int ORD>
struct Lay {
  static constexpr int NV = KIND == ATTR_VEC ? 3 : 1;
  static constexpr int NX = ORD == 1 ? (KIND == ATTR_VEC ? 6 : 3) : 0;
  static constexpr int NC = 4 + NV + NX;
};
static_assert(Lay<ATTR_VEC, 1>::NC <= kMomNC, "tile totals / endpoint sums sized for the widest layout");

// per-point terms of attribute v (vector: ν, scalar: v.x; the a-factor f applied when `scaled`)
template <int KIND, int ORD>
__device__ __forceinline__ void point_terms(float4 x, float4 v, double f, bool scaled, double* o) {
  double a, v0, v1 = 0.0, v2 = 0.0;
  if (KIND == ATTR_VEC) {
    v0 = v.x; v1 = v.y; v2 = v.z;
    if (scaled) {
      v0 *= f; v1 *= f; v2 *= f;
    }
    a = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
  } else {
    v0 = v.x;
    if (scaled) v0 *= f;
    a = fabs(v0);
  }
  const double px = x.x, py = x.y, pz = x.z;
  o[0] = a;
  o[1] = a * px;
  o[2] = a * py;
  o[3] = a * pz;
  o[4] = v0;
  if (KIND == ATTR_VEC) {
    o[5] = v1;
    o[6] = v2;
  }
  if (ORD == 1) {
    constexpr int X = Lay<KIND, ORD>::NC - Lay<KIND, ORD>::NX;
    if (KIND == ATTR_VEC) {
      o[X + 0] = v0 * px;
      o[X + 1] = v1 * py;
      o[X + 2] = v2 * pz;
      o[X + 3] = 0.5 * (v0 * py + v1 * px);
      o[X + 4] = 0.5 * (v0 * pz + v2 * px);
      o[X + 5] = 0.5 * (v1 * pz + v2 * py);
    } else {
      o[X + 0] = v0 * px;
      o[X + 1] = v0 * py;
      o[X + 2] = v0 * pz;
    }
  }
}

// record of a node with ≥ 2 points from its sums d (Σ|ν| = d[0] = 0 exactly iff every ν_j = 0)
template <int KIND, int ORD>
__device__ __forceinline__ void sums_record(int64_t i, int npts, const double* d, const TreeView& tv,
                                            const MomentArgs& m, int tdepth, int topo, int smask) {
  using Ly = Lay<KIND, ORD>;
  Sums S;
  S.W = d[0];
  S.P[0] = d[1]; S.P[1] = d[2]; S.P[2] = d[3];
  S.V[0] = d[4];
  S.V[1] = KIND == ATTR_VEC ? d[5] : 0.0;
  S.V[2] = KIND == ATTR_VEC ? d[6] : 0.0;
  if (m.write_W) tv.sums[8 * i] = S.W;
  write_record<KIND>(i, S, npts, make_float4(0.f, 0.f, 0.f, 0.f), tdepth, topo, smask, m.theta, tv.centroid, m);
  if (ORD == 1) {  // first moment about the fp64 representative (0 for Σ|ν| = 0)
    constexpr int X = Ly::NC - Ly::NX;
    float4 e0 = make_float4(0.f, 0.f, 0.f, 0.f), e1 = e0;
    if (S.W > 0.0) {
      const double Xr = S.P[0] / S.W, Yr = S.P[1] / S.W, Zr = S.P[2] / S.W;
      if (KIND == ATTR_VEC) {
        const double mxx = d[X] - S.V[0] * Xr, myy = d[X + 1] - S.V[1] * Yr, mzz = d[X + 2] - S.V[2] * Zr;
        const double mxy = d[X + 3] - 0.5 * (S.V[0] * Yr + S.V[1] * Xr);
        const double mxz = d[X + 4] - 0.5 * (S.V[0] * Zr + S.V[2] * Xr);
        const double myz = d[X + 5] - 0.5 * (S.V[1] * Zr + S.V[2] * Yr);
        e0 = make_float4((float)mxx, (float)myy, (float)mzz, (float)(mxx + myy + mzz));
        e1 = make_float4((float)mxy, (float)mxz, (float)myz, 0.f);
      } else {
        e0 = make_float4((float)(d[X] - S.V[0] * Xr), (float)(d[X + 1] - S.V[0] * Yr), (float)(d[X + 2] - S.V[0] * Zr),
                         0.f);
      }
    }
    m.out.ext[2 * i] = e0;
    m.out.ext[2 * i + 1] = e1;
  }
}

struct TilePlanView {
  const int4 *small, *large;
  const int32_t *tile_soff, *tile_loff, *cross, *ep_slot, *tile_eoff;
  const int2* onept;
  const uint64_t* ep_key;
  double* epval;  // 2·ncross × kMomNC
  double* ttot;   // ntiles × kMomNC
  int64_t ncross;
  int tile;       // points per tile (wn_tree_s::mom_tile)
};

constexpr int kTileThreads = 256, kTileWarps = kTileThreads / 32;

// warp sum of NC planes over [l0, l1): lanes stride, then a fixed xor butterfly (every lane gets the same bits)
template <int NC>
__device__ __forceinline__ void warp_range_sum(const double* __restrict__ sm, int T, int l0, int l1, int lane,
                                               double* d) {
#pragma unroll
  for (int c = 0; c < NC; ++c) d[c] = 0.0;
  for (int l = l0 + lane; l < l1; l += 32)
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] += sm[c * T + l];
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] += __shfl_xor_sync(0xffffffffu, d[c], o);
}

// d[k] (registers are not indexable at run time: a select chain)
template <int NC>
__device__ __forceinline__ double pick(const double* d, int k) {
  double r = d[0];
#pragma unroll
  for (int c = 1; c < NC; ++c)
    if (k == c) r = d[c];
  return r;
}

template <int KIND, int ORD>
__global__ void __launch_bounds__(kTileThreads) mom_tiles(TreeView tv, MomentArgs m, int64_t n, TilePlanView P) {
  constexpr int NC = Lay<KIND, ORD>::NC;
  extern __shared__ double sm[];  // NC planes of P.tile per-point terms
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
  const bool axpy = KIND == ATTR_VEC && m.axpy_r;
  const bool scaled = m.a_sorted != nullptr;
  const int T = P.tile;
  const int64_t tile = blockIdx.x, base = tile * (int64_t)T;
  const int nv = (int)(n - base < T ? n - base : T);
  for (int jl = threadIdx.x; jl < nv; jl += kTileThreads) {  // coalesced
    const int64_t j = base + jl;
    float4 v = KIND == ATTR_VEC ? m.vec[j] : make_float4(m.scal[j], 0.f, 0.f, 0.f);
    if (axpy) {  // μ' = μ + α r (Alg. 2 line 3), written once here, read by the G traversal
      const float4 r = m.axpy_r[j];
      v = make_float4(fmaf(alpha, r.x, v.x), fmaf(alpha, r.y, v.y), fmaf(alpha, r.z, v.z), 0.f);
      m.axpy_out[j] = v;
    }
    const double f = scaled ? (double)m.a_sorted[j] : 1.0;
    double o[NC];
    point_terms<KIND, ORD>(tv.pts[j], v, f, scaled, o);
#pragma unroll
    for (int c = 0; c < NC; ++c) sm[c * T + jl] = o[c];
    const int2 op = P.onept[j];
    if (op.x >= 0) {  // one-point node: R = (x_j, −1), L, ext (= 0) fixed per tree; V = ν_j, the leaf term's ν
      if (m.write_W) tv.sums[8 * (int64_t)op.x] = o[0];
      const float4 V = KIND == ATTR_VEC ? make_float4((float)o[4], (float)o[5], (float)o[6], __int_as_float(op.y))
                                        : make_float4((float)o[4], 0.f, 0.f, __int_as_float(op.y));
      m.out.rec[kRec * (int64_t)op.x + 1] = V;
    }
  }
  __syncthreads();
  // small nodes: one thread each, points in order
  for (int x = P.tile_soff[tile] + threadIdx.x; x < P.tile_soff[tile + 1]; x += kTileThreads) {
    const int4 d4 = P.small[x];
    const int l0 = d4.y & 0xffff, l1 = d4.y >> 16;
    WN_DCHECK(l0 + 1 < l1 && l1 <= nv, "moment node range");
    double d[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] = sm[c * T + l0];
    for (int l = l0 + 1; l < l1; ++l)
#pragma unroll
      for (int c = 0; c < NC; ++c) d[c] += sm[c * T + l];
    sums_record<KIND, ORD>(d4.x, l1 - l0, d, tv, m, d4.w >> 16, d4.z, d4.w & 0xffff);
  }
  // warp items: the large nodes, the endpoint sums, the tile total
  const int L0 = P.tile_loff[tile], nl = P.tile_loff[tile + 1] - L0;
  const int E0 = P.tile_eoff[tile], ne = P.tile_eoff[tile + 1] - E0;
  for (int w = warp; w < nl + ne + 1; w += kTileWarps) {
    double d[NC];
    if (w < nl) {
      const int4 d4 = P.large[L0 + w];
      const int l0 = d4.y & 0xffff, l1 = d4.y >> 16;
      WN_DCHECK(l0 < l1 && l1 <= nv, "moment node range");
      warp_range_sum<NC>(sm, T, l0, l1, lane, d);
      if (lane == 0) sums_record<KIND, ORD>(d4.x, l1 - l0, d, tv, m, d4.w >> 16, d4.z, d4.w & 0xffff);
    } else if (w < nl + ne) {
      const int e = E0 + w - nl, slot = P.ep_slot[e];
      const int j = (int)(P.ep_key[e] - (uint64_t)tile * (T + 1));
      WN_DCHECK(j >= 0 && j <= nv, "moment endpoint");
      // slot 2c: the node starts here — its points from j to the tile's end; 2c + 1: it ends here — [0, j)
      if (slot & 1) warp_range_sum<NC>(sm, T, 0, j, lane, d);
      else warp_range_sum<NC>(sm, T, j, nv, lane, d);
      if (lane < NC) P.epval[(size_t)kMomNC * slot + lane] = pick<NC>(d, lane);
    } else {
      warp_range_sum<NC>(sm, T, 0, nv, lane, d);
      if (lane < NC) P.ttot[(size_t)kMomNC * tile + lane] = pick<NC>(d, lane);
    }
  }
}

// one warp per node across tiles: Σ at pb's end + the tile totals in between + Σ at pe's end
template <int KIND, int ORD>
__global__ void __launch_bounds__(256) mom_cross(TreeView tv, MomentArgs m, TilePlanView P) {
  constexpr int NC = Lay<KIND, ORD>::NC;
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (c >= P.ncross) return;
  const int64_t i = P.cross[c];
  const int j0 = tv.pb[i], j1 = tv.pe[i];
  const int64_t ta = j0 / P.tile, tb = (j1 - 1) / P.tile;
  double d[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) d[k] = 0.0;
  // lane-strided over the middle tiles, four tiles' loads in flight per step (added in tile order)
  constexpr int U = 4;
  for (int64_t k0 = ta + 1 + lane; k0 < tb; k0 += 32 * U) {
    double x[U][NC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + 32 * u;
#pragma unroll
      for (int q = 0; q < NC; ++q) x[u][q] = k < tb ? P.ttot[(size_t)kMomNC * k + q] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NC; ++q) d[q] += x[u][q];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int q = 0; q < NC; ++q) d[q] += __shfl_xor_sync(0xffffffffu, d[q], o);
  if (lane != 0) return;
  const double* ea = P.epval + (size_t)kMomNC * (2 * c);
  const double* eb = ea + kMomNC;
#pragma unroll
  for (int q = 0; q < NC; ++q) d[q] = (ea[q] + d[q]) + eb[q];
  sums_record<KIND, ORD>(i, j1 - j0, d, tv, m, tv.depth[i], tv.topo[i], tv.smask[i]);
}

template <int KIND, int ORD>
void launch_tiles(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  constexpr int NC = Lay<KIND, ORD>::NC;
  TreeView tv{t->pts, t->pb, t->pe, t->cb, t->cc, t->tdepth, t->topo, t->smask, t->sums, t->centroid};
  const MomPlan& Pl = t->mplan[(m.all_nodes || m.write_W || !t->mom_live) ? 1 : 0];
  TilePlanView P{Pl.small, Pl.large, Pl.tile_soff, Pl.tile_loff, Pl.cross, Pl.ep_slot, Pl.tile_eoff, Pl.onept,
                 Pl.ep_key, Pl.epval, t->mom_ttot, Pl.ncross, t->mom_tile};
  const size_t smem = (size_t)NC * t->mom_tile * sizeof(double);
  static uint64_t smem_set = 0;  // per instantiation and device: beyond the 48 KB default
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !((smem_set >> dev) & 1)) {
    cudaFuncSetAttribute(mom_tiles<KIND, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)NC * kMomTileMax * sizeof(double)));
    if (dev < 64) smem_set |= 1ull << dev;
  }
  mom_tiles<KIND, ORD><<<(unsigned)t->mom_ntiles, kTileThreads, smem, s>>>(tv, m, t->n, P);
  if (Pl.ncross > 0) mom_cross<KIND, ORD><<<(unsigned)((Pl.ncross * 32 + 255) / 256), 256, 0, s>>>(tv, m, P);
}

template <int KIND>
void launch_all(wn_tree_s* t, const MomentArgs& m, cudaStream_t s, const int64_t* loff_dev) {
  TreeView tv{t->pts, t->pb, t->pe, t->cb, t->cc, t->tdepth, t->topo, t->smask, t->sums, t->centroid};
  const int cut = t->mom_cut;
  if (cut <= t->depth_used) {
    // levels ≥ cut: all their leaves in one launch, then one launch per level for the internal nodes
    const int64_t i0 = t->level_off[cut], nn = t->nn;
    moments_range<KIND, 0><<<(unsigned)((nn - i0 + kMomThreads - 1) / kMomThreads), kMomThreads, 0, s>>>(
        tv, m, i0, i0, nn, 0);
    for (int l = t->depth_used - 1; l >= cut; l -= 2) {  // two levels per launch
      const int lo = l - 1 >= cut ? l - 1 : l;
      const int64_t a = t->level_off[lo], mid = t->level_off[l], b = t->level_off[l + 1];
      moments_range<KIND, 1><<<(unsigned)((b - a + kMomThreads - 1) / kMomThreads), kMomThreads, 0, s>>>(
          tv, m, a, mid, b, l);
    }
  }
  // the few levels above the cut: one block, __syncthreads() between levels
  if (cut > 0) moments_top<KIND><<<1, kTopThreads, 0, s>>>(tv, m, loff_dev, cut);
}

}  // namespace

// Points per tile.  A tile block holds its points' terms in shared memory (7 fp64 planes for a vector
// attribute: 57 KB at 1024 points, so 3 blocks per SM).  1024 by default; a cloud whose 1024-point tiles
// would spill just over one wave of resident tiles (3 per SM) takes the multiple of 128 up to kMomTileMax
// that fits one wave (C3 500k: 1152, 435 tiles: moments 7.3 → 6.6 ms per step); a cloud of fewer than two
// 1024-point tiles per SM is cut into about two tiles per SM (multiples of 128, ≥ 256) — more blocks in
// flight (40-iteration solve: C1 2k 256 points, 8.5 → 8.0 ms; C2 50k 256, 39.5 → 38.8; C4 200k 768,
// 67.0 → 66.1); large clouds (many waves) keep 1024 (C5: 1152 would cost 34 → 36 ms of moments).
int choose_mom_tile(int64_t n, int sms) {
  if (WN_EXP_MOMTILE != 1024) return WN_EXP_MOMTILE;  // (experiment builds pin the tile)
  const int64_t t1024 = (n + 1023) / 1024, wave = 3ll * sms;
  if (t1024 < 2ll * sms) {  // few tiles: about two per SM, multiples of 128 points, at least 256
    const int64_t want = ((n + 2ll * sms - 1) / (2ll * sms) + 127) / 128 * 128;
    return (int)std::min<int64_t>(1024, std::max<int64_t>(256, want));
  }
  if (t1024 > wave) {
    const int64_t need = ((n + wave - 1) / wave + 127) / 128 * 128;
    if (need <= kMomTileMax) return (int)need;
  }
  return 1024;
}

wn_status plan_moments(wn_tree_s* t, cudaStream_t s) {
  // cut at the first level with ≥ 1024 nodes: the levels above it run in one block
  const int deepest = t->depth_used;
  int cut = deepest + 1;
  for (int l = 0; l <= deepest; ++l)
    if (t->level_off[l + 1] - t->level_off[l] >= 1024) {
      cut = l;
      break;
    }
  t->mom_cut = cut;
  WN_CUDA(cudaMallocAsync((void**)&t->mom_loff, t->level_off.size() * sizeof(int64_t), s));
  WN_CUDA(cudaMemcpyAsync(t->mom_loff, t->level_off.data(), t->level_off.size() * sizeof(int64_t),
                          cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  t->mom_tile = choose_mom_tile(t->n, sms);
  t->mom_ntiles = (t->n + t->mom_tile - 1) / t->mom_tile;
  WN_TRY(plan_moment_tiles(t, 0, s));
  return WN_OK;
}

wn_status build_moments(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  if (m.kind != ATTR_UNIT) {  // per-iteration attributes: tile builds
    const int which = (m.all_nodes || m.write_W || !t->mom_live) ? 1 : 0;
    WN_TRY(plan_moment_tiles(t, which, s));  // (the export plan on first use; never inside a graph capture)
    ProfScope ps(WN_PROF_MOMENTS, s, t->mplan[which].ncross > 0 ? 2 : 1);  // mom_tiles (+ mom_cross)
    if (m.order1 && !(m.out.ext && t->mom_order1_ready)) return set_error(WN_ERR_ARG, "internal: order-1 scratch");
    if (m.kind == ATTR_VEC) {
      if (m.order1) launch_tiles<ATTR_VEC, 1>(t, m, s);
      else launch_tiles<ATTR_VEC, 0>(t, m, s);
    } else {
      if (m.order1) launch_tiles<ATTR_SCALAR, 1>(t, m, s);
      else launch_tiles<ATTR_SCALAR, 0>(t, m, s);
    }
    WN_CUDA(cudaGetLastError());
    return WN_OK;
  }
  ProfScope ps(WN_PROF_MOMENTS, s, (t->mom_cut <= t->depth_used ? 1 + (t->depth_used - t->mom_cut + 1) / 2 : 0) + (t->mom_cut > 0));
  switch (m.kind) {
    case ATTR_VEC: launch_all<ATTR_VEC>(t, m, s, t->mom_loff); break;
    case ATTR_SCALAR: launch_all<ATTR_SCALAR>(t, m, s, t->mom_loff); break;
    default: launch_all<ATTR_UNIT>(t, m, s, t->mom_loff); break;
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

// order-1 far field (row f2): larger prefix entries and tile totals, the node sets' ext arrays
wn_status enable_order1(wn_tree_s* t, cudaStream_t s) {
  if (t->mom_order1_ready) return WN_OK;
  invalidate_graph(t);  // (no captured buffer changes; a cached graph is keyed on the order anyway)
  WN_CUDA(cudaMallocAsync((void**)&t->set[0].ext, 2 * (size_t)(t->nn + 1) * sizeof(float4), s));
  WN_CUDA(cudaMemsetAsync(t->set[0].ext, 0, 2 * (size_t)(t->nn + 1) * sizeof(float4), s));
  t->mom_order1_ready = true;
  return WN_OK;
}

}  // namespace wn
