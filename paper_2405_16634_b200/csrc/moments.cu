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

// ---------------- prefix-difference builds (per-iteration attributes: ATTR_VEC, ATTR_SCALAR) ----------------
// Every node B covers a contiguous range [pb, pe) of the Morton-sorted points, so its sums are
// E[pe] − E[pb] of one exclusive prefix E over the points' (|ν|, |ν|x, ν) — no level-by-level chain:
// one scan (3 launches) and one fully parallel node launch.  E is double-double (hi + lo, error-free
// two-sum adds; lo stored in fp32), so a difference keeps ≈ 2^-77·|Σ_all| accuracy — far below the bottom-up fp64
// rounding — and an exact integer count of the points with |ν| > 0 decides Σ|ν| = 0 (⇒ centroid)
// exactly.  One-point nodes take their point's own values (exact: rep = the point).  DESIGN.md §Moments.
// First-order far field (ORD = 1): the prefix also carries sym(Σ ν_j x_jᵀ) (vector ν,
// 6 terms) or Σ s_j x_j (scalar, 3), and each node stores its first moment about the representative,
// sym M = sym(Σ ν_j x_jᵀ) − sym(ν_B x_Bᵀ) or D = Σ s_j x_j − s_B x_B, in NodeSet::ext.
#ifndef WN_EXP_SCANITEMS
#define WN_EXP_SCANITEMS 8
#endif
constexpr int kScanThreads = 256, kScanItems = WN_EXP_SCANITEMS, kScanTile = kScanThreads * kScanItems;
constexpr int kScanTopThreads = 256;
#ifndef WN_EXP_FEWTILES
#define WN_EXP_FEWTILES 512
#endif
constexpr int kFewTiles = WN_EXP_FEWTILES;  // up to this many tiles the prefix blocks sum earlier totals themselves

// components per prefix entry; entry j (exclusive: points [0, j)) = hi[EH] fp64 (the NC sums, the count,
// padding) in E_hi and lo[EL] = the double-double low parts rounded to fp32 in E_lo
template <int KIND, int ORD>
struct PreLayout {
  static constexpr int NC = ORD == 0 ? 7 : (KIND == ATTR_VEC ? 13 : 10);
  static constexpr int EH = (NC + 2) & ~1;
  static constexpr int EL = (NC + 3) & ~3;
};
constexpr int kPreDoublesMax = 14 + 8;  // EH + EL/2 of the largest layout (vector, ORD 1)

struct DD {
  double hi, lo;
};

// two-sum based double-double addition (adds only: nothing for the compiler to contract)
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  const double s = __dadd_rn(a.hi, b.hi);
  const double bb = __dsub_rn(s, a.hi);
  double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
  e = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
  const double h = __dadd_rn(s, e);
  return DD{h, __dsub_rn(e, __dsub_rn(h, s))};
}

// per-point terms: (|ν|, |ν|x, |ν|y, |ν|z, ν) and, for ORD 1, sym(ν xᵀ) (xx, yy, zz, xy, xz, yz) or s x;
// v: the attribute (vector: μ, or μ + α r when r is given; scalar: v.x), f: the per-point factor a (or 1)
template <int KIND, int ORD>
__device__ __forceinline__ void point_terms(float4 x, float4 v, const float4* r, float alpha, double f,
                                            bool scaled, double* o) {
  double a, v0, v1 = 0.0, v2 = 0.0;
  if (KIND == ATTR_VEC) {
    if (r)  // μ' = μ + α r (Alg. 2 line 3) — the same fmaf as the record's one-point branch
      v = make_float4(fmaf(alpha, r->x, v.x), fmaf(alpha, r->y, v.y), fmaf(alpha, r->z, v.z), 0.f);
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
  o[5] = v1;
  o[6] = v2;
  if (ORD == 1) {
    if (KIND == ATTR_VEC) {
      o[7] = v0 * px;
      o[8] = v1 * py;
      o[9] = v2 * pz;
      o[10] = 0.5 * (v0 * py + v1 * px);
      o[11] = 0.5 * (v0 * pz + v2 * px);
      o[12] = 0.5 * (v1 * pz + v2 * py);
    } else {
      o[7] = v0 * px;
      o[8] = v0 * py;
      o[9] = v0 * pz;
    }
  }
}

template <int KIND, int ORD>
__device__ __forceinline__ void point_vals(int64_t j, const float4* __restrict__ pts, const MomentArgs& m, float alpha,
                                           double* o) {
  float4 v;
  float4 r;
  if (KIND == ATTR_VEC) {
    v = m.vec[j];
    if (m.axpy_r) r = m.axpy_r[j];
  } else {
    v = make_float4(m.scal[j], 0.f, 0.f, 0.f);
  }
  const bool scaled = m.a_sorted != nullptr;
  point_terms<KIND, ORD>(pts[j], v, KIND == ATTR_VEC && m.axpy_r ? &r : nullptr, alpha,
                         scaled ? (double)m.a_sorted[j] : 1.0, scaled, o);
}

// scan element: NC double-double sums + the number of points with |ν| > 0 (an exact integer)
template <int NC>
struct Elt {
  DD v[NC];
  double cnt;
};

template <int NC>
__device__ __forceinline__ void elt_zero(Elt<NC>& e) {
#pragma unroll
  for (int c = 0; c < NC; ++c) e.v[c] = DD{0.0, 0.0};
  e.cnt = 0.0;
}
template <int NC>
__device__ __forceinline__ void elt_add(Elt<NC>& e, const Elt<NC>& f) {
#pragma unroll
  for (int c = 0; c < NC; ++c) e.v[c] = dd_add(e.v[c], f.v[c]);
  e.cnt += f.cnt;
}
template <int NC>
__device__ __forceinline__ void elt_add_point(Elt<NC>& e, const double* o) {
#pragma unroll
  for (int c = 0; c < NC; ++c) e.v[c] = dd_add(e.v[c], DD{o[c], 0.0});
  e.cnt += o[0] > 0.0 ? 1.0 : 0.0;
}
template <int NC>
__device__ __forceinline__ Elt<NC> elt_shfl_up(const Elt<NC>& e, int d) {
  Elt<NC> r;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    r.v[c].hi = __shfl_up_sync(0xffffffffu, e.v[c].hi, d);
    r.v[c].lo = __shfl_up_sync(0xffffffffu, e.v[c].lo, d);
  }
  r.cnt = __shfl_up_sync(0xffffffffu, e.cnt, d);
  return r;
}
// inclusive warp scan over the first `width` lanes (fixed order)
template <int NC>
__device__ __forceinline__ void warp_inscan(Elt<NC>& x, int lane, int width) {
  for (int o = 1; o < width; o <<= 1) {
    const Elt<NC> y = elt_shfl_up(x, o);
    if (lane >= o) {
      Elt<NC> z = y;
      elt_add(z, x);
      x = z;
    }
  }
}

// block-wide exclusive scan (fixed order: deterministic); e becomes the exclusive prefix, tot the total
template <int NT, int NC>
__device__ __forceinline__ void block_exscan(Elt<NC>& e, Elt<NC>& tot) {
  constexpr int NW = NT / 32;
  __shared__ Elt<NC> ws[NW + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Elt<NC> inc = e;
  warp_inscan(inc, lane, 32);
  if (lane == 31) ws[warp] = inc;
  Elt<NC> prev = elt_shfl_up(inc, 1);
  if (lane == 0) elt_zero(prev);
  __syncthreads();
  if (warp == 0) {  // scan of the warp totals by one warp
    Elt<NC> x;
    if (lane < NW) x = ws[lane];
    else elt_zero(x);
    warp_inscan(x, lane, NW);
    Elt<NC> xp = elt_shfl_up(x, 1);
    if (lane == 0) elt_zero(xp);
    __syncwarp();
    if (lane < NW) ws[lane] = xp;
    if (lane == NW - 1) ws[NW] = x;
  }
  __syncthreads();
  e = ws[warp];
  elt_add(e, prev);
  tot = ws[NW];
  __syncthreads();
}

template <int KIND, int ORD>
__global__ void __launch_bounds__(kScanThreads) mom_tile_sum(const float4* __restrict__ pts, MomentArgs m, int64_t n,
                                                             Elt<PreLayout<KIND, ORD>::NC>* __restrict__ tile_tot) {
  constexpr int NC = PreLayout<KIND, ORD>::NC;
  const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
  Elt<NC> t, tot;
  elt_zero(t);
  // coalesced: item k of thread x is point tile·T + k·256 + x (totals need no ownership order)
  const int64_t j0 = blockIdx.x * (int64_t)kScanTile + threadIdx.x;
#pragma unroll 2
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t j = j0 + k * kScanThreads;
    if (j < n) {
      double o[NC];
      point_vals<KIND, ORD>(j, pts, m, alpha, o);
      elt_add_point(t, o);
    }
  }
  block_exscan<kScanThreads>(t, tot);
  if (threadIdx.x == 0) tile_tot[blockIdx.x] = tot;
}

template <int NC>
__global__ void __launch_bounds__(kScanTopThreads) mom_tile_scan(const Elt<NC>* __restrict__ tile_tot, int64_t ntiles,
                                                                 Elt<NC>* __restrict__ tile_off) {
  const int64_t per = (ntiles + kScanTopThreads - 1) / kScanTopThreads;
  const int64_t t0 = threadIdx.x * per, t1 = min(ntiles, t0 + per);
  Elt<NC> v, tot;
  elt_zero(v);
  for (int64_t t = t0; t < t1; ++t) elt_add(v, tile_tot[t]);
  block_exscan<kScanTopThreads>(v, tot);
  for (int64_t t = t0; t < t1; ++t) {
    tile_off[t] = v;
    elt_add(v, tile_tot[t]);
  }
}

template <int KIND, int ORD>
__device__ __forceinline__ void store_pre(double* __restrict__ Eh, float* __restrict__ El, int64_t j,
                                          const Elt<PreLayout<KIND, ORD>::NC>& t) {
  using Lay = PreLayout<KIND, ORD>;
  double h[Lay::EH];
  float l[Lay::EL];
#pragma unroll
  for (int c = 0; c < Lay::EH; ++c) h[c] = c < Lay::NC ? t.v[c].hi : (c == Lay::NC ? t.cnt : 0.0);
#pragma unroll
  for (int c = 0; c < Lay::EL; ++c) l[c] = c < Lay::NC ? (float)t.v[c].lo : 0.f;
  double2* hp = reinterpret_cast<double2*>(Eh + Lay::EH * j);
#pragma unroll
  for (int c = 0; c < Lay::EH / 2; ++c) hp[c] = make_double2(h[2 * c], h[2 * c + 1]);
  float4* lp = reinterpret_cast<float4*>(El + Lay::EL * j);
#pragma unroll
  for (int c = 0; c < Lay::EL / 4; ++c) lp[c] = make_float4(l[4 * c], l[4 * c + 1], l[4 * c + 2], l[4 * c + 3]);
}

// the prefix stages its tile's inputs in shared memory with coalesced loads (points, attribute, r) and the
// threads then read their consecutive items from there: padded one float4 (float) per 8 so that the
// stride-8 item reads of a warp are free of bank conflicts
constexpr int kStageN = kScanTile + kScanTile / 8;
__device__ __forceinline__ int stage_ix(int jl) { return jl + (jl >> 3); }
template <int KIND>
constexpr size_t stage_bytes() {  // points, attribute (float4 / float), r (vector only)
  return KIND == ATTR_VEC ? 3 * kStageN * sizeof(float4) : kStageN * (sizeof(float4) + sizeof(float));
}

template <int KIND, int ORD>
__global__ void __launch_bounds__(kScanThreads) mom_tile_prefix(const float4* __restrict__ pts, MomentArgs m,
                                                                int64_t n,
                                                                const Elt<PreLayout<KIND, ORD>::NC>* __restrict__ tile_off,
                                                                const Elt<PreLayout<KIND, ORD>::NC>* __restrict__ tile_tot,
                                                                double* __restrict__ Eh, float* __restrict__ El) {
  constexpr int NC = PreLayout<KIND, ORD>::NC;
  extern __shared__ float4 stage[];
  float4* sp = stage;
  float4* sv = stage + kStageN;                                   // vector attribute
  float4* sr = stage + 2 * kStageN;                               // r (μ' = μ + α r)
  float* ss = reinterpret_cast<float*>(stage + kStageN);          // scalar attribute
  const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
  const bool axpy = KIND == ATTR_VEC && m.axpy_r;
  const bool scaled = m.a_sorted != nullptr;
  const int64_t base = blockIdx.x * (int64_t)kScanTile;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {  // coalesced staging
    const int jl = threadIdx.x + k * kScanThreads;
    const int64_t j = base + jl;
    if (j < n) {
      const int x = stage_ix(jl);
      sp[x] = pts[j];
      if (KIND == ATTR_VEC) {
        sv[x] = m.vec[j];
        if (axpy) sr[x] = m.axpy_r[j];
      } else {
        ss[x] = m.scal[j];
      }
    }
  }
  __syncthreads();
  auto vals = [&](int jl, double* o) {
    const int x = stage_ix(jl);
    const float4 v = KIND == ATTR_VEC ? sv[x] : make_float4(ss[x], 0.f, 0.f, 0.f);
    float4 r;
    if (axpy) r = sr[x];
    point_terms<KIND, ORD>(sp[x], v, axpy ? &r : nullptr, alpha, scaled ? (double)m.a_sorted[base + jl] : 1.0,
                           scaled, o);
  };
  Elt<NC> t, tot;
  elt_zero(t);
  const int jl0 = threadIdx.x * kScanItems;  // consecutive ownership
  const int64_t j0 = base + jl0;
  for (int k = 0; k < kScanItems; ++k)
    if (j0 + k < n) {
      double o[NC];
      vals(jl0 + k, o);
      elt_add_point(t, o);
    }
  block_exscan<kScanThreads>(t, tot);
  if (tile_off) {  // the tile offsets of mom_tile_scan
    Elt<NC> z = tile_off[blockIdx.x];
    elt_add(z, t);
    t = z;
  } else if (tile_tot && blockIdx.x > 0) {  // few tiles: this tile's offset = Σ of the earlier totals, here
    Elt<NC> v, z;
    elt_zero(v);
    for (int64_t k = threadIdx.x; k < blockIdx.x; k += kScanThreads) elt_add(v, tile_tot[k]);
    block_exscan<kScanThreads>(v, z);  // z: the block total, a fixed-order reduction
    elt_add(z, t);
    t = z;
  }  // (neither: a single tile, offset 0)
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t j = j0 + k;
    if (j < n) {
      store_pre<KIND, ORD>(Eh, El, j, t);
      double o[NC];
      vals(jl0 + k, o);
      elt_add_point(t, o);
      if (j == n - 1) store_pre<KIND, ORD>(Eh, El, n, t);
    }
  }
  if (axpy) {  // μ' written once here (coalesced), read by the G traversal
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int jl = threadIdx.x + k * kScanThreads;
      if (base + jl < n) {
        const int x = stage_ix(jl);
        const float4 v = sv[x], r = sr[x];
        m.axpy_out[base + jl] = make_float4(fmaf(alpha, r.x, v.x), fmaf(alpha, r.y, v.y), fmaf(alpha, r.z, v.z), 0.f);
      }
    }
  }
}

template <int KIND, int ORD>
__global__ void __launch_bounds__(256) mom_nodes(TreeView tv, MomentArgs m, int64_t nn, const double* __restrict__ Eh,
                                                 const float* __restrict__ El, const int32_t* __restrict__ list) {
  using Lay = PreLayout<KIND, ORD>;
  constexpr int NC = Lay::NC;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nn) return;
  const int64_t i = list ? (int64_t)list[k] : k;  // list: only the nodes a traversal can visit
  WN_DCHECK(i >= 0 && i < (list ? (int64_t)1 << 31 : nn), "moment node index");
  const int j0 = tv.pb[i], j1 = tv.pe[i];
  double d[NC];
  const float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j1 - j0 == 1) {  // one-point node: R = (x_j, −1), L and ext (= 0) are fixed per tree — only V = ν_j
    const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
    double v0, v1 = 0.0, v2 = 0.0;
    if (KIND == ATTR_VEC) {
      float4 v = m.vec[j0];
      if (m.axpy_r) {
        const float4 r = m.axpy_r[j0];
        v = make_float4(fmaf(alpha, r.x, v.x), fmaf(alpha, r.y, v.y), fmaf(alpha, r.z, v.z), 0.f);
      }
      v0 = v.x; v1 = v.y; v2 = v.z;
      if (m.a_sorted) {
        const double f = m.a_sorted[j0];
        v0 *= f; v1 *= f; v2 *= f;
      }
      if (m.write_W) tv.sums[8 * i] = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
    } else {
      v0 = m.scal[j0];
      if (m.a_sorted) v0 *= (double)m.a_sorted[j0];
      if (m.write_W) tv.sums[8 * i] = fabs(v0);
    }
    m.out.rec[kRec * i + 1] = make_float4((float)v0, (float)v1, (float)v2, __int_as_float(tv.topo[i]));
    return;
  } else {
    WN_DCHECK(j0 >= 0 && j0 < j1, "moment point range");
    const double2* a = reinterpret_cast<const double2*>(Eh + Lay::EH * (int64_t)j0);
    const double2* b = reinterpret_cast<const double2*>(Eh + Lay::EH * (int64_t)j1);
    double ah[Lay::EH], bh[Lay::EH];
#pragma unroll
    for (int c = 0; c < Lay::EH / 2; ++c) {
      const double2 x = a[c], y = b[c];
      ah[2 * c] = x.x; ah[2 * c + 1] = x.y;
      bh[2 * c] = y.x; bh[2 * c + 1] = y.y;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) d[c] = 0.0;
    if (bh[NC] != ah[NC]) {  // else no point has |ν| > 0: Σ|ν| = 0 and every ν_j = 0, exactly
      const float4* al = reinterpret_cast<const float4*>(El + Lay::EL * (int64_t)j0);
      const float4* bl = reinterpret_cast<const float4*>(El + Lay::EL * (int64_t)j1);
      float alo[Lay::EL], blo[Lay::EL];
#pragma unroll
      for (int c = 0; c < Lay::EL / 4; ++c) {
        const float4 x = al[c], y = bl[c];
        alo[4 * c] = x.x; alo[4 * c + 1] = x.y; alo[4 * c + 2] = x.z; alo[4 * c + 3] = x.w;
        blo[4 * c] = y.x; blo[4 * c + 1] = y.y; blo[4 * c + 2] = y.z; blo[4 * c + 3] = y.w;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) d[c] = dd_add(DD{bh[c], (double)blo[c]}, DD{-ah[c], -(double)alo[c]}).hi;
    }
  }
  Sums S;
  S.W = d[0];
  S.P[0] = d[1]; S.P[1] = d[2]; S.P[2] = d[3];
  S.V[0] = d[4]; S.V[1] = d[5]; S.V[2] = d[6];
  if (m.write_W) tv.sums[8 * i] = S.W;
  write_record<KIND>(i, S, j1 - j0, p0, tv.depth[i], tv.topo[i], tv.smask[i], m.theta, tv.centroid, m);
  if (ORD == 1) {  // first moment about the fp64 representative (0 for Σ|ν| = 0)
    float4 e0 = make_float4(0.f, 0.f, 0.f, 0.f), e1 = e0;
    if (S.W > 0.0) {
      const double X = S.P[0] / S.W, Y = S.P[1] / S.W, Z = S.P[2] / S.W;
      if (KIND == ATTR_VEC) {
        const double mxx = d[7] - S.V[0] * X, myy = d[8] - S.V[1] * Y, mzz = d[9] - S.V[2] * Z;
        const double mxy = d[10] - 0.5 * (S.V[0] * Y + S.V[1] * X);
        const double mxz = d[11] - 0.5 * (S.V[0] * Z + S.V[2] * X);
        const double myz = d[12] - 0.5 * (S.V[1] * Z + S.V[2] * Y);
        e0 = make_float4((float)mxx, (float)myy, (float)mzz, (float)(mxx + myy + mzz));
        e1 = make_float4((float)mxy, (float)mxz, (float)myz, 0.f);
      } else {
        e0 = make_float4((float)(d[7] - S.V[0] * X), (float)(d[8] - S.V[0] * Y), (float)(d[9] - S.V[0] * Z), 0.f);
      }
    }
    m.out.ext[2 * i] = e0;
    m.out.ext[2 * i + 1] = e1;
  }
}

template <int KIND, int ORD>
void launch_prefix(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  using Lay = PreLayout<KIND, ORD>;
  TreeView tv{t->pts, t->pb, t->pe, t->cb, t->cc, t->tdepth, t->topo, t->smask, t->sums, t->centroid};
  const int64_t nt = t->mom_ntiles;
  Elt<Lay::NC>* tot = reinterpret_cast<Elt<Lay::NC>*>(t->mom_tile);
  Elt<Lay::NC>* off = tot + nt;
  double* Eh = t->mom_pre;
  float* El = reinterpret_cast<float*>(t->mom_pre + Lay::EH * (t->n + 1));
  // a single tile needs no tile totals; up to kFewTiles tiles each prefix block sums the earlier tile
  // totals itself (no one-block scan launch); more tiles go through mom_tile_scan
  const bool scan = nt > kFewTiles;
  if (nt > 1) {
    mom_tile_sum<KIND, ORD><<<(unsigned)nt, kScanThreads, 0, s>>>(t->pts, m, t->n, tot);
    if (scan) mom_tile_scan<Lay::NC><<<1, kScanTopThreads, 0, s>>>(tot, nt, off);
  }
  static bool smem_set = false;  // per instantiation: the staging buffer exceeds the 48 KB default
  if (!smem_set) {
    cudaFuncSetAttribute(mom_tile_prefix<KIND, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)stage_bytes<KIND>());
    smem_set = true;
  }
  mom_tile_prefix<KIND, ORD><<<(unsigned)nt, kScanThreads, stage_bytes<KIND>(), s>>>(
      t->pts, m, t->n, scan ? off : nullptr, nt > 1 ? tot : nullptr, Eh, El);
  // per-iteration builds: only the nodes a traversal can read (chain interiors and the children of
  // pseudo-leaves are never visited); the diagnostic export (write_W) builds every node
  const bool all = m.all_nodes || m.write_W || !t->mom_live;
  const int64_t cnt = all ? t->nn : t->mom_nlive;
  mom_nodes<KIND, ORD><<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(tv, m, cnt, Eh, El, all ? nullptr : t->mom_live);
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
  t->mom_ntiles = (t->n + kScanTile - 1) / kScanTile;
  WN_CUDA(cudaMallocAsync((void**)&t->mom_pre, 12 * (size_t)(t->n + 1) * sizeof(double), s));
  WN_CUDA(cudaMallocAsync((void**)&t->mom_tile, 2 * (size_t)t->mom_ntiles * sizeof(Elt<7>), s));
  return WN_OK;
}

wn_status build_moments(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
#ifndef WN_EXP_OLD_MOM
  if (m.kind != ATTR_UNIT) {  // per-iteration attributes: prefix differences
    ProfScope ps(WN_PROF_MOMENTS, s, t->mom_ntiles > 1 ? (t->mom_ntiles > kFewTiles ? 4 : 3) : 2);
    if (m.order1 && !(m.out.ext && t->mom_order1_ready)) return set_error(WN_ERR_ARG, "internal: order-1 scratch");
    if (m.kind == ATTR_VEC) {
      if (m.order1) launch_prefix<ATTR_VEC, 1>(t, m, s);
      else launch_prefix<ATTR_VEC, 0>(t, m, s);
    } else {
      if (m.order1) launch_prefix<ATTR_SCALAR, 1>(t, m, s);
      else launch_prefix<ATTR_SCALAR, 0>(t, m, s);
    }
    WN_CUDA(cudaGetLastError());
    return WN_OK;
  }
#endif
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
  invalidate_graph(t);  // a cached order-0 graph references the prefix scratch freed here
  cudaFreeAsync(t->mom_pre, s);
  cudaFreeAsync(t->mom_tile, s);
  t->mom_pre = nullptr;
  t->mom_tile = nullptr;
  WN_CUDA(cudaMallocAsync((void**)&t->mom_pre, kPreDoublesMax * (size_t)(t->n + 1) * sizeof(double), s));
  WN_CUDA(cudaMallocAsync((void**)&t->mom_tile, 2 * (size_t)t->mom_ntiles * sizeof(Elt<13>), s));
  WN_CUDA(cudaMallocAsync((void**)&t->set[0].ext, 2 * (size_t)(t->nn + 1) * sizeof(float4), s));
  WN_CUDA(cudaMemsetAsync(t->set[0].ext, 0, 2 * (size_t)(t->nn + 1) * sizeof(float4), s));
  t->mom_order1_ready = true;
  return WN_OK;
}

}  // namespace wn
