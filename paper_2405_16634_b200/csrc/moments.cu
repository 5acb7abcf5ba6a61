// moments.cu — per-application representatives.
//
// PAPER.md:L371-L378 (§4.5, Eqs node-rep-loc / node-rep-vec): for attribute ν,
//     x_{B,ν} = Σ_{i∈B} |ν_i| x_i / Σ_{j∈B} |ν_j| ,   ν_B = Σ_{i∈B} ν_i .
// Readings: Σ|ν| = 0 ⇒ the node's unweighted centroid; a one-point node's rep is the
// point itself; |ν| is the Euclidean norm (vector) or |s| (scalar).
//
// B200 design: fp64 node sums (W, P, V) built bottom-up; an internal node sums its children IN CHILD
// ORDER (deterministic).  One-point leaves (≈60 % of the nodes) are special: their record's position,
// threshold (−1) and remainder never change, so a build rewrites only their attribute word (16 B), and
// they keep no fp64 sums — a parent recomputes a one-point child's contribution from the point itself
// with the same fp64 operations.  No fences, no atomics; kernel boundaries order the levels:
//   1. one launch for every leaf at or below the cut level (the first level with ≥ 1024 nodes);
//   2. one launch per pair of levels, deepest first, for the internal nodes at or below the cut (the
//      upper level of a pair forms its children's sums from the grandchildren in the same order);
//   3. one single-block launch for the few levels above the cut (__syncthreads() between levels).
// Per build: 32 B read per point; per multi-point node 64 B sums + 48 B record written and ≈64 B read;
// 16 B per one-point leaf.
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
  const int32_t *pb, *pe, *cb, *cc, *depth, *topo, *smask;
  double* sums;
  const float4* centroid;
};

__device__ __forceinline__ float thr_of(float theta, int depth) {
  // (c · edge)², edge = 2^{1−depth} of the root cube [−1,1]^3, in fp32 (exact power-of-two scaling)
  float cw = theta * __int_as_float((127 + 1 - depth) << 23);
  return __fmul_rn(cw, cw);
}

__device__ __forceinline__ void add(Sums& S, const Sums& C) {
  S.W += C.W;
  for (int k = 0; k < 3; ++k) {
    S.P[k] += C.P[k];
    S.V[k] += C.V[k];
  }
}

// fp64 contribution of sorted point j: W = |ν_j|, P = |ν_j| x_j, V = ν_j.  WRITE: compute the fused
// axpy μ' = μ + α r and store it; otherwise read the μ' a previous launch stored (same value).
template <int KIND, bool WRITE>
__device__ __forceinline__ Sums point_sums(int j, const TreeView& tv, const MomentArgs& m, float alpha) {
  const float4 x = tv.pts[j];
  double a, v0 = 0, v1 = 0, v2 = 0;
  if (KIND == ATTR_VEC) {
    float4 v;
    if (m.axpy_r) {  // μ' = μ + α r (Alg. 2 line 3), written once, read by the G traversal
      if (WRITE) {
        const float4 mu = m.vec[j], r = m.axpy_r[j];
        v = make_float4(fmaf(alpha, r.x, mu.x), fmaf(alpha, r.y, mu.y), fmaf(alpha, r.z, mu.z), 0.f);
        m.axpy_out[j] = v;
      } else {
        v = m.axpy_out[j];
      }
    } else {
      v = m.vec[j];
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
  }
  Sums S;
  S.W = a;
  S.P[0] = a * (double)x.x;
  S.P[1] = a * (double)x.y;
  S.P[2] = a * (double)x.z;
  S.V[0] = v0;
  S.V[1] = v1;
  S.V[2] = v2;
  return S;
}

__device__ __forceinline__ Sums load_sums(const double* __restrict__ sums, int64_t c) {
  const double2* q = reinterpret_cast<const double2*>(sums + 8 * c);
  const double2 a = q[0], b = q[1], d = q[2], e = q[3];
  return Sums{a.x, {a.y, b.x, b.y}, {d.x, d.y, e.x}};
}

__device__ __forceinline__ void store_sums(double* __restrict__ sums, int64_t i, const Sums& S) {
  double2* o = reinterpret_cast<double2*>(sums + 8 * i);
  o[0] = make_double2(S.W, S.P[0]);
  o[1] = make_double2(S.P[1], S.P[2]);
  o[2] = make_double2(S.V[0], S.V[1]);
  o[3] = make_double2(S.V[2], 0.0);
}

// a child's fp64 sums: a one-point leaf from its point, anything else from the stored sums
template <int KIND>
__device__ __forceinline__ Sums child_sums(int c, bool single, const TreeView& tv, const MomentArgs& m,
                                           float alpha) {
  return single ? point_sums<KIND, false>(tv.pb[c], tv, m, alpha) : load_sums(tv.sums, c);
}

__device__ __forceinline__ float4 attr_word(const Sums& S, int topo, int kind) {
  if (kind == ATTR_SCALAR) return make_float4((float)S.V[0], 0.f, 0.f, __int_as_float(topo));
  return make_float4((float)S.V[0], (float)S.V[1], (float)S.V[2], __int_as_float(topo));
}

// full 48-byte record of a multi-point node
template <int KIND>
__device__ __forceinline__ void write_record(int64_t i, const Sums& S, int depth, int topo, int smask, float theta,
                                             const float4* __restrict__ centroid, const MomentArgs& m) {
  float4 R, L = make_float4(0.f, 0.f, 0.f, 0.f);
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
  L.w = __int_as_float(smask);  // which children are one-point leaves
  float4* rec = m.out.rec + kRec * i;
  rec[0] = R;
  rec[1] = attr_word(S, topo, KIND);
  rec[2] = L;
  if (KIND == ATTR_UNIT) m.centroid_out[i] = make_float4(R.x, R.y, R.z, 0.f);
}

template <int KIND>
__device__ __forceinline__ void process_leaf(int64_t i, int depth, const TreeView& tv, const MomentArgs& m,
                                             float alpha) {
  const int j0 = tv.pb[i], j1 = tv.pe[i];
  if (j1 - j0 == 1) {  // one-point leaf: only the attribute word changes between builds
    const Sums S = point_sums<KIND, true>(j0, tv, m, alpha);
    m.out.rec[kRec * i + 1] = attr_word(S, 0, KIND);
    if (KIND == ATTR_UNIT) {  // once per tree: the static parts, in both record sets
      const float4 x = tv.pts[j0];
      const float4 R = make_float4(x.x, x.y, x.z, -1.0f), L = make_float4(0.f, 0.f, 0.f, 0.f);
      m.out.rec[kRec * i] = R;
      m.out.rec[kRec * i + 2] = L;
      m.out2.rec[kRec * i] = R;
      m.out2.rec[kRec * i + 2] = L;
      m.centroid_out[i] = make_float4(x.x, x.y, x.z, 0.f);
      m.leaf_of_out[j0] = (int32_t)i;
    }
    return;
  }
  Sums S = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};  // multi-point leaf (depth D)
  for (int j = j0; j < j1; ++j) {
    add(S, point_sums<KIND, true>(j, tv, m, alpha));
    if (KIND == ATTR_UNIT) m.leaf_of_out[j] = (int32_t)i;
  }
  store_sums(tv.sums, i, S);
  write_record<KIND>(i, S, depth, 0, 0, m.theta, tv.centroid, m);
}

// internal node: Σ of its children in child order.  DEEP: the children's sums are formed here from the
// grandchildren (same operations, same order as the child's own thread), finishing two levels per launch.
template <int KIND, bool DEEP>
__device__ __forceinline__ void process_internal(int64_t i, int depth, const TreeView& tv, const MomentArgs& m,
                                                 float alpha) {
  Sums S = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  const int nc = tv.cc[i], c0 = tv.cb[i], sm = tv.smask[i];
  for (int k = 0; k < nc; ++k) {
    const int c = c0 + k;
    const bool single = (sm >> k) & 1;
    const int gn = DEEP && !single ? tv.cc[c] : 0;
    if (gn == 0) {
      add(S, child_sums<KIND>(c, single, tv, m, alpha));
    } else {
      Sums C = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
      const int g0 = tv.cb[c], gsm = tv.smask[c];
      for (int g = 0; g < gn; ++g) add(C, child_sums<KIND>(g0 + g, (gsm >> g) & 1, tv, m, alpha));
      add(S, C);
    }
  }
  store_sums(tv.sums, i, S);
  write_record<KIND>(i, S, depth, tv.topo[i], sm, m.theta, tv.centroid, m);
}

// MODE 0: every leaf in [i0, i1) (any level).  MODE 1: the internal nodes of levels `level` ([imid, i1))
// and `level − 1` ([i0, imid)) — the latter from their grandchildren.
template <int KIND, int MODE>
__global__ void __launch_bounds__(kMomThreads) moments_range(TreeView tv, MomentArgs m, int64_t i0, int64_t imid,
                                                             int64_t i1, int level) {
  const int64_t i = i0 + blockIdx.x * (int64_t)kMomThreads + threadIdx.x;
  if (i >= i1) return;
  const bool leaf = tv.cc[i] == 0;
  if (leaf != (MODE == 0)) return;
  const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
  if (MODE == 0) process_leaf<KIND>(i, tv.depth[i], tv, m, alpha);
  else if (i >= imid) process_internal<KIND, false>(i, level, tv, m, alpha);
  else process_internal<KIND, true>(i, level - 1, tv, m, alpha);
}

template <int KIND>
__global__ void __launch_bounds__(kTopThreads) moments_top(TreeView tv, MomentArgs m, const int64_t* __restrict__ loff,
                                                           int cut) {
  const float alpha = (KIND == ATTR_VEC && m.axpy_r) ? (float)(*m.alpha) : 0.f;
  for (int l = cut - 1; l >= 0; --l) {
    const int64_t i0 = loff[l], i1 = loff[l + 1];
    for (int64_t i = i0 + threadIdx.x; i < i1; i += kTopThreads) {
      if (tv.cc[i] == 0) process_leaf<KIND>(i, l, tv, m, alpha);
      else process_internal<KIND, false>(i, l, tv, m, alpha);
    }
    __syncthreads();
  }
}

template <int KIND>
void launch_all(wn_tree_s* t, const MomentArgs& m, cudaStream_t s, const int64_t* loff_dev) {
  TreeView tv{t->pts, t->pb, t->pe, t->cb, t->cc, t->depth, t->topo, t->smask, t->sums, t->centroid};
  const int cut = t->mom_cut;
  if (cut <= t->depth_used) {
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
  if (cut > 0) moments_top<KIND><<<1, kTopThreads, 0, s>>>(tv, m, loff_dev, cut);
}

// diagnostics (wn_moments): store the fp64 sums of the one-point leaves too
template <int KIND>
__global__ void single_leaf_sums(TreeView tv, MomentArgs m, int64_t nn) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn || tv.cc[i] != 0 || tv.pe[i] - tv.pb[i] != 1) return;
  store_sums(tv.sums, i, point_sums<KIND, false>(tv.pb[i], tv, m, 0.f));
}

}  // namespace

wn_status export_single_leaf_sums(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  TreeView tv{t->pts, t->pb, t->pe, t->cb, t->cc, t->depth, t->topo, t->smask, t->sums, t->centroid};
  const unsigned g = (unsigned)((t->nn + 255) / 256);
  if (m.kind == ATTR_SCALAR) single_leaf_sums<ATTR_SCALAR><<<g, 256, 0, s>>>(tv, m, t->nn);
  else single_leaf_sums<ATTR_VEC><<<g, 256, 0, s>>>(tv, m, t->nn);
  count_launches(1);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
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
  return WN_OK;
}

wn_status build_moments(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  const int below = t->mom_cut <= t->depth_used ? 1 + (t->depth_used - t->mom_cut + 1) / 2 : 0;
  ProfScope ps(WN_PROF_MOMENTS, s, below + (t->mom_cut > 0));
  switch (m.kind) {
    case ATTR_VEC: launch_all<ATTR_VEC>(t, m, s, t->mom_loff); break;
    case ATTR_SCALAR: launch_all<ATTR_SCALAR>(t, m, s, t->mom_loff); break;
    default: launch_all<ATTR_UNIT>(t, m, s, t->mom_loff); break;
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

}  // namespace wn
