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
  const int32_t *pb, *pe, *cb, *cc, *depth, *topo, *smask;
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
  write_record<KIND>(i, S, j1 - j0, p0, depth, tv.topo[i], tv.smask[i], m.theta, tv.centroid, m);
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

template <int KIND>
void launch_all(wn_tree_s* t, const MomentArgs& m, cudaStream_t s, const int64_t* loff_dev) {
  TreeView tv{t->pts, t->pb, t->pe, t->cb, t->cc, t->depth, t->topo, t->smask, t->sums, t->centroid};
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
  return WN_OK;
}

wn_status build_moments(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  ProfScope ps(WN_PROF_MOMENTS, s, (t->mom_cut <= t->depth_used ? 1 + (t->depth_used - t->mom_cut + 1) / 2 : 0) + (t->mom_cut > 0));
  switch (m.kind) {
    case ATTR_VEC: launch_all<ATTR_VEC>(t, m, s, t->mom_loff); break;
    case ATTR_SCALAR: launch_all<ATTR_SCALAR>(t, m, s, t->mom_loff); break;
    default: launch_all<ATTR_UNIT>(t, m, s, t->mom_loff); break;
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

}  // namespace wn
