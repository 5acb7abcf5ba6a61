// moments.cu — per-application representatives.
//
// PAPER.md:L371-L378 (§4.5, Eqs node-rep-loc / node-rep-vec): for attribute ν,
//     x_{B,ν} = Σ_{i∈B} |ν_i| x_i / Σ_{j∈B} |ν_j| ,   ν_B = Σ_{i∈B} ν_i .
// Readings: Σ|ν| = 0 ⇒ the node's unweighted centroid; a one-point node's rep is the
// point itself; |ν| is the Euclidean norm (vector) or |s| (scalar).
//
// B200 design: fp64 node sums (W, P, V) built bottom-up, level-synchronously: one launch sums every
// leaf over its points (thread per node), then one launch per level (deepest first) sums the children
// of that level's internal nodes IN CHILD ORDER.  Kernel boundaries order the levels, so there are no
// fences or atomics and the result is deterministic.  Each node writes its 64-byte traversal record
// (rep hi + lo, threshold, ν_B, topology code).  Traffic O(N + Nn): ≈ 32 B/point + 64 B sums +
// 64 B record per node.
#include <cuda_runtime.h>

#include "wn_internal.cuh"

namespace wn {
namespace {

struct Sums {
  double W, P[3], V[3];
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
  L.w = __int_as_float(smask);  // which children are one-point leaves (traversal fast path)
  rec[2] = L;
  if (KIND == ATTR_UNIT) m.centroid_out[i] = make_float4(R.x, R.y, R.z, 0.f);
}

__device__ __forceinline__ void store_sums(double* __restrict__ sums, int64_t i, const Sums& S) {
  double2* o = reinterpret_cast<double2*>(sums + 8 * i);
  o[0] = make_double2(S.W, S.P[0]);
  o[1] = make_double2(S.P[1], S.P[2]);
  o[2] = make_double2(S.V[0], S.V[1]);
  o[3] = make_double2(S.V[2], 0.0);
}

template <int KIND>
__global__ void __launch_bounds__(256) moments_leaves(int64_t nn, const float4* __restrict__ pts,
                                                      const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                                                      const int32_t* __restrict__ cc,
                                                      const int32_t* __restrict__ depth, double* __restrict__ sums,
                                                      MomentArgs m, const float4* __restrict__ centroid) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn || cc[i] != 0) return;
  Sums S = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  const int j0 = pb[i], j1 = pe[i];
  float alpha = 0.f;
  if (KIND == ATTR_VEC && m.axpy_r) alpha = (float)(*m.alpha);
  for (int j = j0; j < j1; ++j) {
    const float4 x = pts[j];
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
    }
    S.W += a;
    S.P[0] += a * (double)x.x;
    S.P[1] += a * (double)x.y;
    S.P[2] += a * (double)x.z;
    S.V[0] += v0;
    S.V[1] += v1;
    S.V[2] += v2;
  }
  store_sums(sums, i, S);
  write_record<KIND>(i, S, j1 - j0, pts[j0], depth[i], 0, 0, m.theta, centroid, m);
  if (KIND == ATTR_UNIT)
    for (int j = j0; j < j1; ++j) m.leaf_of_out[j] = (int32_t)i;
}

template <int KIND>
__global__ void __launch_bounds__(256) moments_level(int64_t i0, int64_t i1, const int32_t* __restrict__ pb,
                                                     const int32_t* __restrict__ pe, const int32_t* __restrict__ cb,
                                                     const int32_t* __restrict__ cc, const int32_t* __restrict__ topo,
                                                     const int32_t* __restrict__ smask, int depth, double* __restrict__ sums, MomentArgs m,
                                                     const float4* __restrict__ centroid) {
  const int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= i1) return;
  const int nc = cc[i];
  if (nc == 0) return;  // leaf: done by moments_leaves
  const int c0 = cb[i];
  Sums T = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  for (int c = c0; c < c0 + nc; ++c) {  // fixed child order ⇒ deterministic sums
    const double2* s = reinterpret_cast<const double2*>(sums + 8 * (int64_t)c);
    const double2 a = s[0], b = s[1], d = s[2], e = s[3];
    T.W += a.x;
    T.P[0] += a.y;
    T.P[1] += b.x;
    T.P[2] += b.y;
    T.V[0] += d.x;
    T.V[1] += d.y;
    T.V[2] += e.x;
  }
  store_sums(sums, i, T);
  write_record<KIND>(i, T, pe[i] - pb[i], make_float4(0, 0, 0, 0), depth, topo[i], smask[i], m.theta, centroid, m);
}

template <int KIND>
void launch_all(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  const int64_t nn = t->nn;
  moments_leaves<KIND><<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(nn, t->pts, t->pb, t->pe, t->cc, t->depth,
                                                                      t->sums, m, t->centroid);
  for (int l = t->depth_used - 1; l >= 0; --l) {
    const int64_t i0 = t->level_off[l], i1 = t->level_off[l + 1];
    moments_level<KIND><<<(unsigned)((i1 - i0 + 255) / 256), 256, 0, s>>>(i0, i1, t->pb, t->pe, t->cb, t->cc,
                                                                           t->topo, t->smask, l, t->sums, m,
                                                                           t->centroid);
  }
}

}  // namespace

wn_status build_moments(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  ProfScope ps(WN_PROF_MOMENTS, s, 1 + t->depth_used);
  switch (m.kind) {
    case ATTR_VEC: launch_all<ATTR_VEC>(t, m, s); break;
    case ATTR_SCALAR: launch_all<ATTR_SCALAR>(t, m, s); break;
    default: launch_all<ATTR_UNIT>(t, m, s); break;
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

}  // namespace wn
