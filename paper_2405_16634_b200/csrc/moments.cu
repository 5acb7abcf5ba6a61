// moments.cu — per-application representatives.
//
// PAPER.md:L371-L378 (§4.5, Eqs node-rep-loc / node-rep-vec): for attribute ν,
//     x_{B,ν} = Σ_{i∈B} |ν_i| x_i / Σ_{j∈B} |ν_j| ,   ν_B = Σ_{i∈B} ν_i .
// Readings: Σ|ν| = 0 ⇒ the node's unweighted centroid; a one-point node's rep is the
// point itself; |ν| is the Euclidean norm (vector) or |s| (scalar).
//
// B200 design: ONE launch per build.  A thread per leaf sums its points in fp64, writes the node's
// fp64 sums and its fp32 traversal record, then walks up: at each parent it bumps an arrival counter
// and the last-arriving child sums the parent's children IN CHILD ORDER (so the result is
// deterministic and independent of scheduling), writes the parent and continues.  Counters are
// reset by the finisher, so the tree carries zeroed counters between builds.  Traffic is O(N + Nn)
// (≈ 16 B/point read + 64 B/node fp64 sums + 32 B/node record); no per-level launches.
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
__device__ __forceinline__ void write_record(int i, const Sums& S, int cnt, float4 p0, int depth, int topo,
                                             float theta, const float4* __restrict__ centroid, NodeSet out,
                                             float4* centroid_out) {
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
      float4 c = centroid[i];
      rx = c.x; ry = c.y; rz = c.z;
    }
    R = make_float4(rx, ry, rz, thr_of(theta, depth));
  }
  if (out.L) out.L[i] = L;
  out.R[i] = R;
  if (KIND == ATTR_SCALAR)
    out.A[i] = make_float4((float)S.V[0], 0.f, 0.f, __int_as_float(topo));
  else
    out.A[i] = make_float4((float)S.V[0], (float)S.V[1], (float)S.V[2], __int_as_float(topo));
  if (KIND == ATTR_UNIT) centroid_out[i] = make_float4(R.x, R.y, R.z, 0.f);
}

template <int KIND>
__global__ void __launch_bounds__(256) moments_up(
    int64_t nn, const float4* __restrict__ pts, const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
    const int32_t* __restrict__ cb, const int32_t* __restrict__ cc, const int32_t* __restrict__ depth,
    const int32_t* __restrict__ parent, int32_t* __restrict__ arrive, double* __restrict__ sums,
    MomentArgs m, const float4* __restrict__ centroid) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn || cc[i] != 0) return;
  // ---- leaf: direct sums over its points ----
  Sums S = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  const int j0 = pb[i], j1 = pe[i];
  float alpha = 0.f;
  if (KIND == ATTR_VEC && m.axpy_r) alpha = (float)(*m.alpha);
  for (int j = j0; j < j1; ++j) {
    const float4 x = pts[j];
    double a, v0 = 0, v1 = 0, v2 = 0;
    if (KIND == ATTR_VEC) {
      float4 v = m.vec[j];
      if (m.axpy_r) {
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
  double* o = sums + 8 * i;
  o[0] = S.W; o[1] = S.P[0]; o[2] = S.P[1]; o[3] = S.P[2]; o[4] = S.V[0]; o[5] = S.V[1]; o[6] = S.V[2];
  write_record<KIND>((int)i, S, j1 - j0, pts[j0], depth[i], 8, m.theta, centroid, m.out, m.centroid_out);
  if (KIND == ATTR_UNIT)
    for (int j = j0; j < j1; ++j) m.leaf_of_out[j] = (int32_t)i;
  // ---- walk up: the last child to arrive finishes the parent ----
  int node = (int)i;
  while (true) {
    const int p = parent[node];
    if (p < 0) break;
    __threadfence();
    const int prev = atomicAdd(&arrive[p], 1);
    const int nc = cc[p];
    if (prev != nc - 1) break;
    arrive[p] = 0;
    __threadfence();
    const int c0 = cb[p];
    Sums T = {0.0, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    for (int c = c0; c < c0 + nc; ++c) {
      const double* s = sums + 8 * (int64_t)c;
      T.W += __ldcg(s + 0);
      T.P[0] += __ldcg(s + 1);
      T.P[1] += __ldcg(s + 2);
      T.P[2] += __ldcg(s + 3);
      T.V[0] += __ldcg(s + 4);
      T.V[1] += __ldcg(s + 5);
      T.V[2] += __ldcg(s + 6);
    }
    double* q = sums + 8 * (int64_t)p;
    q[0] = T.W; q[1] = T.P[0]; q[2] = T.P[1]; q[3] = T.P[2]; q[4] = T.V[0]; q[5] = T.V[1]; q[6] = T.V[2];
    const int topo = (c0 << 4) | (nc - 1);
    write_record<KIND>(p, T, pe[p] - pb[p], make_float4(0, 0, 0, 0), depth[p], topo, m.theta, centroid, m.out,
                       m.centroid_out);
    node = p;
  }
}

}  // namespace

wn_status build_moments(wn_tree_s* t, const MomentArgs& m, cudaStream_t s) {
  unsigned g = (unsigned)((t->nn + 255) / 256);
  ProfScope ps(WN_PROF_MOMENTS, s);
  switch (m.kind) {
    case ATTR_VEC:
      moments_up<ATTR_VEC><<<g, 256, 0, s>>>(t->nn, t->pts, t->pb, t->pe, t->cb, t->cc, t->depth, t->parent,
                                              t->arrive, t->sums, m, t->centroid);
      break;
    case ATTR_SCALAR:
      moments_up<ATTR_SCALAR><<<g, 256, 0, s>>>(t->nn, t->pts, t->pb, t->pe, t->cb, t->cc, t->depth,
                                                 t->parent, t->arrive, t->sums, m, t->centroid);
      break;
    default:
      moments_up<ATTR_UNIT><<<g, 256, 0, s>>>(t->nn, t->pts, t->pb, t->pe, t->cb, t->cc, t->depth, t->parent,
                                               t->arrive, t->sums, m, t->centroid);
      break;
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

}  // namespace wn
