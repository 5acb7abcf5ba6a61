// ops.cu — small fused elementwise / reduction kernels of the solver and the
// host orchestration of Alg. 3 with the grad step of Alg. 2 (L311-L321).
#include <cuda_runtime.h>

#include <cmath>

#include "wn_internal.cuh"
#include "wn_ops.cuh"

namespace wn {
namespace {

// caller order, input frame  →  sorted order, optionally scaled (fp64 product, one rounding)
__global__ void k_gather_vec(int64_t n, const int32_t* __restrict__ perm, const float* __restrict__ v, double scale,
                             float4* __restrict__ out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t j = perm[k];
  out[k] = make_float4((float)((double)v[3 * j] * scale), (float)((double)v[3 * j + 1] * scale),
                       (float)((double)v[3 * j + 2] * scale), 0.f);
}

__global__ void k_gather_vec_a(int64_t n, const int32_t* __restrict__ perm, const float* __restrict__ v,
                               const float* __restrict__ a, float4* __restrict__ mu, float* __restrict__ as,
                               float4* __restrict__ mua) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t j = perm[k];
  const float x = v[3 * j], y = v[3 * j + 1], z = v[3 * j + 2];
  mu[k] = make_float4(x, y, z, 0.f);
  if (a) {
    const double f = a[j];
    as[k] = a[j];
    mua[k] = make_float4((float)(x * f), (float)(y * f), (float)(z * f), 0.f);
  }
}

__global__ void k_gather_scal(int64_t n, const int32_t* __restrict__ perm, const float* __restrict__ v,
                              float* __restrict__ out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  out[k] = v[perm[k]];
}

__global__ void k_scatter_vec(int64_t n, const int32_t* __restrict__ perm, const float4* __restrict__ v, double scale,
                              float* __restrict__ out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t j = perm[k];
  const float4 x = v[k];
  out[3 * j] = (float)((double)x.x * scale);
  out[3 * j + 1] = (float)((double)x.y * scale);
  out[3 * j + 2] = (float)((double)x.z * scale);
}

// xn = (x − c)·scale in fp64, rounded once (the same expression as the tree build)
__global__ void k_normalize_queries(int64_t m, const float* __restrict__ q, double c0, double c1, double c2,
                                    double sc, float4* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  out[i] = make_float4((float)(__dsub_rn((double)q[3 * i], c0) * sc), (float)(__dsub_rn((double)q[3 * i + 1], c1) * sc),
                       (float)(__dsub_rn((double)q[3 * i + 2], c2) * sc), 0.f);
}

// α = Σr² / Σ(Ar)² from fixed-order block partials (0 if the denominator is 0).
// kAlphaBlocks blocks each sum a fixed stride of the partial slots (thread order, then a tree), publish
// their three sums, and the last block to finish (a ticket) adds the block sums in block order: the same
// order on every run and every rank.  alpha[0] = α, alpha[1 .. 3K] the block sums, alpha[3K + 1] the ticket.
constexpr int kAlphaThreads = 256;
__global__ void __launch_bounds__(kAlphaThreads) k_alpha(const double* __restrict__ part, int nblk, int64_t stride,
                                                         double w, double* alpha, double* stats) {
  __shared__ double sh[3][kAlphaThreads];
  __shared__ bool last;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int b = blockIdx.x * kAlphaThreads + threadIdx.x; b < nblk; b += kAlphaBlocks * kAlphaThreads)
    for (int c = 0; c < 3; ++c) acc[c] += part[c * stride + b];
  for (int c = 0; c < 3; ++c) sh[c][threadIdx.x] = acc[c];
  __syncthreads();
  for (int o = kAlphaThreads / 2; o; o >>= 1) {
    if (threadIdx.x < o)
      for (int c = 0; c < 3; ++c) sh[c][threadIdx.x] += sh[c][threadIdx.x + o];
    __syncthreads();
  }
  double* blk = alpha + 1;
  unsigned int* ticket = reinterpret_cast<unsigned int*>(alpha + 1 + 3 * kAlphaBlocks);
  if (threadIdx.x == 0) {
    for (int c = 0; c < 3; ++c) blk[c * kAlphaBlocks + blockIdx.x] = sh[c][0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == kAlphaBlocks - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double E = 0.0, rr = 0.0, qq = 0.0;
  for (int k = 0; k < kAlphaBlocks; ++k) {
    E += __ldcg(blk + k);
    rr += __ldcg(blk + kAlphaBlocks + k);
    qq += __ldcg(blk + 2 * kAlphaBlocks + k);
  }
  const double al = qq > 0.0 ? rr / qq : 0.0;
  *alpha = al;
  stats[0] = E; stats[1] = al; stats[2] = rr; stats[3] = qq; stats[4] = w;
  *ticket = 0u;  // ready for the next α (stream-ordered)
}

// s = ½ − A(0) = ½ for every query and the group partials Σ s² = 0.25 · (queries in the group) — exactly the
// values the A traversal's EPI_S epilogue produces for μ = 0 (every term 0), without the traversal
__global__ void k_s_half(int64_t n, float* __restrict__ s, double* __restrict__ part, int block) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) s[i] = 0.5f;
  if (i * block < n) {
    const int64_t cnt = n - i * block < block ? n - i * block : block;
    part[i] = 0.25 * (double)cnt;
  }
}

// final "Normalize" step of the pipeline figure: n_i = μ_i/|μ_i|, zero stays zero
__global__ void k_unit(int64_t n, const float* __restrict__ mu, float* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = mu[3 * i], y = mu[3 * i + 1], z = mu[3 * i + 2];
  const double l = sqrt(x * x + y * y + z * z);
  const double f = l > 0.0 ? 1.0 / l : 0.0;
  out[3 * i] = (float)(x * f);
  out[3 * i + 1] = (float)(y * f);
  out[3 * i + 2] = (float)(z * f);
}

inline unsigned g256(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void gather_vec(int64_t n, const int32_t* perm, const float* v, double scale, float4* out, cudaStream_t s) {
  k_gather_vec<<<g256(n), 256, 0, s>>>(n, perm, v, scale, out);
  count_launches(1);
}
void gather_vec_a(int64_t n, const int32_t* perm, const float* v, const float* a, float4* mu, float* as, float4* mua,
                  cudaStream_t s) {
  k_gather_vec_a<<<g256(n), 256, 0, s>>>(n, perm, v, a, mu, as, mua);
  count_launches(1);
}
void gather_scal(int64_t n, const int32_t* perm, const float* v, float* out, cudaStream_t s) {
  k_gather_scal<<<g256(n), 256, 0, s>>>(n, perm, v, out);
  count_launches(1);
}
void scatter_vec(int64_t n, const int32_t* perm, const float4* v, double scale, float* out, cudaStream_t s) {
  k_scatter_vec<<<g256(n), 256, 0, s>>>(n, perm, v, scale, out);
  count_launches(1);
}
void normalize_queries(int64_t m, const float* q, const double xf[4], float4* out, cudaStream_t s) {
  k_normalize_queries<<<g256(m), 256, 0, s>>>(m, q, xf[0], xf[1], xf[2], xf[3], out);
  count_launches(1);
}
void alpha_step(const double* part, int nblk, int64_t stride, double w, double* alpha, double* stats, cudaStream_t s) {
  ProfScope ps(WN_PROF_OTHER, s);
  k_alpha<<<kAlphaBlocks, kAlphaThreads, 0, s>>>(part, nblk, stride, w, alpha, stats);
  count_launches(1);
}
void s_half(int64_t n, float* s_out, double* part, cudaStream_t s) {
  k_s_half<<<g256(n), 256, 0, s>>>(n, s_out, part, kPartQ);
  count_launches(1);
}
void unit_normals(int64_t n, const float* mu, float* out, cudaStream_t s) {
  k_unit<<<g256(n), 256, 0, s>>>(n, mu, out);
  count_launches(1);
}

// Alg. 3 width schedule; n = 1 ⇒ w1; handed to the kernels as fp32
float width_at(int k, int n, double w1, double w2) {
  if (n == 1) return (float)w1;
  return (float)(w2 * (double)(n - k) / (double)(n - 1) + w1 * (double)(k - 1) / (double)(n - 1));
}

}  // namespace wn
