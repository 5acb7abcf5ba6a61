// wn_ops.cuh — host wrappers of the small kernels in ops.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace wn {
void gather_vec(int64_t n, const int32_t* perm, const float* v, double scale, float4* out, cudaStream_t s);
void gather_vec_a(int64_t n, const int32_t* perm, const float* v, const float* a, float4* mu, float* as, float4* mua,
                  cudaStream_t s);
void gather_scal(int64_t n, const int32_t* perm, const float* v, float* out, cudaStream_t s);
void scatter_vec(int64_t n, const int32_t* perm, const float4* v, double scale, float* out, cudaStream_t s);
void normalize_queries(int64_t m, const float* q, const double xf[4], float4* out, cudaStream_t s);
void alpha_step(const double* part, int nblk, int64_t stride, double w, double* alpha, double* stats, cudaStream_t s);
void unit_normals(int64_t n, const float* mu, float* out, cudaStream_t s);
// s = ½ and Σs² partials of A(0) (WN_FLAG_MU_ZERO, iteration 1)
void s_half(int64_t n, float* s_out, double* part, cudaStream_t s);
float width_at(int k, int n, double w1, double w2);
}  // namespace wn
