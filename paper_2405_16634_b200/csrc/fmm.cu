// fmm.cu — fast multipole evaluation of the winding-number operators (the paper's future
// work, §6.3 and L409 — an extension, not the paper's Alg. 4 treecode).
//
// One potential carries all three operators (Φ(r) = 1/(4π|r|)):
//     V(y) = Σ_j [ q_j Φ(y − x_j) + ν_j·∇Φ(y − x_j) ]
// A(ν) = V for dipoles ν, G(ν) = −∇V for dipoles (L266), Aᵀ(s) = −∇V for charges q = s
// (L316).  Cells are the octree's nodes (cube centres, radius = half-diagonal); an FMM leaf is a node with
// no children or at most `leaf` (≤ 32) points.  Cartesian Taylor expansions of total degree ≤ p (≤ 6):
//   P2M  M_β = Σ_j [ q_j (−1)^|β| (x_j−c)^β/β! + Σ_k ν_jk (−1)^(|β|−1) (x_j−c)^(β−e_k)/(β−e_k)! ]
//   M2M  M'_β = Σ_{γ≤β} M_γ (c'−c)^(β−γ)/(β−γ)!        M2L  L_γ += Σ_β M_β ∂^(β+γ)Φ(c_t − c_s)
//   L2L  L'_δ = Σ_{γ≥δ} L_γ (c'−c)^(γ−δ)/(γ−δ)!        L2P  V(y) = Σ_γ L_γ (y−c)^γ/γ!  (and ∇V)
// with ∂^δ(1/|R|) = δ! b_δ, |δ| |R|² b_δ = −(2|δ|−1) Σ_i R_i b_(δ−e_i) − (|δ|−1) Σ_i b_(δ−2e_i).
// A cell pair is well separated — one M2L — iff |c_t − c_s| θ_f > r_t + r_s and |c_t − c_s| − r_t − r_s > w
// (every point pair beyond the smoothing cutoff, where the expansion is of the exact kernel); two leaves
// otherwise interact directly (P2P, cutoff r < w decided in fp32 as everywhere, R-prec); else the larger
// cell (the target on ties) is split.  All expansion arithmetic is fp64.
//
// B200 mapping: the interaction lists come from a breadth-first dual traversal on the GPU (one thread per
// cell pair per level, appends by atomics), sorted by (target, source) so that every sum runs in a fixed
// order; P2M / M2M / M2L / L2L run one warp per cell with lanes over the expansion coefficients (the
// derivative tensor of a pair is built degree by degree in shared memory); L2P + P2P one warp per leaf with
// one lane per target point.  The test oracle implements the same algorithm independently in plain fp64 C.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "wn_internal.cuh"

namespace wn {

constexpr int kFmmMaxP = 6;
constexpr int kFmmMaxDeg = 2 * kFmmMaxP;
constexpr int kFmmMaxN = (kFmmMaxP + 1) * (kFmmMaxP + 2) * (kFmmMaxP + 3) / 6;      // 84
constexpr int kFmmMaxT = (kFmmMaxDeg + 1) * (kFmmMaxDeg + 2) * (kFmmMaxDeg + 3) / 6;  // 455
constexpr int kFmmLut = kFmmMaxDeg + 1;

// multi-indices by total degree, then (a, b, c) descending lexicographically — the first count(p) of them
// are exactly the indices of degree ≤ p (the oracle's order)
__constant__ signed char c_mi[kFmmMaxT][3];
__constant__ short c_lut[kFmmLut][kFmmLut][kFmmLut];
__constant__ double c_fact[kFmmMaxDeg + 2];

static int fmm_count(int p) { return (p + 1) * (p + 2) * (p + 3) / 6; }

static wn_status fmm_tables() {
  static bool done = false;
  if (done) return WN_OK;
  signed char mi[kFmmMaxT][3];
  static short lut[kFmmLut][kFmmLut][kFmmLut];
  double fact[kFmmMaxDeg + 2];
  for (int a = 0; a < kFmmLut; ++a)
    for (int b = 0; b < kFmmLut; ++b)
      for (int c = 0; c < kFmmLut; ++c) lut[a][b][c] = -1;
  int n = 0;
  for (int deg = 0; deg <= kFmmMaxDeg; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b) {
        const int c = deg - a - b;
        mi[n][0] = (signed char)a;
        mi[n][1] = (signed char)b;
        mi[n][2] = (signed char)c;
        lut[a][b][c] = (short)n++;
      }
  fact[0] = 1.0;
  for (int k = 1; k < kFmmMaxDeg + 2; ++k) fact[k] = fact[k - 1] * k;
  WN_CUDA(cudaMemcpyToSymbol(c_mi, mi, sizeof(mi)));
  WN_CUDA(cudaMemcpyToSymbol(c_lut, lut, sizeof(lut)));
  WN_CUDA(cudaMemcpyToSymbol(c_fact, fact, sizeof(fact)));
  done = true;
  return WN_OK;
}

__device__ __forceinline__ int fmm_at(int a, int b, int c, int P) {
  if (a < 0 || b < 0 || c < 0 || a + b + c > P) return -1;
  return c_lut[a][b][c];
}

// x^a / a! for a ≤ p (per axis), then a monomial is the product of three of them
__device__ __forceinline__ void fmm_pows(double x, int p, double* o) {
  o[0] = 1.0;
  for (int a = 1; a <= p; ++a) o[a] = o[a - 1] * x / a;
}

struct FmmGeom {
  const int32_t *pb, *pe, *cb, *cc, *depth, *parent;
  const double* ctr;   // nn × 3
  const double* rad;   // nn
  const uint8_t* leaf; // FMM leaf flag
};

// cube centre and half-diagonal of every node from its first sorted point (the tree build's quantization,
// fp64, exact powers of two), the FMM leaf flag, and whether a node is above every FMM leaf (active)
__global__ void k_fmm_geom(int64_t nn, int D, int leafsz, const float4* __restrict__ pts,
                           const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                           const int32_t* __restrict__ cc, const int32_t* __restrict__ depth,
                           double* __restrict__ ctr, double* __restrict__ rad, uint8_t* __restrict__ leaf) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const float4 x = pts[pb[i]];
  const int d = depth[i];
  const double cells = ldexp(1.0, D - 1), qmax = (double)((1u << D) - 1u);
  const double edge = ldexp(1.0, 1 - d);
  const float xs[3] = {x.x, x.y, x.z};
  for (int a = 0; a < 3; ++a) {
    double v = floor(((double)xs[a] + 1.0) * cells);
    v = v < 0.0 ? 0.0 : (v > qmax ? qmax : v);
    const uint32_t q = (uint32_t)v;
    const uint32_t cell = d == 0 ? 0u : q >> (D - d);
    ctr[3 * i + a] = -1.0 + ((double)cell + 0.5) * edge;
  }
  rad[i] = sqrt(3.0) * 0.5 * edge;
  leaf[i] = (cc[i] == 0 || pe[i] - pb[i] <= leafsz) ? 1 : 0;
}

// P2M: one warp per FMM leaf, lanes over the coefficients β
template <int DIM>
__global__ void k_fmm_p2m(int64_t m, const int32_t* __restrict__ list, FmmGeom g, const float4* __restrict__ pts,
                          const float4* __restrict__ vec, const float* __restrict__ scal, int p,
                          double* __restrict__ M) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int64_t id = list[k];
  const int np = (p + 1) * (p + 2) * (p + 3) / 6;
  const double c0 = g.ctr[3 * id], c1 = g.ctr[3 * id + 1], c2 = g.ctr[3 * id + 2];
  for (int b = lane; b < np; b += 32) {
    const int b0 = c_mi[b][0], b1 = c_mi[b][1], b2 = c_mi[b][2], deg = b0 + b1 + b2;
    double acc = 0.0;
    for (int j = g.pb[id]; j < g.pe[id]; ++j) {
      const float4 x = pts[j];
      double px[kFmmMaxP + 1], py[kFmmMaxP + 1], pz[kFmmMaxP + 1];
      fmm_pows((double)x.x - c0, p, px);
      fmm_pows((double)x.y - c1, p, py);
      fmm_pows((double)x.z - c2, p, pz);
      if (DIM == 1) {
        acc += (double)scal[j] * ((deg & 1) ? -1.0 : 1.0) * (px[b0] * py[b1] * pz[b2]);
      } else {
        const float4 v = vec[j];
        const double sg = ((deg - 1) & 1) ? -1.0 : 1.0;
        if (b0 > 0) acc += (double)v.x * sg * (px[b0 - 1] * py[b1] * pz[b2]);
        if (b1 > 0) acc += (double)v.y * sg * (px[b0] * py[b1 - 1] * pz[b2]);
        if (b2 > 0) acc += (double)v.z * sg * (px[b0] * py[b1] * pz[b2 - 1]);
      }
    }
    M[id * np + b] = acc;
  }
}

// M2M: one warp per internal active node of one level, its children in order
__global__ void k_fmm_m2m(int64_t m, const int32_t* __restrict__ list, FmmGeom g, int p, double* __restrict__ M) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int64_t id = list[k];
  const int np = (p + 1) * (p + 2) * (p + 3) / 6;
  for (int b = lane; b < np; b += 32) {
    const int b0 = c_mi[b][0], b1 = c_mi[b][1], b2 = c_mi[b][2];
    double acc = 0.0;
    for (int c = g.cb[id]; c < g.cb[id] + g.cc[id]; ++c) {
      double px[kFmmMaxP + 1], py[kFmmMaxP + 1], pz[kFmmMaxP + 1];  // (c' − c): parent − child
      fmm_pows(g.ctr[3 * id] - g.ctr[3 * c], p, px);
      fmm_pows(g.ctr[3 * id + 1] - g.ctr[3 * c + 1], p, py);
      fmm_pows(g.ctr[3 * id + 2] - g.ctr[3 * c + 2], p, pz);
      const double* Mc = M + (int64_t)c * np;
      for (int g0 = 0; g0 <= b0; ++g0)
        for (int g1 = 0; g1 <= b1; ++g1)
          for (int g2 = 0; g2 <= b2; ++g2) acc += Mc[c_lut[g0][g1][g2]] * (px[b0 - g0] * py[b1 - g1] * pz[b2 - g2]);
    }
    M[id * np + b] = acc;
  }
}

// breadth-first dual traversal, one level of cell pairs: the oracle's fmm_dual decisions, appended by atomics
__global__ void k_fmm_dual(int64_t m, const int2* __restrict__ in, FmmGeom g, double theta, double w,
                           int2* __restrict__ next, unsigned long long* __restrict__ cnt, int64_t cap_next,
                           uint64_t* __restrict__ m2l, int64_t cap_m2l, uint64_t* __restrict__ p2p, int64_t cap_p2p) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int T = in[k].x, S = in[k].y;
  const double dx = g.ctr[3 * T] - g.ctr[3 * S], dy = g.ctr[3 * T + 1] - g.ctr[3 * S + 1],
               dz = g.ctr[3 * T + 2] - g.ctr[3 * S + 2];
  const double d = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  const double rt = g.rad[T], rs = g.rad[S];
  const uint64_t key = ((uint64_t)(uint32_t)T << 32) | (uint32_t)S;
  if (__dmul_rn(d, theta) > __dadd_rn(rt, rs) && __dsub_rn(__dsub_rn(d, rt), rs) > w) {
    const unsigned long long i = atomicAdd(cnt + 1, 1ull);
    if ((int64_t)i < cap_m2l) m2l[i] = key;
    return;
  }
  const bool lt = g.leaf[T], ls = g.leaf[S];
  if (lt && ls) {
    const unsigned long long i = atomicAdd(cnt + 2, 1ull);
    if ((int64_t)i < cap_p2p) p2p[i] = key;
    return;
  }
  const bool split_t = ls || (!lt && rt >= rs);
  const int c0 = split_t ? g.cb[T] : g.cb[S], nc = split_t ? g.cc[T] : g.cc[S];
  const unsigned long long i = atomicAdd(cnt, (unsigned long long)nc);
  for (int c = 0; c < nc; ++c)
    if ((int64_t)(i + c) < cap_next) next[i + c] = split_t ? make_int2(c0 + c, S) : make_int2(T, c0 + c);
}

// CSR offsets of a sorted (target << 32 | source) key list: off[t] = first key with target ≥ t
__global__ void k_fmm_csr(int64_t nn, const uint64_t* __restrict__ keys, int64_t nk, int32_t* __restrict__ off) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > nn) return;
  const uint64_t target = (uint64_t)t << 32;
  int64_t lo = 0, hi = nk;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  off[t] = (int32_t)lo;
}

// M2L: one warp per target cell with a non-empty list; per source cell the derivative tensor of
// R = c_t − c_s is built degree by degree in shared memory (scaled to T_δ = ∂^δΦ on the fly), the source's
// multipole coefficients are staged there too, then lane γ adds Σ_β M_β T_(β+γ)
// index of a multi-index in the degree-then-lexicographic order, arithmetically (no divergent table lookups)
__device__ __forceinline__ int mi_index(int a, int b, int c) {
  const int n = a + b + c, na = n - a;
  return n * (n + 1) * (n + 2) / 6 + na * (na + 1) / 2 + (na - b);
}
__device__ __forceinline__ double fact_small(int k) {  // k! for k ≤ 12, exact in fp64
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return f;
}
constexpr int kFmmWarps = 2;  // (the per-block index tables share the 48 KB of static shared memory)
// M2L: warps stride over the target cells (a resident grid: the index tables below are built once per block);
// per source cell of a target's list the derivative tensor of R = c_t − c_s is built degree by degree in
// shared memory (each entry from its ≤ 6 lower-degree dependencies, looked up in a table), scaled to
// T_δ = ∂^δΦ, the source's coefficients staged beside it, then lane γ adds Σ_β M_β T_(β+γ) through a
// (β, γ) → β + γ index table
__global__ void __launch_bounds__(32 * kFmmWarps) k_fmm_m2l(int64_t nn, const int32_t* __restrict__ off,
                                                            const uint64_t* __restrict__ keys, FmmGeom g, int p,
                                                            const double* __restrict__ M, double* __restrict__ L) {
  __shared__ double sT[kFmmWarps][kFmmMaxT];
  __shared__ double sB[kFmmWarps][kFmmMaxT];
  __shared__ double sM[kFmmWarps][kFmmMaxN];
  __shared__ double sFac[kFmmMaxT];          // δ!/(4π)
  __shared__ short sDep[kFmmMaxT][6];        // δ − e_i (i = 0..2), δ − 2e_i (i = 0..2), or −1
  __shared__ short sSum[kFmmMaxN][kFmmMaxN]; // index of β + γ
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int np = (p + 1) * (p + 2) * (p + 3) / 6, P = 2 * p, nP = (P + 1) * (P + 2) * (P + 3) / 6;
  WN_DCHECK(p >= 1 && p <= kFmmMaxP, "M2L degree");
  for (int e = threadIdx.x; e < nP; e += blockDim.x) {
    const int d0 = c_mi[e][0], d1 = c_mi[e][1], d2 = c_mi[e][2];
    sFac[e] = c_fact[d0] * c_fact[d1] * c_fact[d2] * 0.0795774715459476679;
    sDep[e][0] = d0 > 0 ? (short)mi_index(d0 - 1, d1, d2) : (short)-1;
    sDep[e][1] = d1 > 0 ? (short)mi_index(d0, d1 - 1, d2) : (short)-1;
    sDep[e][2] = d2 > 0 ? (short)mi_index(d0, d1, d2 - 1) : (short)-1;
    sDep[e][3] = d0 > 1 ? (short)mi_index(d0 - 2, d1, d2) : (short)-1;
    sDep[e][4] = d1 > 1 ? (short)mi_index(d0, d1 - 2, d2) : (short)-1;
    sDep[e][5] = d2 > 1 ? (short)mi_index(d0, d1, d2 - 2) : (short)-1;
  }
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int be = e / np, ga = e % np;
    sSum[be][ga] = (short)mi_index(c_mi[be][0] + c_mi[ga][0], c_mi[be][1] + c_mi[ga][1], c_mi[be][2] + c_mi[ga][2]);
  }
  __syncthreads();
  double* b = sB[wp];
  double* Tt = sT[wp];
  double* Ms = sM[wp];
  const int64_t nw = (int64_t)gridDim.x * kFmmWarps;
  for (int64_t T = (int64_t)blockIdx.x * kFmmWarps + wp; T < nn; T += nw) {
    const int k0 = off[T], k1 = off[T + 1];
    if (k0 == k1) continue;
    double acc[3] = {0.0, 0.0, 0.0};  // γ = lane, lane + 32, lane + 64
    for (int k = k0; k < k1; ++k) {
      const int S = (int)(uint32_t)keys[k];
      WN_DCHECK(S >= 0 && S < nn && (int64_t)(keys[k] >> 32) == T, "M2L list entry");
      const double R[3] = {g.ctr[3 * T] - g.ctr[3 * S], g.ctr[3 * T + 1] - g.ctr[3 * S + 1],
                           g.ctr[3 * T + 2] - g.ctr[3 * S + 2]};
      const double r2 = R[0] * R[0] + R[1] * R[1] + R[2] * R[2];
      __syncwarp();
      for (int e = lane; e < np; e += 32) Ms[e] = M[(int64_t)S * np + e];
      if (lane == 0) {
        b[0] = 1.0 / sqrt(r2);
        Tt[0] = b[0] * sFac[0];
      }
      __syncwarp();
      for (int n = 1; n <= P; ++n) {  // the b_δ of degree n from degrees n − 1 and n − 2
        const int lo = n * (n + 1) * (n + 2) / 6, cntn = (n + 1) * (n + 2) / 2;
        const double c1 = 2.0 * n - 1.0, c2 = n - 1.0, inv = 1.0 / (n * r2);
        for (int e = lane; e < cntn; e += 32) {
          const int idx = lo + e;
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int j1 = sDep[idx][i], j2 = sDep[idx][3 + i];
            if (j1 >= 0) s -= c1 * R[i] * b[j1];
            if (j2 >= 0) s -= c2 * b[j2];
          }
          const double bv = s * inv;
          b[idx] = bv;
          Tt[idx] = bv * sFac[idx];  // ∂^δΦ
        }
        __syncwarp();
      }
      for (int q = 0; q < 3; ++q) {
        const int gi = lane + 32 * q;
        if (gi >= np) break;
        double a = 0.0;
        for (int be = 0; be < np; ++be) a += Ms[be] * Tt[sSum[be][gi]];
        acc[q] += a;
      }
    }
    for (int q = 0; q < 3; ++q) {
      const int gi = lane + 32 * q;
      if (gi < np) L[T * np + gi] = acc[q];
    }
  }
}

// L2L: one warp per child of an internal active node of one level: L_c += shift of the parent's L
__global__ void k_fmm_l2l(int64_t m, const int32_t* __restrict__ list, FmmGeom g, int p, double* __restrict__ L) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int64_t c = list[k];  // a node whose parent is an internal active node
  const int64_t par = g.parent[c];
  const int np = (p + 1) * (p + 2) * (p + 3) / 6;
  double px[kFmmMaxP + 1], py[kFmmMaxP + 1], pz[kFmmMaxP + 1];  // (c' − c): child − parent
  fmm_pows(g.ctr[3 * c] - g.ctr[3 * par], p, px);
  fmm_pows(g.ctr[3 * c + 1] - g.ctr[3 * par + 1], p, py);
  fmm_pows(g.ctr[3 * c + 2] - g.ctr[3 * par + 2], p, pz);
  const double* Lp = L + par * np;
  for (int dl = lane; dl < np; dl += 32) {
    const int d0 = c_mi[dl][0], d1 = c_mi[dl][1], d2 = c_mi[dl][2];
    double acc = 0.0;
    for (int gi = 0; gi < np; ++gi) {
      const int g0 = c_mi[gi][0] - d0, g1 = c_mi[gi][1] - d1, g2 = c_mi[gi][2] - d2;
      if (g0 < 0 || g1 < 0 || g2 < 0) continue;
      acc += Lp[gi] * (px[g0] * py[g1] * pz[g2]);
    }
    L[c * np + dl] += acc;
  }
}

// L2P + P2P: one warp per FMM leaf, one lane per target point; V and ∇V in fp64, output per op
template <int DIM>
__global__ void k_fmm_eval(int64_t m, const int32_t* __restrict__ list, FmmGeom g, const int32_t* __restrict__ off,
                           const uint64_t* __restrict__ keys, const float4* __restrict__ pts,
                           const float4* __restrict__ vec, const float* __restrict__ scal, int p,
                           const double* __restrict__ L, float w2f, int op, const int32_t* __restrict__ out_map,
                           float* __restrict__ out, float4* __restrict__ out4, double scale) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int64_t T = list[k];
  const int np = (p + 1) * (p + 2) * (p + 3) / 6;
  // a leaf holds ≤ `leaf` ≤ 32 points unless it is a depth-D cell of duplicates: chunks of 32 targets
  for (int i0 = g.pb[T]; i0 < g.pe[T]; i0 += 32) {
    const int i = i0 + lane;
    const bool valid = i < g.pe[T];
    double V = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      y = pts[i];
      double px[kFmmMaxP + 1], py[kFmmMaxP + 1], pz[kFmmMaxP + 1];
      fmm_pows((double)y.x - g.ctr[3 * T], p, px);
      fmm_pows((double)y.y - g.ctr[3 * T + 1], p, py);
      fmm_pows((double)y.z - g.ctr[3 * T + 2], p, pz);
      const double* Lt = L + T * np;
      for (int gi = 0; gi < np; ++gi) {
        const int g0 = c_mi[gi][0], g1 = c_mi[gi][1], g2 = c_mi[gi][2];
        const double l = Lt[gi];
        V += l * (px[g0] * py[g1] * pz[g2]);
        if (g0 > 0) gx += l * (px[g0 - 1] * py[g1] * pz[g2]);
        if (g1 > 0) gy += l * (px[g0] * py[g1 - 1] * pz[g2]);
        if (g2 > 0) gz += l * (px[g0] * py[g1] * pz[g2 - 1]);
      }
    }
    // P2P: fp32 pair terms (rsqrt, as the treecode's near field), summed per source leaf in fp32 and across
    // leaves in fp64; the cutoff decided in fp32 on d = x_j − y (R-prec)
    for (int kk = off[T]; kk < off[T + 1]; ++kk) {
      const int S = (int)(uint32_t)keys[kk];
      float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
      for (int j = g.pb[S]; j < g.pe[S]; ++j) {
        const float4 x = pts[j];
        const float dxf = x.x - y.x, dyf = x.y - y.y, dzf = x.z - y.z;
        const float d2 = __fmaf_rn(dxf, dxf, __fmaf_rn(dyf, dyf, __fmul_rn(dzf, dzf)));
        const bool live = valid && !(d2 < w2f);
        const float inv = rsqrtf(live ? d2 : __int_as_float(0x7f800000));  // a dead pair: rsqrt(+inf) = 0
        const float inv3 = inv * inv * inv;
        // d = y − x = −(dxf, dyf, dzf)
        if (DIM == 1) {  // q Φ(d): V += q/(4πr), ∇V += −q d/(4πr³) = q (x − y)/(4πr³)
          const float q = scal[j];
          v0 = fmaf(q, inv, v0);
          v1 = fmaf(q * inv3, dxf, v1);
          v2 = fmaf(q * inv3, dyf, v2);
          v3 = fmaf(q * inv3, dzf, v3);
        } else {  // V −= (d·ν)/(4πr³);  ∇V += 3(d·ν)d/(4πr⁵) − ν/(4πr³)
          const float4 v = vec[j];
          const float dn = -(dxf * v.x + dyf * v.y + dzf * v.z);
          const float t5 = 3.0f * dn * inv3 * inv * inv;
          v0 = fmaf(-dn, inv3, v0);
          v1 = fmaf(-t5, dxf, fmaf(-v.x, inv3, v1));
          v2 = fmaf(-t5, dyf, fmaf(-v.y, inv3, v2));
          v3 = fmaf(-t5, dzf, fmaf(-v.z, inv3, v3));
        }
      }
      const double k4 = 0.0795774715459476679;
      V += k4 * v0;
      gx += k4 * v1;
      gy += k4 * v2;
      gz += k4 * v3;
    }
    if (!valid) continue;
    if (out4) {  // the solver's sorted buffers, unscaled: V in .x (A), or −∇V (G, Aᵀ)
      out4[i] = op == OP_A ? make_float4((float)V, 0.f, 0.f, 0.f) : make_float4((float)-gx, (float)-gy, (float)-gz, 0.f);
      continue;
    }
    const int64_t o = out_map ? (int64_t)out_map[i] : i;
    if (op == OP_A) {
      out[o] = (float)(V * scale);
    } else {  // G = −∇V (dipoles), Aᵀ = −∇V (charges)
      out[3 * o] = (float)(-gx * scale);
      out[3 * o + 1] = (float)(-gy * scale);
      out[3 * o + 2] = (float)(-gz * scale);
    }
  }
}

__global__ void k_fmm_flag(int64_t nn, const uint8_t* __restrict__ leaf, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ depth, int mode, int level, uint32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const bool active = parent[i] < 0 || !leaf[parent[i]];  // no FMM leaf above it (the leaf test is monotone)
  bool f = false;
  if (mode == 0) f = active && leaf[i];                                    // the FMM leaves
  else if (mode == 1) f = active && !leaf[i] && depth[i] == level;        // internal active nodes of a level
  else f = active && parent[i] >= 0 && depth[i] == level;                  // active children at a level
  flag[i] = f ? 1u : 0u;
}

__global__ void k_fmm_compact(int64_t nn, const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                              int32_t* __restrict__ list) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nn && flag[i]) list[pos[i]] = (int32_t)i;
}

// exclusive scan helper of tree_build.cu (uint32)
wn_status fmm_scan(const uint32_t* in, uint32_t* out, int64_t m, uint32_t* total, cudaStream_t s);

static inline unsigned g256(int64_t n) { return (unsigned)((n + 255) / 256); }
static inline unsigned gwarps(int64_t n, int wpb) { return (unsigned)((n + wpb - 1) / wpb); }

void fmm_plan_free(FmmPlan& F) {
  for (void* q : F.owned) cudaFreeAsync(q, 0);
  F = FmmPlan();
}

// The per-tree FMM plan (geometry, node lists, sorted interaction lists, expansion scratch) for
// (p, θ_f, leaf, separation width wsep): built once — host-synchronizing, never inside a graph capture —
// and reused by every fmm_run with a cutoff w ≤ wsep (every expanded pair stays beyond the cutoff).
wn_status fmm_plan(wn_tree_s* t, int p, double theta, int leafsz, float wsep, cudaStream_t s) {
  if (p < 1 || p > kFmmMaxP) return set_error(WN_ERR_ARG, "FMM degree must be in 1..6");
  if (leafsz < 1 || leafsz > 32) return set_error(WN_ERR_ARG, "FMM leaf size must be in 1..32");
  if (!(theta > 0.0)) return set_error(WN_ERR_ARG, "FMM separation must be > 0");
  FmmPlan& F = t->fmm;
  if (F.ready && F.p == p && F.theta == theta && F.leaf == leafsz && F.wsep == wsep) return WN_OK;
  invalidate_graph(t);  // a cached graph may hold the old plan's buffers
  WN_CUDA(cudaStreamSynchronize(s));
  fmm_plan_free(F);
  WN_TRY(fmm_tables());
  const int64_t nn = t->nn;
  const int np = fmm_count(p);
  std::vector<void*> tmpv;
  struct Tmp {
    std::vector<void*>& h;
    cudaStream_t s;
    ~Tmp() {
      for (void* q : h) cudaFreeAsync(q, s);
    }
  } tmp_rel{tmpv, s};
  auto alloc = [&](auto** ptr, size_t bytes, bool keep) -> wn_status {
    cudaError_t e = cudaMallocAsync((void**)ptr, std::max<size_t>(bytes, 8), s);
    if (e != cudaSuccess) return cuda_status(e, "FMM scratch");
    (keep ? F.owned : tmpv).push_back((void*)*ptr);
    return WN_OK;
  };
  WN_TRY(alloc(&F.ctr, nn * 3 * sizeof(double), true));
  WN_TRY(alloc(&F.rad, nn * sizeof(double), true));
  WN_TRY(alloc(&F.leaf_flag, nn, true));
  WN_TRY(alloc(&F.M, (size_t)nn * np * sizeof(double), true));
  WN_TRY(alloc(&F.L, (size_t)nn * np * sizeof(double), true));
  k_fmm_geom<<<g256(nn), 256, 0, s>>>(nn, t->D, leafsz, t->pts, t->pb, t->pe, t->cc, t->depth, F.ctr, F.rad,
                                       F.leaf_flag);
  FmmGeom g{t->pb, t->pe, t->cb, t->cc, t->depth, t->parent, F.ctr, F.rad, F.leaf_flag};
  count_launches(1);
  // node lists: FMM leaves, internal active nodes per level, active non-root nodes per level
  uint32_t *flag = nullptr, *pos = nullptr;
  WN_TRY(alloc(&flag, (nn + 1) * sizeof(uint32_t), false));
  WN_TRY(alloc(&pos, (nn + 1) * sizeof(uint32_t), false));
  auto make_list = [&](int mode, int level, int32_t** list, int64_t* m) -> wn_status {
    k_fmm_flag<<<g256(nn), 256, 0, s>>>(nn, F.leaf_flag, t->parent, t->depth, mode, level, flag);
    WN_TRY(fmm_scan(flag, pos, nn, pos + nn, s));
    uint32_t c = 0;
    WN_CUDA(cudaMemcpyAsync(&c, pos + nn, sizeof(c), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    *m = c;
    WN_TRY(alloc(list, (size_t)std::max<uint32_t>(c, 1) * sizeof(int32_t), true));
    k_fmm_compact<<<g256(nn), 256, 0, s>>>(nn, flag, pos, *list);
    count_launches(2);
    return WN_OK;
  };
  WN_TRY(make_list(0, 0, &F.leaves, &F.nleaves));
  const int D = t->depth_used;
  F.inner.assign(D + 1, nullptr);
  F.kids.assign(D + 1, nullptr);
  F.ninner.assign(D + 1, 0);
  F.nkids.assign(D + 1, 0);
  for (int l = 0; l <= D; ++l) {
    WN_TRY(make_list(1, l, &F.inner[l], &F.ninner[l]));
    WN_TRY(make_list(2, l, &F.kids[l], &F.nkids[l]));
  }
  // interaction lists: breadth-first dual traversal from (root, root)
  unsigned long long* cnt = nullptr;
  WN_TRY(alloc(&cnt, 3 * sizeof(unsigned long long), false));
  int64_t cap_f = std::max<int64_t>(1024, 4 * nn), cap_m = std::max<int64_t>(1024, 16 * nn),
          cap_p = std::max<int64_t>(1024, 4 * nn);
  int2 *fa = nullptr, *fb = nullptr;
  uint64_t *m2l = nullptr, *p2p = nullptr;
  WN_TRY(alloc(&fa, cap_f * sizeof(int2), false));
  WN_TRY(alloc(&fb, cap_f * sizeof(int2), false));
  WN_TRY(alloc(&m2l, cap_m * sizeof(uint64_t), false));
  WN_TRY(alloc(&p2p, cap_p * sizeof(uint64_t), false));
  const int2 root = make_int2(0, 0);
  WN_CUDA(cudaMemcpyAsync(fa, &root, sizeof(root), cudaMemcpyHostToDevice, s));
  // a buffer that overflows during a level is regrown (contents kept) and the level runs again
  auto grow = [&](auto** buf, int64_t* cap, int64_t need, int64_t keep, size_t elt) -> wn_status {
    const int64_t nc = std::max<int64_t>(need + need / 2, 2 * *cap);
    void* nb = nullptr;
    WN_TRY(alloc(&nb, (size_t)nc * elt, false));
    if (keep > 0) WN_CUDA(cudaMemcpyAsync(nb, *buf, (size_t)keep * elt, cudaMemcpyDeviceToDevice, s));
    *buf = reinterpret_cast<std::remove_reference_t<decltype(**buf)>*>(nb);
    *cap = nc;
    return WN_OK;
  };
  unsigned long long h[3] = {1, 0, 0};  // frontier size, M2L and P2P counts so far
  while (h[0] > 0) {
    const unsigned long long nf = h[0], m0 = h[1], p0 = h[2];
    for (;;) {
      unsigned long long start[3] = {0, m0, p0};
      WN_CUDA(cudaMemcpyAsync(cnt, start, sizeof(start), cudaMemcpyHostToDevice, s));
      k_fmm_dual<<<g256((int64_t)nf), 256, 0, s>>>((int64_t)nf, fa, g, theta, (double)wsep, fb, cnt, cap_f, m2l,
                                                   cap_m, p2p, cap_p);
      count_launches(1);
      WN_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
      WN_CUDA(cudaStreamSynchronize(s));
      const bool of = (int64_t)h[0] > cap_f, om = (int64_t)h[1] > cap_m, op_ = (int64_t)h[2] > cap_p;
      if (!of && !om && !op_) break;
      if (of) WN_TRY(grow(&fb, &cap_f, (int64_t)h[0], 0, sizeof(int2)));
      if (om) WN_TRY(grow(&m2l, &cap_m, (int64_t)h[1], (int64_t)m0, sizeof(uint64_t)));
      if (op_) WN_TRY(grow(&p2p, &cap_p, (int64_t)h[2], (int64_t)p0, sizeof(uint64_t)));
      if (of) {  // keep the two frontier buffers the same size
        int2* na = nullptr;
        WN_TRY(alloc(&na, (size_t)cap_f * sizeof(int2), false));
        WN_CUDA(cudaMemcpyAsync(na, fa, (size_t)nf * sizeof(int2), cudaMemcpyDeviceToDevice, s));
        fa = na;
      }
    }
    std::swap(fa, fb);
  }
  F.nm2l = (int64_t)h[1];
  F.np2p = (int64_t)h[2];
  WN_TRY(alloc(&F.m2l, std::max<int64_t>(F.nm2l, 1) * sizeof(uint64_t), true));
  WN_TRY(alloc(&F.p2p, std::max<int64_t>(F.np2p, 1) * sizeof(uint64_t), true));
  WN_TRY(alloc(&F.om, (nn + 1) * sizeof(int32_t), true));
  WN_TRY(alloc(&F.op2, (nn + 1) * sizeof(int32_t), true));
  int bits = 1;
  while (bits < 62 && ((int64_t)1 << bits) <= nn) ++bits;
  WN_TRY(sort_keys_u64(m2l, F.nm2l, 32 + bits, F.m2l, s));
  WN_TRY(sort_keys_u64(p2p, F.np2p, 32 + bits, F.p2p, s));
  k_fmm_csr<<<g256(nn + 1), 256, 0, s>>>(nn, F.m2l, F.nm2l, F.om);
  k_fmm_csr<<<g256(nn + 1), 256, 0, s>>>(nn, F.p2p, F.np2p, F.op2);
  count_launches(2);
  WN_CUDA(cudaGetLastError());
  WN_CUDA(cudaStreamSynchronize(s));  // (the temporaries above are freed stream-ordered on return)
  F.p = p;
  F.theta = theta;
  F.leaf = leafsz;
  F.wsep = wsep;
  F.ready = true;
  return WN_OK;
}

// One FMM application with the tree's plan (capturable: launches and a memset only).  Outputs: out (caller
// layout through out_map, or sorted order; float, N or N×3) scaled, or out4 (sorted float4) unscaled.
wn_status fmm_run(wn_tree_s* t, int op, const float4* vec, const float* scal, float w, const int32_t* out_map,
                  float* out, float4* out4, double scale, cudaStream_t s) {
  FmmPlan& F = t->fmm;
  if (!F.ready) return set_error(WN_ERR_ARG, "internal: FMM plan missing");
  if (w > F.wsep) return set_error(WN_ERR_ARG, "internal: FMM cutoff above the plan's separation width");
  const int64_t nn = t->nn;
  const int p = F.p, np = fmm_count(p);
  FmmGeom g{t->pb, t->pe, t->cb, t->cc, t->depth, t->parent, F.ctr, F.rad, F.leaf_flag};
  const int wpb = 8;
  ProfScope ps(op == OP_A ? WN_PROF_TRAV_A : op == OP_AT ? WN_PROF_TRAV_AT : WN_PROF_TRAV_G, s, 0);
  WN_CUDA(cudaMemsetAsync(F.L, 0, (size_t)nn * np * sizeof(double), s));
  if (vec) k_fmm_p2m<3><<<gwarps(F.nleaves, wpb), 32 * wpb, 0, s>>>(F.nleaves, F.leaves, g, t->pts, vec, scal, p, F.M);
  else k_fmm_p2m<1><<<gwarps(F.nleaves, wpb), 32 * wpb, 0, s>>>(F.nleaves, F.leaves, g, t->pts, vec, scal, p, F.M);
  int launches = 1;
  const int D = (int)F.inner.size() - 1;
  for (int l = D; l >= 0; --l)
    if (F.ninner[l]) {
      k_fmm_m2m<<<gwarps(F.ninner[l], wpb), 32 * wpb, 0, s>>>(F.ninner[l], F.inner[l], g, p, F.M);
      ++launches;
    }
  static int m2l_blocks = 0;  // a resident grid (the blocks build their index tables once)
  if (!m2l_blocks) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fmm_m2l, 32 * kFmmWarps, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    m2l_blocks = std::max(1, per_sm * sms);
  }
  k_fmm_m2l<<<(unsigned)std::min<int64_t>(m2l_blocks, gwarps(nn, kFmmWarps)), 32 * kFmmWarps, 0, s>>>(nn, F.om, F.m2l,
                                                                                                   g, p, F.M, F.L);
  ++launches;
  for (int l = 1; l <= D; ++l)
    if (F.nkids[l]) {
      k_fmm_l2l<<<gwarps(F.nkids[l], wpb), 32 * wpb, 0, s>>>(F.nkids[l], F.kids[l], g, p, F.L);
      ++launches;
    }
  const float w2f = w * w;
  if (vec)
    k_fmm_eval<3><<<gwarps(F.nleaves, wpb), 32 * wpb, 0, s>>>(F.nleaves, F.leaves, g, F.op2, F.p2p, t->pts, vec, scal,
                                                             p, F.L, w2f, op, out_map, out, out4, scale);
  else
    k_fmm_eval<1><<<gwarps(F.nleaves, wpb), 32 * wpb, 0, s>>>(F.nleaves, F.leaves, g, F.op2, F.p2p, t->pts, vec, scal,
                                                             p, F.L, w2f, op, out_map, out, out4, scale);
  ++launches;
  count_launches(launches);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

// ---- the solver's elementwise steps around FMM operators (sorted order; Σ partials per 32 points) ----
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// s = ½ − V (Alg. 2: b − A μ, b = ½), partial Σ s²
__global__ void k_fmm_epi_s(int64_t n, const float* __restrict__ V, float* __restrict__ sv, double* __restrict__ part) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double x = 0.0;
  if (i < n) {
    const double v = 0.5 - (double)V[i];
    sv[i] = (float)v;
    x = v * v;
  }
  x = warp_sum_d(x);
  if ((threadIdx.x & 31) == 0 && i < n + 31 && (i >> 5) * 32 < n) part[i >> 5] = x;
}
// partial Σ V² (‖A r‖²)
__global__ void k_fmm_epi_sq(int64_t n, const float* __restrict__ V, double* __restrict__ part) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double x = 0.0;
  if (i < n) {
    const double v = (double)V[i];
    x = v * v;
  }
  x = warp_sum_d(x);
  if ((threadIdx.x & 31) == 0 && (i >> 5) * 32 < n) part[i >> 5] = x;
}
// partial Σ|r|² of r = Aᵀ s (already in place as float4)
__global__ void k_fmm_epi_r(int64_t n, const float4* __restrict__ r, double* __restrict__ part) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double x = 0.0;
  if (i < n) {
    const float4 v = r[i];
    x = (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z;
  }
  x = warp_sum_d(x);
  if ((threadIdx.x & 31) == 0 && (i >> 5) * 32 < n) part[i >> 5] = x;
}
// μ' = μ + α r (Alg. 2 line 3)
__global__ void k_fmm_axpy(int64_t n, const float4* __restrict__ mu, const float4* __restrict__ r,
                           const double* __restrict__ alpha, float4* __restrict__ mup) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float a = (float)*alpha;
  const float4 m = mu[i], v = r[i];
  mup[i] = make_float4(fmaf(a, v.x, m.x), fmaf(a, v.y, m.y), fmaf(a, v.z, m.z), 0.f);
}
// μ = μ̂ |μ'| / |μ̂|, μ' kept if |μ̂| = 0 (Alg. 3)
__global__ void k_fmm_epi_rescale(int64_t n, const float4* __restrict__ hat, const float4* __restrict__ mup,
                                  float4* __restrict__ mu) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 h = hat[i], m = mup[i];
  const double hm = sqrt((double)h.x * h.x + (double)h.y * h.y + (double)h.z * h.z);
  const double mm = sqrt((double)m.x * m.x + (double)m.y * m.y + (double)m.z * m.z);
  float4 o = m;
  if (hm > 0.0) {
    const double f = mm / hm;
    o = make_float4((float)(h.x * f), (float)(h.y * f), (float)(h.z * f), 0.f);
  }
  mu[i] = o;
}

void fmm_epi_s(int64_t n, const float* V, float* sv, double* part, cudaStream_t s) {
  k_fmm_epi_s<<<g256(n), 256, 0, s>>>(n, V, sv, part);
  count_launches(1);
}
void fmm_epi_sq(int64_t n, const float* V, double* part, cudaStream_t s) {
  k_fmm_epi_sq<<<g256(n), 256, 0, s>>>(n, V, part);
  count_launches(1);
}
void fmm_epi_r(int64_t n, const float4* r, double* part, cudaStream_t s) {
  k_fmm_epi_r<<<g256(n), 256, 0, s>>>(n, r, part);
  count_launches(1);
}
void fmm_axpy(int64_t n, const float4* mu, const float4* r, const double* alpha, float4* mup, cudaStream_t s) {
  k_fmm_axpy<<<g256(n), 256, 0, s>>>(n, mu, r, alpha, mup);
  count_launches(1);
}
void fmm_epi_rescale(int64_t n, const float4* hat, const float4* mup, float4* mu, cudaStream_t s) {
  k_fmm_epi_rescale<<<g256(n), 256, 0, s>>>(n, hat, mup, mu);
  count_launches(1);
}

}  // namespace wn
