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
// B200 mapping (DESIGN.md §6 "FMM"): the interaction lists come from a breadth-first dual traversal on the
// GPU (one thread per cell pair per level, appends by atomics), sorted by (target, source) so that every
// sum runs in a fixed order.  Expansion kernels are templated on the degree p: P2M / M2M / L2L one thread
// per cell with the coefficients in registers; M2L grouped by translation vector (one derivative tensor per
// group, computed at plan time; chunks of pairs contracted against it from shared memory, per-pair results
// summed per target in list order); L2P one warp per leaf; P2P in balanced work items of a leaf's direct
// list.  The test oracle implements the same algorithm independently in plain fp64 C.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <utility>
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
  static uint64_t done = 0;  // per device: __constant__ symbols live on each device separately
  int dev = 0;
  WN_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && ((done >> dev) & 1)) return WN_OK;
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
  if (dev < 64) done |= 1ull << dev;
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

// M2L, grouped by translation vector.  Octree cell centres are dyadic: c = −1 + (2k + 1)·2^−d, so
// R = c_t − c_s is an integer vector o in units of 2^−m, m = max(d_t, d_s), and pairs with equal (m, o)
// share one derivative tensor ∂^δΦ(R).  The plan sorts the pairs by that key; each block takes a chunk
// of ≤ kChunk pairs of one group, builds the tensor once in shared memory — in a (2p+1)³ box layout, so
// that the entry of β + γ sits at box(β) + box(γ), box(a, b, c) = (a·E + b)·E + c, E = 2p + 1 — and then
// every thread contracts one pair, L_γ = Σ_β M_β T_(β+γ), its γ loop unrolled at compile time (box(γ) is
// an immediate offset; all lanes read the same T entry: a shared-memory broadcast per FMA).  The per-pair
// results go to Lp (group order); k_fmm_m2l_reduce adds each target's pairs in the (target, source) order
// of the sorted list — the same fixed order for every run.
constexpr int kM2lKeyOff = 18;  // |o_i| < 2^18: 19 bits per component; else the pair is a group of its own

__host__ __device__ constexpr int fmm_np(int p) { return (p + 1) * (p + 2) * (p + 3) / 6; }
// box offset of the j-th multi-index in the degree-then-(a, b) descending order (the c_mi order)
constexpr int fmm_box_of(int j, int E) {
  int n = 0;
  for (int deg = 0; deg < 64; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b) {
        if (n == j) return (a * E + b) * E + (deg - a - b);
        ++n;
      }
  return -1;
}
// component `comp` of the j-th multi-index in the c_mi order
constexpr int fmm_mi_of(int j, int comp) {
  int n = 0;
  for (int deg = 0; deg < 64; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b) {
        if (n == j) return comp == 0 ? a : comp == 1 ? b : deg - a - b;
        ++n;
      }
  return -1;
}
// CHP_ = 0: a full chunk (128 pairs for p ≤ 4, 64 above); else the small-chunk configuration (≤ 32 pairs)
template <int P, int CHP_ = 0>
struct M2lCfg {
  static constexpr int NP = fmm_np(P), E = 2 * P + 1, NT3 = E * E * E;
  static constexpr int PPT = 2;                  // pairs per thread: one tensor read feeds PPT FMAs (4: slower)
  static constexpr int NSPLIT = (NP + 19) / 20;  // γ parts (≤ 20 accumulators per pair each)
  static constexpr int GCH = (NP + NSPLIT - 1) / NSPLIT;
  static constexpr int CHP = CHP_ ? CHP_ : (NP <= 35 ? 128 : 64);  // pairs per block
  static constexpr int HALF = CHP / PPT;         // threads per γ part
  static constexpr int THREADS = HALF * NSPLIT;
};
constexpr int kM2lSmall = 32;  // chunks of at most this many pairs (group remainders, small groups) go to
                               // one-warp blocks instead of occupying a full block's slot
inline int m2l_chunk(int p) { return fmm_np(p) <= 35 ? 128 : 64; }

__global__ void k_fmm_m2l_gkey(int64_t m, const uint64_t* __restrict__ m2l, FmmGeom g, uint64_t* __restrict__ key) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int T = (int)(m2l[i] >> 32), S = (int)(uint32_t)m2l[i];
  const int mx = max(g.depth[T], g.depth[S]);
  uint64_t k = (uint64_t)mx << 57;
  bool ok = mx < 32;
  for (int a = 0; a < 3; ++a) {
    const double o = ldexp(g.ctr[3 * T + a] - g.ctr[3 * S + a], mx);  // exact (dyadic centres)
    ok = ok && o == rint(o) && fabs(o) < (double)(1 << kM2lKeyOff);
    const uint64_t f = ok ? (uint64_t)((int64_t)o + (1 << kM2lKeyOff)) : 0;
    k |= f << (19 * (2 - a));
  }
  key[i] = ok ? k : ((1ull << 62) | (uint64_t)i);
}

// group starts (flags) and the inverse permutation
__global__ void k_fmm_m2l_ginfo(int64_t m, const uint64_t* __restrict__ skey, const int32_t* __restrict__ gidx,
                                uint32_t* __restrict__ gflag, int32_t* __restrict__ ginv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const bool gs = i == 0 || skey[i] != skey[i - 1];
  gflag[i] = gs ? 1u : 0u;
  ginv[gidx[i]] = (int32_t)i;
}
__global__ void k_fmm_gstart(int64_t m, const uint32_t* __restrict__ gflag, const uint32_t* __restrict__ gpos,
                             int64_t ngroups, int32_t* __restrict__ gstart) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m && gflag[i]) gstart[gpos[i]] = (int32_t)i;
  if (i == m) gstart[ngroups] = (int32_t)m;
}
// chunks start at every chunk-th pair of a group; a chunk of ≤ kM2lSmall pairs is a small one
__global__ void k_fmm_chunk_flags(int64_t m, const uint32_t* __restrict__ gflag, const uint32_t* __restrict__ gpos,
                                  const int32_t* __restrict__ gstart, int chunk, uint32_t* __restrict__ big,
                                  uint32_t* __restrict__ small) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t g = (int64_t)gpos[i] + gflag[i] - 1;  // the group of pair i
  const int64_t rel = i - gstart[g], len = min((int64_t)chunk, (int64_t)gstart[g + 1] - i);
  const bool start = rel % chunk == 0;
  big[i] = start && len > kM2lSmall;
  small[i] = start && len <= kM2lSmall;
}
__global__ void k_fmm_chunk_put(int64_t m, const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                const uint32_t* __restrict__ gflag, const uint32_t* __restrict__ gpos,
                                const int32_t* __restrict__ gstart, int chunk, int4* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m || !flag[i]) return;
  const int64_t g = (int64_t)gpos[i] + gflag[i] - 1;
  const int64_t len = min((int64_t)chunk, (int64_t)gstart[g + 1] - i);
  out[pos[i]] = make_int4((int)i, (int)len, (int)g, 0);
}

template <int P, int G0, int... J>
__device__ __forceinline__ void m2l_row(const double (&m)[M2lCfg<P>::PPT], const double* __restrict__ tb,
                                        double (&acc)[M2lCfg<P>::PPT][M2lCfg<P>::GCH],
                                        std::integer_sequence<int, J...>) {
  using C = M2lCfg<P, 0>;
  (
      [&] {
        if constexpr (G0 + J < C::NP) {
          const double tv = tb[std::integral_constant<int, fmm_box_of(G0 + J, C::E)>::value];
#pragma unroll
          for (int q = 0; q < C::PPT; ++q) acc[q][J] = fma(m[q], tv, acc[q][J]);
        }
      }(),
      ...);
}
// PPT pairs (staged coefficients at Ms + q·HALF, stride CHP per β) of one group, the γ of part PART:
// out[q][j] = Σ_β M_q,β T_(β+γ), γ = PART·GCH + j
template <int P, int CHP, int PART>
__device__ __forceinline__ void m2l_contract(const double* Ms, const double* T3,
                                             double (&out)[M2lCfg<P>::PPT][M2lCfg<P>::GCH]) {
  using C = M2lCfg<P, CHP>;
  constexpr int G0 = PART * C::GCH;
#pragma unroll
  for (int q = 0; q < C::PPT; ++q)
#pragma unroll
    for (int j = 0; j < C::GCH; ++j) out[q][j] = 0.0;
#pragma unroll 1
  for (int be = 0; be < C::NP; ++be) {
    const int base = (c_mi[be][0] * C::E + c_mi[be][1]) * C::E + c_mi[be][2];  // warp-uniform
    double m[C::PPT];
#pragma unroll
    for (int q = 0; q < C::PPT; ++q) m[q] = Ms[be * C::CHP + q * C::HALF];
    m2l_row<P, G0>(m, T3 + base, out, std::make_integer_sequence<int, C::GCH>{});
  }
}
template <int P, int CHP, int PART>
__device__ __forceinline__ void m2l_part(int part, const double* Ms, const double* T3,
                                         double (&out)[M2lCfg<P>::PPT][M2lCfg<P>::GCH]) {
  if constexpr (PART < M2lCfg<P, CHP>::NSPLIT) {
    if (part == PART) m2l_contract<P, CHP, PART>(Ms, T3, out);
    else m2l_part<P, CHP, PART + 1>(part, Ms, T3, out);
  }
}

// the j-th multi-index (c_mi order) of degree ≤ 12, arithmetically (no divergent constant-memory lookups)
__device__ __forceinline__ void fmm_mi_dev(int j, int& a, int& b, int& c) {
  int n = 0;
  while (j >= (n + 1) * (n + 2) * (n + 3) / 6) ++n;
  int rem = j - n * (n + 1) * (n + 2) / 6;
  a = n;
  while (rem > n - a) {
    rem -= n - a + 1;
    --a;
  }
  b = n - a - rem;
  c = n - a - b;
}
// the derivative tensor T_δ = ∂^δΦ(R), |δ| ≤ 2P, of every M2L group (plan time: T depends on the geometry
// only), one block per group, graded order.  b_δ by degree:
//   |δ||R|² b_δ = −(2|δ|−1) Σ_i R_i b_(δ−e_i) − (|δ|−1) Σ_i b_(δ−2e_i),  b_0 = 1/|R|,  T_δ = δ! b_δ / (4π)
template <int P>
__global__ void __launch_bounds__(128) k_fmm_m2l_tensor(const int32_t* __restrict__ gstart,
                                                        const int32_t* __restrict__ gidx,
                                                        const uint64_t* __restrict__ m2l, FmmGeom g,
                                                        double* __restrict__ Tg) {
  using C = M2lCfg<P>;
  constexpr int E = C::E, E2 = E * E, NPT = fmm_np(2 * P);
  __shared__ double T3[C::NT3];
  const int tid = threadIdx.x;
  const uint64_t k0 = m2l[gidx[gstart[blockIdx.x]]];
  const int Tn = (int)(k0 >> 32), Sn = (int)(uint32_t)k0;
  const double R0 = g.ctr[3 * Tn] - g.ctr[3 * Sn], R1 = g.ctr[3 * Tn + 1] - g.ctr[3 * Sn + 1],
               R2 = g.ctr[3 * Tn + 2] - g.ctr[3 * Sn + 2];
  const double r2 = R0 * R0 + R1 * R1 + R2 * R2;
  if (tid == 0) T3[0] = 1.0 / sqrt(r2);
  __syncthreads();
  for (int n = 1; n <= 2 * P; ++n) {
    const int cnt = (n + 1) * (n + 2) / 2;
    const double c1 = 2.0 * n - 1.0, c2 = n - 1.0, inv = 1.0 / (n * r2);
    for (int e = tid; e < cnt; e += 128) {
      int a = n, rem = e;  // e-th (a, b) with a descending, then b descending
      while (rem > n - a) {
        rem -= n - a + 1;
        --a;
      }
      const int b = n - a - rem, c = n - a - b;
      const int idx = (a * E + b) * E + c;
      double sacc = 0.0;
      if (a > 0) sacc -= c1 * R0 * T3[idx - E2];
      if (b > 0) sacc -= c1 * R1 * T3[idx - E];
      if (c > 0) sacc -= c1 * R2 * T3[idx - 1];
      if (a > 1) sacc -= c2 * T3[idx - 2 * E2];
      if (b > 1) sacc -= c2 * T3[idx - 2 * E];
      if (c > 1) sacc -= c2 * T3[idx - 2];
      T3[idx] = sacc * inv;
    }
    __syncthreads();
  }
  for (int j = tid; j < NPT; j += 128) {
    int a, b, c;
    fmm_mi_dev(j, a, b, c);
    Tg[(int64_t)blockIdx.x * NPT + j] = T3[(a * E + b) * E + c] * (c_fact[a] * c_fact[b] * c_fact[c] * 0.0795774715459476679);
  }
}

template <int P, int CHP = 0>
constexpr size_t m2l_smem() {
  using C = M2lCfg<P, CHP>;
  return (size_t)(C::NT3 + C::CHP * C::NP) * sizeof(double) + C::CHP * sizeof(int);
}
// one chunk {first pair, pairs, group} of ≤ CHP pairs of one group: the group's tensor into a (2P+1)³ box in
// shared memory, the sources' coefficients staged [β][pair], two pairs per thread, the outputs written
// back as one run
template <int P, int CHP>
__global__ void __launch_bounds__(M2lCfg<P, CHP>::THREADS) k_fmm_m2l_grp(const int4* __restrict__ chunks,
                                                                          const int32_t* __restrict__ gidx,
                                                                          const uint64_t* __restrict__ m2l,
                                                                          const double* __restrict__ Tg,
                                                                          const double* __restrict__ M,
                                                                          double* __restrict__ Lp) {
  using C = M2lCfg<P, CHP>;
  constexpr int E = C::E, NPT = fmm_np(2 * P);
  extern __shared__ double smem[];
  double* T3 = smem;                      // the group's derivative tensor, box layout
  double* sMO = smem + C::NT3;            // the chunk's multipole coefficients [β][pair], then outputs [pair][γ]
  int* sS = reinterpret_cast<int*>(sMO + C::CHP * C::NP);
  const int tid = threadIdx.x;
  const int4 ch = chunks[blockIdx.x];
  const int i0 = ch.x, npair = ch.y;
  const double* Tgr = Tg + (int64_t)ch.z * NPT;
  for (int j = tid; j < NPT; j += C::THREADS) {
    int a, b, c;
    fmm_mi_dev(j, a, b, c);
    T3[(a * E + b) * E + c] = __ldg(Tgr + j);
  }
  for (int e = tid; e < npair; e += C::THREADS) sS[e] = (int)(uint32_t)m2l[gidx[i0 + e]];
  __syncthreads();
  // the sources' coefficients, staged (each pair's np values contiguous in M: coalesced runs); four loads
  // in flight per thread
  {
    const int tot = npair * C::NP;
    int e = tid;
    for (; e + 3 * C::THREADS < tot; e += 4 * C::THREADS) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = e + u * C::THREADS, pr = x / C::NP, be = x - pr * C::NP;
        v[u] = __ldg(M + (int64_t)sS[pr] * C::NP + be);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = e + u * C::THREADS, pr = x / C::NP, be = x - pr * C::NP;
        sMO[be * C::CHP + pr] = v[u];
      }
    }
    for (; e < tot; e += C::THREADS) {
      const int pr = e / C::NP, be = e - pr * C::NP;
      sMO[be * C::CHP + pr] = __ldg(M + (int64_t)sS[pr] * C::NP + be);
    }
  }
  __syncthreads();
  // thread (part, pa): pairs pa + q·HALF (q < PPT; a slot past the chunk is read but its result dropped)
  const int part = tid / C::HALF, pa = tid % C::HALF;
  double out[C::PPT][C::GCH];
  const bool va = pa < npair;
  if (va) m2l_part<P, CHP, 0>(part, sMO + pa, T3, out);
  __syncthreads();  // every thread has read the staged coefficients
  if (va) {
#pragma unroll
    for (int q = 0; q < C::PPT; ++q) {
      const int pr = pa + q * C::HALF;
#pragma unroll
      for (int j = 0; j < C::GCH; ++j) {
        const int gi = part * C::GCH + j;
        if (gi < C::NP && pr < npair) sMO[pr * C::NP + gi] = out[q][j];
      }
    }
  }
  __syncthreads();
  double* dst = Lp + (int64_t)i0 * C::NP;  // the chunk's pairs are consecutive in group order: one coalesced run
  for (int e = tid; e < npair * C::NP; e += C::THREADS) dst[e] = sMO[e];
}

// L_T = Σ of its pairs' local expansions in list order: one thread per (target with a list, γ)
__global__ void k_fmm_m2l_reduce(int64_t m, const int32_t* __restrict__ targets, const int32_t* __restrict__ off,
                                 const int32_t* __restrict__ ginv, int np, const double* __restrict__ Lp,
                                 double* __restrict__ L) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= m * np) return;
  const int64_t T = targets[t / np];
  const int gi = (int)(t % np);
  const int k0 = off[T], k1 = off[T + 1];
  double acc = 0.0;
  for (int k = k0; k < k1; ++k) acc += Lp[(int64_t)ginv[k] * np + gi];
  L[T * np + gi] = acc;
}
// targets with a non-empty M2L list
__global__ void k_fmm_has_list(int64_t nn, const int32_t* __restrict__ off, uint32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nn) flag[i] = off[i + 1] > off[i] ? 1u : 0u;
}

// ---- P2M, M2M, L2L: one thread per cell, the degree P a template parameter, so that every multi-index
// (and every β − γ of a shift) is a compile-time constant and the coefficients stay in registers; the
// β of a cell are done in parts of ≤ kFmmPart accumulators (one part for p ≤ 4) ----
template <int P>
__device__ __forceinline__ void fmm_pows_t(double x, double* o) {
  o[0] = 1.0;
#pragma unroll
  for (int a = 1; a <= P; ++a) o[a] = o[a - 1] * x / a;
}
// L2P of one target: V += Σ_γ L_γ (y−c)^γ/γ!, ∇V likewise (exponents constant after unrolling)
template <int P, int... J>
__device__ __forceinline__ void l2p_terms(const double* __restrict__ Lt, const double* px, const double* py,
                                          const double* pz, double& V, double& gx, double& gy, double& gz,
                                          std::integer_sequence<int, J...>) {
  (
      [&] {
        constexpr int a = fmm_mi_of(J, 0), b = fmm_mi_of(J, 1), c = fmm_mi_of(J, 2);
        const double l = __ldg(Lt + J);
        V += l * (px[a] * py[b] * pz[c]);
        if constexpr (a > 0) gx += l * (px[a > 0 ? a - 1 : 0] * py[b] * pz[c]);
        if constexpr (b > 0) gy += l * (px[a] * py[b > 0 ? b - 1 : 0] * pz[c]);
        if constexpr (c > 0) gz += l * (px[a] * py[b] * pz[c > 0 ? c - 1 : 0]);
      }(),
      ...);
}
constexpr int kFmmPart = 35;
template <int P>
struct ShiftCfg {
  static constexpr int NP = fmm_np(P), NPART = (NP + kFmmPart - 1) / kFmmPart,
                       NB = (NP + NPART - 1) / NPART;
};
template <int J>
struct Mi {
  static constexpr int a = fmm_mi_of(J, 0), b = fmm_mi_of(J, 1), c = fmm_mi_of(J, 2), deg = a + b + c;
};
// the shift of one source coefficient v = src_G into the part's accumulators:
//   UP (M2M): acc_β += v·d^(β−G)/(β−G)!  for β ≥ G;   down (L2L): acc_δ += v·d^(G−δ)/(G−δ)!  for δ ≤ G
template <int P, int B0, bool UP, int G, int... J>
__device__ __forceinline__ void shift_terms(double v, const double* px, const double* py, const double* pz,
                                            double* acc, std::integer_sequence<int, J...>) {
  (
      [&] {
        constexpr int B = B0 + J;
        if constexpr (B < ShiftCfg<P>::NP) {
          constexpr int e0 = UP ? Mi<B>::a - Mi<G>::a : Mi<G>::a - Mi<B>::a;
          constexpr int e1 = UP ? Mi<B>::b - Mi<G>::b : Mi<G>::b - Mi<B>::b;
          constexpr int e2 = UP ? Mi<B>::c - Mi<G>::c : Mi<G>::c - Mi<B>::c;
          if constexpr (e0 >= 0 && e1 >= 0 && e2 >= 0) acc[J] = fma(v, px[e0] * py[e1] * pz[e2], acc[J]);
        }
      }(),
      ...);
}
template <int P, int B0, bool UP, int... G>
__device__ __forceinline__ void shift_all(const double* __restrict__ src, const double* px, const double* py,
                                          const double* pz, double* acc, std::integer_sequence<int, G...>) {
  ((shift_terms<P, B0, UP, G>(__ldg(src + G), px, py, pz, acc, std::make_integer_sequence<int, ShiftCfg<P>::NB>{})),
   ...);
}

// P2M  M_β = Σ_j [ q_j (−1)^|β| (x_j−c)^β/β! + Σ_k ν_jk (−1)^(|β|−1) (x_j−c)^(β−e_k)/(β−e_k)! ], one thread per leaf
template <int DIM, int P, int B0, int... J>
__device__ __forceinline__ void p2m_terms(double q, double vx, double vy, double vz, const double* px,
                                          const double* py, const double* pz, double* acc,
                                          std::integer_sequence<int, J...>) {
  (
      [&] {
        constexpr int B = B0 + J;
        if constexpr (B < ShiftCfg<P>::NP) {
          constexpr int a = Mi<B>::a, b = Mi<B>::b, c = Mi<B>::c;
          if constexpr (DIM == 1) {
            constexpr double sg = (Mi<B>::deg & 1) ? -1.0 : 1.0;
            acc[J] = fma(sg * q, px[a] * py[b] * pz[c], acc[J]);
          } else {
            constexpr double sg = ((Mi<B>::deg + 1) & 1) ? -1.0 : 1.0;  // (−1)^(|β|−1)
            double t = 0.0;
            if constexpr (a > 0) t = fma(vx, px[a > 0 ? a - 1 : 0] * py[b] * pz[c], t);
            if constexpr (b > 0) t = fma(vy, px[a] * py[b > 0 ? b - 1 : 0] * pz[c], t);
            if constexpr (c > 0) t = fma(vz, px[a] * py[b] * pz[c > 0 ? c - 1 : 0], t);
            acc[J] = fma(sg, t, acc[J]);
          }
        }
      }(),
      ...);
}
template <int DIM, int P, int PART>
__device__ __forceinline__ void p2m_part(int64_t id, FmmGeom g, const float4* __restrict__ pts,
                                         const float4* __restrict__ vec, const float* __restrict__ scal,
                                         double* __restrict__ M) {
  using C = ShiftCfg<P>;
  if constexpr (PART < C::NPART) {
    constexpr int B0 = PART * C::NB;
    double acc[C::NB];
#pragma unroll
    for (int j = 0; j < C::NB; ++j) acc[j] = 0.0;
    const double c0 = g.ctr[3 * id], c1 = g.ctr[3 * id + 1], c2 = g.ctr[3 * id + 2];
    for (int j = g.pb[id]; j < g.pe[id]; ++j) {
      const float4 x = pts[j];
      double px[P + 1], py[P + 1], pz[P + 1];
      fmm_pows_t<P>((double)x.x - c0, px);
      fmm_pows_t<P>((double)x.y - c1, py);
      fmm_pows_t<P>((double)x.z - c2, pz);
      double q = 0.0, vx = 0.0, vy = 0.0, vz = 0.0;
      if (DIM == 1) {
        q = (double)scal[j];
      } else {
        const float4 v = vec[j];
        vx = v.x;
        vy = v.y;
        vz = v.z;
      }
      p2m_terms<DIM, P, B0>(q, vx, vy, vz, px, py, pz, acc, std::make_integer_sequence<int, C::NB>{});
    }
#pragma unroll
    for (int j = 0; j < C::NB; ++j)
      if (B0 + j < C::NP) M[id * C::NP + B0 + j] = acc[j];
    p2m_part<DIM, P, PART + 1>(id, g, pts, vec, scal, M);
  }
}
template <int DIM, int P>
__global__ void k_fmm_p2m(int64_t m, const int32_t* __restrict__ list, FmmGeom g, const float4* __restrict__ pts,
                          const float4* __restrict__ vec, const float* __restrict__ scal, double* __restrict__ M) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) p2m_part<DIM, P, 0>(list[k], g, pts, vec, scal, M);
}

// M2M: one thread per internal active node of one level, M_β = Σ_children Σ_(γ≤β) M_c,γ (c_c' − c_c)^(β−γ)/(β−γ)!
// (children in order)
template <int P, int PART>
__device__ __forceinline__ void m2m_part(int64_t id, FmmGeom g, double* __restrict__ M) {
  using C = ShiftCfg<P>;
  if constexpr (PART < C::NPART) {
    constexpr int B0 = PART * C::NB;
    double acc[C::NB];
#pragma unroll
    for (int j = 0; j < C::NB; ++j) acc[j] = 0.0;
    for (int c = g.cb[id]; c < g.cb[id] + g.cc[id]; ++c) {
      double px[P + 1], py[P + 1], pz[P + 1];  // parent − child
      fmm_pows_t<P>(g.ctr[3 * id] - g.ctr[3 * c], px);
      fmm_pows_t<P>(g.ctr[3 * id + 1] - g.ctr[3 * c + 1], py);
      fmm_pows_t<P>(g.ctr[3 * id + 2] - g.ctr[3 * c + 2], pz);
      shift_all<P, B0, true>(M + (int64_t)c * C::NP, px, py, pz, acc, std::make_integer_sequence<int, C::NP>{});
    }
#pragma unroll
    for (int j = 0; j < C::NB; ++j)
      if (B0 + j < C::NP) M[id * C::NP + B0 + j] = acc[j];
    m2m_part<P, PART + 1>(id, g, M);
  }
}
template <int P>
__global__ void k_fmm_m2m(int64_t m, const int32_t* __restrict__ list, FmmGeom g, double* __restrict__ M) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) m2m_part<P, 0>(list[k], g, M);
}

// L2L: one thread per child of an internal active node of one level, L_c,δ += Σ_(γ≥δ) L_γ (c_c − c)^(γ−δ)/(γ−δ)!
template <int P, int PART>
__device__ __forceinline__ void l2l_part(int64_t c, FmmGeom g, double* __restrict__ L) {
  using C = ShiftCfg<P>;
  if constexpr (PART < C::NPART) {
    constexpr int B0 = PART * C::NB;
    const int64_t par = g.parent[c];
    double acc[C::NB];
#pragma unroll
    for (int j = 0; j < C::NB; ++j) acc[j] = 0.0;
    double px[P + 1], py[P + 1], pz[P + 1];  // child − parent
    fmm_pows_t<P>(g.ctr[3 * c] - g.ctr[3 * par], px);
    fmm_pows_t<P>(g.ctr[3 * c + 1] - g.ctr[3 * par + 1], py);
    fmm_pows_t<P>(g.ctr[3 * c + 2] - g.ctr[3 * par + 2], pz);
    shift_all<P, B0, false>(L + par * C::NP, px, py, pz, acc, std::make_integer_sequence<int, C::NP>{});
#pragma unroll
    for (int j = 0; j < C::NB; ++j)
      if (B0 + j < C::NP) L[c * C::NP + B0 + j] += acc[j];
    l2l_part<P, PART + 1>(c, g, L);
  }
}
template <int P>
__global__ void k_fmm_l2l(int64_t m, const int32_t* __restrict__ list, FmmGeom g, double* __restrict__ L) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) l2l_part<P, 0>(list[k], g, L);
}

// L2P: one warp per FMM leaf, one lane per target point: (V, ∇V) of the far field into VG (sorted order)
template <int P>
__global__ void k_fmm_l2p(int64_t m, const int32_t* __restrict__ list, FmmGeom g, const float4* __restrict__ pts,
                          const double* __restrict__ L, double4* __restrict__ VG) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int64_t T = list[k];
  const double c0 = g.ctr[3 * T], c1 = g.ctr[3 * T + 1], c2 = g.ctr[3 * T + 2];
  for (int i = g.pb[T] + lane; i < g.pe[T]; i += 32) {
    const float4 y = pts[i];
    double px[P + 1], py[P + 1], pz[P + 1];
    fmm_pows_t<P>((double)y.x - c0, px);
    fmm_pows_t<P>((double)y.y - c1, py);
    fmm_pows_t<P>((double)y.z - c2, pz);
    double V = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    l2p_terms<P>(L + T * fmm_np(P), px, py, pz, V, gx, gy, gz, std::make_integer_sequence<int, fmm_np(P)>{});
    VG[i] = make_double4(V, gx, gy, gz);
  }
}

// one target's output from its (V, ∇V): the solver's sorted buffers unscaled (V in .x for A, −∇V for G and
// Aᵀ), or the caller's layout through out_map, scaled (G = −∇V for dipoles, Aᵀ = −∇V for charges)
struct FmmOut {
  int op;
  const int32_t* out_map;
  float* out;
  float4* out4;
  double scale;
  __device__ __forceinline__ void put(int i, double V, double gx, double gy, double gz) const {
    if (out4) {
      out4[i] = op == OP_A ? make_float4((float)V, 0.f, 0.f, 0.f) : make_float4((float)-gx, (float)-gy, (float)-gz, 0.f);
      return;
    }
    const int64_t o = out_map ? (int64_t)out_map[i] : i;
    if (op == OP_A) {
      out[o] = (float)(V * scale);
    } else {
      out[3 * o] = (float)(-gx * scale);
      out[3 * o + 1] = (float)(-gy * scale);
      out[3 * o + 2] = (float)(-gz * scale);
    }
  }
};

// P2P work items: the direct list of a target leaf is cut into items of about kFmmItemWork source points
// (× target chunks of 32), so that the leaves of sparse regions — a depth-3 leaf of C3 sums 55k source
// points, the average 870 — spread over many warps instead of one warp ending the launch alone.
// item = {leaf index li, k0, k1, j (item of its leaf)};  linfo[li] = {T, items of the leaf, partial base, 0}
constexpr int kFmmItemWork = 2048;
__global__ void k_fmm_items(int64_t m, const int32_t* __restrict__ leaves, FmmGeom g,
                            const int32_t* __restrict__ off, const uint64_t* __restrict__ keys,
                            const uint32_t* __restrict__ ibase, int4* __restrict__ items, uint32_t* __restrict__ nit) {
  const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (li >= m) return;
  const int T = leaves[li];
  const int chunks = (g.pe[T] - g.pb[T] + 31) / 32;
  const int k0 = off[T], k1 = off[T + 1];
  int n = 0, start = k0;
  int64_t acc = 0;
  for (int k = k0; k < k1; ++k) {
    const int S = (int)(uint32_t)keys[k];
    acc += (int64_t)(g.pe[S] - g.pb[S]) * chunks;
    if (acc >= kFmmItemWork && k + 1 < k1) {
      if (items) items[ibase[li] + n] = make_int4((int)li, start, k + 1, n);
      ++n;
      start = k + 1;
      acc = 0;
    }
  }
  if (items) items[ibase[li] + n] = make_int4((int)li, start, k1, n);
  ++n;
  if (nit) nit[li] = (uint32_t)n;
}
__global__ void k_fmm_linfo(int64_t m, const int32_t* __restrict__ leaves, FmmGeom g, const uint32_t* __restrict__ nit,
                            uint32_t* __restrict__ psize) {
  const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (li >= m) return;
  const int T = leaves[li];
  psize[li] = nit[li] > 1 ? nit[li] * (uint32_t)(g.pe[T] - g.pb[T]) : 0u;
}
__global__ void k_fmm_linfo2(int64_t m, const int32_t* __restrict__ leaves, const uint32_t* __restrict__ nit,
                             const uint32_t* __restrict__ pbase, int4* __restrict__ linfo, uint32_t* __restrict__ mflag) {
  const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (li >= m) return;
  linfo[li] = make_int4(leaves[li], (int)nit[li], (int)pbase[li], 0);
  mflag[li] = nit[li] > 1 ? 1u : 0u;
}

// P2P of one work item: one warp, a leaf of n ≤ 16 targets split into 32 / gs lane groups (gs = the power
// of two ≥ n): lane (grp, t) takes target t and every (32/gs)-th point of each source leaf, the groups'
// sums added by shuffles (a fixed order).  Pair terms in fp32 (rsqrt, as the treecode's near field),
// summed per source leaf in fp32 and across leaves in fp64; the cutoff decided in fp32 on d = x_j − y
// (R-prec).  A leaf of one item starts from its far field VG and writes the outputs; the items of a
// longer list write partial sums, added to VG by k_fmm_combine in item order.
template <int DIM>
__global__ void __launch_bounds__(256) k_fmm_eval(int64_t m, const int4* __restrict__ items,
                                                  const int4* __restrict__ linfo, FmmGeom g,
                                                  const uint64_t* __restrict__ keys, const float4* __restrict__ pts,
                                                  const float4* __restrict__ vec, const float* __restrict__ scal,
                                                  const double4* __restrict__ VG, double4* __restrict__ part,
                                                  float w2f, FmmOut fo) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int4 it = items[k];
  const int4 li = linfo[it.x];
  const int T = li.x;
  const bool single = li.y == 1;
  const int tb = g.pb[T], te = g.pe[T];
  int gs = 32;  // lanes per group
  while (gs > 1 && te - tb <= gs / 2) gs >>= 1;
  const int grp = lane / gs, ng = 32 / gs, tl = lane % gs;
  const int kb = it.y, ke = it.z;
  // a leaf holds ≤ `leaf` ≤ 32 points unless it is a depth-D cell of duplicates: chunks of 32 targets
  for (int i0 = tb; i0 < te; i0 += 32) {
    const int i = i0 + tl;
    const bool valid = i < te;
    double V = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    const float4 y = valid ? pts[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (single && valid && grp == 0) {  // the far field (k_fmm_l2p)
      const double4 f = VG[i];
      V = f.x;
      gx = f.y;
      gy = f.z;
      gz = f.w;
    }
    // the next source leaf's range is loaded while the current one is summed (a dependent-load chain)
    int nb = 0, ne = 0;
    if (kb < ke) {
      const int S0 = (int)(uint32_t)keys[kb];
      nb = g.pb[S0];
      ne = g.pe[S0];
    }
    for (int kk = kb; kk < ke; ++kk) {
      const int jb = nb, je = ne;
      if (kk + 1 < ke) {
        const int S1 = (int)(uint32_t)keys[kk + 1];
        nb = g.pb[S1];
        ne = g.pe[S1];
      }
      float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
      for (int j = jb + grp; j < je; j += ng) {
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
    for (int o = gs; o < 32; o <<= 1) {  // the groups' sums, lane (0, t) ends with all of target t's
      V += __shfl_xor_sync(0xffffffffu, V, o);
      gx += __shfl_xor_sync(0xffffffffu, gx, o);
      gy += __shfl_xor_sync(0xffffffffu, gy, o);
      gz += __shfl_xor_sync(0xffffffffu, gz, o);
    }
    if (!valid || grp != 0) continue;
    if (single) fo.put(i, V, gx, gy, gz);
    else part[li.z + it.w * (te - tb) + (i - tb)] = make_double4(V, gx, gy, gz);
  }
}

// leaves of several items: VG + the items' partial sums in item order, one warp per leaf
__global__ void k_fmm_combine(int64_t m, const int32_t* __restrict__ mleaves, const int4* __restrict__ linfo,
                              FmmGeom g, const double4* __restrict__ VG, const double4* __restrict__ part, FmmOut fo) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (k >= m) return;
  const int4 li = linfo[mleaves[k]];
  const int tb = g.pb[li.x], te = g.pe[li.x];
  for (int i = tb + lane; i < te; i += 32) {
    double4 a = VG[i];
    for (int j = 0; j < li.y; ++j) {
      const double4 q = part[li.z + j * (te - tb) + (i - tb)];
      a.x += q.x;
      a.y += q.y;
      a.z += q.z;
      a.w += q.w;
    }
    fo.put(i, a.x, a.y, a.z, a.w);
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

// dynamic shared memory of the M2L kernels of degree P (above 48 KB for p = 6); set on the current device
// whenever a plan is built (not a stream operation: never inside a graph capture)
template <int P>
static wn_status m2l_attributes() {
  WN_CUDA(cudaFuncSetAttribute(k_fmm_m2l_grp<P, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m2l_smem<P, 0>()));
  WN_CUDA(cudaFuncSetAttribute(k_fmm_m2l_grp<P, kM2lSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)m2l_smem<P, kM2lSmall>()));
  return WN_OK;
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
  switch (p) {
    case 1: WN_TRY(m2l_attributes<1>()); break;
    case 2: WN_TRY(m2l_attributes<2>()); break;
    case 3: WN_TRY(m2l_attributes<3>()); break;
    case 4: WN_TRY(m2l_attributes<4>()); break;
    case 5: WN_TRY(m2l_attributes<5>()); break;
    default: WN_TRY(m2l_attributes<6>()); break;
  }
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
  WN_TRY(alloc(&F.VG, (size_t)std::max<int64_t>(t->n, 1) * sizeof(double4), true));
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
  // M2L groups (pairs with one translation vector) and their chunks
  if (F.nm2l > 0) {
    const int64_t m = F.nm2l;
    uint64_t *gk = nullptr, *sk = nullptr;
    uint32_t *cflag = nullptr, *cpos = nullptr, *gflag = nullptr, *gpos = nullptr;
    WN_TRY(alloc(&gk, m * sizeof(uint64_t), false));
    WN_TRY(alloc(&sk, m * sizeof(uint64_t), false));
    WN_TRY(alloc(&cflag, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&cpos, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&gflag, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&gpos, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&F.gidx, m * sizeof(int32_t), true));
    WN_TRY(alloc(&F.ginv, m * sizeof(int32_t), true));
    k_fmm_m2l_gkey<<<g256(m), 256, 0, s>>>(m, F.m2l, g, gk);
    count_launches(1);
    WN_TRY(sort_keys_u64_perm(gk, m, 63, sk, F.gidx, s));
    k_fmm_m2l_ginfo<<<g256(m), 256, 0, s>>>(m, sk, F.gidx, gflag, F.ginv);
    WN_TRY(fmm_scan(gflag, gpos, m, gpos + m, s));
    uint32_t ng = 0;
    WN_CUDA(cudaMemcpyAsync(&ng, gpos + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    F.ngroups = ng;
    int32_t* gstart = nullptr;
    WN_TRY(alloc(&gstart, (F.ngroups + 1) * sizeof(int32_t), false));
    k_fmm_gstart<<<g256(m + 1), 256, 0, s>>>(m, gflag, gpos, F.ngroups, gstart);
    uint32_t *sflag = nullptr, *spos = nullptr;
    WN_TRY(alloc(&sflag, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&spos, (m + 1) * sizeof(uint32_t), false));
    k_fmm_chunk_flags<<<g256(m), 256, 0, s>>>(m, gflag, gpos, gstart, m2l_chunk(p), cflag, sflag);
    WN_TRY(fmm_scan(cflag, cpos, m, cpos + m, s));
    WN_TRY(fmm_scan(sflag, spos, m, spos + m, s));
    uint32_t tot[2] = {0, 0};
    WN_CUDA(cudaMemcpyAsync(&tot[0], cpos + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaMemcpyAsync(&tot[1], spos + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    F.nchunk = tot[0];
    F.nchunk_small = tot[1];
    WN_TRY(alloc(&F.chunks, std::max<int64_t>(F.nchunk, 1) * sizeof(int4), true));
    WN_TRY(alloc(&F.chunks_small, std::max<int64_t>(F.nchunk_small, 1) * sizeof(int4), true));
    k_fmm_chunk_put<<<g256(m), 256, 0, s>>>(m, cflag, cpos, gflag, gpos, gstart, m2l_chunk(p), F.chunks);
    k_fmm_chunk_put<<<g256(m), 256, 0, s>>>(m, sflag, spos, gflag, gpos, gstart, m2l_chunk(p), F.chunks_small);
    count_launches(4);
    WN_TRY(alloc(&F.Tg, (size_t)std::max<int64_t>(F.ngroups, 1) * fmm_np(2 * p) * sizeof(double), true));
    switch (p) {
      case 1: k_fmm_m2l_tensor<1><<<(unsigned)F.ngroups, 128, 0, s>>>(gstart, F.gidx, F.m2l, g, F.Tg); break;
      case 2: k_fmm_m2l_tensor<2><<<(unsigned)F.ngroups, 128, 0, s>>>(gstart, F.gidx, F.m2l, g, F.Tg); break;
      case 3: k_fmm_m2l_tensor<3><<<(unsigned)F.ngroups, 128, 0, s>>>(gstart, F.gidx, F.m2l, g, F.Tg); break;
      case 4: k_fmm_m2l_tensor<4><<<(unsigned)F.ngroups, 128, 0, s>>>(gstart, F.gidx, F.m2l, g, F.Tg); break;
      case 5: k_fmm_m2l_tensor<5><<<(unsigned)F.ngroups, 128, 0, s>>>(gstart, F.gidx, F.m2l, g, F.Tg); break;
      default: k_fmm_m2l_tensor<6><<<(unsigned)F.ngroups, 128, 0, s>>>(gstart, F.gidx, F.m2l, g, F.Tg); break;
    }
    count_launches(1);
    WN_TRY(alloc(&F.Lp, (size_t)m * np * sizeof(double), true));
    k_fmm_has_list<<<g256(nn), 256, 0, s>>>(nn, F.om, flag);
    WN_TRY(fmm_scan(flag, pos, nn, pos + nn, s));
    uint32_t nt = 0;
    WN_CUDA(cudaMemcpyAsync(&nt, pos + nn, sizeof(nt), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    F.nm2lt = nt;
    WN_TRY(alloc(&F.m2lt, std::max<uint32_t>(nt, 1) * sizeof(int32_t), true));
    k_fmm_compact<<<g256(nn), 256, 0, s>>>(nn, flag, pos, F.m2lt);
    count_launches(4);
  }
  // P2P work items of the target leaves (k_fmm_items), the partial-sum slots of the leaves of several
  {
    const int64_t m = F.nleaves;
    uint32_t *nit = nullptr, *ibase = nullptr, *psize = nullptr, *pbase = nullptr, *mflag = nullptr, *mpos = nullptr;
    WN_TRY(alloc(&nit, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&ibase, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&psize, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&pbase, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&mflag, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&mpos, (m + 1) * sizeof(uint32_t), false));
    WN_TRY(alloc(&F.linfo, std::max<int64_t>(m, 1) * sizeof(int4), true));
    k_fmm_items<<<g256(m), 256, 0, s>>>(m, F.leaves, g, F.op2, F.p2p, nullptr, nullptr, nit);
    k_fmm_linfo<<<g256(m), 256, 0, s>>>(m, F.leaves, g, nit, psize);
    WN_TRY(fmm_scan(nit, ibase, m, ibase + m, s));
    WN_TRY(fmm_scan(psize, pbase, m, pbase + m, s));
    k_fmm_linfo2<<<g256(m), 256, 0, s>>>(m, F.leaves, nit, pbase, F.linfo, mflag);
    WN_TRY(fmm_scan(mflag, mpos, m, mpos + m, s));
    uint32_t tot[3] = {0, 0, 0};
    WN_CUDA(cudaMemcpyAsync(&tot[0], ibase + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaMemcpyAsync(&tot[1], pbase + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaMemcpyAsync(&tot[2], mpos + m, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    F.nitems = tot[0];
    F.nmleaves = tot[2];
    WN_TRY(alloc(&F.items, std::max<int64_t>(F.nitems, 1) * sizeof(int4), true));
    WN_TRY(alloc(&F.part, std::max<uint32_t>(tot[1], 1) * sizeof(double4), true));
    WN_TRY(alloc(&F.mleaves, std::max<int64_t>(F.nmleaves, 1) * sizeof(int32_t), true));
    k_fmm_items<<<g256(m), 256, 0, s>>>(m, F.leaves, g, F.op2, F.p2p, ibase, F.items, nullptr);
    k_fmm_compact<<<g256(m), 256, 0, s>>>(m, mflag, mpos, F.mleaves);
    count_launches(5);
  }
  WN_CUDA(cudaGetLastError());
  WN_CUDA(cudaStreamSynchronize(s));  // (the temporaries above are freed stream-ordered on return)
  F.p = p;
  F.theta = theta;
  F.leaf = leafsz;
  F.wsep = wsep;
  F.ready = true;
  return WN_OK;
}

// the expansions of one application, degree P: P2M, M2M (deepest level first), M2L (grouped, then the
// per-target sums), L2L (top down), L2P into F.VG; returns the number of launches
template <int P>
static int fmm_expansions(wn_tree_s* t, const FmmGeom& g, const float4* vec, const float* scal, cudaStream_t s) {
  FmmPlan& F = t->fmm;
  constexpr int np = fmm_np(P);
  const int wpb = 8;
  int launches = 0;
  if (vec) k_fmm_p2m<3, P><<<g256(F.nleaves), 256, 0, s>>>(F.nleaves, F.leaves, g, t->pts, vec, scal, F.M);
  else k_fmm_p2m<1, P><<<g256(F.nleaves), 256, 0, s>>>(F.nleaves, F.leaves, g, t->pts, vec, scal, F.M);
  ++launches;
  const int D = (int)F.inner.size() - 1;
  for (int l = D; l >= 0; --l)
    if (F.ninner[l]) {
      k_fmm_m2m<P><<<g256(F.ninner[l]), 256, 0, s>>>(F.ninner[l], F.inner[l], g, F.M);
      ++launches;
    }
  if (F.nchunk + F.nchunk_small > 0) {
    if (F.nchunk)
      k_fmm_m2l_grp<P, 0><<<(unsigned)F.nchunk, M2lCfg<P, 0>::THREADS, m2l_smem<P, 0>(), s>>>(F.chunks, F.gidx, F.m2l,
                                                                                          F.Tg, F.M, F.Lp);
    if (F.nchunk_small)
      k_fmm_m2l_grp<P, kM2lSmall><<<(unsigned)F.nchunk_small, M2lCfg<P, kM2lSmall>::THREADS, m2l_smem<P, kM2lSmall>(),
                                    s>>>(F.chunks_small, F.gidx, F.m2l, F.Tg, F.M, F.Lp);
    k_fmm_m2l_reduce<<<g256(F.nm2lt * np), 256, 0, s>>>(F.nm2lt, F.m2lt, F.om, F.ginv, np, F.Lp, F.L);
    launches += 2;
  }
  for (int l = 1; l <= D; ++l)
    if (F.nkids[l]) {
      k_fmm_l2l<P><<<g256(F.nkids[l]), 256, 0, s>>>(F.nkids[l], F.kids[l], g, F.L);
      ++launches;
    }
  k_fmm_l2p<P><<<gwarps(F.nleaves, wpb), 32 * wpb, 0, s>>>(F.nleaves, F.leaves, g, t->pts, F.L, F.VG);
  return launches + 1;
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
  int launches = 0;
  switch (p) {
    case 1: launches = fmm_expansions<1>(t, g, vec, scal, s); break;
    case 2: launches = fmm_expansions<2>(t, g, vec, scal, s); break;
    case 3: launches = fmm_expansions<3>(t, g, vec, scal, s); break;
    case 4: launches = fmm_expansions<4>(t, g, vec, scal, s); break;
    case 5: launches = fmm_expansions<5>(t, g, vec, scal, s); break;
    default: launches = fmm_expansions<6>(t, g, vec, scal, s); break;
  }
  const float w2f = w * w;
  const FmmOut fo{op, out_map, out, out4, scale};
  if (vec)
    k_fmm_eval<3><<<gwarps(F.nitems, wpb), 32 * wpb, 0, s>>>(F.nitems, F.items, F.linfo, g, F.p2p, t->pts, vec, scal,
                                                            F.VG, F.part, w2f, fo);
  else
    k_fmm_eval<1><<<gwarps(F.nitems, wpb), 32 * wpb, 0, s>>>(F.nitems, F.items, F.linfo, g, F.p2p, t->pts, vec, scal,
                                                            F.VG, F.part, w2f, fo);
  if (F.nmleaves) {
    k_fmm_combine<<<gwarps(F.nmleaves, wpb), 32 * wpb, 0, s>>>(F.nmleaves, F.mleaves, F.linfo, g, F.VG, F.part, fo);
    ++launches;
  }
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
