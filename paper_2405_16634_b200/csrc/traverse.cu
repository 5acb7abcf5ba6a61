// traverse.cu — warp-cooperative treecode traversal.
//
// Algorithm 4 apply_A, per query x_i and node B:
//     if |x_i − x_B| > c·width(B):  representative term            ("modified by w")
//     elif B is not a leaf:         recurse into the children
//     else:                         direct sum over the points of B  ("modified by w")
// "Other operators Aᵀ and G are accelerated in the same way" (L406).  Terms (d = x_src − x_i):
//     A  : ∇Φ(x_i − x_src)·ν      =  (d·ν) / (4π r³)                 (Eq wnf-discretization)
//     Aᵀ : s ∇Φ(x_src − x_i)      = −s d / (4π r³)                   (Alg. 2; ν = s, L371)
//     G  : −HΦ(x_i − x_src) ν     = (ν − 3 (d·ν) d / r²) / (4π r³)   (L264-L272)
// and every term is 0 when r < w (§4.4).
//
// B200 design:
//   * one warp = 32 consecutive Morton-sorted queries; a per-warp shared-memory stack of
//     (child group, lane mask) entries; every lane takes ITS OWN opening decision (exact per-query
//     semantics of Alg. 4 — no "open if any lane opens"); the ballot of the lanes that open a node
//     becomes the mask of the pushed child group;
//   * node records are 64-byte AoS (R | V | L | pad): three broadcast LDG.128 from one L1 line;
//   * one-point nodes carry thr = −1, so they always take the representative branch (which equals
//     the leaf branch: rep = the point, ν_B = ν_j) and are never opened;
//   * the kernel term is branch-free (predicated by `live`), rsqrt is one MUFU op (ftz; r ≥ w > 0);
//   * decisions, cutoff and term value all use the fp32 offset d = (hi − x_q) + lo to the representative,
//     d² = fma(dx,dx, fma(dy,dy, dz·dz)) (DESIGN.md R-prec); A accumulates per child group in
//     fp32 and across groups in fp64 (s = ½ − Aμ cancels near convergence);
//   * epilogues fuse the solver's elementwise work (s = ½ − Aμ, Σ partials, rescale).
#include <cuda_runtime.h>

#include "wn_internal.cuh"

namespace wn {
namespace {

constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ float dist2(float dx, float dy, float dz) {
  return __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));
}

// 1/r for a live term, +0 for a dead one (rsqrt(+∞) = +0): live is evaluated as one predicate
__device__ __forceinline__ float inv_live(bool live, float e2) {
  float r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tselp.f32 %0, %2, 0f7F800000, p;\n\t"
      "rsqrt.approx.ftz.f32 %0, %0;\n\t}"
      : "=f"(r)
      : "r"((unsigned)live), "f"(e2));
  return r;
}

template <int OP>
struct Acc {
  float x = 0.f, y = 0.f, z = 0.f;
  double d = 0.0;
  // source at offset e = x_src − x_q (|e|² = e2), attribute V; contributes only if `live`
  // a dead term takes rsqrt(+∞) = +0, so every factor below is 0 and the accumulators are unchanged
  // (x + (±0) = x, all other operands finite): one select per term instead of two
  __device__ __forceinline__ void term(bool live, float ex, float ey, float ez, float e2, const float4& V) {
    const float inv = inv_live(live, e2);
    if (OP == OP_A) {
      const float inv3 = inv * inv * inv;
      x = fmaf(fmaf(ex, V.x, fmaf(ey, V.y, ez * V.z)), inv3, x);
    } else if (OP == OP_AT) {
      const float c = -V.x * (inv * inv * inv);
      x = fmaf(c, ex, x);
      y = fmaf(c, ey, y);
      z = fmaf(c, ez, z);
    } else {
      const float inv2 = inv * inv;
      const float inv3 = inv2 * inv;
      const float t = 3.0f * fmaf(ex, V.x, fmaf(ey, V.y, ez * V.z)) * inv2;
      x = fmaf(inv3, fmaf(-t, ex, V.x), x);
      y = fmaf(inv3, fmaf(-t, ey, V.y), y);
      z = fmaf(inv3, fmaf(-t, ez, V.z), z);
    }
  }
  // first-order far field (row f2): the order-0 term plus Σ_j ∇f(x_B)·d_j from the node's first moments,
  // X0 = (Mxx, Myy, Mzz, tr M), X1 = (Mxy, Mxz, Myz, ·) (sym M, vector ν) or X0 = (D, ·) (scalar s):
  //   A : (e·ν + tr M − 3 eᵀMe/r²) / r³
  //   Aᵀ: −(s e + D − 3 e (e·D)/r²) / r³
  //   G : (ν − 3(e·ν) e/r² − 6 M e/r² + (15 eᵀMe/r² − 3 tr M) e/r²) / r³       (e = x_B − x_q, ×1/(4π) later)
  __device__ __forceinline__ void term1(bool live, float ex, float ey, float ez, float e2, const float4& V,
                                        const float4& X0, const float4& X1) {
    const float inv = inv_live(live, e2);
    const float inv2 = inv * inv;
    const float inv3 = inv2 * inv;
    if (OP == OP_AT) {
      const float eD = fmaf(ex, X0.x, fmaf(ey, X0.y, ez * X0.z));
      const float k = fmaf(-3.0f * eD, inv2, V.x);
      x = fmaf(-inv3, fmaf(k, ex, X0.x), x);
      y = fmaf(-inv3, fmaf(k, ey, X0.y), y);
      z = fmaf(-inv3, fmaf(k, ez, X0.z), z);
      return;
    }
    const float mx = fmaf(X0.x, ex, fmaf(X1.x, ey, X1.y * ez));
    const float my = fmaf(X1.x, ex, fmaf(X0.y, ey, X1.z * ez));
    const float mz = fmaf(X1.y, ex, fmaf(X1.z, ey, X0.z * ez));
    const float uMu = fmaf(ex, mx, fmaf(ey, my, ez * mz));
    const float eV = fmaf(ex, V.x, fmaf(ey, V.y, ez * V.z));
    if (OP == OP_A) {
      x = fmaf(fmaf(-3.0f * uMu, inv2, eV + X0.w), inv3, x);
    } else {
      const float t = 3.0f * eV * inv2;
      const float k = fmaf(inv2, fmaf(15.0f * uMu, inv2, -3.0f * X0.w), -t);
      const float m6 = -6.0f * inv2;
      x = fmaf(inv3, fmaf(k, ex, fmaf(m6, mx, V.x)), x);
      y = fmaf(inv3, fmaf(k, ey, fmaf(m6, my, V.y)), y);
      z = fmaf(inv3, fmaf(k, ez, fmaf(m6, mz, V.z)), z);
    }
  }
  __device__ __forceinline__ void flush() {
    if (OP == OP_A) {
      d += (double)x;
      x = 0.f;
    }
  }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// node record address: one 32-bit byte offset from the base (records are 64 B, Nn < 2^26)
__device__ __forceinline__ const float4* rec_at(const float4* base, int node) {
  return reinterpret_cast<const float4*>(reinterpret_cast<const char*>(base) + ((uint32_t)node << 6));
}

struct Work {  // algorithmic work of one query (counting variant)
  int test = 0, far = 0, near = 0, live = 0;
};

// Visit `node` for the lanes in `mine`: its term (far lanes past the cutoff) and, for the lanes that
// open a leaf-coded node (a multi-point leaf or a pseudo-leaf), the direct sum over its points.
// Returns the ballot of the lanes that open it; *topo_out = its traversal code (0: leaf-coded).
template <int OP, bool COUNT, bool FROZEN, int ORD>
__device__ __forceinline__ uint32_t trav_visit(const TravArgs& a, int node, bool mine, const float4& xq, Acc<OP>& acc,
                                               Work& wk, int& topo_out) {
  const int lane = threadIdx.x & 31;
  const float4* __restrict__ G = a.nodes.rec;           // geometry: R (+0), L (+2)
  const float4* __restrict__ Vr = FROZEN ? a.attr : G;  // attributes: V (+1)
  const float w2 = a.w2;
  WN_DCHECK(node >= 0 && node < a.nnodes, "node index");
  const float4* rp = rec_at(G, node);
  const float4 R = __ldg(rp);
  const float4 V = FROZEN ? __ldg(rec_at(Vr, node) + 1) : __ldg(rp + 1);
  const float4 L = __ldg(rp + 2);
  // d = (hi − x_q) + lo: decisions and value on the same fp32 offset (R-prec)
  const float ex = __fadd_rn(__fsub_rn(R.x, xq.x), L.x), ey = __fadd_rn(__fsub_rn(R.y, xq.y), L.y),
              ez = __fadd_rn(__fsub_rn(R.z, xq.z), L.z);
  const float d2 = dist2(ex, ey, ez);
  const bool far = d2 > R.w;
  const bool live = mine && far && !(d2 < w2);
  if (ORD == 1) {
    const float4 X0 = __ldg(a.nodes.ext + 2 * node);
    const float4 X1 = OP == OP_AT ? X0 : __ldg(a.nodes.ext + 2 * node + 1);
    acc.term1(live, ex, ey, ez, d2, V, X0, X1);
  } else {
    acc.term(live, ex, ey, ez, d2, V);
  }
  if (COUNT && mine) {
    // a collapsed chain (tree_build.cu:topo_codes): Alg. 4 tests its levels from the top until one
    // is far — level k's threshold is the bottom's × 4^(len−1−k), exactly (powers of two)
    const int len = (__float_as_int(L.w) >> 8) & 31;
    int tests = 1;
    if (len > 1) {
      tests = len;
      for (int kk = 0; kk < len; ++kk)
        if (d2 > ldexpf(R.w, 2 * (len - 1 - kk))) {
          tests = kk + 1;
          break;
        }
    }
    wk.test += tests;
    wk.far += far;
    wk.live += live;
  }
  const uint32_t open = __ballot_sync(FULL, mine && !far);
  const int topo = __float_as_int(V.w);
  topo_out = topo;
  if (open && topo == 0) {  // leaf-coded: direct sum for the lanes that opened it
    const bool lm = (open >> lane) & 1u;
    const int j1 = a.nrange_pe[node];
    WN_DCHECK(a.nrange_pb[node] >= 0 && j1 <= a.npts && a.nrange_pb[node] < j1, "leaf point range");
    for (int j = a.nrange_pb[node]; j < j1; ++j) {
      const float4 P = __ldg(a.pts + j);
      float4 Vj;
      if (OP == OP_AT) Vj = make_float4(__ldg(a.scal + j), 0.f, 0.f, 0.f);
      else Vj = __ldg(a.vec + j);
      const float px = __fsub_rn(P.x, xq.x), py = __fsub_rn(P.y, xq.y), pz = __fsub_rn(P.z, xq.z);
      const float p2 = dist2(px, py, pz);
      const bool lv = lm && !(p2 < w2);
      acc.term(lv, px, py, pz, p2, Vj);
      if (COUNT && lm) {
        ++wk.near;
        wk.live += lv;
        wk.test += (__float_as_int(L.w) >> 13) & 1;  // a node whose children are all points
      }
    }
  }
  return open;
}

// Pop child groups (code, lane mask) off this warp's stack until it is empty; every child of a popped
// group is visited, the lanes that open an internal node push its child group.
template <int OP, bool COUNT, bool FROZEN, int ORD>
__device__ __forceinline__ void trav_loop(const TravArgs& a, int2* stk, int sp, const float4& xq, Acc<OP>& acc,
                                          Work& wk) {
  const int lane = threadIdx.x & 31;
  while (sp > 0) {
    --sp;
    const int2 e = stk[sp];
    __syncwarp();
    const int code = e.x;
    const int cb = code >> 4, ncc = (code & 7) + 1;
    const bool mine = ((uint32_t)e.y >> lane) & 1u;
    for (int k = 0; k < ncc; ++k) {
      int topo;
      const uint32_t open = trav_visit<OP, COUNT, FROZEN, ORD>(a, cb + k, mine, xq, acc, wk, topo);
      if (open && topo != 0) {
        WN_DCHECK(sp < a.stack_depth, "traversal stack");
        stk[sp] = make_int2(topo, (int)open);  // every lane writes the same word: no divergence
        ++sp;
      }
    }
    acc.flush();  // (no trailing __syncwarp: every lane writes the same stack words and reads its own)
  }
}

// outputs of one query (fused solver epilogues), its work counts, and its warp group's Σ partial (slot ib)
template <int OP, int EPI, bool COUNT>
__device__ __forceinline__ void trav_epilogue(const TravArgs& a, bool valid, int64_t q, const Acc<OP>& acc,
                                              const Work& wk, bool has_group, int64_t ib) {
  const int lane = threadIdx.x & 31;
  double part = 0.0;
  if (valid) {
    const int64_t oq = a.out_map ? (int64_t)a.out_map[q] : q;
    if (OP == OP_A) {
      const double val = acc.d * 0.0795774715459476679;  // Σ / (4π)
      if (EPI == EPI_PLAIN && a.out_f) a.out_f[oq] = (float)(val * (double)a.scale_out);
      if (EPI == EPI_S) {
        const double sv = 0.5 - val;
        if (a.world) {  // peer-memory exchange: this row into every rank's replica (NVLink stores)
          for (int r = 0; r < a.world; ++r) a.peer_f[r][q] = (float)sv;
        } else {
          a.out_f[q] = (float)sv;
        }
        part = sv * sv;
      }
      if (EPI == EPI_SQ) part = val * val;
    } else {
      const float vx = acc.x * kInv4Pi, vy = acc.y * kInv4Pi, vz = acc.z * kInv4Pi;
      if (EPI == EPI_PLAIN && a.out_v3) {
        a.out_v3[3 * oq + 0] = vx * a.scale_out;
        a.out_v3[3 * oq + 1] = vy * a.scale_out;
        a.out_v3[3 * oq + 2] = vz * a.scale_out;
      }
      if (EPI == EPI_R) {
        const float4 o = make_float4(vx, vy, vz, 0.f);
        if (a.world) {
          for (int r = 0; r < a.world; ++r) a.peer_v4[r][q] = o;
        } else {
          a.out_v4[q] = o;
        }
        part = (double)vx * vx + (double)vy * vy + (double)vz * vz;
      }
      if (EPI == EPI_RESCALE) {  // μ_i = μ̂_i |μ'_i| / |μ̂_i|, μ'_i kept if |μ̂_i| = 0 (Alg. 3)
        const float4 m = a.mup[q];
        const double hm = sqrt((double)vx * vx + (double)vy * vy + (double)vz * vz);
        const double mm = sqrt((double)m.x * m.x + (double)m.y * m.y + (double)m.z * m.z);
        float4 o = m;
        if (hm > 0.0) {
          const double f = mm / hm;
          o = make_float4((float)(vx * f), (float)(vy * f), (float)(vz * f), 0.f);
        }
        if (a.world) {
          for (int r = 0; r < a.world; ++r) a.peer_v4[r][q] = o;
        } else {
          a.out_v4[q] = o;
        }
      }
    }
  }
  if (COUNT) {  // algorithmic work: node tests, representative terms, leaf-point terms, live terms (r ≥ w)
    if (a.qcounts && valid) {
      const int64_t oq = a.out_map ? (int64_t)a.out_map[q] : q;
      a.qcounts[4 * oq + 0] = wk.test;
      a.qcounts[4 * oq + 1] = wk.far;
      a.qcounts[4 * oq + 2] = wk.near;
      a.qcounts[4 * oq + 3] = wk.live;
    }
    if (a.work) {
      unsigned long long c[4] = {(unsigned long long)wk.test, (unsigned long long)wk.far,
                                 (unsigned long long)wk.near, (unsigned long long)wk.live};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int o = 16; o; o >>= 1) c[k] += __shfl_xor_sync(FULL, c[k], o);
        if (lane == 0) atomicAdd((unsigned long long*)a.work + k, c[k]);
      }
    }
  }
  if (EPI == EPI_S || EPI == EPI_SQ || EPI == EPI_R) {  // this warp's group slot ib (schedule position / 32)
    part = warp_sum(part);
    if (lane == 0 && has_group) {
      WN_DCHECK(ib < part_slots(a.npts) || a.queries != a.pts, "partial slot");
      if (a.world) {
        for (int r = 0; r < a.world; ++r) a.peer_part[r][ib] = part;
      } else {
        a.partial[ib] = part;
      }
    }
  }
  if (a.world) {  // signal: every thread's remote stores, then one count per block, the last block tells every rank
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int prev = atomicAdd(a.done, 1u);
      if (prev == gridDim.x - 1) {
        __threadfence_system();
        *a.done = 0u;  // ready for the next exchange (stream-ordered)
        for (int r = 0; r < a.world; ++r) atomicAdd_system(a.peer_sig[r], 1ull);
      }
    }
  }
}

// one warp = 32 consecutive queries of the schedule (positions kq of the lanes), traversing from the root (the
// hot loop: written out here — the same steps as trav_visit / trav_loop, which the compiler schedules worse)
template <int OP, int EPI, bool COUNT, bool FROZEN, int ORD>
__device__ __forceinline__ void trav_group(const TravArgs& a, int2* stk, const int64_t kq) {
  const int lane = threadIdx.x & 31;
  const bool valid = kq < a.q_end;
  const int64_t q = (valid && a.qorder) ? (int64_t)a.qorder[kq] : kq;             // query index
  WN_DCHECK(!valid || (q >= 0 && (a.npts == 0 || a.queries != a.pts || q < a.npts)), "query index");
  const float4 xq = valid ? a.queries[q] : make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t active = __ballot_sync(FULL, valid);
  const float4* __restrict__ G = a.nodes.rec;             // geometry: R (+0), L (+2)
  const float4* __restrict__ Vr = FROZEN ? a.attr : G;    // attributes: V (+1)
  const float w2 = a.w2;
  Acc<OP> acc;
  int ntest = 0, nfar = 0, nnear = 0, nlive = 0, wvis = 0;  // wvis: warp-level visits (counting variant)
  if (active) {
    int sp = 0;
    if (lane == 0) stk[0] = make_int2(0, (int)active);  // the root as a group of one
    sp = 1;
    __syncwarp();
    while (sp > 0) {
      --sp;
      const int2 e = stk[sp];
      __syncwarp();
      // every lane read the same entry; taking lane 0's lets the compiler see a warp-uniform trip count and
      // uniform branches below (loop control and addresses on the uniform datapath, no reconvergence
      // barrier before each vote: C3 Aᵀ −2.8 %, G −2.0 %)
      const int code = __shfl_sync(FULL, e.x, 0);
      const int cb = code >> 4, ncc = (code & 7) + 1;
      const bool mine = ((uint32_t)e.y >> lane) & 1u;
      if (COUNT) wvis += ncc;
      {
        for (int k = 0; k < ncc; ++k) {
          const int node = cb + k;
          WN_DCHECK(node >= 0 && node < a.nnodes, "node index");
          const float4* rp = rec_at(G, node);
          const float4 R = __ldg(rp);
          const float4 V = FROZEN ? __ldg(rec_at(Vr, node) + 1) : __ldg(rp + 1);
          const float4 L = __ldg(rp + 2);
          // d = (hi − x_q) + lo: decisions and value on the same fp32 offset (R-prec)
          const float ex = __fadd_rn(__fsub_rn(R.x, xq.x), L.x), ey = __fadd_rn(__fsub_rn(R.y, xq.y), L.y),
                      ez = __fadd_rn(__fsub_rn(R.z, xq.z), L.z);
          const float d2 = dist2(ex, ey, ez);
          const bool far = d2 > R.w;
          const bool live = mine && far && !(d2 < w2);
          if (ORD == 1) {
            const float4 X0 = __ldg(a.nodes.ext + 2 * node);
            const float4 X1 = OP == OP_AT ? X0 : __ldg(a.nodes.ext + 2 * node + 1);
            acc.term1(live, ex, ey, ez, d2, V, X0, X1);
          } else {
            acc.term(live, ex, ey, ez, d2, V);
          }
          if (COUNT && mine) {
            // a collapsed chain (tree_build.cu:topo_codes): Alg. 4 tests its levels from the top until one
            // is far — level k's threshold is the bottom's × 4^(len−1−k), exactly (powers of two)
            const int len = (__float_as_int(L.w) >> 8) & 31;
            int tests = 1;
            if (len > 1) {
              tests = len;
              for (int kk = 0; kk < len; ++kk)
                if (d2 > ldexpf(R.w, 2 * (len - 1 - kk))) {
                  tests = kk + 1;
                  break;
                }
            }
            ntest += tests;
            nfar += far;
            nlive += live;
          }
          const uint32_t open = __ballot_sync(FULL, mine && !far);
          if (open) {
            const int topo = __shfl_sync(FULL, __float_as_int(V.w), 0);  // (uniform: the same record)
            if (topo != 0) {
              WN_DCHECK(sp < a.stack_depth, "traversal stack");
              stk[sp] = make_int2(topo, (int)open);  // every lane writes the same word: no divergence
              ++sp;
            } else {  // multi-point leaf (depth D): direct sum for the lanes that opened it
              const bool lm = (open >> lane) & 1u;
              const int j0 = __shfl_sync(FULL, a.nrange_pb[node], 0), j1 = __shfl_sync(FULL, a.nrange_pe[node], 0);
              WN_DCHECK(j0 >= 0 && j1 <= a.npts && j0 < j1, "leaf point range");
              if (COUNT) wvis += j1 - j0;
              for (int j = j0; j < j1; ++j) {
                const float4 P = __ldg(a.pts + j);
                float4 Vj;
                if (OP == OP_AT) Vj = make_float4(__ldg(a.scal + j), 0.f, 0.f, 0.f);
                else Vj = __ldg(a.vec + j);
                const float px = __fsub_rn(P.x, xq.x), py = __fsub_rn(P.y, xq.y), pz = __fsub_rn(P.z, xq.z);
                const float p2 = dist2(px, py, pz);
                const bool lv = lm && !(p2 < w2);
                acc.term(lv, px, py, pz, p2, Vj);
                if (COUNT && lm) {
                  ++nnear;
                  nlive += lv;
                  ntest += (__float_as_int(L.w) >> 13) & 1;  // a node whose children are all points
                }
              }
            }
          }
        }
      }
      acc.flush();  // (no trailing __syncwarp: every lane writes the same stack words and reads its own)
    }
  }
  // ---------------- epilogue (shared with the split kernel) ----------------
  if (COUNT && a.wvisits && active && lane == 0) a.wvisits[kq >> 5] = wvis;  // (lane 0's schedule position / 32)
  Work wk;
  wk.test = ntest;
  wk.far = nfar;
  wk.near = nnear;
  wk.live = nlive;
  trav_epilogue<OP, EPI, COUNT>(a, valid, q, acc, wk, active != 0u, kq >> 5);  // (kq: lane's position; q_begin % 32 = 0)
}

#ifndef WN_EXP_LBMIN
#define WN_EXP_LBMIN 6  // 6 resident blocks (48 warps) per SM: ≤ 42 registers, no spills; measured best
#endif
template <int OP, int EPI, bool COUNT, bool FROZEN, int ORD>
__global__ void __launch_bounds__(kTravBlock, (ORD == 1 ? 5 : WN_EXP_LBMIN) * 256 / kTravBlock) trav_kernel(const TravArgs a) {
  extern __shared__ int2 stk_all[];
  int2* stk = stk_all + (threadIdx.x >> 5) * a.stack_depth;
  trav_group<OP, EPI, COUNT, FROZEN, ORD>(a, stk, a.q_begin + (int64_t)blockIdx.x * kTravBlock + threadIdx.x);
}

// Small clouds (few query warps for the GPU): kSplit warps share each group of 32 queries.  All of them
// test the root; the root's children are split between them; the child groups of the children the lanes
// open are dealt round-robin; each warp traverses its share; the partial accumulators are added in warp
// order (a fixed order: deterministic), and one warp per group runs the epilogue.
// kSplit = KS ∈ {4, 8}: 8 for ≤ 512 query groups (capi.cu:split_factor; 2k points: −19 % per solve vs 4)
template <int OP, int EPI, bool COUNT, bool FROZEN, int ORD, int KS>
__global__ void __launch_bounds__(KS * (kTravBlock / 32) * 32) trav_split_kernel(const TravArgs a) {
  constexpr int kSplit = KS, kSplitWarps = KS * (kTravBlock / 32);
  constexpr int NG = kTravBlock / 32;  // query groups per block
  extern __shared__ int2 stk_all[];
  __shared__ uint32_t sm_open[NG][8];
  __shared__ int sm_topo[NG][8];
  __shared__ float sm_v[kSplitWarps][3][32];
  __shared__ double sm_d[kSplitWarps][32];
  __shared__ int sm_w[kSplitWarps][4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = warp / kSplit, sub = warp % kSplit;
  int2* stk = stk_all + warp * a.stack_depth;
  const int64_t kq = a.q_begin + (int64_t)blockIdx.x * kTravBlock + g * 32 + lane;
  const bool valid = kq < a.q_end;
  const int64_t q = (valid && a.qorder) ? (int64_t)a.qorder[kq] : kq;
  WN_DCHECK(!valid || (q >= 0 && (a.npts == 0 || a.queries != a.pts || q < a.npts)), "query index");
  const float4 xq = valid ? a.queries[q] : make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t active = __ballot_sync(FULL, valid);
  if (sub == 0 && lane < 8) sm_open[g][lane] = 0u;
  Acc<OP> acc;
  Work wk;
  uint32_t ropen = 0;
  int rtopo = 0;
  if (active) {  // the root: every warp of the group decides it, warp 0 keeps its term
    Acc<OP> scratch;
    Work wscratch;
    ropen = sub == 0 ? trav_visit<OP, COUNT, FROZEN, ORD>(a, 0, valid, xq, acc, wk, rtopo)
                     : trav_visit<OP, COUNT, FROZEN, ORD>(a, 0, valid, xq, scratch, wscratch, rtopo);
  }
  __syncthreads();
  if (ropen && rtopo != 0) {  // the root's children, child k by warp k mod kSplit
    const int c0 = rtopo >> 4, ncc = (rtopo & 7) + 1;
    for (int k = sub; k < ncc; k += kSplit) {
      int ctopo;
      const uint32_t copen =
          trav_visit<OP, COUNT, FROZEN, ORD>(a, c0 + k, (ropen >> lane) & 1u, xq, acc, wk, ctopo);
      if (lane == 0) {
        sm_open[g][k] = ctopo != 0 ? copen : 0u;
        sm_topo[g][k] = ctopo;
      }
    }
  }
  __syncthreads();
  if (ropen && rtopo != 0) {  // the opened children's groups, dealt round-robin, then this warp's share
    const int ncc = (rtopo & 7) + 1;
    int sp = 0, t = 0;
    for (int k = 0; k < ncc; ++k) {
      const uint32_t m = sm_open[g][k];
      if (!m) continue;
      const int tp = sm_topo[g][k];
      const int gc0 = tp >> 4, gn = (tp & 7) + 1;
      for (int j = 0; j < gn; ++j, ++t)
        if (t % kSplit == sub) {
          if (lane == 0) stk[sp] = make_int2((gc0 + j) << 4, (int)m);  // a group of one node
          ++sp;
        }
    }
    __syncwarp();
    trav_loop<OP, COUNT, FROZEN, ORD>(a, stk, sp, xq, acc, wk);
  }
  acc.flush();
  // the group's kSplit partial sums, added in warp order
  if (OP == OP_A) {
    sm_d[warp][lane] = acc.d;
  } else {
    sm_v[warp][0][lane] = acc.x;
    sm_v[warp][1][lane] = acc.y;
    sm_v[warp][2][lane] = acc.z;
  }
  if (COUNT) {
    sm_w[warp][0][lane] = wk.test;
    sm_w[warp][1][lane] = wk.far;
    sm_w[warp][2][lane] = wk.near;
    sm_w[warp][3][lane] = wk.live;
  }
  __syncthreads();
  if (sub == 0) {
    for (int s2 = 1; s2 < kSplit; ++s2) {
      const int w2 = warp + s2;
      if (OP == OP_A) {
        acc.d += sm_d[w2][lane];
      } else {
        acc.x += sm_v[w2][0][lane];
        acc.y += sm_v[w2][1][lane];
        acc.z += sm_v[w2][2][lane];
      }
      if (COUNT) {
        wk.test += sm_w[w2][0][lane];
        wk.far += sm_w[w2][1][lane];
        wk.near += sm_w[w2][2][lane];
        wk.live += sm_w[w2][3][lane];
      }
    }
  } else {
    wk = Work();
  }
  trav_epilogue<OP, EPI, COUNT>(a, valid && sub == 0, q, acc, wk, sub == 0 && active != 0u, kq >> 5);
}

template <int OP, int EPI, bool C, bool F, int O>
void launch_one(const TravArgs& a, cudaStream_t s, unsigned grid, size_t smem) {
  if (a.split == 8) {
    // eight warps' stacks per group plus the static combine arrays can pass the 48 KB default
    static const cudaError_t opt = cudaFuncSetAttribute(trav_split_kernel<OP, EPI, C, F, O, 8>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    (void)opt;
    trav_split_kernel<OP, EPI, C, F, O, 8><<<grid, 8 * kTravBlock, smem * 8, s>>>(a);
  }
  else if (a.split) {
    static const cudaError_t opt = cudaFuncSetAttribute(trav_split_kernel<OP, EPI, C, F, O, 4>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    (void)opt;
    trav_split_kernel<OP, EPI, C, F, O, 4><<<grid, 4 * kTravBlock, smem * 4, s>>>(a);
  }
  else trav_kernel<OP, EPI, C, F, O><<<grid, kTravBlock, smem, s>>>(a);
}

template <int OP, int EPI>
void launch(const TravArgs& a, cudaStream_t s, unsigned grid, size_t smem) {
  const bool cnt = a.work || a.qcounts || a.wvisits;
  if (OP == OP_A && EPI == EPI_SQ && a.attr) {  // frozen geometry (transpose-mode A(r)); order 0 only
    if (cnt) launch_one<OP, EPI, true, true, 0>(a, s, grid, smem);
    else launch_one<OP, EPI, false, true, 0>(a, s, grid, smem);
    return;
  }
  if (a.order1) {
    if (cnt) launch_one<OP, EPI, true, false, 1>(a, s, grid, smem);
    else launch_one<OP, EPI, false, false, 1>(a, s, grid, smem);
    return;
  }
  if (cnt) launch_one<OP, EPI, true, false, 0>(a, s, grid, smem);
  else launch_one<OP, EPI, false, false, 0>(a, s, grid, smem);
}

}  // namespace

// an empty shard still takes part in the peer-memory exchange: signal every rank
__global__ void k_peer_signal(TravArgs a) {
  __threadfence_system();
  for (int r = 0; r < a.world; ++r) atomicAdd_system(a.peer_sig[r], 1ull);
}

// Warp-level visits of a traversal under a query schedule (the schedule choice's estimate, capi.cu): the
// same walk as trav_kernel — decisions on the same offset, chains and pseudo-leaves as coded — without
// terms or leaf-point loads; per 32-query warp (every wstride-th warp of the schedule), child visits + the
// points of the leaves it opens.
__global__ void __launch_bounds__(kTravBlock) trav_visits_kernel(const TravArgs a) {
  extern __shared__ int2 stk_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int2* stk = stk_all + warp * a.stack_depth;
  const int64_t g = (int64_t)blockIdx.x * (kTravBlock / 32) + warp;  // counted warp → schedule warp g·wstride
  const int64_t kq = a.q_begin + g * a.wstride * 32 + lane;
  const bool valid = kq < a.q_end;
  const int64_t q = (valid && a.qorder) ? (int64_t)a.qorder[kq] : kq;
  const float4 xq = valid ? a.queries[q] : make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t active = __ballot_sync(FULL, valid);
  if (!active) return;
  const float4* __restrict__ G = a.nodes.rec;
  int wv = 0, sp = 1;
  if (lane == 0) stk[0] = make_int2(0, (int)active);
  __syncwarp();
  while (sp > 0) {
    --sp;
    const int2 e = stk[sp];
    __syncwarp();
    const int code = __shfl_sync(FULL, e.x, 0);  // (uniform trip count, as in trav_group)
    const int cb = code >> 4, ncc = (code & 7) + 1;
    const bool mine = ((uint32_t)e.y >> lane) & 1u;
    wv += ncc;
    for (int k = 0; k < ncc; ++k) {
      const int node = cb + k;
      const float4* rp = rec_at(G, node);
      const float4 R = __ldg(rp), L = __ldg(rp + 2);
      const float ex = __fadd_rn(__fsub_rn(R.x, xq.x), L.x), ey = __fadd_rn(__fsub_rn(R.y, xq.y), L.y),
                  ez = __fadd_rn(__fsub_rn(R.z, xq.z), L.z);
      const uint32_t open = __ballot_sync(FULL, mine && !(dist2(ex, ey, ez) > R.w));
      if (open) {
        const int topo = __shfl_sync(FULL, __float_as_int(__ldg(rp + 1).w), 0);
        if (topo != 0) {
          WN_DCHECK(sp < a.stack_depth, "visit-count stack");
          stk[sp] = make_int2(topo, (int)open);
          ++sp;
        } else {
          wv += a.nrange_pe[node] - a.nrange_pb[node];
        }
      }
    }
  }
  if (lane == 0) a.wvisits[g] = wv;
}

wn_status traverse_visits(const TravArgs& a, cudaStream_t s) {
  const int64_t nq = a.q_end - a.q_begin;
  if (nq <= 0) return WN_OK;
  const size_t smem = (size_t)(kTravBlock / 32) * a.stack_depth * sizeof(int2);
  const int64_t nw = ((nq + 31) / 32 + a.wstride - 1) / a.wstride;  // counted warps
  trav_visits_kernel<<<(unsigned)((nw + kTravBlock / 32 - 1) / (kTravBlock / 32)), kTravBlock, smem, s>>>(a);
  count_launches(1);
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

wn_status traverse(const TravArgs& a, cudaStream_t s) {
  const int64_t nq = a.q_end - a.q_begin;
  if (nq <= 0) {
    if (a.world) {
      k_peer_signal<<<1, 1, 0, s>>>(a);
      count_launches(1);
      WN_CUDA(cudaGetLastError());
    }
    return WN_OK;
  }
  const unsigned grid = (unsigned)trav_blocks(nq);
  const size_t smem = (size_t)(kTravBlock / 32) * a.stack_depth * sizeof(int2);
  const int cls = a.op == OP_A ? WN_PROF_TRAV_A : a.op == OP_AT ? WN_PROF_TRAV_AT : WN_PROF_TRAV_G;
  ProfScope ps(a.prof_cls >= 0 ? a.prof_cls : cls, s);
  TravArgs b = a;
  b.work = a.nowork ? nullptr : work_counters(cls);
  if (a.order1 && (!a.nodes.ext || a.attr)) return set_error(WN_ERR_ARG, "internal: order-1 traversal setup");
  switch (a.op * 8 + a.epi) {
    case OP_A * 8 + EPI_PLAIN: launch<OP_A, EPI_PLAIN>(b, s, grid, smem); break;
    case OP_A * 8 + EPI_S: launch<OP_A, EPI_S>(b, s, grid, smem); break;
    case OP_A * 8 + EPI_SQ: launch<OP_A, EPI_SQ>(b, s, grid, smem); break;
    case OP_AT * 8 + EPI_PLAIN: launch<OP_AT, EPI_PLAIN>(b, s, grid, smem); break;
    case OP_AT * 8 + EPI_R: launch<OP_AT, EPI_R>(b, s, grid, smem); break;
    case OP_G * 8 + EPI_PLAIN: launch<OP_G, EPI_PLAIN>(b, s, grid, smem); break;
    case OP_G * 8 + EPI_RESCALE: launch<OP_G, EPI_RESCALE>(b, s, grid, smem); break;
    default: return set_error(WN_ERR_ARG, "internal: unsupported traversal variant");
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

}  // namespace wn
