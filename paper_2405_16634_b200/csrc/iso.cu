// iso.cu — adaptive octree sampling of the winding-number field around its ½ level set (SURVEY §8 row f1:
// "wn_eval on M ≫ N arbitrary queries (a 256³–512³ grid or adaptive octree samples) → WNF iso-surface at ½";
// the reconstruction hand-off of PAPER.md:L1005-L1008, "plugging these normals back into the winding
// number field (WNF)").
//
// The box is cut into 2^L0 cells per axis; per level the field F (Eq. wnf-discretization, PAPER.md:L222,
// through the same Alg. 4 traversal as wn_eval) is evaluated once at every distinct corner of the active
// cells, a cell stays active if its corner values come within `band` of the iso value (min ≤ iso + band and
// max ≥ iso − band), and every active cell is split in eight.  At the finest level the cells the level set
// crosses (min < iso ≤ max) are returned with their eight corner values: the input of a marching-cubes
// mesher.  Corners are keyed on the level's lattice (21 bits per axis), sorted and deduplicated, so a
// corner shared by up to eight cells is evaluated once.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "wn_internal.cuh"

namespace wn {
namespace {

constexpr int kIsoBits = 21;
constexpr uint64_t kIsoMask = (1ull << kIsoBits) - 1;
constexpr int64_t kIsoMaxCells = 1ll << 26;  // active cells per level (8 corner keys each, 32-bit scans)

__host__ __device__ inline uint64_t iso_key(uint64_t i, uint64_t j, uint64_t k) {
  return i | (j << kIsoBits) | (k << (2 * kIsoBits));
}

__global__ void k_iso_base(int level, uint64_t* __restrict__ cells) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t side = 1ll << level;
  if (c >= side * side * side) return;
  cells[c] = iso_key(c % side, (c / side) % side, c / (side * side));
}

__global__ void k_iso_corner_keys(int64_t nc, const uint64_t* __restrict__ cells, uint64_t* __restrict__ ck) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 8 * nc) return;
  const uint64_t c = cells[t >> 3];
  const int b = (int)(t & 7);
  ck[t] = iso_key((c & kIsoMask) + (b & 1), ((c >> kIsoBits) & kIsoMask) + ((b >> 1) & 1),
                  (c >> (2 * kIsoBits)) + ((b >> 2) & 1));
}

__global__ void k_iso_uniq_flag(int64_t m, const uint64_t* __restrict__ sk, uint32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) flag[i] = (i == 0 || sk[i] != sk[i - 1]) ? 1u : 0u;
}

// the distinct corners, and their positions in the input frame: lo + (hi − lo)·idx / 2^level
__global__ void k_iso_uniq(int64_t m, const uint64_t* __restrict__ sk, const uint32_t* __restrict__ flag,
                           const uint32_t* __restrict__ pos, int level, double lx, double ly, double lz, double ex,
                           double ey, double ez, uint64_t* __restrict__ uk, float* __restrict__ q) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m || !flag[i]) return;
  const uint64_t k = sk[i];
  const int64_t u = pos[i];
  uk[u] = k;
  const double inv = ldexp(1.0, -level);
  q[3 * u + 0] = (float)(lx + ex * ((double)(k & kIsoMask) * inv));
  q[3 * u + 1] = (float)(ly + ey * ((double)((k >> kIsoBits) & kIsoMask) * inv));
  q[3 * u + 2] = (float)(lz + ez * ((double)(k >> (2 * kIsoBits)) * inv));
}

__device__ __forceinline__ int64_t iso_find(const uint64_t* __restrict__ uk, int64_t m, uint64_t key) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (uk[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// per cell: its corner values (binary search among the level's distinct corners) and the decision
__global__ void k_iso_decide(int64_t nc, const uint64_t* __restrict__ cells, const uint64_t* __restrict__ uk,
                             int64_t m, const float* __restrict__ F, float iso, float band, int final_level,
                             float* __restrict__ cv, uint32_t* __restrict__ keep) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const uint64_t k = cells[c];
  float lo = 3.4e38f, hi = -3.4e38f;
  for (int b = 0; b < 8; ++b) {
    const uint64_t key = iso_key((k & kIsoMask) + (b & 1), ((k >> kIsoBits) & kIsoMask) + ((b >> 1) & 1),
                                 (k >> (2 * kIsoBits)) + ((b >> 2) & 1));
    const float v = F[iso_find(uk, m, key)];
    cv[8 * c + b] = v;
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  keep[c] = final_level ? (lo < iso && hi >= iso) : (lo <= iso + band && hi >= iso - band);
}

__global__ void k_iso_children(int64_t nc, const uint64_t* __restrict__ cells, const uint32_t* __restrict__ keep,
                               const uint32_t* __restrict__ pos, uint64_t* __restrict__ next) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc || !keep[c]) return;
  const uint64_t k = cells[c];
  const uint64_t i = 2 * (k & kIsoMask), j = 2 * ((k >> kIsoBits) & kIsoMask), l = 2 * (k >> (2 * kIsoBits));
  for (int b = 0; b < 8; ++b) next[8 * (int64_t)pos[c] + b] = iso_key(i + (b & 1), j + ((b >> 1) & 1), l + ((b >> 2) & 1));
}

__global__ void k_iso_out(int64_t nc, const uint64_t* __restrict__ cells, const uint32_t* __restrict__ keep,
                          const uint32_t* __restrict__ pos, const float* __restrict__ cv, int64_t cap,
                          int32_t* __restrict__ out_cells, float* __restrict__ out_vals) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc || !keep[c]) return;
  const int64_t o = pos[c];
  if (o >= cap) return;
  const uint64_t k = cells[c];
  out_cells[3 * o + 0] = (int32_t)(k & kIsoMask);
  out_cells[3 * o + 1] = (int32_t)((k >> kIsoBits) & kIsoMask);
  out_cells[3 * o + 2] = (int32_t)(k >> (2 * kIsoBits));
  for (int b = 0; b < 8; ++b) out_vals[8 * o + b] = cv[8 * c + b];
}

inline unsigned g256(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace
}  // namespace wn

using namespace wn;

extern "C" wn_status wn_iso_cells(wn_tree t, const float* mu, float width, float theta, const float box[6],
                                  int32_t base_level, int32_t max_level, float iso, float band, int64_t capacity,
                                  int32_t* cells, float* values, int64_t* count, int64_t* evals, void* stream) {
  if (!t || !mu || !box || !count) return set_error(WN_ERR_ARG, "tree, mu, box or count is NULL");
  if (base_level < 0 || base_level > 7 || max_level < base_level || max_level > 20)
    return set_error(WN_ERR_ARG, "levels: 0 <= base_level <= 7, base_level <= max_level <= 20");
  if (!(band >= 0.f)) return set_error(WN_ERR_ARG, "band must be >= 0");
  if (capacity < 0 || (capacity > 0 && (!cells || !values))) return set_error(WN_ERR_ARG, "bad output buffers");
  for (int a = 0; a < 3; ++a)
    if (!(box[3 + a] > box[a])) return set_error(WN_ERR_ARG, "box: hi must exceed lo on every axis");
  cudaStream_t s = (cudaStream_t)stream;
  // scratch: `lvl` holds one level's buffers (freed when the level is done), `keep_` the active cells
  std::vector<void*> lvl, keep_;
  struct Rel {
    std::vector<void*>& v;
    cudaStream_t s;
    ~Rel() {
      for (void* p : v) cudaFreeAsync(p, s);
      v.clear();
    }
  } rel_a{lvl, s}, rel_b{keep_, s};
  std::vector<void*>* tgt = &lvl;
  auto alloc = [&](auto** p, size_t bytes) -> wn_status {
    cudaError_t e = cudaMallocAsync((void**)p, std::max<size_t>(bytes, 8), s);
    if (e != cudaSuccess) return cuda_status(e, "wn_iso_cells scratch");
    tgt->push_back((void*)*p);
    return WN_OK;
  };
  const double lx = box[0], ly = box[1], lz = box[2];
  const double ex = (double)box[3] - box[0], ey = (double)box[4] - box[1], ez = (double)box[5] - box[2];
  int64_t nc = 1ll << (3 * base_level);  // ≤ 2^21
  uint64_t* cur = nullptr;
  tgt = &keep_;
  WN_TRY(alloc(&cur, nc * sizeof(uint64_t)));
  tgt = &lvl;
  k_iso_base<<<g256(nc), 256, 0, s>>>(base_level, cur);
  count_launches(1);
  int64_t total_evals = 0;
  for (int level = base_level;; ++level) {
    const bool fin = level == max_level;
    *count = 0;
    if (nc == 0) break;
    // the level's distinct corners
    const int64_t m8 = 8 * nc;
    uint64_t *ck = nullptr, *sk = nullptr, *uk = nullptr;
    uint32_t *flag = nullptr, *pos = nullptr;
    WN_TRY(alloc(&ck, m8 * sizeof(uint64_t)));
    WN_TRY(alloc(&sk, m8 * sizeof(uint64_t)));
    WN_TRY(alloc(&flag, (m8 + 1) * sizeof(uint32_t)));
    WN_TRY(alloc(&pos, (m8 + 1) * sizeof(uint32_t)));
    k_iso_corner_keys<<<g256(m8), 256, 0, s>>>(nc, cur, ck);
    WN_TRY(sort_keys_u64(ck, m8, 3 * kIsoBits, sk, s));
    k_iso_uniq_flag<<<g256(m8), 256, 0, s>>>(m8, sk, flag);
    WN_TRY(scan_u32(flag, pos, m8, pos + m8, s));
    uint32_t m = 0;
    WN_CUDA(cudaMemcpyAsync(&m, pos + m8, sizeof(m), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    float *q = nullptr, *F = nullptr, *cv = nullptr;
    WN_TRY(alloc(&uk, (size_t)m * sizeof(uint64_t)));
    WN_TRY(alloc(&q, (size_t)m * 3 * sizeof(float)));
    WN_TRY(alloc(&F, (size_t)m * sizeof(float)));
    k_iso_uniq<<<g256(m8), 256, 0, s>>>(m8, sk, flag, pos, level, lx, ly, lz, ex, ey, ez, uk, q);
    count_launches(3);
    WN_TRY(eval_field(t, mu, q, m, width, theta, F, s));  // the Alg. 4 traversal of wn_eval
    total_evals += m;
    // decisions
    uint32_t *keep = nullptr, *kpos = nullptr;
    WN_TRY(alloc(&cv, (size_t)nc * 8 * sizeof(float)));
    WN_TRY(alloc(&keep, (nc + 1) * sizeof(uint32_t)));
    WN_TRY(alloc(&kpos, (nc + 1) * sizeof(uint32_t)));
    k_iso_decide<<<g256(nc), 256, 0, s>>>(nc, cur, uk, m, F, iso, band, fin ? 1 : 0, cv, keep);
    WN_TRY(scan_u32(keep, kpos, nc, kpos + nc, s));
    uint32_t nk = 0;
    WN_CUDA(cudaMemcpyAsync(&nk, kpos + nc, sizeof(nk), cudaMemcpyDeviceToHost, s));
    WN_CUDA(cudaStreamSynchronize(s));
    count_launches(1);
    if (fin) {
      if (nk > 0 && capacity > 0) {
        k_iso_out<<<g256(nc), 256, 0, s>>>(nc, cur, keep, kpos, cv, capacity, cells, values);
        count_launches(1);
      }
      *count = nk;
      break;
    }
    const int64_t nn = 8 * (int64_t)nk;
    if (nn > kIsoMaxCells) return set_error(WN_ERR_ARG, "wn_iso_cells: more than 2^26 active cells (lower max_level)");
    uint64_t* next = nullptr;
    for (void* p : keep_) lvl.push_back(p);  // the current cells: freed with this level's buffers
    keep_.clear();
    tgt = &keep_;
    WN_TRY(alloc(&next, nn * sizeof(uint64_t)));
    tgt = &lvl;
    if (nk > 0) {
      k_iso_children<<<g256(nc), 256, 0, s>>>(nc, cur, keep, kpos, next);
      count_launches(1);
    }
    for (void* p : lvl) cudaFreeAsync(p, s);  // stream-ordered: after this level's kernels
    lvl.clear();
    cur = next;
    nc = nn;
  }
  if (evals) *evals = total_evals;
  WN_CUDA(cudaGetLastError());
  WN_CUDA(cudaStreamSynchronize(s));
  return WN_OK;
}
