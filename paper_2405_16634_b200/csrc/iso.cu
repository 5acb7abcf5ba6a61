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
// mesher.  Corners are keyed on the level's lattice (Morton codes, 21 bits per axis), sorted and
// deduplicated, so a corner shared by up to eight cells is evaluated once, and evaluated in Z order — coherent
// warps without the per-call Hilbert schedule of wn_eval.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "wn_internal.cuh"

namespace wn {
namespace {

constexpr int kIsoBits = 21;
constexpr int64_t kIsoMaxCells = 1ll << 26;  // active cells per level (8 corner keys each, 32-bit scans)

// lattice points and cells are keyed by their Morton code (21 bits per axis, interleaved): sorted keys are a
// Z-order walk of the box, so the distinct corners come out spatially coherent for the traversal's warps,
// and a cell's children are its key × 8 + (0..7)
__host__ __device__ inline uint64_t spread3(uint64_t v) {  // 21 bits → every third bit
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}
__host__ __device__ inline uint64_t compact3(uint64_t v) {  // inverse of spread3
  v &= 0x1249249249249249ull;
  v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
  v = (v ^ (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v ^ (v >> 16)) & 0x1f00000000ffffull;
  v = (v ^ (v >> 32)) & 0x1fffff;
  return v;
}
__host__ __device__ inline uint64_t iso_key(uint64_t i, uint64_t j, uint64_t k) {
  return spread3(i) | (spread3(j) << 1) | (spread3(k) << 2);
}
__host__ __device__ inline void iso_ijk(uint64_t key, uint64_t& i, uint64_t& j, uint64_t& k) {
  i = compact3(key);
  j = compact3(key >> 1);
  k = compact3(key >> 2);
}

__global__ void k_iso_base(int level, uint64_t* __restrict__ cells) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t side = 1ll << level;
  if (c >= side * side * side) return;
  cells[c] = iso_key(c % side, (c / side) % side, c / (side * side));  // (any order: corners are sorted)
}

__global__ void k_iso_corner_keys(int64_t nc, const uint64_t* __restrict__ cells, uint64_t* __restrict__ ck) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 8 * nc) return;
  uint64_t i, j, k;
  iso_ijk(cells[t >> 3], i, j, k);
  const int b = (int)(t & 7);
  ck[t] = iso_key(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1));
}
// below the base level the active cells are the eight children of each kept parent, whose corners are the
// parent's 3 × 3 × 3 lattice points on the finer level: 27 keys per parent instead of 64
__global__ void k_iso_corner_keys27(int64_t np, const uint64_t* __restrict__ parents, uint64_t* __restrict__ ck) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 27 * np) return;
  uint64_t i, j, k;
  iso_ijk(parents[t / 27], i, j, k);
  const int b = (int)(t % 27);
  ck[t] = iso_key(2 * i + b % 3, 2 * j + (b / 3) % 3, 2 * k + b / 9);
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
  const uint64_t key = sk[i];
  const int64_t u = pos[i];
  uk[u] = key;
  uint64_t a, b, c;
  iso_ijk(key, a, b, c);
  const double inv = ldexp(1.0, -level);
  q[3 * u + 0] = (float)(lx + ex * ((double)a * inv));
  q[3 * u + 1] = (float)(ly + ey * ((double)b * inv));
  q[3 * u + 2] = (float)(lz + ez * ((double)c * inv));
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
  uint64_t ci, cj, ck3;
  iso_ijk(cells[c], ci, cj, ck3);
  float lo = 3.4e38f, hi = -3.4e38f;
  for (int b = 0; b < 8; ++b) {
    const uint64_t key = iso_key(ci + (b & 1), cj + ((b >> 1) & 1), ck3 + ((b >> 2) & 1));
    const float v = F[iso_find(uk, m, key)];
    cv[8 * c + b] = v;
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  keep[c] = final_level ? (lo < iso && hi >= iso) : (lo <= iso + band && hi >= iso - band);
}

__global__ void k_iso_children(int64_t nc, const uint64_t* __restrict__ cells, const uint32_t* __restrict__ keep,
                               const uint32_t* __restrict__ pos, uint64_t* __restrict__ next,
                               uint64_t* __restrict__ parents) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc || !keep[c]) return;
  parents[pos[c]] = cells[c];
  for (int b = 0; b < 8; ++b) next[8 * (int64_t)pos[c] + b] = cells[c] * 8 + (uint64_t)b;  // (Morton: children)
}

__global__ void k_iso_out(int64_t nc, const uint64_t* __restrict__ cells, const uint32_t* __restrict__ keep,
                          const uint32_t* __restrict__ pos, const float* __restrict__ cv, int64_t cap,
                          int32_t* __restrict__ out_cells, float* __restrict__ out_vals) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc || !keep[c]) return;
  const int64_t o = pos[c];
  if (o >= cap) return;
  uint64_t i, j, k;
  iso_ijk(cells[c], i, j, k);
  out_cells[3 * o + 0] = (int32_t)i;
  out_cells[3 * o + 1] = (int32_t)j;
  out_cells[3 * o + 2] = (int32_t)k;
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
  uint64_t *cur = nullptr, *par = nullptr;  // the level's cells; the previous level's kept cells (parents)
  tgt = &keep_;
  WN_TRY(alloc(&cur, nc * sizeof(uint64_t)));
  tgt = &lvl;
  k_iso_base<<<g256(nc), 256, 0, s>>>(base_level, cur);
  count_launches(1);
  int64_t total_evals = 0;
  const bool verbose = getenv("WN_ISO_VERBOSE") != nullptr;  // (diagnostic: per-level wall times on stderr)
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  for (int level = base_level;; ++level) {
    const auto t_lvl = tnow();
    const bool fin = level == max_level;
    *count = 0;
    if (nc == 0) break;
    // the level's distinct corners: 8 per cell on the base level, 27 per kept parent below it
    const int64_t m8 = level == base_level ? 8 * nc : 27 * (nc / 8);
    uint64_t *ck = nullptr, *sk = nullptr, *uk = nullptr;
    uint32_t *flag = nullptr, *pos = nullptr;
    WN_TRY(alloc(&ck, m8 * sizeof(uint64_t)));
    WN_TRY(alloc(&sk, m8 * sizeof(uint64_t)));
    WN_TRY(alloc(&flag, (m8 + 1) * sizeof(uint32_t)));
    WN_TRY(alloc(&pos, (m8 + 1) * sizeof(uint32_t)));
    if (level == base_level) k_iso_corner_keys<<<g256(m8), 256, 0, s>>>(nc, cur, ck);
    else k_iso_corner_keys27<<<g256(m8), 256, 0, s>>>(nc / 8, par, ck);
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
    const auto t_sort = tnow();
    WN_TRY(eval_field(t, mu, q, m, width, theta, F, s));  // the Alg. 4 traversal of wn_eval
    if (verbose) {
      cudaStreamSynchronize(s);
      fprintf(stderr, "wn_iso_cells level %d: %lld cells, %u corners, keys %.2f ms, F %.2f ms\n", level, (long long)nc, m,
              std::chrono::duration<double, std::milli>(t_sort - t_lvl).count(),
              std::chrono::duration<double, std::milli>(tnow() - t_sort).count());
    }
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
    for (void* p : keep_) lvl.push_back(p);  // the current cells and parents: freed with this level's buffers
    keep_.clear();
    tgt = &keep_;
    WN_TRY(alloc(&next, nn * sizeof(uint64_t)));
    WN_TRY(alloc(&par, std::max<int64_t>(nk, 1) * sizeof(uint64_t)));
    tgt = &lvl;
    if (nk > 0) {
      k_iso_children<<<g256(nc), 256, 0, s>>>(nc, cur, keep, kpos, next, par);
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
