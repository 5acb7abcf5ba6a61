/* oracle/wn_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of what the WNNC hot path computes
 * (Lin, Shi, Liu, "Fast and Globally Consistent Normal Orientation based on the Winding Number
 * Normal Consistency", arXiv 2405.16634).  Citations "PAPER.md:Lnnn (§, Eq/Alg)" point into
 * /root/reference/PAPER.md.  Readings where the paper is silent are the ones listed in
 * DESIGN.md §"Readings" (they follow SURVEY.md §8(c) c.2).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) may load it.
 * It shares nothing with the CUDA path; the two only see the same seeded inputs.
 *
 * Precision: fp64 for every value.  The two decisions that turn floating point into a branch —
 * the opening test |x_i − x_B| > c·width(B) (Alg. 4) and the smoothing cutoff |y| < w (§4.4) —
 * are taken in fp32 (the kernel's precision; the paper fixes none): for a node on the offset
 * d = (hi − y) + lo to its representative held as fp32 hi + lo, for a point on d = x_j − y, with
 * d² = fma(dx,dx, fma(dy,dy, dz·dz)), so that both sides decide identically on identical operands
 * (reading R-prec).
 *
 * Pins (tests/test_oracle_*.py): kernel identities and finite differences; Theorem-1 indicator
 * values; sphere closed forms for A, Aᵀ, G; dense adjointness / symmetry; treecode(c=∞) == dense;
 * treecode error decreasing in c; transpose-mode exact adjointness; tree invariants and SPEC
 * examples; the paper's Table 5 (mean / total solved area, level-7 icosphere); solver energy
 * monotonicity, sphere trajectory and WNNC ablation; the first-order far field (WO_ORDER1, SURVEY
 * §8 row f2 — an extension, not the paper's method) by Taylor decay rates, one-point-node identity,
 * c = ∞ and its error reduction (tests/test_oracle_order1.py).  No function is "parity unpinned".
 */
#include "wn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define WO_4PI (4.0 * 3.14159265358979323846)

/* ------------------------------------------------------------------------------------------ */
/* fp32 decisions (DESIGN.md R-prec)                                                           */
/* ------------------------------------------------------------------------------------------ */
static float d2_f32(const float a[3], const float b[3]) {
  float dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}
/* distance² to a representative held as fp32 hi + lo (lo = fp32 rounding of rep − hi):
   e = (hi − y) + lo per axis, all in fp32 — the fp32 evaluation of |x_B − y| (R-prec) */
static float d2_rep_f32(const float hi[3], const float lo[3], const float y[3]) {
  float ex = (hi[0] - y[0]) + lo[0], ey = (hi[1] - y[1]) + lo[1], ez = (hi[2] - y[2]) + lo[2];
  return fmaf(ex, ex, fmaf(ey, ey, ez * ez));
}

/* ------------------------------------------------------------------------------------------ */
/* Normalization: PAPER.md:L419 (§5.1.1) "normalized to fit into the cube [−1,1]^3 with a margin */
/* of 1/11": bbox-centred, uniform scale so the longest half-extent maps to 10/11.              */
/* ------------------------------------------------------------------------------------------ */
int wo_normalize(const float* raw, int64_t n, float* xn, double xf[4]) {
  if (n < 1) return 1;
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      double v = raw[3 * i + a];
      if (!isfinite(v)) return 2;
      if (v < lo[a]) lo[a] = v;
      if (v > hi[a]) hi[a] = v;
    }
  double half = 0.0;
  for (int a = 0; a < 3; ++a) {
    xf[a] = (lo[a] + hi[a]) * 0.5;
    double h = (hi[a] - lo[a]) * 0.5;
    if (h > half) half = h;
  }
  if (!(half > 0.0)) return 3;
  xf[3] = (10.0 / 11.0) / half;
  wo_normalize_apply(xf, raw, n, xn);
  return 0;
}

void wo_normalize_apply(const double xf[4], const float* raw, int64_t m, float* xn) {
  for (int64_t i = 0; i < m; ++i)
    for (int a = 0; a < 3; ++a) xn[3 * i + a] = (float)(((double)raw[3 * i + a] - xf[a]) * xf[3]);
}

/* Quantization into the 2^D grid of the root cube [−1,1]^3 (exact in fp64). */
static void quantize(const float* x, int D, uint32_t q[3]) {
  double cells = ldexp(1.0, D - 1);
  uint32_t qmax = (1u << D) - 1u;
  for (int a = 0; a < 3; ++a) {
    double v = floor(((double)x[a] + 1.0) * cells);
    if (v < 0.0) v = 0.0;
    if (v > (double)qmax) v = (double)qmax;
    q[a] = (uint32_t)v;
  }
}

/* octant digit of the level-l child (l = 1..D): bit (D−l) of each axis, x most significant */
static int octant(const uint32_t q[3], int D, int l) {
  int s = D - l;
  return (int)((((q[0] >> s) & 1u) << 2) | (((q[1] >> s) & 1u) << 1) | ((q[2] >> s) & 1u));
}

void wo_keys(const float* xn, int64_t n, int D, uint64_t* keys) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t q[3];
    quantize(xn + 3 * i, D, q);
    uint64_t k = 0;
    for (int l = 1; l <= D; ++l) k = (k << 3) | (uint64_t)octant(q, D, l);
    keys[i] = k;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Octree: PAPER.md:L370 (§4.5) "The partitioning stops if the node contains only one point or */
/* if the user-specified maximum depth D is reached."  Recursive stable octant partition.       */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  int depth, nchild;
  int64_t pb, pe;      /* Morton positions [pb, pe) of the points in the node */
  int64_t child[8];    /* node ids, ascending octant digit                    */
} wo_node;

struct wo_tree {
  int64_t n;
  int D;
  const float* xn;     /* borrowed, n×3 normalized fp32 (caller order) */
  uint32_t* q;         /* n×3 quantized */
  int64_t* order;      /* order[k] = caller index of the k-th point in Morton order */
  wo_node* nodes;      /* node 0 = root, ids assigned in DFS order */
  int64_t nn, cap;
  int64_t* bfs;        /* bfs[k] = node id at BFS position k */
  int64_t* bfs_of;     /* bfs_of[id] = BFS position */
  int maxdepth;
};

static int64_t new_node(wo_tree* t, int depth) {
  if (t->nn == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 1024;
    t->nodes = (wo_node*)realloc(t->nodes, (size_t)t->cap * sizeof(wo_node));
  }
  wo_node* nd = &t->nodes[t->nn];
  memset(nd, 0, sizeof(*nd));
  nd->depth = depth;
  if (depth > t->maxdepth) t->maxdepth = depth;
  return t->nn++;
}

static void build_rec(wo_tree* t, int64_t id, const int64_t* idx, int64_t cnt, int64_t* pos) {
  int depth = t->nodes[id].depth;
  t->nodes[id].pb = *pos;
  if (cnt == 1 || depth == t->D) {             /* leaf */
    for (int64_t k = 0; k < cnt; ++k) t->order[(*pos)++] = idx[k];
    t->nodes[id].pe = *pos;
    return;
  }
  int64_t count[8] = {0}, off[8];
  for (int64_t k = 0; k < cnt; ++k) count[octant(t->q + 3 * idx[k], t->D, depth + 1)]++;
  off[0] = 0;
  for (int d = 1; d < 8; ++d) off[d] = off[d - 1] + count[d - 1];
  int64_t* part = (int64_t*)malloc((size_t)cnt * sizeof(int64_t));
  int64_t fill[8];
  memcpy(fill, off, sizeof(fill));
  for (int64_t k = 0; k < cnt; ++k) part[fill[octant(t->q + 3 * idx[k], t->D, depth + 1)]++] = idx[k];
  for (int d = 0; d < 8; ++d) {
    if (!count[d]) continue;
    int64_t c = new_node(t, depth + 1);
    t->nodes[id].child[t->nodes[id].nchild++] = c;
    build_rec(t, c, part + off[d], count[d], pos);
  }
  free(part);
  t->nodes[id].pe = *pos;
}

wo_tree* wo_tree_build(const float* xn, int64_t n, int D) {
  if (n < 1 || D < 1 || D > 21) return NULL;
  wo_tree* t = (wo_tree*)calloc(1, sizeof(wo_tree));
  t->n = n;
  t->D = D;
  t->xn = xn;
  t->q = (uint32_t*)malloc((size_t)n * 3 * sizeof(uint32_t));
  for (int64_t i = 0; i < n; ++i) quantize(xn + 3 * i, D, t->q + 3 * i);
  t->order = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t* idx = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  int64_t pos = 0;
  int64_t root = new_node(t, 0);
  build_rec(t, root, idx, n, &pos);
  free(idx);
  /* BFS relabelling (queue order; children consecutive, ascending digit) */
  t->bfs = (int64_t*)malloc((size_t)t->nn * sizeof(int64_t));
  t->bfs_of = (int64_t*)malloc((size_t)t->nn * sizeof(int64_t));
  int64_t head = 0, tail = 0;
  t->bfs[tail++] = root;
  while (head < tail) {
    int64_t id = t->bfs[head++];
    for (int c = 0; c < t->nodes[id].nchild; ++c) t->bfs[tail++] = t->nodes[id].child[c];
  }
  for (int64_t k = 0; k < t->nn; ++k) t->bfs_of[t->bfs[k]] = k;
  return t;
}

void wo_tree_free(wo_tree* t) {
  if (!t) return;
  free(t->q); free(t->order); free(t->nodes); free(t->bfs); free(t->bfs_of);
  free(t);
}

int64_t wo_tree_num_nodes(const wo_tree* t) { return t->nn; }
int wo_tree_max_depth(const wo_tree* t) { return t->maxdepth; }

void wo_tree_export(const wo_tree* t, int32_t* perm, int32_t* depth, int32_t* pb, int32_t* pe,
                    int32_t* child_begin, int32_t* child_count) {
  for (int64_t k = 0; k < t->n; ++k) perm[k] = (int32_t)t->order[k];
  for (int64_t k = 0; k < t->nn; ++k) {
    const wo_node* nd = &t->nodes[t->bfs[k]];
    depth[k] = nd->depth;
    pb[k] = (int32_t)nd->pb;
    pe[k] = (int32_t)nd->pe;
    child_count[k] = nd->nchild;
    child_begin[k] = nd->nchild ? (int32_t)t->bfs_of[nd->child[0]] : -1;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Representatives: PAPER.md:L371-L378 (§4.5, Eqs node-rep-loc / node-rep-vec)                 */
/*   x_{B,ν} = Σ_{i∈B} |ν_i| x_i / Σ_{j∈B} |ν_j| ,  ν_B = Σ_{i∈B} ν_i                           */
/* Σ|ν| = 0 ⇒ unweighted centroid (values unaffected since ν_B = 0).             */
/* One-point node ⇒ x_B = x_j exactly.  Direct sum over the node's points (plain definition).   */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  double* rep;   /* nn×3 (node id order) */
  float* repf;   /* nn×3 fp32 rounding of rep: hi (decision operand) */
  float* lof;    /* nn×3 fp32 rounding of rep − hi: lo (decision operand) */
  double* V;     /* nn×dim */
  double* W;     /* nn */
  float* thrf;   /* nn: (c·width)^2 in fp32 */
  double* X;     /* first-order moments (WO_ORDER1) or NULL: dim 3: M (nn×9, row-major M_ab =
                    Σ_j ν_j,a (x_j − x_B)_b); dim 1: D (nn×3, D = Σ_j s_j (x_j − x_B)) */
  int dim;
} wo_reps;

static void node_moment(const wo_tree* t, int64_t id, const double* nu, int dim, double rep[3], double* V,
                        double* Wout) {
  const wo_node* nd = &t->nodes[id];
  double W = 0, P[3] = {0, 0, 0}, C[3] = {0, 0, 0};
  for (int c = 0; c < dim; ++c) V[c] = 0;
  for (int64_t k = nd->pb; k < nd->pe; ++k) {
    int64_t j = t->order[k];
    const double* v = nu + (size_t)dim * j;
    double a = dim == 3 ? sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]) : fabs(v[0]);
    W += a;
    for (int c = 0; c < 3; ++c) {
      double x = t->xn[3 * j + c];
      P[c] += a * x;
      C[c] += x;
    }
    for (int c = 0; c < dim; ++c) V[c] += v[c];
  }
  int64_t cnt = nd->pe - nd->pb;
  for (int c = 0; c < 3; ++c) {
    if (cnt == 1) rep[c] = t->xn[3 * t->order[nd->pb] + c];
    else if (W > 0) rep[c] = P[c] / W;
    else rep[c] = C[c] / (double)cnt;
  }
  *Wout = W;
}

/* opening threshold (c·width)^2, width = full cell edge 2^{1−depth} of the root cube [−1,1]^3
   ("c·(the width of B)"; DESIGN.md R-width), fp32 (R-prec). */
static float thr_f32(double theta, int depth) {
  if (isinf(theta)) return INFINITY;
  float cw = (float)theta * ldexpf(1.0f, 1 - depth);
  return cw * cw;
}

/* first-order moments of node id about its representative, from the definition (row f2) */
static void node_moment1(const wo_tree* t, int64_t id, const double* nu, int dim, const double rep[3], double* X) {
  const wo_node* nd = &t->nodes[id];
  int nx = dim == 3 ? 9 : 3;
  for (int c = 0; c < nx; ++c) X[c] = 0;
  for (int64_t k = nd->pb; k < nd->pe; ++k) {
    int64_t j = t->order[k];
    const double* v = nu + (size_t)dim * j;
    double d[3];
    for (int c = 0; c < 3; ++c) d[c] = (double)t->xn[3 * j + c] - rep[c];
    if (dim == 3) {
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) X[3 * a + b] += v[a] * d[b];
    } else {
      for (int c = 0; c < 3; ++c) X[c] += v[0] * d[c];
    }
  }
}

static void reps_compute_o(const wo_tree* t, const double* nu, int dim, double theta, int order1, wo_reps* r);
static void reps_compute(const wo_tree* t, const double* nu, int dim, double theta, wo_reps* r) {
  reps_compute_o(t, nu, dim, theta, 0, r);
}
static void reps_compute_o(const wo_tree* t, const double* nu, int dim, double theta, int order1, wo_reps* r) {
  r->dim = dim;
  r->X = order1 ? (double*)malloc((size_t)t->nn * (dim == 3 ? 9 : 3) * sizeof(double)) : NULL;
  r->rep = (double*)malloc((size_t)t->nn * 3 * sizeof(double));
  r->repf = (float*)malloc((size_t)t->nn * 3 * sizeof(float));
  r->lof = (float*)malloc((size_t)t->nn * 3 * sizeof(float));
  r->V = (double*)malloc((size_t)t->nn * dim * sizeof(double));
  r->W = (double*)malloc((size_t)t->nn * sizeof(double));
  r->thrf = (float*)malloc((size_t)t->nn * sizeof(float));
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t id = 0; id < t->nn; ++id) {
    node_moment(t, id, nu, dim, r->rep + 3 * id, r->V + (size_t)dim * id, r->W + id);
    for (int c = 0; c < 3; ++c) {
      r->repf[3 * id + c] = (float)r->rep[3 * id + c];
      r->lof[3 * id + c] = (float)(r->rep[3 * id + c] - (double)r->repf[3 * id + c]);
    }
    r->thrf[id] = thr_f32(theta, t->nodes[id].depth);
    if (order1) node_moment1(t, id, nu, dim, r->rep + 3 * id, r->X + (size_t)(dim == 3 ? 9 : 3) * id);
  }
}

static void reps_free(wo_reps* r) {
  free(r->rep); free(r->repf); free(r->lof); free(r->V); free(r->W); free(r->thrf); free(r->X);
}

void wo_moments(const wo_tree* t, const double* nu, int dim, double* rep, double* attr, double* W) {
  wo_reps r;
  reps_compute(t, nu, dim, 2.0, &r);
  for (int64_t k = 0; k < t->nn; ++k) {
    int64_t id = t->bfs[k];
    for (int c = 0; c < 3; ++c) rep[3 * k + c] = r.rep[3 * id + c];
    for (int c = 0; c < dim; ++c) attr[(size_t)dim * k + c] = r.V[(size_t)dim * id + c];
    W[k] = r.W[id];
  }
  reps_free(&r);
}

/* ------------------------------------------------------------------------------------------ */
/* Kernels (fp64).  PAPER.md:L213 ∇Φ(y) = −y/(4π|y|^3);                          */
/* HΦ(y) = −I/(4π|y|^3) + 3yyᵀ/(4π|y|^5); both set to 0 if |y| < w (§4.4) —     */
/* the cutoff decision is made by the caller in fp32.                                          */
/* term(op, y, x, ν): contribution of source x with attribute ν to the query y.                */
/* ------------------------------------------------------------------------------------------ */
static void term(int op, const double y[3], const double x[3], const double* nu, double* acc) {
  /* op | WO_ABS: accumulate |contribution| instead (the per-query conditioning scale Σ_j |term_j|) */
  int absm = op & WO_ABS;
  op &= ~(WO_ABS | WO_ORDER1);
  double t[3] = {0, 0, 0};
  double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};     /* d = y − x */
  double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  double r = sqrt(r2);
  double k3 = 1.0 / (WO_4PI * r2 * r);                        /* 1/(4π r^3) */
  if (op == WO_OP_A) {
    /* ∇Φ(y−x)·ν = −(y−x)·ν / (4π r^3)    (Eq wnf-discretization) */
    t[0] = -(d[0] * nu[0] + d[1] * nu[1] + d[2] * nu[2]) * k3;
  } else if (op == WO_OP_G) {
    /* −HΦ(y−x)ν = ν/(4π r^3) − 3 (d·ν) d/(4π r^5) */
    double dn = d[0] * nu[0] + d[1] * nu[1] + d[2] * nu[2];
    double k5 = 3.0 * k3 / r2;
    for (int c = 0; c < 3; ++c) t[c] = nu[c] * k3 - dn * d[c] * k5;
  } else {
    /* ν ∇Φ(x−y) = ν (y−x)/(4π r^3)   (Aᵀ: (Aᵀs)_j = Σ_i s_i ∇Φ(x_i − x_j)) */
    for (int c = 0; c < 3; ++c) t[c] = nu[0] * d[c] * k3;
  }
  if (absm) acc[0] += sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  else for (int c = 0; c < 3; ++c) acc[c] += t[c];
}

/* First-order far field (the paper uses order 0 only, and
   cites Barill et al. for expansions, L409).  For a far node B with sources x_j = x_B + d_j, the
   contribution Σ_j f(x_j) of op's kernel f is expanded to first order in d_j about x_B:
   Σ_j f(x_j) ≈ f(x_B)·(ν_B) + Σ_j ∇_x f(x_B)·d_j.  With u = x_B − y, r = |u|, M_ab = Σ_j ν_j,a d_j,b
   (vector attribute) or D = Σ_j s_j d_j (scalar):
     A : f = u·ν/(4πr³)                    → [tr M − 3 uᵀMu/r²] / (4π r³)
     G : f = [ν − 3(u·ν)u/r²]/(4πr³)       → [−3(Mu + u tr M + Mᵀu) + 15 (uᵀMu) u/r²] / (4π r⁵)
     Aᵀ: f = −s u/(4πr³)                   → −[D − 3 u (u·D)/r²] / (4π r³)
   Adds the correction for source (x_B, X) at query y into t[3]. */
static void term1(int op, const double y[3], const double xB[3], const double* X, double t[3]) {
  double u[3] = {xB[0] - y[0], xB[1] - y[1], xB[2] - y[2]};
  double r2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  double r = sqrt(r2);
  double k3 = 1.0 / (WO_4PI * r2 * r);
  if (op == WO_OP_AT) {
    double uD = u[0] * X[0] + u[1] * X[1] + u[2] * X[2];
    for (int c = 0; c < 3; ++c) t[c] += -(X[c] - 3.0 * u[c] * uD / r2) * k3;
    return;
  }
  double Mu[3], MTu[3], tr = X[0] + X[4] + X[8];
  for (int a = 0; a < 3; ++a) {
    Mu[a] = X[3 * a] * u[0] + X[3 * a + 1] * u[1] + X[3 * a + 2] * u[2];
    MTu[a] = X[a] * u[0] + X[3 + a] * u[1] + X[6 + a] * u[2];
  }
  double uMu = u[0] * Mu[0] + u[1] * Mu[1] + u[2] * Mu[2];
  if (op == WO_OP_A) {
    t[0] += (tr - 3.0 * uMu / r2) * k3;
  } else {
    double k5 = k3 / r2;
    for (int c = 0; c < 3; ++c) t[c] += (-3.0 * (Mu[c] + u[c] * tr + MTu[c]) + 15.0 * uMu * u[c] / r2) * k5;
  }
}

/* far-node contribution: order 0 (term) plus, if X, the first-order correction; |·| under WO_ABS */
static void term_far(int op, const double y[3], const double xB[3], const double* nuB, const double* X,
                     double* acc) {
  int absm = op & WO_ABS, base = op & ~(WO_ABS | WO_ORDER1);
  double t[3] = {0, 0, 0};
  term(base, y, xB, nuB, t);
  if (X) term1(base, y, xB, X, t);
  if (absm) acc[0] += sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  else for (int c = 0; c < 3; ++c) acc[c] += t[c];
}

static int out_dim(int op) { return ((op & ~WO_ORDER1) == WO_OP_A || (op & WO_ABS)) ? 1 : 3; }

/* ------------------------------------------------------------------------------------------ */
/* Dense operators: the O(N^2) definitions.              */
/* ------------------------------------------------------------------------------------------ */
void wo_dense_op(const wo_tree* t, int op, const double* nu, int dim, const float* qf, int64_t m, double w,
                 double* out) {
  const float* Q = qf ? qf : t->xn;
  if (!qf) m = t->n;
  float wf = (float)w, w2f = wf * wf;
  int od = out_dim(op);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < m; ++i) {
    const float* yf = Q + 3 * i;
    double y[3] = {yf[0], yf[1], yf[2]};
    double acc[3] = {0, 0, 0};
    for (int64_t j = 0; j < t->n; ++j) {
      const float* xf = t->xn + 3 * j;
      if (d2_f32(xf, yf) < w2f) continue;
      double x[3] = {xf[0], xf[1], xf[2]};
      term(op, y, x, nu + (size_t)dim * j, acc);
    }
    for (int c = 0; c < od; ++c) out[(size_t)od * i + c] = acc[c];
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Treecode: Algorithm 4 apply_A, literally and recursively:               */
/*   if |x_i − x_B| > c·width(B): representative term ("modified by w")                         */
/*   elif B is not a leaf:        recurse into the children                                     */
/*   else:                        direct sum over the points of B ("modified by w")             */
/* "Other operators Aᵀ and G are accelerated in the same way" (L406) with ν = s for Aᵀ (L371).  */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const wo_tree* t;
  const wo_reps* geo;    /* reps + thresholds that decide (and locate) far terms */
  const double* Vattr;   /* node attribute sums used in far terms (node id order) */
  const double* nu;      /* point attributes (caller order) for leaf terms */
  int dim, op;
  float w2f;
} trav_ctx;

typedef struct { int64_t tests, far, near, ties; } wo_cnt;

static int near_tie(float d2, float thr) { return isfinite(thr) && thr > 0 && fabsf(d2 - thr) <= 1e-5f * thr; }

static void trav(const trav_ctx* c, int64_t id, const double y[3], const float yf[3], double* acc, wo_cnt* k) {
  const wo_node* nd = &c->t->nodes[id];
  float d2 = d2_rep_f32(c->geo->repf + 3 * id, c->geo->lof + 3 * id, yf);
  k->tests++;
  if (near_tie(d2, c->geo->thrf[id])) k->ties++;
  if (d2 > c->geo->thrf[id]) {                                  /* far: representative */
    k->far++;
    if (near_tie(d2, c->w2f)) k->ties++;
    if (!(d2 < c->w2f)) {
      const double* X = c->geo->X ? c->geo->X + (size_t)(c->dim == 3 ? 9 : 3) * id : NULL;
      term_far(c->op, y, c->geo->rep + 3 * id, c->Vattr + (size_t)c->dim * id, X, acc);
    }
  } else if (nd->nchild) {
    for (int ch = 0; ch < nd->nchild; ++ch) trav(c, nd->child[ch], y, yf, acc, k);
  } else {                                                      /* leaf: direct sum */
    for (int64_t p = nd->pb; p < nd->pe; ++p) {
      int64_t j = c->t->order[p];
      const float* xf = c->t->xn + 3 * j;
      float dj = d2_f32(xf, yf);
      k->near++;
      if (near_tie(dj, c->w2f)) k->ties++;
      if (dj < c->w2f) continue;
      double x[3] = {xf[0], xf[1], xf[2]};
      term(c->op, y, x, c->nu + (size_t)c->dim * j, acc);
    }
  }
}

static void run_queries(const trav_ctx* c, const float* qf, const int64_t* qidx, int64_t m, double* out,
                        int64_t* counters) {
  const wo_tree* t = c->t;
  if (!qf && !qidx) m = t->n;
  int od = out_dim(c->op);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < m; ++i) {
    const float* yf = qf ? qf + 3 * i : t->xn + 3 * (qidx ? qidx[i] : i);
    double y[3] = {yf[0], yf[1], yf[2]};
    double acc[3] = {0, 0, 0};
    wo_cnt k = {0, 0, 0, 0};
    trav(c, 0, y, yf, acc, &k);
    for (int d = 0; d < od; ++d) out[(size_t)od * i + d] = acc[d];
    if (counters) {
      counters[4 * i + 0] = k.tests; counters[4 * i + 1] = k.far;
      counters[4 * i + 2] = k.near;  counters[4 * i + 3] = k.ties;
    }
  }
}

void wo_tree_op(const wo_tree* t, int op, const double* nu, int dim, const float* qf, const int64_t* qidx,
                int64_t m, double w, double theta, double* out, int64_t* counters) {
  wo_reps r;
  reps_compute_o(t, nu, dim, theta, (op & WO_ORDER1) != 0, &r);
  float wf = (float)w;
  trav_ctx c = {t, &r, r.V, nu, dim, op, wf * wf};
  run_queries(&c, qf, qidx, m, out, counters);
  reps_free(&r);
}

/* Frozen geometry (north-star transpose form): reps + decisions from mu_geom,
   attribute sums from nu. */
void wo_tree_A_frozen(const wo_tree* t, const double* mu_geom, const double* nu, double w, double theta,
                      double* out) {
  wo_reps g, a;
  reps_compute(t, mu_geom, 3, theta, &g);
  reps_compute(t, nu, 3, theta, &a);
  float wf = (float)w;
  trav_ctx c = {t, &g, a.V, nu, 3, WO_OP_A, wf * wf};
  run_queries(&c, NULL, NULL, t->n, out, NULL);
  reps_free(&g);
  reps_free(&a);
}

/* Exact transpose of the frozen-geometry treecode A: for every query i, each far node B receives
   s_i ∇Φ(x_i − x_B) and each near point j receives s_i ∇Φ(x_i − x_j); then every point collects
   its own term plus the terms of all nodes containing it (push-down). */
static void trav_T(const trav_ctx* c, int64_t id, const double y[3], const float yf[3], double s, double* VB,
                   double* U) {
  const wo_node* nd = &c->t->nodes[id];
  float d2 = d2_rep_f32(c->geo->repf + 3 * id, c->geo->lof + 3 * id, yf);
  if (d2 > c->geo->thrf[id]) {
    if (!(d2 < c->w2f)) {
      const double* x = c->geo->rep + 3 * id;
      double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
      double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      double k3 = 1.0 / (WO_4PI * r2 * sqrt(r2));
      for (int a = 0; a < 3; ++a) VB[3 * id + a] += -s * d[a] * k3;   /* s ∇Φ(y − x_B) */
    }
  } else if (nd->nchild) {
    for (int ch = 0; ch < nd->nchild; ++ch) trav_T(c, nd->child[ch], y, yf, s, VB, U);
  } else {
    for (int64_t p = nd->pb; p < nd->pe; ++p) {
      int64_t j = c->t->order[p];
      const float* xf = c->t->xn + 3 * j;
      if (d2_f32(xf, yf) < c->w2f) continue;
      double d[3] = {y[0] - xf[0], y[1] - xf[1], y[2] - xf[2]};
      double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      double k3 = 1.0 / (WO_4PI * r2 * sqrt(r2));
      for (int a = 0; a < 3; ++a) U[3 * j + a] += -s * d[a] * k3;     /* s ∇Φ(y − x_j) */
    }
  }
}

void wo_tree_AT_transpose(const wo_tree* t, const double* mu_geom, const double* s, double w, double theta,
                          double* out) {
  wo_reps g;
  reps_compute(t, mu_geom, 3, theta, &g);
  float wf = (float)w;
  trav_ctx c = {t, &g, g.V, NULL, 3, WO_OP_A, wf * wf};
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  size_t nv = (size_t)t->nn * 3, nu = (size_t)t->n * 3;
  double* VB = (double*)calloc((size_t)nt * nv, sizeof(double));
  double* U = (double*)calloc((size_t)nt * nu, sizeof(double));
#pragma omp parallel num_threads(nt)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
#pragma omp for schedule(static)
    for (int64_t i = 0; i < t->n; ++i) {
      const float* yf = t->xn + 3 * i;
      double y[3] = {yf[0], yf[1], yf[2]};
      trav_T(&c, 0, y, yf, s[i], VB + (size_t)tid * nv, U + (size_t)tid * nu);
    }
  }
  for (int th = 1; th < nt; ++th) {            /* fixed-order reduction of per-thread partials */
    for (size_t k = 0; k < nv; ++k) VB[k] += VB[(size_t)th * nv + k];
    for (size_t k = 0; k < nu; ++k) U[k] += U[(size_t)th * nu + k];
  }
  /* push-down: out_j = U_j + Σ_{B ∋ j} V_B */
  for (int64_t j = 0; j < t->n; ++j)
    for (int a = 0; a < 3; ++a) out[3 * j + a] = U[3 * j + a];
  for (int64_t id = 0; id < t->nn; ++id) {
    const wo_node* nd = &t->nodes[id];
    for (int64_t p = nd->pb; p < nd->pe; ++p) {
      int64_t j = t->order[p];
      for (int a = 0; a < 3; ++a) out[3 * j + a] += VB[3 * id + a];
    }
  }
  free(VB);
  free(U);
  reps_free(&g);
}

/* ------------------------------------------------------------------------------------------ */
/* Solver: Algorithm 3 with grad_step = Algorithm 2.  */
/*   w_k = w2 (n−k)/(n−1) + w1 (k−1)/(n−1)          (n = 1 ⇒ w1)                   */
/*   s = b − A_w μ (b = ½);  r = A_wᵀ s;  α = rᵀr / ‖A_w r‖² (0 if ‖A_w r‖ = 0);  μ' = μ + α r    */
/*   μ̂ = G_w(μ');  μ_i = μ̂_i |μ'_i| / |μ̂_i|  (keep μ'_i if |μ̂_i| = 0)                           */
/* ------------------------------------------------------------------------------------------ */
static double width_at(int k, int n, double w1, double w2) {
  if (n == 1) return w1;
  return w2 * (double)(n - k) / (double)(n - 1) + w1 * (double)(k - 1) / (double)(n - 1);
}

/* FMM solver backend (row f4): degree, separation θ_f, leaf size (wo_fmm_config); separation width = w2 */
static int g_fmm_p = 4, g_fmm_leaf = 32;
static double g_fmm_theta = 0.5, g_fmm_wsep = 0.0;
void wo_fmm_config(int p, double theta, int leaf) { g_fmm_p = p; g_fmm_theta = theta; g_fmm_leaf = leaf; }

static void apply(const wo_tree* t, int backend, int op, const double* nu, int dim, double w, double theta,
                  double* out) {
  if (backend == 1) wo_dense_op(t, op, nu, dim, NULL, t->n, w, out);
  else if (backend == 2) wo_fmm_op_sep(t, op & ~WO_ORDER1, nu, dim, w, g_fmm_wsep, g_fmm_p, g_fmm_theta, g_fmm_leaf, out,
                                       NULL);
  else wo_tree_op(t, op, nu, dim, NULL, NULL, t->n, w, theta, out, NULL);
}

/* WNNC update's rescale (Alg. 3): μ_i = μ̂_i |μ'_i| / |μ̂_i| — the new direction μ̂_i with
   the length of the grad-step result μ'_i; |μ̂_i| = 0 keeps μ'_i (reading R-rescale). */
void wo_rescale(int64_t n, const double* mp, const double* mh, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double a = sqrt(mp[3 * i] * mp[3 * i] + mp[3 * i + 1] * mp[3 * i + 1] + mp[3 * i + 2] * mp[3 * i + 2]);
    double h = sqrt(mh[3 * i] * mh[3 * i] + mh[3 * i + 1] * mh[3 * i + 1] + mh[3 * i + 2] * mh[3 * i + 2]);
    for (int c = 0; c < 3; ++c) out[3 * i + c] = h > 0 ? mh[3 * i + c] * (a / h) : mp[3 * i + c];
  }
}

int wo_solve(const wo_tree* t, double* mu, double w1, double w2, int iters, int first_iter, int total_iters,
             double theta, int backend, int mode, int wnnc, int order, double* stats) {
  const int o1 = (order == 1 && backend == 0) ? WO_ORDER1 : 0;
  int64_t n = t->n;
  double* s = (double*)malloc((size_t)n * sizeof(double));
  double* r = (double*)malloc((size_t)n * 3 * sizeof(double));
  double* q = (double*)malloc((size_t)n * sizeof(double));
  double* mp = (double*)malloc((size_t)n * 3 * sizeof(double));
  double* mh = (double*)malloc((size_t)n * 3 * sizeof(double));
  int transpose = (mode == 1 && backend == 0);
  g_fmm_wsep = (double)(float)w2;  /* the FMM backend's separation width: the schedule's largest w (fp32, as the GPU) */
  for (int it = 0; it < iters; ++it) {
    int k = first_iter + it;
    /* the width is handed to the kernels as fp32; both sides use the same rounding */
    double w = (double)(float)width_at(k, total_iters, w1, w2);
    /* grad step */
    apply(t, backend, WO_OP_A | o1, mu, 3, w, theta, s);
    double E = 0;
    for (int64_t i = 0; i < n; ++i) { s[i] = 0.5 - s[i]; E += s[i] * s[i]; }
    if (transpose) wo_tree_AT_transpose(t, mu, s, w, theta, r);
    else apply(t, backend, WO_OP_AT | o1, s, 1, w, theta, r);
    if (transpose) wo_tree_A_frozen(t, mu, r, w, theta, q);
    else apply(t, backend, WO_OP_A | o1, r, 3, w, theta, q);
    double rr = 0, qq = 0;
    for (int64_t i = 0; i < n; ++i) {
      rr += r[3 * i] * r[3 * i] + r[3 * i + 1] * r[3 * i + 1] + r[3 * i + 2] * r[3 * i + 2];
      qq += q[i] * q[i];
    }
    double alpha = qq > 0 ? rr / qq : 0.0;
    for (int64_t i = 0; i < 3 * n; ++i) mp[i] = mu[i] + alpha * r[i];
    /* WNNC update + rescale */
    if (wnnc) {
      apply(t, backend, WO_OP_G | o1, mp, 3, w, theta, mh);
      wo_rescale(n, mp, mh, mu);
    } else {
      memcpy(mu, mp, (size_t)n * 3 * sizeof(double));
    }
    if (stats) {
      stats[5 * it + 0] = E; stats[5 * it + 1] = alpha; stats[5 * it + 2] = rr;
      stats[5 * it + 3] = qq; stats[5 * it + 4] = w;
    }
  }
  free(s); free(r); free(q); free(mp); free(mh);
  return 0;
}

int wo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------------------------ */
/* Fast multipole method (SURVEY §8 row f4 — the paper's future work, §6.3 and  */
/* L409; not the paper's method).  The same sums as the dense operators (PAPER.md:L222, L266,  */
/* L316), written as one potential                                                             */
/*   V(y) = Σ_j [ q_j Φ(y − x_j) + ν_j·∇Φ(y − x_j) ],   Φ(r) = 1/(4π|r|)                          */
/* so that A(ν) = V (dipoles ν), G(ν) = −∇V (dipoles ν) and Aᵀ(s) = −∇V (charges q = s).         */
/* Cells = octree nodes (cube centres c, radius = half-diagonal √3·2^−depth); an FMM leaf is a  */
/* node with no children or at most `leaf` points.  Cartesian Taylor expansions of total degree */
/* ≤ p, plain textbook steps:                                                                  */
/*   P2M  M_β = Σ_j [ q_j (−1)^|β| (x_j−c)^β/β! + Σ_k ν_jk (−1)^(|β|−1) (x_j−c)^(β−e_k)/(β−e_k)! ] */
/*        (Taylor of Φ(y − x) in x about c:  V(y) = Σ_β M_β ∂^βΦ(y − c))                         */
/*   M2M  M'_β = Σ_{γ≤β} M_γ (c'−c)^(β−γ)/(β−γ)!                     (child c → parent c')       */
/*   M2L  L_γ += Σ_β M_β ∂^(β+γ)Φ(c_t − c_s)          (local Taylor coefficients L_γ = ∂^γV(c_t)) */
/*   L2L  L'_δ = Σ_{γ≥δ} L_γ (c'−c)^(γ−δ)/(γ−δ)!                      (parent c → child c')       */
/*   L2P  V(y) = Σ_γ L_γ (y−c)^γ/γ!,  ∂_k V(y) = Σ_γ L_γ (y−c)^(γ−e_k)/(γ−e_k)!                   */
/* ∂^δ(1/|R|) = δ! b_δ from the Taylor-coefficient recurrence (b_0 = 1/|R|)                      */
/*   |δ| |R|² b_δ = −(2|δ|−1) Σ_i R_i b_(δ−e_i) − (|δ|−1) Σ_i b_(δ−2e_i).                         */
/* Dual traversal from (root, root): a cell pair is well separated — one M2L — iff              */
/* |c_t − c_s| > (r_t + r_s)/θ_f and |c_t − c_s| − r_t − r_s > w (every pair beyond the smoothing */
/* cutoff: the expansion is of the unsmoothed kernel, exact there); else two leaves interact   */
/* directly (P2P: the definition, cutoff r < w decided in fp32 as in wo_dense_op); else the     */
/* larger cell (the target on ties) is split.  θ_f → 0 makes every pair direct: the dense sums. */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  int p, P, np, nP;      /* expansion degree p, derivative degree P = 2p; coefficient counts */
  int* mi;               /* nP × 3 multi-indices, by total degree, then lexicographic (a, b, c) desc */
  int* lut;              /* (P+1)^3 → index or −1 */
  double* fact;          /* fact[k] = k! */
} fmm_idx;

static int fmm_count(int p) { return (p + 1) * (p + 2) * (p + 3) / 6; }

static void fmm_idx_init(fmm_idx* I, int p) {
  I->p = p;
  I->P = 2 * p;
  I->np = fmm_count(p);
  I->nP = fmm_count(I->P);
  int P1 = I->P + 1;
  I->mi = (int*)malloc((size_t)I->nP * 3 * sizeof(int));
  I->lut = (int*)malloc((size_t)P1 * P1 * P1 * sizeof(int));
  for (int k = 0; k < P1 * P1 * P1; ++k) I->lut[k] = -1;
  int n = 0;
  for (int deg = 0; deg <= I->P; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b) {
        int c = deg - a - b;
        I->mi[3 * n] = a; I->mi[3 * n + 1] = b; I->mi[3 * n + 2] = c;
        I->lut[(a * P1 + b) * P1 + c] = n++;
      }
  I->fact = (double*)malloc((size_t)(I->P + 2) * sizeof(double));
  I->fact[0] = 1.0;
  for (int k = 1; k <= I->P + 1; ++k) I->fact[k] = I->fact[k - 1] * k;
}

static void fmm_idx_free(fmm_idx* I) { free(I->mi); free(I->lut); free(I->fact); }

static int fmm_at(const fmm_idx* I, int a, int b, int c) {
  if (a < 0 || b < 0 || c < 0 || a + b + c > I->P) return -1;
  int P1 = I->P + 1;
  return I->lut[(a * P1 + b) * P1 + c];
}

/* x^α / α! for every |α| ≤ deg (first fmm_count(deg) entries) */
static void fmm_monomials(const fmm_idx* I, const double x[3], int deg, double* out) {
  int n = fmm_count(deg);
  for (int k = 0; k < n; ++k) {
    const int* a = I->mi + 3 * k;
    out[k] = pow(x[0], a[0]) * pow(x[1], a[1]) * pow(x[2], a[2]) / (I->fact[a[0]] * I->fact[a[1]] * I->fact[a[2]]);
  }
}

/* T_δ = ∂^δ Φ(R), |δ| ≤ P, Φ = 1/(4π|R|); b: nP scratch */
static void fmm_derivs(const fmm_idx* I, const double R[3], double* T, double* b) {
  double r2 = R[0] * R[0] + R[1] * R[1] + R[2] * R[2];
  b[0] = 1.0 / sqrt(r2);
  for (int k = 1; k < I->nP; ++k) {
    const int* d = I->mi + 3 * k;
    int n = d[0] + d[1] + d[2];
    double s = 0.0;
    for (int i = 0; i < 3; ++i) {
      int e[3] = {d[0], d[1], d[2]};
      e[i] -= 1;
      int j = fmm_at(I, e[0], e[1], e[2]);
      if (j >= 0) s -= (2.0 * n - 1.0) * R[i] * b[j];
      e[i] -= 1;
      j = fmm_at(I, e[0], e[1], e[2]);
      if (j >= 0) s -= (n - 1.0) * b[j];
    }
    b[k] = s / (n * r2);
  }
  for (int k = 0; k < I->nP; ++k) {
    const int* d = I->mi + 3 * k;
    T[k] = b[k] * I->fact[d[0]] * I->fact[d[1]] * I->fact[d[2]] / WO_4PI;
  }
}

typedef struct {
  const wo_tree* t;
  fmm_idx I;
  int leaf, dim;           /* dim 1: charges q (Aᵀ), dim 3: dipoles ν (A, G) */
  double theta, w, wsep;   /* cutoff w of the direct sums; separation width of the well-separated test */
  float w2f;
  double* ctr;             /* nn × 3 cube centres (node id order) */
  double* rad;             /* nn half-diagonals */
  double* M;               /* nn × np multipole coefficients */
  double* L;               /* nn × np local coefficients */
  const double* nu;        /* caller order */
  double* pot;             /* n × 4: V, ∂V (caller order), accumulated */
  int64_t m2l, p2p;        /* counters: M2L cell pairs, P2P leaf pairs */
} fmm_ctx;

static int fmm_is_leaf(const fmm_ctx* f, int64_t id) {
  const wo_node* nd = &f->t->nodes[id];
  return nd->nchild == 0 || nd->pe - nd->pb <= f->leaf;
}

static void fmm_up(fmm_ctx* f, int64_t id) {
  const wo_node* nd = &f->t->nodes[id];
  const fmm_idx* I = &f->I;
  double* M = f->M + (size_t)id * I->np;
  const double* c = f->ctr + 3 * id;
  if (fmm_is_leaf(f, id)) {  /* P2M */
    double* mono = (double*)malloc((size_t)I->np * sizeof(double));
    for (int64_t k = nd->pb; k < nd->pe; ++k) {
      int64_t j = f->t->order[k];
      double x[3];
      for (int a = 0; a < 3; ++a) x[a] = (double)f->t->xn[3 * j + a] - c[a];
      fmm_monomials(I, x, I->p, mono);
      const double* v = f->nu + (size_t)f->dim * j;
      for (int b = 0; b < I->np; ++b) {
        const int* be = I->mi + 3 * b;
        int deg = be[0] + be[1] + be[2];
        if (f->dim == 1) {
          M[b] += v[0] * ((deg & 1) ? -1.0 : 1.0) * mono[b];
        } else {
          for (int kk = 0; kk < 3; ++kk) {
            int e[3] = {be[0], be[1], be[2]};
            e[kk] -= 1;
            int g = fmm_at(I, e[0], e[1], e[2]);
            if (g >= 0 && g < I->np) M[b] += v[kk] * ((deg - 1) & 1 ? -1.0 : 1.0) * mono[g];
          }
        }
      }
    }
    free(mono);
    return;
  }
  double* shift = (double*)malloc((size_t)I->np * sizeof(double));
  for (int ci = 0; ci < nd->nchild; ++ci) {  /* M2M, children in octant order */
    int64_t ch = nd->child[ci];
    fmm_up(f, ch);
    const double* Mc = f->M + (size_t)ch * I->np;
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = c[a] - f->ctr[3 * ch + a];  /* c' − c (parent − child) */
    fmm_monomials(I, d, I->p, shift);
    for (int b = 0; b < I->np; ++b) {
      const int* be = I->mi + 3 * b;
      for (int g = 0; g <= b; ++g) {
        const int* ge = I->mi + 3 * g;
        int s = fmm_at(I, be[0] - ge[0], be[1] - ge[1], be[2] - ge[2]);
        if (s >= 0) M[b] += Mc[g] * shift[s];
      }
    }
  }
  free(shift);
}

static void fmm_p2p(fmm_ctx* f, int64_t T, int64_t S) {
  const wo_node* nt = &f->t->nodes[T];
  const wo_node* ns = &f->t->nodes[S];
  for (int64_t a = nt->pb; a < nt->pe; ++a) {
    int64_t i = f->t->order[a];
    const float* yf = f->t->xn + 3 * i;
    double* out = f->pot + 4 * i;
    for (int64_t b = ns->pb; b < ns->pe; ++b) {
      int64_t j = f->t->order[b];
      const float* xf = f->t->xn + 3 * j;
      if (d2_f32(xf, yf) < f->w2f) continue;  /* smoothing cutoff (§4.4), fp32 decision (R-prec) */
      double d[3] = {(double)yf[0] - xf[0], (double)yf[1] - xf[1], (double)yf[2] - xf[2]};
      double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2], r = sqrt(r2);
      double k1 = 1.0 / (WO_4PI * r), k3 = k1 / r2, k5 = 3.0 * k3 / r2;
      const double* v = f->nu + (size_t)f->dim * j;
      if (f->dim == 1) {  /* q Φ(d): V += q/(4πr), ∇V += −q d/(4πr³) */
        out[0] += v[0] * k1;
        for (int c = 0; c < 3; ++c) out[1 + c] -= v[0] * d[c] * k3;
      } else {  /* ν·∇Φ(d) = −(d·ν)/(4πr³);  ∇(ν·∇Φ)(d) = HΦ(d)ν = 3(d·ν)d/(4πr⁵) − ν/(4πr³) */
        double dn = d[0] * v[0] + d[1] * v[1] + d[2] * v[2];
        out[0] -= dn * k3;
        for (int c = 0; c < 3; ++c) out[1 + c] += dn * d[c] * k5 - v[c] * k3;
      }
    }
  }
  f->p2p++;  /* one leaf pair */
}

static void fmm_m2l(fmm_ctx* f, int64_t T, int64_t S, double* Tbuf) {
  const fmm_idx* I = &f->I;
  double R[3];
  for (int a = 0; a < 3; ++a) R[a] = f->ctr[3 * T + a] - f->ctr[3 * S + a];
  fmm_derivs(I, R, Tbuf, Tbuf + I->nP);
  const double* M = f->M + (size_t)S * I->np;
  double* L = f->L + (size_t)T * I->np;
  for (int g = 0; g < I->np; ++g) {
    const int* ge = I->mi + 3 * g;
    double acc = 0.0;
    for (int b = 0; b < I->np; ++b) {
      const int* be = I->mi + 3 * b;
      acc += M[b] * Tbuf[fmm_at(I, be[0] + ge[0], be[1] + ge[1], be[2] + ge[2])];
    }
    L[g] += acc;
  }
  f->m2l++;
}

static void fmm_dual(fmm_ctx* f, int64_t T, int64_t S, double* Tbuf) {
  const double* ct = f->ctr + 3 * T;
  const double* cs = f->ctr + 3 * S;
  double d = sqrt((ct[0] - cs[0]) * (ct[0] - cs[0]) + (ct[1] - cs[1]) * (ct[1] - cs[1]) +
                  (ct[2] - cs[2]) * (ct[2] - cs[2]));
  double rt = f->rad[T], rs = f->rad[S];
  if (d * f->theta > rt + rs && d - rt - rs > f->wsep) {
    fmm_m2l(f, T, S, Tbuf);
    return;
  }
  int lt = fmm_is_leaf(f, T), ls = fmm_is_leaf(f, S);
  if (lt && ls) {
    fmm_p2p(f, T, S);
    return;
  }
  const wo_node* nt = &f->t->nodes[T];
  const wo_node* ns = &f->t->nodes[S];
  if (ls || (!lt && rt >= rs)) {
    for (int c = 0; c < nt->nchild; ++c) fmm_dual(f, nt->child[c], S, Tbuf);
  } else {
    for (int c = 0; c < ns->nchild; ++c) fmm_dual(f, T, ns->child[c], Tbuf);
  }
}

static void fmm_down(fmm_ctx* f, int64_t id) {
  const wo_node* nd = &f->t->nodes[id];
  const fmm_idx* I = &f->I;
  const double* L = f->L + (size_t)id * I->np;
  const double* c = f->ctr + 3 * id;
  double* mono = (double*)malloc((size_t)I->np * sizeof(double));
  if (fmm_is_leaf(f, id)) {  /* L2P */
    for (int64_t k = nd->pb; k < nd->pe; ++k) {
      int64_t i = f->t->order[k];
      double y[3];
      for (int a = 0; a < 3; ++a) y[a] = (double)f->t->xn[3 * i + a] - c[a];
      fmm_monomials(I, y, I->p, mono);
      double* out = f->pot + 4 * i;
      for (int g = 0; g < I->np; ++g) {
        const int* ge = I->mi + 3 * g;
        out[0] += L[g] * mono[g];
        for (int kk = 0; kk < 3; ++kk) {
          int e[3] = {ge[0], ge[1], ge[2]};
          e[kk] -= 1;
          int h = fmm_at(I, e[0], e[1], e[2]);
          if (h >= 0) out[1 + kk] += L[g] * mono[h];
        }
      }
    }
    free(mono);
    return;
  }
  for (int ci = 0; ci < nd->nchild; ++ci) {  /* L2L */
    int64_t ch = nd->child[ci];
    double* Lc = f->L + (size_t)ch * I->np;
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = f->ctr[3 * ch + a] - c[a];  /* c' − c (child − parent) */
    fmm_monomials(I, d, I->p, mono);
    for (int dl = 0; dl < I->np; ++dl) {
      const int* de = I->mi + 3 * dl;
      for (int g = 0; g < I->np; ++g) {
        const int* ge = I->mi + 3 * g;
        int s = fmm_at(I, ge[0] - de[0], ge[1] - de[1], ge[2] - de[2]);
        if (s >= 0 && s < I->np) Lc[dl] += L[g] * mono[s];
      }
    }
    fmm_down(f, ch);
  }
  free(mono);
}

void wo_fmm_op(const wo_tree* t, int op, const double* nu, int dim, double w, int p, double theta, int leaf,
               double* out, int64_t* counts) {
  wo_fmm_op_sep(t, op, nu, dim, w, w, p, theta, leaf, out, counts);
}

/* the same with a separation width wsep ≥ w (a solve keeps one set of lists for every iteration's width:
   wsep = the schedule's w2, so every expanded pair is beyond each iteration's cutoff) */
void wo_fmm_op_sep(const wo_tree* t, int op, const double* nu, int dim, double w, double wsep, int p, double theta,
                   int leaf, double* out, int64_t* counts) {
  fmm_ctx f;
  memset(&f, 0, sizeof(f));
  f.t = t;
  fmm_idx_init(&f.I, p);
  f.leaf = leaf;
  f.dim = dim;
  f.theta = theta;
  f.w = w;
  f.wsep = wsep;
  float wf = (float)w;
  f.w2f = wf * wf;
  f.nu = nu;
  f.ctr = (double*)malloc((size_t)t->nn * 3 * sizeof(double));
  f.rad = (double*)malloc((size_t)t->nn * sizeof(double));
  for (int64_t id = 0; id < t->nn; ++id) {  /* cube of the node: its first point's cell at its depth */
    const wo_node* nd = &t->nodes[id];
    const uint32_t* q = t->q + 3 * t->order[nd->pb];
    double edge = ldexp(1.0, 1 - nd->depth);
    for (int a = 0; a < 3; ++a) {
      uint32_t cell = nd->depth == 0 ? 0u : q[a] >> (t->D - nd->depth);
      f.ctr[3 * id + a] = -1.0 + ((double)cell + 0.5) * edge;
    }
    f.rad[id] = sqrt(3.0) * 0.5 * edge;
  }
  f.M = (double*)calloc((size_t)t->nn * f.I.np, sizeof(double));
  f.L = (double*)calloc((size_t)t->nn * f.I.np, sizeof(double));
  f.pot = (double*)calloc((size_t)t->n * 4, sizeof(double));
  double* Tbuf = (double*)malloc((size_t)2 * f.I.nP * sizeof(double));  /* T and the recurrence's b */
  int64_t root = t->bfs[0];
  fmm_up(&f, root);
  fmm_dual(&f, root, root, Tbuf);
  fmm_down(&f, root);
  for (int64_t i = 0; i < t->n; ++i) {
    const double* v = f.pot + 4 * i;
    if (op == WO_OP_A) out[i] = v[0];
    else for (int c = 0; c < 3; ++c) out[3 * i + c] = -v[1 + c];  /* G = −∇V (dipoles), Aᵀ = −∇V (charges) */
  }
  if (counts) { counts[0] = f.m2l; counts[1] = f.p2p; }
  free(Tbuf); free(f.pot); free(f.L); free(f.M); free(f.rad); free(f.ctr);
  fmm_idx_free(&f.I);
}
