/* oracle/wn_oracle.h — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain, slow, fp64 CPU oracle for the WNNC hot path (arXiv 2405.16634).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or helper with the
 * CUDA path under paper_2405_16634_b200/ and never reads anything the CUDA path wrote.
 *
 * Citations "PAPER.md:Lnnn" refer to /root/reference/PAPER.md (LaTeX source of the paper).
 * Every function works in the NORMALIZED frame (§5.1.1) on the fp32 normalized
 * coordinates produced by wo_normalize; frame mapping lives in oracle/__init__.py.
 *
 * Parity status of each function: see the header comment of wn_oracle.c.
 */
#ifndef WN_ORACLE_H
#define WN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wo_tree wo_tree;

enum { WO_OP_A = 0,   /* Σ ∇Φ(y−x_j)·ν_j          (A, and the field F at arbitrary y) */
       WO_OP_G = 1,   /* −Σ HΦ(y−x_j) ν_j         (G, and −∇F at arbitrary y)         */
       WO_OP_AT = 2,  /* Σ ν_i ∇Φ(x_i−y), ν scalar (Aᵀ, gather form)                  */
       WO_ABS = 8,    /* modifier: accumulate |term| (conditioning scale S = Σ_j |term_j|)  */
       WO_ORDER1 = 16 /* modifier: first-order far field (not the paper's):   */
                      /* a far node adds the first-order Taylor term of its sources about x_B  */ };

/* §5.1.1 normalization; returns 0, 1 (empty), 2 (non-finite), 3 (zero extent). */
int wo_normalize(const float* raw, int64_t n, float* xn, double xf[4]);
/* apply an existing transform (queries) */
void wo_normalize_apply(const double xf[4], const float* raw, int64_t m, float* xn);
void wo_keys(const float* xn, int64_t n, int D, uint64_t* keys);

wo_tree* wo_tree_build(const float* xn, int64_t n, int D);
void wo_tree_free(wo_tree* t);
int64_t wo_tree_num_nodes(const wo_tree* t);
int wo_tree_max_depth(const wo_tree* t);
/* BFS layout: perm[k] = caller index of the k-th point in Morton order;
   per BFS node: depth, pb, pe (Morton positions), child_begin (BFS index), child_count */
void wo_tree_export(const wo_tree* t, int32_t* perm, int32_t* depth, int32_t* pb, int32_t* pe,
                    int32_t* child_begin, int32_t* child_count);
/* §4.5 Eqs node-rep-loc / node-rep-vec for attribute nu (caller order, dim 1 or 3); BFS order out */
void wo_moments(const wo_tree* t, const double* nu, int dim, double* rep, double* attr, double* W);

/* dense O(N·M) operator (definition).  qf = m×3 fp32 normalized queries or NULL (queries = sources). */
void wo_dense_op(const wo_tree* t, int op, const double* nu, int dim,
                 const float* qf, int64_t m, double w, double* out);
/* treecode (Alg. 4).  qf as above; if qf == NULL, qidx (m caller indices) selects source queries,
   qidx == NULL means all n sources.  theta = c; theta = +inf ⇒ never use a representative.
   counters (m×4 or NULL): tests, far terms, near terms, tie-band hits. */
void wo_tree_op(const wo_tree* t, int op, const double* nu, int dim, const float* qf,
                const int64_t* qidx, int64_t m, double w, double theta, double* out, int64_t* counters);
/* Treecode A at frozen geometry g = (reps, decisions) of mu_geom, applied to nu (dim 3). */
void wo_tree_A_frozen(const wo_tree* t, const double* mu_geom, const double* nu, double w, double theta,
                      double* out);
/* Exact transpose of wo_tree_A_frozen(mu_geom, ·): out_j = Σ_i s_i ∂(T_g ν)_i/∂ν_j (dim 3). */
void wo_tree_AT_transpose(const wo_tree* t, const double* mu_geom, const double* s, double w, double theta,
                          double* out);

/* FMM (not the paper's method; see wn_oracle.c): op WO_OP_A (nu dim 3: A(ν), n out),
   WO_OP_G (dim 3: G(ν), n×3) or WO_OP_AT (dim 1: Aᵀ(s), n×3) at the n sources, caller order, normalized
   frame; expansion degree p, separation θ_f, at most `leaf` points per FMM leaf; counts (2 or NULL):
   M2L cell pairs, P2P leaf pairs. */
void wo_fmm_op(const wo_tree* t, int op, const double* nu, int dim, double w, int p, double theta, int leaf,
               double* out, int64_t* counts);
/* the same with a separation width wsep ≥ w for the well-separated test (w stays the direct sums' cutoff) */
void wo_fmm_op_sep(const wo_tree* t, int op, const double* nu, int dim, double w, double wsep, int p, double theta,
                   int leaf, double* out, int64_t* counts);
/* wo_solve backend 2 = FMM: degree, θ_f, leaf (the separation width is the solve's w2) */
void wo_fmm_config(int p, double theta, int leaf);

/* WNNC rescale (Alg. 3): out_i = mh_i |mp_i| / |mh_i|, mp_i kept where |mh_i| = 0 (n×3). */
void wo_rescale(int64_t n, const double* mp, const double* mh, double* out);

/* Alg. 3 + Alg. 2 solver in the normalized frame.  mu: n×3 in/out (caller order).
   backend: 0 treecode, 1 dense, 2 FMM (wo_fmm_config; separation width = w2).  mode: 0 gather Aᵀ (paper text), 1 transpose (frozen geometry).
   wnnc: 1 normal, 0 ablation (skip the WNNC update + rescale).
   stats (iters×5 or NULL): E_before, alpha, Σr², Σ(Ar)², w. */
int wo_solve(const wo_tree* t, double* mu, double w1, double w2, int iters, int first_iter,
             int total_iters, double theta, int backend, int mode, int wnnc, int order, double* stats);

int wo_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
