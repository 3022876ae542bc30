/*
 * hcov.h — C ABI of libhcov.so: the B200-native (sm_100a, fp64) hot path of
 * Litvinenko, "HLIBCov" (arXiv 1709.08625): evaluate the Gaussian log-likelihood of a
 * Matern random field with the covariance held as an H-matrix.
 *
 *   L(theta) = -n/2 log(2 pi) - 1/2 log det C(theta) - 1/2 Z^T C(theta)^{-1} Z      Eq. (1)
 *   L~(theta) = -n/2 log(2 pi) - sum_i log L~_ii - 1/2 v^T v,  L~ v = Z              Eq. (2)
 *
 * Stages: A1 cluster tree, A2 block tree (hcov_build_tree);
 * A3-A6 Matern entries, dense leaves, ACA, truncation (hcov_assemble); A7 H-Cholesky
 * (hcov_cholesky); A8-A10 log det, forward H-solve, L (hcov_loglik).
 *
 * Conventions
 *  - All floating point is IEEE fp64.  Pointers named *_dev are CUDA device pointers,
 *    *_host are host pointers.  Arrays are owned by the caller; the library copies what it
 *    keeps into handle-owned device memory.  Handles are owned by the caller and released
 *    with hcov_*_free.  Streams: every call is ordered on the given stream (0 = legacy default).
 *  - Index order: "external" = the caller's order of the n locations; "internal" = cluster-tree
 *    order (perm_e2i / perm_i2e).  Z and sampled vectors are external.
 *  - Errors: every function returns hcov_status; nothing throws across the ABI.  On error the
 *    output handle is left NULL and no memory is leaked.
 *  - Determinism: the same inputs on the same device give bitwise-identical outputs.
 *  - Thread safety: a handle must not be used from several host threads concurrently.
 */
#ifndef HCOV_H
#define HCOV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HCOV_OK = 0,
    HCOV_ERR_INVALID_ARG = 1,   /* sigma2, ell, nu <= 0; nugget, eps < 0; leaf < 1; non-finite coordinates; NULL pointer */
    HCOV_ERR_EMPTY_INPUT = 2,   /* n == 0 */
    HCOV_ERR_NOT_SPD = 3,       /* a diagonal-leaf pivot <= 0 during the H-Cholesky (fail_leaf reports which) */
    HCOV_ERR_OUT_OF_MEMORY = 4, /* device allocation failed */
    HCOV_ERR_CUDA = 5,          /* any other CUDA runtime error */
    HCOV_ERR_RANK_CAPACITY = 6, /* with kmax == 0: an epsilon-rank exceeded the rank capacity, or a
                                   recompression lost accuracy for lack of capacity (acc_loss > 0) */
    HCOV_ERR_STATE = 7          /* call order violated (e.g. loglik on an unfactored matrix) */
} hcov_status;

typedef struct hcov_tree_s *hcov_tree;  /* cluster tree + block tree + theta-independent schedule */
typedef struct hcov_hmat_s *hcov_hmat;  /* device H-matrix: C~ after hcov_assemble, L~ (in place) after hcov_cholesky */
typedef void *hcov_stream;              /* a cudaStream_t */

/* Eq. (3):  C(h) = sigma2 / (2^(nu-1) Gamma(nu)) (h/ell)^nu K_nu(h/ell);
 * nugget tau^2 is added on the diagonal (listing PAPER.md:534). */
typedef struct {
    double sigma2, ell, nu, nugget;
} hcov_theta;

/* Remark 2: per admissible block keep the smallest rank r with
 * sigma_{r+1} <= eps * sigma_1 (adaptive), and r <= kmax (fixed) when kmax > 0.
 * kcap = rank capacity of the device pools (0 = default: kmax if kmax > 0 else 64). */
typedef struct {
    double eps;
    int32_t kmax;
    int32_t kcap;
} hcov_trunc;

typedef struct {
    double loglik;        /* L~(theta), Eq. (2) */
    double logdet;        /* log det C~ = 2 sum log L~_ii */
    double quad;          /* v^T v, L~ v = P_e2i Z */
    int64_t n;
    int32_t max_rank;     /* largest rank of any low-rank block of L~ */
    int32_t cap_binds;    /* number of truncations where kmax bound below the eps-rank */
    double min_pivot;     /* smallest L~_ii^2 */
    int64_t fail_leaf;    /* -1, or the first diagonal leaf whose pivot failed */
    int32_t acc_loss;     /* recompressions that had to cut below their tolerance because a work
                             capacity was exhausted (full-pivot ACA capacity, or an intermediate
                             chunk recompression over 2 kcap; R22/R23).  0 on a clean run;
                             with kmax == 0 a nonzero count returns HCOV_ERR_RANK_CAPACITY. */
    int32_t interm_cuts;  /* with kmax > 0: the same capacity cuts, each keeping a rank >= kmax (every
                             work capacity is >= kmax), so the cut is covered by the rank cap and is
                             not an accuracy loss beyond it (R26) */
} hcov_result;

typedef struct {
    int64_t n, n_pad;       /* locations; padded size 32 * 2^depth (phantom identity rows) */
    int32_t depth, leaf_size;
    int64_t n_leaves;
    int64_t n_dense_tiles;  /* 32x32 tiles of the lower triangle incl. diagonal */
    int64_t n_lowrank;      /* admissible low-rank blocks (lower triangle) */
    int64_t n_tasks, n_waves;   /* n_waves: longest dependency chain of the task DAG (tasks) */
    double eta;
    /* pool sizes (for memory planning): U/V and W elements per unit rank capacity, product slots
     * (slot_a * kcap^2 + slot_b * kcap doubles), cores (kcap^2 each), DAG edges, term-list entries */
    int64_t uv_elems, w_elems, slot_a, slot_b, n_cores, n_edges, n_xterm, max_mq;
    /* 1 if A1 / A2 ran on the device (hcov_build_tree[_ex]: kernels K1 / K2 of tree.cu), 0 for the
     * host planner (hcov_build_tree_host[_ex]); geo_ms: wall time of the device A1 + A2 stage (device
     * path) or of the whole host plan including the task schedule (host path) */
    int32_t tree_on_device;
    double geo_ms;
    int32_t dim;           /* 2 or 3 (hcov_tree_opts.dim) */
} hcov_tree_info;

/* A1 + A2: cluster tree by median bisection on the longest bounding-box axis (leaves <= leaf_size,
 * uniform depth), eta-admissible block tree (min(diam) <= eta * dist, dist > 0; PAPER.md:475,
 * 723-743), and the theta-independent H-Cholesky task schedule.  A1 and A2 run on the device
 * (level-synchronous kernels: segmented bounding boxes + stable radix sort per level; pair
 * classification + scan per level), bitwise equal to the host planner's trees; the task schedule
 * is planned on the host from their output.  Errors: HCOV_ERR_INVALID_ARG for non-finite
 * coordinates or n >= 2^31 - 32, HCOV_ERR_EMPTY_INPUT for n == 0, HCOV_ERR_CUDA on a device error.
 *   s_dev: n x 2 row-major device array of locations (external order).
 *   leaf_size: 32 (the only supported value).  eta: admissibility parameter (2.0; 0 = all dense).
 *   dense_below: admissible blocks with cluster size <= dense_below are stored as dense tiles
 *   (32 = only leaf-level blocks). */
hcov_status hcov_build_tree(const double *s_dev, int64_t n, int32_t leaf_size, double eta,
                            int32_t dense_below, hcov_stream stream, hcov_tree *out);
/* Host-only planning (no device memory is touched; usable without a GPU): same as
 * hcov_build_tree with s_host a host array.  Device arrays are uploaded on first use. */
hcov_status hcov_build_tree_host(const double *s_host, int64_t n, int32_t leaf_size, double eta,
                                 int32_t dense_below, hcov_tree *out);
/* Tree options (hcov_build_tree_ex).  factor_trunc = 1 selects the SPD-preserving variant of the
 * H-Cholesky (NEXT (f4); reading R27): the assembled C~ and the accumulated Schur updates
 * of each low-rank block are kept near-losslessly (eps * 1e-2, no rank cap, within the work capacity
 * kcap), and the (eps, kmax) truncation of Remark 2 (applied per sub-block of L~
 * as Table 4's caption states) is applied to the FACTOR block
 * L_21 = A_21 L_11^{-T} after its solve.  A truncated SVD of L_21 is an orthogonal projection from
 * the right, so the Schur complement A_22 - L~_21 L~_21^T is >= A_22 - L_21 L_21^T in the Loewner
 * order: truncation can only raise the remaining pivots.  Use with kcap > kmax (e.g. kcap = 64,
 * kmax = 20).  factor_trunc = 0 is the paper's order (truncate, then solve). */
typedef struct {
    int32_t leaf_size;     /* 32 */
    double eta;            /* admissibility parameter (2.0; 0 = all dense) */
    int32_t dense_below;   /* 32 */
    int32_t factor_trunc;  /* 0 or 1 */
    int32_t dim;           /* 2 (also 0), or 3: the 3-D variant ("replace dim = 2 by
                            * dim = 3"): s is n x 3, boxes, diameters, distances and the longest-axis
                            * split run over 3 axes (ties -> x, then y), and the Matern argument is the
                            * 3-D distance; everything else is unchanged */
} hcov_tree_opts;
hcov_status hcov_build_tree_ex(const double *s_dev, int64_t n, const hcov_tree_opts *opts, hcov_stream stream,
                               hcov_tree *out);
hcov_status hcov_build_tree_host_ex(const double *s_host, int64_t n, const hcov_tree_opts *opts, hcov_tree *out);
hcov_status hcov_tree_get_info(hcov_tree t, hcov_tree_info *info);
/* Block-tree nodes (lower triangle incl. diagonal), 4 int32 per node: level, i, j, type
 * (0 = inadmissible/subdivided, 1 = low-rank leaf, 2 = dense 32x32 leaf).  With out4 == NULL
 * only *count is set; otherwise cap >= *count is required. */
hcov_status hcov_tree_blocks(hcov_tree t, int32_t *out4, int64_t cap, int64_t *count);
/* Schedule introspection (diagnostics): 6 int32 per task of the DAG in generation order:
 * type (0 FILL, 1 ACA, 2 TAPP, 3 POTRF, 4 TRSM, 5 RAPP, 6 SEG, 7 PROJ, 8 PRR, 9 PHWP, 10 PHWR,
 * 11 NOP, 12 BSEG, 13 BPROJ), phase (0 assembly, 1 H-Cholesky, 2 forward solve, 3 back-solve), and
 * the task arguments a, b, c, d. */
hcov_status hcov_tree_tasks(hcov_tree t, int32_t *out6, int64_t cap, int64_t *count);
/* DAG successors (diagnostics): off has n_tasks + 1 entries, succ has *count entries (CSR).
 * With off == NULL or succ == NULL only *count is set.  Setting the environment variable
 * HCOV_TIMELINE=<file> makes every engine launch write (start_ns, end_ns, cta) as 3 uint64 per
 * task (0 for tasks outside the launched mode) to <file>. */
hcov_status hcov_tree_succ(hcov_tree t, int32_t *off, int32_t *succ, int64_t cap, int64_t *count);
/* Cluster bounding boxes, 2 dim doubles per cluster heap id (2^l - 1 + c): lo_x, lo_y, hi_x, hi_y
 * (dim 2) or lo_x, lo_y, lo_z, hi_x, hi_y, hi_z (dim 3). */
hcov_status hcov_tree_bbox(hcov_tree t, double *bb, int64_t cap);
/* perm_i2e: n_pad int64 (host); entry k = external index of internal position k, -1 for phantom rows. */
hcov_status hcov_tree_perm(hcov_tree t, int64_t *perm_i2e_host);

/* A3-A6: dense leaves filled with Eq. (3) (+nugget), admissible blocks by ACA (Alg. B.1,
 * PAPER.md:759-787) to eps/10, then QR+SVD truncation to (eps, kmax). */
hcov_status hcov_assemble(hcov_tree t, const hcov_theta *theta, const hcov_trunc *trunc,
                          hcov_stream stream, hcov_hmat *out);

/* A7: H-Cholesky C~ = L~ L~^T in place (Eq. (2)).  Synchronises the
 * stream.  fail_leaf (may be NULL) receives -1 or the first failing diagonal leaf. */
hcov_status hcov_cholesky(hcov_hmat h, hcov_stream stream, int64_t *fail_leaf);

/* A8-A10: log det = 2 sum log L~_ii, v = L~^{-1} P_e2i Z (forward H-solve), q = v^T v,
 * L~ = -n/2 log 2pi - logdet/2 - q/2.  Z_dev: n fp64 external order.  Synchronises. */
hcov_status hcov_loglik(hcov_hmat h, const double *Z_dev, hcov_stream stream, hcov_result *out);

/* A3-A10 in one call (assemble + factor + loglik), handle-free for the caller. */
hcov_status hcov_eval(hcov_tree t, const hcov_theta *theta, const hcov_trunc *trunc,
                      const double *Z_dev, hcov_stream stream, hcov_result *out);

/* Theta batch (MLE candidates): evaluates m thetas; loglik_host[i] = -INFINITY and
 * status_host[i] != HCOV_OK for rejected candidates (not SPD, rank capacity); the batch
 * continues.  Returns HCOV_OK unless an argument or CUDA error aborts the batch. */
hcov_status hcov_mle_batch(hcov_tree t, const double *Z_dev, const hcov_theta *thetas_host, int32_t m,
                           const hcov_trunc *trunc, hcov_stream stream, double *loglik_host,
                           hcov_status *status_host);

/* NEXT (f1): the paper's own quadratic-form path (listing PAPER.md:550-555: TCG on C~
 * with the factor as preconditioner, 150 iterations, tolerance 1e-6) and its building blocks.
 * All vectors are n fp64 device arrays in EXTERNAL order; P = the cluster-tree permutation.
 *   hcov_forward_solve: v = P_i2e L~^{-1} P_e2i z   (the Eq. (2) forward solve; v^T v = q)
 *   hcov_backsolve:     u = P_i2e L~^{-T} P_e2i v   (root back-solve, transposed leaf chain)
 *   hcov_solve:         x = C~^{-1} b = P_i2e L~^{-T} L~^{-1} P_e2i b
 *   hcov_matvec:        y = C~ x for an ASSEMBLED (not factored) H-matrix (Table 1),
 *                       lower blocks and their mirror (Remark 1), deterministic order
 *   hcov_pcg:           preconditioned CG for C~ x = b (A assembled, M factored, same tree):
 *                       x0 = 0, preconditioner z = M^{-1} r via hcov_solve; stops after maxit
 *                       iterations or when ||r||_2 <= tol ||b||_2; iters, relres = ||r|| / ||b||.
 * Factored: state after hcov_cholesky (or hcov_eval's handle).  Synchronise the stream. */
hcov_status hcov_forward_solve(hcov_hmat h, const double *z_dev, double *v_dev, hcov_stream stream);
hcov_status hcov_backsolve(hcov_hmat h, const double *v_dev, double *u_dev, hcov_stream stream);
/* NEXT (f4): the point-wise LDL^T form of the factor (the listing's ldl_inv with point_wise
 * pivots; reading R8).  C~ = L' D L'^T with L' = L~ diag(L~)^{-1} unit lower and
 * D = diag(L~)^2: the same factorization (log det = sum log D_i = 2 sum log L~_ii; the forward solve
 * of L' is D^{1/2} times the one of L~).  D_dev: n fp64 device array, EXTERNAL order; D_e is the
 * pivot of point e = its conditional variance given the points before it in the internal order
 * (>= tau^2).  Factored handle required (HCOV_ERR_STATE otherwise); stream-ordered, no sync. */
hcov_status hcov_ldl_diag(hcov_hmat h, double *D_dev, hcov_stream stream);
hcov_status hcov_solve(hcov_hmat h, const double *b_dev, double *x_dev, hcov_stream stream);
hcov_status hcov_matvec(hcov_hmat h, const double *x_dev, double *y_dev, hcov_stream stream);
hcov_status hcov_pcg(hcov_hmat A, hcov_hmat M, const double *b_dev, double *x_dev, int32_t maxit, double tol,
                     hcov_stream stream, int32_t *iters_host, double *relres_host);

/* NEXT (f3): accuracy diagnostics of Sec. 4 (Tables 2-3; Table 4's last
 * column).  Deterministic power iterations from a hashed start vector (seed).
 *   hcov_norm2_diff:  ||A~ - B~||_2 of two ASSEMBLED matrices on the same n points (e.g. B = the exact C
 *                     as an eta = 0 all-dense tree), power iteration on the symmetric difference.
 *   hcov_inv_error:   ||I - M^{-1} A~||_2, A assembled, M factored (M = L~ L~^T), by power iteration on
 *                     E^T E, E = I - M^{-1} A (= ||A M^{-1} - I||_2, the Table 2-3 column with A = C).
 *   hcov_trace_inv:   tr(M^{-1} A) by n solves with the columns of A (the KLD's trace term,
 *                     KLD = (tr(M^{-1} C) - n + log det M - log det C) / 2; feasible for small n).
 * Outputs: one host double.  Iterations: the largest ||E x_k|| (||x_k|| = 1) seen, a lower bound that
 * converges to the norm.  Synchronise the stream. */
hcov_status hcov_norm2_diff(hcov_hmat A, hcov_hmat B, int32_t iters, uint64_t seed, hcov_stream stream,
                            double *out_host);
hcov_status hcov_inv_error(hcov_hmat A, hcov_hmat M, int32_t iters, uint64_t seed, hcov_stream stream,
                           double *out_host);
hcov_status hcov_trace_inv(hcov_hmat M, hcov_hmat A, hcov_stream stream, double *out_host);

/* Support (not timed).  Z = P_i2e L~ xi for a factored matrix (Sec. 5.1);
 * xi_dev, Z_dev: n fp64 (xi in external order too: xi is permuted to internal first). */
hcov_status hcov_sample(hcov_hmat h, const double *xi_dev, double *Z_dev, hcov_stream stream);
/* Columns of the assembled C~ (before hcov_cholesky): out_dev is n x m column-major, external
 * row order; cols_host are external column indices. */
hcov_status hcov_columns(hcov_hmat h, const int64_t *cols_host, int32_t m, double *out_dev,
                         hcov_stream stream);
/* Exact covariance columns C e_j (Eq. (3) + nugget, direct device K_nu without the table), n x m
 * column-major, external row order: the reference side of the sampled-column accuracy check
 * ||C - C~||_F / ||C||_F (BASELINE north_star) at sizes the dense oracle cannot reach. */
hcov_status hcov_cov_columns(hcov_tree t, const hcov_theta *theta, const int64_t *cols_host, int32_t m,
                             double *out_dev, hcov_stream stream);
/* Device memory of an H-matrix handle (bytes), out8_host: [0] dense tiles, [1] U/V pools (rank
 * capacity), [2] cores, [3] W pool capacity, [4] product-slot pool capacity, [5] W used by the last
 * engine run, [6] product slots used, [7] pool overflows of the last run (> 0: it returned
 * HCOV_ERR_OUT_OF_MEMORY).  The per-CTA engine scratch is shared by every handle (not counted). */
hcov_status hcov_hmat_mem_info(hcov_hmat h, int64_t *out8_host);
/* Diagnostics of an H-matrix: bytes of dense tiles and low-rank factors at actual ranks. */
hcov_status hcov_hmat_storage(hcov_hmat h, int64_t *dense_bytes, int64_t *lowrank_bytes,
                              int32_t *max_rank);

/* The H-matrix (factored, L~) of the last hcov_eval on this tree: a BORROWED handle owned by the
 * tree (do not free; invalidated by the next hcov_eval / hcov_tree_free).  For diagnostics
 * (storage, ranks, work model) after an evaluation. */
hcov_status hcov_tree_last_eval(hcov_tree t, hcov_hmat *out);
/* Method-work model of SURVEY.md Sec. 8(d) / App. A.3 evaluated at the measured final ranks of a
 * factored matrix (state >= factored): out[0] total flop of one evaluation; out[1] eager
 * truncations of the low-rank Schur updates (4 m R^2 + 22 R^3 + 4 m R r per update), [2] low-rank
 * products (cores, W = H V), [3] tile updates + TRSM, [4] V <- L^{-1} V solves, [5] POTRF, [6] ACA
 * output truncation, [7] root forward solve.  The denominator of bench.py's roofline fraction. */
hcov_status hcov_model_flops(hcov_hmat h, double *out8_host);

/* Instrumentation (process-wide, not thread-safe).  launches/count: kernels the library launched
 * (always counted).  With events enabled: ms = device time per launch class from CUDA events
 * recorded around each launch on its stream, and the engine's per-task-type busy time (sum over
 * CTAs of globaltimer spans), task counts and algorithmic flop per flop class
 * (0 assembly [kernel evaluations], 1 tile updates, 2 truncation, 3 solves, 4 products).
 * hcov_prof_read synchronises those events.  Names: hcov_prof_class_name / hcov_prof_task_name. */
#define HCOV_PROF_CLASSES 16
typedef struct {
    int64_t launches;                  /* kernels launched since the last reset */
    int32_t n_classes, n_task_types;
    int64_t count[HCOV_PROF_CLASSES];  /* launches per class */
    double ms[HCOV_PROF_CLASSES];      /* device milliseconds per class (0 unless events enabled) */
    double task_busy_ms[HCOV_PROF_CLASSES];
    double task_count[HCOV_PROF_CLASSES];
    double flop[8];
    double phase_ms[16];               /* CTA-time of truncation phases: 0 panel QRs, 1 core product,
                                          2 pivoted QR, 3 SVD, 4 Q applications, 5 full-pivot ACA,
                                          6 dense updates, 8 partial ACA */
    double phase_cls_ms[64];           /* the same per block-size class (phase + 16 * class; classes
                                          m <= 64, <= 256, <= 1024, larger) */
} hcov_prof;
hcov_status hcov_prof_control(int32_t enable_events, int32_t reset);
hcov_status hcov_prof_read(hcov_prof *out);
const char *hcov_prof_class_name(int32_t cls);
const char *hcov_prof_task_name(int32_t type);

/* Unit test of the truncation step A6 on one CTA: X, Y (m x R, col-major device
 * arrays) -> U, V (m x rlim device arrays) with X Y^T ~ U V^T, sigma_{r+1} <= eps sigma_1, r <= kmax
 * (kmax > 0), r <= rlim.  path 0: Householder QRs; 1: shifted CholeskyQR3 (taken when m >= 2R);
 * 2: shared-memory Householder (m <= 1024, m R + R within the CTA's shared memory); 3: the dense-mode
 * pipeline of a small low-rank block (m <= 256): S = X Y^T formed densely, fully pivoted cross
 * approximation to 0.1 eps, then path 2 (R23).  out3_host: rank, cap-bound flag, overflow flag.  Synchronises the device. */
hcov_status hcov_test_truncate(const double *X_dev, const double *Y_dev, int64_t m, int32_t R, double eps,
                               int32_t kmax, int32_t rlim, int32_t path, double *U_dev, double *V_dev,
                               int32_t *out3_host);

void hcov_tree_free(hcov_tree t);
void hcov_hmat_free(hcov_hmat h);
const char *hcov_status_string(hcov_status s);

#ifdef __cplusplus
}
#endif
#endif /* HCOV_H */
