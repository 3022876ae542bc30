// CTA-level fp64 linear algebra used by the task kernels (NT = 128 threads per CTA).
//   * 32x32 tile POTRF / TRSM / GEMM (dense leaves, A7)
//   * Householder QR of tall-skinny panels and application of Q (A6)
//   * one-sided Jacobi SVD of the small core (A6)
//   * truncation  X Y^T -> U V^T  with sigma_{r+1} <= eps sigma_1, r <= kmax   (Remark 2)
//   * partially pivoted ACA on the Matern kernel (Alg. B.1)
//   * fully pivoted cross approximation of a dense Schur block (recompression)
// All matrices are column-major.
#pragma once
#include "dev.cuh"
#include "matern.cuh"

// ------------------------------------------------------------------------------------------
// tiles (shared memory, 32 x 32 col-major)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tile_load(double *s, const double *g)
{
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) s[e] = ldg_cg(g + e);
}
__device__ __forceinline__ void tile_store(double *g, const double *s)
{
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) g[e] = s[e];
}

// In-place lower Cholesky. Returns 0, or k+1 for the first non-positive pivot k.
// On success the strict upper triangle is zeroed; *logsum = sum_k log L_kk, *minpiv = min L_kk^2.
__device__ int tile_potrf(double *A, double *logsum, double *minpiv)
{
    __shared__ int s_fail;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int k = 0; k < 32; ++k) {
        if (threadIdx.x == 0) {
            double d = A[k + 32 * k];
            if (!(d > 0.0) || !isfinite(d)) s_fail = k + 1;
            else A[k + 32 * k] = sqrt(d);
        }
        __syncthreads();
        if (s_fail) break;
        const double dk = A[k + 32 * k];
        if (threadIdx.x > k && threadIdx.x < 32) A[threadIdx.x + 32 * k] /= dk;
        __syncthreads();
        for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
            int i = e & 31, j = e >> 5;
            if (j > k && i >= j) A[i + 32 * j] -= A[i + 32 * k] * A[j + 32 * k];
        }
        __syncthreads();
    }
    int f = s_fail;
    if (f) return f;
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
        int i = e & 31, j = e >> 5;
        if (i < j) A[e] = 0.0;
    }
    if (threadIdx.x == 0) {
        double ls = 0.0, mp = INFINITY;
        for (int k = 0; k < 32; ++k) {
            double d = A[k + 32 * k];
            ls += log(d);
            mp = fmin(mp, d * d);
        }
        *logsum = ls;
        *minpiv = mp;
    }
    __syncthreads();
    return 0;
}

// X <- X L^{-T}  (L lower 32x32), both in shared memory.
__device__ __forceinline__ void tile_trsm_rt(double *X, const double *L)
{
    if (threadIdx.x < 32) {
        const int i = threadIdx.x;
        for (int k = 0; k < 32; ++k) {
            double s = X[i + 32 * k];
            for (int j = 0; j < k; ++j) s -= X[i + 32 * j] * L[k + 32 * j];
            X[i + 32 * k] = s / L[k + 32 * k];
        }
    }
    __syncthreads();
}

// S -= A B^T  (all 32x32 shared)
__device__ __forceinline__ void tile_gemm_nt_sub(double *S, const double *A, const double *B)
{
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
        int i = e & 31, j = e >> 5;
        double s = 0.0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) s += A[i + 32 * k] * B[j + 32 * k];
        S[e] -= s;
    }
    __syncthreads();
}

// ------------------------------------------------------------------------------------------
// Householder QR of a tall-skinny panel in global memory: A (m x R, lda), R <= m.
// Reflector j: v_j = [1; A[j+1:m, j]], H_j = I - tau_j v_j v_j^T; R in the upper triangle.
// ------------------------------------------------------------------------------------------
__device__ void qr_house(double *A, int64_t lda, int64_t m, int R, double *tau, double *red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 0; j < R; ++j) {
        double *aj = A + lda * j;
        double s = 0.0;
        for (int64_t i = j + 1 + threadIdx.x; i < m; i += NT) { double v = aj[i]; s += v * v; }
        s = block_sum(s, red);
        const double alpha = aj[j];
        double t = 0.0, beta = alpha, scale = 0.0;
        if (s > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + s), alpha);
            t = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        __syncthreads();
        if (s > 0.0) {
            for (int64_t i = j + 1 + threadIdx.x; i < m; i += NT) aj[i] *= scale;
        }
        if (threadIdx.x == 0) { aj[j] = beta; tau[j] = t; }
        __syncthreads();
        if (t != 0.0) {
            for (int k = j + 1 + warp; k < R; k += NWARP) {
                double *ak = A + lda * k;
                double w = 0.0;
                for (int64_t i = j + 1 + lane; i < m; i += 32) w += aj[i] * ak[i];
                w = warp_sum(w) + ak[j];
                w *= t;
                if (lane == 0) ak[j] -= w;
                for (int64_t i = j + 1 + lane; i < m; i += 32) ak[i] -= aj[i] * w;
            }
        }
        __syncthreads();
    }
}

// B <- Q B with Q = H_0 H_1 ... H_{R-1} stored by qr_house in A.  B: m x r (ldb).
__device__ void qr_apply_q(const double *A, int64_t lda, int64_t m, int R, const double *tau,
                           double *B, int64_t ldb, int r)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = R - 1; j >= 0; --j) {
        const double t = tau[j];
        if (t == 0.0) continue;
        const double *aj = A + lda * j;
        for (int c = warp; c < r; c += NWARP) {
            double *bc = B + ldb * c;
            double w = 0.0;
            for (int64_t i = j + 1 + lane; i < m; i += 32) w += aj[i] * bc[i];
            w = warp_sum(w) + bc[j];
            w *= t;
            if (lane == 0) bc[j] -= w;
            for (int64_t i = j + 1 + lane; i < m; i += 32) bc[i] -= aj[i] * w;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// One-sided Jacobi SVD of G (K x nc, ld K, global scratch): on return G <- G J (columns mutually
// orthogonal, ||col_i|| = sigma_i) and J (nc x nc, ld nc) orthogonal, so G_in = (G J) J^T.
// Round-robin parallel ordering (nc/2 disjoint pairs per round, one warp per pair).
// ------------------------------------------------------------------------------------------
__device__ void jacobi_svd(double *G, int64_t K, double *J, int nc)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int s_rot;
    for (int e = threadIdx.x; e < nc * nc; e += NT) J[e] = ((e % nc) == (e / nc)) ? 1.0 : 0.0;
    __syncthreads();
    const int Rp = nc + (nc & 1);
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        for (int round = 0; round < Rp - 1; ++round) {
            for (int t = warp; t < Rp / 2; t += NWARP) {
                int a = t, b = Rp - 1 - t;
                int p = (a == 0) ? 0 : 1 + ((a - 1 + round) % (Rp - 1));
                int q = (b == 0) ? 0 : 1 + ((b - 1 + round) % (Rp - 1));
                if (p >= nc || q >= nc) continue;
                double *gp = G + K * p, *gq = G + K * q;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int64_t i = lane; i < K; i += 32) {
                    double x = gp[i], y = gq[i];
                    al += x * x; be += y * y; ga += x * y;
                }
                al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
                if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
                    double zeta = (be - al) / (2.0 * ga);
                    double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
                    for (int64_t i = lane; i < K; i += 32) {
                        double x = gp[i], y = gq[i];
                        gp[i] = c * x - s * y;
                        gq[i] = s * x + c * y;
                    }
                    double *jp = J + (int64_t)nc * p, *jq = J + (int64_t)nc * q;
                    for (int i = lane; i < nc; i += 32) {
                        double x = jp[i], y = jq[i];
                        jp[i] = c * x - s * y;
                        jq[i] = s * x + c * y;
                    }
                    if (lane == 0) s_rot = 1;
                }
            }
            __syncthreads();
        }
        if (!s_rot) break;
        __syncthreads();
    }
    __syncthreads();
}

// Householder QR with column pivoting of the K x K matrix M (ld K, in place), stopped at the
// first step whose largest remaining column norm is <= tol * (largest initial column norm) or
// at rmax steps.  On return: reflectors below the diagonal of the first r columns (tau[0..r)),
// R in the upper trapezoid of rows 0..r-1, piv[k] = original column of column k.  Returns r.
__device__ int qrcp_trunc(double *M, int K, double tol, int rmax, double *tau, int *piv, double *cn,
                          double *redv, int64_t *redi, double *red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = threadIdx.x; k < K; k += NT) piv[k] = k;
    __shared__ double s_n1;
    __shared__ int s_stop;
    int j = 0;
    for (; j < min(K, rmax); ++j) {
        // exact remaining column norms (rows j..K-1) of columns j..K-1
        for (int k = j + warp; k < K; k += NWARP) {
            const double *mk = M + (int64_t)K * k;
            double s = 0.0;
            for (int i = j + lane; i < K; i += 32) s += mk[i] * mk[i];
            s = warp_sum(s);
            if (lane == 0) cn[k] = s;
        }
        __syncthreads();
        double bv = -1.0;
        int64_t bi = K;
        for (int k = j + threadIdx.x; k < K; k += NT)
            if (vi_better(cn[k], k, bv, bi)) { bv = cn[k]; bi = k; }
        ValIdx b = block_argmax(bv, bi, redv, redi);
        if (threadIdx.x == 0) {
            const double nrm = sqrt(fmax(b.v, 0.0));
            if (j == 0) s_n1 = nrm;
            s_stop = !(nrm > tol * s_n1) || !(nrm > 0.0);
        }
        __syncthreads();
        if (s_stop) break;
        const int p = (int)b.i;
        if (p != j) {   // swap columns j and p
            double *mj = M + (int64_t)K * j, *mp = M + (int64_t)K * p;
            for (int i = threadIdx.x; i < K; i += NT) { double t = mj[i]; mj[i] = mp[i]; mp[i] = t; }
            if (threadIdx.x == 0) { int t = piv[j]; piv[j] = piv[p]; piv[p] = t; }
            __syncthreads();
        }
        // Householder reflector of column j, rows j..K-1
        double *aj = M + (int64_t)K * j;
        double s = 0.0;
        for (int i = j + 1 + threadIdx.x; i < K; i += NT) s += aj[i] * aj[i];
        s = block_sum(s, red);
        const double alpha = aj[j];
        double t = 0.0, beta = alpha, scale = 0.0;
        if (s > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + s), alpha);
            t = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        __syncthreads();
        if (s > 0.0)
            for (int i = j + 1 + threadIdx.x; i < K; i += NT) aj[i] *= scale;
        if (threadIdx.x == 0) { aj[j] = beta; tau[j] = t; }
        __syncthreads();
        if (t != 0.0) {
            for (int k = j + 1 + warp; k < K; k += NWARP) {
                double *ak = M + (int64_t)K * k;
                double w = 0.0;
                for (int i = j + 1 + lane; i < K; i += 32) w += aj[i] * ak[i];
                w = warp_sum(w) + ak[j];
                w *= t;
                if (lane == 0) ak[j] -= w;
                for (int i = j + 1 + lane; i < K; i += 32) ak[i] -= aj[i] * w;
            }
        }
        __syncthreads();
    }
    __syncthreads();
    return j;
}

// Truncation workspace for R columns of m rows.
struct CompressWs {
    double *X, *Y;      // m x K each (ld m): inputs, destroyed (Householder vectors)
    double *M, *G, *J;  // K x K, K x K, K x K
    double *tx, *ty, *tm;   // K each
    double *sig, *cn;   // K each
    int *ord, *piv;     // K each
    double *tail;       // first free (8-byte aligned) double after the workspace
};

// Core of the truncation (A6).  Input: upper-triangular R_X, R_Y (R x R, the
// top R rows of RX / RY with leading dimensions ldx / ldy).
//   M = R_X R_Y^T (R x R);  M Pi = Q_M R_M by pivoted QR stopped at tol_q (rank-revealing
//   pre-truncation to r' rows);
//   final (svd = true): SVD of the r' x R matrix B = R_M[:r'] Pi^T by one-sided Jacobi on B^T,
//     keep the smallest r with sigma_{r+1} <= eps sigma_1, then r <= kmax (kmax > 0), r <= rlim;
//     U_core = Q_M [J_r; 0], V_core = (B^T J)_r;
//   intermediate (svd = false): r = min(r', rlim), U_core = Q_M [I; 0], V_core = B^T[:, :r].
// Writes U[0:nr, 0:r] = [U_core; 0] and V[0:nr, 0:r] = [V_core; 0] (ld ldo, nr >= R).  Returns r.
// *cap_bound = 1 if kmax cut below the eps-rank; *overflow = 1 if the rank exceeded rlim
// (with kmax == 0 for the final truncation).
__device__ int compress_core(const CompressWs &w, const double *RX, int64_t ldx, const double *RY, int64_t ldy,
                             int R, double eps, double tol_q, bool svd, int kmax, int rlim, double *U, double *V,
                             int64_t ldo, int64_t nr, int *cap_bound, int *overflow, double *red, double *redv,
                             int64_t *redi)
{
    __shared__ int s_r, s_cb, s_of;
    const int K = R;
    for (int e = threadIdx.x; e < K * K; e += NT) {
        int i = e % K, j = e / K;
        double s = 0.0;
        for (int k = max(i, j); k < K; ++k) s += RX[i + ldx * k] * RY[j + ldy * k];
        w.M[e] = s;
    }
    __syncthreads();
    const int rq = qrcp_trunc(w.M, K, tol_q, svd ? K : rlim + 1, w.tm, w.piv, w.cn, redv, redi, red);
    for (int e = threadIdx.x; e < K * rq; e += NT) {
        int k = e % K, i = e / K;
        w.G[w.piv[k] + (int64_t)K * i] = (k >= i) ? w.M[i + (int64_t)K * k] : 0.0;
    }
    __syncthreads();
    int r;
    if (svd) {
        jacobi_svd(w.G, K, w.J, rq);
        for (int i = threadIdx.x; i < rq; i += NT) {
            double s = 0.0;
            for (int k = 0; k < K; ++k) { double x = w.G[k + (int64_t)K * i]; s += x * x; }
            w.sig[i] = sqrt(s);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < rq; i += NT) {
            int pos = 0;
            double si = w.sig[i];
            for (int j = 0; j < rq; ++j) {
                double sj = w.sig[j];
                if (sj > si || (sj == si && j < i)) ++pos;
            }
            w.ord[pos] = i;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double s1 = rq > 0 ? w.sig[w.ord[0]] : 0.0;
            int rr = 0;
            if (s1 > 0.0)
                while (rr < rq && w.sig[w.ord[rr]] > eps * s1) ++rr;
            int cb = 0, of = 0;
            if (kmax > 0 && rr > kmax) { rr = kmax; cb = 1; }
            if (rr > rlim) { rr = rlim; of = (kmax == 0); }
            s_r = rr; s_cb = cb; s_of = of;
        }
        __syncthreads();
        r = s_r;
        for (int64_t e = threadIdx.x; e < nr * r; e += NT) {
            int64_t i = e % nr;
            int c = (int)(e / nr);
            int src = w.ord[c];
            U[i + ldo * c] = (i < rq) ? w.J[i + (int64_t)rq * src] : 0.0;
            V[i + ldo * c] = (i < K) ? w.G[i + (int64_t)K * src] : 0.0;
        }
    } else {
        if (threadIdx.x == 0) {
            int rr = rq, of = 0;
            if (rr > rlim) { rr = rlim; of = 1; }
            s_r = rr; s_cb = 0; s_of = of;
        }
        __syncthreads();
        r = s_r;
        for (int64_t e = threadIdx.x; e < nr * r; e += NT) {
            int64_t i = e % nr;
            int c = (int)(e / nr);
            U[i + ldo * c] = (i == c) ? 1.0 : 0.0;
            V[i + ldo * c] = (i < K) ? w.G[i + (int64_t)K * c] : 0.0;
        }
    }
    __syncthreads();
    qr_apply_q(w.M, K, K, rq, w.tm, U, ldo, r);   // U_core <- Q_M U_core (rows < K)
    if (threadIdx.x == 0) { *cap_bound = s_cb; *overflow = s_of; }
    __syncthreads();
    return r;
}

// Truncate X Y^T (m x m, rank <= R <= m) to U V^T: [Q_X, R_X] = qr(X), [Q_Y, R_Y] = qr(Y),
// core as above, U = Q_X [U_core; 0], V = Q_Y [V_core; 0].  U, V: m x r (ld ldo), must not
// alias X, Y.  Returns r.
__device__ int compress(const CompressWs &w, int64_t m, int R, double eps, double tol_q, bool svd, int kmax,
                        int rlim, double *U, double *V, int64_t ldo, int *cap_bound, int *overflow, double *red,
                        double *redv, int64_t *redi)
{
    if (R == 0) { if (threadIdx.x == 0) { *cap_bound = 0; *overflow = 0; } __syncthreads(); return 0; }
    qr_house(w.X, m, m, R, w.tx, red);
    qr_house(w.Y, m, m, R, w.ty, red);
    const int r = compress_core(w, w.X, m, w.Y, m, R, eps, tol_q, svd, kmax, rlim, U, V, ldo, m, cap_bound, overflow,
                                red, redv, redi);
    qr_apply_q(w.X, m, m, R, w.tx, U, ldo, r);
    qr_apply_q(w.Y, m, m, R, w.ty, V, ldo, r);
    return r;
}

// ------------------------------------------------------------------------------------------
// Fully pivoted cross approximation of a dense m x m block S (global, ld m), destroyed.
// Appends up to Kmax columns to X, Y (ld m): S ~= X Y^T.  Stops when max |residual| <= tol.
// ------------------------------------------------------------------------------------------
__device__ int aca_full(double *S, int64_t m, double *X, double *Y, int Kmax, double rel_tol,
                        double *redv, int64_t *redi)
{
    const int64_t mm = m * m;
    double bv = 0.0; int64_t bi = 0;
    for (int64_t e = threadIdx.x; e < mm; e += NT) {
        double a = fabs(S[e]);
        if (vi_better(a, e, bv, bi)) { bv = a; bi = e; }
    }
    ValIdx b = block_argmax(bv, bi, redv, redi);
    const double tol = rel_tol * b.v;
    int k = 0;
    while (k < Kmax && b.v > tol && b.v > 0.0) {
        const int64_t is = b.i % m, js = b.i / m;
        const double p = S[is + m * js];
        for (int64_t i = threadIdx.x; i < m; i += NT) {
            X[i + m * k] = S[i + m * js];
            Y[i + m * k] = S[is + m * i] / p;
        }
        __syncthreads();
        bv = 0.0; bi = 0;
        const double *xk = X + m * k, *yk = Y + m * k;
        for (int64_t e = threadIdx.x; e < mm; e += NT) {
            int64_t i = e % m, j = e / m;
            double v = S[e] - xk[i] * yk[j];
            S[e] = v;
            double a = fabs(v);
            if (vi_better(a, e, bv, bi)) { bv = a; bi = e; }
        }
        b = block_argmax(bv, bi, redv, redi);
        ++k;
    }
    __syncthreads();
    return k;
}

// ------------------------------------------------------------------------------------------
// Partially pivoted ACA (Alg. B.1) of the Matern block with rows at internal
// positions r0.., columns c0.. (m x m).  U, V: m x Kmax (ld m).  Reading R4:
// first row i* = 0; ties -> lowest index; column scaled by 1/pivot; a zero residual row is
// skipped (next unused row); stop after adding term k when ||u_k|| ||v_k|| <= eps_aca ||u_1|| ||v_1||.
// ------------------------------------------------------------------------------------------
__device__ int aca_partial(const MaternParams &mp, const double *xs, const double *ys, int64_t r0,
                           int64_t c0, int64_t m, double *U, double *V, int Kmax, double eps_aca,
                           uint8_t *used, double *red, double *redv, int64_t *redi)
{
    for (int64_t i = threadIdx.x; i < m; i += NT) used[i] = 0;
    __syncthreads();
    int64_t istar = 0;
    int k = 0;
    double n1 = 0.0;
    int64_t guard = 0;
    while (k < Kmax && guard++ < m + Kmax) {
        // row residual -> V[:,k]
        const double xi = xs[r0 + istar], yi = ys[r0 + istar];
        double bv = 0.0; int64_t bi = 0;
        double *vk = V + m * k;
        for (int64_t j = threadIdx.x; j < m; j += NT) {
            double a = hcov_cov_entry(mp, xi, yi, xs[c0 + j], ys[c0 + j], (r0 + istar) == (c0 + j));
            for (int l = 0; l < k; ++l) a -= U[istar + m * l] * V[j + m * l];
            vk[j] = a;
            double aa = fabs(a);
            if (vi_better(aa, j, bv, bi)) { bv = aa; bi = j; }
        }
        ValIdx b = block_argmax(bv, bi, redv, redi);
        if (threadIdx.x == 0) used[istar] = 1;
        __syncthreads();
        if (!(b.v > 0.0)) {
            // zero residual row: next unused row (lowest index)
            int64_t cand = m;
            for (int64_t i = threadIdx.x; i < m; i += NT)
                if (!used[i] && i < cand) cand = i;
            ValIdx c = block_argmax(-(double)cand, cand, redv, redi);  // min index
            if (c.i >= m) break;
            istar = c.i;
            continue;
        }
        const int64_t js = b.i;
        const double piv = vk[js];
        const double xj = xs[c0 + js], yj = ys[c0 + js];
        double *uk = U + m * k;
        bv = -1.0; bi = m;
        double su = 0.0, sv = 0.0;
        for (int64_t i = threadIdx.x; i < m; i += NT) {
            double c = hcov_cov_entry(mp, xs[r0 + i], ys[r0 + i], xj, yj, (r0 + i) == (c0 + js));
            for (int l = 0; l < k; ++l) c -= U[i + m * l] * V[js + m * l];
            double u = c / piv;
            uk[i] = u;
            su += u * u;
            double vv = vk[i];
            sv += vv * vv;
            if (!used[i]) {
                double aa = fabs(c);
                if (vi_better(aa, i, bv, bi)) { bv = aa; bi = i; }
            }
        }
        su = block_sum(su, red);
        sv = block_sum(sv, red);
        ValIdx nb = block_argmax(bv, bi, redv, redi);
        ++k;
        const double nn = sqrt(su) * sqrt(sv);
        if (k == 1) n1 = nn;
        else if (nn <= eps_aca * n1) break;
        if (nb.i >= m || nb.v < 0.0) break;   // all rows used
        istar = nb.i;
    }
    __syncthreads();
    return k;
}
