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
// FP64 tensor-core (DMMA) tile update on sm_100a: mma.sync.aligned.m8n8k4.row.col.f64.
// Fragments (PTX ISA, m8n8k4 .f64): lane l, g = l / 4, t = l % 4:  a = A[g][t] (8x4 row),
// b = B[t][g] (4x8 col), c = {C[g][2t], C[g][2t+1]}.
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// S (32 x 32, ld 32) -= A (32 x kd, ld 32) B^T (B 32 x kd, ld 32), all in shared memory; kd is
// padded to a multiple of 4 with zeros.  One warp per 8 x 8 output block (16 blocks).
__device__ __forceinline__ void tile_gemm_nt_sub_k(double *S, const double *A, const double *B, int kd)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    for (int blk = warp; blk < 16; blk += NWARP) {
        const int bi = blk >> 2, bj = blk & 3;
        double c0 = 0.0, c1 = 0.0;
        for (int k0 = 0; k0 < kd; k0 += 4) {
            const int k = k0 + t;
            const double a = (k < kd) ? A[(8 * bi + g) + 32 * k] : 0.0;
            const double b = (k < kd) ? B[(8 * bj + g) + 32 * k] : 0.0;
            dmma_8x8x4(c0, c1, a, b);
        }
        S[(8 * bi + g) + 32 * (8 * bj + 2 * t)] -= c0;
        S[(8 * bi + g) + 32 * (8 * bj + 2 * t + 1)] -= c1;
    }
    __syncthreads();
}

// S -= A B^T  (all 32x32 shared)
__device__ __forceinline__ void tile_gemm_nt_sub(double *S, const double *A, const double *B)
{
    tile_gemm_nt_sub_k(S, A, B, 32);
}

// ------------------------------------------------------------------------------------------
// CTA GEMM update  C(i, j) += alpha * sum_l A(i, l) B(j, l),  i < nr, j < nc, l < kd, with
// A(i, l) = Ap[i + l * lda] (L2 loads, coalesced in i), B(j, l) = Bp[j * bsj + l * bsl] staged
// through shared memory in chunks of GEMM_JC columns j, C(i, j) = Cp[i + j * ldc] (CTA-private).
// Each thread owns rows i and keeps GEMM_JC accumulators: A is read once per column chunk and B
// once in total, instead of once per output entry.  smem: >= GEMM_JC * kd doubles.
// ------------------------------------------------------------------------------------------
#define GEMM_JC 16
__device__ void cta_gemm_nt(double *Cp, int64_t ldc, int64_t nr, int64_t nc, int kd, const double *Ap, int64_t lda,
                            const double *Bp, int64_t bsj, int64_t bsl, double alpha, double *smem,
                            int64_t smem_dbl = 0)
{
    // thread t: row group i = t % rp (rows i, i + rp, ...), column-chunk group g = t / rp; ng chunk
    // groups are staged at once (when there are fewer rows than threads)
    const int rp = (int)(nr < NT ? nr : NT);
    int ng = NT / (rp > 0 ? rp : 1);
    const int64_t per = (int64_t)GEMM_JC * (kd > 0 ? kd : 1);
    if (smem_dbl < per * ng) ng = (int)(smem_dbl / per > 1 ? smem_dbl / per : 1);
    const int g = threadIdx.x / (rp > 0 ? rp : 1);
    const int i0 = threadIdx.x % (rp > 0 ? rp : 1);
    for (int64_t j0 = 0; j0 < nc; j0 += (int64_t)GEMM_JC * ng) {
        __syncthreads();
        for (int e = threadIdx.x; e < GEMM_JC * kd * ng; e += NT) {
            const int gg = e / (GEMM_JC * kd), e2 = e % (GEMM_JC * kd);
            const int jj = e2 % GEMM_JC, l = e2 / GEMM_JC;
            const int64_t j = j0 + (int64_t)gg * GEMM_JC + jj;
            smem[e] = (j < nc) ? __ldcg(Bp + j * bsj + (int64_t)l * bsl) : 0.0;
        }
        __syncthreads();
        const int64_t jg = j0 + (int64_t)g * GEMM_JC;
        if (g < ng && jg < nc) {
            const int jc = (int)(nc - jg < GEMM_JC ? nc - jg : GEMM_JC);
            const double *sb = smem + (int64_t)g * GEMM_JC * kd;
            for (int64_t i = i0; i < nr; i += rp) {
                double acc[GEMM_JC];
#pragma unroll
                for (int jj = 0; jj < GEMM_JC; ++jj) acc[jj] = 0.0;
                for (int l = 0; l < kd; ++l) {
                    const double a = __ldcg(Ap + i + (int64_t)l * lda);
                    const double *bl = sb + GEMM_JC * l;
#pragma unroll
                    for (int jj = 0; jj < GEMM_JC; ++jj) acc[jj] = fma(a, bl[jj], acc[jj]);
                }
                for (int jj = 0; jj < jc; ++jj) Cp[i + (jg + jj) * ldc] += alpha * acc[jj];
            }
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------------------------------
// Householder QR of a tall-skinny panel in global memory: A (m x R, lda), R <= m.
// Reflector j: v_j = [1; A[j+1:m, j]], H_j = I - tau_j v_j v_j^T; R in the upper triangle.
// ------------------------------------------------------------------------------------------
// Apply H = I - t v v^T (v = [1; aj[j+1:m]]) to columns k0..k1-1 of B (ld ldb, rows j..m-1):
// one warp per group of 4 columns, the 4 dot products reduced together (interleaved shuffles).
__device__ __forceinline__ void householder_update(const double *aj, int64_t j, int64_t m, double t, double *B,
                                                   int64_t ldb, int k0, int k1)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = k0 + 4 * warp; k < k1; k += 4 * NWARP) {
        const int nk = min(4, k1 - k);
        double *b0 = B + ldb * k;
        double *b1 = (nk > 1) ? b0 + ldb : b0;
        double *b2 = (nk > 2) ? b0 + 2 * ldb : b0;
        double *b3 = (nk > 3) ? b0 + 3 * ldb : b0;
        double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll 4
        for (int64_t i = j + 1 + lane; i < m; i += 32) {
            const double v = aj[i];
            w0 = fma(v, b0[i], w0);
            w1 = fma(v, b1[i], w1);
            w2 = fma(v, b2[i], w2);
            w3 = fma(v, b3[i], w3);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            w0 += __shfl_xor_sync(0xffffffffu, w0, o);
            w1 += __shfl_xor_sync(0xffffffffu, w1, o);
            w2 += __shfl_xor_sync(0xffffffffu, w2, o);
            w3 += __shfl_xor_sync(0xffffffffu, w3, o);
        }
        w0 = t * (w0 + b0[j]);
        w1 = t * (w1 + b1[j]);
        w2 = t * (w2 + b2[j]);
        w3 = t * (w3 + b3[j]);
        __syncwarp();
        if (lane == 0) {
            b0[j] -= w0;
            if (nk > 1) b1[j] -= w1;
            if (nk > 2) b2[j] -= w2;
            if (nk > 3) b3[j] -= w3;
        }
#pragma unroll 4
        for (int64_t i = j + 1 + lane; i < m; i += 32) {
            const double v = aj[i];
            b0[i] -= v * w0;
            if (nk > 1) b1[i] -= v * w1;
            if (nk > 2) b2[i] -= v * w2;
            if (nk > 3) b3[i] -= v * w3;
        }
        __syncwarp();
    }
}

__device__ void qr_house(double *A, int64_t lda, int64_t m, int R, double *tau, double *red)
{
    for (int j = 0; j < R; ++j) {
        double *aj = A + lda * j;
        double s = 0.0;
#pragma unroll 4
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
        if (t != 0.0) householder_update(aj, j, m, t, A, lda, j + 1, R);
        __syncthreads();
    }
}

// B <- Q B with Q = H_0 H_1 ... H_{R-1} stored by qr_house in A.  B: m x r (ldb).
__device__ void qr_apply_q(const double *A, int64_t lda, int64_t m, int R, const double *tau,
                           double *B, int64_t ldb, int r)
{
    for (int j = R - 1; j >= 0; --j) {
        const double t = tau[j];
        if (t == 0.0) continue;
        householder_update(A + lda * j, j, m, t, B, ldb, 0, r);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// Shared-memory resident Householder QR (one CTA per SM: the engine has ~220 KB of dynamic
// shared memory, enough for a 256 x 96 panel).  Column k is owned by warp k mod NWARP; step j
// applies H_j to every column k > j, and the owner of column j + 1 updates that column first and
// computes reflector j + 1 (look-ahead), so each step costs one CTA barrier.  Same reflector
// convention as qr_house (v_j = [1; A[j+1:m, j]], tau_j, R in the upper triangle).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void house_col_warp(double *A, int lda, int m, int j, double *tau)
{
    const int lane = threadIdx.x & 31;
    double *aj = A + (int64_t)lda * j;
    double s = 0.0;
    for (int i = j + 1 + lane; i < m; i += 32) s = fma(aj[i], aj[i], s);
    s = warp_sum(s);
    const double alpha = aj[j];
    double t = 0.0, beta = alpha, scale = 0.0;
    if (s > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
        for (int i = j + 1 + lane; i < m; i += 32) aj[i] *= scale;
    }
    __syncwarp();
    if (lane == 0) { aj[j] = beta; tau[j] = t; }
    __syncwarp();
}

// Apply H = I - t v v^T (v = [1; v[j+1:m]]) to nk <= 4 columns c0, c0 + cs, ... of B (one warp).
__device__ __forceinline__ void house_apply4(const double *v, int j, int m, double t, double *B, int ldb, int c0,
                                             int cs, int nk)
{
    const int lane = threadIdx.x & 31;
    double *b0 = B + (int64_t)ldb * c0;
    double *b1 = (nk > 1) ? b0 + (int64_t)ldb * cs : b0;
    double *b2 = (nk > 2) ? b0 + (int64_t)ldb * 2 * cs : b0;
    double *b3 = (nk > 3) ? b0 + (int64_t)ldb * 3 * cs : b0;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
    for (int i = j + 1 + lane; i < m; i += 32) {
        const double x = v[i];
        w0 = fma(x, b0[i], w0);
        w1 = fma(x, b1[i], w1);
        w2 = fma(x, b2[i], w2);
        w3 = fma(x, b3[i], w3);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        w0 += __shfl_xor_sync(0xffffffffu, w0, o);
        w1 += __shfl_xor_sync(0xffffffffu, w1, o);
        w2 += __shfl_xor_sync(0xffffffffu, w2, o);
        w3 += __shfl_xor_sync(0xffffffffu, w3, o);
    }
    w0 = t * (w0 + b0[j]);
    w1 = t * (w1 + b1[j]);
    w2 = t * (w2 + b2[j]);
    w3 = t * (w3 + b3[j]);
    __syncwarp();
    if (lane == 0) {
        b0[j] -= w0;
        if (nk > 1) b1[j] -= w1;
        if (nk > 2) b2[j] -= w2;
        if (nk > 3) b3[j] -= w3;
    }
    for (int i = j + 1 + lane; i < m; i += 32) {
        const double x = v[i];
        b0[i] -= x * w0;
        if (nk > 1) b1[i] -= x * w1;
        if (nk > 2) b2[i] -= x * w2;
        if (nk > 3) b3[i] -= x * w3;
    }
    __syncwarp();
}

// QR of A (m x R, ld lda, shared memory, R <= m) in place; tau: R doubles (shared memory).
__device__ void qr_house_sm(double *A, int lda, int m, int R, double *tau)
{
    const int warp = threadIdx.x >> 5;
    if (R <= 0) return;
    if (warp == 0) house_col_warp(A, lda, m, 0, tau);
    __syncthreads();
    for (int j = 0; j < R; ++j) {
        const double t = tau[j];
        const double *v = A + (int64_t)lda * j;
        const int la = j + 1;
        if (la < R && warp == la % NWARP) {
            if (t != 0.0) house_apply4(v, j, m, t, A, lda, la, NWARP, 1);
            house_col_warp(A, lda, m, la, tau);
        }
        if (t != 0.0) {
            // this warp's columns k > la (k = warp mod NWARP), four at a time
            int k0 = warp;
            if (k0 <= la) k0 += NWARP * ((la - warp) / NWARP + 1);
            for (int k = k0; k < R; k += 4 * NWARP) {
                const int nk = min(4, (R - 1 - k) / NWARP + 1);
                house_apply4(v, j, m, t, A, lda, k, NWARP, nk);
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// Blocked variant for panels of m <= 32 QM rows (shared memory, ld lda): panels of 4 columns are
// factored by warp 0 in registers (no CTA barrier inside a panel); the other warps apply the 4
// reflectors to the trailing columns two at a time in registers (one shared-memory read and
// write of the trailing matrix per panel instead of per reflector); warp 0 updates and factors
// the next panel while they do (look-ahead), so each panel costs one CTA barrier.
// ------------------------------------------------------------------------------------------
template <int QM>
__device__ __forceinline__ void hh_coef(const double *A, int lda, int m, int j, double (&cf)[QM])
{
    const int lane = threadIdx.x & 31;
    const double *v = A + (int64_t)lda * j;
#pragma unroll
    for (int q = 0; q < QM; ++q) {
        const int i = lane + 32 * q;
        cf[q] = (i > j && i < m) ? v[i] : (i == j ? 1.0 : 0.0);
    }
}

// Apply H_j (coefficients cf, tau t) to NC register columns b.
template <int QM, int NC>
__device__ __forceinline__ void hh_apply_reg(const double (&cf)[QM], double t, double (&b)[NC][QM])
{
    double w[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < QM; ++q) s = fma(cf[q], b[c][q], s);
        w[c] = s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = 0; c < NC; ++c) w[c] += __shfl_xor_sync(0xffffffffu, w[c], o);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const double tw = t * w[c];
#pragma unroll
        for (int q = 0; q < QM; ++q) b[c][q] = fma(-cf[q], tw, b[c][q]);
    }
}

// Warp-level factorization of the panel columns j0 .. j0+nb-1 (nb <= 4; already updated by all
// earlier reflectors): reflectors and R written to A, tau[j0 ..].
template <int QM>
__device__ __forceinline__ void hh_panel(double *A, int lda, int m, int j0, int nb, double *tau)
{
    const int lane = threadIdx.x & 31;
    double p[4][QM];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            const int i = lane + 32 * q;
            p[c][q] = (c < nb && i < m) ? A[i + (int64_t)lda * (j0 + c)] : 0.0;
        }
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
        if (jj >= nb) break;
        const int j = j0 + jj;
        double s = 0.0, av = 0.0;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            const int i = lane + 32 * q;
            if (i > j && i < m) s = fma(p[jj][q], p[jj][q], s);
            if (q == (j >> 5)) av = p[jj][q];
        }
        s = warp_sum(s);
        const double alpha = __shfl_sync(0xffffffffu, av, j & 31);
        double t = 0.0, beta = alpha, scale = 1.0;
        if (s > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + s), alpha);
            t = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        double cf[QM];
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            const int i = lane + 32 * q;
            if (i > j && i < m) p[jj][q] *= scale;
            if (i == j) p[jj][q] = beta;
            cf[q] = (i > j && i < m) ? p[jj][q] : (i == j ? 1.0 : 0.0);
            if (i < m) A[i + (int64_t)lda * j] = p[jj][q];
        }
        if (lane == 0) tau[j] = t;
        if (t != 0.0) {
            // remaining panel columns jj+1 .. nb-1
            double w[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                double sw = 0.0;
                if (c > jj) {
#pragma unroll
                    for (int q = 0; q < QM; ++q) sw = fma(cf[q], p[c][q], sw);
                }
                w[c] = sw;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c > jj) w[c] += __shfl_xor_sync(0xffffffffu, w[c], o);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c > jj) {
                    const double tw = t * w[c];
#pragma unroll
                    for (int q = 0; q < QM; ++q) p[c][q] = fma(-cf[q], tw, p[c][q]);
                }
        }
    }
    __syncwarp();
}

// Columns k0 .. k1-1 (taken in pairs by the warps w0, w0 + ws, ...): apply H_j0 .. H_{j0+nb-1}.
template <int QM>
__device__ __forceinline__ void hh_trail(double *A, int lda, int m, int j0, int nb, const double *tau, int k0,
                                         int k1, int w0, int ws)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp < w0) return;
    for (int k = k0 + 2 * (warp - w0); k < k1; k += 2 * ws) {
        const bool two = k + 1 < k1;
        double b[2][QM];
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            const int i = lane + 32 * q;
            b[0][q] = (i < m) ? A[i + (int64_t)lda * k] : 0.0;
            b[1][q] = (two && i < m) ? A[i + (int64_t)lda * (k + 1)] : 0.0;
        }
        for (int jj = 0; jj < nb; ++jj) {
            const double t = tau[j0 + jj];
            if (t == 0.0) continue;
            double cf[QM];
            hh_coef<QM>(A, lda, m, j0 + jj, cf);
            hh_apply_reg<QM, 2>(cf, t, b);
        }
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            const int i = lane + 32 * q;
            if (i < m) {
                A[i + (int64_t)lda * k] = b[0][q];
                if (two) A[i + (int64_t)lda * (k + 1)] = b[1][q];
            }
        }
    }
}

template <int QM>
__device__ void qr_house_blk(double *A, int lda, int m, int R, double *tau)
{
    constexpr int NB = 4;
    const int warp = threadIdx.x >> 5;
    if (R <= 0) return;
    if (warp == 0) hh_panel<QM>(A, lda, m, 0, min(NB, R), tau);
    __syncthreads();
    for (int j0 = 0; j0 < R; j0 += NB) {
        const int nb = min(NB, R - j0);
        const int n0 = j0 + nb;
        const int nn = min(NB, R - n0);
        if (nn > 0) {
            // look-ahead: warps 0..3 update one column of the next panel each, then warp 0
            // factors it while warps 1.. finish the trailing update
            if (warp < 4) {
                if (warp < nn) hh_trail<QM>(A, lda, m, j0, nb, tau, n0 + warp, n0 + warp + 1, warp, 1);
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (warp == 0) hh_panel<QM>(A, lda, m, n0, nn, tau);
            }
            hh_trail<QM>(A, lda, m, j0, nb, tau, n0 + nn, R, 1, NWARP - 1);
        }
        __syncthreads();
    }
}

// Householder QR in shared memory: blocked register variant for m <= 256, else qr_house_sm.
__device__ __forceinline__ void qr_sm(double *A, int lda, int m, int R, double *tau)
{
    if (m <= 256) qr_house_blk<8>(A, lda, m, R, tau);
    else qr_house_sm(A, lda, m, R, tau);
}

// B <- Q B, Q = H_0 ... H_{R-1} from qr_house(_sm) (reflectors in shared memory, ld lda, m rows),
// B: m x r (global or shared, ld ldb).  Each warp carries NC columns of B in registers (rows
// lane + 32 q, q < QM, m <= 32 QM) through all R reflectors: no CTA barriers.
template <int QM, int NC>
__device__ void apply_q_reg(const double *A, int lda, int m, int R, const double *tau, double *B, int64_t ldb,
                            int r)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c0 = NC * warp; c0 < r; c0 += NC * NWARP) {
        double b[NC][QM];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int q = 0; q < QM; ++q) {
                const int i = lane + 32 * q;
                b[c][q] = (c0 + c < r && i < m) ? __ldcg(B + i + ldb * (c0 + c)) : 0.0;
            }
        for (int j = R - 1; j >= 0; --j) {
            const double t = tau[j];
            if (t == 0.0) continue;
            const double *v = A + (int64_t)lda * j;
            double cf[QM];
#pragma unroll
            for (int q = 0; q < QM; ++q) {
                const int i = lane + 32 * q;
                cf[q] = (i > j && i < m) ? v[i] : (i == j ? 1.0 : 0.0);
            }
            double w[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < QM; ++q) s = fma(cf[q], b[c][q], s);
                w[c] = s;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int c = 0; c < NC; ++c) w[c] += __shfl_xor_sync(0xffffffffu, w[c], o);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double tw = t * w[c];
#pragma unroll
                for (int q = 0; q < QM; ++q) b[c][q] = fma(-cf[q], tw, b[c][q]);
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int q = 0; q < QM; ++q) {
                const int i = lane + 32 * q;
                if (c0 + c < r && i < m) B[i + ldb * (c0 + c)] = b[c][q];
            }
    }
    __syncthreads();
}

// Dispatch of apply_q_reg by panel height (m <= 1024); returns false if m is too large.
__device__ bool apply_q_sm(const double *A, int lda, int m, int R, const double *tau, double *B, int64_t ldb, int r)
{
    if (m <= 256) {
        if (r <= NWARP) apply_q_reg<8, 1>(A, lda, m, R, tau, B, ldb, r);
        else apply_q_reg<8, 2>(A, lda, m, R, tau, B, ldb, r);
    } else if (m <= 512) {
        if (r <= NWARP) apply_q_reg<16, 1>(A, lda, m, R, tau, B, ldb, r);
        else apply_q_reg<16, 2>(A, lda, m, R, tau, B, ldb, r);
    } else if (m <= 1024) {
        apply_q_reg<32, 1>(A, lda, m, R, tau, B, ldb, r);
    } else {
        return false;
    }
    return true;
}

// Copy a panel (m x R) between global (ld ldg) and shared (ld m) memory.
__device__ __forceinline__ void panel_to_sm(double *S, const double *Gp, int64_t ldg, int m, int R)
{
    for (int e = threadIdx.x; e < m * R; e += NT) {
        const int i = e % m, c = e / m;
        S[e] = Gp[i + ldg * c];
    }
    __syncthreads();
}
__device__ __forceinline__ void panel_from_sm(double *Gp, int64_t ldg, const double *S, int m, int R)
{
    for (int e = threadIdx.x; e < m * R; e += NT) {
        const int i = e % m, c = e / m;
        Gp[i + ldg * c] = S[e];
    }
    __syncthreads();
}

// ------------------------------------------------------------------------------------------
// One-sided Jacobi SVD of G (K x nc, ld K, global scratch): on return G <- G J (columns mutually
// orthogonal, ||col_i|| = sigma_i) and J (nc x nc, ld nc) orthogonal, so G_in = (G J) J^T.
// Round-robin parallel ordering (nc/2 disjoint pairs per round, one warp per pair).  A pair is
// rotated while |g_p^T g_q| > 1e-13 ||g_p|| ||g_q||: the column norms are then the singular values
// to ~1e-13 relative, far below any truncation threshold used (eps >= 1e-11).
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
                if (ga != 0.0 && fabs(ga) > 1e-13 * sqrt(al * be)) {
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

// Same contract as qrcp_trunc with two CTA barriers per step: warp 0 selects the pivot (exact
// remaining column norms kept in cn), swaps and forms the reflector; then every warp applies it
// to its columns (k mod NWARP) and recomputes their exact remaining norms.
__device__ int qrcp_fast(double *M, int K, double tol, int rmax, double *tau, int *piv, double *cn)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double s_n1;
    __shared__ int s_stop;
    for (int k = threadIdx.x; k < K; k += NT) piv[k] = k;
    for (int k = warp; k < K; k += NWARP) {
        const double *mk = M + (int64_t)K * k;
        double sq = 0.0;
        for (int i = lane; i < K; i += 32) sq = fma(mk[i], mk[i], sq);
        sq = warp_sum(sq);
        if (lane == 0) cn[k] = sq;
    }
    __syncthreads();
    const int jmax = min(K, rmax);
    int j = 0;
    for (; j < jmax; ++j) {
        if (warp == 0) {
            double bv = -1.0;
            int bi = K;
            for (int k = j + lane; k < K; k += 32)
                if (cn[k] > bv || (cn[k] == bv && k < bi)) { bv = cn[k]; bi = k; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            const double nrm = sqrt(fmax(bv, 0.0));
            if (j == 0 && lane == 0) s_n1 = nrm;
            __syncwarp();
            const bool stop = !(nrm > tol * s_n1) || !(nrm > 0.0);
            if (lane == 0) s_stop = stop;
            if (!stop) {
                const int p = bi;
                double *aj = M + (int64_t)K * j;
                if (p != j) {
                    double *ap = M + (int64_t)K * p;
                    for (int i = lane; i < K; i += 32) { const double t = aj[i]; aj[i] = ap[i]; ap[i] = t; }
                    if (lane == 0) {
                        const int t = piv[j]; piv[j] = piv[p]; piv[p] = t;
                        cn[p] = cn[j];
                    }
                    __syncwarp();
                }
                double sq = 0.0;
                for (int i = j + 1 + lane; i < K; i += 32) sq = fma(aj[i], aj[i], sq);
                sq = warp_sum(sq);
                const double alpha = aj[j];
                double t = 0.0, beta = alpha;
                if (sq > 0.0) {
                    beta = -copysign(sqrt(alpha * alpha + sq), alpha);
                    t = (beta - alpha) / beta;
                    const double scale = 1.0 / (alpha - beta);
                    for (int i = j + 1 + lane; i < K; i += 32) aj[i] *= scale;
                }
                __syncwarp();
                if (lane == 0) { aj[j] = beta; tau[j] = t; }
            }
        }
        __syncthreads();
        if (s_stop) break;
        const double t = tau[j];
        const double *v = M + (int64_t)K * j;
        int k0 = warp;
        if (k0 <= j) k0 += NWARP * ((j - warp) / NWARP + 1);
        for (int k = k0; k < K; k += 4 * NWARP) {
            const int nk = min(4, (K - 1 - k) / NWARP + 1);
            if (t != 0.0) house_apply4(v, j, K, t, M, K, k, NWARP, nk);
            double sq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q < nk) {
                    const double *mk = M + (int64_t)K * (k + q * NWARP);
                    for (int i = j + 1 + lane; i < K; i += 32) sq[q] = fma(mk[i], mk[i], sq[q]);
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int q = 0; q < 4; ++q) sq[q] += __shfl_xor_sync(0xffffffffu, sq[q], o);
            if (lane == 0)
                for (int q = 0; q < nk; ++q) cn[k + q * NWARP] = sq[q];
        }
        __syncthreads();
    }
    __syncthreads();
    return j;
}

// ------------------------------------------------------------------------------------------
// Cholesky-QR path of the panel QRs (BLAS-3 shaped: streaming Gram products and GEMMs instead of
// one sweep over the panel per Householder reflector).  Shifted CholeskyQR3 (Fukaya et al.):
// column scaling, G = X^T X + s I, R = chol(G), X <- X R^{-1}, then two unshifted passes; the
// product of the triangular factors is R.  A Cholesky breakdown returns false (the caller falls
// back to Householder).
// ------------------------------------------------------------------------------------------

// G(a, b) = sum_i X(i, a) X(i, b) for a <= b (upper triangle, ld K).  4x4 register blocks per
// thread, row strips staged in shared memory (smem_dbl doubles available).
__device__ void gram_upper(const double *X, int64_t m, int64_t ld, int K, double *G, double *smem, int64_t smem_dbl)
{
    const int nb = (K + 3) / 4, W = 4 * nb;
    const int nblk = nb * (nb + 1) / 2;
    int RS = 32;
    while (RS > 1 && (int64_t)RS * W > smem_dbl) RS >>= 1;
    for (int p0 = 0; p0 < nblk; p0 += NT) {
        const int p = p0 + threadIdx.x;
        const bool act = p < nblk;
        int A = 0, off = 0;
        if (act)
            while (off + (nb - A) <= p) { off += nb - A; ++A; }
        const int B = A + (p - off);
        double acc[16];
#pragma unroll
        for (int z = 0; z < 16; ++z) acc[z] = 0.0;
        for (int64_t r0 = 0; r0 < m; r0 += RS) {
            const int rows = (int)(m - r0 < RS ? m - r0 : RS);
            __syncthreads();
            for (int e = threadIdx.x; e < RS * W; e += NT) {
                const int r = e % RS, cc = e / RS;
                smem[e] = (r < rows && cc < K) ? X[r0 + r + ld * cc] : 0.0;
            }
            __syncthreads();
            if (act) {
                const double *sa = smem + RS * 4 * A, *sb = smem + RS * 4 * B;
                for (int r = 0; r < rows; ++r) {
                    const double a0 = sa[r], a1 = sa[r + RS], a2 = sa[r + 2 * RS], a3 = sa[r + 3 * RS];
                    const double b0 = sb[r], b1 = sb[r + RS], b2 = sb[r + 2 * RS], b3 = sb[r + 3 * RS];
                    acc[0] = fma(a0, b0, acc[0]); acc[1] = fma(a0, b1, acc[1]);
                    acc[2] = fma(a0, b2, acc[2]); acc[3] = fma(a0, b3, acc[3]);
                    acc[4] = fma(a1, b0, acc[4]); acc[5] = fma(a1, b1, acc[5]);
                    acc[6] = fma(a1, b2, acc[6]); acc[7] = fma(a1, b3, acc[7]);
                    acc[8] = fma(a2, b0, acc[8]); acc[9] = fma(a2, b1, acc[9]);
                    acc[10] = fma(a2, b2, acc[10]); acc[11] = fma(a2, b3, acc[11]);
                    acc[12] = fma(a3, b0, acc[12]); acc[13] = fma(a3, b1, acc[13]);
                    acc[14] = fma(a3, b2, acc[14]); acc[15] = fma(a3, b3, acc[15]);
                }
            }
        }
        if (act)
            for (int u = 0; u < 4; ++u)
                for (int v = 0; v < 4; ++v) {
                    const int a = 4 * A + u, bb = 4 * B + v;
                    if (a <= bb && bb < K) G[a + (int64_t)K * bb] = acc[4 * u + v];
                }
    }
    __syncthreads();
}

// Upper Cholesky G = R^T R in place (upper triangle, ld K) by one warp (warp-synchronous).
// Returns false on a non-positive or non-finite pivot.
__device__ bool chol_upper_warp(double *G, int K)
{
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < K; ++k) {
        const double d = G[k + (int64_t)K * k];
        if (!(d > 0.0) || !isfinite(d)) return false;
        const double rk = sqrt(d);
        __syncwarp();
        for (int j = k + lane; j < K; j += 32) G[k + (int64_t)K * j] = (j == k) ? rk : G[k + (int64_t)K * j] / rk;
        __syncwarp();
        for (int j = k + 1 + lane; j < K; j += 32) {
            const double gkj = G[k + (int64_t)K * j];
            for (int i = k + 1; i <= j; ++i) G[i + (int64_t)K * j] -= G[k + (int64_t)K * i] * gkj;
        }
        __syncwarp();
    }
    return true;
}

// Ri = R^{-1} (upper triangular, ld K), one column per thread (back substitution).
__device__ void tri_inv_upper(const double *R, int K, double *Ri)
{
    for (int j = threadIdx.x; j < K; j += NT) {
        for (int i = j + 1; i < K; ++i) Ri[i + (int64_t)K * j] = 0.0;
        Ri[j + (int64_t)K * j] = 1.0 / R[j + (int64_t)K * j];
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int l = i + 1; l <= j; ++l) s += R[i + (int64_t)K * l] * Ri[l + (int64_t)K * j];
            Ri[i + (int64_t)K * j] = -s / R[i + (int64_t)K * i];
        }
    }
    __syncthreads();
}

// C = A B (A: m x K ld lda, B: K x K upper triangular ld K, C: m x K ld ldc, C != A)
__device__ void gemm_upper(double *C, int64_t ldc, const double *A, int64_t lda, int64_t m, int K, const double *B,
                           double *smem)
{
    for (int64_t e = threadIdx.x; e < m * (int64_t)K; e += NT) {
        const int64_t i = e % m, j = e / m;
        C[i + ldc * j] = 0.0;
    }
    __syncthreads();
    // C(i, j) += sum_l A(i, l) B(l, j) = sum_l A(i, l) Bt(j, l),  Bt(j, l) = B[l + K j]
    cta_gemm_nt(C, ldc, m, K, K, A, lda, B, K, 1, 1.0, smem);
}

// Shifted CholeskyQR3 of X (m x K, ld m) into Q (overwrites Xq, which must not alias X: the
// passes alternate X -> Xq -> X -> Xq) and R (upper, ld K; includes the column scaling).
// Returns false on breakdown.  smem: the engine's dynamic shared memory (smem_dbl doubles).
__device__ bool cholqr3(double *X, double *Xq, int64_t m, int K, double *R, double *Racc, double *G, double *Ri,
                        double *dcol, double *smem, int64_t smem_dbl, double *red, double **Qout)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int s_ok;
    // column scaling to unit norms
    for (int c = warp; c < K; c += NWARP) {
        double s = 0.0;
        for (int64_t i = lane; i < m; i += 32) s += X[i + m * c] * X[i + m * c];
        s = warp_sum(s);
        if (lane == 0) dcol[c] = (s > 0.0) ? sqrt(s) : 1.0;
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < m * (int64_t)K; e += NT) X[e] /= dcol[e / m];
    for (int e = threadIdx.x; e < K * K; e += NT) Racc[e] = ((e % K) == (e / K)) ? 1.0 : 0.0;
    __syncthreads();
    double *src = X, *dst = Xq;
    for (int pass = 0; pass < 3; ++pass) {
        // pass 0 is shifted; a later pass that breaks down (numerically rank-deficient panel) is
        // retried once with the shift 11 (m K + K (K + 1)) u tr(G)  (tr(G) >= ||X||_2^2)
        for (int attempt = (pass == 0 ? 1 : 0); attempt < 2; ++attempt) {
            gram_upper(src, m, m, K, G, smem, smem_dbl);
            if (attempt == 1 && threadIdx.x == 0) {
                double tr = 0.0;
                for (int a = 0; a < K; ++a) tr += G[a + (int64_t)K * a];
                const double sh = 11.0 * ((double)m * K + (double)K * (K + 1)) * 1.1102230246251565e-16 * tr;
                for (int a = 0; a < K; ++a) G[a + (int64_t)K * a] += sh;
            }
            __syncthreads();
            if (warp == 0) {
                const bool ok = chol_upper_warp(G, K);
                if (lane == 0) s_ok = ok;
            }
            __syncthreads();
            if (s_ok) break;
        }
        if (!s_ok) return false;
        // Racc <- R_pass Racc (both upper)
        for (int e = threadIdx.x; e < K * K; e += NT) {
            const int i = e % K, j = e / K;
            double sum = 0.0;
            for (int l = i; l <= j; ++l) sum += G[i + (int64_t)K * l] * Racc[l + (int64_t)K * j];
            R[e] = (i <= j) ? sum : 0.0;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < K * K; e += NT) Racc[e] = R[e];
        tri_inv_upper(G, K, Ri);
        gemm_upper(dst, m, src, m, m, K, Ri, smem);
        double *t = src; src = dst; dst = t;
    }
    // R = Racc diag(d)
    for (int e = threadIdx.x; e < K * K; e += NT) R[e] = Racc[e] * dcol[e / K];
    __syncthreads();
    *Qout = src;
    return true;
}

// Truncation workspace for R columns of m rows.
struct CompressWs {
    double *X, *Y;      // m x K each (ld m): inputs, destroyed (Householder vectors / Q factors)
    double *M, *G, *J;  // K x K, K x K, K x K
    double *tx, *ty, *tm;   // K each
    double *sig, *cn;   // K each
    int *ord, *piv;     // K each
    double *RX, *RY, *UC, *VC, *Ri;   // K x K each (Cholesky-QR path)
    double *T1, *T2;    // m x K each: Cholesky-QR ping-pong panels (Q_X ends in T1, Q_Y in T2)
    double *dX, *dY;    // K each (column scales)
    double *tail;       // first free (8-byte aligned) double after the workspace
    double *tsr;        // gang members with more than 256 rows: in-CTA TSQR region (ts_region_doubles)
    int K;              // column capacity of the panels and K x K arrays
};

// The core's K x K work arrays (M, G, J and vectors) in shared memory when they fit (R x R each).
__device__ __forceinline__ CompressWs core_ws_sm(const CompressWs &w, double *sm, int64_t dbl, int R)
{
    const int64_t RR = (int64_t)R * R;
    if (!sm || 3 * RR + 6 * (int64_t)R + 8 > dbl) return w;
    CompressWs c = w;
    c.M = sm;
    c.G = c.M + RR;
    c.J = c.G + RR;
    c.tm = c.J + RR;
    c.sig = c.tm + R;
    c.cn = c.sig + R;
    c.ord = (int *)(c.cn + R);
    c.piv = (int *)(c.cn + 2 * R);
    return c;
}

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
    PH_BEGIN(t1);
    for (int e = threadIdx.x; e < K * K; e += NT) {
        int i = e % K, j = e / K;
        double s = 0.0;
        for (int k = max(i, j); k < K; ++k) s += RX[i + ldx * k] * RY[j + ldy * k];
        w.M[e] = s;
    }
    __syncthreads();
    PH_END(1, t1);
    PH_BEGIN(t2);
    const int rq = qrcp_fast(w.M, K, tol_q, svd ? K : rlim + 1, w.tm, w.piv, w.cn);
    PH_END(2, t2);
    PH_BEGIN(t3);
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
    PH_END(3, t3);
    // U_core <- Q_M U_core (rows < K): registers when K <= 1024, else the global sweep
    if (!apply_q_sm(w.M, K, K, rq, w.tm, U, ldo, r)) qr_apply_q(w.M, K, K, rq, w.tm, U, ldo, r);
    if (threadIdx.x == 0) { *cap_bound = s_cb; *overflow = s_of; }
    __syncthreads();
    return r;
}

// Truncate X Y^T (m x m, rank <= R <= m) to U V^T: [Q_X, R_X] = qr(X), [Q_Y, R_Y] = qr(Y),
// core as above, U = Q_X [U_core; 0], V = Q_Y [V_core; 0].  U, V: m x r (ld ldo), must not
// alias X, Y.  Returns r.
__device__ int compress(const CompressWs &w, int64_t m, int R, double eps, double tol_q, bool svd, int kmax,
                        int rlim, double *U, double *V, int64_t ldo, int *cap_bound, int *overflow, double *red,
                        double *redv, int64_t *redi, double *smem = nullptr, int64_t smem_dbl = 0,
                        int qr_path = 2)
{
    if (R == 0) { if (threadIdx.x == 0) { *cap_bound = 0; *overflow = 0; } __syncthreads(); return 0; }
    if (smem && qr_path == 2 && m <= 1024 && m * (int64_t)R + R <= smem_dbl) {
        // shared-memory path: Householder QR of X and Y in shared memory (reflectors written back),
        // core, then Q_X / Q_Y applied to [U_core; 0] / [V_core; 0] held in registers
        const int mi = (int)m;
        double *As = smem, *ts = smem + m * (int64_t)R;
        PH_BEGIN(tc);
        panel_to_sm(As, w.X, m, mi, R);
        qr_sm(As, mi, mi, R, ts);
        for (int e = threadIdx.x; e < R; e += NT) w.tx[e] = ts[e];
        panel_from_sm(w.X, m, As, mi, R);
        panel_to_sm(As, w.Y, m, mi, R);
        qr_sm(As, mi, mi, R, ts);
        for (int e = threadIdx.x; e < R; e += NT) w.ty[e] = ts[e];
        panel_from_sm(w.Y, m, As, mi, R);
        PH_END(0, tc);
        const int r = compress_core(core_ws_sm(w, smem, smem_dbl, R), w.X, m, w.Y, m, R, eps, tol_q, svd, kmax, rlim,
                                    U, V, ldo, m, cap_bound, overflow, red, redv, redi);
        PH_BEGIN(t4);
        if (r > 0) {
            for (int e = threadIdx.x; e < R; e += NT) ts[e] = w.tx[e];
            panel_to_sm(As, w.X, m, mi, R);
            apply_q_sm(As, mi, mi, R, ts, U, ldo, r);
            for (int e = threadIdx.x; e < R; e += NT) ts[e] = w.ty[e];
            panel_to_sm(As, w.Y, m, mi, R);
            apply_q_sm(As, mi, mi, R, ts, V, ldo, r);
        }
        PH_END(4, t4);
        return r;
    }
    if (smem && qr_path != 0 && m >= 2 * R) {
        // BLAS-3 path: shifted CholeskyQR3 of X and Y, core, U = Q_X U_core, V = Q_Y V_core
        PH_BEGIN(tc);
        double *QX = nullptr, *QY = nullptr;
        bool ok = cholqr3(w.X, w.T1, m, R, w.RX, w.M, w.G, w.Ri, w.dX, smem, smem_dbl, red, &QX);
        if (ok) ok = cholqr3(w.Y, w.T2, m, R, w.RY, w.M, w.G, w.Ri, w.dY, smem, smem_dbl, red, &QY);
        PH_END(0, tc);
        if (!ok) {
            // breakdown (non-finite data): report as a rank-capacity failure
            if (threadIdx.x == 0) { *cap_bound = 0; *overflow = 1; }
            __syncthreads();
            return 0;
        }
        const int r = compress_core(w, w.RX, R, w.RY, R, R, eps, tol_q, svd, kmax, rlim, w.UC, w.VC, R, R, cap_bound,
                                    overflow, red, redv, redi);
        PH_BEGIN(t4c);
        for (int64_t e = threadIdx.x; e < m * (int64_t)r; e += NT) {
            const int64_t i = e % m, j = e / m;
            U[i + ldo * j] = 0.0;
            V[i + ldo * j] = 0.0;
        }
        __syncthreads();
        if (r > 0) {
            cta_gemm_nt(U, ldo, m, r, R, QX, m, w.UC, R, 1, 1.0, smem);
            cta_gemm_nt(V, ldo, m, r, R, QY, m, w.VC, R, 1, 1.0, smem);
        }
        PH_END(4, t4c);
        return r;
    }
    PH_BEGIN(t0);
    qr_house(w.X, m, m, R, w.tx, red);
    qr_house(w.Y, m, m, R, w.ty, red);
    PH_END(0, t0);
    const int r = compress_core(w, w.X, m, w.Y, m, R, eps, tol_q, svd, kmax, rlim, U, V, ldo, m, cap_bound, overflow,
                                red, redv, redi);
    PH_BEGIN(t4);
    qr_apply_q(w.X, m, m, R, w.tx, U, ldo, r);
    qr_apply_q(w.Y, m, m, R, w.ty, V, ldo, r);
    PH_END(4, t4);
    return r;
}

// ------------------------------------------------------------------------------------------
// Fully pivoted cross approximation of a dense m x m block S (global, ld m), destroyed.
// Appends up to Kmax columns to X, Y (ld m): S ~= X Y^T.  Stops when max |residual| <=
// rel_tol max |S| or ||residual||_F <= rel_fro ||S||_F (the residual is known exactly).
// ------------------------------------------------------------------------------------------
__device__ int aca_full(double *S, int64_t m, double *X, double *Y, int Kmax, double rel_tol, double rel_fro,
                        double *red, double *redv, int64_t *redi)
{
    // entries e = threadIdx.x + NT q (all threads busy for any m); the argmax ties go to the
    // lowest e, so the pivots do not depend on the traversal
    double bv = 0.0, ss = 0.0;
    int64_t bi = 0;
    const int64_t mm = m * m;
    const int mi = (int)m, mmi = (int)mm;   // m <= HCOV_DENSE_MAX (512)
    const int sh = ((mi & (mi - 1)) == 0) ? 31 - __clz(mi) : -1;
    for (int64_t e = threadIdx.x; e < mm; e += NT) {
        const double v = S[e], a = fabs(v);
        ss += v * v;
        if (vi_better(a, e, bv, bi)) { bv = a; bi = e; }
    }
    ValIdx b = block_argmax(bv, bi, redv, redi);
    const double fro0 = sqrt(block_sum(ss, red));
    const double tol = rel_tol * b.v, tolf = rel_fro * fro0;
    double fro = fro0;
    int k = 0;
    while (k < Kmax && b.v > tol && fro > tolf && b.v > 0.0) {
        const int64_t is = b.i % m, js = b.i / m;
        const double p = S[is + m * js];
        for (int64_t i = threadIdx.x; i < m; i += NT) {
            X[i + m * k] = S[i + m * js];
            Y[i + m * k] = S[is + m * i] / p;
        }
        __syncthreads();
        bv = 0.0; bi = 0; ss = 0.0;
        const double *xk = X + m * k, *yk = Y + m * k;
        // (i, j) of entry e in 32-bit arithmetic, by a shift when m is a power of two (every cluster
        // size is): the 64-bit division per entry was a sizeable part of this pass
        for (int e = threadIdx.x; e < mmi; e += NT) {
            const int j = sh >= 0 ? (e >> sh) : e / mi, i = e - j * mi;
            const double v = S[e] - xk[i] * yk[j];
            S[e] = v;
            ss += v * v;
            const double a = fabs(v);
            if (vi_better(a, (int64_t)e, bv, bi)) { bv = a; bi = e; }
        }
        b = block_argmax(bv, bi, redv, redi);
        fro = sqrt(block_sum(ss, red));
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
__device__ int aca_partial(const MaternParams &mp, const Pts P, int64_t r0,
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
        const bool d3 = P.z != nullptr;
        const double xi = P.x[r0 + istar], yi = P.y[r0 + istar], zi = d3 ? P.z[r0 + istar] : 0.0;
        double bv = 0.0; int64_t bi = 0;
        double *vk = V + m * k;
        for (int64_t j = threadIdx.x; j < m; j += NT) {
            double a = hcov_cov_entry_d(mp, xi, yi, zi, P.x[c0 + j], P.y[c0 + j], d3 ? P.z[c0 + j] : 0.0,
                                        (r0 + istar) == (c0 + j), d3);
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
        const double xj = P.x[c0 + js], yj = P.y[c0 + js], zj = d3 ? P.z[c0 + js] : 0.0;
        double *uk = U + m * k;
        bv = -1.0; bi = m;
        double su = 0.0, sv = 0.0;
        for (int64_t i = threadIdx.x; i < m; i += NT) {
            double c = hcov_cov_entry_d(mp, P.x[r0 + i], P.y[r0 + i], d3 ? P.z[r0 + i] : 0.0, xj, yj, zj,
                                        (r0 + i) == (c0 + js), d3);
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
