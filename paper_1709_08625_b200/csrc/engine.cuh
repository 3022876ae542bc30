// Task bodies of the DAG engine, one CTA (NT threads) per task.
// Data: dense 32x32 tiles, low-rank blocks U V^T (capacity kcap columns), pending
// Schur-complement terms (DTerm), forward-solve right-hand sides, product slots.
//
// Memory visibility: a task reads data written by other CTAs of the same persistent launch,
// so every load of mutable data goes through L2 (__ldcg); producers fence before they release
// their successors (hcov.cu, k_engine).
#pragma once
#include "hcov_internal.h"
#include "la.cuh"

// algorithmic flop counters per task class
enum FlopCls { FC_ASM = 0, FC_TILE = 1, FC_TRUNC = 2, FC_SOLVE = 3, FC_PROD = 4, FC_N = 5 };

struct Ctx {
    // ---- plan (theta-independent) ----
    const DNode *nodes;
    const int32_t *tile_node;
    const DRBlk *rblk;
    const DTerm *terms;
    const int32_t *xterm;
    const int64_t *fac_row0;
    const int32_t *fac_nrows;
    const int32_t *fac_rank_src;
    const int64_t *fac_off;
    const int8_t *fac_pool;
    const DSolve *solves;
    const int32_t *solve_rhs;
    const DSlot *slots;
    const DCtr *ctr;
    const DPhw *phw;
    const int32_t *col_r;
    const DTask *tasks;
    const int32_t *succ_off, *succ;
    const int32_t *diag_tile;
    const double *xs, *ys;
    const int64_t *perm_i2e;
    int32_t depth, n_r, root_solve, pad0;
    int64_t n_pad, n_leaves, n_real, n_tiles;
    // ---- numeric (per H-matrix) ----
    double *tiles;
    double *U, *V;
    int32_t *rank;
    double *cores;
    double *W;
    double *P;                 // product slots
    double *vbuf;              // root right-hand side / solution (internal order)
    double *logdet_part, *minpiv_part, *quad_part;
    int32_t *fail_leaf;        // min over failing leaves (init INT32_MAX)
    int32_t *flags;            // [0] cap binds, [1] rank overflow, [2] max rank
    int32_t kcap, kmax;
    double eps;
    MaternParams mp;
    // ---- engine ----
    int32_t *indeg;            // working copy of the in-degrees
    int32_t *queue[2];
    uint32_t *qctl;            // [0,1] head per queue, [2,3] tail per queue, [4] abort
    int32_t nq[2];
    int32_t nbig;              // CTAs serving queue 1
    int32_t pad1;
    double *scr;               // per-CTA scratch (normal CTAs), scr_stride doubles each
    int64_t scr_stride;
    double *bscr;              // per-CTA scratch of the big CTAs
    int64_t bscr_stride;
    double *flop;              // FC_N accumulators
    unsigned long long timeout_ns;
};

// ---------------------------------------------------------------------------------------------
struct Fac {
    const double *p;
    int64_t ld, row0;
    int32_t nrows, ncols;
};
__device__ __forceinline__ Fac get_fac(const Ctx &c, int f)
{
    Fac F;
    const int64_t off = c.fac_off[f] * (int64_t)c.kcap;
    F.p = (c.fac_pool[f] == 0 ? c.U : c.W) + off;
    F.nrows = c.fac_nrows[f];
    F.ld = F.nrows;
    F.row0 = c.fac_row0[f];
    F.ncols = __ldcg(c.rank + c.fac_rank_src[f]);
    return F;
}
__device__ __forceinline__ int64_t cl_size(const Ctx &c, int level) { return (int64_t)HCOV_LEAF << (c.depth - level); }
__device__ __forceinline__ double *r_U(const Ctx &c, int r) { return c.U + c.rblk[r].uv_off * (int64_t)c.kcap; }
__device__ __forceinline__ double *r_V(const Ctx &c, int r) { return c.V + c.rblk[r].uv_off * (int64_t)c.kcap; }
__device__ __forceinline__ double *slot_ptr(const Ctx &c, int s)
{
    const DSlot sl = c.slots[s];
    return c.P + sl.offa * (int64_t)c.kcap * c.kcap + sl.offb * (int64_t)c.kcap;
}

// Shared-memory layout of the tile tasks.
struct TileSmem {
    double *S, *A, *B, *K, *T, *L;
};
__host__ __device__ inline int64_t tile_smem_doubles(int kcap)
{
    int64_t w = 32 * (int64_t)(kcap > 32 ? kcap : 32);
    return 1024 + 3 * w + (int64_t)kcap * kcap + 1024 + 64;
}
__device__ __forceinline__ TileSmem tile_smem(double *base, int kcap)
{
    int64_t w = 32 * (int64_t)(kcap > 32 ? kcap : 32);
    TileSmem s;
    s.S = base;
    s.A = s.S + 1024;
    s.B = s.A + w;
    s.T = s.B + w;
    s.K = s.T + w;
    s.L = s.K + (int64_t)kcap * kcap;
    return s;
}

// S (32x32 smem) -= term, for a target tile at global rows R0.., cols C0..  Returns flops.
__device__ double tile_apply_term(const Ctx &c, const DTerm &t, int64_t R0, int64_t C0, const TileSmem &sm)
{
    if (t.kind == TM_TT) {
        tile_load(sm.A, c.tiles + (int64_t)t.a * HCOV_TILE);
        tile_load(sm.B, c.tiles + (int64_t)t.b * HCOV_TILE);
        __syncthreads();
        tile_gemm_nt_sub(sm.S, sm.A, sm.B);
        return 2.0 * 32 * 32 * 32;
    }
    Fac A = get_fac(c, t.a), B = get_fac(c, t.b);
    const int ra = A.ncols, rb = B.ncols;
    if (ra == 0 || rb == 0) return 0.0;
    const int64_t ao = R0 - A.row0, bo = C0 - B.row0;
    for (int e = threadIdx.x; e < 32 * ra; e += NT) {
        int i = e & 31, k = e >> 5;
        sm.A[e] = __ldcg(A.p + ao + i + A.ld * k);
    }
    for (int e = threadIdx.x; e < 32 * rb; e += NT) {
        int i = e & 31, k = e >> 5;
        sm.B[e] = __ldcg(B.p + bo + i + B.ld * k);
    }
    const double *T1 = sm.A;
    double fl = 2.0 * 32 * 32 * rb;
    if (t.core >= 0) {
        const double *K = c.cores + (int64_t)t.core * c.kcap * c.kcap;
        for (int e = threadIdx.x; e < ra * rb; e += NT) {
            int a = e % ra, b = e / ra;
            sm.K[e] = __ldcg(K + a + (int64_t)c.kcap * b);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 32 * rb; e += NT) {
            int i = e & 31, b = e >> 5;
            double s = 0.0;
            for (int a = 0; a < ra; ++a) s += sm.A[i + 32 * a] * sm.K[a + ra * b];
            sm.T[e] = s;
        }
        T1 = sm.T;
        fl += 2.0 * 32 * ra * rb;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
        int i = e & 31, j = e >> 5;
        double s = 0.0;
        for (int b = 0; b < rb; ++b) s += T1[i + 32 * b] * sm.B[j + 32 * b];
        sm.S[e] -= s;
    }
    __syncthreads();
    return fl;
}

// ---------------------------------------------------------------------------------------------
// A4: dense tiles of C~ (Eq. (3) + nugget on the diagonal)
__device__ void task_fill(const Ctx &c, const DTask &tk, double &fl)
{
    for (int t = tk.a; t < tk.a + tk.b; ++t) {
        const DNode x = c.nodes[c.tile_node[t]];
        const int64_t r0 = (int64_t)x.i * HCOV_LEAF, c0 = (int64_t)x.j * HCOV_LEAF;
        double *T = c.tiles + (int64_t)t * HCOV_TILE;
        for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
            int i = e & 31, j = e >> 5;
            int64_t a = r0 + i, b = c0 + j;
            __stcg(T + e, hcov_cov_entry(c.mp, c.xs[a], c.ys[a], c.xs[b], c.ys[b], a == b));
        }
    }
    fl += (double)tk.b * HCOV_TILE;   // kernel evaluations
}

// Scratch needs (doubles) for an ACA / RAPP task of block size m: two m x K panel pairs
// (inputs and outputs of an intermediate recompression), three K x K cores, vectors.
__host__ __device__ inline int aca_kmax(int64_t m, int kcap)
{
    int64_t k = 2 * (int64_t)kcap + 32;
    return (int)(k < m ? k : m);
}
__host__ __device__ inline int kbuf_of(int kcap) { return 3 * kcap + 32; }
__host__ __device__ inline int64_t task_scratch(int64_t m, int kcap)
{
    int64_t K = kbuf_of(kcap);
    return 4 * m * K + 3 * K * K + 8 * K + m / 8 + 64;
}

__device__ __forceinline__ CompressWs make_ws(double *base, int64_t m, int K, double **X2, double **Y2)
{
    CompressWs w;
    w.X = base;
    w.Y = w.X + m * K;
    *X2 = w.Y + m * K;
    *Y2 = *X2 + m * K;
    w.M = *Y2 + m * K;
    w.G = w.M + (int64_t)K * K;
    w.J = w.G + (int64_t)K * K;
    w.tx = w.J + (int64_t)K * K;
    w.ty = w.tx + K;
    w.tm = w.ty + K;
    w.sig = w.tm + K;
    w.cn = w.sig + K;
    w.ord = (int *)(w.cn + K);
    w.piv = w.ord + K;
    return w;
}

__device__ void record_rank(const Ctx &c, int r, int rk, int cb, int of)
{
    if (threadIdx.x == 0) {
        __stcg(c.rank + r, rk);
        if (cb) atomicAdd(c.flags + 0, 1);
        if (of) atomicAdd(c.flags + 1, 1);
        atomicMax(c.flags + 2, rk);
    }
    __syncthreads();
}

__device__ __forceinline__ double final_tol(double eps, int R) { return eps / (10.0 * sqrt((double)(R > 0 ? R : 1))); }
__device__ __forceinline__ double interm_tol(double eps) { return fmax(eps * 1e-4, 1e-15); }

__device__ __forceinline__ double compress_flops(int64_t m, int R, int r)
{
    // 2 Householder QRs, the core product, one-sided Jacobi (~6 sweeps), two Q applications
    return 2.0 * (4.0 * m * R * R - 4.0 * R * R * R / 3.0) + 2.0 * R * R * R / 3.0 + 6.0 * 9.0 * R * R * R +
           2.0 * 4.0 * m * R * r;
}

// A5 + A6: ACA of the admissible block (Alg. B.1) to eps/10, then QR + SVD truncation to (eps, kmax).
__device__ void task_aca(const Ctx &c, const DTask &tk, double *scr, double *red, double *redv, int64_t *redi,
                         double &fl_asm, double &fl_tr)
{
    const int r = tk.a;
    const DRBlk b = c.rblk[r];
    const int64_t m = b.m;
    const int K = aca_kmax(m, c.kcap);
    double *X2, *Y2;
    CompressWs w = make_ws(scr, m, kbuf_of(c.kcap), &X2, &Y2);
    uint8_t *used = (uint8_t *)(w.piv + kbuf_of(c.kcap) + 2);
    int k = aca_partial(c.mp, c.xs, c.ys, b.row0, b.col0, m, w.X, w.Y, K, 0.1 * c.eps, used, red, redv, redi);
    int cb = 0, of = 0;
    int rk = compress(w, m, k, c.eps, final_tol(c.eps, k), true, c.kmax, c.kcap, r_U(c, r), r_V(c, r), m, &cb, &of,
                      red, redv, redi);
    record_rank(c, r, rk, cb, of);
    fl_asm += 2.0 * m * k;                       // kernel evaluations (rows + columns)
    fl_tr += 2.0 * m * k * k + compress_flops(m, k, rk);
}

// ---------------------------------------------------------------------------------------------
// A7 tiles: apply pending terms [b, c) of xterm; then (POTRF) factor or (TRSM) X <- X L^{-T}.
__device__ void task_tile(const Ctx &c, const DTask &tk, double *smem, double &fl)
{
    TileSmem sm = tile_smem(smem, c.kcap);
    const int t = tk.a;
    const DNode x = c.nodes[c.tile_node[t]];
    double *Tg = c.tiles + (int64_t)t * HCOV_TILE;
    tile_load(sm.S, Tg);
    __syncthreads();
    const int64_t R0 = (int64_t)x.i * HCOV_LEAF, C0 = (int64_t)x.j * HCOV_LEAF;
    for (int k = tk.b; k < tk.c; ++k) fl += tile_apply_term(c, c.terms[c.xterm[k]], R0, C0, sm);
    if (tk.type == TK_POTRF) {
        double ls = 0.0, mp = 0.0;
        int f = tile_potrf(sm.S, &ls, &mp);
        if (threadIdx.x == 0) {
            if (f) {
                atomicMin(c.fail_leaf, x.i);
                c.logdet_part[x.i] = NAN;
                c.minpiv_part[x.i] = 0.0;
            } else {
                c.logdet_part[x.i] = ls;
                c.minpiv_part[x.i] = mp;
            }
        }
        fl += 32.0 * 32 * 32 / 3.0;
    } else if (tk.type == TK_TRSM) {
        tile_load(sm.L, c.tiles + (int64_t)tk.d * HCOV_TILE);
        __syncthreads();
        tile_trsm_rt(sm.S, sm.L);
        fl += 32.0 * 32 * 32;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) __stcg(Tg + e, sm.S[e]);
}

// A7 low-rank blocks: S = U V^T - sum of all pending terms, accumulated in factored form
// X = [U, -A_1 K_1, ...], Y = [V, B_1, ...] (in scratch).  When the panel is full it is
// recompressed near-losslessly (pivoted QR at eps*1e-4, no SVD); at the end X Y^T is truncated
// to (eps, kmax) by QR + SVD (A6; Remark 2).
__device__ void task_rapp(const Ctx &c, const DTask &tk, double *scr, double *red, double *redv, int64_t *redi,
                          double &fl)
{
    const int r = tk.a;
    const DRBlk blk = c.rblk[r];
    const int64_t m = blk.m;
    const int64_t R0 = blk.row0, C0 = blk.col0;
    double *U = r_U(c, r), *V = r_V(c, r);
    const int r0 = __ldcg(c.rank + r);
    int cb = 0, of = 0;
    const int K = kbuf_of(c.kcap);
    const int maxw = max(32, c.kcap);
    double *X2, *Y2;
    CompressWs w = make_ws(scr, m, K, &X2, &Y2);
    if (m <= K) {
        // small block: exact dense accumulation S = U V^T - sum of terms, then X = S, Y = I
        double *S = w.X;
        for (int64_t e = threadIdx.x; e < m * m; e += NT) {
            const int64_t i = e % m, j = e / m;
            double sum = 0.0;
            for (int l = 0; l < r0; ++l) sum += __ldcg(U + i + m * l) * __ldcg(V + j + m * l);
            S[e] = sum;
            w.Y[e] = (i == j) ? 1.0 : 0.0;
        }
        fl += 2.0 * m * m * r0;
        __syncthreads();
        for (int kk = tk.b; kk < tk.c; ++kk) {
            const DTerm t = c.terms[c.xterm[kk]];
            if (t.kind == TM_TT) {
                const DNode na = c.nodes[c.tile_node[t.a]], nb = c.nodes[c.tile_node[t.b]];
                const int64_t ar = (int64_t)na.i * HCOV_LEAF - R0, br = (int64_t)nb.i * HCOV_LEAF - C0;
                const double *A = c.tiles + (int64_t)t.a * HCOV_TILE, *B = c.tiles + (int64_t)t.b * HCOV_TILE;
                for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
                    int i = e & 31, j = e >> 5;
                    double sum = 0.0;
                    for (int l = 0; l < 32; ++l) sum += __ldcg(A + i + 32 * l) * __ldcg(B + j + 32 * l);
                    S[(ar + i) + m * (br + j)] -= sum;
                }
                fl += 2.0 * 32 * 32 * 32;
            } else {
                Fac A = get_fac(c, t.a), B = get_fac(c, t.b);
                const int ra = A.ncols, rb = B.ncols;
                if (ra == 0 || rb == 0) continue;
                const int64_t r_lo = max(R0, A.row0), r_hi = min(R0 + m, A.row0 + A.nrows);
                const int64_t c_lo = max(C0, B.row0), c_hi = min(C0 + m, B.row0 + B.nrows);
                const int64_t nr = r_hi - r_lo, nc = c_hi - c_lo;
                const double *Kc = (t.core >= 0) ? c.cores + (int64_t)t.core * c.kcap * c.kcap : nullptr;
                double *T1 = X2;   // nr x rb
                for (int64_t e = threadIdx.x; e < nr * (int64_t)rb; e += NT) {
                    int64_t i = e % nr;
                    int b = (int)(e / nr);
                    double sum;
                    if (Kc) {
                        sum = 0.0;
                        for (int a = 0; a < ra; ++a)
                            sum += __ldcg(A.p + (r_lo - A.row0) + i + A.ld * a) * __ldcg(Kc + a + (int64_t)c.kcap * b);
                    } else {
                        sum = __ldcg(A.p + (r_lo - A.row0) + i + A.ld * b);
                    }
                    T1[e] = sum;
                }
                __syncthreads();
                for (int64_t e = threadIdx.x; e < nr * nc; e += NT) {
                    const int64_t i = e % nr, j = e / nr;
                    double sum = 0.0;
                    for (int b = 0; b < rb; ++b) sum += T1[i + nr * b] * __ldcg(B.p + (c_lo - B.row0) + j + B.ld * b);
                    S[(r_lo - R0 + i) + m * (c_lo - C0 + j)] -= sum;
                }
                fl += 2.0 * nr * nc * rb + (Kc ? 2.0 * nr * ra * rb : 0.0);
            }
            __syncthreads();
        }
        int rk = compress(w, m, (int)m, c.eps, final_tol(c.eps, (int)m), true, c.kmax, c.kcap, U, V, m, &cb, &of,
                          red, redv, redi);
        fl += compress_flops(m, (int)m, rk);
        record_rank(c, r, rk, cb, of);
        return;
    }
    int cur = r0;
    for (int64_t e = threadIdx.x; e < m * (int64_t)r0; e += NT) { w.X[e] = __ldcg(U + e); w.Y[e] = __ldcg(V + e); }
    __syncthreads();
    for (int kk = tk.b; kk < tk.c; ++kk) {
        const DTerm t = c.terms[c.xterm[kk]];
        int width;
        if (t.kind == TM_TT) width = 32;
        else width = __ldcg(c.rank + c.fac_rank_src[t.b]);
        if (width == 0) continue;
        if (t.kind == TM_LR && __ldcg(c.rank + c.fac_rank_src[t.a]) == 0) continue;
        if (cur + width > K) {
            int icb = 0, iof = 0;
            int rk = compress(w, m, cur, c.eps, interm_tol(c.eps), false, 0, K - maxw, X2, Y2, m, &icb, &iof, red,
                              redv, redi);
            fl += compress_flops(m, cur, rk);
            if (iof && threadIdx.x == 0) atomicAdd(c.flags + 3, 1);
            double *tx = w.X, *ty = w.Y;
            w.X = X2; w.Y = Y2; X2 = tx; Y2 = ty;
            cur = rk;
        }
        double *xc = w.X + m * cur, *yc = w.Y + m * cur;
        for (int64_t e = threadIdx.x; e < m * (int64_t)width; e += NT) { xc[e] = 0.0; yc[e] = 0.0; }
        __syncthreads();
        if (t.kind == TM_TT) {
            const DNode na = c.nodes[c.tile_node[t.a]], nb = c.nodes[c.tile_node[t.b]];
            const int64_t ar = (int64_t)na.i * HCOV_LEAF - R0, br = (int64_t)nb.i * HCOV_LEAF - C0;
            const double *A = c.tiles + (int64_t)t.a * HCOV_TILE, *B = c.tiles + (int64_t)t.b * HCOV_TILE;
            for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
                int i = e & 31, k = e >> 5;
                xc[ar + i + m * k] = -__ldcg(A + e);
                yc[br + i + m * k] = __ldcg(B + e);
            }
        } else {
            Fac A = get_fac(c, t.a), B = get_fac(c, t.b);
            const int ra = A.ncols, rb = B.ncols;
            const int64_t r_lo = max(R0, A.row0), r_hi = min(R0 + m, A.row0 + A.nrows);
            const int64_t c_lo = max(C0, B.row0), c_hi = min(C0 + m, B.row0 + B.nrows);
            const double *Kc = (t.core >= 0) ? c.cores + (int64_t)t.core * c.kcap * c.kcap : nullptr;
            for (int64_t e = threadIdx.x; e < (r_hi - r_lo) * (int64_t)rb; e += NT) {
                int64_t i = e % (r_hi - r_lo);
                int b = (int)(e / (r_hi - r_lo));
                double s;
                if (Kc) {
                    s = 0.0;
                    for (int a = 0; a < ra; ++a)
                        s += __ldcg(A.p + (r_lo - A.row0) + i + A.ld * a) * __ldcg(Kc + a + (int64_t)c.kcap * b);
                } else {
                    s = __ldcg(A.p + (r_lo - A.row0) + i + A.ld * b);
                }
                xc[(r_lo - R0) + i + m * b] = -s;
            }
            for (int64_t e = threadIdx.x; e < (c_hi - c_lo) * (int64_t)rb; e += NT) {
                int64_t i = e % (c_hi - c_lo);
                int b = (int)(e / (c_hi - c_lo));
                yc[(c_lo - C0) + i + m * b] = __ldcg(B.p + (c_lo - B.row0) + i + B.ld * b);
            }
            if (Kc) fl += 2.0 * (r_hi - r_lo) * ra * rb;
        }
        __syncthreads();
        cur += width;
    }
    int rk = compress(w, m, cur, c.eps, final_tol(c.eps, cur), true, c.kmax, c.kcap, U, V, m, &cb, &of, red, redv,
                      redi);
    fl += compress_flops(m, cur, rk);
    record_rank(c, r, rk, cb, of);
}

// ---------------------------------------------------------------------------------------------
// Right-hand sides of a solve: column j of the concatenated RHS -> pointer to Y(row0_s.., j).
struct Rhs {
    int cnt;          // number of R entries (0 = root vector)
    int off;
    int64_t m, row0;
};
__device__ __forceinline__ Rhs get_rhs(const Ctx &c, int s)
{
    const DSolve sv = c.solves[s];
    Rhs h;
    h.cnt = sv.rhs_cnt;
    h.off = sv.rhs_off;
    h.m = sv.m;
    h.row0 = sv.row0;
    return h;
}

#define SEG_MAXCOL 64   // right-hand-side columns processed per pass of a SEG / PHWR task

// Column map of a pass: smem arrays colp[k] = base pointer of column k of Y (rows relative to
// the solve's row0), for columns [k0, k0 + nk) of the concatenated right-hand side.
__device__ int rhs_columns(const Ctx &c, const Rhs &h, int k0, double **colp, int *total)
{
    // returns nk, fills colp (thread 0 only; caller syncs)
    if (h.cnt == 0) {
        *total = 1;
        if (k0 == 0) { colp[0] = c.vbuf + h.row0; return 1; }
        return 0;
    }
    int k = 0, nk = 0;
    for (int q = 0; q < h.cnt; ++q) {
        const int r = c.solve_rhs[h.off + q];
        const int rk = __ldcg(c.rank + r);
        double *Vr = r_V(c, r);
        for (int j = 0; j < rk; ++j, ++k)
            if (k >= k0 && nk < SEG_MAXCOL) colp[nk++] = Vr + h.m * (int64_t)j;
    }
    *total = k;
    return nk;
}

// A7 (V <- L_ss^{-1} V) and A9 (v = L^{-1} z): rows of one leaf segment i of solve s.
//   Y_i -= sum_{tiles (i,j), j < i} L_ij Y_j + sum_{low-rank b over row i} U_b[i] P_b;  Y_i <- L_ii^{-1} Y_i
__device__ void task_seg(const Ctx &c, const DTask &tk, double *smem, double &fl)
{
    const Rhs h = get_rhs(c, tk.a);
    const int64_t i = tk.b;
    const int64_t ro = i * HCOV_LEAF - h.row0;   // local row offset of the segment
    double *Ys = smem;                            // 32 x SEG_MAXCOL
    double *Ts = Ys + 32 * SEG_MAXCOL;            // 32 x 32 tile
    double *Xs = Ts + HCOV_TILE;                  // 32 x SEG_MAXCOL (Y_j) / kcap x SEG_MAXCOL (P)
    double *Us = Xs + (int64_t)max(32, c.kcap) * SEG_MAXCOL;   // 32 x kcap
    double **colp = (double **)(Us + 32 * (int64_t)c.kcap);
    __shared__ int s_nk, s_total;
    int k0 = 0;
    double q = 0.0;
    while (true) {
        if (threadIdx.x == 0) { int tot; s_nk = rhs_columns(c, h, k0, colp, &tot); s_total = tot; }
        __syncthreads();
        const int nk = s_nk;
        if (nk == 0) break;
        for (int e = threadIdx.x; e < 32 * nk; e += NT) {
            int rr = e & 31, k = e >> 5;
            Ys[e] = __ldcg(colp[k] + ro + rr);
        }
        __syncthreads();
        for (int z = tk.c; z < tk.d; ++z) {
            const DCtr ct = c.ctr[z];
            if (ct.kind == 0) {
                tile_load(Ts, c.tiles + (int64_t)ct.id * HCOV_TILE);
                const int64_t jo = (int64_t)ct.aux * HCOV_LEAF - h.row0;
                for (int e = threadIdx.x; e < 32 * nk; e += NT) {
                    int rr = e & 31, k = e >> 5;
                    Xs[e] = __ldcg(colp[k] + jo + rr);
                }
                __syncthreads();
                for (int e = threadIdx.x; e < 32 * nk; e += NT) {
                    int rr = e & 31, k = e >> 5;
                    double s = 0.0;
#pragma unroll 8
                    for (int l = 0; l < 32; ++l) s += Ts[rr + 32 * l] * Xs[l + 32 * k];
                    Ys[e] -= s;
                }
                fl += 2.0 * 32 * 32 * nk;
            } else {
                const int r = ct.id;
                const int rk = __ldcg(c.rank + r);
                if (rk == 0) continue;
                const DRBlk b = c.rblk[r];
                const double *Ub = r_U(c, r);
                const double *Pb = slot_ptr(c, ct.aux);
                const int64_t uo = i * HCOV_LEAF - b.row0;
                for (int e = threadIdx.x; e < 32 * rk; e += NT) {
                    int rr = e & 31, l = e >> 5;
                    Us[e] = __ldcg(Ub + uo + rr + (int64_t)b.m * l);
                }
                for (int e = threadIdx.x; e < rk * nk; e += NT) {
                    int l = e % rk, k = e / rk;
                    Xs[e] = __ldcg(Pb + l + (int64_t)c.kcap * (k0 + k));
                }
                __syncthreads();
                for (int e = threadIdx.x; e < 32 * nk; e += NT) {
                    int rr = e & 31, k = e >> 5;
                    double s = 0.0;
                    for (int l = 0; l < rk; ++l) s += Us[rr + 32 * l] * Xs[l + rk * k];
                    Ys[e] -= s;
                }
                fl += 2.0 * 32 * rk * nk;
            }
            __syncthreads();
        }
        // Y_i <- L_ii^{-1} Y_i (forward substitution, one thread per column)
        tile_load(Ts, c.tiles + (int64_t)c.diag_tile[i] * HCOV_TILE);
        __syncthreads();
        for (int k = threadIdx.x; k < nk; k += NT) {
            double *y = Ys + 32 * k;
            for (int a = 0; a < 32; ++a) {
                double s = y[a];
                for (int l = 0; l < a; ++l) s -= Ts[a + 32 * l] * y[l];
                y[a] = s / Ts[a + 32 * a];
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 32 * nk; e += NT) {
            int rr = e & 31, k = e >> 5;
            __stcg(colp[k] + ro + rr, Ys[e]);
            if (h.cnt == 0) q += Ys[e] * Ys[e];
        }
        fl += 32.0 * 32 * nk;
        k0 += nk;
        __syncthreads();
        if (k0 >= s_total) break;
    }
    if (h.cnt == 0) {
        __shared__ double red[NWARP];
        q = block_sum(q, red);
        if (threadIdx.x == 0) c.quad_part[i] = q;
    }
}

// P = V_b^T Y[cols of b]  (rank_b x ctot, ld kcap)
__device__ void task_proj(const Ctx &c, const DTask &tk, double *smem, double &fl)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Rhs h = get_rhs(c, tk.a);
    const int r = tk.b;
    const DRBlk b = c.rblk[r];
    const int rk = __ldcg(c.rank + r);
    const double *Vb = r_V(c, r);
    double *Pb = slot_ptr(c, tk.c);
    double **colp = (double **)smem;
    __shared__ int s_nk, s_total;
    const int64_t co = b.col0 - h.row0;
    int k0 = 0;
    while (true) {
        if (threadIdx.x == 0) { int tot; s_nk = rhs_columns(c, h, k0, colp, &tot); s_total = tot; }
        __syncthreads();
        const int nk = s_nk;
        if (nk == 0) break;
        for (int pq = warp; pq < rk * nk; pq += NWARP) {
            const int l = pq % rk, k = pq / rk;
            const double *vl = Vb + (int64_t)b.m * l;
            const double *y = colp[k] + co;
            double s = 0.0;
            for (int64_t q = lane; q < b.m; q += 32) s += __ldcg(vl + q) * __ldcg(y + q);
            s = warp_sum(s);
            if (lane == 0) __stcg(Pb + l + (int64_t)c.kcap * (k0 + k), s);
        }
        fl += 2.0 * b.m * rk * nk;
        k0 += nk;
        __syncthreads();
        if (k0 >= s_total) break;
    }
}

// K = V_a^T V_b  (Schur term core of two low-rank entries of one column)
__device__ void task_prr(const Ctx &c, const DTask &tk, double &fl)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ra = __ldcg(c.rank + tk.a), rb = __ldcg(c.rank + tk.b);
    const int64_t m = c.rblk[tk.a].m;
    const double *Va = r_V(c, tk.a), *Vb = r_V(c, tk.b);
    double *K = c.cores + (int64_t)tk.c * c.kcap * c.kcap;
    for (int pq = warp; pq < ra * rb; pq += NWARP) {
        int a = pq % ra, b = pq / ra;
        double s = 0.0;
        for (int64_t i = lane; i < m; i += 32) s += __ldcg(Va + i + m * a) * __ldcg(Vb + i + m * b);
        s = warp_sum(s);
        if (lane == 0) __stcg(K + a + (int64_t)c.kcap * b, s);
    }
    fl += 2.0 * m * ra * rb;
}

// Q_x = V_x^T V_p[cols of x] for every partner p (Q: kcap x (kcap * part_cnt))
__device__ void task_phwp(const Ctx &c, const DTask &tk, double &fl)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const DPhw q = c.phw[tk.a];
    const DNode hn = c.nodes[q.hnode];
    const int64_t sig0 = (int64_t)hn.j * q.m;
    const int x = tk.b;
    const DRBlk bx = c.rblk[x];
    const int rx = __ldcg(c.rank + x);
    const double *Vx = r_V(c, x);
    double *Q = slot_ptr(c, tk.c);
    const int64_t co = bx.col0 - sig0;
    for (int p = 0; p < q.part_cnt; ++p) {
        const int rp_id = c.col_r[q.part_off + p];
        const int rp = __ldcg(c.rank + rp_id);
        const double *Vp = r_V(c, rp_id);
        for (int pq = warp; pq < rx * rp; pq += NWARP) {
            const int l = pq % rx, k = pq / rx;
            double s = 0.0;
            for (int64_t i = lane; i < bx.m; i += 32) s += __ldcg(Vx + i + (int64_t)bx.m * l) * __ldcg(Vp + co + i + (int64_t)q.m * k);
            s = warp_sum(s);
            if (lane == 0) __stcg(Q + l + (int64_t)c.kcap * (p * c.kcap + k), s);
        }
        fl += 2.0 * bx.m * rx * rp;
    }
}

// W[rows of segment i] = H(rows, :) [V_p]  for every partner p
__device__ void task_phwr(const Ctx &c, const DTask &tk, double *smem, double &fl)
{
    const DPhw q = c.phw[tk.a];
    const DNode hn = c.nodes[q.hnode];
    const int64_t rho0 = (int64_t)hn.i * q.m, sig0 = (int64_t)hn.j * q.m;
    const int64_t i = tk.b;
    const int64_t ro = i * HCOV_LEAF - rho0;
    double *Ws = smem;                        // 32 x kcap
    double *Ts = Ws + 32 * (int64_t)c.kcap;   // 32 x 32
    double *Xs = Ts + HCOV_TILE;              // 32 x kcap
    double *Us = Xs + 32 * (int64_t)max(32, c.kcap);
    for (int p = 0; p < q.part_cnt; ++p) {
        const int rp_id = c.col_r[q.part_off + p];
        const int rp = __ldcg(c.rank + rp_id);
        const double *Vp = r_V(c, rp_id);
        double *Wp = c.W + (q.w_off + (int64_t)p * q.m) * c.kcap;
        if (rp == 0) continue;
        for (int e = threadIdx.x; e < 32 * rp; e += NT) Ws[e] = 0.0;
        __syncthreads();
        for (int z = tk.c; z < tk.d; ++z) {
            const DCtr ct = c.ctr[z];
            if (ct.kind == 0) {
                tile_load(Ts, c.tiles + (int64_t)ct.id * HCOV_TILE);
                const int64_t jo = (int64_t)ct.aux * HCOV_LEAF - sig0;
                for (int e = threadIdx.x; e < 32 * rp; e += NT) {
                    int rr = e & 31, k = e >> 5;
                    Xs[e] = __ldcg(Vp + jo + rr + (int64_t)q.m * k);
                }
                __syncthreads();
                for (int e = threadIdx.x; e < 32 * rp; e += NT) {
                    int rr = e & 31, k = e >> 5;
                    double s = 0.0;
#pragma unroll 8
                    for (int l = 0; l < 32; ++l) s += Ts[rr + 32 * l] * Xs[l + 32 * k];
                    Ws[e] += s;
                }
                fl += 2.0 * 32 * 32 * rp;
            } else {
                const int x = ct.id;
                const int rx = __ldcg(c.rank + x);
                if (rx == 0) continue;
                const DRBlk bx = c.rblk[x];
                const double *Ux = r_U(c, x);
                const double *Qx = slot_ptr(c, ct.aux);
                const int64_t uo = i * HCOV_LEAF - bx.row0;
                for (int e = threadIdx.x; e < 32 * rx; e += NT) {
                    int rr = e & 31, l = e >> 5;
                    Us[e] = __ldcg(Ux + uo + rr + (int64_t)bx.m * l);
                }
                for (int e = threadIdx.x; e < rx * rp; e += NT) {
                    int l = e % rx, k = e / rx;
                    Xs[e] = __ldcg(Qx + l + (int64_t)c.kcap * (p * c.kcap + k));
                }
                __syncthreads();
                for (int e = threadIdx.x; e < 32 * rp; e += NT) {
                    int rr = e & 31, k = e >> 5;
                    double s = 0.0;
                    for (int l = 0; l < rx; ++l) s += Us[rr + 32 * l] * Xs[l + rx * k];
                    Ws[e] += s;
                }
                fl += 2.0 * 32 * rx * rp;
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < 32 * rp; e += NT) {
            int rr = e & 31, k = e >> 5;
            __stcg(Wp + ro + rr + (int64_t)q.m * k, Ws[e]);
        }
        __syncthreads();
    }
}

// shared memory (doubles) of the engine's task bodies
__host__ __device__ inline int64_t engine_smem_doubles(int kcap)
{
    int64_t a = tile_smem_doubles(kcap);
    int64_t k = kcap > 32 ? kcap : 32;
    int64_t b = 32 * SEG_MAXCOL + HCOV_TILE + k * SEG_MAXCOL + 32 * (int64_t)kcap + SEG_MAXCOL + 8;
    int64_t cc = 32 * (int64_t)kcap + HCOV_TILE + 32 * k + 32 * (int64_t)kcap + 8;
    int64_t m = a > b ? a : b;
    return m > cc ? m : cc;
}
