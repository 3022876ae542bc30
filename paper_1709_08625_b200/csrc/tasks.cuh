// Task bodies of the lazy column-oriented H-Cholesky, one CTA (NT threads)
// per task.  Data: dense 32x32 tiles, low-rank blocks U V^T (capacity kcap columns), pending
// Schur-complement terms (DTerm) attached to block-tree nodes.
#pragma once
#include "hcov_internal.h"
#include "la.cuh"

struct Ctx {
    // ---- plan (theta-independent) ----
    const DNode *nodes;
    const int32_t *children;
    const DTerm *terms;
    const DTask *tasks;
    const DRBlk *rblk;
    const int32_t *tile_node;
    const DPhw *phw;
    const int32_t *phw_part;
    const int32_t *hleaf;
    const int32_t *col_r_off, *col_r;
    const DOp *ops;
    const int32_t *op_beg, *op_end;
    const int64_t *fac_row0;
    const int32_t *fac_nrows;
    const int32_t *fac_rank_src;
    const int64_t *fac_off;
    const int8_t *fac_pool;
    const int32_t *row_off, *row_nodes;
    const double *xs, *ys;
    const int64_t *perm_i2e;
    int32_t depth;
    int32_t n_r;
    int64_t n_pad, n_leaves, n_real;
    // ---- numeric (per H-matrix) ----
    double *tiles;
    double *U, *V;
    int32_t *rank;
    double *cores;
    double *W;
    double *logdet_part, *minpiv_part;
    int32_t *fail_leaf;        // min over failing leaves (init INT32_MAX)
    int32_t *flags;            // [0] cap binds (count), [1] rank overflow (count), [2] max rank
    int32_t kcap, kmax;
    double eps;
    MaternParams mp;
    // ---- scratch slots ----
    double *scr[2];
    int64_t scr_stride[2];     // doubles per slot
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

// Shared-memory layout for tile finalisation.
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

// S (32x32 smem) -= term, for a target tile at global rows R0.., cols C0..
__device__ void tile_apply_term(const Ctx &c, const DTerm &t, int64_t R0, int64_t C0, const TileSmem &sm)
{
    if (t.kind == TM_TT) {
        tile_load(sm.A, c.tiles + (int64_t)t.a * HCOV_TILE);
        tile_load(sm.B, c.tiles + (int64_t)t.b * HCOV_TILE);
        __syncthreads();
        tile_gemm_nt_sub(sm.S, sm.A, sm.B);
        return;
    }
    Fac A = get_fac(c, t.a), B = get_fac(c, t.b);
    const int ra = A.ncols, rb = B.ncols;
    if (ra == 0 || rb == 0) return;
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
    }
    __syncthreads();
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
        int i = e & 31, j = e >> 5;
        double s = 0.0;
        for (int b = 0; b < rb; ++b) s += T1[i + 32 * b] * sm.B[j + 32 * b];
        sm.S[e] -= s;
    }
    __syncthreads();
}

// S = C~_tile - sum of all pending terms of the node and its ancestors.
__device__ void tile_finalize(const Ctx &c, int nd, const TileSmem &sm)
{
    const DNode x = c.nodes[nd];
    tile_load(sm.S, c.tiles + (int64_t)x.idx * HCOV_TILE);
    __syncthreads();
    const int64_t R0 = (int64_t)x.i * HCOV_LEAF, C0 = (int64_t)x.j * HCOV_LEAF;
    for (int y = nd; y >= 0; y = c.nodes[y].parent) {
        const DNode ny = c.nodes[y];
        for (int k = 0; k < ny.term_cnt; ++k) tile_apply_term(c, c.terms[ny.term_off + k], R0, C0, sm);
    }
}

__device__ void task_potrf(const Ctx &c, const DTask &tk, double *smem)
{
    TileSmem sm = tile_smem(smem, c.kcap);
    tile_finalize(c, tk.a, sm);
    const DNode x = c.nodes[tk.a];
    double ls = 0.0, mp = 0.0;
    int f = tile_potrf(sm.S, &ls, &mp);
    __shared__ double s_ls, s_mp;
    if (threadIdx.x == 0) { s_ls = ls; s_mp = mp; }
    __syncthreads();
    if (f) {
        if (threadIdx.x == 0) {
            atomicMin(c.fail_leaf, x.i);
            c.logdet_part[x.i] = NAN;
            c.minpiv_part[x.i] = 0.0;
        }
    } else if (threadIdx.x == 0) {
        c.logdet_part[x.i] = s_ls;
        c.minpiv_part[x.i] = s_mp;
    }
    tile_store(c.tiles + (int64_t)x.idx * HCOV_TILE, sm.S);
}

__device__ void task_trsm(const Ctx &c, const DTask &tk, double *smem)
{
    TileSmem sm = tile_smem(smem, c.kcap);
    tile_finalize(c, tk.a, sm);
    tile_load(sm.L, c.tiles + (int64_t)tk.b * HCOV_TILE);
    __syncthreads();
    tile_trsm_rt(sm.S, sm.L);
    const DNode x = c.nodes[tk.a];
    tile_store(c.tiles + (int64_t)x.idx * HCOV_TILE, sm.S);
}

// ---------------------------------------------------------------------------------------------
// Dense m x m block helpers (global scratch, ld m), used by the R finalisation.
// S[rows r_lo..r_hi) x [cols c_lo..c_hi) (block-relative) -= A[arow..] K B[brow..]^T
__device__ void dense_sub_term(const Ctx &c, const DTerm &t, double *S, int64_t m, int64_t R0, int64_t C0,
                               double *T1scr)
{
    if (t.kind == TM_TT) {
        const DNode na = c.nodes[c.tile_node[t.a]], nb = c.nodes[c.tile_node[t.b]];
        const int64_t ar = (int64_t)na.i * HCOV_LEAF - R0, br = (int64_t)nb.i * HCOV_LEAF - C0;
        if (ar < 0 || ar >= m || br < 0 || br >= m) return;   // (cannot happen for owned sub-terms)
        const double *A = c.tiles + (int64_t)t.a * HCOV_TILE, *B = c.tiles + (int64_t)t.b * HCOV_TILE;
        for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
            int i = e & 31, j = e >> 5;
            double s = 0.0;
            for (int k = 0; k < 32; ++k) s += __ldcg(A + i + 32 * k) * __ldcg(B + j + 32 * k);
            S[(ar + i) + m * (br + j)] -= s;
        }
        __syncthreads();
        return;
    }
    Fac A = get_fac(c, t.a), B = get_fac(c, t.b);
    const int ra = A.ncols, rb = B.ncols;
    if (ra == 0 || rb == 0) return;
    const int64_t r_lo = max(R0, A.row0), r_hi = min(R0 + m, A.row0 + A.nrows);
    const int64_t c_lo = max(C0, B.row0), c_hi = min(C0 + m, B.row0 + B.nrows);
    if (r_lo >= r_hi || c_lo >= c_hi) return;
    const int64_t nr = r_hi - r_lo, nc = c_hi - c_lo;
    const double *Ap = A.p + (r_lo - A.row0);
    const double *Bp = B.p + (c_lo - B.row0);
    const double *T1 = Ap;
    int64_t ldt = A.ld;
    if (t.core >= 0) {
        const double *K = c.cores + (int64_t)t.core * c.kcap * c.kcap;
        for (int64_t e = threadIdx.x; e < nr * rb; e += NT) {
            int64_t i = e % nr;
            int b = (int)(e / nr);
            double s = 0.0;
            for (int a = 0; a < ra; ++a) s += __ldcg(Ap + i + A.ld * a) * __ldcg(K + a + (int64_t)c.kcap * b);
            T1scr[i + nr * b] = s;
        }
        __syncthreads();
        T1 = T1scr;
        ldt = nr;
    }
    for (int64_t e = threadIdx.x; e < nr * nc; e += NT) {
        int64_t i = e % nr, j = e / nr;
        double s = 0.0;
        for (int b = 0; b < rb; ++b) s += T1[i + ldt * b] * __ldcg(Bp + j + B.ld * b);
        S[(r_lo - R0 + i) + m * (c_lo - C0 + j)] -= s;
    }
    __syncthreads();
}

// Scratch needs (doubles) of the R finalisation / assembly for block size m.
__host__ __device__ inline int aca_kmax(int64_t m, int kcap)
{
    int64_t k = 2 * (int64_t)kcap + 32;
    return (int)(k < m ? k : m);
}
#define HCOV_DENSE_MAX 512
#define HCOV_FACTOR_BATCH 64
__host__ __device__ inline int64_t rfin_scratch(int64_t m, int kcap)
{
    if (m <= HCOV_DENSE_MAX) {
        int64_t K = aca_kmax(m, kcap);
        return m * m + 2 * m * K + 2 * K * K + 4 * K + m * (int64_t)kcap + 64;
    }
    int64_t K = kcap + HCOV_FACTOR_BATCH + 32;
    return 2 * m * K + 2 * K * K + 4 * K + m * 32 + m * (int64_t)kcap + 64;
}
__host__ __device__ inline int64_t assemble_scratch(int64_t m, int kcap)
{
    int64_t K = aca_kmax(m, kcap);
    return 2 * m * K + 2 * K * K + 4 * K + m / 8 + 64;
}
__host__ __device__ inline int64_t solve_scratch(int64_t m, int ctot, int kcap)
{
    return m * (int64_t)ctot + (int64_t)kcap * ctot + 64;
}

__device__ __forceinline__ CompressWs make_ws(double *base, int64_t m, int K)
{
    CompressWs w;
    w.X = base;
    w.Y = w.X + m * K;
    w.M = w.Y + m * K;
    w.J = w.M + (int64_t)K * K;
    w.tx = w.J + (int64_t)K * K;
    w.ty = w.tx + K;
    w.sig = w.ty + K;
    w.ord = (int *)(w.sig + K);
    return w;
}

__device__ void record_rank(const Ctx &c, int r, int rk, int cb, int of)
{
    if (threadIdx.x == 0) {
        c.rank[r] = rk;
        if (cb) atomicAdd(c.flags + 0, 1);
        if (of) atomicAdd(c.flags + 1, 1);
        atomicMax(c.flags + 2, rk);
    }
    __syncthreads();
}

__device__ void task_rfin(const Ctx &c, const DTask &tk, double *scr, double *red, double *redv, int64_t *redi)
{
    const DNode x = c.nodes[tk.a];
    const int r = x.idx;
    const DRBlk blk = c.rblk[r];
    const int64_t m = blk.m;
    const int64_t R0 = blk.row0, C0 = blk.col0;
    double *U = r_U(c, r), *V = r_V(c, r);
    const int r0 = __ldcg(c.rank + r);
    int cb = 0, of = 0;
    if (m <= HCOV_DENSE_MAX) {
        const int K = aca_kmax(m, c.kcap);
        double *S = scr;
        CompressWs w = make_ws(S + m * m, m, K);
        double *T1 = (double *)(w.ord + K + 2);
        // S = U V^T
        for (int64_t e = threadIdx.x; e < m * m; e += NT) {
            int64_t i = e % m, j = e / m;
            double s = 0.0;
            for (int l = 0; l < r0; ++l) s += __ldcg(U + i + m * l) * __ldcg(V + j + m * l);
            S[e] = s;
        }
        __syncthreads();
        for (int y = tk.a; y >= 0; y = c.nodes[y].parent) {
            const DNode ny = c.nodes[y];
            for (int k = 0; k < ny.term_cnt; ++k) dense_sub_term(c, c.terms[ny.term_off + k], S, m, R0, C0, T1);
        }
        const double rel = 0.1 * c.eps / (double)m;
        int k = aca_full(S, m, w.X, w.Y, K, rel, redv, redi);
        int rk = compress(w, m, k, c.eps, c.kmax, c.kcap, U, V, m, &cb, &of, red);
        record_rank(c, r, rk, cb, of);
        return;
    }
    // factor path: X = [U, -A_1 K_1, ...], Y = [V, B_1, ...]; recompress every batch
    const int K = c.kcap + HCOV_FACTOR_BATCH + 32;
    CompressWs w = make_ws(scr, m, K);
    double *T1 = (double *)(w.ord + K + 2);
    double *Ut = T1 + m * 32;   // m x kcap temporary output of intermediate compressions
    int cur = r0;
    for (int64_t e = threadIdx.x; e < m * (int64_t)r0; e += NT) { w.X[e] = __ldcg(U + e); w.Y[e] = __ldcg(V + e); }
    __syncthreads();
    for (int y = tk.a; y >= 0; y = c.nodes[y].parent) {
        const DNode ny = c.nodes[y];
        for (int kk = 0; kk < ny.term_cnt; ++kk) {
            const DTerm t = c.terms[ny.term_off + kk];
            int width;
            if (t.kind == TM_TT) width = 32;
            else width = __ldcg(c.rank + c.fac_rank_src[t.b]);
            if (width == 0) continue;
            if (cur + width > K) {
                int rk = compress(w, m, cur, c.eps, c.kmax, c.kcap, Ut, U, m, &cb, &of, red);
                // U holds V-part temporarily; copy back into X, Y
                for (int64_t e = threadIdx.x; e < m * (int64_t)rk; e += NT) { w.X[e] = Ut[e]; w.Y[e] = U[e]; }
                __syncthreads();
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
            }
            __syncthreads();
            cur += width;
        }
    }
    int rk = compress(w, m, cur, c.eps, c.kmax, c.kcap, U, V, m, &cb, &of, red);
    record_rank(c, r, rk, cb, of);
}

// ---------------------------------------------------------------------------------------------
// Forward H-solve program on Y (m_sig x ncol, ld m_sig), rows relative to sig0.  Executes the
// post-order ops of the cluster `sig` whose rows lie inside [sig0, sig0 + msig).
__device__ void run_solve_program(const Ctx &c, int64_t sig, int64_t sig0, int64_t msig, double *Y, int ncol,
                                  double *tscr, double *smL)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = c.op_beg[sig], e = c.op_end[sig];
    for (int o = b; o < e; ++o) {
        const DOp op = c.ops[o];
        if (op.row0 >= sig0 + msig) continue;
        const int64_t ro = op.row0 - sig0, co = op.col0 - sig0;
        if (op.kind == OP_TRSM) {
            tile_load(smL, c.tiles + (int64_t)op.id * HCOV_TILE);
            __syncthreads();
            for (int col = threadIdx.x; col < ncol; col += NT) {
                double *y = Y + ro + msig * col;
                double v[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = y[k];
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    double s = v[k];
                    for (int j = 0; j < k; ++j) s -= smL[k + 32 * j] * v[j];
                    v[k] = s / smL[k + 32 * k];
                }
#pragma unroll
                for (int k = 0; k < 32; ++k) y[k] = v[k];
            }
            __syncthreads();
        } else if (op.kind == OP_UPD_T) {
            tile_load(smL, c.tiles + (int64_t)op.id * HCOV_TILE);
            __syncthreads();
            for (int64_t q = threadIdx.x; q < 32 * (int64_t)ncol; q += NT) {
                int i = (int)(q & 31);
                int64_t col = q >> 5;
                const double *x = Y + co + msig * col;
                double s = 0.0;
#pragma unroll 8
                for (int k = 0; k < 32; ++k) s += smL[i + 32 * k] * x[k];
                Y[ro + i + msig * col] -= s;
            }
            __syncthreads();
        } else {
            const int r = op.id;
            const int rk = __ldcg(c.rank + r);
            if (rk == 0) continue;
            const int64_t m = op.m;
            const double *U = r_U(c, r), *V = r_V(c, r);
            // t = V^T Y[co..co+m)   (rk x ncol)
            for (int pq = warp; pq < rk * ncol; pq += NWARP) {
                int l = pq % rk, col = pq / rk;
                const double *vl = V + m * l;
                const double *x = Y + co + msig * col;
                double s = 0.0;
                for (int64_t i = lane; i < m; i += 32) s += __ldcg(vl + i) * x[i];
                s = warp_sum(s);
                if (lane == 0) tscr[l + rk * col] = s;
            }
            __syncthreads();
            for (int64_t q = threadIdx.x; q < m * (int64_t)ncol; q += NT) {
                int64_t i = q % m, col = q / m;
                double s = 0.0;
                for (int l = 0; l < rk; ++l) s += __ldcg(U + i + m * l) * tscr[l + rk * col];
                Y[ro + i + msig * col] -= s;
            }
            __syncthreads();
        }
    }
}

__device__ void task_solve(const Ctx &c, const DTask &tk, double *scr, double *smL)
{
    const int64_t sig = tk.a;
    int level = 0;
    while ((((int64_t)2 << level) - 1) <= sig) ++level;
    const int64_t cidx = sig - (((int64_t)1 << level) - 1);
    const int64_t msig = cl_size(c, level), sig0 = cidx * msig;
    const int b = c.col_r_off[sig], e = c.col_r_off[sig + 1];
    int ctot = 0;
    for (int k = b; k < e; ++k) ctot += __ldcg(c.rank + c.col_r[k]);
    double *Y = scr;
    double *tscr = Y + msig * (int64_t)ctot;
    int off = 0;
    for (int k = b; k < e; ++k) {
        const int r = c.col_r[k];
        const int rk = __ldcg(c.rank + r);
        const double *V = r_V(c, r);
        for (int64_t q = threadIdx.x; q < msig * (int64_t)rk; q += NT) Y[msig * off + q] = __ldcg(V + q);
        off += rk;
    }
    __syncthreads();
    if (ctot > 0) run_solve_program(c, sig, sig0, msig, Y, ctot, tscr, smL);
    off = 0;
    for (int k = b; k < e; ++k) {
        const int r = c.col_r[k];
        const int rk = __ldcg(c.rank + r);
        double *V = r_V(c, r);
        for (int64_t q = threadIdx.x; q < msig * (int64_t)rk; q += NT) V[q] = Y[msig * off + q];
        off += rk;
    }
    __syncthreads();
}

// K = V_a^T V_b
__device__ void task_prr(const Ctx &c, const DTask &tk)
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
        if (lane == 0) K[a + (int64_t)c.kcap * b] = s;
    }
}

// W = H * [V_p]  for an H entry and all R partners of its column.
__device__ void task_phw(const Ctx &c, const DTask &tk, double *smT, double *tsm)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const DPhw q = c.phw[tk.b];
    const DNode h = c.nodes[q.hnode];
    const int64_t m = q.m;
    const int64_t rho0 = (int64_t)h.i * m, sig0 = (int64_t)h.j * m;
    double *W = c.W + q.w_off * (int64_t)c.kcap;
    const int ldw = (int)m;
    const int np = q.part_cnt;
    // zero W
    for (int64_t e = threadIdx.x; e < m * (int64_t)c.kcap * np; e += NT) W[e] = 0.0;
    __syncthreads();
    for (int li = 0; li < h.leaf_cnt; ++li) {
        const DNode x = c.nodes[c.hleaf[h.leaf_off + li]];
        const int64_t mx = cl_size(c, x.level);
        const int64_t xr = (int64_t)x.i * mx - rho0, xc = (int64_t)x.j * mx - sig0;
        if (x.type == ND_T) {
            tile_load(smT, c.tiles + (int64_t)x.idx * HCOV_TILE);
            __syncthreads();
            for (int p = 0; p < np; ++p) {
                const int r = c.phw_part[q.part_off + p];
                const int rk = __ldcg(c.rank + r);
                const double *Vp = r_V(c, r);
                double *Wp = W + (int64_t)ldw * c.kcap * p;
                for (int64_t e = threadIdx.x; e < 32 * (int64_t)rk; e += NT) {
                    int i = (int)(e & 31);
                    int col = (int)(e >> 5);
                    double s = 0.0;
#pragma unroll 8
                    for (int k = 0; k < 32; ++k) s += smT[i + 32 * k] * __ldcg(Vp + xc + k + m * col);
                    Wp[xr + i + (int64_t)ldw * col] += s;
                }
            }
            __syncthreads();
        } else {
            const int rx = __ldcg(c.rank + x.idx);
            if (rx == 0) continue;
            const double *Ux = r_U(c, x.idx), *Vx = r_V(c, x.idx);
            for (int p = 0; p < np; ++p) {
                const int r = c.phw_part[q.part_off + p];
                const int rk = __ldcg(c.rank + r);
                if (rk == 0) continue;
                const double *Vp = r_V(c, r);
                double *Wp = W + (int64_t)ldw * c.kcap * p;
                for (int pq = warp; pq < rx * rk; pq += NWARP) {
                    int l = pq % rx, col = pq / rx;
                    double s = 0.0;
                    for (int64_t i = lane; i < mx; i += 32) s += __ldcg(Vx + i + mx * l) * __ldcg(Vp + xc + i + m * col);
                    s = warp_sum(s);
                    if (lane == 0) tsm[l + rx * col] = s;
                }
                __syncthreads();
                for (int64_t e = threadIdx.x; e < mx * (int64_t)rk; e += NT) {
                    int64_t i = e % mx;
                    int col = (int)(e / mx);
                    double s = 0.0;
                    for (int l = 0; l < rx; ++l) s += __ldcg(Ux + i + mx * l) * tsm[l + rx * col];
                    Wp[xr + i + (int64_t)ldw * col] += s;
                }
                __syncthreads();
            }
        }
    }
}
