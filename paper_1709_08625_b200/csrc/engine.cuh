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

// qctl layout (engine control words, hcov.cu)
#define QC_HEAD1 0      // gang queue: next ticket
#define QC_TAIL1 1      // gang queue: published tickets
#define QC_ABORT 2      // watchdog / pool overflow: every CTA leaves its loop
#define QC_DONE0 3      // completed queue-0 tasks
#define QC_BHEAD 4      // HCOV_BANDS band heads
#define QC_BTAIL (4 + HCOV_BANDS)
#define QC_N (4 + 2 * HCOV_BANDS)

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
    const double *zs;          // 3-D variant (tree option dim = 3); nullptr for 2-D locations
    const int64_t *perm_i2e;
    int32_t depth, n_r, root_solve, ntasks;
    int64_t n_pad, n_leaves, n_real, n_tiles;
    // ---- numeric (per H-matrix) ----
    double *tiles;
    double *U, *V;
    int32_t *rank;
    double *cores;
    double *W;                 // pool of W = H V blocks, allocated at run time with actual ranks (woff)
    double *P;                 // pool of product slots (PROJ / PHWP results), allocated at run time (poff)
    int64_t *woff, *poff;      // per PHW / per slot: offset in its pool (-1 = not yet allocated)
    unsigned long long *mem;   // [0] W bump, [1] P bump, [2] pool overflows
    int64_t wcap, pcap;        // pool capacities (doubles)
    double *vbuf;              // root right-hand side / solution (internal order)
    double *tbuf;              // back-solve projections t_b = U_b^T u (n_r x kcap)
    double *logdet_part, *minpiv_part, *quad_part;
    int32_t *fail_leaf;        // min over failing leaves (init INT32_MAX)
    int32_t *flags;            // [0] cap binds, [1] rank overflow, [2] max rank, [3] accuracy losses
                               // (a recompression cut below its tolerance for lack of work capacity,
                               // kmax == 0), [4] the same cuts under a rank cap kmax > 0 (the kept
                               // rank is >= kmax, so the cut is covered by the cap; not a loss)
    int32_t kcap, kmax;
    double eps;
    double interm_rel;         // intermediate (chunk) recompression tolerance, relative to eps (R22)
    MaternParams mp;
    // ---- engine ----
    int32_t *indeg;            // working copy of the in-degrees
    int32_t *queue[2];         // [0]: HCOV_BANDS priority rings (band_off x ninst), [1]: unused
    const int32_t *band_off;   // HCOV_BANDS + 1
    uint32_t *qctl;            // see QC_* in hcov.cu
    int32_t nq[2];
    int32_t ninst;             // instances (H-matrices of one tree) run by this engine launch
    int32_t kcore;             // leading dimension / stride of the PRR cores (kcap; kmax in the
                               // SPD-preserving mode, where products see truncated factors only)
    int32_t factor_trunc;      // 1: SPD-preserving mode (tree option; R27): C~ and the pending
                               // updates kept near-losslessly, the (eps, kmax) truncation applied to the
                               // factor block L_21 = A_21 L_11^{-T} after its solve (a TRUNC task)
    int32_t *gbar;             // per-task gang barrier counters
    int32_t *gslot;            // per-task: CTA index of the gang's member 0 (-1 until it joined)
    int64_t gshared_off;       // offset (doubles) of the shared gang workspace in a gang CTA's scratch
    double *scr;               // per-CTA scratch (normal CTAs), scr_stride doubles each
    int64_t scr_stride;
    double *bscr;              // big-member scratch: n_bgrp groups of HCOV_GANG member slots
    int64_t bscr_stride;       // doubles per member slot
    int32_t *bgrp_busy;        // per group: 1 while a gang holds it
    int32_t *bgrp_cta;         // per CTA (member 0 of a gang): the group its gang holds
    int32_t big_mq;            // gang members with more rows than this use a big-member slot
    int32_t dense_max;         // low-rank blocks up to this size use the dense-mode RAPP (PlanOpts.big_m)
    int32_t dense_dmma;        // dense-mode S += XA YB^T on the FP64 tensor cores (HCOV_DENSE_DMMA, default 1)
    int32_t term_min;          // a pending term A K B^T enters a panel with min(rank A, rank B) columns:
                               // [-A K, B] (rank B columns) or [-A, B K^T] (rank A), HCOV_TERM_MIN, default 1
    int32_t n_bgrp;
    double *flop;              // FC_N accumulators
    int64_t smem_dbl;          // dynamic shared memory of the engine (doubles)
    unsigned long long timeout_ns;
};

// ---------------------------------------------------------------------------------------------
struct Fac {
    const double *p;
    int64_t ld, row0;
    int32_t nrows, ncols;
};
__device__ __forceinline__ int partner_prefix(const Ctx &c, const DPhw &q, int p)
{
    int s = 0;
    for (int k = 0; k < p; ++k) s += __ldcg(c.rank + c.col_r[q.part_off + k]);
    return s;
}
__device__ __forceinline__ double *w_base(const Ctx &c, int qid) { return c.W + __ldcg(c.woff + qid); }
__device__ __forceinline__ const double *slot_get(const Ctx &c, int s) { return c.P + __ldcg(c.poff + s); }

// Bump allocation from a pool (thread 0); an overflow is counted (reported as out of memory) and
// the allocation aliases offset 0.
__device__ __forceinline__ int64_t pool_bump(const Ctx &c, int which, int64_t size, int64_t cap)
{
    int64_t off = (int64_t)atomicAdd(c.mem + which, (unsigned long long)size);
    if (off + size > cap) {
        // overflow: counted, reported as out of memory; the engine is stopped at once (the
        // aliased allocation below is never used for a result)
        atomicAdd(c.mem + 2, 1ull);
        atomicExch(c.qctl + QC_ABORT, 1u);
        off = 0;
    }
    return off;
}
// Product slot s of `size` doubles (single producer task; CTA-collective).  A slot keeps its offset
// until the next assembly resets poff[]: later solve-mode runs on the same factor (hcov_solve, PCG,
// the diagnostics) reuse it (the slot's size depends only on the factor's ranks) instead of
// growing the pool.
__device__ double *slot_alloc(const Ctx &c, int s, int64_t size)
{
    __shared__ int64_t s_off;
    if (threadIdx.x == 0) {
        int64_t off = (int64_t)__ldcg(c.poff + s);
        if (off < 0) {
            off = pool_bump(c, 1, size, c.pcap);
            atomicExch((unsigned long long *)(c.poff + s), (unsigned long long)off);
        }
        s_off = off;
    }
    __syncthreads();
    return c.P + s_off;
}
// W block of PHW q (m x sum of partner ranks): the first of its row tasks allocates, the others
// wait for the published offset (CTA-collective).
__device__ double *w_acquire(const Ctx &c, int qid, int64_t size)
{
    __shared__ int64_t s_off;
    if (threadIdx.x == 0) {
        unsigned long long *slot = (unsigned long long *)(c.woff + qid);
        unsigned long long cur = atomicCAS(slot, ~0ull, ~1ull);
        int64_t off;
        if (cur == ~0ull) {
            off = pool_bump(c, 0, size, c.wcap);
            __threadfence();
            atomicExch(slot, (unsigned long long)off);
        } else {
            while ((int64_t)(cur = *(volatile unsigned long long *)slot) < 0) __nanosleep(64);
            off = (int64_t)cur;
        }
        s_off = off;
    }
    __syncthreads();
    return c.W + s_off;
}

__device__ __forceinline__ Fac get_fac(const Ctx &c, int f)
{
    Fac F;
    F.nrows = c.fac_nrows[f];
    F.ld = F.nrows;
    F.row0 = c.fac_row0[f];
    F.ncols = __ldcg(c.rank + c.fac_rank_src[f]);
    if (c.fac_pool[f] == 0) {
        F.p = c.U + c.fac_off[f] * (int64_t)c.kcap;
    } else {   // W slice (phw id, partner index)
        const int64_t code = c.fac_off[f];
        const int qid = (int)(code >> 20), p = (int)(code & 0xFFFFF);
        const DPhw q = c.phw[qid];
        F.p = w_base(c, qid) + (int64_t)q.m * partner_prefix(c, q, p);
    }
    return F;
}
__device__ __forceinline__ int64_t cl_size(const Ctx &c, int level) { return (int64_t)HCOV_LEAF << (c.depth - level); }
__device__ __forceinline__ double *r_U(const Ctx &c, int r) { return c.U + c.rblk[r].uv_off * (int64_t)c.kcap; }
__device__ __forceinline__ double *r_V(const Ctx &c, int r) { return c.V + c.rblk[r].uv_off * (int64_t)c.kcap; }

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
        const double *K = c.cores + (int64_t)t.core * c.kcore * c.kcore;
        for (int e = threadIdx.x; e < ra * rb; e += NT) {
            int a = e % ra, b = e / ra;
            sm.K[e] = __ldcg(K + a + (int64_t)c.kcore * b);
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
    tile_gemm_nt_sub_k(sm.S, T1, sm.B, rb);   // DMMA
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
            __stcg(T + e, pts_cov(c.mp, Pts{c.xs, c.ys, c.zs}, a, b));
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
#ifndef HCOV_KBUF_MULT
#define HCOV_KBUF_MULT 3   // panel width of a chunked accumulation: HCOV_KBUF_MULT kcap + 32 columns
#endif
__host__ __device__ inline int kbuf_of(int kcap) { return HCOV_KBUF_MULT * kcap + 32; }
// In-CTA TSQR of a member's rows (> 256): chunks of <= 256 rows, per side nc x K taus and nc
// node slots of (2 K x K panel + K taus).
__host__ __device__ inline int ts_nchunks(int64_t mq) { return (int)((mq + 255) / 256); }
__host__ __device__ inline int64_t ts_slot(int K) { return 2 * (int64_t)K * K + K; }
__host__ __device__ inline int64_t ts_region_doubles(int64_t mq, int K)
{
    if (mq <= 256) return 0;
    return 2 * (int64_t)ts_nchunks(mq) * (K + ts_slot(K));
}
__host__ __device__ inline int64_t task_scratch_base(int64_t m, int kcap, int npanels)
{
    int64_t K = kbuf_of(kcap);
    int64_t panels = npanels * m * K;
    if (m <= HCOV_DENSE_MAX) panels = m * m + npanels * m * K;
    return panels + 8 * K * K + 10 * K + m / 8 + 64;
}
__host__ __device__ inline int64_t task_scratch(int64_t m, int kcap, int npanels = 6)
{
    const int64_t b = task_scratch_base(m, kcap, npanels);
    return npanels == 4 ? b + ts_region_doubles(m, kbuf_of(kcap)) : b;
}


__device__ __forceinline__ CompressWs make_ws(double *base, int64_t m, int K, double **X2, double **Y2, int npanels = 6)
{
    CompressWs w;
    w.X = base;
    w.Y = w.X + m * K;
    *X2 = w.Y + m * K;
    *Y2 = *X2 + m * K;
    w.T1 = (npanels >= 6) ? *Y2 + m * K : nullptr;
    w.T2 = (npanels >= 6) ? w.T1 + m * K : nullptr;
    w.M = *Y2 + m * K * (npanels - 3);
    w.G = w.M + (int64_t)K * K;
    w.J = w.G + (int64_t)K * K;
    w.RX = w.J + (int64_t)K * K;
    w.RY = w.RX + (int64_t)K * K;
    w.UC = w.RY + (int64_t)K * K;
    w.VC = w.UC + (int64_t)K * K;
    w.Ri = w.VC + (int64_t)K * K;
    w.tx = w.Ri + (int64_t)K * K;
    w.ty = w.tx + K;
    w.tm = w.ty + K;
    w.sig = w.tm + K;
    w.cn = w.sig + K;
    w.dX = w.cn + K;
    w.dY = w.dX + K;
    w.ord = (int *)(w.dY + K);
    w.piv = (int *)(w.dY + 2 * K);
    w.tail = w.dY + 3 * K;
    w.tsr = nullptr;
    w.K = K;
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

// Rank of a near-lossless (not yet final) representation: stored, not counted in the rank
// statistics; a cut for lack of capacity is counted like an intermediate cut.
__device__ void record_interm(const Ctx &c, int r, int rk, int of)
{
    if (threadIdx.x == 0) {
        __stcg(c.rank + r, rk);
        if (of) atomicAdd(c.flags + (c.kmax > 0 ? 4 : 3), 1);
    }
    __syncthreads();
}

// Index of the flag counting a recompression cut made for lack of work capacity: an accuracy
// loss (flags[3]) without a rank cap, else a cut covered by the cap (flags[4]; every work capacity
// is >= kmax).
__device__ __forceinline__ int cut_flag(const Ctx &c) { return c.kmax > 0 ? 4 : 3; }

__device__ __forceinline__ double final_tol(double eps, int R) { return eps / (10.0 * sqrt((double)(R > 0 ? R : 1))); }
__device__ __forceinline__ double interm_tol(const Ctx &c) { return fmax(c.eps * c.interm_rel, 1e-15); }

__device__ __forceinline__ double compress_flops(int64_t m, int R, int r)
{
    // 2 Householder QRs, the core product, one-sided Jacobi (~6 sweeps), two Q applications
    return 2.0 * (4.0 * m * R * R - 4.0 * R * R * R / 3.0) + 2.0 * R * R * R / 3.0 + 6.0 * 9.0 * R * R * R +
           2.0 * 4.0 * m * R * r;
}


// ---------------------------------------------------------------------------------------------
// Gang tasks: HCOV_GANG CTAs cooperate on one big block.  The block's rows (and, for ACA, its
// columns) are partitioned: member g owns rows [q0, q0 + mq) and keeps its panel rows in its own
// CTA scratch; the small shared workspace (stacked R factors, cores, partials) lives in member
// 0's scratch.  Members synchronise through a per-task counter.  Gangs are formed from
// consecutive tickets of queue 1.
struct Gang {
    int g, G;
    int32_t *bar;
    const uint32_t *abort;     // the engine's watchdog flag: a partly formed gang never spins forever
    int nb;
    int64_t mq, q0;
    double *shared;
    int split;                 // side-split gang: members [0, G/2) hold X rows, [G/2, G) Y rows
    int side, gs, Gs;          // side (0 X, 1 Y; -1 both), index within the side, members per side
};
// Rows of a gang member: m / Gs each (Gs = G, or G/2 per side when side-split), the last member
// of a side also takes the remainder.
__device__ __forceinline__ void gang_rows(Gang &gg, int64_t m)
{
    gg.Gs = gg.split ? gg.G / 2 : gg.G;
    gg.side = gg.split ? gg.g / gg.Gs : -1;
    gg.gs = gg.split ? gg.g % gg.Gs : gg.g;
    const int64_t base = m / gg.Gs;
    gg.q0 = (int64_t)gg.gs * base;
    gg.mq = (gg.gs == gg.Gs - 1) ? m - (int64_t)(gg.Gs - 1) * base : base;
}
__device__ __forceinline__ void gang_sync(Gang &gg)
{
    PH_BEGIN(tw);
    __syncthreads();
    ++gg.nb;
    if (threadIdx.x == 0) {
        // the Gang fields in registers for the spin (a reference into the engine's local frame)
        volatile int32_t *bar = gg.bar;
        volatile const uint32_t *abort = gg.abort;
        const int target = gg.nb * gg.G;
        __threadfence();
        atomicAdd(gg.bar, 1);
        unsigned spin = 0;
        while (*bar < target) {
            if ((++spin & 63u) == 0 && *abort) break;
            __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
    PH_END(13, tw);
}

struct GangWs {
    // per side (X, Y): G blocks of R x R (ld R: the current R factors of the TSQR tree), G node
    // slots of (2K x K panel + K taus) (tree node (g, s) in slot g + s), G blocks of R x r (ld R:
    // the cores pushed down the tree)
    double *BX, *BY, *NX, *NY, *CX, *CY;
    double *pv;            // 2 x G partial values
    int64_t *pi;           // 2 x G partial indices
    double *ps;            // 2 x G x 2 partial sums
    double *urow, *vrow;   // K each: published pivot row of U / pivot column of V (ACA)
    int32_t *ires;         // [0] r, [1] cb, [2] of
    int64_t nslot;         // doubles per node slot
};
__host__ __device__ inline int64_t gang_shared_doubles(int K, int G)
{
    return 2 * (int64_t)G * (2 * (int64_t)K * K + (2 * (int64_t)K * K + K)) + 2 * (int64_t)K + 8 * (int64_t)G + 64;
}
__device__ __forceinline__ GangWs make_gws(double *base, int K, int G)
{
    GangWs gw;
    const int64_t GK2 = (int64_t)G * K * K;
    gw.nslot = 2 * (int64_t)K * K + K;
    gw.BX = base;
    gw.BY = gw.BX + GK2;
    gw.CX = gw.BY + GK2;
    gw.CY = gw.CX + GK2;
    gw.NX = gw.CY + GK2;
    gw.NY = gw.NX + G * gw.nslot;
    gw.urow = gw.NY + G * gw.nslot;
    gw.vrow = gw.urow + K;
    gw.pv = gw.vrow + K;
    gw.pi = (int64_t *)(gw.pv + 2 * G);
    gw.ps = (double *)(gw.pi + 2 * G);
    gw.ires = (int32_t *)(gw.ps + 4 * G);
    return gw;
}

// Local Householder QR of a member's panel (mq x R, ld mq): in shared memory when mq <= 256,
// else an in-CTA TSQR over nc chunks of <= 256 rows (chunk QRs in shared memory, then a binary
// tree of 2R x R node QRs; region: nc x K taus, then nc node slots (node (b, s) in slot b + s)).
// The R factor of the whole panel ends in the upper triangle of rows 0..R-1.
__device__ __forceinline__ int64_t ts_c0(int64_t mq, int nc, int c) { return (mq * c) / nc; }

// 0: global Householder, 1: one shared-memory panel, 2: in-CTA TSQR over chunks
__device__ __forceinline__ int local_mode(int64_t mq, int R, const double *reg, int64_t smem_dbl)
{
    if (mq <= 256) return (R <= mq && mq * R + R <= smem_dbl) ? 1 : 0;
    const int nc = ts_nchunks(mq);
    if (reg && 256 * (int64_t)R + R <= smem_dbl && 2 * (int64_t)R * R + R <= smem_dbl && mq / nc >= R) return 2;
    return 0;
}

__device__ void local_qr(double *P, int64_t mq, int R, double *tau, double *reg, int K, double *smem,
                         int64_t smem_dbl, double *red)
{
    const int mode = local_mode(mq, R, reg, smem_dbl);
    if (mode == 0) {
        qr_house(P, mq, mq, R, tau, red);
        return;
    }
    if (mode == 1) {
        double *ts = smem + mq * R;
        panel_to_sm(smem, P, mq, (int)mq, R);
        qr_sm(smem, (int)mq, (int)mq, R, ts);
        for (int e = threadIdx.x; e < R; e += NT) tau[e] = ts[e];
        panel_from_sm(P, mq, smem, (int)mq, R);
        return;
    }
    const int nc = ts_nchunks(mq);
    const int64_t nslot = ts_slot(K);
    double *taus = reg, *nodes = reg + (int64_t)nc * K;
    for (int cix = 0; cix < nc; ++cix) {
        const int64_t r0 = ts_c0(mq, nc, cix);
        const int rows = (int)(ts_c0(mq, nc, cix + 1) - r0);
        double *ts = smem + (int64_t)rows * R;
        panel_to_sm(smem, P + r0, mq, rows, R);
        qr_sm(smem, rows, rows, R, ts);
        for (int e = threadIdx.x; e < R; e += NT) taus[(int64_t)cix * K + e] = ts[e];
        panel_from_sm(P + r0, mq, smem, rows, R);
    }
    const int R2 = 2 * R;
    for (int s = 1; s < nc; s *= 2)
        for (int b = 0; b + s < nc; b += 2 * s) {
            double *Pb = P + ts_c0(mq, nc, b), *Pc = P + ts_c0(mq, nc, b + s);
            double *slot = nodes + (int64_t)(b + s) * nslot;
            double *ts = smem + (int64_t)R2 * R;
            for (int e = threadIdx.x; e < R2 * R; e += NT) {
                const int i = e % R2, k = e / R2;
                const int ii = i < R ? i : i - R;
                smem[e] = (k >= ii) ? (i < R ? Pb : Pc)[ii + mq * k] : 0.0;
            }
            __syncthreads();
            qr_sm(smem, R2, R2, R, ts);
            for (int e = threadIdx.x; e < R2 * R; e += NT) slot[e] = smem[e];
            for (int e = threadIdx.x; e < R; e += NT) slot[2 * (int64_t)R * R + e] = ts[e];
            for (int e = threadIdx.x; e < R * R; e += NT) {
                const int i = e % R, k = e / R;
                if (k >= i) Pb[i + mq * k] = smem[i + (int64_t)R2 * k];
            }
            __syncthreads();
        }
}

// B <- Q B for the local QR above (B: mq x r, ld ldb; only rows 0..R-1 nonzero on entry).
__device__ void local_apply(const double *P, int64_t mq, int R, const double *tau, const double *reg, int K,
                            double *B, int64_t ldb, int r, double *tmp, double *smem, int64_t smem_dbl)
{
    const int mode = local_mode(mq, R, reg, smem_dbl);
    if (mode == 0) {
        qr_apply_q(P, mq, mq, R, tau, B, ldb, r);
        return;
    }
    if (mode == 1) {
        double *ts = smem + mq * R;
        for (int e = threadIdx.x; e < R; e += NT) ts[e] = tau[e];
        panel_to_sm(smem, P, mq, (int)mq, R);
        apply_q_sm(smem, (int)mq, (int)mq, R, ts, B, ldb, r);
        return;
    }
    const int nc = ts_nchunks(mq);
    const int64_t nslot = ts_slot(K);
    const double *taus = reg, *nodes = reg + (int64_t)nc * K;
    const int R2 = 2 * R;
    int top = 1;
    while (2 * top < nc) top *= 2;
    for (int s = top; s >= 1; s /= 2)
        for (int b = 0; b + s < nc; b += 2 * s) {
            double *Bb = B + ts_c0(mq, nc, b), *Bc = B + ts_c0(mq, nc, b + s);
            const double *slot = nodes + (int64_t)(b + s) * nslot;
            double *ts = smem + (int64_t)R2 * R;
            for (int e = threadIdx.x; e < R2 * r; e += NT) {
                const int i = e % R2, cc = e / R2;
                tmp[e] = (i < R) ? Bb[i + ldb * cc] : 0.0;
            }
            for (int e = threadIdx.x; e < R2 * R; e += NT) smem[e] = slot[e];
            for (int e = threadIdx.x; e < R; e += NT) ts[e] = slot[2 * (int64_t)R * R + e];
            __syncthreads();
            apply_q_sm(smem, R2, R2, R, ts, tmp, R2, r);
            for (int e = threadIdx.x; e < R2 * r; e += NT) {
                const int i = e % R2, cc = e / R2;
                if (i < R) Bb[i + ldb * cc] = tmp[e];
                else Bc[(i - R) + ldb * cc] = tmp[e];
            }
            __syncthreads();
        }
    for (int cix = 0; cix < nc; ++cix) {
        const int64_t r0 = ts_c0(mq, nc, cix);
        const int rows = (int)(ts_c0(mq, nc, cix + 1) - r0);
        double *ts = smem + (int64_t)rows * R;
        for (int e = threadIdx.x; e < R; e += NT) ts[e] = taus[(int64_t)cix * K + e];
        panel_to_sm(smem, P + r0, mq, rows, R);
        apply_q_sm(smem, rows, rows, R, ts, B + r0, ldb, r);
    }
}

// TSQR tree node (b, s) of one side: [B_b; B_{b+s}] = Q_node [R'; 0]; panel + taus -> slot b + s,
// R' -> B_b.  2R x R in shared memory (2R <= 1024 rows fits for R <= 96 with the engine's 220 KB).
__device__ void tsqr_node_up(double *Bk, double *Nd, int64_t nslot, int b, int s, int R, double *smem,
                             int64_t smem_dbl, double *red)
{
    const int R2 = 2 * R;
    const int64_t RR = (int64_t)R * R;
    double *slot = Nd + (int64_t)(b + s) * nslot;
    const bool sm = (int64_t)R2 * R + R <= smem_dbl;
    double *P = sm ? smem : slot;
    double *ts = sm ? smem + (int64_t)R2 * R : slot + 2 * RR;
    for (int e = threadIdx.x; e < R2 * R; e += NT) {
        const int i = e % R2, k = e / R2;
        const double *src = (i < R) ? Bk + (int64_t)b * RR + i + (int64_t)R * k
                                    : Bk + (int64_t)(b + s) * RR + (i - R) + (int64_t)R * k;
        P[e] = __ldcg(src);
    }
    __syncthreads();
    if (sm) qr_sm(P, R2, R2, R, ts);
    else qr_house(P, R2, R2, R, ts, red);
    for (int e = threadIdx.x; e < RR; e += NT) {
        const int i = e % R, k = e / R;
        __stcg(Bk + (int64_t)b * RR + e, (k >= i) ? P[i + (int64_t)R2 * k] : 0.0);
    }
    if (sm) {
        for (int e = threadIdx.x; e < R2 * R; e += NT) __stcg(slot + e, P[e]);
        for (int e = threadIdx.x; e < R; e += NT) __stcg(slot + 2 * RR + e, ts[e]);
    }
    __syncthreads();
}

// Push the core down node (b, s): [C_b; 0] (2R x r) <- Q_node [C_b; 0]; top half -> C_b, bottom
// half -> C_{b+s}.  tmp: 2R x r private scratch.
__device__ void tsqr_node_down(double *Ck, const double *Nd, int64_t nslot, int b, int s, int R, int r, double *tmp,
                               double *smem, int64_t smem_dbl)
{
    const int R2 = 2 * R;
    const int64_t RR = (int64_t)R * R, Rr = (int64_t)R * r;
    const double *slot = Nd + (int64_t)(b + s) * nslot;
    for (int e = threadIdx.x; e < R2 * r; e += NT) {
        const int i = e % R2, c = e / R2;
        tmp[e] = (i < R) ? __ldcg(Ck + (int64_t)b * Rr + i + (int64_t)R * c) : 0.0;
    }
    const bool sm = (int64_t)R2 * R + R <= smem_dbl;
    if (sm) {
        double *ts = smem + (int64_t)R2 * R;
        for (int e = threadIdx.x; e < R2 * R; e += NT) smem[e] = __ldcg(slot + e);
        for (int e = threadIdx.x; e < R; e += NT) ts[e] = __ldcg(slot + 2 * RR + e);
        __syncthreads();
        apply_q_sm(smem, R2, R2, R, ts, tmp, R2, r);
    } else {
        __syncthreads();
        qr_apply_q(slot, R2, R2, R, slot + 2 * RR, tmp, R2, r);
    }
    for (int e = threadIdx.x; e < R2 * r; e += NT) {
        const int i = e % R2, c = e / R2;
        double *dst = (i < R) ? Ck + (int64_t)b * Rr + i + (int64_t)R * c
                              : Ck + (int64_t)(b + s) * Rr + (i - R) + (int64_t)R * c;
        __stcg(dst, tmp[e]);
    }
    __syncthreads();
}

// Gang truncation of X Y^T (m x m, R columns; member rows in the local panels w.X, w.Y with
// ld mq >= R).  TSQR: every member factors its rows (local QR); the R factors are combined by a
// binary tree (node (b, s) merges blocks b and b + s; the X tree runs on member b, the Y tree on
// member b + s, so both proceed in parallel); member 0 truncates the core M = R_X R_Y^T
// (compress_core); the core factors are pushed down the trees, and every member applies its local
// Q to its block [C_g; 0] of the result U, V (global, ld ldo, rows q0..q0+mq).
__device__ __noinline__ int gang_compress(const CompressWs &w, const GangWs &gw, Gang &gg, int R, double eps, double tol_q,
                             bool svd, int kmax, int rlim, double *U, double *V, int64_t ldo, int *cb, int *of,
                             double *red, double *redv, int64_t *redi, double *smem, int64_t smem_dbl)
{
    if (R == 0) { *cb = 0; *of = 0; return 0; }
    const int G = gg.G, g = gg.g;
    const int64_t mq = gg.mq, q0 = gg.q0;
    const int64_t RR = (int64_t)R * R;
    // phase 1 (all members): local QR, R factor -> B_g
    PH_BEGIN(t1);
    const int K = w.K;
    local_qr(w.X, mq, R, w.tx, w.tsr, K, smem, smem_dbl, red);
    local_qr(w.Y, mq, R, w.ty, w.tsr ? w.tsr + ts_region_doubles(mq, K) / 2 : nullptr, K, smem, smem_dbl, red);
    for (int e = threadIdx.x; e < RR; e += NT) {
        const int i = e % R, k = e / R;
        __stcg(gw.BX + (int64_t)g * RR + e, (k >= i) ? w.X[i + mq * k] : 0.0);
        __stcg(gw.BY + (int64_t)g * RR + e, (k >= i) ? w.Y[i + mq * k] : 0.0);
    }
    PH_END(9, t1);
    gang_sync(gg);
    // phase 2: up the trees
    PH_BEGIN(t2);
    int top = 1;
    while (2 * top < G) top *= 2;
    for (int s = 1; s < G; s *= 2) {
        if (g % (2 * s) == 0 && g + s < G) tsqr_node_up(gw.BX, gw.NX, gw.nslot, g, s, R, smem, smem_dbl, red);
        if (g % (2 * s) == s) tsqr_node_up(gw.BY, gw.NY, gw.nslot, g - s, s, R, smem, smem_dbl, red);
        gang_sync(gg);
    }
    PH_END(10, t2);
    // phase 3: core truncation (member 0) -> C_0 (R x r each side)
    if (g == 0) {
        PH_BEGIN(t3);
        for (int e = threadIdx.x; e < RR; e += NT) {
            w.RX[e] = __ldcg(gw.BX + e);
            w.RY[e] = __ldcg(gw.BY + e);
        }
        __syncthreads();
        int c1 = 0, o1 = 0;
        const int rr = compress_core(core_ws_sm(w, smem, smem_dbl, R), w.RX, R, w.RY, R, R, eps, tol_q, svd, kmax,
                                     rlim, gw.CX, gw.CY, R, R, &c1, &o1, red, redv, redi);
        if (threadIdx.x == 0) { gw.ires[0] = rr; gw.ires[1] = c1; gw.ires[2] = o1; }
        PH_END(11, t3);
    }
    gang_sync(gg);
    const int r = __ldcg(gw.ires);
    // phase 4: down the trees
    PH_BEGIN(t4);
    if (r > 0) {
        for (int s = top; s >= 1; s /= 2) {
            if (g % (2 * s) == 0 && g + s < G)
                tsqr_node_down(gw.CX, gw.NX, gw.nslot, g, s, R, r, w.G, smem, smem_dbl);
            if (g % (2 * s) == s) tsqr_node_down(gw.CY, gw.NY, gw.nslot, g - s, s, R, r, w.G, smem, smem_dbl);
            gang_sync(gg);
        }
    }
    PH_END(10, t4);
    // phase 5 (all members): rows of U = Q_g [C_g; 0], V likewise
    PH_BEGIN(t5);
    const int64_t Rr = (int64_t)R * r;
    for (int64_t e = threadIdx.x; e < mq * r; e += NT) {
        const int64_t i = e % mq;
        const int cc = (int)(e / mq);
        U[q0 + i + ldo * cc] = (i < R) ? __ldcg(gw.CX + (int64_t)g * Rr + i + (int64_t)R * cc) : 0.0;
        V[q0 + i + ldo * cc] = (i < R) ? __ldcg(gw.CY + (int64_t)g * Rr + i + (int64_t)R * cc) : 0.0;
    }
    *cb = __ldcg(gw.ires + 1);
    *of = __ldcg(gw.ires + 2);
    __syncthreads();
    if (r > 0) {
        local_apply(w.X, mq, R, w.tx, w.tsr, K, U + q0, ldo, r, w.G, smem, smem_dbl);
        local_apply(w.Y, mq, R, w.ty, w.tsr ? w.tsr + ts_region_doubles(mq, K) / 2 : nullptr, K, V + q0, ldo, r, w.G,
                    smem, smem_dbl);
    }
    PH_END(12, t5);
    gang_sync(gg);
    return r;
}

// Side-split gang truncation of X Y^T: members [0, Gs) hold rows of X (their panel w.X), members
// [Gs, 2 Gs) rows of Y (panel w.Y); every member factors ONE local panel, the two TSQR trees run on
// their own members (node (b, s) of a side on that side's member b), member 0 truncates the core,
// the cores go down the trees and each member writes its rows of U (X side) or V (Y side).  Same
// arithmetic as gang_compress with the per-side row partition.
__device__ __noinline__ int gang_compress_split(const CompressWs &w, const GangWs &gw, Gang &gg, int R, double eps,
                                   double tol_q, bool svd, int kmax, int rlim, double *U, double *V, int64_t ldo,
                                   int *cb, int *of, double *red, double *redv, int64_t *redi, double *smem,
                                   int64_t smem_dbl)
{
    if (R == 0) { *cb = 0; *of = 0; return 0; }
    const int Gs = gg.Gs, gs = gg.gs, side = gg.side;
    const int64_t mq = gg.mq, q0 = gg.q0;
    const int64_t RR = (int64_t)R * R;
    const int K = w.K;
    double *Pn = side ? w.Y : w.X;
    double *tau = side ? w.ty : w.tx;
    double *Bk = side ? gw.BY : gw.BX, *Nd = side ? gw.NY : gw.NX, *Ck = side ? gw.CY : gw.CX;
    PH_BEGIN(t1);
    local_qr(Pn, mq, R, tau, w.tsr, K, smem, smem_dbl, red);
    for (int e = threadIdx.x; e < RR; e += NT) {
        const int i = e % R, k = e / R;
        __stcg(Bk + (int64_t)gs * RR + e, (k >= i) ? Pn[i + mq * k] : 0.0);
    }
    PH_END(9, t1);
    gang_sync(gg);
    PH_BEGIN(t2);
    int top = 1;
    while (2 * top < Gs) top *= 2;
    for (int s = 1; s < Gs; s *= 2) {
        if (gs % (2 * s) == 0 && gs + s < Gs) tsqr_node_up(Bk, Nd, gw.nslot, gs, s, R, smem, smem_dbl, red);
        gang_sync(gg);
    }
    PH_END(10, t2);
    if (gg.g == 0) {
        PH_BEGIN(t3);
        for (int e = threadIdx.x; e < RR; e += NT) {
            w.RX[e] = __ldcg(gw.BX + e);
            w.RY[e] = __ldcg(gw.BY + e);
        }
        __syncthreads();
        int c1 = 0, o1 = 0;
        const int rr = compress_core(core_ws_sm(w, smem, smem_dbl, R), w.RX, R, w.RY, R, R, eps, tol_q, svd, kmax,
                                     rlim, gw.CX, gw.CY, R, R, &c1, &o1, red, redv, redi);
        if (threadIdx.x == 0) { gw.ires[0] = rr; gw.ires[1] = c1; gw.ires[2] = o1; }
        PH_END(11, t3);
    }
    gang_sync(gg);
    const int r = __ldcg(gw.ires);
    PH_BEGIN(t4);
    if (r > 0) {
        for (int s = top; s >= 1; s /= 2) {
            if (gs % (2 * s) == 0 && gs + s < Gs) tsqr_node_down(Ck, Nd, gw.nslot, gs, s, R, r, w.G, smem, smem_dbl);
            gang_sync(gg);
        }
    }
    PH_END(10, t4);
    PH_BEGIN(t5);
    const int64_t Rr = (int64_t)R * r;
    double *Out = side ? V : U;
    for (int64_t e = threadIdx.x; e < mq * r; e += NT) {
        const int64_t i = e % mq;
        const int cc = (int)(e / mq);
        Out[q0 + i + ldo * cc] = (i < R) ? __ldcg(Ck + (int64_t)gs * Rr + i + (int64_t)R * cc) : 0.0;
    }
    *cb = __ldcg(gw.ires + 1);
    *of = __ldcg(gw.ires + 2);
    __syncthreads();
    if (r > 0) local_apply(Pn, mq, R, tau, w.tsr, K, Out + q0, ldo, r, w.G, smem, smem_dbl);
    PH_END(12, t5);
    gang_sync(gg);
    return r;
}

// Gang ACA (Alg. B.1) of a big admissible block with the readings of
// aca_partial (first row 0, ties -> lowest index, scaled column, zero-row skip, stop at eps_aca).
// Member g evaluates the columns j and rows i in [q0, q0 + mq) of each cross; the pivot row of U
// and the pivot column of V are published through the shared workspace.  Ul, Vl: local panels
// (mq x Kmax, ld mq).  Returns k.
__device__ int gang_aca(const MaternParams &mp, const Pts P, int64_t R0, int64_t C0, int64_t m,
                        double *Ul, double *Vl, uint8_t *used, int Kmax, double eps_aca, const GangWs &gw, Gang &gg,
                        double *red, double *redv, int64_t *redi)
{
    const int G = gg.G, g = gg.g;
    const int64_t mq = gg.mq, q0 = gg.q0;
    for (int64_t i = threadIdx.x; i < mq; i += NT) used[i] = 0;
    int64_t istar = 0;
    int k = 0, par = 0;
    double n1 = 0.0;
    int64_t guard = 0;
    gang_sync(gg);
    while (k < Kmax && guard++ < m + Kmax) {
        // row residual of row istar (U[istar, :k] published in urow)
        const bool d3 = P.z != nullptr;
        const double xi = P.x[R0 + istar], yi = P.y[R0 + istar], zi = d3 ? P.z[R0 + istar] : 0.0;
        double *vk = Vl + mq * k;
        double bv = 0.0;
        int64_t bi = 0;
        for (int64_t j = threadIdx.x; j < mq; j += NT) {
            double a = hcov_cov_entry_d(mp, xi, yi, zi, P.x[C0 + q0 + j], P.y[C0 + q0 + j], d3 ? P.z[C0 + q0 + j] : 0.0,
                                        (R0 + istar) == (C0 + q0 + j), d3);
            for (int l = 0; l < k; ++l) a -= __ldcg(gw.urow + l) * Vl[j + mq * l];
            vk[j] = a;
            const double aa = fabs(a);
            if (vi_better(aa, q0 + j, bv, bi)) { bv = aa; bi = q0 + j; }
        }
        ValIdx b = block_argmax(bv, bi, redv, redi);
        if (threadIdx.x == 0) {
            __stcg(gw.pv + par * G + g, b.v);
            __stcg(gw.pi + par * G + g, b.i);
        }
        if (istar >= q0 && istar < q0 + mq && threadIdx.x == 0) used[istar - q0] = 1;
        gang_sync(gg);
        ValIdx best{__ldcg(gw.pv + par * G), __ldcg(gw.pi + par * G)};
        for (int h = 1; h < G; ++h) {
            double v2 = __ldcg(gw.pv + par * G + h);
            int64_t i2 = __ldcg(gw.pi + par * G + h);
            if (vi_better(v2, i2, best.v, best.i)) { best.v = v2; best.i = i2; }
        }
        par ^= 1;
        if (!(best.v > 0.0)) {
            // zero residual row: next unused row (lowest index)
            int64_t cand = m;
            for (int64_t i = threadIdx.x; i < mq; i += NT)
                if (!used[i] && q0 + i < cand) cand = q0 + i;
            ValIdx cmin = block_argmax(-(double)cand, cand, redv, redi);
            if (threadIdx.x == 0) __stcg(gw.pi + par * G + g, cmin.i);
            gang_sync(gg);
            int64_t c2 = m;
            for (int h = 0; h < G; ++h) c2 = min(c2, (int64_t)__ldcg(gw.pi + par * G + h));
            par ^= 1;
            if (c2 >= m) break;
            istar = c2;
            // publish U[istar, :k] (owner)
            if (istar >= q0 && istar < q0 + mq)
                for (int l = threadIdx.x; l < k; l += NT) __stcg(gw.urow + l, Ul[(istar - q0) + mq * l]);
            gang_sync(gg);
            continue;
        }
        const int64_t js = best.i;
        // publish V[js, :k+1] (owner of column js)
        if (js >= q0 && js < q0 + mq)
            for (int l = threadIdx.x; l <= k; l += NT) __stcg(gw.vrow + l, Vl[(js - q0) + mq * l]);
        gang_sync(gg);
        const double piv = __ldcg(gw.vrow + k);
        const bool d3j = P.z != nullptr;
        const double xj = P.x[C0 + js], yj = P.y[C0 + js], zj = d3j ? P.z[C0 + js] : 0.0;
        double *uk = Ul + mq * k;
        bv = -1.0;
        bi = m;
        double su = 0.0, sv = 0.0;
        for (int64_t i = threadIdx.x; i < mq; i += NT) {
            double cc = hcov_cov_entry_d(mp, P.x[R0 + q0 + i], P.y[R0 + q0 + i], d3j ? P.z[R0 + q0 + i] : 0.0, xj, yj, zj,
                                         (R0 + q0 + i) == (C0 + js), d3j);
            for (int l = 0; l < k; ++l) cc -= Ul[i + mq * l] * __ldcg(gw.vrow + l);
            const double u = cc / piv;
            uk[i] = u;
            su += u * u;
            const double vv = vk[i];
            sv += vv * vv;
            if (!used[i]) {
                const double aa = fabs(cc);
                if (vi_better(aa, q0 + i, bv, bi)) { bv = aa; bi = q0 + i; }
            }
        }
        su = block_sum(su, red);
        sv = block_sum(sv, red);
        ValIdx nb = block_argmax(bv, bi, redv, redi);
        if (threadIdx.x == 0) {
            __stcg(gw.pv + par * G + g, nb.v);
            __stcg(gw.pi + par * G + g, nb.i);
            __stcg(gw.ps + 2 * (par * G + g), su);
            __stcg(gw.ps + 2 * (par * G + g) + 1, sv);
        }
        gang_sync(gg);
        double tsu = 0.0, tsv = 0.0;
        ValIdx nbest{-1.0, m};
        for (int h = 0; h < G; ++h) {
            tsu += __ldcg(gw.ps + 2 * (par * G + h));
            tsv += __ldcg(gw.ps + 2 * (par * G + h) + 1);
            double v2 = __ldcg(gw.pv + par * G + h);
            int64_t i2 = __ldcg(gw.pi + par * G + h);
            if (vi_better(v2, i2, nbest.v, nbest.i)) { nbest.v = v2; nbest.i = i2; }
        }
        par ^= 1;
        ++k;
        const double nn = sqrt(tsu) * sqrt(tsv);
        bool stop = false;
        if (k == 1) n1 = nn;
        else if (nn <= eps_aca * n1) stop = true;
        if (nbest.i >= m || nbest.v < 0.0) stop = true;
        if (stop) break;
        istar = nbest.i;
        // publish U[istar, :k] (owner of row istar)
        if (istar >= q0 && istar < q0 + mq)
            for (int l = threadIdx.x; l < k; l += NT) __stcg(gw.urow + l, Ul[(istar - q0) + mq * l]);
        gang_sync(gg);
    }
    gang_sync(gg);
    return k;
}

// A5 + A6: ACA of the admissible block (Alg. B.1) to eps/10, then QR + SVD truncation to (eps, kmax).
// gg == nullptr: one CTA; else one member of a gang (scr = this CTA's private scratch).
__device__ void task_aca(const Ctx &c, const DTask &tk, double *scr, double *smem, double *red, double *redv,
                         int64_t *redi, double &fl_asm, double &fl_tr, Gang *gg)
{
    const int r = tk.a;
    const DRBlk b = c.rblk[r];
    const int64_t m = b.m;
    const int K = aca_kmax(m, c.kcap);
    const int KB = kbuf_of(c.kcap);
    // SPD-preserving mode: C~ near-lossless (eps * interm_rel, no rank cap; the (eps, kmax) truncation
    // comes after the block's solve, R27)
    const double ea = c.factor_trunc ? interm_tol(c) : c.eps;
    const int km = c.factor_trunc ? 0 : c.kmax;
    double *X2, *Y2;
    int cb = 0, of = 0, k, rk;
    if (!gg) {
        CompressWs w = make_ws(scr, m, KB, &X2, &Y2);
        uint8_t *used = (uint8_t *)w.tail;
        PH_BEGIN(tp);
        k = aca_partial(c.mp, Pts{c.xs, c.ys, c.zs}, b.row0, b.col0, m, w.X, w.Y, K, 0.1 * ea, used, red, redv, redi);
        PH_END(8, tp);
        if (k == K && K < m && threadIdx.x == 0) atomicAdd(c.flags + cut_flag(c), 1);   // ACA not converged
        rk = compress(w, m, k, ea, final_tol(ea, k), true, km, c.kcap, r_U(c, r), r_V(c, r), m, &cb, &of,
                      red, redv, redi, smem, c.smem_dbl);
        if (c.factor_trunc) record_interm(c, r, rk, of);
        else record_rank(c, r, rk, cb, of);
    } else {
        gang_rows(*gg, m);
        CompressWs w = make_ws(scr, gg->mq, KB, &X2, &Y2, 4);
        w.tsr = scr + task_scratch_base(gg->mq, c.kcap, 4);
        GangWs gw = make_gws(gg->shared, KB, gg->G);
        k = gang_aca(c.mp, Pts{c.xs, c.ys, c.zs}, b.row0, b.col0, m, w.X, w.Y, (uint8_t *)w.tail, K, 0.1 * ea, gw, *gg, red,
                     redv, redi);
        if (k == K && K < m && gg->g == 0 && threadIdx.x == 0) atomicAdd(c.flags + cut_flag(c), 1);
        rk = gang_compress(w, gw, *gg, k, ea, final_tol(ea, k), true, km, c.kcap, r_U(c, r), r_V(c, r), m,
                           &cb, &of, red, redv, redi, smem, c.smem_dbl);
        if (gg->g == 0) {
            if (c.factor_trunc) record_interm(c, r, rk, of);
            else record_rank(c, r, rk, cb, of);
        }
    }
    const double share = gg ? 1.0 / gg->G : 1.0;
    fl_asm += share * 2.0 * m * k;                       // kernel evaluations (rows + columns)
    fl_tr += share * (2.0 * m * k * k + compress_flops(m, k, rk));
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

// S (m x m, ld m) += XA YB^T, XA and YB m x W (ld m, global).  Row blocks of 16 MA rows per pass;
// thread (ty, tx) of the 16 x 32 grid owns rows ty + 16 a and columns tx + 32 b; k staged through
// shared memory (sb: 32 (16 MA + 32 NB) doubles).
template <int MA, int NB>
__device__ void dense_gemm_add(double *S, int m, const double *XA, const double *YB, int W, double *sb)
{
    constexpr int KC = 32, PR = 16 * MA, CN = 32 * NB;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double *xs = sb, *ys = sb + KC * PR;
    for (int c0 = 0; c0 < m; c0 += CN)
    for (int p0 = 0; p0 < m; p0 += PR) {
        double acc[MA][NB];
#pragma unroll
        for (int a = 0; a < MA; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b) acc[a][b] = 0.0;
        for (int k0 = 0; k0 < W; k0 += KC) {
            __syncthreads();
            for (int e = threadIdx.x; e < KC * PR; e += NT) {
                const int k = e / PR, i = e % PR;
                xs[e] = (p0 + i < m && k0 + k < W) ? __ldcg(XA + (p0 + i) + (int64_t)m * (k0 + k)) : 0.0;
            }
            for (int e = threadIdx.x; e < KC * CN; e += NT) {
                const int k = e / CN, j = e % CN;
                ys[e] = (c0 + j < m && k0 + k < W) ? __ldcg(YB + c0 + j + (int64_t)m * (k0 + k)) : 0.0;
            }
            __syncthreads();
#pragma unroll 4
            for (int k = 0; k < KC; ++k) {
                double xa[MA], yb[NB];
#pragma unroll
                for (int a = 0; a < MA; ++a) xa[a] = xs[k * PR + ty + 16 * a];
#pragma unroll
                for (int b = 0; b < NB; ++b) yb[b] = ys[k * CN + tx + 32 * b];
#pragma unroll
                for (int a = 0; a < MA; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) acc[a][b] = fma(xa[a], yb[b], acc[a][b]);
            }
        }
#pragma unroll
        for (int a = 0; a < MA; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int i = p0 + ty + 16 * a, j = c0 + tx + 32 * b;
                if (i < m && j < m) S[i + (int64_t)m * j] += acc[a][b];
            }
    }
    __syncthreads();
}

// S (m x m, ld m) += XA YB^T on the FP64 tensor cores (the U V^T low-rank-update product of the
// dense-mode accumulation; north_star: DMMA for the truly dense contractions).  XA, YB: m x W (ld m,
// global scratch).  CTA tile (8 WM WGM) x (8 WN WGN), warp grid WGM x WGN (= NWARP warps), every
// warp WM x WN mma.sync.m8n8k4.f64 blocks; k staged through shared memory in chunks of 32, row
// stride (tile + 4) doubles so the four k of a fragment load fall into disjoint banks.
// sb: 32 (TM + TN + 8) doubles.
template <int WM, int WN, int WGM, int WGN>
__device__ void dense_gemm_add_dmma(double *S, int m, const double *XA, const double *YB, int W, double *sb)
{
    static_assert(WGM * WGN == NWARP, "warp grid must cover the CTA");
    constexpr int KC = 32, TM = 8 * WM * WGM, TN = 8 * WN * WGN, LX = TM + 4, LY = TN + 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % WGM, wn = warp / WGM;
    const int g = lane >> 2, q = lane & 3;
    double *xs = sb, *ys = sb + KC * LX;
    for (int c0 = 0; c0 < m; c0 += TN)
    for (int p0 = 0; p0 < m; p0 += TM) {
        double acc[WM][WN][2];
#pragma unroll
        for (int u = 0; u < WM; ++u)
#pragma unroll
            for (int v = 0; v < WN; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
        for (int k0 = 0; k0 < W; k0 += KC) {
            __syncthreads();
            for (int e = threadIdx.x; e < KC * TM; e += NT) {
                const int k = e / TM, i = e % TM;
                xs[k * LX + i] = (p0 + i < m && k0 + k < W) ? __ldcg(XA + (p0 + i) + (int64_t)m * (k0 + k)) : 0.0;
            }
            for (int e = threadIdx.x; e < KC * TN; e += NT) {
                const int k = e / TN, j = e % TN;
                ys[k * LY + j] = (c0 + j < m && k0 + k < W) ? __ldcg(YB + (c0 + j) + (int64_t)m * (k0 + k)) : 0.0;
            }
            __syncthreads();
            const int kc = min(KC, (W - k0 + 3) & ~3);
            const double *xw = xs + 8 * WM * wm + g, *yw = ys + 8 * WN * wn + g;
#pragma unroll 2
            for (int kk = 0; kk < kc; kk += 4) {
                double a[WM], b[WN];
#pragma unroll
                for (int u = 0; u < WM; ++u) a[u] = xw[(kk + q) * LX + 8 * u];
#pragma unroll
                for (int v = 0; v < WN; ++v) b[v] = yw[(kk + q) * LY + 8 * v];
#pragma unroll
                for (int u = 0; u < WM; ++u)
#pragma unroll
                    for (int v = 0; v < WN; ++v) dmma_8x8x4(acc[u][v][0], acc[u][v][1], a[u], b[v]);
            }
        }
#pragma unroll
        for (int u = 0; u < WM; ++u)
#pragma unroll
            for (int v = 0; v < WN; ++v) {
                const int i = p0 + 8 * (WM * wm + u) + g, j = c0 + 8 * (WN * wn + v) + 2 * q;
                if (i < m && j < m) S[i + (int64_t)m * j] += acc[u][v][0];
                if (i < m && j + 1 < m) S[i + (int64_t)m * (j + 1)] += acc[u][v][1];
            }
    }
    __syncthreads();
}

// Columns of one pending term in the batched GEMM of the dense accumulation (0 if a factor has rank
// 0; 0 for a tile x tile term, which is applied directly to its 32 x 32 target, tt_apply).
__device__ __forceinline__ int term_width(const Ctx &c, const DTerm &t)
{
    if (t.kind == TM_TT) return 0;
    const int ra = __ldcg(c.rank + c.fac_rank_src[t.a]), rb = __ldcg(c.rank + c.fac_rank_src[t.b]);
    if (ra == 0 || rb == 0) return 0;
    return (t.core >= 0 && c.term_min && ra < rb) ? ra : rb;
}

// S[ar + i, br + j] -= sum_k A(i, k) B(j, k) for the 32 x 32 target of a tile x tile term (the
// tiles staged in shared memory, 2 x 32 x 32 doubles of sb); all threads of the CTA, in term order.
__device__ __forceinline__ void tt_apply(const Ctx &c, const DTerm &t, double *S, int64_t m, int64_t R0, int64_t C0,
                                         double *sb)
{
    const DNode na = c.nodes[c.tile_node[t.a]], nb = c.nodes[c.tile_node[t.b]];
    const int64_t ar = (int64_t)na.i * HCOV_LEAF - R0, br = (int64_t)nb.i * HCOV_LEAF - C0;
    const double *A = c.tiles + (int64_t)t.a * HCOV_TILE, *B = c.tiles + (int64_t)t.b * HCOV_TILE;
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
        sb[e] = __ldcg(A + e);
        sb[HCOV_TILE + e] = __ldcg(B + e);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
        const int i = e & 31, j = e >> 5;
        double s = 0.0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) s = fma(sb[i + 32 * k], sb[HCOV_TILE + j + 32 * k], s);
        const int64_t gi = ar + i, gj = br + j;
        if (gi >= 0 && gi < m && gj >= 0 && gj < m) S[gi + m * gj] -= s;
    }
    __syncthreads();
}

// Dense-mode accumulation (m <= c.dense_max): S += U V^T - sum_k terms_k (S zero on entry), in
// batches of at most Wcap columns gathered into XA / YB (m x Wcap each, global scratch) for the
// low-rank terms; tile x tile terms go straight to their 32 x 32 target (tt_apply) instead of
// being zero-padded to m rows.  Returns the flops.
#define DENSE_BATCH 128
__device__ double dense_accumulate(const Ctx &c, const DTask &tk, double *S, int64_t m, int64_t R0, int64_t C0,
                                   const double *U, const double *V, int r0, double *XA, int64_t Wcap, double *sb,
                                   int64_t sb_dbl)
{
    const int kbw = (int)min((int64_t)512, sb_dbl / NWARP);   // per-warp core staging (gather phase)
    __shared__ int s_off[DENSE_BATCH + 1], s_kk[DENSE_BATCH];
    __shared__ int s_nt, s_next, s_w;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *YB = XA + m * Wcap;
    double fl = 0.0;
    int kk = tk.b;
    bool first = true;
    while (first || kk < tk.c) {
        // widths of the next DENSE_BATCH terms in parallel, then the batch's prefix by thread 0
        const int cand = min(DENSE_BATCH, tk.c - kk);
        for (int q = threadIdx.x; q < cand; q += NT) s_kk[q] = term_width(c, c.terms[c.xterm[kk + q]]);
        __syncthreads();
        if (threadIdx.x == 0) {
            int W = (first ? r0 : 0), nt = 0;
            while (nt < cand) {
                const int w = s_kk[nt];
                if (W + w > Wcap) break;
                s_off[nt] = W;
                W += w;
                ++nt;
            }
            s_off[nt] = W;
            s_nt = nt;
            s_next = kk + nt;
            s_w = W;
        }
        __syncthreads();
        const int nt = s_nt, W = s_w;
        if (first && r0 > 0)
            for (int64_t e = threadIdx.x; e < m * r0; e += NT) {
                XA[e] = __ldcg(U + e);
                YB[e] = __ldcg(V + e);
            }
        for (int j = warp; j < nt; j += NWARP) {
            const DTerm t = c.terms[c.xterm[kk + j]];
            const int off = s_off[j], w = s_off[j + 1] - off;
            if (w == 0) continue;
            double *xc = XA + m * off, *yc = YB + m * off;
            if (t.kind == TM_TT) {
                continue;   // tt_apply below
            } else {
                const Fac A = get_fac(c, t.a), B = get_fac(c, t.b);
                const int ra = A.ncols, rbn = B.ncols;
                const int64_t r_lo = max(R0, A.row0), r_hi = min(R0 + m, A.row0 + A.nrows);
                const int64_t c_lo = max(C0, B.row0), c_hi = min(C0 + m, B.row0 + B.nrows);
                const double *Kc = (t.core >= 0) ? c.cores + (int64_t)t.core * c.kcore * c.kcore : nullptr;
                // the core K (ra x rbn) staged in this warp's slice of shared memory: kb[a + ra b]
                double *kb = sb + (int64_t)warp * kbw;
                const bool kstaged = Kc && ra * rbn <= kbw;
                if (kstaged) {
                    for (int e = lane; e < ra * rbn; e += 32) kb[e] = __ldcg(Kc + (e % ra) + (int64_t)c.kcore * (e / ra));
                    __syncwarp();
                }
                // the product side: [-A K, B] (w = rbn columns) or, when A has the lower rank,
                // [-A, B K^T] (w = ra columns; term_width).  F: the factor multiplied by the core
                // (nin columns), M(l, o) = km[l sl + o so] the core as seen from F.
                const bool swp = Kc && w < rbn;
                const int nin = swp ? rbn : ra;
                const double *km = kstaged ? kb : Kc;
                const int64_t kld = kstaged ? ra : c.kcore;
                const int64_t sl = swp ? kld : 1, so = swp ? 1 : kld;
                const double sgn = swp ? 1.0 : -1.0;
                for (int64_t i = lane; i < m; i += 32) {
                    const int64_t gi = R0 + i, gj = C0 + i;
                    const bool inr = gi >= r_lo && gi < r_hi, inc = gj >= c_lo && gj < c_hi;
                    const double *Ar = A.p + (gi - A.row0), *Br = B.p + (gj - B.row0);
                    double *pc = swp ? yc : xc;          // the product panel, the plain-copy panel
                    double *cc = swp ? xc : yc;
                    const bool inp = swp ? inc : inr, inq = swp ? inr : inc;
                    const double *Fr = swp ? Br : Ar, *Gr = swp ? Ar : Br;
                    const int64_t fld = swp ? B.ld : A.ld, gld = swp ? A.ld : B.ld;
                    const double csg = swp ? -1.0 : 1.0;  // sign of the copied panel (X carries the minus)
                    if (!inp) {
                        for (int b = 0; b < w; ++b) pc[i + m * b] = 0.0;
                    } else if (!Kc) {
                        for (int b = 0; b < w; ++b) pc[i + m * b] = -__ldcg(Fr + fld * b);
                    } else if (kstaged && nin <= 24) {
                        // the row of F in registers first: nin independent L2 loads in flight (one
                        // latency per row; inside the a-loop below they were exposed four at a time,
                        // once per block of 8 output columns)
                        double fa[24];
#pragma unroll
                        for (int a = 0; a < 24; ++a) fa[a] = (a < nin) ? __ldcg(Fr + fld * a) : 0.0;
                        for (int b0 = 0; b0 < w; b0 += 8) {
                            double acc[8];
#pragma unroll
                            for (int bb = 0; bb < 8; ++bb) acc[bb] = 0.0;
#pragma unroll
                            for (int a = 0; a < 24; ++a) {
                                if (a < nin) {
#pragma unroll
                                    for (int bb = 0; bb < 8; ++bb)
                                        if (b0 + bb < w) acc[bb] = fma(fa[a], km[a * sl + (b0 + bb) * so], acc[bb]);
                                }
                            }
#pragma unroll
                            for (int bb = 0; bb < 8; ++bb)
                                if (b0 + bb < w) pc[i + m * (b0 + bb)] = sgn * acc[bb];
                        }
                    } else {
                        for (int b0 = 0; b0 < w; b0 += 8) {
                            double acc[8];
#pragma unroll
                            for (int bb = 0; bb < 8; ++bb) acc[bb] = 0.0;
                            for (int a0 = 0; a0 < nin; a0 += 4) {
                                double xa[4];
#pragma unroll
                                for (int u = 0; u < 4; ++u) xa[u] = (a0 + u < nin) ? __ldcg(Fr + fld * (a0 + u)) : 0.0;
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const int a = a0 + u;
                                    if (a < nin) {
#pragma unroll
                                        for (int bb = 0; bb < 8; ++bb)
                                            if (b0 + bb < w) {
                                                const double kv = kstaged ? km[a * sl + (b0 + bb) * so]
                                                                          : __ldcg(km + a * sl + (b0 + bb) * so);
                                                acc[bb] = fma(xa[u], kv, acc[bb]);
                                            }
                                    }
                                }
                            }
#pragma unroll
                            for (int bb = 0; bb < 8; ++bb)
                                if (b0 + bb < w) pc[i + m * (b0 + bb)] = sgn * acc[bb];
                        }
                    }
                    for (int b = 0; b < w; ++b)
                        cc[i + m * b] = inq ? csg * __ldcg(Gr + gld * b) : 0.0;
                }
                if (Kc) fl += 2.0 * (swp ? c_hi - c_lo : r_hi - r_lo) * ra * rbn;
            }
        }
        __syncthreads();
        PH_BEGIN(tdg);
        if (W > 0) {
            if (c.dense_dmma) {
                if (m <= 64) dense_gemm_add_dmma<2, 2, 4, 4>(S, (int)m, XA, YB, W, sb);
                else dense_gemm_add_dmma<4, 4, 4, 4>(S, (int)m, XA, YB, W, sb);
            } else if (m <= 64) dense_gemm_add<4, 2>(S, (int)m, XA, YB, W, sb);
            else if (m <= 128) dense_gemm_add<8, 4>(S, (int)m, XA, YB, W, sb);
            else dense_gemm_add<4, 8>(S, (int)m, XA, YB, W, sb);
            fl += 2.0 * m * m * W;
        }
        for (int j = 0; j < nt; ++j) {
            const DTerm t = c.terms[c.xterm[kk + j]];
            if (t.kind == TM_TT) {
                tt_apply(c, t, S, m, R0, C0, sb);
                fl += 2.0 * HCOV_TILE * 32;
            }
        }
        PH_END(15, tdg);
        kk = s_next;
        first = false;
        __syncthreads();
    }
    return fl;
}

// A7 low-rank blocks: S = U V^T - sum of all pending terms, accumulated in factored form
// X = [U, -A_1 K_1, ...], Y = [V, B_1, ...] (in scratch).  When the panel is full it is
// recompressed near-losslessly (pivoted QR at eps * interm_rel, no SVD; R22); at the end X Y^T is truncated
// to (eps, kmax) by QR + SVD (A6; Remark 2).
__device__ void task_rapp(const Ctx &c, const DTask &tk, double *scr, double *smem, double *red, double *redv,
                          int64_t *redi, double &fl, Gang *gg)
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
    if (gg) gang_rows(*gg, m);
    if (m <= c.dense_max) {
        // small block: exact dense accumulation S = U V^T - sum of terms (m x m), fully pivoted
        // cross approximation of S to 0.1 eps |S|_max / m (so |S - X Y^T|_2 <= 0.1 eps |S|_2), then
        // QR + SVD truncation to (eps, kmax)
        // S lives in shared memory when it leaves room for the GEMM staging (m <= 128)
        const int64_t stage = m <= 64 ? 32 * 136 : m <= 128 ? 32 * 264 : 32 * 320;   // dense_gemm_add(_dmma) staging
        const bool s_sm = m * m + stage <= c.smem_dbl;
        double *S = s_sm ? smem : scr;
        double *gs = s_sm ? smem + m * m : smem;
        CompressWs wd = make_ws(scr + m * m, m, K, &X2, &Y2);   // X, Y panels (m x K) follow S
        PH_BEGIN(tg);
        // S = U V^T - sum of terms as S = XA YB^T, batch by batch: the factor columns of a batch of
        // terms (XA = [U, -A_1 K_1, -T_a, ...], YB = [V, B_1, T_b, ...], zero outside each term's
        // rows) are gathered warp-parallel into the panel scratch, then one CTA GEMM adds them
        for (int64_t e = threadIdx.x; e < m * m; e += NT) S[e] = 0.0;
        // batch capacity: the whole per-CTA scratch after S (sized for the largest gang member)
        const int64_t wcap = max((int64_t)3 * K, (c.scr_stride - m * m - 64) / (2 * m));
        fl += dense_accumulate(c, tk, S, m, R0, C0, U, V, r0, wd.X, wcap, gs,
                               s_sm ? c.smem_dbl - m * m : c.smem_dbl);
        PH_END(6, tg);
        const int KA = (int)(m < K ? m : K);
        PH_BEGIN(ta);
        int k = aca_full(S, m, wd.X, wd.Y, KA, 0.1 * c.eps / (double)m, 0.1 * c.eps, red, redv, redi);
        PH_END(5, ta);
        fl += 2.0 * m * m * k;
        if (k == KA && KA < m && threadIdx.x == 0) atomicAdd(c.flags + cut_flag(c), 1);
        // tk.d == 2: the pre-solve state of the SPD-preserving mode (near-lossless, no cap, R27)
        const bool pre = (tk.d == 2);
        const double ed = pre ? interm_tol(c) : c.eps;
        int rk = compress(wd, m, k, ed, final_tol(ed, k), true, pre ? 0 : c.kmax, c.kcap, U, V, m, &cb, &of, red,
                          redv, redi, smem, c.smem_dbl);
        fl += compress_flops(m, k, rk);
        if (pre) record_interm(c, r, rk, of);
        else record_rank(c, r, rk, cb, of);
        return;
    }
    // factor mode (m > c.dense_max); rows [q0, q0 + mq) belong to this CTA (the whole block
    // without a gang); the panels w.X, w.Y, X2, Y2 hold those rows (ld mq).
    CompressWs w = make_ws(scr, gg ? gg->mq : m, K, &X2, &Y2, gg ? 4 : 6);
    if (gg) w.tsr = scr + task_scratch_base(gg->mq, c.kcap, 4);
    const int64_t mq = gg ? gg->mq : m, q0 = gg ? gg->q0 : 0;
    GangWs gw{};
    if (gg) gw = make_gws(gg->shared, K, gg->G);
    int cur = r0;
    // side-split gangs: a member builds (and factors) only its side's panel
    const bool doX = !gg || gg->side != 1, doY = !gg || gg->side != 0;
    const bool split = gg && gg->split;
    PH_BEGIN(tl0);
    for (int64_t e = threadIdx.x; e < mq * (int64_t)r0; e += NT) {
        const int64_t i = e % mq, l = e / mq;
        if (doX) w.X[i + mq * l] = __ldcg(U + q0 + i + m * l);
        if (doY) w.Y[i + mq * l] = __ldcg(V + q0 + i + m * l);
    }
    __syncthreads();
    PH_END(14, tl0);
    for (int kk = tk.b; kk < tk.c; ++kk) {
        const DTerm t = c.terms[c.xterm[kk]];
        int width;
        bool swp = false;   // LR term with rank A < rank B: appended as [-A, B K^T] (rank A columns)
        if (t.kind == TM_TT) width = 32;
        else {
            width = __ldcg(c.rank + c.fac_rank_src[t.b]);
            const int wa = __ldcg(c.rank + c.fac_rank_src[t.a]);
            if (wa == 0) continue;
            if (t.core >= 0 && c.term_min && wa < width) { width = wa; swp = true; }
        }
        if (width == 0) continue;
        if (cur + width > K) {
            int icb = 0, iof = 0, rk;
            if (split)
                rk = gang_compress_split(w, gw, *gg, cur, c.eps, interm_tol(c), false, 0, K - maxw, X2 - q0, Y2 - q0,
                                         mq, &icb, &iof, red, redv, redi, smem, c.smem_dbl);
            else if (gg)
                rk = gang_compress(w, gw, *gg, cur, c.eps, interm_tol(c), false, 0, K - maxw, X2 - q0, Y2 - q0, mq,
                                   &icb, &iof, red, redv, redi, smem, c.smem_dbl);
            else
                rk = compress(w, m, cur, c.eps, interm_tol(c), false, 0, K - maxw, X2, Y2, m, &icb, &iof, red,
                              redv, redi, smem, c.smem_dbl);
            fl += (gg ? 1.0 / gg->G : 1.0) * compress_flops(m, cur, rk);
            if (iof && threadIdx.x == 0 && (!gg || gg->g == 0)) atomicAdd(c.flags + cut_flag(c), 1);
            double *tx = w.X, *ty = w.Y;
            w.X = X2; w.Y = Y2; X2 = tx; Y2 = ty;
            cur = rk;
        }
        PH_BEGIN(tap);
        double *xc = w.X + mq * cur, *yc = w.Y + mq * cur;
        for (int64_t e = threadIdx.x; e < mq * (int64_t)width; e += NT) {
            if (doX) xc[e] = 0.0;
            if (doY) yc[e] = 0.0;
        }
        __syncthreads();
        if (t.kind == TM_TT) {
            const DNode na = c.nodes[c.tile_node[t.a]], nb = c.nodes[c.tile_node[t.b]];
            const int64_t ar = (int64_t)na.i * HCOV_LEAF - R0 - q0, br = (int64_t)nb.i * HCOV_LEAF - C0 - q0;
            const double *A = c.tiles + (int64_t)t.a * HCOV_TILE, *B = c.tiles + (int64_t)t.b * HCOV_TILE;
            for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
                int i = e & 31, k = e >> 5;
                if (doX && ar + i >= 0 && ar + i < mq) xc[ar + i + mq * k] = -__ldcg(A + e);
                if (doY && br + i >= 0 && br + i < mq) yc[br + i + mq * k] = __ldcg(B + e);
            }
        } else {
            Fac A = get_fac(c, t.a), B = get_fac(c, t.b);
            const int ra = A.ncols, rb = B.ncols;
            const int64_t r_lo = max(R0 + q0, A.row0), r_hi = min(R0 + q0 + mq, A.row0 + A.nrows);
            const int64_t c_lo = max(C0 + q0, B.row0), c_hi = min(C0 + q0 + mq, B.row0 + B.nrows);
            const double *Kc = (t.core >= 0) ? c.cores + (int64_t)t.core * c.kcore * c.kcore : nullptr;
            if (doX && r_hi > r_lo) {
                if (Kc && !swp) {   // xc = -A K  (columns b < rb), staged GEMM
                    cta_gemm_nt(xc + (r_lo - R0 - q0), mq, r_hi - r_lo, rb, ra, A.p + (r_lo - A.row0), A.ld, Kc, c.kcore,
                                1, -1.0, smem);
                    fl += 2.0 * (r_hi - r_lo) * ra * rb;
                } else {
                    for (int64_t e = threadIdx.x; e < (r_hi - r_lo) * (int64_t)width; e += NT) {
                        int64_t i = e % (r_hi - r_lo);
                        int b = (int)(e / (r_hi - r_lo));
                        xc[(r_lo - R0 - q0) + i + mq * b] = -__ldcg(A.p + (r_lo - A.row0) + i + A.ld * b);
                    }
                }
            }
            if (doY && c_hi > c_lo) {
                if (swp) {   // yc = B K^T  (columns a < ra), staged GEMM
                    cta_gemm_nt(yc + (c_lo - C0 - q0), mq, c_hi - c_lo, ra, rb, B.p + (c_lo - B.row0), B.ld, Kc, 1,
                                c.kcore, 1.0, smem);
                    fl += 2.0 * (c_hi - c_lo) * ra * rb;
                } else {
                    for (int64_t e = threadIdx.x; e < (c_hi - c_lo) * (int64_t)rb; e += NT) {
                        int64_t i = e % (c_hi - c_lo);
                        int b = (int)(e / (c_hi - c_lo));
                        yc[(c_lo - C0 - q0) + i + mq * b] = __ldcg(B.p + (c_lo - B.row0) + i + B.ld * b);
                    }
                }
            }
        }
        __syncthreads();
        PH_END(14, tap);
        cur += width;
    }
    // last chunk: truncation to (eps, kmax) into capacity kcap; else near-lossless into 2 kcap
    const bool fin = (tk.d == 1);
    const double tq = fin ? final_tol(c.eps, cur) : interm_tol(c);
    const int kmx = fin ? c.kmax : 0, rl = fin ? c.kcap : 2 * c.kcap;
    int rk;
    if (split) {
        rk = gang_compress_split(w, gw, *gg, cur, c.eps, tq, fin, kmx, rl, U, V, m, &cb, &of, red, redv, redi, smem,
                                 c.smem_dbl);
        fl += compress_flops(m, cur, rk) / gg->G;
    } else if (gg) {
        rk = gang_compress(w, gw, *gg, cur, c.eps, tq, fin, kmx, rl, U, V, m, &cb, &of, red, redv, redi, smem,
                           c.smem_dbl);
        fl += compress_flops(m, cur, rk) / gg->G;
    } else {
        rk = compress(w, m, cur, c.eps, tq, fin, kmx, rl, U, V, m, &cb, &of, red, redv, redi, smem, c.smem_dbl);
        fl += compress_flops(m, cur, rk);
    }
    if (!fin) {
        if (of && threadIdx.x == 0 && (!gg || gg->g == 0)) atomicAdd(c.flags + cut_flag(c), 1);
        cb = 0;
        of = 0;
    }
    if (!gg || gg->g == 0) {
        if (fin) record_rank(c, r, rk, cb, of);
        else {
            if (threadIdx.x == 0) __stcg(c.rank + r, rk);
            __syncthreads();
        }
    }
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

#define SEG_MAXCOL 128  // right-hand-side columns processed per pass of a SEG task

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
#define SEG_BATCH 32
#define SEG_RHS_MAX 128   // right-hand-side blocks whose ranks / bases a SEG task caches
__device__ void task_seg(const Ctx &c, const DTask &tk, double *smem, double &fl)
{
    const Rhs h = get_rhs(c, tk.a);
    const int64_t i = tk.b;
    const int64_t ro = i * HCOV_LEAF - h.row0;   // local row offset of the segment
    double *Ys = smem;                            // 32 x SEG_MAXCOL
    double *Ts = Ys + 32 * SEG_MAXCOL;            // 32 x 32 tile (diagonal block)
    double **colp = (double **)(Ts + HCOV_TILE);  // SEG_MAXCOL column pointers, then the batch area
    __shared__ int s_nk, s_total, s_bn;
    __shared__ int s_boff[SEG_BATCH], s_brk[SEG_BATCH];
    __shared__ int s_rrk[SEG_RHS_MAX];
    __shared__ double *s_rvp[SEG_RHS_MAX];
    int k0 = 0;
    double q = 0.0;
    while (true) {
        if (h.cnt > 0 && h.cnt <= SEG_RHS_MAX) {
            // ranks and V bases of the right-hand-side blocks loaded in parallel (once per task)
            if (k0 == 0) {
                for (int q = threadIdx.x; q < h.cnt; q += NT) {
                    const int r = c.solve_rhs[h.off + q];
                    s_rrk[q] = __ldcg(c.rank + r);
                    s_rvp[q] = r_V(c, r);
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                int k = 0, nk = 0;
                for (int q = 0; q < h.cnt; ++q)
                    for (int j = 0; j < s_rrk[q]; ++j, ++k)
                        if (k >= k0 && nk < SEG_MAXCOL) colp[nk++] = s_rvp[q] + h.m * (int64_t)j;
                s_nk = nk;
                s_total = k;
            }
        } else if (threadIdx.x == 0) {
            int tot;
            s_nk = rhs_columns(c, h, k0, colp, &tot);
            s_total = tot;
        }
        __syncthreads();
        const int nk = s_nk;
        if (nk == 0) break;
        for (int e = threadIdx.x; e < 32 * nk; e += NT) {
            int rr = e & 31, k = e >> 5;
            Ys[e] = __ldcg(colp[k] + ro + rr);
        }
        __syncthreads();
        // contributions in batches: all operands of a batch are loaded into shared memory at once
        // (independent loads, one latency), then each thread accumulates its entries over the batch
        double *bb = (double *)(colp + SEG_MAXCOL);   // batch area (the rest of shared memory)
        const int64_t bcap = c.smem_dbl - (int64_t)(bb - smem) - 8;
        for (int z0 = tk.c; z0 < tk.d;) {
            if (threadIdx.x == 0) {
                int64_t off = 0;
                int z = z0, nb = 0;
                while (z < tk.d && nb < SEG_BATCH) {
                    const DCtr ct = c.ctr[z];
                    const int rk = (ct.kind == 0) ? 32 : __ldcg(c.rank + ct.id);
                    const int64_t need = (ct.kind == 0) ? HCOV_TILE + 32 * nk : 32 * (int64_t)rk + (int64_t)rk * nk;
                    if (off + need > bcap && nb > 0) break;
                    s_boff[nb] = (int)off;
                    s_brk[nb] = rk;
                    off += need;
                    ++nb;
                    ++z;
                }
                s_bn = nb;
            }
            __syncthreads();
            const int nbt = s_bn;
            for (int j = 0; j < nbt; ++j) {
                const DCtr ct = c.ctr[z0 + j];
                double *A = bb + s_boff[j];
                const int rk = s_brk[j];
                if (ct.kind == 0) {
                    const double *T = c.tiles + (int64_t)ct.id * HCOV_TILE;
                    double *X = A + HCOV_TILE;
                    const int64_t jo = (int64_t)ct.aux * HCOV_LEAF - h.row0;
                    for (int e = threadIdx.x; e < HCOV_TILE; e += NT) A[e] = __ldcg(T + e);
                    for (int e = threadIdx.x; e < 32 * nk; e += NT) X[e] = __ldcg(colp[e >> 5] + jo + (e & 31));
                } else if (rk > 0) {
                    const DRBlk b = c.rblk[ct.id];
                    const double *Ub = r_U(c, ct.id);
                    const double *Pb = slot_get(c, ct.aux);
                    const int64_t uo = i * HCOV_LEAF - b.row0;
                    double *X = A + 32 * rk;
                    for (int e = threadIdx.x; e < 32 * rk; e += NT)
                        A[e] = __ldcg(Ub + uo + (e & 31) + (int64_t)b.m * (e >> 5));
                    for (int e = threadIdx.x; e < rk * nk; e += NT) {
                        const int l = e % rk, k = e / rk;
                        X[e] = __ldcg(Pb + l + (int64_t)rk * (k0 + k));
                    }
                }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < 32 * nk; e += NT) {
                const int rr = e & 31, k = e >> 5;
                double sacc = 0.0;
                for (int j = 0; j < nbt; ++j) {
                    const double *A = bb + s_boff[j];
                    const int rk = s_brk[j];
                    if (rk == 0) continue;
                    const double *X = A + 32 * rk;   // dense: rk = 32, A = tile
#pragma unroll 8
                    for (int l = 0; l < rk; ++l) sacc = fma(A[rr + 32 * l], X[l + rk * k], sacc);
                }
                Ys[e] -= sacc;
            }
            for (int j = 0; j < nbt; ++j) fl += 2.0 * 32 * s_brk[j] * nk;
            z0 += nbt;
            __syncthreads();
        }
        // Y_i <- L_ii^{-1} Y_i (forward substitution, one thread per column)
        tile_load(Ts, c.tiles + (int64_t)c.diag_tile[i] * HCOV_TILE);
        __syncthreads();
        // one warp per group of 4 columns, lane = row: 32 steps of (broadcast y_a, update rows > a)
        {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            const double dinv = 1.0 / Ts[lane + 32 * lane];
            for (int k0c = 4 * warp; k0c < nk; k0c += 4 * NWARP) {
                double y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) y[u] = (k0c + u < nk) ? Ys[lane + 32 * (k0c + u)] : 0.0;
#pragma unroll 4
                for (int a = 0; a < 32; ++a) {
                    const double da = __shfl_sync(0xffffffffu, dinv, a);
                    const double la = Ts[lane + 32 * a];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double ya = __shfl_sync(0xffffffffu, y[u], a) * da;
                        if (lane == a) y[u] = ya;
                        else if (lane > a) y[u] = fma(-la, ya, y[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (k0c + u < nk) Ys[lane + 32 * (k0c + u)] = y[u];
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

// P = V_b^T Y[cols of b]  (rank_b x ctot, ld rank_b; allocated here with actual sizes)
__device__ void task_proj(const Ctx &c, const DTask &tk, double *smem, double &fl)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Rhs h = get_rhs(c, tk.a);
    const int r = tk.b;
    const DRBlk b = c.rblk[r];
    const int rk = __ldcg(c.rank + r);
    const double *Vb = r_V(c, r);
    int total = 1;
    if (h.cnt > 0) {
        total = 0;
        for (int q = 0; q < h.cnt; ++q) total += __ldcg(c.rank + c.solve_rhs[h.off + q]);
    }
    double *Pb = slot_alloc(c, tk.c, (int64_t)rk * total + 1);
    double **colp = (double **)smem;
    __shared__ int s_nk, s_total;
    __shared__ int s_rrk[SEG_RHS_MAX];
    __shared__ double *s_rvp[SEG_RHS_MAX];
    const int64_t co = b.col0 - h.row0;
    int k0 = 0;
    while (true) {
        if (h.cnt > 0 && h.cnt <= SEG_RHS_MAX) {
            // ranks and V bases of the right-hand-side blocks loaded in parallel (once per task)
            if (k0 == 0) {
                for (int q = threadIdx.x; q < h.cnt; q += NT) {
                    const int r = c.solve_rhs[h.off + q];
                    s_rrk[q] = __ldcg(c.rank + r);
                    s_rvp[q] = r_V(c, r);
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                int k = 0, nk = 0;
                for (int q = 0; q < h.cnt; ++q)
                    for (int j = 0; j < s_rrk[q]; ++j, ++k)
                        if (k >= k0 && nk < SEG_MAXCOL) colp[nk++] = s_rvp[q] + h.m * (int64_t)j;
                s_nk = nk;
                s_total = k;
            }
        } else if (threadIdx.x == 0) {
            int tot;
            s_nk = rhs_columns(c, h, k0, colp, &tot);
            s_total = tot;
        }
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
            if (lane == 0) __stcg(Pb + l + (int64_t)rk * (k0 + k), s);
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
    double *K = c.cores + (int64_t)tk.c * c.kcore * c.kcore;
    for (int pq = warp; pq < ra * rb; pq += NWARP) {
        int a = pq % ra, b = pq / ra;
        double s = 0.0;
        for (int64_t i = lane; i < m; i += 32) s += __ldcg(Va + i + m * a) * __ldcg(Vb + i + m * b);
        s = warp_sum(s);
        if (lane == 0) __stcg(K + a + (int64_t)c.kcore * b, s);
    }
    fl += 2.0 * m * ra * rb;
}

// Q_x = V_x^T V_p[cols of x] for every partner p (Q: rank_x x sum of partner ranks, ld rank_x)
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
    const int tot = partner_prefix(c, q, q.part_cnt);
    double *Q = slot_alloc(c, tk.c, (int64_t)rx * tot + 1);
    const int64_t co = bx.col0 - sig0;
    int pre = 0;
    for (int p = 0; p < q.part_cnt; ++p) {
        const int rp_id = c.col_r[q.part_off + p];
        const int rp = __ldcg(c.rank + rp_id);
        const double *Vp = r_V(c, rp_id);
        for (int pq = warp; pq < rx * rp; pq += NWARP) {
            const int l = pq % rx, k = pq / rx;
            double s = 0.0;
            for (int64_t i = lane; i < bx.m; i += 32) s += __ldcg(Vx + i + (int64_t)bx.m * l) * __ldcg(Vp + co + i + (int64_t)q.m * k);
            s = warp_sum(s);
            if (lane == 0) __stcg(Q + l + (int64_t)rx * (pre + k), s);
        }
        fl += 2.0 * bx.m * rx * rp;
        pre += rp;
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
    double *Xs = Ts + HCOV_TILE;              // 32 x rp (tile branch) or the rx x rp core slice
    double *Us = Xs + max(32 * (int64_t)max(32, c.kcap), (int64_t)c.kcap * c.kcap);   // 32 x rx
    const int tot = partner_prefix(c, q, q.part_cnt);
    double *Wq = w_acquire(c, tk.a, (int64_t)q.m * tot + 1);
    int pre = 0;
    for (int p = 0; p < q.part_cnt; ++p) {
        const int rp_id = c.col_r[q.part_off + p];
        const int rp = __ldcg(c.rank + rp_id);
        const double *Vp = r_V(c, rp_id);
        double *Wp = Wq + (int64_t)q.m * pre;
        pre += rp;
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
                const double *Qx = slot_get(c, ct.aux);
                const int64_t uo = i * HCOV_LEAF - bx.row0;
                for (int e = threadIdx.x; e < 32 * rx; e += NT) {
                    int rr = e & 31, l = e >> 5;
                    Us[e] = __ldcg(Ux + uo + rr + (int64_t)bx.m * l);
                }
                for (int e = threadIdx.x; e < rx * rp; e += NT) {
                    int l = e % rx, k = e / rx;
                    Xs[e] = __ldcg(Qx + l + (int64_t)rx * (pre - rp + k));
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

// ---------------------------------------------------------------------------------------------
// Root back-solve u = L~^{-T} v in place in vbuf (NEXT (f1); the transpose of the root forward
// solve).  Segment i: y = v_i - sum over the strictly-lower leaves over column i of
//   tile (rho, i):      T^T u_rho                  (kind 0, aux = rho)
//   low-rank b = U V^T: V_b[rows of i] t_b         (kind 1, t_b = U_b^T u[rows of b] from BPROJ)
// then u_i = L_ii^{-T} y.  Each warp accumulates a fixed subset of the contributions; the partial
// vectors are summed in warp order (deterministic).
__device__ void task_bseg(const Ctx &c, const DTask &tk, double *smem, double &fl)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = tk.b;
    double *part = smem;                          // NWARP x 32 partial sums
    double *Ts = part + 32 * NWARP;               // NWARP padded 32 x 33 tiles
    double *mine = Ts + (int64_t)warp * 32 * 33;
    double acc = 0.0;                             // this warp's partial, entry `lane`
    for (int z = tk.c + warp; z < tk.d; z += NWARP) {
        const DCtr ct = c.ctr[z];
        if (ct.kind == 0) {
            const double *T = c.tiles + (int64_t)ct.id * HCOV_TILE;
            const double *u = c.vbuf + (int64_t)ct.aux * HCOV_LEAF;
            for (int cc = 0; cc < 32; ++cc) mine[lane + 33 * cc] = __ldcg(T + lane + 32 * cc);   // coalesced
            const double ul = __ldcg(u + lane);
            __syncwarp();
            // (T^T u)[lane] = sum_rr T[rr, lane] u[rr]
            double s = 0.0;
#pragma unroll 8
            for (int rr = 0; rr < 32; ++rr) s = fma(mine[rr + 33 * lane], __shfl_sync(0xffffffffu, ul, rr), s);
            acc += s;
            __syncwarp();
            fl += 2.0 * 32 * 32;
        } else {
            const DRBlk b = c.rblk[ct.id];
            const int rk = __ldcg(c.rank + ct.id);
            const double *V = r_V(c, ct.id) + (i * HCOV_LEAF - b.col0) + lane;
            const double *t = c.tbuf + (int64_t)ct.id * c.kcap;
            double s = 0.0;
            for (int l = 0; l < rk; ++l) s = fma(__ldcg(V + (int64_t)b.m * l), __ldcg(t + l), s);
            acc += s;
            fl += 2.0 * 32 * rk;
        }
    }
    part[warp * 32 + lane] = acc;
    __syncthreads();
    if (warp == 0) {
        double y = __ldcg(c.vbuf + i * HCOV_LEAF + lane);
        for (int w = 0; w < NWARP; ++w) y -= part[w * 32 + lane];
        // L_ii^T u = y: u_a = y_a / L_aa for a = 31..0, then y_b -= L_ab u_a for b < a
        const double *L = c.tiles + (int64_t)c.diag_tile[i] * HCOV_TILE;
        for (int cc = 0; cc < 32; ++cc) mine[lane + 33 * cc] = __ldcg(L + lane + 32 * cc);
        __syncwarp();
        for (int a = 31; a >= 0; --a) {
            const double ua = __shfl_sync(0xffffffffu, y, a) / mine[a + 33 * a];
            if (lane == a) y = ua;
            else if (lane < a) y = fma(-mine[a + 33 * lane], ua, y);
        }
        __stcg(c.vbuf + i * HCOV_LEAF + lane, y);
        fl += 32.0 * 32;
    }
}

// t_b = U_b^T u[rows of b] (rank_b values into tbuf): one warp per column of U_b.
__device__ void task_bproj(const Ctx &c, const DTask &tk, double &fl)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = tk.b;
    const DRBlk b = c.rblk[r];
    const int rk = __ldcg(c.rank + r);
    const double *U = r_U(c, r);
    const double *u = c.vbuf + b.row0;
    for (int l = warp; l < rk; l += NWARP) {
        const double *ul = U + (int64_t)b.m * l;
        double s = 0.0;
        for (int64_t q = lane; q < b.m; q += 32) s = fma(__ldcg(ul + q), __ldcg(u + q), s);
        s = warp_sum(s);
        if (lane == 0) __stcg(c.tbuf + (int64_t)r * c.kcap + l, s);
    }
    fl += 2.0 * b.m * rk;
}

// shared memory (doubles) of the engine's task bodies
__host__ __device__ inline int64_t engine_smem_doubles(int kcap)
{
    int64_t a = tile_smem_doubles(kcap);
    int64_t k = kcap > 32 ? kcap : 32;
    int64_t b = 32 * SEG_MAXCOL + HCOV_TILE + k * SEG_MAXCOL + 32 * (int64_t)kcap + SEG_MAXCOL + 8;
    int64_t cc = 32 * (int64_t)kcap + HCOV_TILE + (32 * k > (int64_t)kcap * kcap ? 32 * k : (int64_t)kcap * kcap) +
                 32 * (int64_t)kcap + 8;   // task_phwr
    int64_t m = a > b ? a : b;
    m = m > cc ? m : cc;
    const int64_t floor_dbl = (NT >= 512) ? HCOV_SMEM_DBL : 0;   // one CTA per SM: panels resident in shared memory
    return m > floor_dbl ? m : floor_dbl;
}
