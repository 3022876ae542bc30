// libhcov: C ABI (include/hcov.h), the persistent DAG engine and its auxiliary kernels.
//
// One evaluation of L~(theta) (hcov_eval) is: a reset kernel, the permutation of Z, ONE
// persistent engine launch that executes the whole task DAG of the plan (assembly A3-A6,
// H-Cholesky A7, forward H-solve A9; plan.cpp), and a fixed-order reduction (A8, A10).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

#include "../../include/hcov.h"
#include "engine.cuh"
#include "plan.h"

namespace {

#define CK(x)                                                 \
    do {                                                      \
        cudaError_t e_ = (x);                                 \
        if (e_ != cudaSuccess) return map_err_at(e_, __LINE__); \
    } while (0)

static bool verbose()
{
    static int v = -1;
    if (v < 0) { const char *e = std::getenv("HCOV_VERBOSE"); v = (e && *e && *e != '0') ? 1 : 0; }
    return v == 1;
}

hcov_status map_err(cudaError_t e);
hcov_status map_err_at(cudaError_t e, int line)
{
    if (verbose()) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        std::fprintf(stderr, "hcov: hcov.cu:%d: CUDA error %d, device memory free %.2f of %.2f GB\n", line, (int)e,
                     fr / 1e9, tot / 1e9);
    }
    return map_err(e);
}

hcov_status map_err(cudaError_t e)
{
    if (verbose()) std::fprintf(stderr, "hcov: CUDA error %d (%s)\n", (int)e, cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) return HCOV_ERR_OUT_OF_MEMORY;
    return HCOV_ERR_CUDA;
}

template <class T>
cudaError_t upload(T **d, const std::vector<T> &h)
{
    size_t bytes = std::max<size_t>(1, h.size()) * sizeof(T);
    cudaError_t e = cudaMalloc((void **)d, bytes);
    if (e != cudaSuccess) return e;
    if (!h.empty()) e = cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

// ------------------------------------------------------------------------------------------
// instrumentation: launch counter, per-class CUDA-event timing, engine counters (hcov_prof_*)
// ------------------------------------------------------------------------------------------
enum ProfCls { PC_ENGINE = 0, PC_RESET = 1, PC_PERM = 2, PC_REDUCE = 3, PC_AUX = 4, PC_N = 5 };
const char *const PROF_NAMES[PC_N] = {"engine", "reset", "permute", "reduce", "aux"};
const char *const TASK_NAMES[TK_NTYPES] = {"fill", "aca", "tapp", "potrf", "trsm", "rapp", "seg",
                                           "proj", "prr", "phwp", "phwr", "nop", "bseg", "bproj"};
struct ProfEv { int cls; cudaEvent_t a, b; };
struct Prof {
    int64_t launches = 0;
    int64_t count[PC_N] = {};
    bool events = false;
    std::vector<ProfEv> evs;
    std::vector<cudaEvent_t> pool;
    double ms[PC_N] = {};
    double busy_ns[TK_NTYPES] = {};
    double tasks[TK_NTYPES] = {};
    double flop[FC_N] = {};
    double phase_ns[64] = {};
};
Prof g_prof;

cudaEvent_t prof_event()
{
    if (!g_prof.pool.empty()) { cudaEvent_t e = g_prof.pool.back(); g_prof.pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
int prof_begin(int cls, cudaStream_t st)
{
    g_prof.launches++;
    g_prof.count[cls]++;
    if (!g_prof.events) return -1;
    ProfEv p{cls, prof_event(), prof_event()};
    cudaEventRecord(p.a, st);
    g_prof.evs.push_back(p);
    return (int)g_prof.evs.size() - 1;
}
void prof_end(int k, cudaStream_t st)
{
    if (k >= 0) cudaEventRecord(g_prof.evs[k].b, st);
}
void prof_collect()
{
    for (ProfEv &p : g_prof.evs) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess)
            g_prof.ms[p.cls] += ms;
        g_prof.pool.push_back(p.a);
        g_prof.pool.push_back(p.b);
    }
    g_prof.evs.clear();
}
#define LAUNCH(cls, st, ...)                     \
    do {                                         \
        int pk_ = prof_begin((cls), (st));       \
        __VA_ARGS__;                             \
        prof_end(pk_, (st));                     \
    } while (0)

// ------------------------------------------------------------------------------------------
// engine
// ------------------------------------------------------------------------------------------
struct EngineStats {
    unsigned long long busy_ns[TK_NTYPES];
    unsigned long long tasks[TK_NTYPES];
    double flop[FC_N];
};

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int ld_volatile(const int32_t *p) { return *(volatile const int32_t *)p; }
__device__ __forceinline__ uint4 ld_volatile_v4(const uint32_t *p)
{
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}


// Queue entries: (global task id << QE_SHIFT) | gang member, global task id = instance * ntasks +
// task (an engine launch runs the DAGs of c.ninst H-matrices of the same tree: a theta batch).  A
// gang task of G CTAs occupies G consecutive entries.  Band b of the ring holds ninst x its
// per-instance capacity.
#define QE_SHIFT 3
__device__ __forceinline__ void push_ready(const Ctx &c, int32_t inst, int32_t s)
{
    const int b = c.tasks[s].band;
    const int G = max(1, c.tasks[s].qcls);
    const uint32_t pos = atomicAdd(c.qctl + QC_BTAIL + b, (uint32_t)G);
    int32_t *q = c.queue[0] + (int64_t)c.band_off[b] * c.ninst + pos;
    const int32_t e0 = (inst * c.ntasks + s) << QE_SHIFT;
    for (int g = 0; g < G; ++g) atomicExch(q + g, e0 + g);
}

// Release the successors of task t of instance inst (all threads of the CTA; NOP joins complete
// inline).  c: the instance's context (its in-degrees).
__device__ void release(const Ctx &c, int32_t inst, int32_t t, int mask, const int8_t *phase)
{
    const int b = c.succ_off[t], e = c.succ_off[t + 1];
    for (int k = b + threadIdx.x; k < e; k += blockDim.x) {
        int32_t s = c.succ[k];
        if (!(mask & (1 << phase[s]))) continue;
        if (atomicSub(c.indeg + s, 1) != 1) continue;
        int32_t stack[24];
        int sp = 0;
        stack[sp++] = s;
        while (sp > 0) {
            int32_t u = stack[--sp];
            if (c.tasks[u].type != TK_NOP) { push_ready(c, inst, u); continue; }
            __threadfence();
            for (int z = c.succ_off[u]; z < c.succ_off[u + 1]; ++z) {
                int32_t v = c.succ[z];
                if (!(mask & (1 << phase[v]))) continue;
                if (atomicSub(c.indeg + v, 1) == 1) {
                    if (sp < 24) stack[sp++] = v;
                    else push_ready(c, inst, v);
                }
            }
        }
    }
}

// The persistent engine: every CTA claims the head entry of the most urgent non-empty band, runs
// the task with its instance's context (copied to shared memory), releases the successors.
// c: engine-level fields (queue, control words, scratch; identical in every instance context);
// ictx[i]: the full context of instance i.
__global__ void __launch_bounds__(NT, 512 / NT) k_engine(Ctx c, const Ctx *__restrict__ ictx, int mask,
                                                         const int8_t *phase, EngineStats *stats,
                                                         unsigned long long *tl)
{
    extern __shared__ double smem[];
    __shared__ double red[NWARP], redv[NWARP];
    __shared__ int64_t redi[NWARP];
    __shared__ int32_t s_entry;
    __shared__ Ctx s_ctx;
    double *scr = c.scr + (int64_t)blockIdx.x * c.scr_stride;
    double fl[FC_N] = {0, 0, 0, 0, 0};
    unsigned long long busy[TK_NTYPES] = {}, cnt[TK_NTYPES] = {};
    const int ninst = c.ninst;
    while (true) {
        if (threadIdx.x == 0) {
            int32_t v = -1;
            const unsigned long long t0 = gtimer();
            unsigned ns = 32;
            // take the head of the most urgent non-empty band (try-claim by CAS)
            while (true) {
                if (ld_volatile((const int32_t *)c.qctl + QC_DONE0) >= c.nq[0]) break;
                if (ld_volatile((const int32_t *)c.qctl + QC_ABORT)) break;
                bool got = false;
                // one pass of independent 16-byte loads over the band heads and tails (the per-band
                // head -> entry chain of dependent L2 loads made an idle scan ~16 x 2 L2 latencies)
                static_assert(HCOV_BANDS == 16, "vectorised band scan");
                unsigned nonempty = 0;
                {
                    uint4 hv[4], tv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) hv[i] = ld_volatile_v4(c.qctl + QC_BHEAD + 4 * i);
#pragma unroll
                    for (int i = 0; i < 4; ++i) tv[i] = ld_volatile_v4(c.qctl + QC_BTAIL + 4 * i);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        nonempty |= (hv[i].x < tv[i].x ? 1u : 0u) << (4 * i);
                        nonempty |= (hv[i].y < tv[i].y ? 1u : 0u) << (4 * i + 1);
                        nonempty |= (hv[i].z < tv[i].z ? 1u : 0u) << (4 * i + 2);
                        nonempty |= (hv[i].w < tv[i].w ? 1u : 0u) << (4 * i + 3);
                    }
                }
                while (nonempty && !got) {
                    const int b = 31 - __clz(nonempty);
                    nonempty &= ~(1u << b);
                    const int64_t base = (int64_t)c.band_off[b] * ninst;
                    const uint32_t cap = (uint32_t)((c.band_off[b + 1] - c.band_off[b]) * ninst);
                    while (true) {
                        const uint32_t h = (uint32_t)ld_volatile((const int32_t *)c.qctl + QC_BHEAD + b);
                        if (h >= cap) break;
                        const int32_t e = ld_volatile(c.queue[0] + base + h);
                        if (e < 0) break;
                        if (atomicCAS(c.qctl + QC_BHEAD + b, h, h + 1) == h) { v = e; got = true; break; }
                    }
                }
                if (got) break;
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
                if (gtimer() - t0 > c.timeout_ns) { atomicExch(c.qctl + QC_ABORT, 1u); break; }
            }
            __threadfence();
            s_entry = v;
        }
        __syncthreads();
        const int32_t v = s_entry;
        if (v < 0) break;
        const int32_t gt = v >> QE_SHIFT, member = v & ((1 << QE_SHIFT) - 1);
        const int32_t inst = gt / c.ntasks, t = gt - inst * c.ntasks;
        {
            const unsigned long long *src = (const unsigned long long *)(ictx + inst);
            unsigned long long *dst = (unsigned long long *)&s_ctx;
            for (int k = threadIdx.x; k < (int)(sizeof(Ctx) / 8); k += NT) dst[k] = __ldg(src + k);
        }
        __syncthreads();
        const Ctx &ci = s_ctx;
        const DTask tk = c.tasks[t];
        Gang gang{member, tk.qcls, ci.gbar + t, c.qctl + QC_ABORT, 0, 0, 0, nullptr, tk.type == TK_RAPP && tk.pad == 1,
                  -1, member, tk.qcls};
        Gang *gg = nullptr;
        double *tscr = scr;
        bool use_big = false;
        __shared__ int32_t s_bgrp;
        if (tk.qcls > 0) {
            // member 0 (the first entry of the gang) lends the shared workspace of its scratch
            __shared__ int32_t s_cta0;
            if (threadIdx.x == 0) {
                if (gang.g == 0) {
                    atomicExch(ci.gslot + t, (int32_t)blockIdx.x);
                    s_cta0 = blockIdx.x;
                } else {
                    int32_t w;
                    while ((w = ld_volatile(ci.gslot + t)) < 0) {
                        if (ld_volatile((const int32_t *)c.qctl + QC_ABORT)) break;
                        __nanosleep(64);
                    }
                    if (w < 0) w = blockIdx.x;   // aborted: the task body exits at its first gang barrier
                    s_cta0 = w;
                }
                __threadfence();
            }
            __syncthreads();
            gg = &gang;
            gang.shared = c.scr + (int64_t)s_cta0 * c.scr_stride + c.gshared_off;
            // members with more rows than the per-CTA scratch holds take a slot of a big-member
            // group: once the gang has formed (all members present), member 0 claims a free group
            // (only formed gangs hold groups, so a waiting gang never blocks the holder); member g
            // uses slot g of it.  Released by member 0 after the task body (every member has passed
            // the body's last gang barrier by then).
            if (c.n_bgrp > 0 && (tk.type == TK_ACA || tk.type == TK_RAPP)) {
                const int64_t m = c.rblk[tk.a].m;
                const int Gs = gang.split ? tk.qcls / 2 : tk.qcls;
                const int64_t mq_last = m - (int64_t)(Gs - 1) * (m / Gs);
                if (mq_last > c.big_mq) {
                    gang_sync(gang);
                    if (gang.g == 0 && threadIdx.x == 0) {
                        int k = -1;
                        unsigned ns = 64;
                        const unsigned long long tw0 = gtimer();
                        while (k < 0) {
                            for (int q = 0; q < c.n_bgrp && k < 0; ++q)
                                if (atomicCAS(c.bgrp_busy + q, 0, 1) == 0) k = q;
                            if (k >= 0) break;
                            if (ld_volatile((const int32_t *)c.qctl + QC_ABORT)) { k = 0; break; }
                            if (gtimer() - tw0 > c.timeout_ns) { atomicExch(c.qctl + QC_ABORT, 1u); k = 0; break; }
                            __nanosleep(ns);
                            if (ns < 1024) ns <<= 1;
                        }
                        __stcg(c.bgrp_cta + blockIdx.x, k);
                        s_bgrp = k;
                    }
                    gang_sync(gang);
                    if (threadIdx.x == 0) s_bgrp = __ldcg(c.bgrp_cta + s_cta0);
                    __syncthreads();
                    tscr = c.bscr + ((int64_t)s_bgrp * HCOV_GANG + gang.g) * c.bscr_stride;
                    use_big = true;
                }
            }
        }
        const unsigned long long t0 = gtimer();
        if (threadIdx.x == 0) {
            int pc = 0;
            if (tk.type == TK_RAPP || tk.type == TK_ACA) {
                const int64_t m = c.rblk[tk.a].m;
                pc = m <= 64 ? 0 : m <= 256 ? 1 : m <= 1024 ? 2 : 3;
            }
            s_phase_cls = pc;
        }
        __syncthreads();
        // flop counters of this task in call-local scalars (registers; an element of fl[] passed by
        // reference was reloaded and stored through local memory in every inner-loop iteration)
        double f1 = 0.0, f2 = 0.0;
        int c1 = FC_ASM, c2 = FC_TRUNC;
        switch (tk.type) {
        case TK_FILL: task_fill(ci, tk, f1); break;
        case TK_ACA: task_aca(ci, tk, tscr, smem, red, redv, redi, f1, f2, gg); break;
        case TK_TAPP:
        case TK_POTRF:
        case TK_TRSM: task_tile(ci, tk, smem, f1); c1 = FC_TILE; break;
        case TK_RAPP: task_rapp(ci, tk, tscr, smem, red, redv, redi, f1, gg); c1 = FC_TRUNC; break;
        case TK_SEG: task_seg(ci, tk, smem, f1); c1 = FC_SOLVE; break;
        case TK_PROJ: task_proj(ci, tk, smem, f1); c1 = FC_SOLVE; break;
        case TK_PRR: task_prr(ci, tk, f1); c1 = FC_PROD; break;
        case TK_PHWP: task_phwp(ci, tk, f1); c1 = FC_PROD; break;
        case TK_PHWR: task_phwr(ci, tk, smem, f1); c1 = FC_PROD; break;
        case TK_BSEG: task_bseg(ci, tk, smem, f1); c1 = FC_SOLVE; break;
        case TK_BPROJ: task_bproj(ci, tk, f1); c1 = FC_SOLVE; break;
        default: break;
        }
        if (threadIdx.x == 0) {
            for (int k = 0; k < FC_N; ++k) {
                if (k == c1) fl[k] += f1;
                if (k == c2 && tk.type == TK_ACA) fl[k] += f2;
            }
        }
        __threadfence();
        __syncthreads();
        if (use_big && gang.g == 0 && threadIdx.x == 0) atomicExch(c.bgrp_busy + s_bgrp, 0);
        if (gang.g == 0) {
            if (threadIdx.x == 0) {
                const unsigned long long t1 = gtimer();
                busy[tk.type] += t1 - t0;
                cnt[tk.type] += 1;
                if (tl && ninst == 1) { tl[3 * (int64_t)t] = t0; tl[3 * (int64_t)t + 1] = t1; tl[3 * (int64_t)t + 2] = blockIdx.x; }
            }
            release(ci, inst, t, mask, phase);
            __syncthreads();
            if (threadIdx.x == 0) { __threadfence(); atomicAdd(c.qctl + QC_DONE0, 1u); }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && stats) {
        for (int k = 0; k < TK_NTYPES; ++k) {
            if (cnt[k]) {
                atomicAdd(stats->busy_ns + k, busy[k]);
                atomicAdd(stats->tasks + k, cnt[k]);
            }
        }
        for (int k = 0; k < FC_N; ++k)
            if (fl[k] != 0.0) atomicAdd(stats->flop + k, fl[k]);
    }
}

// Per instance: working in-degrees of the mode, gang barriers and member-0 slots.
__global__ void k_reset_inst(Ctx c, const int32_t *indeg_mode, int64_t ntasks)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntasks; k += stride) {
        c.indeg[k] = indeg_mode[k];
        c.gbar[k] = 0;
        c.gslot[k] = -1;
    }
}

// The batch's ready queue: band b holds, for instance 0, 1, ..., the mode's initially ready entries
// of the band (q0init, plan order), then -1; control words reset (band tails = ninst x initial).
__global__ void k_qinit(Ctx c, const int32_t *q0init, const int32_t *q0tail)
{
    const int ninst = c.ninst;
    const int64_t total = (int64_t)c.band_off[HCOV_BANDS] * ninst;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t p = tid; p < total; p += stride) {
        int b = 0;
        while (b + 1 < HCOV_BANDS && (int64_t)c.band_off[b + 1] * ninst <= p) ++b;
        const int64_t local = p - (int64_t)c.band_off[b] * ninst;
        const int64_t qt = q0tail[b];
        int32_t e = -1;
        if (local < qt * ninst) {
            const int64_t inst = local / qt, k = local - inst * qt;
            const int32_t v = q0init[c.band_off[b] + k];   // plan entries: task * 32 + member
            e = (int32_t)(((inst * c.ntasks + (v >> 5)) << QE_SHIFT) | (v & 31));
        }
        c.queue[0][p] = e;
    }
    if (tid < QC_N) {
        uint32_t v = 0;
        if (tid >= QC_BTAIL && tid < QC_BTAIL + HCOV_BANDS) v = (uint32_t)(q0tail[tid - QC_BTAIL] * ninst);
        c.qctl[tid] = v;
    }
}

__global__ void k_permute_in(Ctx c, const double *Zext, double *y)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < c.n_pad; p += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = c.perm_i2e[p];
        y[p] = (e >= 0) ? Zext[e] : 0.0;
    }
}
__global__ void k_permute_out(Ctx c, const double *y, double *Zext)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < c.n_pad; p += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = c.perm_i2e[p];
        if (e >= 0) Zext[e] = y[p];
    }
}

// Point-wise LDL^T read-out (NEXT (f4)): D_e = L~_pp^2 for the internal position p of point e
// (the diagonal of the factor's diagonal leaf tiles, col-major 32 x 32).
__global__ void k_ldl_diag(Ctx c, double *Dext)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < c.n_pad; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = c.perm_i2e[p];
        if (e < 0) continue;
        const int64_t leaf = p / HCOV_LEAF, i = p % HCOV_LEAF;
        const double l = c.tiles[(int64_t)c.diag_tile[leaf] * HCOV_TILE + i + HCOV_LEAF * i];
        Dext[e] = l * l;
    }
}

// out[0] = log det, out[1] = quad, out[2] = min pivot (fixed-order reductions, one CTA)
__global__ void __launch_bounds__(NT) k_reduce(Ctx c, double *out)
{
    __shared__ double red[NWARP];
    __shared__ double mred[NT];
    double ld = 0.0, q = 0.0, mp = INFINITY;
    for (int64_t k = threadIdx.x; k < c.n_leaves; k += NT) {
        ld += c.logdet_part[k];
        q += c.quad_part[k];
        mp = fmin(mp, c.minpiv_part[k]);
    }
    ld = block_sum(ld, red);
    q = block_sum(q, red);
    mred[threadIdx.x] = mp;
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = INFINITY;
        for (int k = 0; k < NT; ++k) x = fmin(x, mred[k]);
        out[0] = 2.0 * ld;
        out[1] = q;
        out[2] = x;
    }
}

// Per-theta K_nu Chebyshev table (general nu, matern.cuh): one thread per interval.
__global__ void k_ktab(double nu, double *coef)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < KTAB_NI) hcov_matern_table_row(nu, i, coef + i * KTAB_NC);
}

// hcov_sample: t_b = V_b^T x[cols of b] for every R block
__global__ void __launch_bounds__(NT) k_sample_t(Ctx c, const double *x, double *t)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = blockIdx.x; r < c.n_r; r += gridDim.x) {
        const DRBlk b = c.rblk[r];
        const int rk = c.rank[r];
        const double *V = r_V(c, r);
        for (int l = warp; l < rk; l += NWARP) {
            double s = 0.0;
            for (int64_t i = lane; i < b.m; i += 32) s += V[i + b.m * l] * x[b.col0 + i];
            s = warp_sum(s);
            if (lane == 0) t[(int64_t)r * c.kcap + l] = s;
        }
    }
}
// y_seg = sum over the row's lower-triangular leaves (T: tile x_cols; R: U[seg rows] t_b)
__global__ void __launch_bounds__(32) k_sample_rows(Ctx c, const int32_t *row_off, const int32_t *row_nodes,
                                                    const double *x, const double *t, double *y)
{
    for (int64_t seg = blockIdx.x; seg < c.n_leaves; seg += gridDim.x) {
        const int i = threadIdx.x;
        double s = 0.0;
        for (int k = row_off[seg]; k < row_off[seg + 1]; ++k) {
            const DNode nd = c.nodes[row_nodes[k]];
            if (nd.type == ND_T) {
                const double *T = c.tiles + (int64_t)nd.idx * HCOV_TILE;
                const int64_t c0 = (int64_t)nd.j * HCOV_LEAF;
                for (int j = 0; j < 32; ++j) s += T[i + 32 * j] * x[c0 + j];
            } else {
                const DRBlk b = c.rblk[nd.idx];
                const int rk = c.rank[nd.idx];
                const double *U = r_U(c, nd.idx);
                const int64_t ro = seg * HCOV_LEAF - b.row0 + i;
                for (int l = 0; l < rk; ++l) s += U[ro + b.m * l] * t[(int64_t)nd.idx * c.kcap + l];
            }
        }
        y[seg * HCOV_LEAF + i] = s;
    }
}

// hcov_columns: out (n_pad x m internal rows) for internal columns pc[k] of the assembled C~.
__global__ void __launch_bounds__(NT) k_columns(Ctx c, const int32_t *leafnodes, int nleafnodes, const int64_t *pc,
                                                int mcols, double *out)
{
    for (int q = blockIdx.x; q < nleafnodes; q += gridDim.x) {
        const DNode nd = c.nodes[leafnodes[q]];
        const int64_t mb = cl_size(c, nd.level);
        const int64_t r0 = (int64_t)nd.i * mb, c0 = (int64_t)nd.j * mb;
        for (int k = 0; k < mcols; ++k) {
            const int64_t p = pc[k];
            double *o = out + c.n_pad * (int64_t)k;
            if (p >= c0 && p < c0 + mb) {
                const int64_t jj = p - c0;
                for (int64_t i = threadIdx.x; i < mb; i += NT) {
                    double v;
                    if (nd.type == ND_T) v = c.tiles[(int64_t)nd.idx * HCOV_TILE + i + 32 * jj];
                    else {
                        const int rk = c.rank[nd.idx];
                        const double *U = r_U(c, nd.idx), *V = r_V(c, nd.idx);
                        v = 0.0;
                        for (int l = 0; l < rk; ++l) v += U[i + mb * l] * V[jj + mb * l];
                    }
                    o[r0 + i] = v;
                }
            }
            if (nd.i != nd.j && p >= r0 && p < r0 + mb) {
                const int64_t ii = p - r0;
                for (int64_t j = threadIdx.x; j < mb; j += NT) {
                    double v;
                    if (nd.type == ND_T) v = c.tiles[(int64_t)nd.idx * HCOV_TILE + ii + 32 * j];
                    else {
                        const int rk = c.rank[nd.idx];
                        const double *U = r_U(c, nd.idx), *V = r_V(c, nd.idx);
                        v = 0.0;
                        for (int l = 0; l < rk; ++l) v += U[ii + mb * l] * V[j + mb * l];
                    }
                    o[c0 + j] = v;
                }
            }
        }
    }
}
// hcov_cov_columns: exact Eq. (3) columns C e_j (direct K_nu, no table), external row order.
__global__ void k_cov_columns(Ctx c, const int64_t *pc, int mcols, double *out)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c.n_pad * (int64_t)mcols;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = e % c.n_pad, k = e / c.n_pad;
        const int64_t ex = c.perm_i2e[p];
        if (ex < 0) continue;
        const int64_t q = pc[k];
        out[ex + c.n_real * k] = pts_cov(c.mp, Pts{c.xs, c.ys, c.zs}, p, q);
    }
}

__global__ void k_columns_perm(Ctx c, const double *in, int mcols, double *out)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c.n_pad * (int64_t)mcols;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = e % c.n_pad, k = e / c.n_pad;
        int64_t ex = c.perm_i2e[p];
        if (ex >= 0) out[ex + c.n_real * k] = in[e];
    }
}

// ---- H-matvec y = C~ x of an assembled H-matrix (Table 1 row "C~ z"), internal order.
// k_mv_t: per low-rank block, t1_b = V_b^T x[cols of b], t2_b = U_b^T x[rows of b].
__global__ void __launch_bounds__(NT) k_mv_t(Ctx c, const double *x, double *t1, double *t2)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = blockIdx.x; r < c.n_r; r += gridDim.x) {
        const DRBlk b = c.rblk[r];
        const int rk = c.rank[r];
        const double *U = r_U(c, r), *V = r_V(c, r);
        for (int q = warp; q < 2 * rk; q += NWARP) {
            const int l = q % rk;
            const bool tv = q < rk;
            const double *F = (tv ? V : U) + (int64_t)b.m * l;
            const double *xx = x + (tv ? b.col0 : b.row0);
            double s = 0.0;
            for (int64_t i = lane; i < b.m; i += 32) s = fma(F[i], xx[i], s);
            s = warp_sum(s);
            if (lane == 0) (tv ? t1 : t2)[(int64_t)r * c.kcap + l] = s;
        }
    }
}
// k_mv_rows: one warp per leaf segment i, lane = row: y_i = sum over the leaves of row i (T x_j,
// U_b[i] t1_b) + sum over the strictly-lower leaves of column i (T^T x_rho, V_b[i] t2_b), in the
// fixed CSR order (deterministic).  The symmetric upper triangle is the mirror (Remark 1, R10).
__global__ void __launch_bounds__(256) k_mv_rows(Ctx c, const int32_t *row_off, const int32_t *row_nodes,
                                                 const int32_t *col_off, const int32_t *col_nodes, const double *x,
                                                 const double *t1, const double *t2, double *y)
{
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t seg = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); seg < c.n_leaves; seg += nw) {
        double s = 0.0;
        for (int k = row_off[seg]; k < row_off[seg + 1]; ++k) {
            const DNode nd = c.nodes[row_nodes[k]];
            if (nd.type == ND_T) {
                const double *T = c.tiles + (int64_t)nd.idx * HCOV_TILE + lane;
                const double *xx = x + (int64_t)nd.j * HCOV_LEAF;
                for (int j = 0; j < 32; ++j) s = fma(T[32 * j], xx[j], s);
            } else {
                const DRBlk b = c.rblk[nd.idx];
                const int rk = c.rank[nd.idx];
                const double *U = r_U(c, nd.idx) + (seg * HCOV_LEAF - b.row0 + lane);
                const double *t = t1 + (int64_t)nd.idx * c.kcap;
                for (int l = 0; l < rk; ++l) s = fma(U[(int64_t)b.m * l], t[l], s);
            }
        }
        for (int k = col_off[seg]; k < col_off[seg + 1]; ++k) {
            const DNode nd = c.nodes[col_nodes[k]];
            if (nd.type == ND_T) {
                const double *T = c.tiles + (int64_t)nd.idx * HCOV_TILE + 32 * lane;
                const double *xx = x + (int64_t)nd.i * HCOV_LEAF;
                for (int j = 0; j < 32; ++j) s = fma(T[j], xx[j], s);
            } else {
                const DRBlk b = c.rblk[nd.idx];
                const int rk = c.rank[nd.idx];
                const double *V = r_V(c, nd.idx) + (seg * HCOV_LEAF - b.col0 + lane);
                const double *t = t2 + (int64_t)nd.idx * c.kcap;
                for (int l = 0; l < rk; ++l) s = fma(V[(int64_t)b.m * l], t[l], s);
            }
        }
        y[seg * HCOV_LEAF + lane] = s;
    }
}

// ---- vector kernels of the PCG (external order).  Dot products in a fixed order: 148 x 256 partials
// (grid-stride, fixed assignment), then one CTA sums them in index order.
#define DOT_BLOCKS 148
__global__ void __launch_bounds__(256) k_dot_part(const double *a, const double *b, int64_t n, double *part)
{
    __shared__ double red[8];
    double s = 0.0;
    for (int64_t k = blockIdx.x * 256 + threadIdx.x; k < n; k += (int64_t)DOT_BLOCKS * 256) s = fma(a[k], b[k], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}
__global__ void k_dot_sum(const double *part, double *out)
{
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < DOT_BLOCKS; ++k) t += part[k];
        *out = t;
    }
}
// y = a x + b y
__global__ void k_axpby(int64_t n, double a, const double *x, double b, double *y)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        y[k] = fma(a, x[k], b * y[k]);
}

// Unit-test kernel for the truncation (A6): one CTA truncates X Y^T (m x m, R columns).
__global__ void __launch_bounds__(NT) k_test_truncate(double *scr, int64_t m, int R, int K, double eps, int kmax,
                                                      int rlim, int path, double *U, double *V, int *rank,
                                                      int64_t smem_dbl, const double *Xin, const double *Yin)
{
    extern __shared__ double smem[];
    __shared__ double red[NWARP], redv[NWARP];
    __shared__ int64_t redi[NWARP];
    double *X2, *Y2;
    int cb = 0, of = 0;
    if (path == 3) {
        // the dense-mode pipeline of a small low-rank block (task_rapp, m <= HCOV_DENSE_MAX): S = X Y^T
        // formed densely (in shared memory when it leaves the GEMM staging room), fully pivoted cross
        // approximation to 0.1 eps, then the shared-memory truncation path
        const bool s_sm = m * m + 32 * 256 <= smem_dbl;
        double *S = s_sm ? smem : scr;
        CompressWs w = make_ws(scr + m * m, m, K, &X2, &Y2);
        for (int64_t e = threadIdx.x; e < m * m; e += NT) {
            const int64_t i = e % m, j = e / m;
            double a = 0.0;
            for (int l = 0; l < R; ++l) a = fma(Xin[i + m * l], Yin[j + m * l], a);
            S[e] = a;
        }
        __syncthreads();
        const int KA = (int)(m < K ? m : K);
        const int k = aca_full(S, m, w.X, w.Y, KA, 0.1 * eps / (double)m, 0.1 * eps, red, redv, redi);
        const int r = compress(w, m, k, eps, final_tol(eps, k), true, kmax, rlim, U, V, m, &cb, &of, red, redv, redi,
                               smem, smem_dbl, 2);
        if (threadIdx.x == 0) { rank[0] = r; rank[1] = cb; rank[2] = of; }
        return;
    }
    CompressWs w = make_ws(scr, m, K, &X2, &Y2);
    const int r = compress(w, m, R, eps, final_tol(eps, R), true, kmax, rlim, U, V, m, &cb, &of, red, redv, redi,
                           path >= 1 ? smem : nullptr, smem_dbl, path);
    if (threadIdx.x == 0) { rank[0] = r; rank[1] = cb; rank[2] = of; }
}

}  // namespace

// ------------------------------------------------------------------------------------------
// handles
// ------------------------------------------------------------------------------------------
// Engine resources shared by every H-matrix of a tree (one persistent launch at a time per tree):
// per-CTA scratch, big-member groups, the ready queue and control words, the per-instance
// context array of a batched launch, statistics.
struct Engine {
    int kcap = -1, grid = 0, ninst_cap = 0, nbg = 0;
    int64_t smem = 0, scr_stride = 0, bstride = 0, gshared_off = 0;
    double *scr = nullptr, *bscr = nullptr;
    int32_t *bgrp = nullptr, *q0 = nullptr, *q1 = nullptr;
    uint32_t *qctl = nullptr;
    Ctx *d_ctx = nullptr;
    EngineStats *stats = nullptr, *stats_host = nullptr;
    void release()
    {
        void *ps[] = {scr, bscr, bgrp, q0, q1, qctl, d_ctx, stats};
        for (void *p : ps) cudaFree(p);
        if (stats_host) cudaFreeHost(stats_host);
        scr = bscr = nullptr;
        bgrp = q0 = q1 = nullptr;
        qctl = nullptr;
        d_ctx = nullptr;
        stats = stats_host = nullptr;
        kcap = -1;
        ninst_cap = 0;
    }
};

struct hcov_tree_s {
    Plan P;
    bool uploaded = false;
    bool tree_on_device = false;             // A1 / A2 built by tree.cu's kernels
    double geo_ms = 0.0;                     // wall time of A1 + A2
    DNode *d_nodes = nullptr;
    int32_t *d_tile_node = nullptr;
    DRBlk *d_rblk = nullptr;
    DTerm *d_terms = nullptr;
    int32_t *d_xterm = nullptr;
    int64_t *d_fac_row0 = nullptr;
    int32_t *d_fac_nrows = nullptr, *d_fac_rank_src = nullptr;
    int64_t *d_fac_off = nullptr;
    int8_t *d_fac_pool = nullptr;
    DSolve *d_solves = nullptr;
    int32_t *d_solve_rhs = nullptr;
    DSlot *d_slots = nullptr;
    DCtr *d_ctr = nullptr;
    DPhw *d_phw = nullptr;
    int32_t *d_col_r = nullptr;
    DTask *d_tasks = nullptr;
    int8_t *d_phase = nullptr;
    int32_t *d_succ_off = nullptr, *d_succ = nullptr;
    int32_t *d_indeg[HCOV_MODES] = {};
    int32_t *d_roots[HCOV_MODES][2] = {};
    int32_t *d_q0init[HCOV_MODES] = {}, *d_q0tail[HCOV_MODES] = {};
    int32_t *d_col_off = nullptr, *d_col_nodes = nullptr;
    int32_t *d_band_off = nullptr;
    int32_t *d_diag_tile = nullptr;
    double *d_xs = nullptr, *d_ys = nullptr, *d_zs = nullptr;   // d_zs: 3-D variant only
    int64_t *d_perm_i2e = nullptr;
    int32_t *d_leafnodes = nullptr;
    int32_t n_leafnodes = 0;
    int32_t *d_row_off = nullptr, *d_row_nodes = nullptr;
    Engine eng;
    hcov_hmat cached = nullptr;              // instance 0 of hcov_eval / hcov_mle_batch
    std::vector<hcov_hmat> extra;            // instances 1.. of the last theta batch
    // W / product-slot words used by the most demanding run so far at capacity est_kcap (per-instance
    // pool sizing of theta batches)
    int est_kcap = -1, est_kmax = -1;
    double est_eps = -1.0;
    int64_t est_w = 0, est_p = 0;
    ~hcov_tree_s();
};

struct hcov_hmat_s {
    hcov_tree t = nullptr;
    Ctx ctx{};
    hcov_theta theta{};
    hcov_trunc trunc{};
    int state = 0;   // 1 assembled, 2 factored, 3 solved
    int kcap_alloc = -1, kcore_alloc = -1;
    double *tiles = nullptr, *U = nullptr, *V = nullptr, *cores = nullptr, *W = nullptr, *P = nullptr;
    double *vbuf = nullptr, *tbuf = nullptr, *logdet_part = nullptr, *minpiv_part = nullptr, *quad_part = nullptr;
    int32_t *rank = nullptr, *fail = nullptr, *flags = nullptr;
    int32_t *indeg = nullptr, *gbar = nullptr, *gslot = nullptr;
    double *res = nullptr, *res_host = nullptr;
    double *ktab = nullptr;
    int64_t *woff = nullptr, *poff = nullptr;
    unsigned long long *mem = nullptr;
    int64_t wcap = 0, pcap = 0;
    int64_t w_budget = 0, p_budget = 0;   // > 0: pool sizes (words) fixed by a theta batch
    void release_pools()
    {
        cudaFree(W);
        cudaFree(P);
        W = P = nullptr;
        wcap = pcap = 0;
        ctx.W = ctx.P = nullptr;
        ctx.wcap = ctx.pcap = 0;
    }
    void release_all()
    {
        release_pools();
        void *ps[] = {tiles, U, V, cores, vbuf, tbuf, logdet_part, minpiv_part, quad_part, rank, fail, flags,
                      indeg, gbar, gslot, res, woff, poff, mem};
        for (void *p : ps) cudaFree(p);
        tiles = U = V = cores = vbuf = tbuf = logdet_part = minpiv_part = quad_part = nullptr;
        rank = fail = flags = indeg = gbar = gslot = nullptr;
        res = nullptr;
        woff = poff = nullptr;
        mem = nullptr;
        kcap_alloc = -1;
    }
    ~hcov_hmat_s()
    {
        release_all();
        cudaFree(ktab);
        if (res_host) cudaFreeHost(res_host);
    }
};

hcov_tree_s::~hcov_tree_s()
{
    if (cached) delete cached;
    for (hcov_hmat h : extra) delete h;
    eng.release();
    void *ps[] = {d_nodes, d_tile_node, d_rblk, d_terms, d_xterm, d_fac_row0, d_fac_nrows, d_fac_rank_src,
                  d_fac_off, d_fac_pool, d_solves, d_solve_rhs, d_slots, d_ctr, d_phw, d_col_r, d_tasks, d_phase,
                  d_succ_off, d_succ, d_diag_tile, d_xs, d_ys, d_zs, d_perm_i2e, d_leafnodes, d_row_off, d_row_nodes,
                  d_col_off, d_col_nodes};
    for (void *p : ps) cudaFree(p);
    for (int m = 0; m < HCOV_MODES; ++m) {
        cudaFree(d_indeg[m]);
        cudaFree(d_roots[m][0]);
        cudaFree(d_roots[m][1]);
        cudaFree(d_q0init[m]);
        cudaFree(d_q0tail[m]);
    }
    cudaFree(d_band_off);
}

namespace {


hcov_status tree_upload(hcov_tree t)
{
    if (t->uploaded) return HCOV_OK;
    Plan &P = t->P;
    CK(upload(&t->d_nodes, P.nodes));
    CK(upload(&t->d_tile_node, P.tile_node));
    CK(upload(&t->d_rblk, P.rblk));
    CK(upload(&t->d_terms, P.terms));
    CK(upload(&t->d_xterm, P.xterm));
    CK(upload(&t->d_fac_row0, P.fac_row0));
    CK(upload(&t->d_fac_nrows, P.fac_nrows));
    CK(upload(&t->d_fac_rank_src, P.fac_rank_src));
    CK(upload(&t->d_fac_off, P.fac_off));
    CK(upload(&t->d_fac_pool, P.fac_pool));
    CK(upload(&t->d_solves, P.solves));
    CK(upload(&t->d_solve_rhs, P.solve_rhs));
    CK(upload(&t->d_slots, P.slots));
    CK(upload(&t->d_ctr, P.ctr));
    CK(upload(&t->d_phw, P.phw));
    CK(upload(&t->d_col_r, P.col_r));
    CK(upload(&t->d_tasks, P.tasks));
    CK(upload(&t->d_phase, P.phase));
    CK(upload(&t->d_succ_off, P.succ_off));
    CK(upload(&t->d_succ, P.succ));
    CK(upload(&t->d_col_off, P.col_off));
    CK(upload(&t->d_col_nodes, P.col_nodes));
    for (int m = 0; m < HCOV_MODES; ++m) {
        CK(upload(&t->d_indeg[m], P.indeg[m]));
        CK(upload(&t->d_roots[m][0], P.roots[m][0]));
        CK(upload(&t->d_roots[m][1], P.roots[m][1]));
        CK(upload(&t->d_q0init[m], P.q0init[m]));
        CK(upload(&t->d_q0tail[m], P.q0tail[m]));
    }
    CK(upload(&t->d_band_off, P.band_off));
    CK(upload(&t->d_diag_tile, P.diag_tile));
    CK(upload(&t->d_xs, P.xs));
    CK(upload(&t->d_ys, P.ys));
    if (P.dim == 3) CK(upload(&t->d_zs, P.zs));
    CK(upload(&t->d_perm_i2e, P.perm_i2e));
    std::vector<int32_t> leafnodes;
    std::vector<std::vector<int32_t>> rows(P.n_leaves);
    for (size_t k = 0; k < P.nodes.size(); ++k) {
        const DNode &x = P.nodes[k];
        if (x.type == ND_H) continue;
        leafnodes.push_back((int32_t)k);
        int64_t span = (int64_t)1 << (P.depth - x.level);
        for (int64_t seg = (int64_t)x.i * span; seg < (int64_t)(x.i + 1) * span; ++seg) rows[seg].push_back((int32_t)k);
    }
    t->n_leafnodes = (int32_t)leafnodes.size();
    CK(upload(&t->d_leafnodes, leafnodes));
    std::vector<int32_t> ro(P.n_leaves + 1, 0), rn;
    for (int64_t s = 0; s < P.n_leaves; ++s) {
        ro[s] = (int32_t)rn.size();
        rn.insert(rn.end(), rows[s].begin(), rows[s].end());
    }
    ro[P.n_leaves] = (int32_t)rn.size();
    CK(upload(&t->d_row_off, ro));
    CK(upload(&t->d_row_nodes, rn));
    t->uploaded = true;
    return HCOV_OK;
}

hcov_status check_theta(const hcov_theta *th, const hcov_trunc *tr)
{
    if (!th || !tr) return HCOV_ERR_INVALID_ARG;
    if (!(th->sigma2 > 0) || !(th->ell > 0) || !(th->nu > 0) || !(th->nugget >= 0)) return HCOV_ERR_INVALID_ARG;
    if (!std::isfinite(th->sigma2) || !std::isfinite(th->ell) || !std::isfinite(th->nu) || !std::isfinite(th->nugget))
        return HCOV_ERR_INVALID_ARG;
    if (!(tr->eps >= 0) || tr->kmax < 0 || tr->kcap < 0 || tr->kcap > 64) return HCOV_ERR_INVALID_ARG;
    if (tr->kmax > 0 && tr->kcap > 0 && tr->kmax > tr->kcap) return HCOV_ERR_INVALID_ARG;
    return HCOV_OK;
}

int eff_kcap(const hcov_trunc *tr)
{
    if (tr->kcap > 0) return tr->kcap;
    if (tr->kmax > 0) return tr->kmax;
    return 64;
}
// Core capacity: the products of the SPD-preserving mode see factors truncated to kmax only.
int eff_kcore(const Plan &P, const hcov_trunc *tr)
{
    const int kc = eff_kcap(tr);
    return (P.opt.factor_trunc && tr->kmax > 0) ? std::min(kc, (int)tr->kmax) : kc;
}


// Device bytes of one H-matrix instance outside its W / product-slot pools (memory planning of
// theta batches; must follow hmat_alloc).
int64_t inst_fixed_bytes(const Plan &P, int64_t kc, int64_t kco)
{
    const int64_t ntk = (int64_t)P.tasks.size();
    return 8 * (P.n_tiles() * HCOV_TILE + 2 * P.uv_elems * kc + (int64_t)P.n_cores * kco * kco + P.n_pad +
                P.n_r() * kc + 3 * P.n_leaves + (int64_t)P.phw.size() + (int64_t)P.slots.size()) +
           4 * (P.n_r() + 3 * ntk) + (int64_t)KTAB_NI * KTAB_NC * 8 + (1 << 20);
}

// (Re)allocate the numeric buffers of h for the tree's plan and capacity kcap.
hcov_status hmat_alloc(hcov_hmat h, int kcap, int kcore)
{
    hcov_tree t = h->t;
    Plan &P = t->P;
    if (h->tiles && h->kcap_alloc == kcap && h->kcore_alloc == kcore) return HCOV_OK;
    h->release_all();
    const int64_t kc = kcap;
    h->kcore_alloc = kcore;
    CK(cudaMalloc(&h->tiles, std::max<int64_t>(1, P.n_tiles()) * HCOV_TILE * sizeof(double)));
    CK(cudaMalloc(&h->U, std::max<int64_t>(1, P.uv_elems * kc) * sizeof(double)));
    CK(cudaMalloc(&h->V, std::max<int64_t>(1, P.uv_elems * kc) * sizeof(double)));
    CK(cudaMalloc(&h->cores, std::max<int64_t>(1, (int64_t)P.n_cores * kcore * kcore) * sizeof(double)));
    CK(cudaMalloc(&h->woff, std::max<size_t>(1, P.phw.size()) * sizeof(int64_t)));
    CK(cudaMalloc(&h->poff, std::max<size_t>(1, P.slots.size()) * sizeof(int64_t)));
    CK(cudaMalloc(&h->mem, 4 * sizeof(unsigned long long)));
    CK(cudaMemset(h->mem, 0, 4 * sizeof(unsigned long long)));
    CK(cudaMalloc(&h->vbuf, P.n_pad * sizeof(double)));
    CK(cudaMalloc(&h->tbuf, std::max<int64_t>(1, P.n_r() * kc) * sizeof(double)));
    CK(cudaMalloc(&h->logdet_part, P.n_leaves * sizeof(double)));
    CK(cudaMalloc(&h->minpiv_part, P.n_leaves * sizeof(double)));
    CK(cudaMalloc(&h->quad_part, P.n_leaves * sizeof(double)));
    CK(cudaMalloc(&h->rank, std::max<int64_t>(1, P.n_r()) * sizeof(int32_t)));
    CK(cudaMalloc(&h->fail, sizeof(int32_t)));
    CK(cudaMalloc(&h->flags, 5 * sizeof(int32_t)));
    const int64_t ntk = (int64_t)P.tasks.size();
    CK(cudaMalloc(&h->indeg, std::max<int64_t>(1, ntk) * sizeof(int32_t)));
    CK(cudaMalloc(&h->gbar, std::max<int64_t>(1, ntk) * sizeof(int32_t)));
    CK(cudaMalloc(&h->gslot, std::max<int64_t>(1, ntk) * sizeof(int32_t)));
    CK(cudaMalloc(&h->res, 8 * sizeof(double)));
    if (!h->res_host) CK(cudaMallocHost(&h->res_host, 8 * sizeof(double)));
    h->kcap_alloc = kcap;
    return HCOV_OK;
}

// The tree's engine resources for rank capacity kcap and ninst instances per launch.
hcov_status engine_alloc(hcov_tree t, int kcap, int ninst)
{
    Engine &E = t->eng;
    const Plan &P = t->P;
    if (E.kcap != kcap) {
        E.release();
        E.smem = engine_smem_doubles(kcap) * (int64_t)sizeof(double);
        CK(cudaFuncSetAttribute(k_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)E.smem));
        int dev = 0, nsm = 0, occ = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_engine, NT, (size_t)E.smem));
        occ = std::max(1, std::min(occ, 512 / NT));
        E.grid = nsm * occ;
        // every gang forms only if the CTAs that partly formed gangs can hold (at most one per band)
        // leave at least one free CTA
        if (E.grid <= HCOV_BANDS * (HCOV_GANG - 1)) return HCOV_ERR_INVALID_ARG;
        // per-CTA scratch: single-CTA tasks (blocks < HCOV_GANG_MIN, 6 panels) or a gang member's rows
        // (m / G rows, 4 panels) followed by the gang's shared workspace (used when the CTA is member
        // 0); members of more than HCOV_BIG_MQ rows (gangs on the largest blocks) use one of
        // HCOV_BIG_GROUPS shared big-member groups instead
        const int64_t med_m = std::min<int64_t>(std::max<int64_t>(HCOV_GANG_MIN / 2, P.opt.big_m),
                                                std::max<int64_t>(P.max_rm, 32));
        E.gshared_off = 0;
        E.scr_stride = task_scratch(med_m, kcap);
        E.bstride = 0;
        E.nbg = 0;
        if (P.max_mq > 0) {
            E.gshared_off = task_scratch(std::min<int64_t>(P.max_mq, HCOV_BIG_MQ), kcap, 4);
            E.scr_stride = std::max<int64_t>(E.scr_stride, E.gshared_off + gang_shared_doubles(kbuf_of(kcap), HCOV_GANG));
            if (P.max_mq > HCOV_BIG_MQ) {
                E.bstride = task_scratch(P.max_mq, kcap, 4);
                E.nbg = HCOV_BIG_GROUPS;
            }
        }
        CK(cudaMalloc(&E.scr, E.scr_stride * (int64_t)E.grid * sizeof(double)));
        CK(cudaMalloc(&E.bscr, std::max<int64_t>(1, E.bstride * HCOV_GANG * E.nbg) * sizeof(double)));
        CK(cudaMalloc(&E.bgrp, (HCOV_BIG_GROUPS + E.grid) * sizeof(int32_t)));
        CK(cudaMemset(E.bgrp, 0, (HCOV_BIG_GROUPS + E.grid) * sizeof(int32_t)));
        CK(cudaMalloc(&E.q1, sizeof(int32_t)));
        CK(cudaMalloc(&E.qctl, QC_N * sizeof(uint32_t)));
        CK(cudaMemset(E.qctl, 0, QC_N * sizeof(uint32_t)));
        CK(cudaMalloc(&E.stats, sizeof(EngineStats)));
        CK(cudaMallocHost(&E.stats_host, sizeof(EngineStats)));
        E.kcap = kcap;
    }
    if (ninst > E.ninst_cap) {
        cudaFree(E.q0);
        cudaFree(E.d_ctx);
        E.q0 = nullptr;
        E.d_ctx = nullptr;
        E.ninst_cap = 0;
        CK(cudaMalloc(&E.q0, std::max<int64_t>(1, (int64_t)P.band_off[HCOV_BANDS] * ninst) * sizeof(int32_t)));
        CK(cudaMalloc(&E.d_ctx, ninst * sizeof(Ctx)));
        E.ninst_cap = ninst;
    }
    return HCOV_OK;
}

// The W and product-slot pools (H-Cholesky and solves only; an assembly-only H-matrix never holds
// them).  W and the slots are bump-allocated at run time with the actual ranks.  Sizes: the
// instance's budget when a theta batch fixed one; else the capacity-based sizes when they fit,
// else the free device memory (minus 3 GB headroom) split 70 / 30.  An overflow stops the engine
// and is reported as HCOV_ERR_OUT_OF_MEMORY.
hcov_status pools_alloc(hcov_hmat h)
{
    if (h->W) return HCOV_OK;
    const Plan &P = h->t->P;
    const int64_t kc = h->kcap_alloc;
    // SPD-preserving mode: the solves inside the factorization see the pre-truncation blocks (ranks up
    // to 2 kcap for blocks > HCOV_DENSE_MAX), so product slots may need up to 4x the capacity bound
    const int64_t fm = P.opt.factor_trunc ? 4 : 1;
    const int64_t wfull = fm * P.w_elems * kc + (int64_t)P.phw.size() + 64;
    const int64_t pfull = fm * (P.slot_a * kc * kc + P.slot_b * kc) + (int64_t)P.slots.size() + 64;
    if (h->w_budget > 0) {
        h->wcap = std::min(wfull, h->w_budget);
        h->pcap = std::min(pfull, h->p_budget);
    } else {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const int64_t avail = std::max<int64_t>(0, (int64_t)fr / 8 - ((int64_t)3 << 27));
        if (wfull + pfull <= avail) { h->wcap = wfull; h->pcap = pfull; }
        else {
            h->wcap = std::min<int64_t>(wfull, (int64_t)(0.7 * avail));
            h->pcap = std::min<int64_t>(pfull, avail - h->wcap);
        }
    }
    CK(cudaMalloc(&h->W, std::max<int64_t>(1, h->wcap) * sizeof(double)));
    CK(cudaMalloc(&h->P, std::max<int64_t>(1, h->pcap) * sizeof(double)));
    h->ctx.W = h->W; h->ctx.P = h->P; h->ctx.wcap = h->wcap; h->ctx.pcap = h->pcap;
    return HCOV_OK;
}

void fill_ctx(hcov_hmat h)
{
    hcov_tree t = h->t;
    Plan &P = t->P;
    Ctx &c = h->ctx;
    c.nodes = t->d_nodes; c.tile_node = t->d_tile_node; c.rblk = t->d_rblk; c.terms = t->d_terms;
    c.xterm = t->d_xterm; c.fac_row0 = t->d_fac_row0; c.fac_nrows = t->d_fac_nrows;
    c.fac_rank_src = t->d_fac_rank_src; c.fac_off = t->d_fac_off; c.fac_pool = t->d_fac_pool;
    c.solves = t->d_solves; c.solve_rhs = t->d_solve_rhs; c.slots = t->d_slots; c.ctr = t->d_ctr;
    c.phw = t->d_phw; c.col_r = t->d_col_r; c.tasks = t->d_tasks; c.succ_off = t->d_succ_off; c.succ = t->d_succ;
    c.diag_tile = t->d_diag_tile; c.xs = t->d_xs; c.ys = t->d_ys; c.zs = t->d_zs; c.perm_i2e = t->d_perm_i2e;
    c.depth = P.depth; c.n_r = (int32_t)P.n_r(); c.root_solve = P.root_solve; c.ntasks = (int32_t)P.tasks.size();
    c.n_pad = P.n_pad; c.n_leaves = P.n_leaves; c.n_real = P.n; c.n_tiles = P.n_tiles();
    c.tiles = h->tiles; c.U = h->U; c.V = h->V; c.rank = h->rank; c.cores = h->cores; c.W = h->W; c.P = h->P;
    c.woff = h->woff; c.poff = h->poff; c.mem = h->mem; c.wcap = h->wcap; c.pcap = h->pcap;
    c.vbuf = h->vbuf; c.tbuf = h->tbuf; c.logdet_part = h->logdet_part; c.minpiv_part = h->minpiv_part; c.quad_part = h->quad_part;
    c.fail_leaf = h->fail; c.flags = h->flags;
    c.kcap = h->kcap_alloc; c.kcore = h->kcore_alloc; c.kmax = h->trunc.kmax; c.eps = h->trunc.eps;
    {
        // R22: intermediate chunk recompressions at eps * interm_rel (default 1e-2; HCOV_INTERM_REL
        // overrides it for the accuracy study in tests/test_gpu_accuracy.py)
        const char *ir = std::getenv("HCOV_INTERM_REL");
        const double v = ir ? std::atof(ir) : 1e-2;
        c.interm_rel = (v > 0 && v <= 1) ? v : 1e-2;
    }
    c.mp = hcov_matern_params(h->theta.sigma2, h->theta.ell, h->theta.nu, h->theta.nugget);
    if (c.mp.kind == 3) c.mp.tab = h->ktab;
    c.indeg = h->indeg; c.gbar = h->gbar; c.gslot = h->gslot;
    c.band_off = t->d_band_off;
    c.factor_trunc = P.opt.factor_trunc ? 1 : 0;
    c.dense_max = (int32_t)P.opt.big_m;
    {
        const char *dm = std::getenv("HCOV_DENSE_DMMA");   // A/B switch: scalar DFMA accumulation when 0
        c.dense_dmma = (dm && *dm == '0') ? 0 : 1;
        const char *tm = std::getenv("HCOV_TERM_MIN");     // A/B switch: terms always rank-B wide when 0
        c.term_min = (tm && *tm == '0') ? 0 : 1;
    }
    c.flop = nullptr;
    const char *wd = std::getenv("HCOV_WATCHDOG_S");
    double wds = wd ? std::atof(wd) : 300.0;
    if (!(wds > 0)) wds = 300.0;
    c.timeout_ns = (unsigned long long)(wds * 1e9);
}

// Engine-level fields of a context (identical in every instance of a launch).
void engine_fields(Ctx &c, const Engine &E, int ninst)
{
    c.queue[0] = E.q0; c.queue[1] = E.q1; c.qctl = E.qctl;
    c.ninst = ninst;
    c.scr = E.scr; c.scr_stride = E.scr_stride; c.gshared_off = E.gshared_off;
    c.bscr = E.bscr; c.bscr_stride = E.bstride; c.n_bgrp = E.nbg; c.big_mq = HCOV_BIG_MQ;
    c.bgrp_busy = E.bgrp; c.bgrp_cta = E.bgrp + HCOV_BIG_GROUPS;
    c.smem_dbl = E.smem / (int64_t)sizeof(double);
}

// Run the engine in mode md (0 eval, 1 assembly, 2 Cholesky, 3 forward solve, 4 back-solve) on st
// for nb H-matrices of the same tree and rank capacity in ONE persistent launch (their DAGs share
// the priority queue; a theta batch).
hcov_status engine_run_batch(hcov_hmat *hs, int nb, int md, cudaStream_t st)
{
    hcov_tree t = hs[0]->t;
    Plan &P = t->P;
    static const int mask[HCOV_MODES] = {7, 1, 2, 4, 8};
    const int64_t ntk = (int64_t)P.tasks.size();
    if (((int64_t)nb * ntk) >= ((int64_t)1 << (31 - QE_SHIFT))) return HCOV_ERR_INVALID_ARG;
    for (int i = 0; i < nb; ++i)
        if (hs[i]->t != t || hs[i]->kcap_alloc != hs[0]->kcap_alloc) return HCOV_ERR_INVALID_ARG;
    // the engine's scratch first: the W / P pools of a first run take all the free memory left
    hcov_status es = engine_alloc(t, hs[0]->kcap_alloc, nb);
    if (es) return es;
    for (int i = 0; i < nb; ++i) {
        if (md == 0 || md == 2 || md == 3) {
            hcov_status ps = pools_alloc(hs[i]);
            if (ps) return ps;
        }
    }
    Engine &E = t->eng;
    std::vector<Ctx> cx(nb);
    for (int i = 0; i < nb; ++i) {
        engine_fields(hs[i]->ctx, E, nb);
        cx[i] = hs[i]->ctx;
        cx[i].nq[0] = nb * P.n_q[md][0];
        cx[i].nq[1] = 0;
    }
    if (cx[0].nq[0] == 0) return HCOV_OK;
    CK(cudaMemcpyAsync(E.d_ctx, cx.data(), nb * sizeof(Ctx), cudaMemcpyHostToDevice, st));
    for (int i = 0; i < nb; ++i)
        LAUNCH(PC_RESET, st, k_reset_inst<<<296, 256, 0, st>>>(cx[i], t->d_indeg[md], ntk));
    LAUNCH(PC_RESET, st, k_qinit<<<296, 256, 0, st>>>(cx[0], t->d_q0init[md], t->d_q0tail[md]));
    EngineStats *stats = g_prof.events ? E.stats : nullptr;
    if (stats) CK(cudaMemsetAsync(E.stats, 0, sizeof(EngineStats), st));
    {
        static const unsigned long long zeros[64] = {};
        const int on = stats ? 1 : 0;
        CK(cudaMemcpyToSymbolAsync(g_phase_on, &on, sizeof(int), 0, cudaMemcpyHostToDevice, st));
        if (on) CK(cudaMemcpyToSymbolAsync(g_phase_ns, zeros, sizeof(zeros), 0, cudaMemcpyHostToDevice, st));
    }
    const char *tlpath = std::getenv("HCOV_TIMELINE");
    unsigned long long *tl = nullptr;
    if (tlpath && nb == 1) {
        CK(cudaMalloc(&tl, 3 * std::max<int64_t>(1, ntk) * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(tl, 0, 3 * std::max<int64_t>(1, ntk) * sizeof(unsigned long long), st));
    }
    LAUNCH(PC_ENGINE, st, k_engine<<<E.grid, NT, E.smem, st>>>(cx[0], E.d_ctx, mask[md], t->d_phase, stats, tl));
    CK(cudaGetLastError());
    // the context array's host copy (cx) must outlive the asynchronous upload
    CK(cudaStreamSynchronize(st));
    if (tl) {
        std::vector<unsigned long long> hv(3 * ntk);
        CK(cudaMemcpyAsync(hv.data(), tl, hv.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cudaFree(tl);
        FILE *f = std::fopen(tlpath, "wb");
        if (f) {
            std::fwrite(hv.data(), 8, hv.size(), f);
            std::fclose(f);
        }
    }
    if (stats) {
        CK(cudaMemcpyAsync(E.stats_host, E.stats, sizeof(EngineStats), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int k = 0; k < TK_NTYPES; ++k) {
            g_prof.busy_ns[k] += (double)E.stats_host->busy_ns[k];
            g_prof.tasks[k] += (double)E.stats_host->tasks[k];
        }
        for (int k = 0; k < FC_N; ++k) g_prof.flop[k] += E.stats_host->flop[k];
        unsigned long long ph[64];
        CK(cudaMemcpyFromSymbol(ph, g_phase_ns, sizeof(ph)));
        for (int k = 0; k < 64; ++k) g_prof.phase_ns[k] += (double)ph[k];
    }
    return HCOV_OK;
}

hcov_status engine_run(hcov_hmat h, int md, cudaStream_t st) { return engine_run_batch(&h, 1, md, st); }

hcov_status assemble_setup(hcov_hmat h, const hcov_theta *theta, const hcov_trunc *trunc, cudaStream_t st)
{
    hcov_tree t = h->t;
    const int kcap = eff_kcap(trunc);
    hcov_status s = tree_upload(t);
    if (s) return s;
    h->theta = *theta;
    h->trunc = *trunc;
    if ((s = hmat_alloc(h, kcap, eff_kcore(t->P, trunc)))) return s;
    if (!h->ktab) CK(cudaMalloc(&h->ktab, KTAB_NI * KTAB_NC * sizeof(double)));
    {
        const MaternParams mp = hcov_matern_params(theta->sigma2, theta->ell, theta->nu, theta->nugget);
        if (mp.kind == 3) {
            LAUNCH(PC_AUX, st, k_ktab<<<1, KTAB_NI, 0, st>>>(theta->nu, h->ktab));
            CK(cudaGetLastError());
        }
    }
    fill_ctx(h);
    Plan &P = t->P;
    CK(cudaMemsetAsync(h->rank, 0, std::max<int64_t>(1, P.n_r()) * sizeof(int32_t), st));
    CK(cudaMemsetAsync(h->flags, 0, 5 * sizeof(int32_t), st));
    CK(cudaMemsetAsync(h->fail, 0x7f, sizeof(int32_t), st));
    CK(cudaMemsetAsync(h->quad_part, 0, P.n_leaves * sizeof(double), st));
    CK(cudaMemsetAsync(h->woff, 0xff, std::max<size_t>(1, P.phw.size()) * sizeof(int64_t), st));
    CK(cudaMemsetAsync(h->poff, 0xff, std::max<size_t>(1, P.slots.size()) * sizeof(int64_t), st));
    CK(cudaMemsetAsync(h->mem, 0, 4 * sizeof(unsigned long long), st));
    return HCOV_OK;
}

hcov_status check_abort(hcov_hmat h, cudaStream_t st, int32_t *hf)
{
    uint32_t ab = 0;
    unsigned long long mem[4] = {0, 0, 0, 0};
    CK(cudaMemcpyAsync(mem, h->mem, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (h->t->eng.qctl) CK(cudaMemcpyAsync(&ab, h->t->eng.qctl + QC_ABORT, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hf, h->fail, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hf + 1, h->flags, 5 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (mem[2]) {   // a pool overflow also raises the abort flag
        if (verbose())
            std::fprintf(stderr, "hcov: pool overflow: W used %llu of %lld, P used %llu of %lld, overflows %llu\n",
                         mem[0], (long long)h->wcap, mem[1], (long long)h->pcap, mem[2]);
        return HCOV_ERR_OUT_OF_MEMORY;
    }
    {
        // pool words this run used: sizing of later theta batches on this tree
        hcov_tree t = h->t;
        if (t->est_kcap != h->kcap_alloc || t->est_eps != h->trunc.eps || t->est_kmax != h->trunc.kmax) {
            t->est_kcap = h->kcap_alloc; t->est_eps = h->trunc.eps; t->est_kmax = h->trunc.kmax;
            t->est_w = 0; t->est_p = 0;
        }
        t->est_w = std::max<int64_t>(t->est_w, (int64_t)mem[0]);
        t->est_p = std::max<int64_t>(t->est_p, (int64_t)mem[1]);
    }
    if (ab) return HCOV_ERR_CUDA;
    return HCOV_OK;
}

hcov_status finish_result(hcov_hmat h, cudaStream_t st, hcov_result *out)
{
    Plan &P = h->t->P;
    LAUNCH(PC_REDUCE, st, k_reduce<<<1, NT, 0, st>>>(h->ctx, h->res));
    CK(cudaGetLastError());
    int32_t hf[6];
    CK(cudaMemcpyAsync(h->res_host, h->res, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    hcov_status s = check_abort(h, st, hf);
    if (s) return s;
    const double ld = h->res_host[0], q = h->res_host[1];
    std::memset(out, 0, sizeof(*out));
    out->n = P.n;
    out->logdet = ld;
    out->quad = q;
    out->loglik = -0.5 * (double)P.n * std::log(2.0 * M_PI) - 0.5 * ld - 0.5 * q;
    out->min_pivot = h->res_host[2];
    out->fail_leaf = (hf[0] == 0x7f7f7f7f) ? -1 : hf[0];
    out->cap_binds = hf[1];
    out->max_rank = hf[3];
    out->acc_loss = hf[4];
    out->interm_cuts = hf[5];
    if (out->fail_leaf >= 0) { out->loglik = -INFINITY; return HCOV_ERR_NOT_SPD; }
    if ((hf[2] > 0 || hf[4] > 0) && h->trunc.kmax == 0) { out->loglik = -INFINITY; return HCOV_ERR_RANK_CAPACITY; }
    return HCOV_OK;
}


// Release the extra instances of the last theta batch.
void free_extra(hcov_tree t)
{
    for (hcov_hmat h : t->extra) delete h;
    t->extra.clear();
}

// Evaluate L~ for nb thetas on nb instances of one tree in ONE engine launch (A3-A10 each);
// out[i] / sts[i] per instance (sts == nullptr: nb == 1, the status is returned).
hcov_status eval_instances(hcov_hmat *hs, int nb, const hcov_theta *const *th, const hcov_trunc *trunc,
                           const double *Z_dev, cudaStream_t st, hcov_result *out, hcov_status *sts)
{
    hcov_status s;
    for (int i = 0; i < nb; ++i) {
        if ((s = assemble_setup(hs[i], th[i], trunc, st))) return s;
        LAUNCH(PC_PERM, st, k_permute_in<<<256, 256, 0, st>>>(hs[i]->ctx, Z_dev, hs[i]->vbuf));
    }
    s = engine_run_batch(hs, nb, 0, st);
    if (s) {
        if (!sts) return s;
        for (int i = 0; i < nb; ++i) { sts[i] = s; out[i] = hcov_result{}; out[i].loglik = -INFINITY; }
        return (s == HCOV_ERR_OUT_OF_MEMORY) ? HCOV_OK : s;
    }
    for (int i = 0; i < nb; ++i) {
        hs[i]->state = 3;
        const hcov_status r = finish_result(hs[i], st, out + i);
        if (!sts) return r;
        sts[i] = r;
    }
    return HCOV_OK;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
extern "C" {

const char *hcov_status_string(hcov_status s)
{
    switch (s) {
    case HCOV_OK: return "ok";
    case HCOV_ERR_INVALID_ARG: return "invalid argument";
    case HCOV_ERR_EMPTY_INPUT: return "empty input";
    case HCOV_ERR_NOT_SPD: return "matrix not positive definite";
    case HCOV_ERR_OUT_OF_MEMORY: return "out of device memory";
    case HCOV_ERR_CUDA: return "CUDA error";
    case HCOV_ERR_RANK_CAPACITY: return "rank capacity exceeded";
    case HCOV_ERR_STATE: return "invalid call order";
    }
    return "unknown";
}

// schedule-granularity experiments (not part of the method): HCOV_RCHUNK = pending terms per RAPP
// chunk of a large low-rank block, HCOV_TCHUNK = pending terms per TAPP task
static void plan_env_overrides(PlanOpts &o)
{
    if (const char *e = std::getenv("HCOV_RCHUNK")) { const int v = std::atoi(e); if (v >= 1 && v <= 16) o.rchunk = v; }
    if (const char *e = std::getenv("HCOV_TCHUNK")) { const int v = std::atoi(e); if (v >= 1 && v <= 64) o.chunk = v; }
    if (const char *e = std::getenv("HCOV_GANG1_BELOW")) o.gang1_below = std::atoll(e);
    if (const char *e = std::getenv("HCOV_GANG_ROWS")) o.gang_rows = std::atoll(e);
    if (const char *e = std::getenv("HCOV_GANG_MAX_SMALL")) o.gang_max_small = std::atoi(e);
    if (const char *e = std::getenv("HCOV_RAPP512")) o.rapp512 = std::atoi(e);
    if (const char *e = std::getenv("HCOV_BIG_M")) { const int v = std::atoi(e); if (v == 64 || v == 128 || v == 256 || v == 512) o.big_m = v; }
}

hcov_status hcov_build_tree_host_ex(const double *s_host, int64_t n, const hcov_tree_opts *opts, hcov_tree *out)
{
    if (!out || !opts) return HCOV_ERR_INVALID_ARG;
    *out = nullptr;
    if (n == 0) return HCOV_ERR_EMPTY_INPUT;
    if (!s_host || n < 0 || opts->leaf_size != HCOV_LEAF || !(opts->eta >= 0) || opts->dense_below < 0 ||
        (opts->factor_trunc != 0 && opts->factor_trunc != 1) || (opts->dim != 0 && opts->dim != 2 && opts->dim != 3))
        return HCOV_ERR_INVALID_ARG;
    std::unique_ptr<hcov_tree_s> t(new (std::nothrow) hcov_tree_s());
    if (!t) return HCOV_ERR_OUT_OF_MEMORY;
    PlanOpts o;
    o.eta = opts->eta;
    o.dense_below = opts->dense_below;
    o.factor_trunc = opts->factor_trunc != 0;
    o.dim = opts->dim == 3 ? 3 : 2;
    plan_env_overrides(o);
    const auto g0 = std::chrono::steady_clock::now();
    int rc = plan_build(t->P, s_host, n, o);
    t->geo_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - g0).count();
    if (rc == 2) return HCOV_ERR_EMPTY_INPUT;
    if (rc) return HCOV_ERR_INVALID_ARG;
    *out = t.release();
    return HCOV_OK;
}

hcov_status hcov_build_tree_host(const double *s_host, int64_t n, int32_t leaf_size, double eta, int32_t dense_below,
                                 hcov_tree *out)
{
    const hcov_tree_opts o{leaf_size, eta, dense_below, 0, 2};
    return hcov_build_tree_host_ex(s_host, n, &o, out);
}

hcov_status hcov_build_tree_ex(const double *s_dev, int64_t n, const hcov_tree_opts *opts, hcov_stream stream,
                               hcov_tree *out)
{
    if (!out) return HCOV_ERR_INVALID_ARG;
    *out = nullptr;
    if (n == 0) return HCOV_ERR_EMPTY_INPUT;
    if (!s_dev || n < 0 || !opts) return HCOV_ERR_INVALID_ARG;
    if (opts->leaf_size != HCOV_LEAF || !(opts->eta >= 0) || opts->dense_below < 0 ||
        (opts->factor_trunc != 0 && opts->factor_trunc != 1) || (opts->dim != 0 && opts->dim != 2 && opts->dim != 3))
        return HCOV_ERR_INVALID_ARG;
    // A1 / A2 on the device (tree.cu: K1 cluster tree, K2 block tree); the task DAG is planned on
    // the host from their output
    std::unique_ptr<hcov_tree_s> tp(new (std::nothrow) hcov_tree_s());
    if (!tp) return HCOV_ERR_OUT_OF_MEMORY;
    PlanOpts o;
    o.eta = opts->eta;
    o.dense_below = opts->dense_below;
    o.factor_trunc = opts->factor_trunc != 0;
    o.dim = opts->dim == 3 ? 3 : 2;
    plan_env_overrides(o);
    {
        PlanGeo geo;
        const auto g0 = std::chrono::steady_clock::now();
        const int rg = tree_geo_device(s_dev, n, o, (cudaStream_t)stream, geo);
        tp->geo_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - g0).count();
        if (rg == 2) return HCOV_ERR_EMPTY_INPUT;
        if (rg == 1) return HCOV_ERR_INVALID_ARG;
        if (rg) return HCOV_ERR_CUDA;
        const int rc = plan_build(tp->P, nullptr, n, o, &geo);
        if (rc == 2) return HCOV_ERR_EMPTY_INPUT;
        if (rc == 3) return HCOV_ERR_CUDA;    // device trees inconsistent with the planner's rules
        if (rc) return HCOV_ERR_INVALID_ARG;
    }
    tp->tree_on_device = true;
    hcov_tree t = tp.release();
    hcov_status st = tree_upload(t);
    if (st) { delete t; return st; }
    *out = t;
    return HCOV_OK;
}

hcov_status hcov_build_tree(const double *s_dev, int64_t n, int32_t leaf_size, double eta, int32_t dense_below,
                            hcov_stream stream, hcov_tree *out)
{
    const hcov_tree_opts o{leaf_size, eta, dense_below, 0, 2};
    return hcov_build_tree_ex(s_dev, n, &o, stream, out);
}

hcov_status hcov_tree_get_info(hcov_tree t, hcov_tree_info *info)
{
    if (!t || !info) return HCOV_ERR_INVALID_ARG;
    const Plan &P = t->P;
    info->n = P.n; info->n_pad = P.n_pad; info->depth = P.depth; info->leaf_size = HCOV_LEAF;
    info->n_leaves = P.n_leaves; info->n_dense_tiles = P.n_tiles(); info->n_lowrank = P.n_r();
    info->n_tasks = (int64_t)P.tasks.size(); info->n_waves = P.crit_len; info->eta = P.opt.eta;
    info->uv_elems = P.uv_elems; info->w_elems = P.w_elems; info->slot_a = P.slot_a; info->slot_b = P.slot_b;
    info->n_cores = P.n_cores; info->n_edges = (int64_t)P.succ.size(); info->n_xterm = (int64_t)P.xterm.size();
    info->max_mq = P.max_mq;
    info->tree_on_device = t->tree_on_device ? 1 : 0;
    info->geo_ms = t->geo_ms;
    info->dim = P.dim;
    return HCOV_OK;
}

hcov_status hcov_tree_perm(hcov_tree t, int64_t *perm)
{
    if (!t || !perm) return HCOV_ERR_INVALID_ARG;
    std::memcpy(perm, t->P.perm_i2e.data(), t->P.n_pad * sizeof(int64_t));
    return HCOV_OK;
}

hcov_status hcov_tree_blocks(hcov_tree t, int32_t *out4, int64_t cap, int64_t *count)
{
    if (!t || !count) return HCOV_ERR_INVALID_ARG;
    const Plan &P = t->P;
    *count = (int64_t)P.nodes.size();
    if (!out4) return HCOV_OK;
    if (cap < *count) return HCOV_ERR_INVALID_ARG;
    for (size_t k = 0; k < P.nodes.size(); ++k) {
        out4[4 * k + 0] = P.nodes[k].level;
        out4[4 * k + 1] = P.nodes[k].i;
        out4[4 * k + 2] = P.nodes[k].j;
        out4[4 * k + 3] = P.nodes[k].type;
    }
    return HCOV_OK;
}

hcov_status hcov_tree_tasks(hcov_tree t, int32_t *out6, int64_t cap, int64_t *count)
{
    if (!t || !count) return HCOV_ERR_INVALID_ARG;
    const Plan &P = t->P;
    *count = (int64_t)P.tasks.size();
    if (!out6) return HCOV_OK;
    if (cap < *count) return HCOV_ERR_INVALID_ARG;
    for (size_t k = 0; k < P.tasks.size(); ++k) {
        const DTask &tk = P.tasks[k];
        int32_t *o = out6 + 6 * k;
        o[0] = tk.type; o[1] = P.phase[k]; o[2] = tk.a; o[3] = tk.b; o[4] = tk.c; o[5] = tk.d;
    }
    return HCOV_OK;
}

hcov_status hcov_tree_succ(hcov_tree t, int32_t *off, int32_t *succ, int64_t cap, int64_t *count)
{
    if (!t || !count) return HCOV_ERR_INVALID_ARG;
    const Plan &P = t->P;
    *count = (int64_t)P.succ.size();
    if (!off || !succ) return HCOV_OK;
    if (cap < *count) return HCOV_ERR_INVALID_ARG;
    std::memcpy(off, P.succ_off.data(), P.succ_off.size() * sizeof(int32_t));
    std::memcpy(succ, P.succ.data(), P.succ.size() * sizeof(int32_t));
    return HCOV_OK;
}

hcov_status hcov_tree_bbox(hcov_tree t, double *bb, int64_t cap)
{
    if (!t || !bb || cap < (int64_t)t->P.bb.size()) return HCOV_ERR_INVALID_ARG;
    std::memcpy(bb, t->P.bb.data(), t->P.bb.size() * sizeof(double));
    return HCOV_OK;
}

hcov_status hcov_assemble(hcov_tree t, const hcov_theta *theta, const hcov_trunc *trunc, hcov_stream stream,
                          hcov_hmat *out)
{
    if (!out) return HCOV_ERR_INVALID_ARG;
    *out = nullptr;
    if (!t) return HCOV_ERR_INVALID_ARG;
    hcov_status s = check_theta(theta, trunc);
    if (s) return s;
    hcov_hmat h = new (std::nothrow) hcov_hmat_s();
    if (!h) return HCOV_ERR_OUT_OF_MEMORY;
    h->t = t;
    cudaStream_t st = (cudaStream_t)stream;
    s = assemble_setup(h, theta, trunc, st);
    if (!s) s = engine_run(h, 1, st);
    if (!s) {
        int32_t hf[6];
        s = check_abort(h, st, hf);
    }
    if (s) { delete h; return s; }
    h->state = 1;
    *out = h;
    return HCOV_OK;
}

hcov_status hcov_cholesky(hcov_hmat h, hcov_stream stream, int64_t *fail_leaf)
{
    if (!h) return HCOV_ERR_INVALID_ARG;
    if (h->state != 1) return HCOV_ERR_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    hcov_status s = engine_run(h, 2, st);
    if (s) return s;
    int32_t hf[6];
    if ((s = check_abort(h, st, hf))) return s;
    h->state = 2;
    int64_t fl = (hf[0] == 0x7f7f7f7f) ? -1 : hf[0];
    if (fail_leaf) *fail_leaf = fl;
    if (fl >= 0) return HCOV_ERR_NOT_SPD;
    if ((hf[2] > 0 || hf[4] > 0) && h->trunc.kmax == 0) return HCOV_ERR_RANK_CAPACITY;
    return HCOV_OK;
}

hcov_status hcov_loglik(hcov_hmat h, const double *Z_dev, hcov_stream stream, hcov_result *out)
{
    if (!h || !Z_dev || !out) return HCOV_ERR_INVALID_ARG;
    if (h->state < 2) return HCOV_ERR_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    LAUNCH(PC_PERM, st, k_permute_in<<<256, 256, 0, st>>>(h->ctx, Z_dev, h->vbuf));
    hcov_status s = engine_run(h, 3, st);
    if (s) return s;
    h->state = 3;
    return finish_result(h, st, out);
}

hcov_status hcov_eval(hcov_tree t, const hcov_theta *theta, const hcov_trunc *trunc, const double *Z_dev,
                      hcov_stream stream, hcov_result *out)
{
    if (!t || !Z_dev || !out) return HCOV_ERR_INVALID_ARG;
    hcov_status s = check_theta(theta, trunc);
    if (s) return s;
    if (!t->cached) {
        t->cached = new (std::nothrow) hcov_hmat_s();
        if (!t->cached) return HCOV_ERR_OUT_OF_MEMORY;
        t->cached->t = t;
    }
    hcov_hmat h = t->cached;
    cudaStream_t st = (cudaStream_t)stream;
    s = eval_instances(&h, 1, &theta, trunc, Z_dev, st, out, nullptr);
    if (s == HCOV_ERR_OUT_OF_MEMORY && (h->w_budget > 0 || !t->extra.empty())) {
        // pools sized for a theta batch were too small for this theta: all free memory, once more
        free_extra(t);
        h->release_pools();
        h->w_budget = h->p_budget = 0;
        s = eval_instances(&h, 1, &theta, trunc, Z_dev, st, out, nullptr);
    }
    return s;
}

hcov_status hcov_mle_batch(hcov_tree t, const double *Z_dev, const hcov_theta *thetas, int32_t m,
                           const hcov_trunc *trunc, hcov_stream stream, double *loglik_host, hcov_status *status_host)
{
    if (!t || !Z_dev || !thetas || m < 0 || !trunc || !loglik_host || !status_host) return HCOV_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    auto record = [&](int k, hcov_status s, const hcov_result &r) -> hcov_status {
        status_host[k] = s;
        if (s == HCOV_OK) { loglik_host[k] = r.loglik; return HCOV_OK; }
        loglik_host[k] = -INFINITY;
        if (s == HCOV_ERR_NOT_SPD || s == HCOV_ERR_RANK_CAPACITY || s == HCOV_ERR_INVALID_ARG) return HCOV_OK;
        return s;   // out of memory / CUDA: abort the batch
    };
    std::vector<int> todo;
    for (int32_t k = 0; k < m; ++k) {
        if (check_theta(thetas + k, trunc)) { status_host[k] = HCOV_ERR_INVALID_ARG; loglik_host[k] = -INFINITY; }
        else todo.push_back(k);
    }
    if (todo.empty()) return HCOV_OK;
    hcov_status s = tree_upload(t);
    if (s) return s;
    const int kcap = eff_kcap(trunc);
    size_t next = 0;
    // pool sizes of the batch instances come from the words an earlier run on this tree used; without
    // that, the first candidate runs alone (all free memory) and provides it
    if (t->est_kcap != kcap || t->est_eps != trunc->eps || t->est_kmax != trunc->kmax || t->est_w + t->est_p == 0 ||
        !t->cached) {
        hcov_result r{};
        const int k = todo[next++];
        if ((s = record(k, hcov_eval(t, thetas + k, trunc, Z_dev, stream, &r), r))) return s;
    }
    if (next == todo.size()) return HCOV_OK;
    // batch size B: instance 0 (t->cached) plus B - 1 extra instances, every instance with pools of
    // 1.3 x the estimate, 2 GB headroom (HCOV_MAX_BATCH at most; env HCOV_BATCH overrides downwards)
    free_extra(t);
    t->cached->release_pools();
    const Plan &P = t->P;
    const int64_t wb = (int64_t)(1.3 * (double)t->est_w) + ((int64_t)1 << 20);
    const int64_t pb = (int64_t)(1.3 * (double)t->est_p) + ((int64_t)1 << 20);
    const int64_t fixed = inst_fixed_bytes(P, kcap, eff_kcore(P, trunc)), pools = 8 * (wb + pb);
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const int64_t avail = (int64_t)fr - ((int64_t)2 << 30);
    int B = 1;
    if (avail > pools) B = 1 + (int)std::min<int64_t>(HCOV_MAX_BATCH - 1, (avail - pools) / (fixed + pools));
    if (const char *eb = std::getenv("HCOV_BATCH")) B = std::max(1, std::min(B, std::atoi(eb)));
    B = std::min<int>(B, (int)(todo.size() - next));
    std::vector<hcov_hmat> inst(1, t->cached);
    for (int i = 1; i < B; ++i) {
        hcov_hmat h = new (std::nothrow) hcov_hmat_s();
        if (!h) break;
        h->t = t;
        t->extra.push_back(h);
        if (hmat_alloc(h, kcap, eff_kcore(P, trunc))) { free_extra(t); inst.resize(1); break; }   // (fixed memory only: B shrinks)
        inst.push_back(h);
    }
    B = (int)inst.size();
    for (hcov_hmat h : inst) { h->w_budget = B > 1 ? wb : 0; h->p_budget = B > 1 ? pb : 0; }
    std::vector<int> retry;
    while (next < todo.size()) {
        const int nb = (int)std::min<size_t>(B, todo.size() - next);
        std::vector<const hcov_theta *> th(nb);
        std::vector<hcov_result> res(nb);
        std::vector<hcov_status> sts(nb);
        for (int i = 0; i < nb; ++i) th[i] = thetas + todo[next + i];
        s = eval_instances(inst.data(), nb, th.data(), trunc, Z_dev, st, res.data(), sts.data());
        if (s) return s;
        for (int i = 0; i < nb; ++i) {
            const int k = todo[next + i];
            // a pool overflow stops the whole launch: every candidate of it that did not finish is
            // evaluated again on its own
            if (sts[i] == HCOV_ERR_OUT_OF_MEMORY || sts[i] == HCOV_ERR_CUDA) retry.push_back(k);
            else if ((s = record(k, sts[i], res[i]))) return s;
        }
        next += nb;
    }
    free_extra(t);
    t->cached->release_pools();
    t->cached->w_budget = t->cached->p_budget = 0;
    for (int k : retry) {
        hcov_result r{};
        if ((s = record(k, hcov_eval(t, thetas + k, trunc, Z_dev, stream, &r), r))) return s;
    }
    return HCOV_OK;
}

}  // extern "C"

namespace {
// in (external) -> vbuf -> [forward] -> [back] -> out (external); factored H-matrix.
hcov_status solve_ext(hcov_hmat h, const double *in, double *out, bool fwd, bool back, cudaStream_t st)
{
    LAUNCH(PC_AUX, st, k_permute_in<<<256, 256, 0, st>>>(h->ctx, in, h->vbuf));
    hcov_status s;
    if (fwd && (s = engine_run(h, 3, st))) return s;
    if (back && (s = engine_run(h, 4, st))) return s;
    LAUNCH(PC_AUX, st, k_permute_out<<<256, 256, 0, st>>>(h->ctx, h->vbuf, out));
    int32_t hf[6];
    return check_abort(h, st, hf);
}

hcov_status matvec_ext(hcov_hmat h, const double *x, double *y, double *xi, double *yi, double *t12, cudaStream_t st)
{
    hcov_tree t = h->t;
    const Plan &P = t->P;
    LAUNCH(PC_AUX, st, k_permute_in<<<256, 256, 0, st>>>(h->ctx, x, xi));
    double *t1 = t12, *t2 = t12 + std::max<int64_t>(1, P.n_r()) * h->ctx.kcap;
    if (P.n_r() > 0) LAUNCH(PC_AUX, st, k_mv_t<<<(int)std::min<int64_t>(P.n_r(), 65535), NT, 0, st>>>(h->ctx, xi, t1, t2));
    LAUNCH(PC_AUX, st, k_mv_rows<<<(int)std::min<int64_t>((P.n_leaves + 7) / 8, 65535), 256, 0, st>>>(
                           h->ctx, t->d_row_off, t->d_row_nodes, t->d_col_off, t->d_col_nodes, xi, t1, t2, yi));
    LAUNCH(PC_AUX, st, k_permute_out<<<256, 256, 0, st>>>(h->ctx, yi, y));
    CK(cudaGetLastError());
    return HCOV_OK;
}

struct DevBuf {
    std::vector<void *> ps;
    ~DevBuf() { for (void *p : ps) cudaFree(p); }
    template <class T> cudaError_t get(T **p, int64_t n)
    {
        cudaError_t e = cudaMalloc((void **)p, std::max<int64_t>(1, n) * sizeof(T));
        if (e == cudaSuccess) ps.push_back(*p);
        return e;
    }
};

double dot_dev(const double *a, const double *b, int64_t n, double *part, double *res, double *res_host, cudaStream_t st)
{
    k_dot_part<<<DOT_BLOCKS, 256, 0, st>>>(a, b, n, part);
    k_dot_sum<<<1, 32, 0, st>>>(part, res);
    g_prof.launches += 2;
    cudaMemcpyAsync(res_host, res, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return *res_host;
}
}  // namespace

extern "C" {

hcov_status hcov_forward_solve(hcov_hmat h, const double *z_dev, double *v_dev, hcov_stream stream)
{
    if (!h || !z_dev || !v_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state < 2) return HCOV_ERR_STATE;
    return solve_ext(h, z_dev, v_dev, true, false, (cudaStream_t)stream);
}

hcov_status hcov_ldl_diag(hcov_hmat h, double *D_dev, hcov_stream stream)
{
    if (!h || !D_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state < 2) return HCOV_ERR_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    LAUNCH(PC_AUX, st, k_ldl_diag<<<256, 256, 0, st>>>(h->ctx, D_dev));
    CK(cudaGetLastError());
    return HCOV_OK;
}

hcov_status hcov_backsolve(hcov_hmat h, const double *v_dev, double *u_dev, hcov_stream stream)
{
    if (!h || !v_dev || !u_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state < 2) return HCOV_ERR_STATE;
    return solve_ext(h, v_dev, u_dev, false, true, (cudaStream_t)stream);
}

hcov_status hcov_solve(hcov_hmat h, const double *b_dev, double *x_dev, hcov_stream stream)
{
    if (!h || !b_dev || !x_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state < 2) return HCOV_ERR_STATE;
    return solve_ext(h, b_dev, x_dev, true, true, (cudaStream_t)stream);
}

hcov_status hcov_matvec(hcov_hmat h, const double *x_dev, double *y_dev, hcov_stream stream)
{
    if (!h || !x_dev || !y_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state != 1) return HCOV_ERR_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    const Plan &P = h->t->P;
    DevBuf B;
    double *xi, *yi, *t12;
    CK(B.get(&xi, P.n_pad));
    CK(B.get(&yi, P.n_pad));
    CK(B.get(&t12, 2 * std::max<int64_t>(1, P.n_r()) * h->ctx.kcap));
    hcov_status s = matvec_ext(h, x_dev, y_dev, xi, yi, t12, st);
    if (s) return s;
    CK(cudaStreamSynchronize(st));
    return HCOV_OK;
}

hcov_status hcov_pcg(hcov_hmat A, hcov_hmat M, const double *b_dev, double *x_dev, int32_t maxit, double tol,
                     hcov_stream stream, int32_t *iters, double *relres)
{
    if (!A || !M || !b_dev || !x_dev || maxit < 0 || !(tol >= 0) || !iters || !relres) return HCOV_ERR_INVALID_ARG;
    if (A->state != 1 || M->state < 2) return HCOV_ERR_STATE;
    if (A->t != M->t) return HCOV_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const Plan &P = A->t->P;
    const int64_t n = P.n;
    DevBuf B;
    double *r, *z, *p, *q, *xi, *yi, *t12, *part, *res, *resh;
    CK(B.get(&r, n)); CK(B.get(&z, n)); CK(B.get(&p, n)); CK(B.get(&q, n));
    CK(B.get(&xi, P.n_pad)); CK(B.get(&yi, P.n_pad));
    CK(B.get(&t12, 2 * std::max<int64_t>(1, P.n_r()) * A->ctx.kcap));
    CK(B.get(&part, DOT_BLOCKS)); CK(B.get(&res, 1));
    CK(cudaMallocHost(&resh, sizeof(double)));
    std::unique_ptr<double, cudaError_t (*)(void *)> resh_guard(resh, cudaFreeHost);
    const int gb = 592;
    // x0 = 0, r0 = b, z0 = M^{-1} r0, p0 = z0  (TCG with preconditioner A_inv, listing PAPER.md:550-555)
    CK(cudaMemsetAsync(x_dev, 0, n * sizeof(double), st));
    CK(cudaMemcpyAsync(r, b_dev, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    hcov_status s;
    if ((s = solve_ext(M, r, z, true, true, st))) return s;
    CK(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    const double bb = std::sqrt(dot_dev(b_dev, b_dev, n, part, res, resh, st));
    double rz = dot_dev(r, z, n, part, res, resh, st);
    int it = 0;
    double rr = bb;
    *relres = bb > 0 ? 1.0 : 0.0;
    while (it < maxit && bb > 0) {
        if ((s = matvec_ext(A, p, q, xi, yi, t12, st))) return s;
        const double pq = dot_dev(p, q, n, part, res, resh, st);
        if (!(pq > 0)) break;   // A~ not positive definite along p
        const double alpha = rz / pq;
        k_axpby<<<gb, 256, 0, st>>>(n, alpha, p, 1.0, x_dev);
        k_axpby<<<gb, 256, 0, st>>>(n, -alpha, q, 1.0, r);
        g_prof.launches += 2;
        ++it;
        rr = std::sqrt(dot_dev(r, r, n, part, res, resh, st));
        *relres = rr / bb;
        if (rr <= tol * bb) break;
        if ((s = solve_ext(M, r, z, true, true, st))) return s;
        const double rz1 = dot_dev(r, z, n, part, res, resh, st);
        const double beta = rz1 / rz;
        rz = rz1;
        k_axpby<<<gb, 256, 0, st>>>(n, 1.0, z, beta, p);
        g_prof.launches += 1;
    }
    *iters = it;
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return HCOV_OK;
}

// ---- NEXT (f3): accuracy diagnostics of Sec. 4 (Tables 2-4) ----------
namespace {
// x_i in [-1/2, 1/2): a counter-based hash of (i, seed) (deterministic start vector of the power
// iterations)
__global__ void k_start_vec(int64_t n, uint64_t seed, double *x)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        x[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    }
}
// y = a * x (n)
__global__ void k_scale(int64_t n, double a, const double *x, double *y)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        y[k] = a * x[k];
}
// acc[0] += x[j] (one thread: the trace accumulates in column order)
__global__ void k_pick_add(const double *x, int64_t j, double *acc)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) acc[0] += x[j];
}

struct DiagBufs {
    DevBuf B;
    double *xi, *yi, *t12, *part, *res, *resh = nullptr;
    ~DiagBufs() { if (resh) cudaFreeHost(resh); }
    hcov_status init(const Plan &P, int kcap)
    {
        CK(B.get(&xi, P.n_pad)); CK(B.get(&yi, P.n_pad));
        CK(B.get(&t12, 2 * std::max<int64_t>(1, P.n_r()) * std::max(1, kcap)));
        CK(B.get(&part, DOT_BLOCKS)); CK(B.get(&res, 1));
        CK(cudaMallocHost(&resh, sizeof(double)));
        return HCOV_OK;
    }
};
}  // namespace

hcov_status hcov_norm2_diff(hcov_hmat A, hcov_hmat Bm, int32_t iters, uint64_t seed, hcov_stream stream, double *out)
{
    if (!A || !Bm || !out || iters < 1) return HCOV_ERR_INVALID_ARG;
    if (A->state != 1 || Bm->state != 1) return HCOV_ERR_STATE;
    if (A->t->P.n != Bm->t->P.n) return HCOV_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = A->t->P.n;
    DiagBufs da, db;
    hcov_status s;
    if ((s = da.init(A->t->P, A->ctx.kcap)) || (s = db.init(Bm->t->P, Bm->ctx.kcap))) return s;
    DevBuf B;
    double *x, *y, *z;
    CK(B.get(&x, n)); CK(B.get(&y, n)); CK(B.get(&z, n));
    k_start_vec<<<296, 256, 0, st>>>(n, seed, x);
    double nx = std::sqrt(dot_dev(x, x, n, da.part, da.res, da.resh, st));
    k_scale<<<296, 256, 0, st>>>(n, 1.0 / nx, x, x);
    g_prof.launches += 2;
    double lam = 0.0;
    for (int it = 0; it < iters; ++it) {
        // y = (A - B) x
        if ((s = matvec_ext(A, x, y, da.xi, da.yi, da.t12, st))) return s;
        if ((s = matvec_ext(Bm, x, z, db.xi, db.yi, db.t12, st))) return s;
        k_axpby<<<296, 256, 0, st>>>(n, -1.0, z, 1.0, y);
        g_prof.launches += 1;
        const double ny = std::sqrt(dot_dev(y, y, n, da.part, da.res, da.resh, st));
        lam = std::max(lam, ny);                 // ||(A - B) x|| with ||x|| = 1: -> |lambda|_max
        if (!(ny > 0)) break;
        k_scale<<<296, 256, 0, st>>>(n, 1.0 / ny, y, x);
        g_prof.launches += 1;
    }
    CK(cudaStreamSynchronize(st));
    *out = lam;
    return HCOV_OK;
}

hcov_status hcov_inv_error(hcov_hmat A, hcov_hmat M, int32_t iters, uint64_t seed, hcov_stream stream, double *out)
{
    if (!A || !M || !out || iters < 1) return HCOV_ERR_INVALID_ARG;
    if (A->state != 1 || M->state < 2) return HCOV_ERR_STATE;
    if (A->t->P.n != M->t->P.n) return HCOV_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = A->t->P.n;
    DiagBufs da;
    hcov_status s;
    if ((s = da.init(A->t->P, A->ctx.kcap))) return s;
    DevBuf B;
    double *x, *y, *e, *w;
    CK(B.get(&x, n)); CK(B.get(&y, n)); CK(B.get(&e, n)); CK(B.get(&w, n));
    k_start_vec<<<296, 256, 0, st>>>(n, seed, x);
    double nx = std::sqrt(dot_dev(x, x, n, da.part, da.res, da.resh, st));
    k_scale<<<296, 256, 0, st>>>(n, 1.0 / nx, x, x);
    g_prof.launches += 2;
    double best = 0.0;
    for (int it = 0; it < iters; ++it) {
        // e = E x = x - M^{-1} A x;  w = E^T e = e - A M^{-1} e  (A, M symmetric)
        if ((s = matvec_ext(A, x, y, da.xi, da.yi, da.t12, st))) return s;
        if ((s = solve_ext(M, y, e, true, true, st))) return s;
        k_axpby<<<296, 256, 0, st>>>(n, 1.0, x, -1.0, e);
        const double ne = std::sqrt(dot_dev(e, e, n, da.part, da.res, da.resh, st));
        best = std::max(best, ne);               // ||E x||, ||x|| = 1: -> ||E||_2
        if ((s = solve_ext(M, e, y, true, true, st))) return s;
        if ((s = matvec_ext(A, y, w, da.xi, da.yi, da.t12, st))) return s;
        k_axpby<<<296, 256, 0, st>>>(n, 1.0, e, -1.0, w);
        const double nw = std::sqrt(dot_dev(w, w, n, da.part, da.res, da.resh, st));
        g_prof.launches += 2;
        if (!(nw > 0)) break;
        k_scale<<<296, 256, 0, st>>>(n, 1.0 / nw, w, x);
        g_prof.launches += 1;
    }
    CK(cudaStreamSynchronize(st));
    *out = best;
    return HCOV_OK;
}

hcov_status hcov_trace_inv(hcov_hmat M, hcov_hmat A, hcov_stream stream, double *out)
{
    if (!M || !A || !out) return HCOV_ERR_INVALID_ARG;
    if (A->state != 1 || M->state < 2) return HCOV_ERR_STATE;
    if (A->t->P.n != M->t->P.n) return HCOV_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = A->t->P.n;
    const int mc = 64;
    DevBuf B;
    double *cols, *x, *acc;
    CK(B.get(&cols, n * mc)); CK(B.get(&x, n)); CK(B.get(&acc, 1));
    CK(cudaMemsetAsync(acc, 0, sizeof(double), st));
    std::vector<int64_t> ids(mc);
    hcov_status s;
    for (int64_t j0 = 0; j0 < n; j0 += mc) {
        const int m = (int)std::min<int64_t>(mc, n - j0);
        for (int k = 0; k < m; ++k) ids[k] = j0 + k;
        if ((s = hcov_columns(A, ids.data(), m, cols, stream))) return s;
        for (int k = 0; k < m; ++k) {
            if ((s = solve_ext(M, cols + n * k, x, true, true, st))) return s;
            k_pick_add<<<1, 32, 0, st>>>(x, j0 + k, acc);
            g_prof.launches += 1;
        }
    }
    CK(cudaMemcpyAsync(out, acc, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return HCOV_OK;
}

hcov_status hcov_sample(hcov_hmat h, const double *xi_dev, double *Z_dev, hcov_stream stream)
{
    if (!h || !xi_dev || !Z_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state < 2) return HCOV_ERR_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    Plan &P = h->t->P;
    double *x = nullptr, *y = nullptr, *tt = nullptr;
    CK(cudaMalloc(&x, P.n_pad * sizeof(double)));
    CK(cudaMalloc(&y, P.n_pad * sizeof(double)));
    CK(cudaMalloc(&tt, std::max<int64_t>(1, P.n_r()) * h->ctx.kcap * sizeof(double)));
    LAUNCH(PC_AUX, st, k_permute_in<<<256, 256, 0, st>>>(h->ctx, xi_dev, x));
    if (P.n_r() > 0) LAUNCH(PC_AUX, st, k_sample_t<<<(int)std::min<int64_t>(P.n_r(), 65535), NT, 0, st>>>(h->ctx, x, tt));
    LAUNCH(PC_AUX, st, k_sample_rows<<<(int)std::min<int64_t>(P.n_leaves, 65535), 32, 0, st>>>(
                           h->ctx, h->t->d_row_off, h->t->d_row_nodes, x, tt, y));
    LAUNCH(PC_AUX, st, k_permute_out<<<256, 256, 0, st>>>(h->ctx, y, Z_dev));
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(x); cudaFree(y); cudaFree(tt);
    if (e != cudaSuccess) return map_err(e);
    CK(cudaGetLastError());
    return HCOV_OK;
}

hcov_status hcov_columns(hcov_hmat h, const int64_t *cols_host, int32_t m, double *out_dev, hcov_stream stream)
{
    if (!h || !cols_host || m < 0 || !out_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state != 1) return HCOV_ERR_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    hcov_tree t = h->t;
    Plan &P = t->P;
    std::vector<int64_t> e2i(P.n, -1);
    for (int64_t p = 0; p < P.n_pad; ++p)
        if (P.perm_i2e[p] >= 0) e2i[P.perm_i2e[p]] = p;
    std::vector<int64_t> pc(m);
    for (int k = 0; k < m; ++k) {
        if (cols_host[k] < 0 || cols_host[k] >= P.n) return HCOV_ERR_INVALID_ARG;
        pc[k] = e2i[cols_host[k]];
    }
    int64_t *d_pc = nullptr;
    double *tmp = nullptr;
    CK(cudaMalloc(&d_pc, std::max(1, m) * sizeof(int64_t)));
    CK(cudaMalloc(&tmp, std::max<int64_t>(1, P.n_pad * m) * sizeof(double)));
    CK(cudaMemcpyAsync(d_pc, pc.data(), m * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    LAUNCH(PC_AUX, st, k_columns<<<std::min(t->n_leafnodes, 65535), NT, 0, st>>>(h->ctx, t->d_leafnodes,
                                                                                 t->n_leafnodes, d_pc, m, tmp));
    LAUNCH(PC_AUX, st, k_columns_perm<<<512, 256, 0, st>>>(h->ctx, tmp, m, out_dev));
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d_pc); cudaFree(tmp);
    if (e != cudaSuccess) return map_err(e);
    return HCOV_OK;
}

hcov_status hcov_cov_columns(hcov_tree t, const hcov_theta *theta, const int64_t *cols_host, int32_t m,
                             double *out_dev, hcov_stream stream)
{
    if (!t || !theta || !cols_host || m < 0 || !out_dev) return HCOV_ERR_INVALID_ARG;
    hcov_trunc tr{0.0, 0, 0};
    hcov_status s = check_theta(theta, &tr);
    if (s) return s;
    if ((s = tree_upload(t))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    Plan &P = t->P;
    std::vector<int64_t> e2i(P.n, -1);
    for (int64_t p = 0; p < P.n_pad; ++p)
        if (P.perm_i2e[p] >= 0) e2i[P.perm_i2e[p]] = p;
    std::vector<int64_t> pc(std::max(1, m));
    for (int k = 0; k < m; ++k) {
        if (cols_host[k] < 0 || cols_host[k] >= P.n) return HCOV_ERR_INVALID_ARG;
        pc[k] = e2i[cols_host[k]];
    }
    Ctx c{};
    c.xs = t->d_xs; c.ys = t->d_ys; c.zs = t->d_zs; c.perm_i2e = t->d_perm_i2e; c.n_pad = P.n_pad; c.n_real = P.n;
    c.mp = hcov_matern_params(theta->sigma2, theta->ell, theta->nu, theta->nugget);   // tab = null: direct K_nu
    int64_t *d_pc = nullptr;
    CK(cudaMalloc(&d_pc, std::max(1, m) * sizeof(int64_t)));
    CK(cudaMemcpyAsync(d_pc, pc.data(), m * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    LAUNCH(PC_AUX, st, k_cov_columns<<<1184, 256, 0, st>>>(c, d_pc, m, out_dev));
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d_pc);
    if (e != cudaSuccess) return map_err(e);
    return HCOV_OK;
}

hcov_status hcov_hmat_mem_info(hcov_hmat h, int64_t *out)
{
    if (!h || !out) return HCOV_ERR_INVALID_ARG;
    const Plan &P = h->t->P;
    const int64_t kc = std::max(0, h->kcap_alloc);
    unsigned long long mem[4] = {0, 0, 0, 0};
    if (h->mem) CK(cudaMemcpy(mem, h->mem, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    out[0] = P.n_tiles() * HCOV_TILE * 8;
    out[1] = 2 * P.uv_elems * kc * 8;
    out[2] = (int64_t)P.n_cores * std::max(0, h->kcore_alloc) * std::max(0, h->kcore_alloc) * 8;
    out[3] = h->wcap * 8;
    out[4] = h->pcap * 8;
    out[5] = (int64_t)mem[0] * 8;
    out[6] = (int64_t)mem[1] * 8;
    out[7] = (int64_t)mem[2];
    return HCOV_OK;
}

hcov_status hcov_hmat_storage(hcov_hmat h, int64_t *dense_bytes, int64_t *lowrank_bytes, int32_t *max_rank)
{
    if (!h || !dense_bytes || !lowrank_bytes || !max_rank) return HCOV_ERR_INVALID_ARG;
    Plan &P = h->t->P;
    std::vector<int32_t> rk(P.n_r());
    if (P.n_r()) CK(cudaMemcpy(rk.data(), h->rank, P.n_r() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    int64_t lr = 0;
    int32_t mx = 0;
    for (int64_t r = 0; r < P.n_r(); ++r) { lr += 2 * (int64_t)P.rblk[r].m * rk[r] * 8; mx = std::max(mx, rk[r]); }
    *dense_bytes = P.n_tiles() * HCOV_TILE * 8;
    *lowrank_bytes = lr;
    *max_rank = mx;
    return HCOV_OK;
}

hcov_status hcov_tree_last_eval(hcov_tree t, hcov_hmat *out)
{
    if (!t || !out) return HCOV_ERR_INVALID_ARG;
    *out = t->cached;
    return t->cached ? HCOV_OK : HCOV_ERR_STATE;
}

hcov_status hcov_model_flops(hcov_hmat h, double *out)
{
    // SURVEY.md Sec. 8(d) / App. A.3 method-work model at the MEASURED final ranks r_b of L~:
    // every Schur-complement term applied to every leaf it covers, low-rank targets truncated
    // eagerly after each term (4 m R^2 + 22 R^3 + 4 m R r_b with R = r_b + term width), tile updates,
    // POTRF / TRSM, the V <- L^{-1} V solves and W = H V products as 2 x (words of the operator) x
    // (columns), the ACA output truncation, and the root forward solve (2 x words of L~).
    if (!h || !out) return HCOV_ERR_INVALID_ARG;
    if (h->state < 2) return HCOV_ERR_STATE;
    const Plan &P = h->t->P;
    std::vector<int32_t> rk(std::max<int64_t>(1, P.n_r()), 0);
    if (P.n_r()) CK(cudaMemcpy(rk.data(), h->rank, P.n_r() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    auto ncols = [&](int f) { return (double)rk[P.fac_rank_src[f]]; };
    auto trunc = [](double m, double R, double r) { return 4.0 * m * R * R + 22.0 * R * R * R + 4.0 * m * R * r; };
    // words of L~ below each node (lower triangle)
    std::vector<double> words(P.nodes.size(), 0.0);
    for (int64_t k = (int64_t)P.nodes.size() - 1; k >= 0; --k) {   // children have larger ids (preorder)
        const DNode &x = P.nodes[k];
        if (x.type == ND_T) words[k] = HCOV_TILE;
        else if (x.type == ND_R) words[k] = 2.0 * P.rblk[x.idx].m * rk[x.idx];
        else
            for (int c = 0; c < 4; ++c)
                if (P.children[4 * k + c] >= 0) words[k] += words[P.children[4 * k + c]];
    }
    std::vector<int32_t> diag_node(P.n_clusters, -1);
    for (size_t k = 0; k < P.nodes.size(); ++k)
        if (P.nodes[k].i == P.nodes[k].j) diag_node[((int64_t)1 << P.nodes[k].level) - 1 + P.nodes[k].i] = (int32_t)k;
    double f_trunc = 0, f_prod = 0, f_tile = 0, f_solve = 0, f_potrf = 0, f_aca = 0, f_root = 0;
    for (int64_t r = 0; r < P.n_r(); ++r) f_aca += trunc(P.rblk[r].m, rk[r], rk[r]);
    for (const DTask &tk : P.tasks) {
        switch (tk.type) {
        case TK_TAPP: case TK_POTRF: case TK_TRSM:
            for (int k = tk.b; k < tk.c; ++k) {
                const DTerm &t = P.terms[P.xterm[k]];
                if (t.kind == TM_TT) f_tile += 2.0 * 32 * 32 * 32;
                else {
                    const double ra = ncols(t.a), rb = ncols(t.b);
                    f_tile += 2.0 * 32 * 32 * rb + (t.core >= 0 ? 2.0 * 32 * ra * rb : 0.0);
                }
            }
            if (tk.type == TK_POTRF) f_potrf += 32.0 * 32 * 32 / 3.0;
            if (tk.type == TK_TRSM) f_tile += 32.0 * 32 * 32;
            break;
        case TK_RAPP: {
            const double m = P.rblk[tk.a].m, ro = rk[tk.a];
            for (int k = tk.b; k < tk.c; ++k) {
                const DTerm &t = P.terms[P.xterm[k]];
                double w = 32.0;
                if (t.kind == TM_LR) {
                    w = ncols(t.b);
                    if (w == 0 || ncols(t.a) == 0) continue;
                    if (t.core >= 0) f_prod += 2.0 * m * ncols(t.a) * w;
                }
                f_trunc += trunc(m, ro + w, ro);
            }
            break;
        }
        case TK_PRR: f_prod += 2.0 * P.rblk[tk.a].m * rk[tk.a] * rk[tk.b]; break;
        default: break;
        }
    }
    for (size_t s = 0; s < P.solves.size(); ++s) {
        const DSolve &sv = P.solves[s];
        const int32_t dn = diag_node[((int64_t)1 << sv.level) - 1 + sv.c];
        if ((int)s == P.root_solve) { f_root += 2.0 * words[dn]; continue; }
        double cols = 0;
        for (int q = 0; q < sv.rhs_cnt; ++q) cols += rk[P.solve_rhs[sv.rhs_off + q]];
        f_solve += 2.0 * words[dn] * cols;
    }
    for (const DPhw &q : P.phw) {
        double cols = 0;
        for (int p = 0; p < q.part_cnt; ++p) cols += rk[P.col_r[q.part_off + p]];
        f_prod += 2.0 * words[q.hnode] * cols;
    }
    out[1] = f_trunc; out[2] = f_prod; out[3] = f_tile; out[4] = f_solve; out[5] = f_potrf; out[6] = f_aca;
    out[7] = f_root;
    out[0] = f_trunc + f_prod + f_tile + f_solve + f_potrf + f_aca + f_root;
    return HCOV_OK;
}

hcov_status hcov_prof_control(int32_t enable_events, int32_t reset)
{
    if (reset) {
        prof_collect();
        g_prof.launches = 0;
        for (int k = 0; k < PC_N; ++k) { g_prof.count[k] = 0; g_prof.ms[k] = 0.0; }
        for (int k = 0; k < TK_NTYPES; ++k) { g_prof.busy_ns[k] = 0; g_prof.tasks[k] = 0; }
        for (int k = 0; k < FC_N; ++k) g_prof.flop[k] = 0;
        for (int k = 0; k < 64; ++k) g_prof.phase_ns[k] = 0;
    }
    g_prof.events = enable_events != 0;
    return HCOV_OK;
}

hcov_status hcov_prof_read(hcov_prof *out)
{
    if (!out) return HCOV_ERR_INVALID_ARG;
    prof_collect();
    std::memset(out, 0, sizeof(*out));
    out->launches = g_prof.launches;
    out->n_classes = PC_N;
    for (int k = 0; k < PC_N; ++k) {
        out->ms[k] = g_prof.ms[k];
        out->count[k] = g_prof.count[k];
    }
    out->n_task_types = TK_NTYPES;
    for (int k = 0; k < TK_NTYPES; ++k) {
        out->task_busy_ms[k] = g_prof.busy_ns[k] * 1e-6;
        out->task_count[k] = g_prof.tasks[k];
    }
    for (int k = 0; k < FC_N; ++k) out->flop[k] = g_prof.flop[k];
    for (int k = 0; k < 64; ++k) {
        out->phase_ms[k % 16] += g_prof.phase_ns[k] * 1e-6;
        out->phase_cls_ms[k] = g_prof.phase_ns[k] * 1e-6;
    }
    return HCOV_OK;
}

const char *hcov_prof_class_name(int32_t cls)
{
    return (cls >= 0 && cls < PC_N) ? PROF_NAMES[cls] : "";
}

const char *hcov_prof_task_name(int32_t type)
{
    return (type >= 0 && type < TK_NTYPES) ? TASK_NAMES[type] : "";
}

hcov_status hcov_test_truncate(const double *X_dev, const double *Y_dev, int64_t m, int32_t R, double eps,
                               int32_t kmax, int32_t rlim, int32_t path, double *U_dev, double *V_dev,
                               int32_t *out3_host)
{
    if (!X_dev || !Y_dev || !U_dev || !V_dev || !out3_host || m < 1 || R < 0 || R > 224 || rlim < 1) return HCOV_ERR_INVALID_ARG;
    if (path == 3 && m > HCOV_DENSE_MAX) return HCOV_ERR_INVALID_ARG;
    const int K = path == 3 ? (int)std::max<int64_t>(m, R) : (R > 0 ? R : 1);
    const int64_t need = (path == 3 ? m * m : 0) + 6 * m * K + 8 * (int64_t)K * K + 10 * K + m / 8 + 64;
    double *scr = nullptr;
    int *rk = nullptr;
    CK(cudaMalloc(&scr, need * sizeof(double)));
    CK(cudaMalloc(&rk, 3 * sizeof(int)));
    if (path != 3) {
        CK(cudaMemcpy(scr, X_dev, m * (int64_t)R * sizeof(double), cudaMemcpyDeviceToDevice));
        CK(cudaMemcpy(scr + m * K, Y_dev, m * (int64_t)R * sizeof(double), cudaMemcpyDeviceToDevice));
    }
    const int64_t smem = HCOV_SMEM_DBL * sizeof(double);
    CK(cudaFuncSetAttribute(k_test_truncate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_test_truncate<<<1, NT, smem, 0>>>(scr, m, R, K, eps, kmax, rlim, path, U_dev, V_dev, rk, HCOV_SMEM_DBL,
                                        X_dev, Y_dev);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(out3_host, rk, 3 * sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(scr);
    cudaFree(rk);
    return e == cudaSuccess ? HCOV_OK : map_err(e);
}

void hcov_tree_free(hcov_tree t) { delete t; }
void hcov_hmat_free(hcov_hmat h) { delete h; }

}  // extern "C"
