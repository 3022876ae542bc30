// libhcov: C ABI (include/hcov.h) + kernels + wave executor.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

#include "../../include/hcov.h"
#include "plan.h"
#include "tasks.cuh"

namespace {

#define CK(x)                                                 \
    do {                                                      \
        cudaError_t e_ = (x);                                 \
        if (e_ != cudaSuccess) return map_err(e_);            \
    } while (0)

hcov_status map_err(cudaError_t e)
{
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
// instrumentation: launch counter and per-class CUDA-event timing (hcov_prof_*)
// ------------------------------------------------------------------------------------------
enum ProfCls { PC_FILL = 0, PC_ACA = 1, PC_POTRF = 2, PC_TRSM = 3, PC_RFIN = 4, PC_LRSOLVE = 5, PC_PRR = 6,
               PC_PHW = 7, PC_FWD = 8, PC_REDUCE = 9, PC_AUX = 10, PC_N = 11 };
const char *const PROF_NAMES[PC_N] = {"fill_tiles", "aca_trunc", "potrf", "trsm", "rfin", "lr_solve", "prr",
                                      "phw", "fwd_solve", "reduce", "aux"};
struct ProfEv { int cls; cudaEvent_t a, b; };
struct Prof {
    int64_t launches = 0;
    int64_t count[PC_N] = {};
    bool events = false;
    std::vector<ProfEv> evs;
    std::vector<cudaEvent_t> pool;
    double ms[PC_N] = {};
};
Prof g_prof;

cudaEvent_t prof_event()
{
    if (!g_prof.pool.empty()) { cudaEvent_t e = g_prof.pool.back(); g_prof.pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
// Open a launch record of class cls on stream st; returns the index to close.
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
// kernels
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_fill_tiles(Ctx c, int64_t ntiles)
{
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const DNode x = c.nodes[c.tile_node[t]];
        const int64_t r0 = (int64_t)x.i * HCOV_LEAF, c0 = (int64_t)x.j * HCOV_LEAF;
        double *T = c.tiles + t * HCOV_TILE;
        for (int e = threadIdx.x; e < HCOV_TILE; e += NT) {
            int i = e & 31, j = e >> 5;
            int64_t a = r0 + i, b = c0 + j;
            T[e] = hcov_cov_entry(c.mp, c.xs[a], c.ys[a], c.xs[b], c.ys[b], a == b);
        }
    }
}

__global__ void __launch_bounds__(NT) k_assemble_r(Ctx c, const int32_t *list, int cnt, int cls)
{
    __shared__ double red[NWARP], redv[NWARP];
    __shared__ int64_t redi[NWARP];
    double *scr = c.scr[cls] + c.scr_stride[cls] * blockIdx.x;
    for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
        const int r = list[q];
        const DRBlk b = c.rblk[r];
        const int64_t m = b.m;
        const int K = aca_kmax(m, c.kcap);
        CompressWs w = make_ws(scr, m, K);
        uint8_t *used = (uint8_t *)(w.ord + K + 2);
        int k = aca_partial(c.mp, c.xs, c.ys, b.row0, b.col0, m, w.X, w.Y, K, 0.1 * c.eps, used, red, redv, redi);
        int cb = 0, of = 0;
        int rk = compress(w, m, k, c.eps, c.kmax, c.kcap, r_U(c, r), r_V(c, r), m, &cb, &of, red);
        record_rank(c, r, rk, cb, of);
    }
}

__global__ void __launch_bounds__(NT) k_exec(Ctx c, const int32_t *ids, int cnt, int cls)
{
    extern __shared__ double smem[];
    __shared__ double red[NWARP], redv[NWARP];
    __shared__ int64_t redi[NWARP];
    double *scr = c.scr[cls] ? c.scr[cls] + c.scr_stride[cls] * blockIdx.x : nullptr;
    for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
        const DTask tk = c.tasks[ids[q]];
        switch (tk.type) {
        case TK_POTRF: task_potrf(c, tk, smem); break;
        case TK_TRSM: task_trsm(c, tk, smem); break;
        case TK_RFIN: task_rfin(c, tk, scr, red, redv, redi); break;
        case TK_SOLVE: task_solve(c, tk, scr, smem); break;
        case TK_PRR: task_prr(c, tk); break;
        case TK_PHW: task_phw(c, tk, smem, smem + HCOV_TILE); break;
        default: break;
        }
        __syncthreads();
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

// Forward solve v = L^{-1} y over the whole matrix (root program), one CTA.
__global__ void __launch_bounds__(NT) k_fwd_solve(Ctx c, double *y, double *tscr)
{
    __shared__ double smL[HCOV_TILE];
    run_solve_program(c, 0, 0, c.n_pad, y, 1, tscr, smL);
}

// out[0] = log det, out[1] = quad, out[2] = min pivot (fixed-order reductions, one CTA)
__global__ void __launch_bounds__(NT) k_reduce(Ctx c, const double *v, double *out)
{
    __shared__ double red[NWARP];
    double ld = 0.0, q = 0.0, mp = INFINITY;
    for (int64_t k = threadIdx.x; k < c.n_leaves; k += NT) { ld += c.logdet_part[k]; mp = fmin(mp, c.minpiv_part[k]); }
    for (int64_t k = threadIdx.x; k < c.n_pad; k += NT) q += v[k] * v[k];
    ld = block_sum(ld, red);
    q = block_sum(q, red);
    // min
    __shared__ double mred[NT];
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
// y_seg = sum over the row's blocks (T: tile x_cols; R: U[seg rows] t_b)
__global__ void __launch_bounds__(32) k_sample_rows(Ctx c, const double *x, const double *t, double *y)
{
    for (int64_t seg = blockIdx.x; seg < c.n_leaves; seg += gridDim.x) {
        const int i = threadIdx.x;
        double s = 0.0;
        for (int k = c.row_off[seg]; k < c.row_off[seg + 1]; ++k) {
            const DNode nd = c.nodes[c.row_nodes[k]];
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

// hcov_columns: out (n_pad x m internal rows) for internal columns pc[k].
__global__ void __launch_bounds__(NT) k_columns(Ctx c, const int32_t *leafnodes, int nleafnodes, const int64_t *pc, int mcols,
                                                double *out)
{
    for (int q = blockIdx.x; q < nleafnodes; q += gridDim.x) {
        const DNode nd = c.nodes[leafnodes[q]];
        const int64_t mb = cl_size(c, nd.level);
        const int64_t r0 = (int64_t)nd.i * mb, c0 = (int64_t)nd.j * mb;
        for (int k = 0; k < mcols; ++k) {
            const int64_t p = pc[k];
            double *o = out + c.n_pad * (int64_t)k;
            if (p >= c0 && p < c0 + mb) {   // column part: rows r0..r0+mb
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
            if (nd.i != nd.j && p >= r0 && p < r0 + mb) {   // transposed part: rows c0..c0+mb
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
__global__ void k_columns_perm(Ctx c, const double *in, int mcols, double *out)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c.n_pad * (int64_t)mcols;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = e % c.n_pad, k = e / c.n_pad;
        int64_t ex = c.perm_i2e[p];
        if (ex >= 0) out[ex + c.n_real * k] = in[e];
    }
}

}  // namespace

// ------------------------------------------------------------------------------------------
// handles
// ------------------------------------------------------------------------------------------
struct Launch {
    int32_t type, cls, off, cnt;
};

struct hcov_tree_s {
    Plan P;
    bool uploaded = false;
    // device plan arrays
    DNode *d_nodes = nullptr;
    int32_t *d_children = nullptr;
    DTerm *d_terms = nullptr;
    DTask *d_tasks = nullptr;
    DRBlk *d_rblk = nullptr;
    int32_t *d_tile_node = nullptr;
    DPhw *d_phw = nullptr;
    int32_t *d_phw_part = nullptr, *d_hleaf = nullptr, *d_col_r_off = nullptr, *d_col_r = nullptr;
    DOp *d_ops = nullptr;
    int32_t *d_op_beg = nullptr, *d_op_end = nullptr;
    int64_t *d_fac_row0 = nullptr;
    int32_t *d_fac_nrows = nullptr, *d_fac_rank_src = nullptr;
    int64_t *d_fac_off = nullptr;
    int8_t *d_fac_pool = nullptr;
    int32_t *d_row_off = nullptr, *d_row_nodes = nullptr;
    double *d_xs = nullptr, *d_ys = nullptr;
    int64_t *d_perm_i2e = nullptr;
    int32_t *d_exec_ids = nullptr;
    int32_t *d_asm_ids = nullptr;
    int32_t *d_leafnodes = nullptr;
    int32_t n_leafnodes = 0;
    // schedule, computed for a given kcap
    int32_t sched_kcap = -1;
    std::vector<Launch> launches;
    std::vector<Launch> asm_launches;
    int64_t scr_need[2] = {0, 0};
    int32_t scr_slots[2] = {0, 0};
    hcov_hmat cached = nullptr;
    ~hcov_tree_s();
};

struct hcov_hmat_s {
    hcov_tree t = nullptr;
    Ctx ctx{};
    hcov_theta theta{};
    hcov_trunc trunc{};
    int state = 0;   // 1 assembled, 2 factored
    double *tiles = nullptr, *U = nullptr, *V = nullptr, *cores = nullptr, *W = nullptr;
    double *logdet_part = nullptr, *minpiv_part = nullptr;
    int32_t *rank = nullptr, *fail = nullptr, *flags = nullptr;
    double *scr[2] = {nullptr, nullptr};
    double *vbuf = nullptr, *tbuf = nullptr, *res = nullptr, *res_host = nullptr;
    ~hcov_hmat_s()
    {
        cudaFree(tiles); cudaFree(U); cudaFree(V); cudaFree(cores); cudaFree(W);
        cudaFree(logdet_part); cudaFree(minpiv_part); cudaFree(rank); cudaFree(fail); cudaFree(flags);
        cudaFree(scr[0]); cudaFree(scr[1]); cudaFree(vbuf); cudaFree(tbuf); cudaFree(res);
        if (res_host) cudaFreeHost(res_host);
    }
};

hcov_tree_s::~hcov_tree_s()
{
    if (cached) delete cached;
    void *ps[] = {d_nodes, d_children, d_terms, d_tasks, d_rblk, d_tile_node, d_phw, d_phw_part, d_hleaf,
                  d_col_r_off, d_col_r, d_ops, d_op_beg, d_op_end, d_fac_row0, d_fac_nrows, d_fac_rank_src,
                  d_fac_off, d_fac_pool, d_row_off, d_row_nodes, d_xs, d_ys, d_perm_i2e, d_exec_ids, d_asm_ids,
                  d_leafnodes};
    for (void *p : ps) cudaFree(p);
}

namespace {

const int SMALL_SLOTS = 296;
const int BIG_SLOTS_MAX = 8;
const int64_t SMALL_LIMIT = (int64_t)3 << 20;   // doubles (24 MB) per small slot at most

hcov_status tree_upload(hcov_tree t)
{
    if (t->uploaded) return HCOV_OK;
    Plan &P = t->P;
    CK(upload(&t->d_nodes, P.nodes));
    CK(upload(&t->d_children, P.children));
    CK(upload(&t->d_terms, P.terms));
    CK(upload(&t->d_tasks, P.tasks));
    CK(upload(&t->d_rblk, P.rblk));
    CK(upload(&t->d_tile_node, P.tile_node));
    CK(upload(&t->d_phw, P.phw));
    CK(upload(&t->d_phw_part, P.phw_part));
    CK(upload(&t->d_hleaf, P.hleaf));
    CK(upload(&t->d_col_r_off, P.col_r_off));
    CK(upload(&t->d_col_r, P.col_r));
    CK(upload(&t->d_ops, P.ops));
    CK(upload(&t->d_op_beg, P.op_beg));
    CK(upload(&t->d_op_end, P.op_end));
    CK(upload(&t->d_fac_row0, P.fac_row0));
    CK(upload(&t->d_fac_nrows, P.fac_nrows));
    CK(upload(&t->d_fac_rank_src, P.fac_rank_src));
    CK(upload(&t->d_fac_off, P.fac_off));
    CK(upload(&t->d_fac_pool, P.fac_pool));
    CK(upload(&t->d_row_off, P.row_off));
    CK(upload(&t->d_row_nodes, P.row_nodes));
    CK(upload(&t->d_xs, P.xs));
    CK(upload(&t->d_ys, P.ys));
    CK(upload(&t->d_perm_i2e, P.perm_i2e));
    std::vector<int32_t> leafnodes;
    for (size_t k = 0; k < P.nodes.size(); ++k)
        if (P.nodes[k].type != ND_H) leafnodes.push_back((int32_t)k);
    t->n_leafnodes = (int32_t)leafnodes.size();
    CK(upload(&t->d_leafnodes, leafnodes));
    t->uploaded = true;
    return HCOV_OK;
}

// Group the tasks of every wave by (type, scratch class) for a given rank capacity.
hcov_status tree_schedule(hcov_tree t, int kcap)
{
    if (t->sched_kcap == kcap) return HCOV_OK;
    Plan &P = t->P;
    const size_t nt = P.tasks.size();
    std::vector<int64_t> need(nt, 0);
    for (size_t k = 0; k < nt; ++k) {
        const DTask &tk = P.tasks[k];
        if (tk.type == TK_RFIN) {
            const DRBlk &b = P.rblk[P.nodes[tk.a].idx];
            need[k] = rfin_scratch(b.m, kcap);
        } else if (tk.type == TK_SOLVE) {
            int level = 0;
            while ((((int64_t)2 << level) - 1) <= tk.a) ++level;
            int64_t msig = P.cluster_size(level);
            int cnt = P.col_r_off[tk.a + 1] - P.col_r_off[tk.a];
            need[k] = solve_scratch(msig, cnt * kcap, kcap);
        }
    }
    int64_t nsmall = 0, nbig = 0;
    std::vector<int8_t> cls(nt, 0);
    for (size_t k = 0; k < nt; ++k) {
        if (need[k] == 0) continue;
        if (need[k] <= SMALL_LIMIT) { cls[k] = 0; nsmall = std::max(nsmall, need[k]); }
        else { cls[k] = 1; nbig = std::max(nbig, need[k]); }
    }
    // assembly requirements
    std::vector<int32_t> asm_small, asm_big;
    for (size_t r = 0; r < P.rblk.size(); ++r) {
        int64_t nd = assemble_scratch(P.rblk[r].m, kcap);
        if (nd <= SMALL_LIMIT) { asm_small.push_back((int32_t)r); nsmall = std::max(nsmall, nd); }
        else { asm_big.push_back((int32_t)r); nbig = std::max(nbig, nd); }
    }
    t->scr_need[0] = nsmall;
    t->scr_need[1] = nbig;
    // exec order: by wave, then type, then class, then generation order
    std::vector<int32_t> ids(P.wave_tasks);
    std::stable_sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) {
        if (P.task_wave[a] != P.task_wave[b]) return P.task_wave[a] < P.task_wave[b];
        if (P.tasks[a].type != P.tasks[b].type) return P.tasks[a].type < P.tasks[b].type;
        return cls[a] < cls[b];
    });
    t->launches.clear();
    int32_t maxbig = 0, maxsmall = 0;
    for (size_t k = 0; k < ids.size();) {
        size_t e = k;
        const int32_t w = P.task_wave[ids[k]], ty = P.tasks[ids[k]].type, c = cls[ids[k]];
        while (e < ids.size() && P.task_wave[ids[e]] == w && P.tasks[ids[e]].type == ty && cls[ids[e]] == c) ++e;
        t->launches.push_back(Launch{ty, c, (int32_t)k, (int32_t)(e - k)});
        if (need[ids[k]] > 0) {
            if (c == 1) maxbig = std::max(maxbig, (int32_t)(e - k));
            else maxsmall = std::max(maxsmall, (int32_t)(e - k));
        }
        k = e;
    }
    std::vector<int32_t> asm_ids(asm_small);
    asm_ids.insert(asm_ids.end(), asm_big.begin(), asm_big.end());
    t->asm_launches.clear();
    if (!asm_small.empty()) t->asm_launches.push_back(Launch{-1, 0, 0, (int32_t)asm_small.size()});
    if (!asm_big.empty()) t->asm_launches.push_back(Launch{-1, 1, (int32_t)asm_small.size(), (int32_t)asm_big.size()});
    maxsmall = std::max(maxsmall, (int32_t)asm_small.size());
    maxbig = std::max(maxbig, (int32_t)asm_big.size());
    t->scr_slots[0] = nsmall ? std::min(SMALL_SLOTS, std::max(1, maxsmall)) : 0;
    t->scr_slots[1] = nbig ? std::min(BIG_SLOTS_MAX, std::max(1, maxbig)) : 0;
    cudaFree(t->d_exec_ids);
    cudaFree(t->d_asm_ids);
    t->d_exec_ids = nullptr;
    t->d_asm_ids = nullptr;
    CK(upload(&t->d_exec_ids, ids));
    CK(upload(&t->d_asm_ids, asm_ids));
    t->sched_kcap = kcap;
    return HCOV_OK;
}

int64_t exec_smem_bytes(int kcap)
{
    int64_t a = tile_smem_doubles(kcap);
    int64_t b = HCOV_TILE + (int64_t)kcap * kcap + 64;
    return std::max(a, b) * (int64_t)sizeof(double);
}

hcov_status check_theta(const hcov_theta *th, const hcov_trunc *tr)
{
    if (!th || !tr) return HCOV_ERR_INVALID_ARG;
    if (!(th->sigma2 > 0) || !(th->ell > 0) || !(th->nu > 0) || !(th->nugget >= 0)) return HCOV_ERR_INVALID_ARG;
    if (!std::isfinite(th->sigma2) || !std::isfinite(th->ell) || !std::isfinite(th->nu) || !std::isfinite(th->nugget))
        return HCOV_ERR_INVALID_ARG;
    if (!(tr->eps >= 0) || tr->kmax < 0 || tr->kcap < 0 || tr->kcap > 256) return HCOV_ERR_INVALID_ARG;
    if (tr->kmax > 0 && tr->kcap > 0 && tr->kmax > tr->kcap) return HCOV_ERR_INVALID_ARG;
    return HCOV_OK;
}

int eff_kcap(const hcov_trunc *tr)
{
    if (tr->kcap > 0) return tr->kcap;
    if (tr->kmax > 0) return tr->kmax;
    return 64;
}

// (Re)allocate the numeric buffers of h for the tree's plan and capacity kcap.
hcov_status hmat_alloc(hcov_hmat h, int kcap)
{
    hcov_tree t = h->t;
    Plan &P = t->P;
    if (h->tiles && h->ctx.kcap == kcap) return HCOV_OK;
    cudaFree(h->tiles); cudaFree(h->U); cudaFree(h->V); cudaFree(h->cores); cudaFree(h->W);
    cudaFree(h->logdet_part); cudaFree(h->minpiv_part); cudaFree(h->rank); cudaFree(h->fail); cudaFree(h->flags);
    cudaFree(h->scr[0]); cudaFree(h->scr[1]); cudaFree(h->vbuf); cudaFree(h->tbuf); cudaFree(h->res);
    h->tiles = h->U = h->V = h->cores = h->W = h->logdet_part = h->minpiv_part = nullptr;
    h->rank = h->fail = h->flags = nullptr;
    h->scr[0] = h->scr[1] = h->vbuf = h->tbuf = h->res = nullptr;
    CK(cudaMalloc(&h->tiles, std::max<int64_t>(1, P.n_tiles()) * HCOV_TILE * sizeof(double)));
    CK(cudaMalloc(&h->U, std::max<int64_t>(1, P.uv_elems * kcap) * sizeof(double)));
    CK(cudaMalloc(&h->V, std::max<int64_t>(1, P.uv_elems * kcap) * sizeof(double)));
    CK(cudaMalloc(&h->cores, std::max<int64_t>(1, (int64_t)P.n_cores * kcap * kcap) * sizeof(double)));
    CK(cudaMalloc(&h->W, std::max<int64_t>(1, P.w_elems * kcap) * sizeof(double)));
    CK(cudaMalloc(&h->logdet_part, P.n_leaves * sizeof(double)));
    CK(cudaMalloc(&h->minpiv_part, P.n_leaves * sizeof(double)));
    CK(cudaMalloc(&h->rank, std::max<int64_t>(1, P.n_r()) * sizeof(int32_t)));
    CK(cudaMalloc(&h->fail, sizeof(int32_t)));
    CK(cudaMalloc(&h->flags, 4 * sizeof(int32_t)));
    for (int k = 0; k < 2; ++k)
        if (t->scr_slots[k] > 0) CK(cudaMalloc(&h->scr[k], t->scr_need[k] * t->scr_slots[k] * sizeof(double)));
    CK(cudaMalloc(&h->vbuf, P.n_pad * sizeof(double)));
    CK(cudaMalloc(&h->tbuf, std::max<int64_t>((int64_t)kcap * kcap + 64, std::max<int64_t>(1, P.n_r()) * kcap) * sizeof(double)));
    CK(cudaMalloc(&h->res, 8 * sizeof(double)));
    if (!h->res_host) CK(cudaMallocHost(&h->res_host, 8 * sizeof(double)));
    return HCOV_OK;
}

void fill_ctx(hcov_hmat h)
{
    hcov_tree t = h->t;
    Plan &P = t->P;
    Ctx &c = h->ctx;
    c.nodes = t->d_nodes; c.children = t->d_children; c.terms = t->d_terms; c.tasks = t->d_tasks;
    c.rblk = t->d_rblk; c.tile_node = t->d_tile_node; c.phw = t->d_phw; c.phw_part = t->d_phw_part;
    c.hleaf = t->d_hleaf; c.col_r_off = t->d_col_r_off; c.col_r = t->d_col_r; c.ops = t->d_ops;
    c.op_beg = t->d_op_beg; c.op_end = t->d_op_end; c.fac_row0 = t->d_fac_row0; c.fac_nrows = t->d_fac_nrows;
    c.fac_rank_src = t->d_fac_rank_src; c.fac_off = t->d_fac_off; c.fac_pool = t->d_fac_pool;
    c.row_off = t->d_row_off; c.row_nodes = t->d_row_nodes; c.xs = t->d_xs; c.ys = t->d_ys;
    c.perm_i2e = t->d_perm_i2e;
    c.depth = P.depth; c.n_r = (int32_t)P.n_r(); c.n_pad = P.n_pad; c.n_leaves = P.n_leaves; c.n_real = P.n;
    c.tiles = h->tiles; c.U = h->U; c.V = h->V; c.rank = h->rank; c.cores = h->cores; c.W = h->W;
    c.logdet_part = h->logdet_part; c.minpiv_part = h->minpiv_part; c.fail_leaf = h->fail; c.flags = h->flags;
    c.kmax = h->trunc.kmax; c.eps = h->trunc.eps;
    c.mp = hcov_matern_params(h->theta.sigma2, h->theta.ell, h->theta.nu, h->theta.nugget);
    for (int k = 0; k < 2; ++k) { c.scr[k] = h->scr[k]; c.scr_stride[k] = t->scr_need[k]; }
}

hcov_status assemble_into(hcov_hmat h, const hcov_theta *theta, const hcov_trunc *trunc, cudaStream_t st)
{
    hcov_tree t = h->t;
    const int kcap = eff_kcap(trunc);
    hcov_status s = tree_upload(t);
    if (s) return s;
    if ((s = tree_schedule(t, kcap))) return s;
    if ((s = hmat_alloc(h, kcap))) return s;
    h->theta = *theta;
    h->trunc = *trunc;
    h->ctx.kcap = kcap;
    fill_ctx(h);
    Plan &P = t->P;
    CK(cudaMemsetAsync(h->rank, 0, std::max<int64_t>(1, P.n_r()) * sizeof(int32_t), st));
    CK(cudaMemsetAsync(h->flags, 0, 4 * sizeof(int32_t), st));
    CK(cudaMemsetAsync(h->fail, 0x7f, sizeof(int32_t), st));
    if (P.n_tiles() > 0) {
        int grid = (int)std::min<int64_t>(P.n_tiles(), 148 * 16);
        LAUNCH(PC_FILL, st, k_fill_tiles<<<grid, NT, 0, st>>>(h->ctx, P.n_tiles()));
    }
    for (const Launch &L : t->asm_launches) {
        int grid = std::min(L.cnt, t->scr_slots[L.cls]);
        LAUNCH(PC_ACA, st, k_assemble_r<<<grid, NT, 0, st>>>(h->ctx, t->d_asm_ids + L.off, L.cnt, L.cls));
    }
    CK(cudaGetLastError());
    h->state = 1;
    return HCOV_OK;
}

hcov_status cholesky_run(hcov_hmat h, cudaStream_t st, int64_t *fail_leaf)
{
    if (!h || h->state != 1) return HCOV_ERR_STATE;
    hcov_tree t = h->t;
    const int64_t smem = exec_smem_bytes(h->ctx.kcap);
    CK(cudaFuncSetAttribute(k_exec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (const Launch &L : t->launches) {
        int grid;
        const bool scratch = (L.type == TK_RFIN || L.type == TK_SOLVE);
        if (scratch) grid = std::min(L.cnt, t->scr_slots[L.cls]);
        else grid = std::min(L.cnt, 65535);
        Ctx c = h->ctx;
        if (!scratch) { c.scr[0] = c.scr[1] = nullptr; }
        static const int cls_of[7] = {PC_POTRF, PC_TRSM, PC_RFIN, PC_LRSOLVE, PC_PRR, PC_PHW, PC_AUX};
        LAUNCH(cls_of[L.type], st, k_exec<<<grid, NT, smem, st>>>(c, t->d_exec_ids + L.off, L.cnt, scratch ? L.cls : 0));
    }
    CK(cudaGetLastError());
    int32_t hf[5];
    CK(cudaMemcpyAsync(hf, h->fail, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hf + 1, h->flags, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    h->state = 2;
    int64_t fl = (hf[0] == 0x7f7f7f7f) ? -1 : hf[0];
    if (fail_leaf) *fail_leaf = fl;
    if (fl >= 0) return HCOV_ERR_NOT_SPD;
    if (hf[2] > 0 && h->trunc.kmax == 0) return HCOV_ERR_RANK_CAPACITY;
    return HCOV_OK;
}

hcov_status loglik_run(hcov_hmat h, const double *Z, cudaStream_t st, hcov_result *out)
{
    if (!h || h->state != 2) return HCOV_ERR_STATE;
    Plan &P = h->t->P;
    LAUNCH(PC_REDUCE, st, k_permute_in<<<256, 256, 0, st>>>(h->ctx, Z, h->vbuf));
    LAUNCH(PC_FWD, st, k_fwd_solve<<<1, NT, 0, st>>>(h->ctx, h->vbuf, h->tbuf));
    LAUNCH(PC_REDUCE, st, k_reduce<<<1, NT, 0, st>>>(h->ctx, h->vbuf, h->res));
    CK(cudaGetLastError());
    int32_t hf[5];
    CK(cudaMemcpyAsync(h->res_host, h->res, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hf, h->fail, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hf + 1, h->flags, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const double ld = h->res_host[0], q = h->res_host[1];
    out->n = P.n;
    out->logdet = ld;
    out->quad = q;
    out->loglik = -0.5 * (double)P.n * std::log(2.0 * M_PI) - 0.5 * ld - 0.5 * q;
    out->min_pivot = h->res_host[2];
    out->fail_leaf = (hf[0] == 0x7f7f7f7f) ? -1 : hf[0];
    out->cap_binds = hf[1];
    out->max_rank = hf[3];
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

hcov_status hcov_build_tree_host(const double *s_host, int64_t n, int32_t leaf_size, double eta, int32_t dense_below,
                                 hcov_tree *out)
{
    if (!out) return HCOV_ERR_INVALID_ARG;
    *out = nullptr;
    if (n == 0) return HCOV_ERR_EMPTY_INPUT;
    if (!s_host || n < 0 || leaf_size != HCOV_LEAF || !(eta >= 0) || dense_below < 0) return HCOV_ERR_INVALID_ARG;
    std::unique_ptr<hcov_tree_s> t(new (std::nothrow) hcov_tree_s());
    if (!t) return HCOV_ERR_OUT_OF_MEMORY;
    int rc = plan_build(t->P, s_host, n, eta, dense_below);
    if (rc == 2) return HCOV_ERR_EMPTY_INPUT;
    if (rc) return HCOV_ERR_INVALID_ARG;
    *out = t.release();
    return HCOV_OK;
}

hcov_status hcov_build_tree(const double *s_dev, int64_t n, int32_t leaf_size, double eta, int32_t dense_below,
                            hcov_stream stream, hcov_tree *out)
{
    if (!out) return HCOV_ERR_INVALID_ARG;
    *out = nullptr;
    if (n == 0) return HCOV_ERR_EMPTY_INPUT;
    if (!s_dev || n < 0) return HCOV_ERR_INVALID_ARG;
    std::vector<double> s(2 * n);
    CK(cudaMemcpyAsync(s.data(), s_dev, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    hcov_tree t = nullptr;
    hcov_status st = hcov_build_tree_host(s.data(), n, leaf_size, eta, dense_below, &t);
    if (st) return st;
    st = tree_upload(t);
    if (st) { delete t; return st; }
    *out = t;
    return HCOV_OK;
}

hcov_status hcov_tree_get_info(hcov_tree t, hcov_tree_info *info)
{
    if (!t || !info) return HCOV_ERR_INVALID_ARG;
    const Plan &P = t->P;
    info->n = P.n; info->n_pad = P.n_pad; info->depth = P.depth; info->leaf_size = HCOV_LEAF;
    info->n_leaves = P.n_leaves; info->n_dense_tiles = P.n_tiles(); info->n_lowrank = P.n_r();
    info->n_tasks = (int64_t)P.tasks.size(); info->n_waves = P.n_waves; info->eta = P.eta;
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
    s = assemble_into(h, theta, trunc, (cudaStream_t)stream);
    if (s) { delete h; return s; }
    *out = h;
    return HCOV_OK;
}

hcov_status hcov_cholesky(hcov_hmat h, hcov_stream stream, int64_t *fail_leaf)
{
    if (!h) return HCOV_ERR_INVALID_ARG;
    return cholesky_run(h, (cudaStream_t)stream, fail_leaf);
}

hcov_status hcov_loglik(hcov_hmat h, const double *Z_dev, hcov_stream stream, hcov_result *out)
{
    if (!h || !Z_dev || !out) return HCOV_ERR_INVALID_ARG;
    return loglik_run(h, Z_dev, (cudaStream_t)stream, out);
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
    if ((s = assemble_into(h, theta, trunc, st))) return s;
    int64_t fl = -1;
    s = cholesky_run(h, st, &fl);
    if (s == HCOV_ERR_NOT_SPD || s == HCOV_ERR_RANK_CAPACITY) {
        std::memset(out, 0, sizeof(*out));
        out->n = t->P.n;
        out->loglik = -INFINITY;
        out->fail_leaf = fl;
        return s;
    }
    if (s) return s;
    return loglik_run(h, Z_dev, st, out);
}

hcov_status hcov_mle_batch(hcov_tree t, const double *Z_dev, const hcov_theta *thetas, int32_t m,
                           const hcov_trunc *trunc, hcov_stream stream, double *loglik_host, hcov_status *status_host)
{
    if (!t || !Z_dev || !thetas || m < 0 || !trunc || !loglik_host || !status_host) return HCOV_ERR_INVALID_ARG;
    for (int32_t k = 0; k < m; ++k) {
        hcov_result r;
        hcov_status s = hcov_eval(t, thetas + k, trunc, Z_dev, stream, &r);
        status_host[k] = s;
        if (s == HCOV_OK) loglik_host[k] = r.loglik;
        else if (s == HCOV_ERR_NOT_SPD || s == HCOV_ERR_RANK_CAPACITY || s == HCOV_ERR_INVALID_ARG)
            loglik_host[k] = -INFINITY;
        else return s;
    }
    return HCOV_OK;
}

hcov_status hcov_sample(hcov_hmat h, const double *xi_dev, double *Z_dev, hcov_stream stream)
{
    if (!h || !xi_dev || !Z_dev) return HCOV_ERR_INVALID_ARG;
    if (h->state != 2) return HCOV_ERR_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    Plan &P = h->t->P;
    double *x = nullptr, *y = nullptr, *tt = nullptr;
    CK(cudaMalloc(&x, P.n_pad * sizeof(double)));
    CK(cudaMalloc(&y, P.n_pad * sizeof(double)));
    CK(cudaMalloc(&tt, std::max<int64_t>(1, P.n_r()) * h->ctx.kcap * sizeof(double)));
    k_permute_in<<<256, 256, 0, st>>>(h->ctx, xi_dev, x);
    if (P.n_r() > 0) k_sample_t<<<(int)std::min<int64_t>(P.n_r(), 65535), NT, 0, st>>>(h->ctx, x, tt);
    k_sample_rows<<<(int)std::min<int64_t>(P.n_leaves, 65535), 32, 0, st>>>(h->ctx, x, tt, y);
    k_permute_out<<<256, 256, 0, st>>>(h->ctx, y, Z_dev);
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
    k_columns<<<std::min(t->n_leafnodes, 65535), NT, 0, st>>>(h->ctx, t->d_leafnodes, t->n_leafnodes, d_pc, m, tmp);
    k_columns_perm<<<512, 256, 0, st>>>(h->ctx, tmp, m, out_dev);
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d_pc); cudaFree(tmp);
    if (e != cudaSuccess) return map_err(e);
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

hcov_status hcov_prof_control(int32_t enable_events, int32_t reset)
{
    if (reset) {
        prof_collect();
        g_prof.launches = 0;
        for (int k = 0; k < PC_N; ++k) { g_prof.count[k] = 0; g_prof.ms[k] = 0.0; }
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
    return HCOV_OK;
}

const char *hcov_prof_class_name(int32_t cls)
{
    return (cls >= 0 && cls < PC_N) ? PROF_NAMES[cls] : "";
}

void hcov_tree_free(hcov_tree t) { delete t; }
void hcov_hmat_free(hcov_hmat h) { delete h; }

}  // extern "C"
