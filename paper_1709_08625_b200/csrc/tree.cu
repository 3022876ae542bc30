// Device cluster tree (A1, kernel K1) and block tree (A2, kernel K2).
//
//  A1 — Def. A.1 with the split rule of the listing's
//       TAutoBSPPartStrat(adaptive_split_axis) as read in DESIGN.md R5: per cluster,
//       the tight bounding box of its points; split the longest axis (ties -> x) at the cardinality
//       median, left child gets ceil(m/2); the order inside a cluster is a STABLE sort on the split
//       coordinate.  Level-synchronous on the device: per level one segmented bounding-box
//       reduction and one segmented stable sort of all clusters at once, done as an LSD radix sort
//       of the composite key (cluster id, order-preserving bits of the coordinate); radix passes
//       are stable, so equal coordinates keep their current order exactly as std::stable_sort.
//  A2 — Def. A.2 son rule with TStdGeomAdmCond(2.0, use_min_diam)
//       (PAPER.md:475): a pair (tau, sigma) is admissible iff dist > 0 and
//       min(diam tau, diam sigma) <= eta * dist.  Level-synchronous expansion of the lower block
//       tree: every pair of level l is classified (R: admissible low-rank leaf, T: dense leaf,
//       H: inner node) and the children of the H nodes (3 below a diagonal pair, 4 below an
//       off-diagonal pair) are emitted with one scan.
//
//  Bitwise agreement with the host planner (plan.cpp, whose rules are pinned against an
//  independent Python mirror in tests/test_plan.py) is tested in tests/test_gpu_tree.py: the
//  geometry below uses explicitly rounded operations (__dmul_rn / __dadd_rn / __dsqrt_rn, no FMA
//  contraction) so that bounding boxes, diameters, distances and admissibility decisions are the
//  same IEEE results as the host's.
//
//  The task DAG of the factorization (scheduling, not a stage of the method) is planned on the
//  host from the device-built trees (plan_build with a PlanGeo).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "plan.h"

namespace {

constexpr int RB = 8;                 // radix bits per pass
constexpr int RD = 1 << RB;           // digits
constexpr int TILE = 1024;            // elements per warp tile (radix histogram / scatter)
constexpr int WPB = 8;                // warps per block in the radix kernels
constexpr int SCAN_NT = 1024;         // threads of the scan kernels
constexpr int SCAN_ITEMS = 4;         // elements per thread in a scan block

#define TCK(x)                                   \
    do {                                         \
        if ((x) != cudaSuccess) return -1;       \
    } while (0)

__device__ __forceinline__ uint64_t order_bits(double v)
{
    // order-preserving map of a finite double to uint64; -0.0 and +0.0 compare equal on the host
    // (std::stable_sort with operator<), so both map to the bits of +0.0
    v = v + 0.0;
    const uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// std::min / std::max semantics (first argument returned unless the second compares strictly)
__device__ __forceinline__ double hmin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double hmax(double a, double b) { return (a < b) ? b : a; }

__global__ void k_finite(const double *s, int64_t n2, int *bad)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n2; k += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(s[k])) atomicExch(bad, 1);
}

__global__ void k_iota(int32_t *p, int64_t n)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        p[k] = (int32_t)k;
}

// Bounding box and split axis of every cluster of one level (one CTA per cluster, grid-stride).
// s: n x D row-major; box layout lo[0..D), hi[0..D) (as the host planner).
__global__ void __launch_bounds__(256) k_seg_bbox(const double *s, int D, const int32_t *perm, const int64_t *rs,
                                                  int64_t nseg, int64_t heap0, double *bb, int8_t *axis)
{
    __shared__ double red[6][8];
    for (int64_t c = blockIdx.x; c < nseg; c += gridDim.x) {
        const int64_t a = rs[c], b = rs[c + 1];
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t k = a + threadIdx.x; k < b; k += blockDim.x) {
            const int64_t e = perm[k];
            for (int d = 0; d < D; ++d) {
                const double x = s[D * e + d];
                lo[d] = fmin(lo[d], x); hi[d] = fmax(hi[d], x);
            }
        }
        // min / max are exact (order-independent) for finite values
        for (int d = 0; d < D; ++d)
            for (int o = 16; o > 0; o >>= 1) {
                lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
                hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
            }
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0)
            for (int d = 0; d < D; ++d) { red[d][w] = lo[d]; red[3 + d][w] = hi[d]; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
                for (int d = 0; d < D; ++d) { lo[d] = fmin(lo[d], red[d][k]); hi[d] = fmax(hi[d], red[3 + d][k]); }
            double *o = bb + 2 * D * (heap0 + c);
            if (b > a) {
                // with both -0.0 and +0.0 among the coordinates the stored zero's sign may differ
                // from the host's (which keeps the first met); every use of a box is a difference
                // followed by a square or a comparison, so the trees are the same either way
                for (int d = 0; d < D; ++d) { o[d] = lo[d]; o[D + d] = hi[d]; }
                // longest extent, ties -> lowest axis
                int ax = 0;
                for (int d = 1; d < D; ++d)
                    if (__dsub_rn(hi[d], lo[d]) > __dsub_rn(hi[ax], lo[ax])) ax = d;
                axis[c] = (int8_t)ax;
            } else {
                for (int d = 0; d < 2 * D; ++d) o[d] = __longlong_as_double(0x7ff8000000000000ll);
                axis[c] = 0;
            }
        }
        __syncthreads();
    }
}

// Sort keys of one level: coordinate bits on the cluster's split axis, and the cluster id.
__global__ void k_keys(const double *s, int D, const int32_t *perm, const int64_t *rs, int64_t nseg,
                       const int8_t *axis, int64_t n, uint64_t *key, uint32_t *seg)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        // cluster containing position k: last c with rs[c] <= k
        int64_t lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (rs[mid] <= k) lo = mid; else hi = mid - 1;
        }
        const int64_t e = perm[k];
        key[k] = order_bits(s[D * e + axis[lo]]);
        seg[k] = (uint32_t)lo;
    }
}

__device__ __forceinline__ uint32_t digit_of(const uint64_t *key, const uint32_t *seg, int64_t k, int pass)
{
    // passes 0..7: coordinate bytes (least significant first); 8, 9: cluster id bytes
    return pass < 8 ? (uint32_t)(key[k] >> (RB * pass)) & (RD - 1) : (seg[k] >> (RB * (pass - 8))) & (RD - 1);
}

__global__ void __launch_bounds__(32 * WPB) k_rhist(const uint64_t *key, const uint32_t *seg, int64_t n, int pass,
                                                    int64_t ntiles, int32_t *hist)
{
    __shared__ int32_t cnt[WPB][RD];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = (int64_t)blockIdx.x * WPB + w;
    for (int d = lane; d < RD; d += 32) cnt[w][d] = 0;
    __syncwarp();
    if (tile < ntiles) {
        const int64_t k0 = tile * TILE, k1 = (n < k0 + TILE) ? n : k0 + TILE;
        for (int64_t k = k0 + lane; k < k1; k += 32) atomicAdd(&cnt[w][digit_of(key, seg, k, pass)], 1);
        __syncwarp();
        for (int d = lane; d < RD; d += 32) hist[(int64_t)d * ntiles + tile] = cnt[w][d];
    }
}

// Stable scatter: one warp per tile, 32 elements per step in order; ranks among equal digits of a
// step from __match_any_sync, running per-digit counters in shared memory.
__global__ void __launch_bounds__(32 * WPB) k_rscatter(const uint64_t *key, const uint32_t *seg, const int32_t *val,
                                                       int64_t n, int pass, int64_t ntiles, const int32_t *offs,
                                                       uint64_t *key2, uint32_t *seg2, int32_t *val2)
{
    __shared__ int32_t cnt[WPB][RD];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = (int64_t)blockIdx.x * WPB + w;
    if (tile >= ntiles) return;
    for (int d = lane; d < RD; d += 32) cnt[w][d] = offs[(int64_t)d * ntiles + tile];
    __syncwarp();
    const int64_t k0 = tile * TILE, k1 = (n < k0 + TILE) ? n : k0 + TILE;
    for (int64_t kb = k0; kb < k1; kb += 32) {
        const int64_t k = kb + lane;
        const bool on = k < k1;
        const unsigned act = __ballot_sync(0xffffffffu, on);
        if (!on) break;
        const uint32_t d = digit_of(key, seg, k, pass);
        const unsigned peers = __match_any_sync(act, d);
        const int r = __popc(peers & ((1u << lane) - 1u));
        const int base = cnt[w][d];
        __syncwarp(act);
        if (r == 0) cnt[w][d] = base + __popc(peers);
        __syncwarp(act);
        const int64_t p = base + r;
        key2[p] = key[k];
        seg2[p] = seg[k];
        val2[p] = val[k];
    }
}

// ---- exclusive scan of int32 counts (int64 totals), three kernels ------------------------------
__global__ void __launch_bounds__(SCAN_NT) k_scan_blocks(const int32_t *in, int64_t n, int64_t *out, int64_t *bsum)
{
    __shared__ int64_t ws[SCAN_NT / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_NT * SCAN_ITEMS + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS], t = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        t += v[i];
    }
    // inclusive warp scan of thread totals
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = t;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t y = lane < SCAN_NT / 32 ? ws[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        if (lane < SCAN_NT / 32) ws[lane] = y;
    }
    __syncthreads();
    int64_t run = x - t + (w ? ws[w - 1] : 0);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (threadIdx.x == SCAN_NT - 1) bsum[blockIdx.x] = run;
}

__global__ void k_scan_serial(int64_t *bsum, int64_t nb, int64_t *total)
{
    // nb <= a few thousand: one thread, fixed order
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t r = 0;
        for (int64_t b = 0; b < nb; ++b) { const int64_t v = bsum[b]; bsum[b] = r; r += v; }
        *total = r;
    }
}

__global__ void k_scan_add(int64_t *out, int64_t n, const int64_t *bsum)
{
    const int64_t per = (int64_t)SCAN_NT * SCAN_ITEMS;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[k] += bsum[k / per];
}

__global__ void k_to_i32(const int64_t *a, int64_t n, int32_t *b)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        b[k] = (int32_t)a[k];
}

// Leaf level: padded internal order (32 positions per leaf; phantoms -1 / NaN).
__global__ void k_leaves(const double *s, int D, const int32_t *perm, const int64_t *rs, int64_t nleaf, int64_t *i2e,
                         double *xs, double *ys, double *zs)
{
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nleaf * HCOV_LEAF;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = q / HCOV_LEAF, o = q % HCOV_LEAF;
        const int64_t k = rs[c] + o;
        if (k < rs[c + 1]) {
            const int64_t e = perm[k];
            i2e[q] = e; xs[q] = s[D * e]; ys[q] = s[D * e + 1];
            if (zs) zs[q] = s[D * e + 2];
        } else {
            i2e[q] = -1;
            xs[q] = ys[q] = qnan;
            if (zs) zs[q] = qnan;
        }
    }
}

// ---- A2 ------------------------------------------------------------------------------------
struct Pair { int32_t i, j, forced; };

__device__ __forceinline__ double diam_of(const double *b, int D)
{
    double s2 = 0.0;
    for (int d = 0; d < D; ++d) {
        const double e = __dsub_rn(b[D + d], b[d]);
        s2 = (d == 0) ? __dmul_rn(e, e) : __dadd_rn(s2, __dmul_rn(e, e));
    }
    return __dsqrt_rn(s2);
}

__device__ __forceinline__ bool admissible(const double *bb, int D, int64_t heap0, int32_t i, int32_t j, double eta)
{
    if (eta <= 0.0) return false;
    const double *a = bb + 2 * D * (heap0 + i), *b = bb + 2 * D * (heap0 + j);
    double s2 = 0.0;
    for (int d = 0; d < D; ++d) {
        const double g = hmax(0.0, hmax(__dsub_rn(a[d], b[D + d]), __dsub_rn(b[d], a[D + d])));
        s2 = (d == 0) ? __dmul_rn(g, g) : __dadd_rn(s2, __dmul_rn(g, g));
    }
    const double dd = __dsqrt_rn(s2);
    if (!(dd > 0.0)) return false;
    return hmin(diam_of(a, D), diam_of(b, D)) <= __dmul_rn(eta, dd);
}

__global__ void k_bclass(const Pair *pr, int64_t np, const double *bb, int D, int l, int L, int64_t csize,
                         int dense_below, double eta, int8_t *type, int32_t *nchild)
{
    const int64_t heap0 = ((int64_t)1 << l) - 1;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
        const Pair x = pr[p];
        int t, nc = 0;
        if (x.i == x.j) {
            t = (l == L) ? ND_T : ND_H;
            nc = (t == ND_H) ? 3 : 0;
        } else {
            const bool adm = !x.forced && admissible(bb, D, heap0, x.i, x.j, eta);
            if (adm && l < L && csize > dense_below) t = ND_R;
            else if (l == L) t = ND_T;
            else t = ND_H;
            nc = (t == ND_H) ? 4 : 0;
            // the child's forced flag (forced || adm) is recomputed in k_bexpand
        }
        type[p] = (int8_t)t;
        nchild[p] = nc;
    }
}

__global__ void k_bexpand(const Pair *pr, int64_t np, const int8_t *type, const int64_t *off, const double *bb, int D,
                          int l, double eta, Pair *out)
{
    const int64_t heap0 = ((int64_t)1 << l) - 1;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
        if (type[p] != ND_H) continue;
        const Pair x = pr[p];
        Pair *o = out + off[p];
        if (x.i == x.j) {
            o[0] = {2 * x.i, 2 * x.j, x.forced};
            o[1] = {2 * x.i + 1, 2 * x.j, x.forced};
            o[2] = {2 * x.i + 1, 2 * x.j + 1, x.forced};
        } else {
            const int f = (x.forced || admissible(bb, D, heap0, x.i, x.j, eta)) ? 1 : 0;
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) o[2 * a + b] = {2 * x.i + a, 2 * x.j + b, f};
        }
    }
}

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    ~DBuf() { if (p) cudaFree(p); }
    int alloc(size_t k)
    {
        if (k <= n) return 0;
        if (p) cudaFree(p);
        p = nullptr; n = 0;
        if (cudaMalloc(&p, std::max<size_t>(k, 1) * sizeof(T)) != cudaSuccess) return -1;
        n = k;
        return 0;
    }
};

inline int grid_for(int64_t n, int nt = 256) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + nt - 1) / nt, 148 * 16)); }

// exclusive scan of in[0, n) (int32) into out (int64); returns the total via *total_h
int scan_counts(const int32_t *in, int64_t n, int64_t *out, DBuf<int64_t> &bsum, DBuf<int64_t> &tot, cudaStream_t st,
                int64_t *total_h)
{
    const int64_t per = (int64_t)SCAN_NT * SCAN_ITEMS;
    const int64_t nb = std::max<int64_t>(1, (n + per - 1) / per);
    if (bsum.alloc(nb) || tot.alloc(1)) return -1;
    k_scan_blocks<<<(unsigned)nb, SCAN_NT, 0, st>>>(in, n, out, bsum.p);
    k_scan_serial<<<1, 32, 0, st>>>(bsum.p, nb, tot.p);
    k_scan_add<<<grid_for(n), 256, 0, st>>>(out, n, bsum.p);
    if (total_h) {
        TCK(cudaMemcpyAsync(total_h, tot.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        TCK(cudaStreamSynchronize(st));
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace

// Host driver: K1 + K2 on the device; the results are copied into PlanGeo for the DAG planner.
// Returns 0 ok, 1 invalid input (non-finite coordinates / n >= 2^31), 2 empty input, -1 CUDA error.
int tree_geo_device(const double *s, int64_t n, const PlanOpts &opt, cudaStream_t st, PlanGeo &g)
{
    if (n <= 0) return 2;
    if (n >= ((int64_t)1 << 31) - HCOV_LEAF) return 1;
    const int D = opt.dim;
    if (D != 2 && D != 3) return 1;
    {
        DBuf<int> bad;
        if (bad.alloc(1)) return -1;
        TCK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        k_finite<<<grid_for(D * n), 256, 0, st>>>(s, D * n, bad.p);
        int h = 0;
        TCK(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        TCK(cudaStreamSynchronize(st));
        if (h) return 1;
    }
    int L = 0;
    while (((int64_t)HCOV_LEAF << L) < n) ++L;
    const int64_t nleaf = (int64_t)1 << L, npad = (int64_t)HCOV_LEAF << L, ncl = ((int64_t)2 << L) - 1;
    const int dense_below = std::max(opt.dense_below, HCOV_LEAF);
    g.depth = L;
    // cluster boundaries per level depend on n only (left child gets ceil(m/2))
    std::vector<std::vector<int64_t>> rs(L + 1);
    rs[0] = {0, n};
    for (int l = 0; l < L; ++l) {
        const int64_t nc = (int64_t)1 << l;
        rs[l + 1].resize(2 * nc + 1);
        for (int64_t c = 0; c < nc; ++c) {
            const int64_t a = rs[l][c], b = rs[l][c + 1], m1 = (b - a + 1) / 2;
            rs[l + 1][2 * c] = a;
            rs[l + 1][2 * c + 1] = a + m1;
        }
        rs[l + 1][2 * nc] = n;
    }
    DBuf<int32_t> perm, perm2, hist;
    DBuf<uint64_t> key, key2;
    DBuf<uint32_t> seg, seg2;
    DBuf<int64_t> offs, bsum, tot, drs, i2e;
    DBuf<double> bb, xs, ys, zs;
    DBuf<int8_t> axis;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    if (perm.alloc(n) || perm2.alloc(n) || key.alloc(n) || key2.alloc(n) || seg.alloc(n) || seg2.alloc(n) ||
        hist.alloc((size_t)RD * ntiles) || offs.alloc((size_t)RD * ntiles) || bb.alloc(2 * D * ncl) ||
        axis.alloc(nleaf) || drs.alloc(nleaf + 1) || i2e.alloc(npad) || xs.alloc(npad) || ys.alloc(npad) ||
        (D == 3 && zs.alloc(npad)))
        return -1;
    k_iota<<<grid_for(n), 256, 0, st>>>(perm.p, n);
    for (int l = 0; l <= L; ++l) {
        const int64_t nseg = (int64_t)1 << l;
        TCK(cudaMemcpyAsync(drs.p, rs[l].data(), (nseg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        k_seg_bbox<<<(unsigned)std::min<int64_t>(nseg, 148 * 8), 256, 0, st>>>(s, D, perm.p, drs.p, nseg, nseg - 1,
                                                                                bb.p, axis.p);
        if (l == L) break;
        k_keys<<<grid_for(n), 256, 0, st>>>(s, D, perm.p, drs.p, nseg, axis.p, n, key.p, seg.p);
        const int npass = 8 + (l + RB - 1) / RB;     // coordinate bytes, then the cluster id bytes
        for (int pass = 0; pass < npass; ++pass) {
            const unsigned nb = (unsigned)((ntiles + WPB - 1) / WPB);
            k_rhist<<<nb, 32 * WPB, 0, st>>>(key.p, seg.p, n, pass, ntiles, hist.p);
            if (scan_counts(hist.p, RD * ntiles, offs.p, bsum, tot, st, nullptr)) return -1;
            k_to_i32<<<grid_for(RD * ntiles), 256, 0, st>>>(offs.p, RD * ntiles, hist.p);
            k_rscatter<<<nb, 32 * WPB, 0, st>>>(key.p, seg.p, perm.p, n, pass, ntiles, hist.p, key2.p, seg2.p, perm2.p);
            std::swap(key.p, key2.p); std::swap(seg.p, seg2.p); std::swap(perm.p, perm2.p);
        }
    }
    k_leaves<<<grid_for(npad), 256, 0, st>>>(s, D, perm.p, drs.p, nleaf, i2e.p, xs.p, ys.p, D == 3 ? zs.p : nullptr);
    TCK(cudaGetLastError());
    g.perm_i2e.resize(npad); g.xs.resize(npad); g.ys.resize(npad); g.bb.resize(2 * D * ncl);
    if (D == 3) g.zs.resize(npad);
    TCK(cudaMemcpyAsync(g.perm_i2e.data(), i2e.p, npad * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    TCK(cudaMemcpyAsync(g.xs.data(), xs.p, npad * sizeof(double), cudaMemcpyDeviceToHost, st));
    TCK(cudaMemcpyAsync(g.ys.data(), ys.p, npad * sizeof(double), cudaMemcpyDeviceToHost, st));
    TCK(cudaMemcpyAsync(g.bb.data(), bb.p, 2 * D * ncl * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (D == 3) TCK(cudaMemcpyAsync(g.zs.data(), zs.p, npad * sizeof(double), cudaMemcpyDeviceToHost, st));
    TCK(cudaStreamSynchronize(st));

    // ---- A2: level-synchronous block tree ------------------------------------------------------
    DBuf<Pair> pa, pb;
    DBuf<int8_t> ty;
    DBuf<int32_t> nch;
    DBuf<int64_t> coff;
    if (pa.alloc(1)) return -1;
    const Pair root{0, 0, 0};
    TCK(cudaMemcpyAsync(pa.p, &root, sizeof(Pair), cudaMemcpyHostToDevice, st));
    int64_t np = 1;
    g.level_pairs.assign(L + 1, {});
    g.level_types.assign(L + 1, {});
    for (int l = 0; l <= L && np > 0; ++l) {
        if (ty.alloc(np) || nch.alloc(np) || coff.alloc(np)) return -1;
        k_bclass<<<grid_for(np), 256, 0, st>>>(pa.p, np, bb.p, D, l, L, (int64_t)HCOV_LEAF << (L - l), dense_below,
                                              opt.eta, ty.p, nch.p);
        int64_t nnext = 0;
        if (scan_counts(nch.p, np, coff.p, bsum, tot, st, &nnext)) return -1;
        std::vector<Pair> hp(np);
        g.level_types[l].resize(np);
        TCK(cudaMemcpyAsync(hp.data(), pa.p, np * sizeof(Pair), cudaMemcpyDeviceToHost, st));
        TCK(cudaMemcpyAsync(g.level_types[l].data(), ty.p, np, cudaMemcpyDeviceToHost, st));
        if (nnext > 0) {
            if (pb.alloc(nnext)) return -1;
            k_bexpand<<<grid_for(np), 256, 0, st>>>(pa.p, np, ty.p, coff.p, bb.p, D, l, opt.eta, pb.p);
        }
        TCK(cudaStreamSynchronize(st));
        TCK(cudaGetLastError());
        g.level_pairs[l].resize(np);
        for (int64_t p = 0; p < np; ++p) g.level_pairs[l][p] = {hp[p].i, hp[p].j};
        std::swap(pa.p, pb.p); std::swap(pa.n, pb.n);
        np = nnext;
    }
    return 0;
}
