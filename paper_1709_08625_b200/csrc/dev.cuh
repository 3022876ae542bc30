// CTA-level helpers: reductions with deterministic ordering.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef HCOV_NT
#define HCOV_NT 512
#endif
#define NT HCOV_NT      // threads per CTA for every task kernel
#define NWARP (NT / 32)

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum; result broadcast to all threads.  red: >= NWARP doubles of shared memory.
__device__ __forceinline__ double block_sum(double v, double *red)
{
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < NWARP; ++k) t += red[k];
    return t;
}

// argmax |v| with ties -> lowest index; returns (value, index) to all threads.
struct ValIdx { double v; int64_t i; };
__device__ __forceinline__ bool vi_better(double av, int64_t ai, double bv, int64_t bi)
{
    return (av > bv) || (av == bv && ai < bi);
}
__device__ __forceinline__ ValIdx warp_argmax(double v, int64_t i)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (vi_better(ov, oi, v, i)) { v = ov; i = oi; }
    }
    return ValIdx{v, i};
}
__device__ __forceinline__ ValIdx block_argmax(double v, int64_t i, double *redv, int64_t *redi)
{
    ValIdx r = warp_argmax(v, i);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { redv[w] = r.v; redi[w] = r.i; }
    __syncthreads();
    ValIdx b{redv[0], redi[0]};
#pragma unroll
    for (int k = 1; k < NWARP; ++k)
        if (vi_better(redv[k], redi[k], b.v, b.i)) { b.v = redv[k]; b.i = redi[k]; }
    return b;
}

// Loads that bypass L1 (data written by other CTAs in earlier launches/waves is always in
// L2; within a launch no task reads data another task of the same launch writes).
__device__ __forceinline__ double ldg_cg(const double *p) { return __ldcg(p); }

// Phase timers (diagnostics, hcov_prof with events enabled): thread 0 of a CTA accumulates
// globaltimer spans of the truncation phases into g_phase_ns.
__device__ unsigned long long g_phase_ns[64];   // phase + 16 * size class
__device__ int g_phase_on;
__shared__ int s_phase_cls;                      // size class of the running task (0..3)
__device__ __forceinline__ unsigned long long ph_now()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PH_BEGIN(v) const unsigned long long v = (g_phase_on && threadIdx.x == 0) ? ph_now() : 0ull
#define PH_END(k, v)                                                  \
    do {                                                              \
        if (g_phase_on && threadIdx.x == 0) atomicAdd(&g_phase_ns[(k) + 16 * s_phase_cls], ph_now() - (v)); \
    } while (0)
