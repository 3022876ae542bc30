// Measured fp64 peaks of this B200 (MEASURED_PEAKS.json has none): a DFMA loop and a
// DMMA (mma.sync.m8n8k4.f64) loop, all SMs, CUDA-event timed, best of 5.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters)
{
    double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double *out, int iters)
{
    double acc[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
    if (s == 12345.678) out[0] = s;
}

int main()
{
    double *d;
    cudaMalloc(&d, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, threads = 512, blocks = nsm * 4;
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    double fl = 2.0 * 8 * (double)iters * threads * blocks;
    printf("{\"dfma_tflops\": %.3f, ", fl / best * 1e-9);
    best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(d, iters / 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    // one m8n8k4 per warp = 2*8*8*4 = 512 flop
    fl = 512.0 * 4 * (double)(iters / 4) * (threads / 32) * blocks;
    printf("\"dmma_tflops\": %.3f, \"sms\": %d}\n", fl / best * 1e-9, nsm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
