// FP64 throughput probes on sm_100a: scalar DFMA and DMMA (mma.sync m8n8k4 f64), issue-bound
// loops with independent accumulators.  Prints TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters, double a, double b) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
    double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i], av, bv);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

#ifdef HAS_M16
__device__ __forceinline__ void dmma16(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__global__ void k_dmma16(double* out, int iters, double a, double b) {
    double c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = threadIdx.x * 1e-3 + i;
    double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma16(c[i], av, av, bv);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0) out[0] = s;
}
#endif

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps = 4; warps <= 32; warps *= 2) {
        const int blocks = nsm * 2, thr = warps * 32 / 2;
        k_dfma<<<blocks, thr>>>(d, 10, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dfma<<<blocks, thr>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * iters * (double)blocks * thr;
        printf("DFMA   warps/SM %2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
        k_dmma<<<blocks, thr>>>(d, 10, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dmma<<<blocks, thr>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 256 * 8 * iters * (double)blocks * (thr / 32);
        printf("DMMA8  warps/SM %2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
#ifdef HAS_M16
        k_dmma16<<<blocks, thr>>>(d, 10, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dmma16<<<blocks, thr>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 512 * 4 * iters * (double)blocks * (thr / 32);
        printf("DMMA16 warps/SM %2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
#endif
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
