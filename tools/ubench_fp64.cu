// FP64 throughput on this GPU: CUDA-core DFMA vs the legacy FP64 tensor path
// (mma.sync m8n8k4 f64, DMMA).  Prints achieved TFLOP/s for each.
#include <cstdio>

__global__ void k_dfma(int iters, double *out) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double b = 0.999999, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dmma(int iters, double *out) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
}

int main() {
    double *out;
    cudaMalloc(&out, 8 * 148 * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        for (int threads : {256, 1024}) {
            const int grid = nsm * 4;
            cudaEventRecord(e0);
            k_dfma<<<grid, threads>>>(iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 64 * iters * (double)grid * threads;
            printf("DFMA  grid %d x %d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, flops / ms / 1e9);
            cudaEventRecord(e0);
            k_dmma<<<grid, threads>>>(iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            // one m8n8k4 per warp = 8*8*4*2 flops; 32 per iteration per warp
            const double f2 = 512.0 * 32 * iters * (double)grid * (threads / 32);
            printf("DMMA  grid %d x %d: %.3f ms  %.2f TFLOP/s  (%s)\n", grid, threads, ms, f2 / ms / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
