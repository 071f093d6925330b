// Micro-benchmarks for the sweep kernels' building blocks (not part of libtsb):
// panel triangle solves in isolation, TMA bulk-copy and plain-load streaming
// rates per CTA and for a full grid.  Built by tools/ubench.py.
#include "../paper_2306_05893_b200/csrc/ldlt.cu"

namespace tsb {  // libtsb's accounting hooks, stubbed for the stand-alone bench
void count_launch(int64_t) {}
void set_last_error(const std::string &) {}
}  // namespace tsb

namespace ub {
using namespace tsb;

__global__ void k_forward(const double *blob, int64_t tri_len, int w, int iters, long long *cycles,
                          double *out) {
    extern __shared__ __align__(128) double sm[];
    double *tri = sm;                 // column-packed copy followed by the row-packed copy
    double *tri_u = sm + tri_len / 2;
    double *seg = sm + tri_len;
    double *yv = seg + kMaxW;
    double *red = yv + kMaxW;
    for (int64_t i = threadIdx.x; i < tri_len; i += blockDim.x) tri[i] = blob[i];
    for (int i = threadIdx.x; i < w; i += blockDim.x) seg[i] = 1.0 + 0.001 * i;
    __syncthreads();
    const int tid = threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < iters; ++r) {
        panel_lower(tri, w, seg, yv, red, tid);
        __syncthreads();
    }
    long long t1 = clock64();
    for (int r = 0; r < iters; ++r) {
        panel_upper(tri_u, w, yv, seg, red, tid);
        __syncthreads();
    }
    long long t2 = clock64();
    if (threadIdx.x == 0) {
        cycles[0] = (t1 - t0) / iters;
        cycles[1] = (t2 - t1) / iters;
    }
    if (threadIdx.x < w) out[threadIdx.x] = seg[threadIdx.x];
}

__global__ void k_tma(const double *src, int64_t stride_doubles, uint32_t bytes, int iters, long long *ns) {
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < iters; ++r) {
        const double *s = src + ((int64_t)blockIdx.x * iters + r) * stride_doubles;
        if (threadIdx.x == 0) tma_load_1d(sm, s, bytes, &bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) ns[blockIdx.x] = (long long)(t1 - t0);
}

__global__ void k_ldg(const double *src, int64_t stride_doubles, uint32_t bytes, int iters, long long *ns,
                      double *sink) {
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    double acc = 0.0;
    const int n2 = bytes / 16;
    for (int r = 0; r < iters; ++r) {
        const double2 *s = reinterpret_cast<const double2 *>(src + ((int64_t)blockIdx.x * iters + r) * stride_doubles);
#pragma unroll 8
        for (int i = threadIdx.x; i < n2; i += blockDim.x) {
            double2 v = __ldcs(s + i);
            acc += v.x + v.y;
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) ns[blockIdx.x] = (long long)(t1 - t0);
    if (acc == 12345.678) sink[0] = acc;
}

__device__ __forceinline__ void gsync(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_barrier(unsigned *bar, int iters, long long *ns) {
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) gsync(bar);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0 && blockIdx.x == 0) ns[0] = (long long)(t1 - t0);
}

}  // namespace ub

extern "C" int ub_barrier(unsigned *bar, int iters, int grid, long long *ns) {
    void *args[] = {&bar, &iters, &ns};
    cudaLaunchCooperativeKernel((const void *)ub::k_barrier, dim3(grid), dim3(256), args, 0, 0);
    return (int)cudaDeviceSynchronize();
}

extern "C" int ub_forward(const double *blob, int64_t tri_len, int w, int iters, long long *cycles, double *out) {
    size_t smem = (tri_len + 256 + 512) * sizeof(double);
    cudaFuncSetAttribute(ub::k_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ub::k_forward<<<1, 256, smem>>>(blob, tri_len, w, iters, cycles, out);
    return (int)cudaDeviceSynchronize();
}

extern "C" int ub_tma(const double *src, int64_t stride, uint32_t bytes, int iters, int grid, long long *ns) {
    cudaFuncSetAttribute(ub::k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    ub::k_tma<<<grid, 256, bytes>>>(src, stride, bytes, iters, ns);
    return (int)cudaDeviceSynchronize();
}

extern "C" int ub_ldg(const double *src, int64_t stride, uint32_t bytes, int iters, int grid, long long *ns,
                      double *sink) {
    ub::k_ldg<<<grid, 256>>>(src, stride, bytes, iters, ns, sink);
    return (int)cudaDeviceSynchronize();
}
