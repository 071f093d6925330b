// Read-streaming ceiling on the B200 for the sweep's access pattern:
// persistent CTAs each pull chunks of CHUNK bytes with cp.async.bulk (TMA)
// into a ring of S shared-memory stages and reduce them (as the sweep items
// do), versus a plain LDG.128 grid-stride reduction.  Prints GB/s per config.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_stream tools/ubench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_reduce(const double2 *__restrict__ a, int64_t n2, double *out) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        double2 v = __ldcs(a + i);
        s += v.x * 1.0000001 + v.y;
    }
    if (s == 123.456) out[0] = s;
}

// each CTA streams chunks c = blockIdx.x, + gridDim.x, ... through S stages
__global__ void tma_reduce(const char *__restrict__ a, int64_t nchunks, int chunk, int S, double *out) {
    extern __shared__ __align__(128) char smem[];
    __shared__ uint64_t bars[8];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t c, int s) {
        if (threadIdx.x == 0 && c < nchunks) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(chunk)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(smem + (int64_t)s * chunk)),
                "l"(a + c * chunk), "r"(chunk), "r"(su32(&bars[s]))
                : "memory");
        }
    };
    int64_t c = blockIdx.x;
    for (int s = 0; s < S; ++s) issue(c + (int64_t)s * gridDim.x, s);
    double acc = 0.0;
    uint32_t ph = 0;
    int s = 0;
    for (; c < nchunks; c += gridDim.x) {
        asm volatile(
            "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                su32(&bars[s])),
            "r"((ph >> s) & 1u)
            : "memory");
        ph ^= 1u << s;
        const double2 *v = reinterpret_cast<const double2 *>(smem + (int64_t)s * chunk);
        for (int k = threadIdx.x; k < chunk / 16; k += blockDim.x) acc += v[k].x * 1.0000001 + v[k].y;
        __syncthreads();
        issue(c + (int64_t)S * gridDim.x, s);
        s = (s + 1 == S) ? 0 : s + 1;
    }
    if (acc == 123.456) out[0] = acc;
}

int main() {
    const int64_t bytes = 2800ll << 20;
    char *a;
    double *out;
    cudaMalloc(&a, bytes);
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, bytes);
    char *flush;
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaMemsetAsync(flush, r, 512 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r) best = ms < best ? ms : best;
        }
        return best;
    };
    for (int bpsm : {2, 4, 8}) {
        float ms = timeit([&] { ldg_reduce<<<148 * bpsm, 256>>>((const double2 *)a, bytes / 16, out); });
        printf("LDG.128 grid=148x%d        %.3f ms  %.0f GB/s\n", bpsm, ms, bytes / (ms * 1e-3) / 1e9);
    }
    for (int chunk : {16384, 32768, 49152}) {
        for (int S : {1, 2, 3, 4}) {
            for (int cps : {1, 2, 3, 4}) {
                size_t sm = (size_t)chunk * S;
                if (sm * cps > 220 * 1024 || sm > 227 * 1024) continue;
                cudaFuncSetAttribute(tma_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                int64_t nch = bytes / chunk;
                float ms = timeit([&] { tma_reduce<<<148 * cps, 256, sm>>>(a, nch, chunk, S, out); });
                printf("TMA chunk=%2dKB stages=%d ctas/sm=%d  %.3f ms  %.0f GB/s  (in flight/SM %d KB)\n", chunk / 1024, S,
                       cps, ms, bytes / (ms * 1e-3) / 1e9, chunk * S * cps / 1024);
            }
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
