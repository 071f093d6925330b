// Block-level all-reduce over peer memory (csrc/peer.cu): the exchange tail
// shared by the standalone peer all-reduce and the fused compute + exchange
// kernels (the SpMV whose last CTA exchanges the top rows, spmv.cu).
#pragma once

#include "tsb_common.cuh"

namespace tsb {

struct PeerArgs {
    int64_t m;                 // rows exchanged
    int world, rank;
    double *const *bufs;       // [world] exchange buffers (2 x half doubles), as mapped here
    int64_t *const *flags;     // [world] epoch words, as mapped here
    const int32_t *idx;        // rows of x (NULL: the first m)
    int64_t epoch;             // unused: derived on the device (exchange_block)
    int64_t half;
};

__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// One CTA: gather x's rows into this rank's buffer half (epoch & 1), publish
// the epoch (release, system scope), wait for every peer's, then x's rows :=
// the sum over ranks in rank order.  x may have been written by other CTAs of
// the same kernel (read through L2).
// The epoch is derived on the device -- one more than this rank's own epoch
// word, which only this rank's exchanges write, in stream order -- so every
// rank numbers the same sequence of exchanges identically and the kernels
// replay inside CUDA graphs (P.epoch is not used).
__device__ __forceinline__ void exchange_block(const PeerArgs &P, double *x) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t epoch = *((volatile const int64_t *)P.flags[P.rank]) + 1;
    const int64_t off = (epoch & 1) * P.half;
    double *mine = P.bufs[P.rank] + off;
    for (int64_t i = tid; i < P.m; i += nt) mine[i] = __ldcg(x + (P.idx ? P.idx[i] : i));
    __syncthreads();
    if (tid == 0) {
        __threadfence_system();
        st_release_sys(P.flags[P.rank], epoch);
    }
    if (tid < P.world && tid != P.rank) {
        const int64_t *f = P.flags[tid];
        while (ld_acquire_sys(f) < epoch) __nanosleep(64);
    }
    __syncthreads();
    for (int64_t i = tid; i < P.m; i += nt) {
        double a = 0.0;
        for (int r = 0; r < P.world; ++r) a += __ldcv(P.bufs[r] + off + i);
        x[P.idx ? P.idx[i] : i] = a;
    }
}

}  // namespace tsb
