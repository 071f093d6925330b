// Shared device/host helpers for libtsb (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "tsb.h"

namespace tsb {

// ---------------------------------------------------------------------------
// Error plumbing: every C entry point runs its body through guard(), which
// turns exceptions into a status code and a per-thread message.
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);
void count_launch(int64_t n = 1);

inline void check_cuda(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        throw Error(TSB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define TSB_CUDA(x) ::tsb::check_cuda((x), #x)
#define TSB_LAUNCHED()                                               \
    do {                                                             \
        ::tsb::check_cuda(cudaGetLastError(), "kernel launch");      \
        ::tsb::count_launch();                                       \
    } while (0)

template <class F>
int guard(F &&body) {
    try {
        body();
        return TSB_OK;
    } catch (const Error &e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        set_last_error(e.what());
        return TSB_E_ARG;
    }
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Opt a kernel into the device's full dynamic shared memory once, so handles
// with different footprints (several factor images, block subsets) can all
// launch it; occupancy is still computed from each launch's actual size.
template <class K>
inline void allow_max_smem(K kernel) {
    int dev = 0, optin = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    check_cuda(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem optin");
    cudaFuncAttributes fa{};
    check_cuda(cudaFuncGetAttributes(&fa, (const void *)kernel), "cudaFuncGetAttributes");
    check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    optin - (int)fa.sharedSizeBytes),
               "cudaFuncSetAttribute(max dynamic smem)");
}

constexpr int kNumSM = 148;

// ---------------------------------------------------------------------------
// Exactly-rounded arithmetic without FMA contraction: the reference (NumPy)
// rounds every product and every sum, so kernels that must reproduce its
// values bit for bit use these instead of the operators.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// ---------------------------------------------------------------------------
// Deterministic block reduction (fixed shuffle tree + fixed smem order).
// All threads of the block must call; result valid in thread 0.
// ---------------------------------------------------------------------------
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double *smem) {
    static_assert(BLOCK % 32 == 0 && BLOCK <= 1024, "block size");
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (warp == 0) {
        constexpr int NW = BLOCK / 32;
        r = lane < NW ? smem[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// NumPy's pairwise summation of `n` terms term(i), i in [0, n): the order
// np.add.reduce / reduceat use for float64 (8 partial sums for 8 <= n <= 128,
// halves rounded to a multiple of 8 above).  Single-thread version, used for
// rows longer than the 8-lane fast path handles.
// ---------------------------------------------------------------------------
template <class Term>
__device__ double pairwise_serial(Term term, int64_t lo, int64_t n) {
    // explicit stack instead of recursion: (lo, n, state)
    struct Frame { int64_t lo, n; double left; int stage; };
    Frame st[40];
    int sp = 0;
    st[0] = {lo, n, 0.0, 0};
    double ret = 0.0;
    while (true) {
        Frame &f = st[sp];
        if (f.n <= 128) {
            double res;
            if (f.n < 8) {
                res = -0.0;
                for (int64_t i = 0; i < f.n; ++i) res = add(res, term(f.lo + i));
            } else {
                double r[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = term(f.lo + j);
                int64_t i = 8;
                for (; i < f.n - (f.n % 8); i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) r[j] = add(r[j], term(f.lo + i + j));
                }
                res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
                for (; i < f.n; ++i) res = add(res, term(f.lo + i));
            }
            ret = res;
            // pop
            while (true) {
                if (sp == 0) return ret;
                --sp;
                Frame &p = st[sp];
                int64_t n2 = p.n / 2;
                n2 -= n2 % 8;
                if (p.stage == 0) {
                    p.left = ret;
                    p.stage = 1;
                    st[++sp] = {p.lo + n2, p.n - n2, 0.0, 0};
                    break;
                } else {
                    ret = add(p.left, ret);
                }
            }
        } else {
            int64_t n2 = f.n / 2;
            n2 -= n2 % 8;
            f.stage = 0;
            st[++sp] = {f.lo, n2, 0.0, 0};
        }
    }
}

}  // namespace tsb
