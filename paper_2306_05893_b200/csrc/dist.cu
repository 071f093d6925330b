// Vector kernels of the sharded (multi-GPU) PCG loop, paper_2306_05893_b200/shard.py.
//
// One rank holds full-length vectors in dissection (permuted) order but only
// its owned rows and the replicated top-separator rows are live.  Reductions
// are weighted (owned rows 1, top rows 1 on rank 0 only, else 0) so that the
// all-reduce of the rank partials counts every row once; they are two-pass
// and fixed-order (deterministic for a given grid).  The scalars alpha/beta
// stay on the device: the kernels read them from the all-reduced sums, the
// host only reads the residual norm for the stop test (krylov.py:150-153).
#include "tsb_common.cuh"

namespace tsb {

constexpr int kVecBlock = 256;
constexpr int kVecGrid = kNumSM * 2;

// ops: 0 dot(a, b); 1 update x += alpha p, r -= alpha ap, reduce r.r
//      (alpha = s[0] / s[1]); 2 direction p = z + beta p (beta = s[0] / s[1]),
//      then s[1] := s[0] for the next iteration (rz_old)
template <int OP>
__global__ void __launch_bounds__(kVecBlock)
vec_kernel(int64_t n, const double *__restrict__ w, double *a, double *b, double *c, double *d,
           const double *__restrict__ sc, double *__restrict__ part, const int32_t *done) {
    __shared__ double red[32];
    if (done != nullptr && *((volatile const int32_t *)done)) return;  // uniform per launch
    double acc = 0.0;
    double coef = 0.0;
    if (OP == 1 || OP == 2) coef = sc[0] / sc[1];
    for (int64_t i = (int64_t)blockIdx.x * kVecBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kVecBlock) {
        if (OP == 0) {
            acc += w[i] * (a[i] * b[i]);
        } else if (OP == 1) {  // a = x, b = p, c = r, d = ap
            a[i] = a[i] + coef * b[i];
            const double ri = c[i] - coef * d[i];
            c[i] = ri;
            acc += w[i] * (ri * ri);
        } else {               // a = p, b = z
            a[i] = b[i] + coef * a[i];
        }
    }
    if (OP != 2) {
        const double s = block_sum<kVecBlock>(acc, red);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}

__global__ void finish_kernel(int nparts, const double *__restrict__ part, double *__restrict__ out,
                              const int32_t *done) {
    __shared__ double red[32];
    if (done != nullptr && *((volatile const int32_t *)done)) return;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kVecBlock) acc += part[i];
    const double s = block_sum<kVecBlock>(acc, red);
    if (threadIdx.x == 0) out[0] = s;
}

__global__ void roll_kernel(double *sc, const int32_t *done) {
    if (done == nullptr || !*done) sc[1] = sc[0];
}

__global__ void check_kernel(const double *rr, double bnorm, double tol, int64_t max_it, int32_t *done,
                             int64_t *it, double *res) {
    if (*done) return;
    const int64_t k = *it + 1;
    *it = k;
    const double r = sqrt(*rr) / bnorm;
    *res = r;
    if (r <= tol || k >= max_it) *done = 1;
}

__global__ void gather_kernel(int64_t m, const int32_t *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

__global__ void scatter_kernel(int64_t m, const int32_t *__restrict__ idx, const double *__restrict__ src,
                               double *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        dst[idx[i]] = src[i];
}

static int grid_for(int64_t n, int per = kVecBlock) {
    int64_t g = (n + per - 1) / per;
    if (g > kVecGrid) g = kVecGrid;
    return (int)(g > 0 ? g : 1);
}

}  // namespace tsb

// out[0] = sum_i w_i a_i b_i; `part` is scratch of kNumSM * 2 doubles.
extern "C" int tsb_wdot(int64_t n, const double *d_w, const double *d_a, const double *d_b, double *d_part,
                        double *d_out, void *stream) {
    using namespace tsb;
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        const int g = grid_for(n);
        vec_kernel<0><<<g, kVecBlock, 0, s>>>(n, d_w, const_cast<double *>(d_a), const_cast<double *>(d_b),
                                              nullptr, nullptr, nullptr, d_part, nullptr);
        finish_kernel<<<1, kVecBlock, 0, s>>>(g, d_part, d_out, nullptr);
        count_launch(2);
        TSB_CUDA(cudaGetLastError());
    });
}

// alpha = d_sc[0] / d_sc[1]; x += alpha p; r -= alpha ap; d_out[0] = sum w r^2
extern "C" int tsb_pcg_update(int64_t n, const double *d_w, double *d_x, const double *d_p, double *d_r,
                              const double *d_ap, const double *d_sc, double *d_part, double *d_out,
                              const int32_t *d_done, void *stream) {
    using namespace tsb;
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        const int g = grid_for(n);
        vec_kernel<1><<<g, kVecBlock, 0, s>>>(n, d_w, d_x, const_cast<double *>(d_p), d_r,
                                              const_cast<double *>(d_ap), d_sc, d_part, d_done);
        finish_kernel<<<1, kVecBlock, 0, s>>>(g, d_part, d_out, d_done);
        count_launch(2);
        TSB_CUDA(cudaGetLastError());
    });
}

// beta = d_sc[0] / d_sc[1]; p = z + beta p; then d_sc[1] = d_sc[0]
extern "C" int tsb_pcg_direction(int64_t n, double *d_p, const double *d_z, double *d_sc, const int32_t *d_done,
                                 void *stream) {
    using namespace tsb;
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        vec_kernel<2><<<grid_for(n), kVecBlock, 0, s>>>(n, nullptr, d_p, const_cast<double *>(d_z), nullptr,
                                                        nullptr, d_sc, nullptr, d_done);
        roll_kernel<<<1, 1, 0, s>>>(d_sc, d_done);
        count_launch(2);
        TSB_CUDA(cudaGetLastError());
    });
}

extern "C" int tsb_pcg_check(const double *d_rr, double bnorm, double tol, int64_t max_it, int32_t *d_done,
                             int64_t *d_it, double *d_res, void *stream) {
    using namespace tsb;
    return guard([&] {
        check_kernel<<<1, 1, 0, as_stream(stream)>>>(d_rr, bnorm, tol, max_it, d_done, d_it, d_res);
        count_launch();
        TSB_CUDA(cudaGetLastError());
    });
}

extern "C" int tsb_gather_rows(int64_t m, const int32_t *d_idx, const double *d_src, double *d_dst, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (m <= 0) return;
        gather_kernel<<<grid_for(m), kVecBlock, 0, as_stream(stream)>>>(m, d_idx, d_src, d_dst);
        count_launch();
        TSB_CUDA(cudaGetLastError());
    });
}

extern "C" int tsb_scatter_rows(int64_t m, const int32_t *d_idx, const double *d_src, double *d_dst, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (m <= 0) return;
        scatter_kernel<<<grid_for(m), kVecBlock, 0, as_stream(stream)>>>(m, d_idx, d_src, d_dst);
        count_launch();
        TSB_CUDA(cudaGetLastError());
    });
}
