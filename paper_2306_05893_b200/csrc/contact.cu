// Plane-contact stage on the device (contact.py:89-257 of the reference):
// detection, compliance columns, Gram matrix, projected Gauss-Seidel and the
// motion correction.  With LDL^T factors the compliance is formed without
// the m full applies of the reference:
//     W = J A^-1 J^T = Y^T D^-1 Y,   Y = L^-1 P J^T   (lower sweeps only)
//     S lambda = P^T L^-T D^-1 (Y lambda)             (ONE upper sweep)
// Every reduction runs in a fixed order (bit-reproducible).
#include "tsb_common.cuh"

namespace tsb {
namespace ct {

constexpr int kBlock = 256;

// Ordered compaction of the nodes below the plane (one CTA; nodes ascending)
// + the maximum penetration max(plane - z, 0).
__global__ void __launch_bounds__(1024) plane_kernel(int64_t N, const double *__restrict__ pos, double plane_z,
                                                     int32_t *__restrict__ nodes, double *__restrict__ pen,
                                                     int64_t *__restrict__ count, double *__restrict__ maxpen) {
    __shared__ int32_t wsum[32];
    __shared__ int64_t base;
    __shared__ double wmax[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) base = 0;
    double mx = 0.0;
    __syncthreads();
    for (int64_t i0 = 0; i0 < N; i0 += 1024) {
        const int64_t i = i0 + tid;
        double p = 0.0;
        bool hit = false;
        if (i < N) {
            p = plane_z - pos[3 * i + 2];
            hit = p > 0.0;
            mx = fmax(mx, p);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int off = 0, tot = 0;
        for (int w = 0; w < 32; ++w) {
            if (w < warp) off += wsum[w];
            tot += wsum[w];
        }
        if (hit) {
            const int64_t k = base + off + __popc(bal & ((1u << lane) - 1u));
            if (nodes != nullptr) {
                nodes[k] = (int32_t)i;
                pen[k] = p;
            }
        }
        __syncthreads();
        if (tid == 0) base += tot;
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) wmax[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < 32; ++w) m = fmax(m, wmax[w]);
        *count = base;
        *maxpen = m;
    }
}

// R[:, i] = row i of J scattered (through iperm when given); R zeroed by the caller.
__global__ void rhs_kernel(int64_t m, const int64_t *__restrict__ indptr, const int32_t *__restrict__ cols,
                           const double *__restrict__ coefs, const int32_t *__restrict__ iperm, int64_t n,
                           double *__restrict__ R) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t q = indptr[i]; q < indptr[i + 1]; ++q) {
            const int64_t c = iperm ? iperm[cols[q]] : cols[q];
            R[i * n + c] += coefs[q];
        }
}

// Gram partials: part[chunk][i][j] = sum_{r in chunk} (Y_ri Y_rj) w_r  (w = 1/d or 1)
constexpr int kGT = 16;       // 16 x 16 output tile per CTA
constexpr int kChunk = 2048;  // rows per chunk
__global__ void __launch_bounds__(256) gram_kernel(int64_t n, int64_t m, const double *__restrict__ Y,
                                                   const double *__restrict__ d, double *__restrict__ part) {
    __shared__ double yi[64][kGT + 1], yj[64][kGT + 1], ws[64];
    const int ti = threadIdx.x & 15, tj = threadIdx.x >> 4;
    const int64_t i = blockIdx.x * kGT + ti, j = blockIdx.y * kGT + tj;
    const int64_t r0 = (int64_t)blockIdx.z * kChunk, r1 = min(n, r0 + kChunk);
    double acc = 0.0;
    for (int64_t rb = r0; rb < r1; rb += 64) {
        for (int q = threadIdx.x; q < 64 * kGT; q += 256) {
            const int rr = q & 63, c = q >> 6;
            const int64_t r = rb + rr;
            const int64_t ci = blockIdx.x * kGT + c, cj = blockIdx.y * kGT + c;
            yi[rr][c] = (r < r1 && ci < m) ? Y[ci * n + r] : 0.0;
            yj[rr][c] = (r < r1 && cj < m) ? Y[cj * n + r] : 0.0;
        }
        if (threadIdx.x < 64) {
            const int64_t r = rb + threadIdx.x;
            ws[threadIdx.x] = r < r1 ? (d ? 1.0 / d[r] : 1.0) : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int rr = 0; rr < 64; ++rr) acc = fma(yi[rr][ti] * yj[rr][tj], ws[rr], acc);
        __syncthreads();
    }
    if (i < m && j < m) part[((int64_t)blockIdx.z * m + i) * m + j] = acc;
}

__global__ void gram_reduce(int64_t m, int nchunk, const double *__restrict__ part, double scale,
                            double *__restrict__ W) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m * m; k += (int64_t)gridDim.x * blockDim.x) {
        double a = 0.0;
        for (int c = 0; c < nchunk; ++c) a += part[(int64_t)c * m * m + k];
        W[k] = scale * a;
    }
}

// W_ij = (J S)_ij = sum_q coef_q S[col_q, j] over row i of J, symmetrised by
// averaging (contact.py:119-124)
__device__ __forceinline__ double jrow_dot(const int64_t *indptr, const int32_t *cols, const double *coefs,
                                           const double *Sj, int64_t i) {
    double a = 0.0;
    for (int64_t q = indptr[i]; q < indptr[i + 1]; ++q) a += coefs[q] * Sj[cols[q]];
    return a;
}
__global__ void jsym_kernel(int64_t m, int64_t n, const int64_t *__restrict__ indptr, const int32_t *__restrict__ cols,
                            const double *__restrict__ coefs, const double *__restrict__ S, double scale,
                            double *__restrict__ W) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m * m; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = k / m, j = k - i * m;
        const double wij = jrow_dot(indptr, cols, coefs, S + j * n, i), wji = jrow_dot(indptr, cols, coefs, S + i * n, j);
        W[k] = scale * (0.5 * (wij + wji));
    }
}

// Projected Gauss-Seidel (contact.py:128-166), one warp: row dot products
// lane-strided with a fixed shuffle tree; lambda in shared memory.
// info: [0] sweeps, [1] complementarity residual sum |lam (W lam - rhs)|, [2] dropped rows
__global__ void __launch_bounds__(32) pgs_kernel(int64_t m, const double *W, const double *__restrict__ rhs,
                                                 const uint8_t *__restrict__ unilateral, double tol, int max_sweeps,
                                                 double *__restrict__ lam_out, double *__restrict__ info,
                                                 bool W_in_smem) {
    extern __shared__ double lam[];  // [m] multipliers, then W itself when it fits (row dots from smem)
    const int lane = threadIdx.x;
    for (int64_t i = lane; i < m; i += 32) lam[i] = 0.0;
    double *Ws = lam + ((m + 1) & ~1);
    if (W_in_smem) {
        for (int64_t i = lane; i < m * m; i += 32) Ws[i] = W[i];
        W = Ws;
    }
    __syncwarp();
    int dropped = 0;
    for (int64_t i = 0; i < m; ++i) dropped += W[i * m + i] == 0.0;
    int sweeps = 0;
    for (int s = 0; s < max_sweeps; ++s) {
        ++sweeps;
        double dmax = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            const double dii = W[i * m + i];
            double a = 0.0;
            for (int64_t j = lane; j < m; j += 32) a = fma(W[i * m + j], lam[j], a);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            double nv = 0.0;
            if (dii != 0.0) {
                nv = lam[i] + (rhs[i] - a) / dii;
                if (unilateral[i] && nv < 0.0) nv = 0.0;
            }
            dmax = fmax(dmax, fabs(nv - lam[i]));
            __syncwarp();
            if (lane == 0) lam[i] = nv;
            __syncwarp();
        }
        double sc = 0.0;
        for (int64_t i = lane; i < m; i += 32) sc = fmax(sc, fabs(lam[i]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
        if (dmax <= tol * sc || sc == 0.0) break;
    }
    double res = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        double a = 0.0;
        for (int64_t j = lane; j < m; j += 32) a = fma(W[i * m + j], lam[j], a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        res += fabs(lam[i] * (a - rhs[i]));
    }
    for (int64_t i = lane; i < m; i += 32) lam_out[i] = lam[i];
    if (lane == 0) {
        info[0] = sweeps;
        info[1] = res;
        info[2] = dropped;
    }
}

// out[r] = sum_i Y[r, i] lam_i (fixed column order)
__global__ void gemv_cols(int64_t n, int64_t m, const double *__restrict__ Y, const double *__restrict__ lam,
                          double *__restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        double a = 0.0;
        for (int64_t i = 0; i < m; ++i) a = fma(Y[i * n + r], lam[i], a);
        out[r] = a;
    }
}

// acc[c] = acc_free[c] - delta[iperm ? iperm[c] : c]
__global__ void correct_kernel(int64_t n, const double *__restrict__ acc_free, const double *__restrict__ delta,
                               const int32_t *__restrict__ iperm, double *__restrict__ acc) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
        acc[c] = acc_free[c] - delta[iperm ? iperm[c] : c];
}

inline int grid_of(int64_t n) {
    int64_t g = (n + kBlock - 1) / kBlock;
    if (g > kNumSM * 8) g = kNumSM * 8;
    return (int)(g > 0 ? g : 1);
}

}  // namespace ct
}  // namespace tsb

extern "C" int tsb_plane_contacts(int64_t n_nodes, const double *d_pos, double plane_z, int32_t *d_nodes,
                                  double *d_pen, int64_t *d_count, double *d_maxpen, void *stream) {
    using namespace tsb;
    return guard([&] {
        ct::plane_kernel<<<1, 1024, 0, as_stream(stream)>>>(n_nodes, d_pos, plane_z, d_nodes, d_pen, d_count, d_maxpen);
        TSB_LAUNCHED();
    });
}

extern "C" int tsb_contact_rhs(int64_t m, const int64_t *d_indptr, const int32_t *d_cols, const double *d_coefs,
                               const int32_t *d_iperm, int64_t n, double *d_R, void *stream) {
    using namespace tsb;
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        TSB_CUDA(cudaMemsetAsync(d_R, 0, sizeof(double) * n * m, s));
        if (m > 0) {
            ct::rhs_kernel<<<ct::grid_of(m), ct::kBlock, 0, s>>>(m, d_indptr, d_cols, d_coefs, d_iperm, n, d_R);
            TSB_LAUNCHED();
        }
    });
}

extern "C" int64_t tsb_gram_scratch(int64_t n, int64_t m) {
    return ((n + tsb::ct::kChunk - 1) / tsb::ct::kChunk) * m * m;
}

extern "C" int tsb_gram(int64_t n, int64_t m, const double *d_Y, const double *d_d, double scale, double *d_part,
                        double *d_W, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (m <= 0) return;
        cudaStream_t s = as_stream(stream);
        const int nchunk = (int)((n + ct::kChunk - 1) / ct::kChunk);
        dim3 g((unsigned)((m + ct::kGT - 1) / ct::kGT), (unsigned)((m + ct::kGT - 1) / ct::kGT), (unsigned)nchunk);
        ct::gram_kernel<<<g, 256, 0, s>>>(n, m, d_Y, d_d, d_part);
        ct::gram_reduce<<<ct::grid_of(m * m), ct::kBlock, 0, s>>>(m, nchunk, d_part, scale, d_W);
        count_launch(2);
        TSB_CUDA(cudaGetLastError());
    });
}

extern "C" int tsb_compliance_from_columns(int64_t m, int64_t n, const int64_t *d_indptr, const int32_t *d_cols,
                                           const double *d_coefs, const double *d_S, double scale, double *d_W,
                                           void *stream) {
    using namespace tsb;
    return guard([&] {
        if (m <= 0) return;
        ct::jsym_kernel<<<ct::grid_of(m * m), ct::kBlock, 0, as_stream(stream)>>>(m, n, d_indptr, d_cols, d_coefs, d_S,
                                                                                 scale, d_W);
        TSB_LAUNCHED();
    });
}

extern "C" int tsb_pgs(int64_t m, const double *d_W, const double *d_rhs, const uint8_t *d_unilateral, double tol,
                       int32_t max_sweeps, double *d_lam, double *d_info, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (m <= 0) return;
        size_t smem = sizeof(double) * (size_t)((m + 1) & ~1);
        if (smem > 200 * 1024) throw Error(TSB_E_ARG, "too many constraints for the shared-memory PGS");
        const bool w_smem = smem + sizeof(double) * (size_t)(m * m) <= 200 * 1024;
        if (w_smem) smem += sizeof(double) * (size_t)(m * m);
        static bool once = [] {
            allow_max_smem(ct::pgs_kernel);
            return true;
        }();
        (void)once;
        ct::pgs_kernel<<<1, 32, smem, as_stream(stream)>>>(m, d_W, d_rhs, d_unilateral, tol, max_sweeps, d_lam, d_info,
                                                          w_smem);
        TSB_LAUNCHED();
    });
}

extern "C" int tsb_gemv_cols(int64_t n, int64_t m, const double *d_Y, const double *d_lam, double *d_out,
                             void *stream) {
    using namespace tsb;
    return guard([&] {
        ct::gemv_cols<<<ct::grid_of(n), ct::kBlock, 0, as_stream(stream)>>>(n, m, d_Y, d_lam, d_out);
        TSB_LAUNCHED();
    });
}

extern "C" int tsb_contact_correct(int64_t n, const double *d_acc_free, const double *d_delta, const int32_t *d_iperm,
                                   double *d_acc, void *stream) {
    using namespace tsb;
    return guard([&] {
        ct::correct_kernel<<<ct::grid_of(n), ct::kBlock, 0, as_stream(stream)>>>(n, d_acc_free, d_delta, d_iperm, d_acc);
        TSB_LAUNCHED();
    });
}
