// CSR SpMV (bit-exact with krylov.spmv, krylov.py:73-96) and CSR diagonal
// extraction (CsrMatrix.diagonal, assembly.py:154-159).
#include "peer_exchange.cuh"
#include "spmv_exact.cuh"

namespace tsb {

constexpr int kSpmvBlock = 256;  // 32 rows per CTA (8 lanes per row)

__global__ void __launch_bounds__(kSpmvBlock, 8)
spmv_kernel(int64_t nrows, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
            const double *__restrict__ val, const double *__restrict__ x, double *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int lane8 = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const int64_t groups = (int64_t)gridDim.x * (kSpmvBlock / 8);
    XPlain xa{x};
    for (int64_t row = (int64_t)blockIdx.x * (kSpmvBlock / 8) + (threadIdx.x >> 3); row < nrows;
         row += groups) {
        const int lo = __ldg(rp + row), hi = __ldg(rp + row + 1);
        const double s = row_sum_exact(lo, hi - lo, ci, val, xa, lane8, gmask);
        if (lane8 == 0) y[row] = s;
    }
}

// SpMV followed by the peer all-reduce of the rows shared between ranks, in
// ONE kernel: every CTA computes its rows; the last CTA to finish (atomic
// ticket after a device fence) exchanges the shared rows over peer memory
// and resets the ticket -- the exchange starts the moment the local product
// is complete, without a kernel boundary or a host-issued collective.
__global__ void __launch_bounds__(kSpmvBlock, 8)
spmv_exchange_kernel(int64_t nrows, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                     const double *__restrict__ val, const double *__restrict__ x, double *y, PeerArgs P,
                     int32_t *ticket) {
    const int lane = threadIdx.x & 31;
    const int lane8 = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const int64_t groups = (int64_t)gridDim.x * (kSpmvBlock / 8);
    XPlain xa{x};
    for (int64_t row = (int64_t)blockIdx.x * (kSpmvBlock / 8) + (threadIdx.x >> 3); row < nrows;
         row += groups) {
        const int lo = __ldg(rp + row), hi = __ldg(rp + row + 1);
        const double s = row_sum_exact(lo, hi - lo, ci, val, xa, lane8, gmask);
        if (lane8 == 0) y[row] = s;
    }
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    exchange_block(P, y);
    if (threadIdx.x == 0) *ticket = 0;
}

__global__ void csr_diag_kernel(int64_t nrows, int64_t ncols, const int32_t *__restrict__ rp,
                                const int32_t *__restrict__ ci, const double *__restrict__ val,
                                double *__restrict__ d) {
    const int64_t nd = nrows < ncols ? nrows : ncols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        const int lo = rp[i], hi = rp[i + 1];
        // columns are strictly increasing per row: binary search
        int a = lo, b = hi;
        while (a < b) {
            int mid = (a + b) >> 1;
            if (ci[mid] < i) a = mid + 1; else b = mid;
        }
        if (a < hi && ci[a] == i) v = val[a];
        d[i] = v;
    }
}

int spmv_grid(int64_t nrows) {
    int64_t need = (nrows + (kSpmvBlock / 8) - 1) / (kSpmvBlock / 8);
    int64_t cap = (int64_t)kNumSM * 8;
    return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

void launch_spmv(int64_t nrows, const int32_t *rp, const int32_t *ci, const double *val,
                 const double *x, double *y, cudaStream_t s) {
    if (nrows <= 0) return;
    spmv_kernel<<<spmv_grid(nrows), kSpmvBlock, 0, s>>>(nrows, rp, ci, val, x, y);
    TSB_LAUNCHED();
}

void launch_csr_diag(int64_t nrows, int64_t ncols, const int32_t *rp, const int32_t *ci,
                     const double *val, double *d, cudaStream_t s) {
    int64_t nd = nrows < ncols ? nrows : ncols;
    if (nd <= 0) return;
    int grid = (int)((nd + 255) / 256);
    if (grid > kNumSM * 8) grid = kNumSM * 8;
    csr_diag_kernel<<<grid, 256, 0, s>>>(nrows, ncols, rp, ci, val, d);
    TSB_LAUNCHED();
}

}  // namespace tsb

extern "C" int tsb_spmv(int64_t nrows, const int32_t *d_row_ptr, const int32_t *d_col_ind,
                        const double *d_values, const double *d_x, double *d_y, void *stream) {
    return tsb::guard([&] {
        if (nrows < 0) throw tsb::Error(TSB_E_ARG, "nrows must be >= 0");
        tsb::launch_spmv(nrows, d_row_ptr, d_col_ind, d_values, d_x, d_y, tsb::as_stream(stream));
    });
}

extern "C" int tsb_csr_diagonal(int64_t nrows, int64_t ncols, const int32_t *d_row_ptr,
                                const int32_t *d_col_ind, const double *d_values, double *d_diag,
                                void *stream) {
    return tsb::guard([&] {
        tsb::launch_csr_diag(nrows, ncols, d_row_ptr, d_col_ind, d_values, d_diag,
                             tsb::as_stream(stream));
    });
}

// y = A x (local rows), then the rows d_idx[0..m) of y all-reduced over the
// ranks' peer memory (see tsb_peer_allreduce), in one kernel.  d_ticket: one
// int32, zero before the first call (the kernel leaves it zero).
extern "C" int tsb_spmv_peer(int64_t nrows, const int32_t *d_row_ptr, const int32_t *d_col_ind,
                             const double *d_values, const double *d_x, double *d_y, int64_t m, int32_t world,
                             int32_t rank, double *const *d_bufs, int64_t *const *d_flags, const int32_t *d_idx,
                             int64_t epoch, int64_t half, int32_t *d_ticket, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (nrows <= 0) throw Error(TSB_E_ARG, "nrows must be > 0");
        if (m < 0 || m > half || world < 1 || rank < 0 || rank >= world) throw Error(TSB_E_ARG, "bad peer arguments");
        PeerArgs P{m, world, rank, d_bufs, d_flags, d_idx, epoch, half};
        spmv_exchange_kernel<<<spmv_grid(nrows), kSpmvBlock, 0, as_stream(stream)>>>(
            nrows, d_row_ptr, d_col_ind, d_values, d_x, d_y, P, d_ticket);
        TSB_LAUNCHED();
    });
}
