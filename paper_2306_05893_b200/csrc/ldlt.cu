// Nested-dissection LDL^T apply on the B200: one persistent, dependency-driven
// kernel per triangular sweep (the paper's level-scheduled GPU Cholesky apply,
// with the level barriers replaced by per-block completion counters).
//
// Replaces solve_lower (ndprecond.py:647-671, _forward_block 623-631),
// solve_upper (674-691, _backward_block 634-644) and apply (694-700).  Factor
// values come from the host factorisation (ldlt_factor, ndprecond.py:501-572)
// and are re-packed on the host (paper_2306_05893_b200/_ldlt_pack.py) into one
// matrix per dissection block,
//     G_b = [inv(L11) - I ; L21 inv(L11)]          (layout: include/tsb.h),
// i.e. the reference's t x t tile inverses (ndprecond.py:575-587) widened to
// the whole diagonal block and folded into the coupling panel.  The in-block
// dependency chain of the tile substitution disappears: every block is one
// GEMV per sweep, split into many independent row chunks (lower) or column
// slab x row tiles (upper), so the only serial chain left is the depth of
// the dissection tree (one hop per level).
// Work items (dispatched in a precomputed topological, critical-path-first
// order through one atomic ticket counter; every CTA is resident, so an item
// only ever waits on items dispensed before it) are tiles of 32 rows of G_b
// (lower) or G_b^T (upper), lane-interleaved so each lane owns one row, staged
// by TMA bulk copies issued before the item's wait:
//   lower  triangle rows give y_b, M rows give the contributions to the
//          ancestors (column-major pre-accumulation, paper Fig. solveBlock)
//          written to row-contiguous slots; x_b = input - contributions is
//          summed in a fixed order (deterministic, no atomics on data) by the
//          block's own items or once by the child item that completes it.
//   upper  z_b = w_b + G_b^T [w_b; -z_anc] for a range of the block's columns
//          (row-major pull); only -z_anc waits for the parent.
// Counters are reset by the last CTA to leave, so the kernels replay inside
// the persistent PCG without memsets.
#include <cstdlib>
#include <mutex>
#include <vector>

#include "ldlt_sweep.cuh"
#include "peer_exchange.cuh"

struct tsb_ldlt {
    tsb_ldlt_desc d;
    uint64_t serial;
};

namespace tsb {

template <bool TRACE, bool MULTI = false>
__global__ void __launch_bounds__(kSweepBlock) lower_sweep(tsb_ldlt_desc D, SweepArgs A) {
    extern __shared__ __align__(128) double smem[];
    __shared__ SweepRing R;
    if (A.done != nullptr && *((volatile const int32_t *)A.done)) {
        lower_exit(D);
        return;
    }
    ring_init(R);
    lower_sweep_body<TRACE, MULTI>(D, A, smem, R);
}

template <bool TRACE>
__global__ void __launch_bounds__(kSweepBlock) upper_sweep(tsb_ldlt_desc D, SweepArgs A) {
    extern __shared__ __align__(128) double smem[];
    __shared__ SweepRing R;
    if (A.done != nullptr && *((volatile const int32_t *)A.done)) {
        upper_exit(D);
        return;
    }
    ring_init(R);
    upper_sweep_body<TRACE>(D, A, smem, R);
}

__global__ void permute_kernel(int64_t n, const int32_t *__restrict__ perm, const double *__restrict__ r,
                               double *__restrict__ out, const int32_t *done) {
    if (done != nullptr && *((volatile const int32_t *)done)) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __ldg(r + perm[i]);
}

static uint64_t g_serial = 0;
static std::mutex g_serial_mu;

// Co-resident (cooperative) launch: items only ever wait on earlier tickets,
// which is deadlock-free exactly when every CTA of the grid is resident.
template <class K>
static void launch_coop(K kernel, int grid, size_t smem, cudaStream_t st, tsb_ldlt_desc &D, SweepArgs &a) {
    sync_pub_direct();
    // TSB_SHARED_DEVICE=1: several processes share one GPU (the 2-rank shard test
    // on a 1-GPU box), where the driver refuses cooperative launches; the grid
    // (<= one CTA per SM there) is still co-resident, launch it plainly
    static const bool shared = getenv("TSB_SHARED_DEVICE") != nullptr;
    if (shared) {
        kernel<<<grid, kSweepBlock, smem, st>>>(D, a);
        TSB_CUDA(cudaGetLastError());
    } else {
        void *args[] = {&D, &a};
        TSB_CUDA(cudaLaunchCooperativeKernel((const void *)kernel, dim3(grid), dim3(kSweepBlock), args, smem, st));
    }
    count_launch();
}

void ldlt_enqueue(tsb_ldlt_t h, int mode, const double *r, double *out, const int32_t *done,
                  cudaStream_t st) {
    // mode 0: lower (r permuted -> out permuted); 1: upper; 2: apply
    tsb_ldlt_desc &D = h->d;
    if (D.n == 0) return;
    const int grid = D.grid;
    if (mode == 2 && D.d_rin != nullptr) {  // r through perm once: the sweep's items then read it directly
        int g = (int)((D.n + 255) / 256);
        if (g > kNumSM * 8) g = kNumSM * 8;
        permute_kernel<<<g, 256, 0, st>>>(D.n, D.d_perm, r, D.d_rin, done);
        TSB_LAUNCHED();
    }
    if (mode == 0 || mode == 2) {
        const bool pre = mode == 2 && D.d_rin != nullptr;
        SweepArgs a{pre ? D.d_rin : r, (mode == 2 && !pre) ? D.d_perm : nullptr, nullptr, mode == 2 ? D.d_y : out,
                    nullptr, nullptr, done};
        if (D.d_trace_lower)
            launch_coop(lower_sweep<true>, grid, sweep_smem_lower(D), st, D, a);
        else
            launch_coop(lower_sweep<false>, grid, sweep_smem_lower(D), st, D, a);
    }
    if (mode == 1 || mode == 2) {
        // apply: w = y / d read from d_y, z (permuted) into d_x, scattered through perm
        SweepArgs a{mode == 2 ? D.d_y : r, nullptr, mode == 2 ? D.d_d : nullptr, mode == 2 ? D.d_x : out,
                    mode == 2 ? D.d_perm : nullptr, mode == 2 ? out : nullptr, done};
        if (D.d_trace_upper)
            launch_coop(upper_sweep<true>, grid, sweep_smem_upper(D), st, D, a);
        else
            launch_coop(upper_sweep<false>, grid, sweep_smem_upper(D), st, D, a);
    }
}

__global__ void ext_sums_kernel(tsb_ldlt_desc D, double *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D.n_ext; i += (int64_t)gridDim.x * blockDim.x) {
        const int row = D.d_ext_rows[i];
        out[row] = contrib_sum<true>(D.d_cbuf, D.d_cin_ptr[row], D.d_cin_ptr[row + 1]);
    }
}

// external sums + the peer all-reduce of the shared rows in one kernel (the
// last CTA exchanges, as spmv_exchange_kernel)
__global__ void ext_sums_peer_kernel(tsb_ldlt_desc D, double *out, PeerArgs P, int32_t *ticket) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D.n_ext; i += (int64_t)gridDim.x * blockDim.x) {
        const int row = D.d_ext_rows[i];
        out[row] = contrib_sum<true>(D.d_cbuf, D.d_cin_ptr[row], D.d_cin_ptr[row + 1]);
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
    exchange_block(P, out);
    if (threadIdx.x == 0) *ticket = 0;
}

void ldlt_enqueue_ext(tsb_ldlt_t h, int mode, const double *r, const double *ext, double *out, cudaStream_t st) {
    tsb_ldlt_desc &D = h->d;
    if (D.n == 0 || D.n_blocks == 0) return;
    if (mode == 0) {  // lower with external contributions
        SweepArgs a{r, nullptr, nullptr, out, nullptr, nullptr, nullptr, ext};
        launch_coop(lower_sweep<false>, D.grid, sweep_smem_lower(D), st, D, a);
    } else if (mode == 1) {  // upper with D scaling, in place into out (permuted)
        SweepArgs a{r, nullptr, D.d_d, out, nullptr, nullptr, nullptr, nullptr};
        launch_coop(upper_sweep<false>, D.grid, sweep_smem_upper(D), st, D, a);
    } else {
        if (D.n_ext == 0) return;
        int g = (int)((D.n_ext + 255) / 256);
        if (g > kNumSM * 4) g = kNumSM * 4;
        ext_sums_kernel<<<g, 256, 0, st>>>(D, out);
        TSB_LAUNCHED();
    }
}

const tsb_ldlt_desc &ldlt_desc(tsb_ldlt_t h) { return h->d; }
uint64_t ldlt_serial(tsb_ldlt_t h) { return h->serial; }

}  // namespace tsb

extern "C" int tsb_ldlt_create(const tsb_ldlt_desc *desc, tsb_ldlt_t *out) {
    using namespace tsb;
    return guard([&] {
        if (desc == nullptr || out == nullptr) throw Error(TSB_E_ARG, "null desc/out");
        if (desc->max_v > kMaxV || desc->max_v < 1)
            throw Error(TSB_E_ARG, "item window larger than the vector staging buffer");
        if (desc->max_cb < 0 || desc->max_cb > 4096) throw Error(TSB_E_ARG, "bad contribution staging size");
        auto *h = new tsb_ldlt;
        h->d = *desc;
        const size_t ls = sweep_smem_lower(*desc), us = sweep_smem_upper(*desc);
        for (auto fn : {lower_sweep<false>, lower_sweep<true>})
            allow_max_smem(fn);
        for (auto fn : {upper_sweep<false>, upper_sweep<true>})
            allow_max_smem(fn);
        int per_sm_l = 0, per_sm_u = 0;
        TSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_l, lower_sweep<true>, kSweepBlock, ls));
        TSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_u, upper_sweep<true>, kSweepBlock, us));
        int per_sm = per_sm_l < per_sm_u ? per_sm_l : per_sm_u;
        if (per_sm < 1) {
            delete h;
            throw Error(TSB_E_ARG, "sweep kernels do not fit on an SM");
        }
        int dev = 0, nsm = kNumSM;
        TSB_CUDA(cudaGetDevice(&dev));
        TSB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        // persistent grid: every CTA resident (items only wait on earlier tickets)
        int want = desc->grid > 0 ? desc->grid : nsm * per_sm;
        h->d.grid = want < nsm * per_sm ? want : nsm * per_sm;
        {
            std::lock_guard<std::mutex> lk(g_serial_mu);
            h->serial = ++g_serial;
        }
        *out = h;
    });
}

extern "C" int tsb_ldlt_destroy(tsb_ldlt_t h) {
    delete h;
    return TSB_OK;
}

extern "C" int tsb_ldlt_lower(tsb_ldlt_t h, const double *d_r, double *d_y, void *stream) {
    return tsb::guard([&] { tsb::ldlt_enqueue(h, 0, d_r, d_y, nullptr, tsb::as_stream(stream)); });
}

extern "C" int tsb_ldlt_upper(tsb_ldlt_t h, const double *d_w, double *d_z, void *stream) {
    return tsb::guard([&] { tsb::ldlt_enqueue(h, 1, d_w, d_z, nullptr, tsb::as_stream(stream)); });
}

extern "C" int tsb_ldlt_apply(tsb_ldlt_t h, const double *d_r, double *d_z, void *stream) {
    return tsb::guard([&] { tsb::ldlt_enqueue(h, 2, d_r, d_z, nullptr, tsb::as_stream(stream)); });
}

// y_j = L^-1 r_j for nr right-hand sides in one sweep (every factor tile read
// once for all of them); r, y: [nr][n] permuted; scratch: cbuf [nr][ld_cb]
// (ld_cb >= contribution slots), x [nr][n], part [nr][ld_part] (>= the lower
// segment partials).
extern "C" int tsb_ldlt_lower_multi(tsb_ldlt_t h, int32_t nr, const double *d_r, double *d_y, double *d_cbuf,
                                    int64_t ld_cb, double *d_x, double *d_part, int64_t ld_part, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (h == nullptr || nr < 1) throw Error(TSB_E_ARG, "bad multi-RHS lower sweep");
        tsb_ldlt_desc D = h->d;
        if (D.n == 0) return;
        const size_t smem = sweep_smem_lower(D, nr);
        int dev = 0, optin = 0;
        TSB_CUDA(cudaGetDevice(&dev));
        TSB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        if (smem + 8192 > (size_t)optin) throw Error(TSB_E_ARG, "too many right-hand sides for the staging buffer");
        D.d_cbuf = d_cbuf;
        D.d_x = d_x;
        D.d_part_lower = d_part;
        SweepArgs a{d_r, nullptr, nullptr, d_y, nullptr, nullptr, nullptr, nullptr};
        a.nr = nr;
        a.ld = D.n;
        a.ld_cb = ld_cb;
        a.ld_part = ld_part;
        // the grid of the handle was sized for the 1-RHS footprint: keep it co-resident
        int per_sm = 0;
        static bool once = [] {
            allow_max_smem(lower_sweep<false, true>);
            return true;
        }();
        (void)once;
        if (nr > 8) throw Error(TSB_E_ARG, "at most 8 right-hand sides per multi-RHS sweep");
        TSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lower_sweep<false, true>, kSweepBlock, smem));
        int nsm = kNumSM;
        TSB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int grid = D.grid < nsm * per_sm ? D.grid : nsm * per_sm;
        if (grid < 1) throw Error(TSB_E_ARG, "multi-RHS lower sweep does not fit on an SM");
        launch_coop(lower_sweep<false, true>, grid, smem, as_stream(stream), D, a);
    });
}

extern "C" int tsb_ldlt_lower_ext(tsb_ldlt_t h, const double *d_r, const double *d_ext, double *d_y, void *stream) {
    return tsb::guard([&] { tsb::ldlt_enqueue_ext(h, 0, d_r, d_ext, d_y, tsb::as_stream(stream)); });
}

extern "C" int tsb_ldlt_upper_scaled(tsb_ldlt_t h, const double *d_y, double *d_z, void *stream) {
    return tsb::guard([&] { tsb::ldlt_enqueue_ext(h, 1, d_y, nullptr, d_z, tsb::as_stream(stream)); });
}

extern "C" int tsb_ldlt_external_sums(tsb_ldlt_t h, double *d_out, void *stream) {
    return tsb::guard([&] { tsb::ldlt_enqueue_ext(h, 2, nullptr, nullptr, d_out, tsb::as_stream(stream)); });
}

// tsb_ldlt_external_sums followed by the peer all-reduce of d_out's rows
// d_idx[0..m) (see tsb_peer_allreduce), in one kernel; d_ticket: one int32,
// initially zero.
extern "C" int tsb_ldlt_external_sums_peer(tsb_ldlt_t h, double *d_out, int64_t m, int32_t world, int32_t rank,
                                           double *const *d_bufs, int64_t *const *d_flags, const int32_t *d_idx,
                                           int64_t epoch, int64_t half, int32_t *d_ticket, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (h == nullptr) throw Error(TSB_E_ARG, "null ldlt handle");
        if (m < 0 || m > half || world < 1 || rank < 0 || rank >= world) throw Error(TSB_E_ARG, "bad peer arguments");
        const tsb_ldlt_desc &D = ldlt_desc(h);
        int g = (int)((D.n_ext + 255) / 256);
        if (g > kNumSM * 4) g = kNumSM * 4;
        if (g < 1) g = 1;
        PeerArgs P{m, world, rank, d_bufs, d_flags, d_idx, epoch, half};
        ext_sums_peer_kernel<<<g, 256, 0, as_stream(stream)>>>(D, d_out, P, d_ticket);
        TSB_LAUNCHED();
    });
}
