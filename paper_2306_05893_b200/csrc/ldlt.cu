// Nested-dissection LDL^T apply on the B200: one persistent, dependency-driven
// kernel per triangular sweep (the paper's level-scheduled GPU Cholesky apply,
// with the level barriers replaced by per-panel completion counters).
//
// Replaces solve_lower (ndprecond.py:647-671, _forward_block 623-631),
// solve_upper (674-691, _backward_block 634-644) and apply (694-700).  Factor
// values come from the host factorisation (ldlt_factor, ndprecond.py:501-572)
// and are re-cut on the host (paper_2306_05893_b200/_ldlt_pack.py) into
// PANELS: every dissection block is split into column panels of <= 128
// columns.  Panel p of block b owns columns [c0, c0+w) and stores
//   tri    the explicit inverse of its unit-lower w x w diagonal triangle --
//          the reference's tile_inv (ndprecond.py:575-587) widened from 16 to
//          the whole panel, so the in-panel solve is one dependency-free GEMV
//          (column-packed copy for the lower sweep, row-packed for the upper,
//          each read by its sweep only; staged in shared memory by one TMA copy);
//   P      its below panel: rows (block rows >= c0+w) U anc(b), w columns,
//          row-major, rows padded to an even stride -- [L11[c0+w:, c0:c0+w];
//          L21[:, c0:c0+w]] -- streamed chunk by chunk with TMA bulk copies.
// Work items (dispatched in a precomputed topological, critical-path-first
// order through one atomic ticket counter; every CTA is resident, so an item
// only ever waits on items dispensed before it):
//   lower  DIAG(p)        rows of p = input - contributions pre-accumulated by
//                         earlier panels (row-contiguous, summed in a fixed
//                         order -> deterministic, no atomics on data), then
//                         y_p = inv(L_pp) x_p
//          OFFDIAG(p,k)   contributions of y_p to a chunk of p's below rows
//                         (column-major pre-accumulation, paper Fig. solveBlock)
//   upper  OFFDIAG_T(p,k) partial sums P[k rows]^T z[below]        (row-major pull)
//          DIAG_T(p)      z_p = inv(L_pp)^T (w_p - sum of partials in chunk order)
// Counters (int32 per panel) are reset by the last CTA to leave, so the kernel
// can be replayed inside the PCG graph without extra memsets.
#include <mutex>
#include <vector>

#include "ldlt_sweep.cuh"

struct tsb_ldlt {
    tsb_ldlt_desc d;
    uint64_t serial;
};

namespace tsb {

template <bool TRACE>
__global__ void __launch_bounds__(kSweepBlock) lower_sweep(tsb_ldlt_desc D, SweepArgs A) {
    extern __shared__ __align__(128) double smem[];
    __shared__ uint64_t bar;
    if (A.done != nullptr && *((volatile const int32_t *)A.done)) {
        sweep_exit(D, D.d_ctl, D.d_cnt0, D.d_cnt1);
        return;
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    lower_sweep_body<TRACE>(D, A, smem, bar, phase);
}

template <bool TRACE>
__global__ void __launch_bounds__(kSweepBlock) upper_sweep(tsb_ldlt_desc D, SweepArgs A) {
    extern __shared__ __align__(128) double smem[];
    __shared__ uint64_t bar;
    if (A.done != nullptr && *((volatile const int32_t *)A.done)) {
        sweep_exit(D, D.d_ctl + 2, D.d_cnt2, D.d_cnt3);
        return;
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    upper_sweep_body<TRACE>(D, A, smem, bar, phase);
}

static uint64_t g_serial = 0;
static std::mutex g_serial_mu;

// Co-resident (cooperative) launch: items only ever wait on earlier tickets,
// which is deadlock-free exactly when every CTA of the grid is resident.
template <class K>
static void launch_coop(K kernel, int grid, size_t smem, cudaStream_t st, tsb_ldlt_desc &D, SweepArgs &a) {
    void *args[] = {&D, &a};
    TSB_CUDA(cudaLaunchCooperativeKernel((const void *)kernel, dim3(grid), dim3(kSweepBlock), args, smem, st));
    count_launch();
}

void ldlt_enqueue(tsb_ldlt_t h, int mode, const double *r, double *out, const int32_t *done,
                  cudaStream_t st) {
    // mode 0: lower (r permuted -> out permuted); 1: upper; 2: apply
    tsb_ldlt_desc &D = h->d;
    if (D.n == 0) return;
    const int grid = D.grid;
    if (mode == 0 || mode == 2) {
        SweepArgs a{r, mode == 2 ? D.d_perm : nullptr, nullptr, mode == 2 ? D.d_y : out, nullptr, nullptr, done};
        if (D.d_trace_lower)
            launch_coop(lower_sweep<true>, grid, sweep_smem_lower(D), st, D, a);
        else
            launch_coop(lower_sweep<false>, grid, sweep_smem_lower(D), st, D, a);
    }
    if (mode == 1 || mode == 2) {
        SweepArgs a{mode == 2 ? D.d_y : r, nullptr, mode == 2 ? D.d_d : nullptr, mode == 2 ? D.d_y : out,
                    mode == 2 ? D.d_perm : nullptr, mode == 2 ? out : nullptr, done};
        if (D.d_trace_upper)
            launch_coop(upper_sweep<true>, grid, sweep_smem_upper(D), st, D, a);
        else
            launch_coop(upper_sweep<false>, grid, sweep_smem_upper(D), st, D, a);
    }
}

const tsb_ldlt_desc &ldlt_desc(tsb_ldlt_t h) { return h->d; }
uint64_t ldlt_serial(tsb_ldlt_t h) { return h->serial; }

}  // namespace tsb

extern "C" int tsb_ldlt_create(const tsb_ldlt_desc *desc, tsb_ldlt_t *out) {
    using namespace tsb;
    return guard([&] {
        if (desc == nullptr || out == nullptr) throw Error(TSB_E_ARG, "null desc/out");
        if (desc->tile != kT) throw Error(TSB_E_ARG, "device tile must be 16");
        if (desc->panel_width > kMaxW) throw Error(TSB_E_ARG, "panel width exceeds 128");
        auto *h = new tsb_ldlt;
        h->d = *desc;
        const size_t ls = sweep_smem_lower(*desc), us = sweep_smem_upper(*desc);
        for (auto fn : {lower_sweep<false>, lower_sweep<true>})
            TSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ls));
        for (auto fn : {upper_sweep<false>, upper_sweep<true>})
            TSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)us));
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
