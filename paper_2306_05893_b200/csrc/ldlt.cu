// Nested-dissection LDL^T apply on the B200: one persistent, dependency-driven
// kernel per triangular sweep (the paper's level-scheduled GPU Cholesky apply,
// with the level barriers replaced by per-panel completion counters).
//
// Replaces solve_lower (ndprecond.py:647-671, _forward_block 623-631),
// solve_upper (674-691, _backward_block 634-644) and apply (694-700).  Factor
// values come from the host factorisation (ldlt_factor, ndprecond.py:501-572)
// and are re-cut on the host (paper_2306_05893_b200/ndprecond.py,
// DeviceFactors) into PANELS: every dissection block is split into column
// panels of <= 128 columns.  Panel p of block b owns columns [c0, c0+w) and
//   tri    the strict-lower w x w triangle as 16-wide tile-column panels plus
//          the 16x16 tile inverses (the reference's tile_inv, t = 16) --
//          contiguous, so one TMA bulk copy stages it in shared memory;
//   P      its "below" panel: rows (block rows >= c0+w) U anc(b), w columns,
//          row-major -- [L11[c0+w:, c0:c0+w]; L21[:, c0:c0+w]].
// Work items (dispatched in a precomputed topological, critical-path-first
// order through one atomic ticket counter; every CTA is resident, so an item
// only ever waits on items dispensed before it):
//   lower  DIAG(p)        rows of p = input - pre-accumulated contributions
//                         (gathered in a fixed order -> deterministic, no
//                         atomics on data), then the tile chain in smem
//                         (tile_inv matvec, column-major push) -> y[p]
//          OFFDIAG(p,k)   contributions of y[p] to a chunk of p's below rows
//                         (column-major pre-accumulation, paper Fig. solveBlock)
//   upper  OFFDIAG_T(p,k) partial sums of P[k rows]^T z[below]   (row-major pull)
//          DIAG_T(p)      w - sum of partials (chunk order), backward tile chain
//                         with tile_inv^T -> z[p]
// Counters (int32 per panel) are reset by the last CTA to leave, so the kernel
// can be replayed inside the PCG graph without extra memsets.
#include <mutex>
#include <vector>

#include "tsb_common.cuh"

struct tsb_ldlt {
    tsb_ldlt_desc d;
    uint64_t serial;
};

namespace tsb {

constexpr int kSweepBlock = 256;
constexpr int kT = 16;        // diagonal tile (the reference's default tile)
constexpr int kMaxW = 128;    // panel width
enum { IT_DIAG = 0, IT_OFF = 1, IT_OFFT = 2, IT_DIAGT = 3 };

struct Item {
    int32_t type, panel, r0, r1, dep_off, dep_cnt, out_off, pad;
};

// ---- small PTX helpers -----------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void spin_until_geq(const int *p, int target) {
    if (ld_acquire(p) >= target) return;
    int ns = 32;
    while (ld_acquire(p) < target) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

// Optional per-item timeline (globaltimer ns): [take, ready, end, smid].
__device__ __forceinline__ void trace(int64_t *buf, int iid, int slot) {
    if (buf != nullptr && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        buf[(int64_t)iid * 4 + slot] = (int64_t)t;
        if (slot == 0) {
            uint32_t sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            buf[(int64_t)iid * 4 + 3] = sm;
        }
    }
}

struct SweepArgs {
    const double *in;        // input vector (lower: r; upper: w)
    const int32_t *in_perm;  // lower apply: gather input through perm
    const double *dscale;    // upper apply: divide input by D
    double *x;               // lower: y (permuted)   upper: z (permuted)
    const int32_t *out_perm; // upper apply: scatter z through perm
    double *out;             // upper apply: output in original order
    const int32_t *done;     // PCG stop flag (skip when set)
};

// Exit protocol: the last CTA out zeroes the counters for the next replay.
__device__ __forceinline__ void sweep_exit(const tsb_ldlt_desc &D, int32_t *ctl, int32_t *c0, int32_t *c1) {
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ctl + 1, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    for (int64_t i = threadIdx.x; i < D.n_panels; i += blockDim.x) {
        c0[i] = 0;
        c1[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ctl[0] = 0;
        ctl[1] = 0;
        __threadfence();
    }
}

// ---------------------------------------------------------------------------
// lower sweep: L y = r
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSweepBlock)
lower_sweep(tsb_ldlt_desc D, SweepArgs A) {
    extern __shared__ __align__(128) double smem[];
    double *tri = smem;                               // staged tri + tinv of a DIAG panel
    double *seg = smem + D.tri_smem_doubles;          // panel rows (w <= 128)
    __shared__ uint64_t bar;
    __shared__ int item_id;
    __shared__ double tvec[kT];
    int32_t *ctl = D.d_ctl;
    int32_t *contrib = D.d_cnt0, *flag = D.d_cnt1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (A.done != nullptr && *((volatile const int32_t *)A.done)) {
        sweep_exit(D, ctl, contrib, flag);
        return;
    }
    if (tid == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    const Item *items = reinterpret_cast<const Item *>(D.d_items_lower);
    while (true) {
        if (tid == 0) item_id = atomicAdd(ctl, 1);
        __syncthreads();
        const int iid = item_id;
        if (iid >= D.n_items_lower) break;
        trace(D.d_trace_lower, iid, 0);
        const Item it = items[iid];
        const int p = it.panel;
        const int pstart = D.d_p_start[p], w = D.d_p_w[p];
        if (it.type == IT_DIAG) {
            const int ntiles = (w + kT - 1) / kT;
            const int64_t tbytes = D.d_p_tri_len[p] * 8;
            if (tid == 0) tma_load_1d(tri, D.d_tri + D.d_p_tri[p], (uint32_t)tbytes, &bar);
            if (tid == 0) spin_until_geq(contrib + p, it.dep_cnt);
            __syncthreads();
            trace(D.d_trace_lower, iid, 1);
            // rows: input - contributions pre-accumulated by earlier panels.  8 lanes
            // per row, lane-strided sums + xor tree: a fixed order (deterministic).
            for (int kb = warp * 4; kb < w; kb += kSweepBlock / 8) {
                const int k = kb + (lane >> 3), l8 = lane & 7;
                double acc = 0.0;
                if (k < w) {
                    const int row = pstart + k;
                    const int64_t q0 = D.d_cin_ptr[row], q1 = D.d_cin_ptr[row + 1];
#pragma unroll 4
                    for (int64_t q = q0 + l8; q < q1; q += 8) acc += __ldcg(D.d_cbuf + D.d_cin_idx[q]);
                }
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                if (k < w && l8 == 0) {
                    const int row = pstart + k;
                    seg[k] = A.in[A.in_perm ? A.in_perm[row] : row] - acc;
                }
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            __syncthreads();
            const double *tinv = tri + D.d_p_tri_len[p] - ntiles * kT * kT;
            const double *tp = tri;
            for (int t = 0; t < ntiles; ++t) {
                const int t0 = t * kT, tw = min(kT, w - t0), t1 = t0 + tw;
                if (warp == 0) {
                    double acc = 0.0;
                    if (lane < tw) {
                        const double *ti = tinv + t * kT * kT + lane * kT;
                        for (int j = 0; j < tw; ++j) acc += ti[j] * seg[t0 + j];
                    }
                    __syncwarp();
                    if (lane < tw) {
                        seg[t0 + lane] = acc;
                        tvec[lane] = acc;
                    } else if (lane < kT) {
                        tvec[lane] = 0.0;
                    }
                }
                __syncthreads();
                // trailing rows inside the panel: 4 lanes per row, 4 columns each
                const int nrows = w - t1;
                for (int rb = (tid >> 5) * 8; rb < nrows; rb += kSweepBlock / 4) {
                    const int r = rb + (lane >> 2);
                    double part = 0.0;
                    if (r < nrows) {
                        const double *pr = tp + r * kT + (lane & 3) * 4;
#pragma unroll
                        for (int c = 0; c < 4; ++c) part += pr[c] * tvec[(lane & 3) * 4 + c];
                    }
                    part += __shfl_xor_sync(0xffffffffu, part, 1);
                    part += __shfl_xor_sync(0xffffffffu, part, 2);
                    if ((lane & 3) == 0 && r < nrows) seg[t1 + r] -= part;
                }
                tp += nrows * kT;
                __syncthreads();
            }
            for (int k = tid; k < w; k += kSweepBlock) A.x[pstart + k] = seg[k];
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicExch(flag + p, 1);
            trace(D.d_trace_lower, iid, 2);
        } else {  // IT_OFF: contributions of panel p to below rows [r0, r1)
            if (tid == 0) spin_until_geq(flag + p, 1);
            __syncthreads();
            trace(D.d_trace_lower, iid, 1);
            for (int k = tid; k < w; k += kSweepBlock) seg[k] = __ldcg(A.x + pstart + k);
            __syncthreads();
            const double *P = D.d_pan + D.d_p_pan[p];
            double *cb = D.d_cbuf + D.d_p_cb[p];
            for (int j0 = it.r0 + warp * 2; j0 < it.r1; j0 += (kSweepBlock / 32) * 2) {
                const double *pa = P + (int64_t)j0 * w;
                const bool two = j0 + 1 < it.r1;
                double a0 = 0.0, a1 = 0.0;
                for (int c = lane; c < w; c += 32) {
                    const double s = seg[c];
                    a0 += __ldg(pa + c) * s;
                    if (two) a1 += __ldg(pa + w + c) * s;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                }
                if (lane == 0) {
                    cb[j0] = a0;
                    if (two) cb[j0 + 1] = a1;
                }
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                for (int q = 0; q < it.dep_cnt; ++q) atomicAdd(contrib + D.d_deps[it.dep_off + q], 1);
            }
            trace(D.d_trace_lower, iid, 2);
        }
    }
    sweep_exit(D, ctl, contrib, flag);
}

// ---------------------------------------------------------------------------
// upper sweep: L^T z = w
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSweepBlock)
upper_sweep(tsb_ldlt_desc D, SweepArgs A) {
    extern __shared__ __align__(128) double smem[];
    double *tri = smem;
    double *seg = smem + D.tri_smem_doubles;          // w doubles
    double *red = seg + kMaxW;                        // kSweepBlock doubles
    double *zb = red + kSweepBlock;                   // chunk rows of z[below]
    __shared__ uint64_t bar;
    __shared__ int item_id;
    __shared__ double tvec[kT];
    int32_t *ctl = D.d_ctl + 2;
    int32_t *ready = D.d_cnt2, *flag = D.d_cnt3;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (A.done != nullptr && *((volatile const int32_t *)A.done)) {
        sweep_exit(D, ctl, ready, flag);
        return;
    }
    if (tid == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    const Item *items = reinterpret_cast<const Item *>(D.d_items_upper);
    while (true) {
        if (tid == 0) item_id = atomicAdd(ctl, 1);
        __syncthreads();
        const int iid = item_id;
        if (iid >= D.n_items_upper) break;
        trace(D.d_trace_upper, iid, 0);
        const Item it = items[iid];
        const int p = it.panel;
        const int pstart = D.d_p_start[p], w = D.d_p_w[p];
        if (it.type == IT_OFFT) {
            // partial[c] = sum_{j in [r0,r1)} P[j][c] * z[below[j]]
            if (tid == 0) {
                for (int q = 0; q < it.dep_cnt; ++q) spin_until_geq(flag + D.d_deps[it.dep_off + q], 1);
            }
            __syncthreads();
            trace(D.d_trace_upper, iid, 1);
            const int32_t *below = D.d_below + D.d_p_below[p];
            for (int j = it.r0 + tid; j < it.r1; j += kSweepBlock) zb[j - it.r0] = __ldcg(A.x + below[j]);
            __syncthreads();
            const double *P = D.d_pan + D.d_p_pan[p];
            const int wp = w <= 16 ? 16 : (w <= 32 ? 32 : (w <= 64 ? 64 : 128));
            const int c = tid % wp, rg = tid / wp, ng = kSweepBlock / wp;
            double acc = 0.0;
            if (c < w) {
                int j = it.r0 + rg;
                for (; j + ng < it.r1; j += 2 * ng)
                    acc += __ldg(P + (int64_t)j * w + c) * zb[j - it.r0] +
                           __ldg(P + (int64_t)(j + ng) * w + c) * zb[j + ng - it.r0];
                if (j < it.r1) acc += __ldg(P + (int64_t)j * w + c) * zb[j - it.r0];
            }
            red[tid] = acc;
            __syncthreads();
            if (tid < w) {
                double s = 0.0;
                for (int g = 0; g < ng; ++g) s += red[g * wp + tid];
                D.d_part[it.out_off + tid] = s;
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(ready + p, 1);
            trace(D.d_trace_upper, iid, 2);
        } else {  // IT_DIAGT
            const int ntiles = (w + kT - 1) / kT;
            if (tid == 0) tma_load_1d(tri, D.d_tri + D.d_p_tri[p], (uint32_t)(D.d_p_tri_len[p] * 8), &bar);
            if (tid == 0) spin_until_geq(ready + p, it.dep_cnt);
            __syncthreads();
            trace(D.d_trace_upper, iid, 1);
            for (int k = tid; k < w; k += kSweepBlock) {
                double v = A.in[pstart + k];
                if (A.dscale) v = v / A.dscale[pstart + k];
                double s = 0.0;
                for (int q = 0; q < it.dep_cnt; ++q) s += __ldcg(D.d_part + it.out_off + q * w + k);
                seg[k] = v - s;
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            __syncthreads();
            const double *tinv = tri + D.d_p_tri_len[p] - ntiles * kT * kT;
            // offsets of the tile-column panels inside tri
            int64_t toff = 0;
            for (int t = 0; t < ntiles; ++t) toff += (int64_t)(w - min(t * kT + kT, w)) * kT;
            for (int t = ntiles - 1; t >= 0; --t) {
                const int t0 = t * kT, tw = min(kT, w - t0), t1 = t0 + tw;
                const int nrows = w - t1;
                toff -= (int64_t)nrows * kT;
                const double *tp = tri + toff;
                // acc_c = sum_{r < nrows} tp[r][c] * seg[t1 + r]   (16 row groups)
                {
                    const int cc = tid & (kT - 1), g = tid >> 4;
                    double a = 0.0;
                    for (int r = g; r < nrows; r += kSweepBlock / kT) a += tp[r * kT + cc] * seg[t1 + r];
                    red[tid] = a;
                }
                __syncthreads();
                if (warp == 0) {
                    double v = 0.0;
                    if (lane < tw) {
                        double a = 0.0;
                        for (int g = 0; g < kSweepBlock / kT; ++g) a += red[g * kT + lane];
                        v = seg[t0 + lane] - a;
                        tvec[lane] = v;
                    }
                    __syncwarp();
                    if (lane < tw) {
                        double z = 0.0;
                        const double *ti = tinv + t * kT * kT;
                        for (int q = 0; q < tw; ++q) z += ti[q * kT + lane] * tvec[q];
                        seg[t0 + lane] = z;
                    }
                }
                __syncthreads();
            }
            for (int k = tid; k < w; k += kSweepBlock) {
                const double v = seg[k];
                A.x[pstart + k] = v;
                if (A.out_perm) A.out[A.out_perm[pstart + k]] = v;
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicExch(flag + p, 1);
            trace(D.d_trace_upper, iid, 2);
        }
    }
    sweep_exit(D, ctl, ready, flag);
}

static uint64_t g_serial = 0;
static std::mutex g_serial_mu;

static size_t lower_smem(const tsb_ldlt_desc &D) { return (D.tri_smem_doubles + kMaxW) * sizeof(double); }
static size_t upper_smem(const tsb_ldlt_desc &D) {
    return (D.tri_smem_doubles + kMaxW + kSweepBlock + D.max_chunk_rows) * sizeof(double);
}

void ldlt_enqueue(tsb_ldlt_t h, int mode, const double *r, double *out, const int32_t *done,
                  cudaStream_t st) {
    // mode 0: lower (r permuted -> out permuted); 1: upper; 2: apply
    const tsb_ldlt_desc &D = h->d;
    if (D.n == 0) return;
    const int grid = D.grid;
    if (mode == 0 || mode == 2) {
        SweepArgs a{r, mode == 2 ? D.d_perm : nullptr, nullptr, mode == 2 ? D.d_y : out, nullptr, nullptr, done};
        lower_sweep<<<grid, kSweepBlock, lower_smem(D), st>>>(D, a);
        TSB_LAUNCHED();
    }
    if (mode == 1 || mode == 2) {
        SweepArgs a{mode == 2 ? D.d_y : r, nullptr, mode == 2 ? D.d_d : nullptr, mode == 2 ? D.d_y : out,
                    mode == 2 ? D.d_perm : nullptr, mode == 2 ? out : nullptr, done};
        upper_sweep<<<grid, kSweepBlock, upper_smem(D), st>>>(D, a);
        TSB_LAUNCHED();
    }
}

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
        const size_t ls = lower_smem(*desc), us = upper_smem(*desc);
        TSB_CUDA(cudaFuncSetAttribute(lower_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ls));
        TSB_CUDA(cudaFuncSetAttribute(upper_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)us));
        int per_sm_l = 0, per_sm_u = 0;
        TSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_l, lower_sweep, kSweepBlock, ls));
        TSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_u, upper_sweep, kSweepBlock, us));
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
