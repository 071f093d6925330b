// Persistent sweep bodies of the nested-dissection LDL^T apply, shared by the
// stand-alone sweep kernels (ldlt.cu) and the persistent PCG solver (pcg.cu).
// See ldlt.cu for the panel layout and the work-item protocol.
#pragma once

#include "tsb_common.cuh"

namespace tsb {

constexpr int kSweepBlock = 256;
constexpr int kT = 16;        // device tile parameter (ABI: panels start at multiples of it)
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
// one-thread TMA bulk copy global -> shared, completion on the mbarrier
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

// Optional per-item timeline (globaltimer ns): [take, ready, end, smid, staged, computed].
__device__ __forceinline__ void trace(int64_t *buf, int iid, int slot) {
    if (buf != nullptr && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        buf[(int64_t)iid * 8 + slot] = (int64_t)t;
        if (slot == 0) {
            uint32_t sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            buf[(int64_t)iid * 8 + 3] = sm;
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

// dynamic shared memory of the sweep bodies
inline size_t sweep_smem_lower(const tsb_ldlt_desc &D) {
    return (D.stage_doubles + 2 * kMaxW + kSweepBlock + (kMaxW + 2)) * sizeof(double) +
           ((D.max_chunk_rows + 1) & ~1) * sizeof(int32_t);
}
inline size_t sweep_smem_upper(const tsb_ldlt_desc &D) {
    return (D.stage_doubles + kMaxW + kSweepBlock + kMaxW + D.max_chunk_rows) * sizeof(double);
}

// ---------------------------------------------------------------------------
// Diagonal-panel GEMVs with the explicit inverse of the unit-lower triangle.
// The factor blocks are well conditioned (cond(L11) <= 3.4 on the beams); the
// panel-inverse sweeps agree with the tile-16 reference to ~6e-16.
// Both put one output per thread, two partial sums (column/row parity), so
// consecutive threads read consecutive shared-memory words.
// ---------------------------------------------------------------------------
// column-packed strict lower: column j holds rows j+1..w-1 at j*(2w-j-1)/2
__device__ __forceinline__ int col_off(int j, int w) { return (j * (2 * w - j - 1)) >> 1; }
// row-packed strict lower: row i holds columns 0..i-1 at i*(i-1)/2
__device__ __forceinline__ int row_off(int i) { return (i * (i - 1)) >> 1; }

// y = inv(L_pp) x   (lower sweep): thread per row i, columns j < i of one parity
__device__ __forceinline__ void panel_lower(const double *Lc, int w, const double *x, double *y, double *red,
                                            int tid) {
    const int i = tid & (kMaxW - 1), h = tid / kMaxW;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (i < w) {
        int j = h;
        for (; j + 6 < i; j += 8) {  // four independent chains hide the LDS latency
            a0 += Lc[col_off(j, w) + i - j - 1] * x[j];
            a1 += Lc[col_off(j + 2, w) + i - j - 3] * x[j + 2];
            a2 += Lc[col_off(j + 4, w) + i - j - 5] * x[j + 4];
            a3 += Lc[col_off(j + 6, w) + i - j - 7] * x[j + 6];
        }
        for (; j < i; j += 2) a0 += Lc[col_off(j, w) + i - j - 1] * x[j];
    }
    red[tid] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (tid < w) y[tid] = x[tid] + (red[tid] + red[tid + kMaxW]);
}

// z = inv(L_pp)^T v   (upper sweep): thread per column j, rows i > j of one parity
__device__ __forceinline__ void panel_upper(const double *Lr, int w, const double *v, double *z, double *red,
                                            int tid) {
    const int j = tid & (kMaxW - 1), h = tid / kMaxW;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (j < w) {
        int i = j + 1;
        if ((i & 1) != h) ++i;
        for (; i + 6 < w; i += 8) {
            a0 += Lr[row_off(i) + j] * v[i];
            a1 += Lr[row_off(i + 2) + j] * v[i + 2];
            a2 += Lr[row_off(i + 4) + j] * v[i + 4];
            a3 += Lr[row_off(i + 6) + j] * v[i + 6];
        }
        for (; i < w; i += 2) a0 += Lr[row_off(i) + j] * v[i];
    }
    red[tid] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (tid < w) z[tid] = v[tid] + (red[tid] + red[tid + kMaxW]);
}

// ---------------------------------------------------------------------------
// lower sweep: L y = r
// shared memory: [stage][seg 128][yv 128][red 256][row pointers 130 x int64][dst slots]
// ---------------------------------------------------------------------------
template <bool TRACE>
__device__ __forceinline__ void lower_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                            uint64_t &bar, uint32_t &phase) {
    double *stage = smem;                             // TMA staging: panel inverse or factor chunk
    double *seg = smem + D.stage_doubles;             // gathered panel rows
    double *yv = seg + kMaxW;                         // solved panel rows
    double *red = yv + kMaxW;                         // 256 partial sums
    int64_t *rptr = reinterpret_cast<int64_t *>(red + kSweepBlock);  // contribution row pointers
    int32_t *dsts = reinterpret_cast<int32_t *>(rptr + kMaxW + 2);   // chunk rows' cbuf slots
    __shared__ int item_id;
    int32_t *ctl = D.d_ctl;
    int32_t *contrib = D.d_cnt0, *flag = D.d_cnt1;
    int64_t *const tbuf = TRACE ? D.d_trace_lower : nullptr;  // folds away when off
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Item *items = reinterpret_cast<const Item *>(D.d_items_lower);
    while (true) {
        if (tid == 0) item_id = atomicAdd(ctl, 1);
        __syncthreads();
        const int iid = item_id;
        if (iid >= D.n_items_lower) break;
        trace(tbuf, iid, 0);
        const Item it = items[iid];
        const int p = it.panel;
        const int pstart = D.d_p_start[p], w = D.d_p_w[p];
        if (it.type == IT_DIAG) {
            // everything that does not depend on the contributions is fetched
            // before the wait: the panel inverse (TMA), row pointers, the input
            const int k = tid >> 1, h = tid & 1;
            double xin = 0.0;
            int64_t q0 = 0, q1 = 0;
            if (tid == 0) tma_load_1d(stage, D.d_tri + D.d_p_tri[p], (uint32_t)(D.d_p_tri_len[p] * 8), &bar);
            if (k < w) {
                const int row = pstart + k;
                q0 = __ldg(D.d_cin_ptr + row) + h;
                q1 = __ldg(D.d_cin_ptr + row + 1);
                if (h == 0) xin = __ldcg(A.in + (A.in_perm ? A.in_perm[row] : row));  // L2: may be produced in-kernel
            }
            if (tid == 0) spin_until_geq(contrib + p, it.dep_cnt);
            __syncthreads();
            trace(tbuf, iid, 1);
            // rows: input - contributions.  Two threads per row (w <= 128), each
            // summing every other contribution with its loads in flight, then one
            // xor step: a fixed summation order (deterministic)
            {
                double acc0 = 0.0, acc1 = 0.0;
                int64_t q = q0;
                for (; q + 2 < q1; q += 4) {
                    acc0 += __ldcg(D.d_cbuf + q);
                    acc1 += __ldcg(D.d_cbuf + q + 2);
                }
                if (q < q1) acc0 += __ldcg(D.d_cbuf + q);
                double acc = acc0 + acc1;
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                if (k < w && h == 0) seg[k] = xin - acc;
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            __syncthreads();
            trace(tbuf, iid, 4);
            panel_lower(stage, w, seg, yv, red, tid);
            __syncthreads();
            for (int k = tid; k < w; k += kSweepBlock) A.x[pstart + k] = yv[k];
            trace(tbuf, iid, 5);
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicExch(flag + p, 1);
            trace(tbuf, iid, 2);
        } else {  // IT_OFF: contributions of panel p to below rows [r0, r1)
            // the factor chunk does not depend on the sweep: stage it with TMA while
            // waiting for the panel's solution
            const int ws = w + (w & 1), nr = it.r1 - it.r0;
            if (tid == 0) {
                tma_load_1d(stage, D.d_pan + D.d_p_pan[p] + (int64_t)it.r0 * ws, (uint32_t)(nr * ws * 8), &bar);
                spin_until_geq(flag + p, 1);
            }
            const int32_t *slot = D.d_cslot + D.d_p_cb[p] + it.r0;
            for (int j = tid; j < nr; j += kSweepBlock) dsts[j] = __ldg(slot + j);
            __syncthreads();
            trace(tbuf, iid, 1);
            for (int k = tid; k < w; k += kSweepBlock) seg[k] = __ldcg(A.x + pstart + k);
            mbar_wait(&bar, phase);
            phase ^= 1;
            __syncthreads();
            trace(tbuf, iid, 4);
            // G lanes per below row (G = 32/16/8 for wide/medium/narrow panels),
            // two rows in flight per group, lanes over the panel columns; each
            // result goes to the row's contiguous contribution slot
            {
                const int G = w > 64 ? 32 : (w > 32 ? 16 : 8);
                const int gl = lane & (G - 1), gpw = 32 / G;
                // warp-uniform trip count: the xor shuffles need every lane
                for (int jb = warp * gpw * 2; jb < nr; jb += (kSweepBlock / 32) * gpw * 2) {
                    const int j = jb + (lane / G) * 2;
                    const bool one = j < nr, two = j + 1 < nr;
                    const double *pa = stage + j * ws;
                    double a0 = 0.0, a1 = 0.0;
                    for (int c = gl; c < w; c += G) {
                        const double s = seg[c];
                        if (one) a0 += pa[c] * s;
                        if (two) a1 += pa[ws + c] * s;
                    }
                    for (int o = G >> 1; o > 0; o >>= 1) {
                        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                    }
                    if (gl == 0 && one) {
                        D.d_cbuf[dsts[j]] = a0;
                        if (two) D.d_cbuf[dsts[j + 1]] = a1;
                    }
                }
            }
            trace(tbuf, iid, 5);
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                for (int q = 0; q < it.dep_cnt; ++q) atomicAdd(contrib + D.d_deps[it.dep_off + q], 1);
            }
            trace(tbuf, iid, 2);
        }
    }
    sweep_exit(D, ctl, contrib, flag);
}

// ---------------------------------------------------------------------------
// upper sweep: L^T z = w
// shared memory: [stage][seg 128][red 256][zv 128][zb max chunk rows]
// ---------------------------------------------------------------------------
template <bool TRACE>
__device__ __forceinline__ void upper_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                            uint64_t &bar, uint32_t &phase) {
    double *stage = smem;
    double *seg = smem + D.stage_doubles;
    double *red = seg + kMaxW;
    double *zv = red + kSweepBlock;
    double *zb = zv + kMaxW;
    __shared__ int item_id;
    int32_t *ctl = D.d_ctl + 2;
    int32_t *ready = D.d_cnt2, *flag = D.d_cnt3;
    int64_t *const tbuf = TRACE ? D.d_trace_upper : nullptr;
    const int tid = threadIdx.x;
    const Item *items = reinterpret_cast<const Item *>(D.d_items_upper);
    while (true) {
        if (tid == 0) item_id = atomicAdd(ctl, 1);
        __syncthreads();
        const int iid = item_id;
        if (iid >= D.n_items_upper) break;
        trace(tbuf, iid, 0);
        const Item it = items[iid];
        const int p = it.panel;
        const int pstart = D.d_p_start[p], w = D.d_p_w[p];
        if (it.type == IT_OFFT) {
            // partial[c] = sum_{j in [r0,r1)} P[j][c] * z[below[j]]; the factor chunk
            // is staged by TMA while the owners of its rows finish
            const int ws = w + (w & 1), nr = it.r1 - it.r0;
            if (tid == 0) {
                tma_load_1d(stage, D.d_pan + D.d_p_pan[p] + (int64_t)it.r0 * ws, (uint32_t)(nr * ws * 8), &bar);
                for (int q = 0; q < it.dep_cnt; ++q) spin_until_geq(flag + D.d_deps[it.dep_off + q], 1);
            }
            __syncthreads();
            trace(tbuf, iid, 1);
            const int32_t *below = D.d_below + D.d_p_below[p] + it.r0;
            for (int j = tid; j < nr; j += kSweepBlock) zb[j] = __ldcg(A.x + below[j]);
            mbar_wait(&bar, phase);
            phase ^= 1;
            __syncthreads();
            trace(tbuf, iid, 4);
            const int wp = w <= 16 ? 16 : (w <= 32 ? 32 : (w <= 64 ? 64 : 128));
            const int c = tid % wp, rg = tid / wp, ng = kSweepBlock / wp;
            double a0 = 0.0, a1 = 0.0;
            if (c < w) {
                int j = rg;
                for (; j + ng < nr; j += 2 * ng) {
                    a0 += stage[j * ws + c] * zb[j];
                    a1 += stage[(j + ng) * ws + c] * zb[j + ng];
                }
                if (j < nr) a0 += stage[j * ws + c] * zb[j];
            }
            red[tid] = a0 + a1;
            __syncthreads();
            if (tid < w) {
                double s = 0.0;
                for (int g = 0; g < ng; ++g) s += red[g * wp + tid];
                D.d_part[it.out_off + tid] = s;
            }
            trace(tbuf, iid, 5);
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(ready + p, 1);
            trace(tbuf, iid, 2);
        } else {  // IT_DIAGT
            const int k = tid >> 1, h = tid & 1;
            double vin = 0.0;
            if (tid == 0) tma_load_1d(stage, D.d_tri_u + D.d_p_tri[p], (uint32_t)(D.d_p_tri_len[p] * 8), &bar);
            if (k < w && h == 0) {  // input (and D scaling) does not depend on the wait
                vin = __ldcg(A.in + pstart + k);
                if (A.dscale) vin = vin / A.dscale[pstart + k];
            }
            if (tid == 0) spin_until_geq(ready + p, it.dep_cnt);
            __syncthreads();
            trace(tbuf, iid, 1);
            {
                // two threads per row sum the chunk partials of one parity (fixed order)
                double s0 = 0.0, s1 = 0.0;
                if (k < w) {
                    int q = h;
                    for (; q + 2 < it.dep_cnt; q += 4) {
                        s0 += __ldcg(D.d_part + it.out_off + q * w + k);
                        s1 += __ldcg(D.d_part + it.out_off + (q + 2) * w + k);
                    }
                    if (q < it.dep_cnt) s0 += __ldcg(D.d_part + it.out_off + q * w + k);
                }
                double s = s0 + s1;
                s += __shfl_xor_sync(0xffffffffu, s, 1);
                if (k < w && h == 0) seg[k] = vin - s;
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            __syncthreads();
            trace(tbuf, iid, 4);
            panel_upper(stage, w, seg, zv, red, tid);
            __syncthreads();
            for (int k = tid; k < w; k += kSweepBlock) {
                const double v = zv[k];
                A.x[pstart + k] = v;
                if (A.out_perm) A.out[A.out_perm[pstart + k]] = v;
            }
            trace(tbuf, iid, 5);
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicExch(flag + p, 1);
            trace(tbuf, iid, 2);
        }
    }
    sweep_exit(D, ctl, ready, flag);
}

}  // namespace tsb
