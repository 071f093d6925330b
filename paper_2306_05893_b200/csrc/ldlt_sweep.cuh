// Persistent sweep bodies of the nested-dissection LDL^T apply, shared by the
// stand-alone sweep kernels (ldlt.cu) and the persistent PCG solver (pcg.cu).
// Block-inverse layout and item protocol: include/tsb.h (tsb_ldlt_desc) and
// ldlt.cu.
#pragma once

#include "tsb_common.cuh"

namespace tsb {

constexpr int kSweepBlock = 256;
constexpr int kMaxV = 8192;         // largest m + na whose vector is staged in shared memory
constexpr int kMaxChunkRows = 512;  // rows of an item (host packer caps it)

struct Item {
    int32_t block, r0, r1, pad;
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
    if (bytes > 0)
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
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until_geq(const int *p, int target) {
    if (ld_acquire(p) >= target) return;
    int ns = 32;
    while (ld_acquire(p) < target) {
        __nanosleep(ns);
        if (ns < 128) ns <<= 1;
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

// Row r of G_b (lower; m = block size): triangle rows r < m hold r entries
// (padded to even), then the M rows with stride m rounded up to even.
__device__ __forceinline__ int64_t g_row_off(int r, int m) {
    if (r < m) return ((int64_t)r * r) >> 1;
    return (((int64_t)m * m) >> 1) + (int64_t)(r - m) * (m + (m & 1));
}
// Row c of G_b^T (upper; K = m + na - 1): v-entries [c+1, K+1), length K - c
// padded to even; offset = sum_{j=K-c+1..K} (j + (j & 1)).
__device__ __forceinline__ int64_t gt_row_off(int c, int K) {
    if (c <= 0) return 0;
    const int64_t a = (int64_t)K - c + 1;
    return ((K + a) * (K - a + 1)) / 2 + (((int64_t)K + 1) >> 1) - (a >> 1);
}

struct SweepArgs {
    const double *in;        // input vector (lower: r; upper: w)
    const int32_t *in_perm;  // lower apply: gather input through perm
    const double *dscale;    // upper apply: divide input by D
    double *x;               // lower: y (permuted)   upper: z (permuted)
    const int32_t *out_perm; // upper apply: scatter z through perm
    double *out;             // upper apply: output in original order
    const int32_t *done;     // stop flag (skip the sweep when set)
};

// Exit protocol: the last CTA out zeroes the counters for the next replay.
__device__ __forceinline__ void sweep_exit(int32_t *ctl, int32_t *c0, int64_t n0, int32_t *c1, int64_t n1) {
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ctl + 1, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    for (int64_t i = threadIdx.x; i < n0; i += blockDim.x) c0[i] = 0;
    for (int64_t i = threadIdx.x; i < n1; i += blockDim.x) c1[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        ctl[0] = 0;
        ctl[1] = 0;
        __threadfence();
    }
}

// dynamic shared memory of the sweep bodies
inline size_t sweep_smem_lower(const tsb_ldlt_desc &D) {
    return (size_t)(D.stage_doubles + ((D.max_m + 1) & ~1) + ((D.max_cb + 1) & ~1)) * sizeof(double) +
           (((D.max_m + 2) & ~1) + kMaxChunkRows) * sizeof(int32_t);
}
inline size_t sweep_smem_upper(const tsb_ldlt_desc &D) {
    return (size_t)(D.stage_doubles + ((D.max_v + 1) & ~1)) * sizeof(double);
}

// Sum of a row's contributions cb[a0, a1) in the fixed order every finaliser
// uses (even slots into c0, odd into c1, then c0 + c1).
template <bool GLOBAL>
__device__ __forceinline__ double contrib_sum(const double *cb, int64_t a0, int64_t a1) {
    double c0 = 0.0, c1 = 0.0;
    int64_t q = a0;
    for (; q + 1 < a1; q += 2) {
        c0 += GLOBAL ? __ldcg(cb + q) : cb[q];
        c1 += GLOBAL ? __ldcg(cb + q + 1) : cb[q + 1];
    }
    if (q < a1) c0 += GLOBAL ? __ldcg(cb + q) : cb[q];
    return c0 + c1;
}

// Cooperative coalesced copy global -> shared of n doubles, all loads in flight.
__device__ __forceinline__ void stage_copy(double *dst, const double *src, int n) {
    constexpr int U = 8;
    for (int k0 = threadIdx.x; k0 < n; k0 += U * kSweepBlock) {
        double t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * kSweepBlock;
            t[u] = k < n ? __ldcg(src + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * kSweepBlock;
            if (k < n) dst[k] = t[u];
        }
    }
}

// One warp: dot products of 8 staged rows with the shared vector v.  Row k
// holds the entries of v[lo_k, hi_k) at p_k.  Lanes stride v (each v[t] read
// once for the 8 rows), then a butterfly transpose-reduction (7 + 2 shuffles
// for 8 rows, fixed order).  Returns the row sum in the lanes with
// (lane & 3) == 0; *krow = which of the 8 rows.
__device__ __forceinline__ double rows8_dot(const double *const p[8], const int lo[8], const int hi[8],
                                            const double *v, int lane, int *krow) {
    int tmin = lo[0], tmax = hi[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        tmin = min(tmin, lo[k]);
        tmax = max(tmax, hi[k]);
    }
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
    for (int t = tmin + lane; t < tmax; t += 32) {
        const double vt = v[t];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (t >= lo[k] && t < hi[k]) acc[k] += p[k][t - lo[k]] * vt;
    }
    const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double send = b16 ? acc[k] : acc[k + 4];
        const double keep = b16 ? acc[k + 4] : acc[k];
        acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double send = b8 ? acc[k] : acc[k + 2];
        const double keep = b8 ? acc[k + 2] : acc[k];
        acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
        const double send = b4 ? acc[0] : acc[1];
        const double keep = b4 ? acc[1] : acc[0];
        acc[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    double r = acc[0];
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    *krow = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
    return r;
}

__device__ __forceinline__ double lower_input(const SweepArgs &A, int row) {
    return __ldcg(A.in + (A.in_perm ? A.in_perm[row] : row));  // may be produced in-kernel (L2)
}

// Strided per-thread loops with their global loads issued in batches of 4
// (the loads of one batch are independent; results land in shared memory).
// dst[j] = f(j) for j = tid, tid + 256, ... < n
template <class F>
__device__ __forceinline__ void batched(int n, F f) {
    constexpr int U = 4;
    for (int j0 = threadIdx.x; j0 < n; j0 += U * kSweepBlock) {
        double t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + u * kSweepBlock;
            if (j < n) t[u] = f.load(j);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + u * kSweepBlock;
            if (j < n) f.store(j, t[u]);
        }
    }
}

// ---------------------------------------------------------------------------
// lower sweep: L y = r   (column-major pre-accumulation, one GEMV per block)
//   item (b, rows [r0, r1) of G_b): stage the rows by TMA and the block's
//   input before the wait, form x_b = input - contributions, then
//       triangle row i:  y_i = x_i + sum_{j<i} Linv_ij x_j          -> x[start+i]
//       M row k:         c_k = sum_j M_kj x_j                        -> cbuf slot
//   and count the item on the parent; a mode-2 parent's contribution sums
//   are formed once by the item that completes it.
// shared memory: [stage][xs max_m][cbs max_cb][offs int32 max_m+2][dsts int32]
// ---------------------------------------------------------------------------
template <bool TRACE>
__device__ __forceinline__ void lower_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                                 uint64_t &bar, uint32_t &phase) {
    double *stage = smem;
    double *xs = smem + D.stage_doubles;
    double *cbs = xs + ((D.max_m + 1) & ~1);
    int32_t *offs = reinterpret_cast<int32_t *>(cbs + ((D.max_cb + 1) & ~1));
    int32_t *dsts = offs + ((D.max_m + 2) & ~1);
    __shared__ int item_id, fin_parent;
    int32_t *ctl = D.d_ctl;
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
        const tsb_ldlt_block B = D.d_blocks[it.block];
        const int m = B.m, s = B.start, nr = it.r1 - it.r0;
        const int64_t o0 = g_row_off(it.r0, m);
        // everything that does not depend on the sweep's progress is fetched
        // before the wait: the factor rows (TMA), the block's input, the slots
        if (tid == 0) tma_load_1d(stage, D.d_g + B.g_off + o0, (uint32_t)((g_row_off(it.r1, m) - o0) * 8), &bar);
        {
            struct In {
                const SweepArgs &A;
                double *xs;
                int s;
                __device__ double load(int j) const { return lower_input(A, s + j); }
                __device__ void store(int j, double v) const { xs[j] = v; }
            };
            batched(m, In{A, xs, s});
        }
        const int mr0 = max(it.r0, m);
        for (int j = mr0 + tid; j < it.r1; j += kSweepBlock) dsts[j - mr0] = __ldg(D.d_cslot + B.anc_off + (j - m));
        if (B.mode == 1)
            for (int j = tid; j <= m; j += kSweepBlock) offs[j] = (int32_t)(__ldg(D.d_cin_ptr + s + j) - B.cb_off);
        if (tid == 0) {
            if (B.mode == 1) spin_until_geq(D.d_cnt_l + it.block, B.target_l);
            else if (B.mode == 2) spin_until_geq(D.d_ready_l + it.block, 1);
        }
        __syncthreads();
        trace(tbuf, iid, 1);
        // x_b = input - (contributions of the descendants)
        if (B.mode == 1) {
            stage_copy(cbs, D.d_cbuf + B.cb_off, B.ncb);
            __syncthreads();
            for (int j = tid; j < m; j += kSweepBlock) xs[j] = xs[j] - contrib_sum<false>(cbs, offs[j], offs[j + 1]);
        } else if (B.mode == 2) {
            struct Sub {
                const double *src;
                double *xs;
                __device__ double load(int j) const { return __ldcg(src + j); }
                __device__ void store(int j, double v) const { xs[j] = xs[j] - v; }
            };
            batched(m, Sub{D.d_x + s, xs});
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        __syncthreads();
        trace(tbuf, iid, 4);
        for (int j0 = warp * 8; j0 < nr; j0 += 8 * (kSweepBlock / 32)) {  // warp-uniform trips
            const double *p[8];
            int lo[8], hi[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const bool ok = j0 + k < nr;
                const int r = it.r0 + (ok ? j0 + k : 0);
                lo[k] = 0;
                hi[k] = ok ? (r < m ? r : m) : 0;
                p[k] = stage + (g_row_off(r, m) - o0);
            }
            int k;
            const double a = rows8_dot(p, lo, hi, xs, lane, &k);
            const int j = j0 + k;
            if ((lane & 3) == 0 && j < nr) {
                const int r = it.r0 + j;
                if (r < m)
                    A.x[s + r] = xs[r] + a;
                else
                    D.d_cbuf[dsts[r - mr0]] = a;
            }
        }
        trace(tbuf, iid, 5);
        __syncthreads();
        if (tid == 0) {
            fin_parent = -1;
            if (B.parent >= 0) {
                __threadfence();
                const int old = atomicAdd(D.d_cnt_l + B.parent, 1);
                const tsb_ldlt_block &Pb = D.d_blocks[B.parent];
                if (Pb.mode == 2 && old == Pb.target_l - 1) {
                    __threadfence();
                    fin_parent = B.parent;
                }
            }
        }
        __syncthreads();
        if (fin_parent >= 0) {
            // Every child item is done: the parent's contribution sums, formed once
            // here (row-contiguous in cbuf; staged piece by piece with coalesced loads
            // together with the per-row offsets, one thread per row sums in order).
            const tsb_ldlt_block P = D.d_blocks[fin_parent];
            int32_t *fo = reinterpret_cast<int32_t *>(xs);  // free: this item's GEMV is done
            const int64_t qe = P.cb_off + P.ncb;
            int i0 = 0;
            while (i0 < P.m) {
                const int64_t qb = __ldg(D.d_cin_ptr + P.start + i0);
                int i1 = P.m;
                if (qe - qb > D.stage_doubles) {  // rows [i0, i1) whose contributions fit (>= 1 row)
                    int lo = i0 + 1, hi = P.m;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (__ldg(D.d_cin_ptr + P.start + mid) - qb <= D.stage_doubles) lo = mid; else hi = mid - 1;
                    }
                    i1 = lo;
                }
                const int cnt = (int)(__ldg(D.d_cin_ptr + P.start + i1) - qb);
                const bool staged = cnt <= D.stage_doubles;
                if (staged) stage_copy(stage, D.d_cbuf + qb, cnt);
                for (int i = i0 + tid; i <= i1; i += kSweepBlock)
                    fo[i - i0] = (int32_t)(__ldg(D.d_cin_ptr + P.start + i) - qb);
                __syncthreads();
                for (int i = i0 + tid; i < i1; i += kSweepBlock)
                    D.d_x[P.start + i] = staged ? contrib_sum<false>(stage, fo[i - i0], fo[i - i0 + 1])
                                                : contrib_sum<true>(D.d_cbuf + qb, fo[i - i0], fo[i - i0 + 1]);
                __syncthreads();
                i0 = i1;
            }
            if (tid == 0) {
                __threadfence();
                st_release(D.d_ready_l + fin_parent, 1);
            }
        }
        trace(tbuf, iid, 2);
    }
    sweep_exit(ctl, D.d_cnt_l, D.n_blocks, D.d_ready_l, D.n_blocks);
}

// ---------------------------------------------------------------------------
// upper sweep: L^T z = w   (row-major pull, one GEMV per block)
//   z_b = w_b + G_b^T v,  v = [w_b ; -z_anc]
//   item (b, rows [c0, c1) of G_b^T = columns of G_b): stage the rows by TMA
//   and w_b before the wait (only -z_anc depends on the parent), then
//   z_c = v_c + sum_{t > c} G^T[c][t] v_t for the item's columns.
// shared memory: [stage][v max_v]
// ---------------------------------------------------------------------------
template <bool TRACE>
__device__ __forceinline__ void upper_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                                 uint64_t &bar, uint32_t &phase) {
    double *stage = smem;
    double *v = smem + D.stage_doubles;
    __shared__ int item_id;
    int32_t *ctl = D.d_ctl + 2;
    int64_t *const tbuf = TRACE ? D.d_trace_upper : nullptr;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Item *items = reinterpret_cast<const Item *>(D.d_items_upper);
    while (true) {
        if (tid == 0) item_id = atomicAdd(ctl, 1);
        __syncthreads();
        const int iid = item_id;
        if (iid >= D.n_items_upper) break;
        trace(tbuf, iid, 0);
        const Item it = items[iid];
        const tsb_ldlt_block B = D.d_blocks[it.block];
        const int m = B.m, s = B.start, na = B.na, K = m + na - 1, nr = it.r1 - it.r0;
        const int64_t o0 = gt_row_off(it.r0, K);
        if (tid == 0) tma_load_1d(stage, D.d_gt + B.gt_off + o0, (uint32_t)((gt_row_off(it.r1, K) - o0) * 8), &bar);
        for (int t = it.r0 + tid; t < m; t += kSweepBlock) {  // w_b: produced before this sweep
            double w = __ldcg(A.in + s + t);
            if (A.dscale) w = w / A.dscale[s + t];
            v[t] = w;
        }
        for (int k = tid; k < na; k += kSweepBlock)  // ancestor rows, parked in v until the wait is over
            v[m + k] = __longlong_as_double((long long)__ldg(D.d_anc + B.anc_off + k));
        if (na > 0 && tid == 0) spin_until_geq(D.d_done_u + B.parent, D.d_blocks[B.parent].n_u);
        __syncthreads();
        trace(tbuf, iid, 1);
        {
            struct Anc {
                const double *x;
                double *va;
                __device__ double load(int k) const { return __ldcg(x + __double_as_longlong(va[k])); }
                __device__ void store(int k, double z) const { va[k] = -z; }
            };
            batched(na, Anc{A.x, v + m});
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        __syncthreads();
        trace(tbuf, iid, 4);
        for (int j0 = warp * 8; j0 < nr; j0 += 8 * (kSweepBlock / 32)) {
            const double *p[8];
            int lo[8], hi[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const bool ok = j0 + k < nr;
                const int c = it.r0 + (ok ? j0 + k : 0);
                lo[k] = c + 1;
                hi[k] = ok ? K + 1 : c + 1;
                p[k] = stage + (gt_row_off(c, K) - o0);
            }
            int k;
            const double a = rows8_dot(p, lo, hi, v, lane, &k);
            const int j = j0 + k;
            if ((lane & 3) == 0 && j < nr) {
                const int c = it.r0 + j;
                const double z = v[c] + a;
                A.x[s + c] = z;
                if (A.out_perm) A.out[A.out_perm[s + c]] = z;
            }
        }
        trace(tbuf, iid, 5);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(D.d_done_u + it.block, 1);
        }
        trace(tbuf, iid, 2);
    }
    sweep_exit(ctl, D.d_done_u, D.n_blocks, D.d_pad, 0);
}

}  // namespace tsb
