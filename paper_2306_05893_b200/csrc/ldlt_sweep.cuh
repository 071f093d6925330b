// Persistent sweep bodies of the nested-dissection LDL^T apply, shared by the
// stand-alone sweep kernels (ldlt.cu) and the persistent PCG solver (pcg.cu).
// Block-inverse layout and item protocol: include/tsb.h (tsb_ldlt_desc) and
// ldlt.cu.
#pragma once

#include "tsb_common.cuh"

namespace tsb {

constexpr int kSweepBlock = 256;
constexpr int kMaxSW = 32;      // upper-sweep column slab width (doubles)
constexpr int kMaxXs = 8192;    // largest block whose x_b is staged in shared memory
constexpr int kMaxChunkRows = 512;  // rows of a lower item (host packer caps it)

struct LItem {
    int32_t block, r0, r1, pad;
};
struct UItem {
    int32_t block, slab, ra, rb, tile, has_dep, p0, p1;
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

// Row r of G_b (m = block size): triangle rows r < m hold r entries (padded to
// even), then the M rows with stride m rounded up to even.  Every row offset
// is even (16-byte aligned).
__device__ __forceinline__ int64_t g_row_off(int r, int m) {
    if (r < m) return ((int64_t)r * r) >> 1;
    return (((int64_t)m * m) >> 1) + (int64_t)(r - m) * (m + (m & 1));
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
    return (size_t)(D.stage_doubles + ((D.max_m + 1) & ~1)) * sizeof(double) +
           (((D.max_m + 2) & ~1) + kMaxChunkRows) * sizeof(int32_t);
}
inline size_t sweep_smem_upper(const tsb_ldlt_desc &D) {
    return (size_t)(D.stage_doubles + ((D.max_tile_rows + 1) & ~1) + kSweepBlock) * sizeof(double) +
           ((D.max_tile_rows + 1) & ~1) * sizeof(int32_t);
}

// ---------------------------------------------------------------------------
// lower sweep: L y = r   (column-major pre-accumulation, one GEMV per block)
//   item (b, rows [r0, r1) of G_b):
//     stage the rows by TMA (before any wait), wait until x_b is final (the
//     last child item finalises it), stage x_b, then
//       triangle row i:  y_i = x_i + sum_{j<i} Linv_ij x_j          -> x[start+i]
//       M row k:         c_k = sum_j M_kj x_j                        -> cbuf slot
//     publish to the parent's counter; the item that completes the parent's
//     inputs finalises x_parent = in - (contributions, fixed order).
// shared memory: [stage][xs max_m]
// ---------------------------------------------------------------------------
__device__ __forceinline__ double lower_input(const SweepArgs &A, int row) {
    return __ldcg(A.in + (A.in_perm ? A.in_perm[row] : row));  // may be produced in-kernel (L2)
}

// Sum of the contributions cbuf[a0, a1) in the fixed order both finalisers use
// (even slots into c0, odd into c1, then c0 + c1); loads issued ahead.
__device__ __forceinline__ double contrib_sum(const double *cb, int64_t a0, int64_t a1) {
    double c0 = 0.0, c1 = 0.0;
    int64_t q = a0;
    for (; q + 3 < a1; q += 4) {
        const double t0 = __ldcg(cb + q), t1 = __ldcg(cb + q + 1), t2 = __ldcg(cb + q + 2), t3 = __ldcg(cb + q + 3);
        c0 += t0;
        c1 += t1;
        c0 += t2;
        c1 += t3;
    }
    for (; q + 1 < a1; q += 2) {
        c0 += __ldcg(cb + q);
        c1 += __ldcg(cb + q + 1);
    }
    if (q < a1) c0 += __ldcg(cb + q);
    return c0 + c1;
}

// One warp: dot products of 8 consecutive G rows [j0, j0+8) of the staged chunk
// with xs (lanes stride the columns, xs read once per 8 rows), then a butterfly
// transpose-reduction (7 + 2 shuffles for 8 rows, fixed order).  Returns the
// row sum in lanes with (lane & 3) == 0; *krow = which of the 8 rows.
__device__ __forceinline__ double rows8_dot(const double *stage, int64_t o0, int r0, int j0, int nr, int m,
                                            const double *xs, int lane, int *krow) {
    const double *rp[8];
    int len[8];
    int maxlen = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int j = j0 + k;
        const bool ok = j < nr;
        const int r = r0 + (ok ? j : 0);
        len[k] = ok ? (r < m ? r : m) : 0;
        rp[k] = stage + (g_row_off(r, m) - o0);
        maxlen = max(maxlen, len[k]);
    }
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
    for (int c = lane; c < maxlen; c += 32) {
        const double xc = xs[c];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (c < len[k]) acc[k] += rp[k][c] * xc;
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
    double v = acc[0];
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    *krow = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
    return v;
}

template <bool TRACE>
__device__ __forceinline__ void lower_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                                 uint64_t &bar, uint32_t &phase) {
    double *stage = smem;
    double *xs = smem + D.stage_doubles;
    int32_t *offs = reinterpret_cast<int32_t *>(xs + ((D.max_m + 1) & ~1));  // per-row contribution offsets
    int32_t *dsts = offs + ((D.max_m + 2) & ~1);                             // cbuf slots of the M rows
    __shared__ int item_id, fin_parent;
    __shared__ int64_t qbase;
    int32_t *ctl = D.d_ctl;
    int64_t *const tbuf = TRACE ? D.d_trace_lower : nullptr;  // folds away when off
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const LItem *items = reinterpret_cast<const LItem *>(D.d_items_lower);
    while (true) {
        if (tid == 0) item_id = atomicAdd(ctl, 1);
        __syncthreads();
        const int iid = item_id;
        if (iid >= D.n_items_lower) break;
        trace(tbuf, iid, 0);
        const LItem it = items[iid];
        const tsb_ldlt_block B = D.d_blocks[it.block];
        const int m = B.m, s = B.start, nr = it.r1 - it.r0;
        const int64_t o0 = g_row_off(it.r0, m);
        const double *gb = D.d_g + B.g_off;
        // everything that does not depend on the sweep's progress is fetched
        // before the wait: the factor rows (TMA), the block's input, the slots
        if (tid == 0) tma_load_1d(stage, gb + o0, (uint32_t)((g_row_off(it.r1, m) - o0) * 8), &bar);
        for (int j = tid; j < m; j += kSweepBlock) xs[j] = lower_input(A, s + j);
        const int mr0 = max(it.r0, m);
        for (int j = mr0 + tid; j < it.r1; j += kSweepBlock) dsts[j - mr0] = __ldg(D.d_cslot + B.anc_off + (j - m));
        if (B.mode == 1) {
            const int64_t q0 = __ldg(D.d_cin_ptr + s);
            for (int j = tid; j <= m; j += kSweepBlock) offs[j] = (int32_t)(__ldg(D.d_cin_ptr + s + j) - q0);
            if (tid == 0) qbase = q0;
        }
        if (tid == 0) {
            if (B.mode == 1) spin_until_geq(D.d_cnt_l + it.block, B.target_l);
            else if (B.mode == 2) spin_until_geq(D.d_ready_l + it.block, 1);
        }
        __syncthreads();
        trace(tbuf, iid, 1);
        // x_b = input - (contributions of the descendants)
        if (B.mode == 1) {
            const double *cb = D.d_cbuf + qbase;
            for (int j = tid; j < m; j += kSweepBlock) xs[j] = xs[j] - contrib_sum(cb, offs[j], offs[j + 1]);
        } else if (B.mode == 2) {
            for (int j = tid; j < m; j += kSweepBlock) xs[j] = xs[j] - __ldcg(D.d_x + s + j);
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        __syncthreads();
        trace(tbuf, iid, 4);
        for (int j0 = warp * 8; j0 < nr; j0 += 8 * (kSweepBlock / 32)) {  // warp-uniform trips
            int k;
            const double a = rows8_dot(stage, o0, it.r0, j0, nr, m, xs, lane, &k);
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
            // Every child item is done: S_parent = sum of its rows' contributions
            // (row-contiguous in cbuf).  Stage them piece by piece with coalesced
            // loads (all in flight at once) together with the per-row offsets,
            // then one thread per row sums its slots in order.
            const tsb_ldlt_block P = D.d_blocks[fin_parent];
            int32_t *fo = reinterpret_cast<int32_t *>(xs);  // free: this item's GEMV is done
            const int64_t qe = __ldg(D.d_cin_ptr + P.start + P.m);
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
                if (staged) {
                    constexpr int U = 8;
                    for (int k0 = tid; k0 < cnt; k0 += U * kSweepBlock) {
                        double t[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int k = k0 + u * kSweepBlock;
                            t[u] = k < cnt ? __ldcg(D.d_cbuf + qb + k) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int k = k0 + u * kSweepBlock;
                            if (k < cnt) stage[k] = t[u];
                        }
                    }
                }
                for (int i = i0 + tid; i <= i1; i += kSweepBlock)
                    fo[i - i0] = (int32_t)(__ldg(D.d_cin_ptr + P.start + i) - qb);
                __syncthreads();
                for (int i = i0 + tid; i < i1; i += kSweepBlock) {
                    const int a0 = fo[i - i0], a1 = fo[i - i0 + 1];
                    double c0 = 0.0, c1 = 0.0;
                    int q = a0;
                    if (staged) {
                        for (; q + 1 < a1; q += 2) {
                            c0 += stage[q];
                            c1 += stage[q + 1];
                        }
                        if (q < a1) c0 += stage[q];
                    } else {  // a single row with more contributions than the buffer
                        for (; q + 1 < a1; q += 2) {
                            c0 += __ldcg(D.d_cbuf + qb + q);
                            c1 += __ldcg(D.d_cbuf + qb + q + 1);
                        }
                        if (q < a1) c0 += __ldcg(D.d_cbuf + qb + q);
                    }
                    D.d_x[P.start + i] = c0 + c1;
                }
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
// upper sweep: L^T z = w   (row-major pull)
//   z_b = w_b + G_b^T v,  v = [w_b ; -z_anc]
//   item (b, slab, G rows [ra, rb)): partial sums of the slab's columns over
//   the tile rows (cp.async-staged before the wait; triangle-only tiles have
//   no dependency, M tiles wait for the parent's z); the last tile of a slab
//   adds the partials in tile order and publishes z for the slab's columns.
// shared memory: [stage tile_rows x sw][v max_tile_rows][red 256]
// ---------------------------------------------------------------------------
template <bool TRACE>
__device__ __forceinline__ void upper_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                                 uint64_t &bar, uint32_t &phase) {
    (void)bar;
    (void)phase;
    double *stage = smem;
    double *v = smem + D.stage_doubles;
    double *red = v + ((D.max_tile_rows + 1) & ~1);
    int32_t *ancs = reinterpret_cast<int32_t *>(red + kSweepBlock);
    __shared__ int item_id, last;
    int32_t *ctl = D.d_ctl + 2;
    int64_t *const tbuf = TRACE ? D.d_trace_upper : nullptr;
    const int tid = threadIdx.x;
    const UItem *items = reinterpret_cast<const UItem *>(D.d_items_upper);
    while (true) {
        if (tid == 0) item_id = atomicAdd(ctl, 1);
        __syncthreads();
        const int iid = item_id;
        if (iid >= D.n_items_upper) break;
        trace(tbuf, iid, 0);
        const UItem it = items[iid];
        const tsb_ldlt_block B = D.d_blocks[it.block];
        const int m = B.m, s = B.start, sw = B.sw, nr = it.rb - it.ra;
        const int c0 = (it.slab - B.slab_base) * sw;
        const int cw = min(sw, m - c0);
        const double *gb = D.d_g + B.g_off;
        // stage G[ra:rb, c0:c0+sw) (16-byte pieces; missing triangle entries -> 0)
        {
            const int pr = sw >> 1;
            for (int q = tid; q < nr * pr; q += kSweepBlock) {
                const int rr = q / pr, pc = (q - rr * pr) * 2;
                const int r = it.ra + rr, c = c0 + pc;
                double *dst = stage + rr * sw + pc;
                const int lim = r < m ? r : c0 + cw;  // triangle row r stores columns < r
                if (c < lim)
                    cp_async16(dst, gb + g_row_off(r, m) + c);
                else
                    dst[0] = dst[1] = 0.0;
            }
            cp_async_commit();
        }
        // the triangle rows' values and the M rows' ancestor indices do not
        // depend on the sweep: fetch them before the wait
        for (int j = tid; j < nr; j += kSweepBlock) {
            const int r = it.ra + j;
            if (r < m) {
                double vj = __ldcg(A.in + s + r);  // produced earlier in the same (persistent) kernel
                if (A.dscale) vj = vj / A.dscale[s + r];
                v[j] = vj;
            } else {
                ancs[j] = __ldg(D.d_anc + B.anc_off + (r - m));
            }
        }
        if (it.has_dep && tid == 0) spin_until_geq(D.d_done_u + B.parent, D.d_blocks[B.parent].nslabs);
        __syncthreads();
        trace(tbuf, iid, 1);
        if (it.has_dep)
            for (int j = tid; j < nr; j += kSweepBlock)
                if (it.ra + j >= m) v[j] = -__ldcg(A.x + ancs[j]);
        cp_async_wait_all();
        __syncthreads();
        trace(tbuf, iid, 4);
        {
            const int cc = tid % sw, g = tid / sw, ng = kSweepBlock / sw;
            double a0 = 0.0, a1 = 0.0;
            int j = g;
            for (; j + ng < nr; j += 2 * ng) {
                a0 += stage[j * sw + cc] * v[j];
                a1 += stage[(j + ng) * sw + cc] * v[j + ng];
            }
            if (j < nr) a0 += stage[j * sw + cc] * v[j];
            red[tid] = a0 + a1;
            __syncthreads();
            if (tid < cw) {
                double p = 0.0;
                for (int q = 0; q < ng; ++q) p += red[q * sw + tid];
                D.d_part[D.d_slab_part[it.slab] + (int64_t)it.tile * sw + tid] = p;
            }
        }
        trace(tbuf, iid, 5);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            last = atomicAdd(D.d_cnt_s + it.slab, 1) == D.d_slab_ntiles[it.slab] - 1;
            if (last) __threadfence();
        }
        __syncthreads();
        if (last) {  // all tiles of the slab are in: z = w + partials (tile order)
            if (tid < cw) {
                const int nt = D.d_slab_ntiles[it.slab];
                const double *pp = D.d_part + D.d_slab_part[it.slab] + tid;
                double acc = 0.0;
                for (int t = 0; t < nt; ++t) acc += __ldcg(pp + (int64_t)t * sw);
                const int row = s + c0 + tid;
                double w = __ldcg(A.in + row);
                if (A.dscale) w = w / A.dscale[row];
                const double z = w + acc;
                A.x[row] = z;
                if (A.out_perm) A.out[A.out_perm[row]] = z;
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(D.d_done_u + it.block, 1);
            }
        }
        trace(tbuf, iid, 2);
    }
    sweep_exit(ctl, D.d_cnt_s, D.n_slabs, D.d_done_u, D.n_blocks);
}

}  // namespace tsb
