// Persistent sweep bodies of the nested-dissection LDL^T apply, shared by the
// stand-alone sweep kernels (ldlt.cu) and the persistent PCG solver (pcg.cu).
// Tiled block-inverse layout and item protocol: include/tsb.h (tsb_ldlt_desc),
// ldlt.cu and paper_2306_05893_b200/_ldlt_pack.py.
//
// Warp roles inside a sweep (256-thread CTA):
//   warp 7 (producer, lane 0) takes the item tickets, posts each item id in a
//          two-entry mailbox and streams the item's factor data -- one TMA
//          bulk copy per small-tile group or per 40 KB column segment --
//          through a two-stage shared-memory ring, running up to two items /
//          two copies ahead of the consumers;
//   warps 0-6 (consumers, 224 threads, named barrier 1) stage each item's
//          vector window, wait for its dependency, form the block input,
//          run the GEMV out of the ring and publish.
// So the ticket atomic, the descriptor loads and the factor copies of the next
// item overlap the current item's dependency wait, input staging and math: the
// per-item latency chain no longer gates the HBM stream.  Consumers process
// their CTA's tickets in ticket order and every dependency points to an
// earlier ticket, so the persistent grid stays deadlock-free.
#pragma once

#include <cstdlib>

#include "tsb_common.cuh"

namespace tsb {

constexpr int kSweepBlock = 256;
constexpr int kWarps = 7;               // consumer warps
constexpr int kCThreads = kWarps * 32;  // consumer threads
constexpr int kProducerWarp = 7;
constexpr int kTile = 32;               // rows per tile (one per lane)
constexpr int kStage = 5120;            // doubles per ring stage (40 KB; 2 stages + vectors fit 2 CTAs/SM)
constexpr int kStages = 2;
constexpr int kSegPairs = 80;           // pairs per column segment of a large tile (40 KB)
constexpr int kMaxV = 8192;             // largest item window staged in shared memory
constexpr int kGroupsPerItem = 8;       // TMA groups (<= kWarps small tiles, <= 40 KB each) per small-tile item (max)
constexpr int kMailTiles = kGroupsPerItem * kWarps;
constexpr int kMaxItemRows = kMailTiles * kTile;

constexpr int kWhole = 1 << 20;  // Item.seg of a whole-tiles item (see below)

// seg = kWhole: whole large tiles [t0, t1), each one chunk (<= t1 - t0 <= kMailTiles
// tiles, their segments streamed one TMA each, every tile's rows emitted from the
// warp reduction -- no partial slots);
// seg = 0: small tiles [t0, t1), streamed as up to kGroupsPerItem TMA groups
// (greedy: <= kWarps tiles and <= 40 KB per group); seg = c + 1 (chunk item of a large
// tile): column segments [c*t1, min(c*t1 + t1, nsegs)) of tile t0, one TMA
// each (t1 = segments per chunk); seg < 0: finaliser of rows [t0, t1).
struct Item {
    int32_t block, t0, t1, seg;
};

// ---- small PTX helpers -----------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one-thread TMA bulk copy global -> shared, completion on the mbarrier
// (bytes == 0: the arrive alone completes the phase)
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
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
// barrier of the consumer warps only (the producer warp runs its own loop)
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(kCThreads) : "memory"); }
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Release / acquire-release counter updates: issued by consumer thread 0 after
// a csync(), they publish every write the consumers made before the barrier
// (bar.sync orders them before thread 0's release; release is cumulative).
__device__ __forceinline__ void red_add_release(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel(int *p, int v) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until_geq(const int *p, int target) {
    for (int k = 0; k < 16; ++k)
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

struct SweepArgs {
    const double *in;        // input vector (lower: r; upper: w)
    const int32_t *in_perm;  // lower apply: gather input through perm
    const double *dscale;    // upper apply: divide input by D
    double *x;               // lower: y (permuted)   upper: z (permuted)
    const int32_t *out_perm; // upper apply: scatter z through perm
    double *out;             // upper apply: output in original order
    const int32_t *done;     // stop flag (skip the sweep when set)
    const double *ext;       // lower: contributions from outside the handle's blocks (subtracted), or NULL
    // multi-RHS lower sweep (tsb_ldlt_lower_multi): nr right-hand sides, vector j
    // of in / x / d_x at j * ld, of the contributions at j * ld_cb, of the
    // chunk partial sums at j * ld_part
    int nr = 1;
    int64_t ld = 0, ld_cb = 0, ld_part = 0;
};

// Producer/consumer ring of one CTA (static shared memory of the kernel; its
// sequence counters persist across the sweeps of one launch, e.g. inside the
// persistent PCG).  TMA copy q uses stage q % 2 (barrier parity (q / 2) & 1);
// item k uses mailbox entry k % 2.
// A mailbox entry carries everything the consumers need about an item, loaded
// by the producer while the consumers work on the previous one: the item, its
// block, its tiles (small groups: up to kWarps; chunks: the tile) and its
// vector window.
struct MailEntry {
    int32_t iid, w0, w1, dep_target;
    const int32_t *dep;  // counter the item waits for (>= dep_target) or nullptr
    Item it;
    tsb_ldlt_block B;
    tsb_ldlt_tile T[kMailTiles];
};
// Publication queue: the consumers hand each finished item's counter update
// (a gpu-scope release of the item's outputs) to the producer lane, which
// issues it between its copies -- the release fence's round trip then costs
// the consumers nothing.  Entry j % 2 holds publication j (nullptr = the
// consumers left the sweep).
struct SweepRing {
    uint64_t full[kStages], empty[kStages];  // stage landed / stage read by the consumers
    uint64_t posted[2], taken[2];            // mailbox entry written / consumed
    uint64_t pub_full[2], pub_done[2];       // publication posted / issued
    MailEntry mail[2];
    int32_t *pub[2];
    uint32_t q_prod, k_prod, q_cons, k_cons, p_prod, p_cons;
};

__device__ __forceinline__ void ring_init(SweepRing &R) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < kStages; ++k) {
            mbar_init(&R.full[k], 1);
            mbar_init(&R.empty[k], 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&R.posted[k], 1);
            mbar_init(&R.taken[k], 1);
            mbar_init(&R.pub_full[k], 1);
            mbar_init(&R.pub_done[k], 1);
        }
        R.q_prod = R.k_prod = R.q_cons = R.k_cons = R.p_prod = R.p_cons = 0;
    }
    __syncthreads();
}

// Exit protocol: the last CTA out zeroes the counters for the next replay.
__device__ __forceinline__ void sweep_exit(int32_t *ctl, int32_t *c0, int64_t n0, int32_t *c1, int64_t n1,
                                           int32_t *c2, int64_t n2) {
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
    for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) c2[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        ctl[0] = 0;
        ctl[1] = 0;
        __threadfence();
    }
}
__device__ __forceinline__ void lower_exit(const tsb_ldlt_desc &D) {
    sweep_exit(D.d_ctl, D.d_cnt_l, D.n_blocks, D.d_ready_l, D.n_blocks, D.d_tcnt_lower, D.n_tiles_lower);
}
__device__ __forceinline__ void upper_exit(const tsb_ldlt_desc &D) {
    sweep_exit(D.d_ctl + 2, D.d_done_u, D.n_blocks, D.d_tcnt_upper, D.n_tiles_upper, D.d_pad, 0);
}

constexpr int kFinRows = 1024;          // rows per piece of a mode-2 finalisation

// dynamic shared memory of the sweep bodies (max_v = widest item window;
// nr right-hand sides stage nr windows)
inline size_t sweep_smem_lower(const tsb_ldlt_desc &D, int nr = 1) {
    const int offs = (D.max_v + 2 > kFinRows + 2 ? D.max_v + 2 : kFinRows + 2);
    return (size_t)(kStages * kStage + nr * ((D.max_v + 3) & ~1) + ((D.max_cb + 1) & ~1)) * sizeof(double) +
           (((offs + 1) & ~1) + kMaxItemRows) * sizeof(int32_t) +
           (nr > 1 ? (size_t)nr * kSweepBlock * sizeof(double) : 0);  // multi-RHS chunk partials
}
inline size_t sweep_smem_upper(const tsb_ldlt_desc &D) {
    return (size_t)(kStages * kStage + ((D.max_v + 3) & ~1)) * sizeof(double);
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

// Consumer-cooperative coalesced copy global -> shared of n doubles, all loads in flight.
__device__ __forceinline__ void stage_copy(double *dst, const double *src, int n) {
    constexpr int U = 8;
    for (int k0 = threadIdx.x; k0 < n; k0 += U * kCThreads) {
        double t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * kCThreads;
            t[u] = k < n ? __ldcg(src + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * kCThreads;
            if (k < n) dst[k] = t[u];
        }
    }
}

// Strided per-consumer-thread loops with their global loads issued in batches
// of 4 (the loads of one batch are independent; results land in shared memory).
// dst[j] = f(j) for j = tid, tid + 224, ... < n
// j = tid, tid + NT, ... < n with U loads in flight per thread (consumer
// threads [0, NT) take part)
template <class F, int NT = kCThreads>
__device__ __forceinline__ void batched(int n, F f) {
    constexpr int U = 4;
    if ((int)threadIdx.x >= NT) return;
    for (int j0 = threadIdx.x; j0 < n; j0 += U * NT) {
        double t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + u * NT;
            if (j < n) t[u] = f.load(j);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + u * NT;
            if (j < n) f.store(j, t[u]);
        }
    }
}

// One warp, one staged tile: lane k accumulates row k of the tile over the
// column pairs p = p0, p0 + ps, ... < p1 (pairs-major, 32 lanes x double2:
// 512 contiguous bytes per pair, conflict-free; v read as a broadcast
// double2).  Fixed summation order (deterministic).
__device__ __forceinline__ double tile_dot(const double *d, const double *v, int p0, int p1, int ps, int lane) {
    const double2 *g = reinterpret_cast<const double2 *>(d) + lane;
    const double2 *vv = reinterpret_cast<const double2 *>(v);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int p = p0;
    for (; p + ps < p1; p += 2 * ps) {
        const double2 g0 = g[p * kTile], g1 = g[(p + ps) * kTile];
        const double2 x0 = vv[p], x1 = vv[p + ps];
        a0 += g0.x * x0.x;
        a1 += g0.y * x0.y;
        a2 += g1.x * x1.x;
        a3 += g1.y * x1.y;
    }
    if (p < p1) {
        const double2 g0 = g[p * kTile], x0 = vv[p];
        a0 += g0.x * x0.x;
        a1 += g0.y * x0.y;
    }
    return (a0 + a1) + (a2 + a3);
}

// segments [s0, s1) of a chunk item's tile (see Item)
__device__ __forceinline__ void chunk_range(const Item &it, const tsb_ldlt_tile &T, int &s0, int &s1) {
    const int nsegs = (T.np + kSegPairs - 1) / kSegPairs;
    s0 = (it.seg - 1) * it.t1;
    s1 = min(s0 + it.t1, nsegs);
}

// end of the TMA group of a small-tile item that starts at tile g0 (of nt):
// the longest run of <= kWarps tiles whose data fit one stage
__device__ __forceinline__ int group_end(const tsb_ldlt_tile *T, int nt, int g0) {
    int g1 = g0, tot = 0;
    while (g1 < nt && g1 - g0 < kWarps) {
        const int b = T[g1].np * 2 * kTile;
        if (tot + b > kStage) break;
        tot += b;
        ++g1;
    }
    return g1 > g0 ? g1 : g0 + 1;
}

// v-columns [w0, w1) an item reads (lim = width of its vector: m or m + na);
// T = the item's tiles.
__device__ __forceinline__ bool is_chunk(const Item &it) { return it.seg > 0 && it.seg != kWhole; }
__device__ __forceinline__ void item_window(const Item &it, const tsb_ldlt_tile *T, int lim, int &w0, int &w1) {
    if (is_chunk(it)) {
        int s0, s1;
        chunk_range(it, T[0], s0, s1);
        w0 = T[0].tl + 2 * s0 * kSegPairs;
        w1 = min(T[0].tl + 2 * min(s1 * kSegPairs, T[0].np), lim);
    } else {
        w0 = T[0].tl;  // tiles are in row order: the first has the smallest tl
        int hi = 0;
        for (int t = 0; t < it.t1 - it.t0; ++t) hi = max(hi, T[t].tl + 2 * T[t].np);
        w1 = min(hi, lim);
    }
}

// ---- producer warp ---------------------------------------------------------
// Lane 0 of the producer warp: ticket -> mailbox -> the item's ring copies
// (one per small-tile group or chunk segment; a finaliser reserves one stage
// as scratch), until the ticket runs past the item list (that sentinel is
// posted too, so the consumers stop).
// Issue every publication the consumers have posted (in order); returns false
// once the consumers' end-of-sweep marker has been seen.
__device__ __forceinline__ bool serve_pubs(SweepRing &R, uint32_t &p) {
    while (true) {
        const int e = p & 1;
        if (!mbar_test(&R.pub_full[e], (p >> 1) & 1u)) return true;
        int32_t *addr = R.pub[e];
        if (addr != nullptr) red_add_release(addr, 1);
        mbar_arrive(&R.pub_done[e]);
        ++p;
        if (addr == nullptr) return false;
    }
}
// mbar_wait that keeps issuing publications meanwhile
__device__ __forceinline__ void wait_serving(SweepRing &R, uint64_t *bar, uint32_t phase, uint32_t &p, bool &live) {
    while (!mbar_test(bar, phase))
        if (live) live = serve_pubs(R, p);
}

__device__ __forceinline__ void sweep_producer(SweepRing &R, const tsb_ldlt_desc &D, int32_t *ticket,
                                               int64_t n_items, const Item *items, const tsb_ldlt_block *blocks,
                                               const tsb_ldlt_tile *tiles, const double *base, double *stage,
                                               bool upper) {
    if ((threadIdx.x & 31) != 0) return;
    uint32_t q = R.q_prod, k = R.k_prod, p = R.p_prod;
    bool live = true;
    while (true) {
        const int iid = atomicAdd(ticket, 1);
        const int e = k & 1;
        MailEntry &M = R.mail[e];
        Item it{0, 0, 0, 0};
        tsb_ldlt_tile T0{};
        if (iid < n_items) {  // descriptors: loaded while the entry may still be in use
            it = items[iid];
            const tsb_ldlt_block B = blocks[it.block];
            if (it.seg >= 0) T0 = tiles[it.t0];
            if (k >= 2) wait_serving(R, &R.taken[e], ((k >> 1) - 1) & 1u, p, live);
            M.it = it;
            M.B = B;
            if (is_chunk(it)) {
                M.T[0] = T0;
            } else if (it.seg >= 0) {  // small groups / whole tiles: every tile
                for (int t = it.t0; t < it.t1; ++t) M.T[t - it.t0] = t == it.t0 ? T0 : tiles[t];
            }
            if (it.seg >= 0) item_window(it, M.T, B.m + (upper ? B.na : 0), M.w0, M.w1);
            // the item's dependency (the counter its consumers would spin on)
            const int32_t *dep = nullptr;
            int32_t tgt = 0;
            if (upper) {  // -z_anc in the window: the parent's items (a parent outside the handle is solved before)
                if (B.parent >= 0 && M.w1 > B.m) {
                    dep = D.d_done_u + B.parent;
                    tgt = B.nu_parent;
                }
            } else if (it.seg < 0 || B.mode == 1) {  // finaliser / items summing contributions: the children
                dep = D.d_cnt_l + it.block;
                tgt = B.target_l;
            } else if (B.mode == 2) {  // x_b formed by the block's finalisers
                dep = D.d_ready_l + it.block;
                tgt = B.nfin;
            }
            M.dep = dep;
            M.dep_target = tgt;
        } else if (k >= 2) {
            wait_serving(R, &R.taken[e], ((k >> 1) - 1) & 1u, p, live);
        }
        M.iid = iid;
        mbar_arrive(&R.posted[e]);
        ++k;
        if (iid >= n_items) break;
        int s0 = 0, s1 = 1, g0 = 0;
        const int nt = it.t1 - it.t0;
        if (is_chunk(it)) chunk_range(it, T0, s0, s1);
        if (it.seg == kWhole) {  // every segment of every tile, in order
            for (int t = 0; t < nt; ++t) {
                const tsb_ldlt_tile &Tt = M.T[t];
                const int ns = (Tt.np + kSegPairs - 1) / kSegPairs;
                for (int sg = 0; sg < ns; ++sg, ++q) {
                    const int st = q % kStages;
                    if (q >= (uint32_t)kStages) wait_serving(R, &R.empty[st], ((q / kStages) - 1) & 1u, p, live);
                    const int p0 = sg * kSegPairs, cnt = min(kSegPairs, Tt.np - p0);
                    tma_load_1d(stage + st * kStage, base + Tt.off + (int64_t)p0 * (2 * kTile),
                                (uint32_t)(cnt * 2 * kTile * 8), &R.full[st]);
                }
            }
            continue;
        }
        for (int sg = s0; it.seg == 0 ? g0 < nt : sg < s1; ++sg, ++q) {
            const int st = q % kStages;
            if (q >= (uint32_t)kStages) wait_serving(R, &R.empty[st], ((q / kStages) - 1) & 1u, p, live);
            double *dst = stage + st * kStage;
            if (it.seg < 0) {
                tma_load_1d(dst, base, 0u, &R.full[st]);  // finaliser: the stage is its scratch
            } else if (it.seg == 0) {  // one group of small tiles
                const int g1 = group_end(M.T, nt, g0);
                const tsb_ldlt_tile &Tl = M.T[g1 - 1];
                const int64_t end = Tl.off + (int64_t)Tl.np * (2 * kTile);
                tma_load_1d(dst, base + M.T[g0].off, (uint32_t)((end - M.T[g0].off) * 8), &R.full[st]);
                g0 = g1;
            } else {
                const int p0 = sg * kSegPairs, cnt = min(kSegPairs, T0.np - p0);
                tma_load_1d(dst, base + T0.off + (int64_t)p0 * (2 * kTile), (uint32_t)(cnt * 2 * kTile * 8),
                            &R.full[st]);
            }
        }
    }
    while (live) live = serve_pubs(R, p);  // until the consumers leave the sweep
    R.q_prod = q;
    R.k_prod = k;
    R.p_prod = p;
}

// Consumers: the item's dependency (computed by the producer into the mailbox)
// is waited on by consumer thread kDepThread alone while the first kLoaders
// threads fetch the item's input window -- the acquire round trip overlaps
// those loads instead of following them.
constexpr int kDepThread = kCThreads - 32;  // lane 0 of the last consumer warp (a warp of its own:
constexpr int kLoaders = kCThreads - 32;    // its spin does not serialise a loading warp)
__device__ __forceinline__ void dep_spin(const MailEntry &M) {
    if (threadIdx.x == kDepThread && M.dep != nullptr) spin_until_geq(M.dep, M.dep_target);
}

// ---- consumer side ---------------------------------------------------------
// Next mailbox entry (all consumer threads); hand it back with mail_done()
// once the item is finished.
__device__ __forceinline__ const MailEntry &next_item(SweepRing &R, uint32_t k) {
    const int e = k & 1;
    mbar_wait(&R.posted[e], (k >> 1) & 1u);
    return R.mail[e];
}
__device__ __forceinline__ void mail_done(SweepRing &R, uint32_t &k) {  // after a csync()
    if (threadIdx.x == 0) mbar_arrive(&R.taken[k & 1]);
    ++k;
}
// Post a publication (consumer thread 0, after a csync()): the producer lane
// issues red.release.gpu(addr, 1); addr == nullptr ends the sweep's queue.
// tuning switch (TSB_PUB_DIRECT=1): the consumers issue their releases
// themselves instead of handing them to the producer lane; one copy per
// translation unit, set by sync_pub_direct() before its first sweep launch
static __device__ int g_pub_direct;
static inline void sync_pub_direct() {
    static bool done = false;
    if (done) return;
    const char *e = getenv("TSB_PUB_DIRECT");
    const int v = (e != nullptr && atoi(e) != 0) ? 1 : 0;
    cudaMemcpyToSymbol(g_pub_direct, &v, sizeof(int));
    done = true;
}

__device__ __forceinline__ void publish(SweepRing &R, uint32_t &p, int32_t *addr) {
    if (addr != nullptr && g_pub_direct) {
        if (threadIdx.x == 0) red_add_release(addr, 1);
        return;
    }
    if (threadIdx.x == 0) {
        const int e = p & 1;
        if (p >= 2) mbar_wait(&R.pub_done[e], ((p >> 1) - 1) & 1u);
        R.pub[e] = addr;
        mbar_arrive(&R.pub_full[e]);
    }
    ++p;
}
// Wait for ring copy q; returns its stage.
__device__ __forceinline__ double *ring_wait(SweepRing &R, uint32_t q, double *stage) {
    const int st = q % kStages;
    mbar_wait(&R.full[st], (q / kStages) & 1u);
    return stage + st * kStage;
}
// Hand ring copy q's stage back to the producer (after a csync()).
__device__ __forceinline__ void ring_release(SweepRing &R, uint32_t q) {
    if (threadIdx.x == 0) mbar_arrive(&R.empty[q % kStages]);
}

// GEMV of an item against the shared vector v (v[t] = column t).
// emit(row, value) once per tile row (block-relative row index).  A chunk
// item of a large tile consumes its segments from the ring in order, each
// consumer warp accumulating its share of every segment's pairs; the chunk's
// 32 partial sums go to the tile's scratch and the last chunk to finish adds
// them in chunk order and emits.  q = the item's first ring copy (advanced).
template <class Emit>
__device__ __forceinline__ void item_gemv(SweepRing &R, uint32_t &q, const Item &it, const tsb_ldlt_tile *tiles,
                                          double *stage, const double *v, double *red, double *part, int32_t *tcnt,
                                          const Emit &emit) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (it.seg == 0) {  // tiles = the item's tiles (mailbox), one ring copy per group, one warp per tile
        const int nt = it.t1 - it.t0;
        for (int g0 = 0; g0 < nt; ++q) {
            const int g1 = group_end(tiles, nt, g0);
            const double *sd = ring_wait(R, q, stage);
            const int64_t off0 = tiles[g0].off;
            if (g0 + warp < g1) {
                const tsb_ldlt_tile T = tiles[g0 + warp];
                const double a = tile_dot(sd + (T.off - off0), v + T.tl, 0, T.np, 1, lane);
                if (lane < T.nrows) emit(T.row0 + lane, a);
            }
            csync();
            ring_release(R, q);
            g0 = g1;
        }
        return;
    }
    if (it.seg == kWhole) {  // whole tiles, one after the other: segments split over the warps
        const int nt = it.t1 - it.t0;
        for (int t = 0; t < nt; ++t) {
            const tsb_ldlt_tile T = tiles[t];
            const int ns = (T.np + kSegPairs - 1) / kSegPairs;
            double acc = 0.0;
            for (int sg = 0; sg < ns; ++sg, ++q) {
                const double *sd = ring_wait(R, q, stage);
                const int p0 = sg * kSegPairs, cnt = min(kSegPairs, T.np - p0);
                acc += tile_dot(sd, v + T.tl + 2 * p0, warp, cnt, kWarps, lane);
                csync();
                ring_release(R, q);
            }
            red[warp * 32 + lane] = acc;
            csync();
            if (threadIdx.x < 32) {  // the sum a one-chunk item of the tile emits
                double a = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) a += red[w * 32 + threadIdx.x];
                if ((int)threadIdx.x < T.nrows) emit(T.row0 + threadIdx.x, 0.0 + a);
            }
        }
        return;
    }
    __shared__ int last_seg;
    const tsb_ldlt_tile T = tiles[0];
    int s0, s1;
    chunk_range(it, T, s0, s1);
    double acc = 0.0;
    for (int sg = s0; sg < s1; ++sg, ++q) {
        const double *sd = ring_wait(R, q, stage);
        const int p0 = sg * kSegPairs, cnt = min(kSegPairs, T.np - p0);
        acc += tile_dot(sd, v + T.tl + 2 * p0, warp, cnt, kWarps, lane);
        csync();  // every consumer warp is done with the stage
        ring_release(R, q);
    }
    red[warp * 32 + lane] = acc;
    csync();
    if (T.nseg == 1) {  // the whole tile in this item: emit without the partials' round trip
        if (threadIdx.x < 32) {
            double a = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) a += red[w * 32 + threadIdx.x];
            if ((int)threadIdx.x < T.nrows) emit(T.row0 + threadIdx.x, 0.0 + a);  // = the one-chunk sum below
        }
        return;
    }
    if (threadIdx.x < 32) {
        double a = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) a += red[w * 32 + threadIdx.x];
        part[((int64_t)T.part + it.seg - 1) * kTile + threadIdx.x] = a;
    }
    csync();
    if (threadIdx.x == 0) last_seg = atom_add_acq_rel(tcnt + it.t0, 1) == T.nseg - 1;
    csync();
    if (last_seg && threadIdx.x < 32) {
        double a = 0.0;
        for (int c = 0; c < T.nseg; ++c) a += __ldcg(part + ((int64_t)T.part + c) * kTile + threadIdx.x);
        if ((int)threadIdx.x < T.nrows) emit(T.row0 + threadIdx.x, a);
    }
}

__device__ __forceinline__ double lower_input(const SweepArgs &A, int row, int j = 0) {
    const double v = __ldcg(A.in + j * A.ld + (A.in_perm ? A.in_perm[row] : row));  // may be produced in-kernel (L2)
    return A.ext ? v - __ldcg(A.ext + row) : v;
}

// tile_dot for NR right-hand sides at once: every tile pair is read from
// shared memory once and applied to the NR vectors (v_j = v + j * vstride);
// per right-hand side the same four accumulators and summation order as
// tile_dot, so each result is bit-identical to a single-vector sweep.
template <int NR>
__device__ __forceinline__ void tile_dot_multi(const double *d, const double *v, int vstride, int p0, int p1, int ps,
                                               int lane, double *out) {
    const double2 *g = reinterpret_cast<const double2 *>(d) + lane;
    double a0[NR], a1[NR], a2[NR], a3[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) a0[j] = a1[j] = a2[j] = a3[j] = 0.0;
    int p = p0;
    for (; p + ps < p1; p += 2 * ps) {
        const double2 g0 = g[p * kTile], g1 = g[(p + ps) * kTile];
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const double2 *vv = reinterpret_cast<const double2 *>(v + j * vstride);
            const double2 x0 = vv[p], x1 = vv[p + ps];
            a0[j] += g0.x * x0.x;
            a1[j] += g0.y * x0.y;
            a2[j] += g1.x * x1.x;
            a3[j] += g1.y * x1.y;
        }
    }
    if (p < p1) {
        const double2 g0 = g[p * kTile];
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const double2 x0 = reinterpret_cast<const double2 *>(v + j * vstride)[p];
            a0[j] += g0.x * x0.x;
            a1[j] += g0.y * x0.y;
        }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) out[j] = (a0[j] + a1[j]) + (a2[j] + a3[j]);
}

// out[0..nr) for a runtime nr <= 8 (compile-time unrolled per width)
__device__ __forceinline__ void tile_dot_nr(int nr, const double *d, const double *v, int vstride, int p0, int p1,
                                            int ps, int lane, double *out) {
    switch (nr) {
        case 1: tile_dot_multi<1>(d, v, vstride, p0, p1, ps, lane, out); break;
        case 2: tile_dot_multi<2>(d, v, vstride, p0, p1, ps, lane, out); break;
        case 3: tile_dot_multi<3>(d, v, vstride, p0, p1, ps, lane, out); break;
        case 4: tile_dot_multi<4>(d, v, vstride, p0, p1, ps, lane, out); break;
        case 5: tile_dot_multi<5>(d, v, vstride, p0, p1, ps, lane, out); break;
        case 6: tile_dot_multi<6>(d, v, vstride, p0, p1, ps, lane, out); break;
        case 7: tile_dot_multi<7>(d, v, vstride, p0, p1, ps, lane, out); break;
        default: tile_dot_multi<8>(d, v, vstride, p0, p1, ps, lane, out); break;
    }
}

// item_gemv for nr <= 8 right-hand sides: each staged tile pair read once for
// all of them; chunk partials of all right-hand sides reduced after one
// barrier (red: [nr][7 warps][32]); emit(row, j, value).
template <class Emit>
__device__ __forceinline__ void item_gemv_multi(SweepRing &R, uint32_t &q, const Item &it, const tsb_ldlt_tile *tiles,
                                                double *stage, const double *v, int vstride, int nr, double *red,
                                                double *part, int64_t ld_part, int32_t *tcnt, const Emit &emit) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double out[8];
    if (it.seg == 0) {
        const int nt = it.t1 - it.t0;
        for (int g0 = 0; g0 < nt; ++q) {
            const int g1 = group_end(tiles, nt, g0);
            const double *sd = ring_wait(R, q, stage);
            const int64_t off0 = tiles[g0].off;
            if (g0 + warp < g1) {
                const tsb_ldlt_tile T = tiles[g0 + warp];
                tile_dot_nr(nr, sd + (T.off - off0), v + T.tl, vstride, 0, T.np, 1, lane, out);
                if (lane < T.nrows)
                    for (int j = 0; j < nr; ++j) emit(T.row0 + lane, j, out[j]);
            }
            csync();
            ring_release(R, q);
            g0 = g1;
        }
        return;
    }
    if (it.seg == kWhole) {  // as item_gemv
        const int nt = it.t1 - it.t0;
        for (int t = 0; t < nt; ++t) {
            const tsb_ldlt_tile T = tiles[t];
            const int ns = (T.np + kSegPairs - 1) / kSegPairs;
            double acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.0;
            for (int sg = 0; sg < ns; ++sg, ++q) {
                const double *sd = ring_wait(R, q, stage);
                const int p0 = sg * kSegPairs, cnt = min(kSegPairs, T.np - p0);
                tile_dot_nr(nr, sd, v + T.tl + 2 * p0, vstride, warp, cnt, kWarps, lane, out);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] += out[j];
                csync();
                ring_release(R, q);
            }
            for (int j = 0; j < nr; ++j) red[(j * kWarps + warp) * 32 + lane] = acc[j];
            csync();
            for (int idx = threadIdx.x; idx < 32 * nr; idx += kCThreads) {
                const int j = idx >> 5, l = idx & 31;
                double a = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) a += red[(j * kWarps + w) * 32 + l];
                if (l < T.nrows) emit(T.row0 + l, j, 0.0 + a);
            }
            csync();  // red is rewritten by the next tile
        }
        return;
    }
    __shared__ int last_seg_m;
    const tsb_ldlt_tile T = tiles[0];
    int s0, s1;
    chunk_range(it, T, s0, s1);
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    for (int sg = s0; sg < s1; ++sg, ++q) {
        const double *sd = ring_wait(R, q, stage);
        const int p0 = sg * kSegPairs, cnt = min(kSegPairs, T.np - p0);
        tile_dot_nr(nr, sd, v + T.tl + 2 * p0, vstride, warp, cnt, kWarps, lane, out);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += out[j];
        csync();
        ring_release(R, q);
    }
    for (int j = 0; j < nr; ++j) red[(j * kWarps + warp) * 32 + lane] = acc[j];
    csync();
    if (T.nseg == 1) {  // whole tile: emit directly (as item_gemv)
        for (int idx = threadIdx.x; idx < 32 * nr; idx += kCThreads) {
            const int j = idx >> 5, l = idx & 31;
            double a = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) a += red[(j * kWarps + w) * 32 + l];
            if (l < T.nrows) emit(T.row0 + l, j, 0.0 + a);
        }
        return;
    }
    for (int idx = threadIdx.x; idx < 32 * nr; idx += kCThreads) {
        const int j = idx >> 5, l = idx & 31;
        double a = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) a += red[(j * kWarps + w) * 32 + l];
        part[j * ld_part + ((int64_t)T.part + it.seg - 1) * kTile + l] = a;
    }
    csync();
    if (threadIdx.x == 0) last_seg_m = atom_add_acq_rel(tcnt + it.t0, 1) == T.nseg - 1;
    csync();
    if (last_seg_m && threadIdx.x < 32) {
        for (int j = 0; j < nr; ++j) {
            double a = 0.0;
            for (int c = 0; c < T.nseg; ++c) a += __ldcg(part + j * ld_part + ((int64_t)T.part + c) * kTile + threadIdx.x);
            if ((int)threadIdx.x < T.nrows) emit(T.row0 + threadIdx.x, j, a);
        }
    }
}

// ---------------------------------------------------------------------------
// lower sweep: L y = r   (column-major pre-accumulation, one GEMV per block)
//   item (b, tiles of G_b rows): stage the block's input window while the
//   item's tiles stream in, form x_b = input - contributions, then
//       triangle row i:  y_i = x_i + sum_{j<i} Linv_ij x_j          -> x[start+i]
//       M row k:         c_k = sum_j M_kj x_j                        -> cbuf slot
//   and count the item on the parent; a mode-2 parent's contribution sums
//   are formed once by its finaliser items.
// shared memory: [ring stages][xs max_v+2][cbs max_cb][offs int32][dsts int32]
// ---------------------------------------------------------------------------
template <bool TRACE, bool MULTI = false>
__device__ __forceinline__ void lower_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                                 SweepRing &R) {
    double *stage = smem;
    const Item *items = reinterpret_cast<const Item *>(D.d_items_lower);
    if ((threadIdx.x >> 5) == kProducerWarp) {
        sweep_producer(R, D, D.d_ctl, D.n_items_lower, items, D.d_blocks, D.d_tiles_lower, D.d_g, stage, false);
        lower_exit(D);
        return;
    }
    double *xs = smem + kStages * kStage;             // x_b over the item's window [w0, w1) (nr windows)
    const int nr = MULTI ? A.nr : 1, xstride = (D.max_v + 3) & ~1;
    double *cbs = xs + nr * xstride;
    int32_t *offs = reinterpret_cast<int32_t *>(cbs + ((D.max_cb + 1) & ~1));
    const int noffs = (D.max_v + 2 > kFinRows + 2 ? D.max_v + 2 : kFinRows + 2);
    int32_t *dsts = offs + ((noffs + 1) & ~1);
    double *redm = reinterpret_cast<double *>(dsts + kMaxItemRows);  // MULTI: [nr][7 warps][32] chunk partials
    __shared__ double red[kSweepBlock];
    int64_t *const tbuf = TRACE ? D.d_trace_lower : nullptr;  // folds away when off
    const int tid = threadIdx.x;
    uint32_t q = R.q_cons, k = R.k_cons, pc = R.p_cons;
    while (true) {
        const MailEntry &M = next_item(R, k);
        const int iid = M.iid;
        if (iid >= D.n_items_lower) {
            csync();
            mail_done(R, k);
            publish(R, pc, nullptr);  // end of this CTA's publications
            break;
        }
        trace(tbuf, iid, 0);
        const Item it = M.it;
        const tsb_ldlt_block B = M.B;
        const int m = B.m, s = B.start;
        if (it.seg < 0) {
            // finaliser item (mode 2): x_b = input - contributions for rows
            // [t0, t1), once the children are done; contributions staged piece
            // by piece in the item's ring stage, one thread per row sums in order
            double *scratch = ring_wait(R, q, stage);
            dep_spin(M);
            csync();
            trace(tbuf, iid, 1);
            int i0 = it.t0;
            while (i0 < it.t1) {
                const int64_t qb = __ldg(D.d_cin_ptr + s + i0);
                int i1 = min(it.t1, i0 + kFinRows);
                if (__ldg(D.d_cin_ptr + s + i1) - qb > kStage) {  // rows whose contributions fit (>= 1 row)
                    int lo = i0 + 1, hi = i1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (__ldg(D.d_cin_ptr + s + mid) - qb <= kStage) lo = mid; else hi = mid - 1;
                    }
                    i1 = lo;
                }
                const int cnt = (int)(__ldg(D.d_cin_ptr + s + i1) - qb);
                const bool staged = cnt <= kStage;
                for (int i = i0 + tid; i <= i1; i += kCThreads) offs[i - i0] = (int32_t)(__ldg(D.d_cin_ptr + s + i) - qb);
                for (int j = 0; j < nr; ++j) {  // right-hand side j (nr > 1: multi-RHS sweep)
                    const double *cbj = D.d_cbuf + j * A.ld_cb + qb;
                    if (staged) stage_copy(scratch, cbj, cnt);
                    csync();
                    for (int i = i0 + tid; i < i1; i += kCThreads)
                        D.d_x[j * A.ld + s + i] =
                            lower_input(A, s + i, j) -
                            (staged ? contrib_sum<false>(scratch, offs[i - i0], offs[i - i0 + 1])
                                    : contrib_sum<true>(cbj, offs[i - i0], offs[i - i0 + 1]));
                    csync();
                }
                i0 = i1;
            }
            ring_release(R, q);
            ++q;
            mail_done(R, k);
            publish(R, pc, D.d_ready_l + it.block);
            trace(tbuf, iid, 2);
            continue;
        }
        const int w0 = M.w0, w1 = M.w1;
        const int nw = w1 - w0;
        // everything that does not depend on the sweep's progress is fetched
        // before the wait: the window's input, the contribution slots (the
        // factor tiles are already streaming in through the ring)
        {
            struct In {
                const SweepArgs &A;
                double *xs;
                int s, r;
                __device__ double load(int j) const { return lower_input(A, s + j, r); }
                __device__ void store(int j, double v) const { xs[j] = v; }
            };
            dep_spin(M);  // the dependency thread, meanwhile the others fetch:
            if (B.mode != 2)  // mode 2: x_b comes from the finalisers
                for (int j = 0; j < nr; ++j) batched<In, kLoaders>(nw, In{A, xs + j * xstride, s + w0, j});
        }
        if (tid < nr) xs[tid * xstride + nw] = 0.0;  // column pad of odd-width tiles
        const tsb_ldlt_tile &Tf = M.T[0], &Tb = M.T[is_chunk(it) ? 0 : it.t1 - 1 - it.t0];
        const int r_hi = Tb.row0 + Tb.nrows, mr0 = max(Tf.row0, m);
        const int64_t cb0 = B.mode == 1 ? __ldg(D.d_cin_ptr + s + w0) : 0;
        if (tid < kLoaders) {
            for (int j = mr0 + tid; j < r_hi; j += kLoaders) dsts[j - mr0] = __ldg(D.d_cslot + B.anc_off + (j - m));
            if (B.mode == 1)
                for (int j = tid; j <= nw; j += kLoaders) offs[j] = (int32_t)(__ldg(D.d_cin_ptr + s + w0 + j) - cb0);
        }
        csync();  // dependency met; the window's staged input / offsets / destinations
        trace(tbuf, iid, 1);
        // x_b = input - (contributions of the descendants) over the window
        if (B.mode == 1) {  // rows in pieces whose contributions fit the buffer, per right-hand side
            for (int j = 0; j < nr; ++j) {
                double *xj = xs + j * xstride;
                const double *cbj = D.d_cbuf + j * A.ld_cb + cb0;
                int i0 = 0;
                while (i0 < nw) {
                    int i1 = nw;
                    if (offs[nw] - offs[i0] > D.max_cb) {
                        int lo = i0 + 1, hi = nw;
                        while (lo < hi) {
                            const int mid = (lo + hi + 1) >> 1;
                            if (offs[mid] - offs[i0] <= D.max_cb) lo = mid; else hi = mid - 1;
                        }
                        i1 = lo;
                    }
                    const int base = offs[i0], cnt = offs[i1] - base;
                    const bool fits = cnt <= D.max_cb;
                    if (fits) stage_copy(cbs, cbj + base, cnt);
                    csync();
                    for (int jj = i0 + tid; jj < i1; jj += kCThreads)
                        xj[jj] = xj[jj] - (fits ? contrib_sum<false>(cbs, offs[jj] - base, offs[jj + 1] - base)
                                                : contrib_sum<true>(cbj, offs[jj], offs[jj + 1]));
                    csync();
                    i0 = i1;
                }
            }
        } else if (B.mode == 2) {  // formed by the block's finaliser items
            struct Ld {
                const double *src;
                double *xs;
                __device__ double load(int j) const { return __ldcg(src + j); }
                __device__ void store(int j, double v) const { xs[j] = v; }
            };
            for (int j = 0; j < nr; ++j) batched(nw, Ld{D.d_x + j * A.ld + s + w0, xs + j * xstride});
        }
        csync();
        trace(tbuf, iid, 4);
        if (!MULTI) {
            auto emit = [&](int r, double a) {
                if (r < m)
                    A.x[s + r] = a;  // unit diagonal stored: y_r = sum_{j <= r} Linv_rj x_j
                else
                    D.d_cbuf[dsts[r - mr0]] = a;
            };
            item_gemv(R, q, it, M.T, stage, xs - w0, red, D.d_part_lower, D.d_tcnt_lower, emit);
        } else {
            auto emit = [&](int r, int j, double a) {
                if (r < m)
                    A.x[j * A.ld + s + r] = a;
                else
                    D.d_cbuf[j * A.ld_cb + dsts[r - mr0]] = a;
            };
            item_gemv_multi(R, q, it, M.T, stage, xs - w0, xstride, nr, redm, D.d_part_lower, A.ld_part,
                            D.d_tcnt_lower, emit);
        }
        trace(tbuf, iid, 5);
        csync();
        mail_done(R, k);
        if (B.parent >= 0) publish(R, pc, D.d_cnt_l + B.parent);
        trace(tbuf, iid, 2);
    }
    if (tid == 0) {
        R.q_cons = q;
        R.k_cons = k;
        R.p_cons = pc;
    }
    lower_exit(D);
}

// ---------------------------------------------------------------------------
// upper sweep: L^T z = w   (row-major pull, one GEMV per block)
//   z_b = w_b + G_b^T v,  v = [w_b ; -z_anc]
//   item (b, tiles of G_b^T rows = columns of G_b): w_b is staged before the
//   wait (only -z_anc depends on the parent), the tiles stream through the
//   ring, then z_c = v_c + sum_{t > c} G^T[c][t] v_t for the item's columns.
// shared memory: [ring stages][v max_v+2]
// ---------------------------------------------------------------------------
template <bool TRACE>
__device__ __forceinline__ void upper_sweep_body(const tsb_ldlt_desc &D, const SweepArgs &A, double *smem,
                                                 SweepRing &R) {
    double *stage = smem;
    const Item *items = reinterpret_cast<const Item *>(D.d_items_upper);
    if ((threadIdx.x >> 5) == kProducerWarp) {
        sweep_producer(R, D, D.d_ctl + 2, D.n_items_upper, items, D.d_blocks, D.d_tiles_upper, D.d_gt, stage, true);
        upper_exit(D);
        return;
    }
    double *v = smem + kStages * kStage;  // [w_b; -z_anc] over the item's window [w0, w1)
    __shared__ double red[kSweepBlock];
    int64_t *const tbuf = TRACE ? D.d_trace_upper : nullptr;
    const int tid = threadIdx.x;
    uint32_t q = R.q_cons, k = R.k_cons, pc = R.p_cons;
    while (true) {
        const MailEntry &M = next_item(R, k);
        const int iid = M.iid;
        if (iid >= D.n_items_upper) {
            csync();
            mail_done(R, k);
            publish(R, pc, nullptr);  // end of this CTA's publications
            break;
        }
        trace(tbuf, iid, 0);
        const Item it = M.it;
        const tsb_ldlt_block B = M.B;
        const int m = B.m, s = B.start;
        const int w0 = M.w0, w1 = M.w1;
        const int nw = w1 - w0;
        dep_spin(M);  // -z_anc in the window: the parent's items; meanwhile the others fetch:
        const int k0 = max(w0, m) - m, k1 = w1 - m;  // ancestor entries in the window
        if (tid < kLoaders) {
            for (int t = w0 + tid; t < min(w1, m); t += kLoaders) {  // w_b: produced before this sweep
                double w = __ldcg(A.in + s + t);
                if (A.dscale) w = w / A.dscale[s + t];
                v[t - w0] = w;
            }
            for (int kk = k0 + tid; kk < k1; kk += kLoaders)  // rows parked in v until the wait is over
                v[m + kk - w0] = __longlong_as_double((long long)__ldg(D.d_anc + B.anc_off + kk));
        }
        if (tid == 0) v[nw] = 0.0;  // column pad of odd-width tiles
        csync();
        trace(tbuf, iid, 1);
        if (k1 > k0) {
            struct Anc {
                const double *x;
                double *va;
                __device__ double load(int j) const { return __ldcg(x + __double_as_longlong(va[j])); }
                __device__ void store(int j, double z) const { va[j] = -z; }
            };
            batched(k1 - k0, Anc{A.x, v + (m + k0 - w0)});
        }
        csync();
        trace(tbuf, iid, 4);
        {
            auto emit = [&](int c, double z) {  // unit diagonal stored: z_c = sum_{t >= c} G^T[c][t] v_t
                A.x[s + c] = z;
                if (A.out_perm) A.out[A.out_perm[s + c]] = z;
            };
            item_gemv(R, q, it, M.T, stage, v - w0, red, D.d_part_upper, D.d_tcnt_upper, emit);
        }
        trace(tbuf, iid, 5);
        csync();
        mail_done(R, k);
        publish(R, pc, D.d_done_u + it.block);
        trace(tbuf, iid, 2);
    }
    if (tid == 0) {
        R.q_cons = q;
        R.k_cons = k;
        R.p_cons = pc;
    }
    upper_exit(D);
}

}  // namespace tsb
