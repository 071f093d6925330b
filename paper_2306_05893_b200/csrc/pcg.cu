// Device-resident preconditioned conjugate gradient (krylov.pcg, krylov.py:120-158)
// as ONE persistent cooperative kernel per solve.
//
// Every CTA of a co-resident grid runs the whole solve; phases are separated
// by a software grid barrier:
//     P1  ap = A p with p = z + beta p_old fused into the bit-exact SpMV gather
//         (krylov.py:145, 156); p.ap block partials
//     P2  x += alpha p; r -= alpha ap; ||r||^2 (and z = r/diag, r.z for the
//         diagonal preconditioners) -> convergence test (krylov.py:147-153)
//     [LDL^T: the two persistent sweep bodies (ldlt_sweep.cuh) run by the same
//      CTAs, then r.z -> beta]
// Reductions: each CTA writes its block partial, and after the barrier EVERY
// CTA sums all partials in the same fixed order, so alpha/beta/the stop test
// are computed redundantly and identically everywhere -- no second barrier,
// no host round-trip, deterministic results for a given grid.  One report is
// read back per solve.  Vector updates round exactly like NumPy (no FMA
// contraction): x + (alpha*p), r - (alpha*ap), z + (beta*p), r * (1/diag).
#include <cuda_runtime.h>

#include <cstdlib>

#include "ldlt_sweep.cuh"
#include "spmv_exact.cuh"

namespace tsb {
const tsb_ldlt_desc &ldlt_desc(tsb_ldlt_t h);
}

namespace tsb {

struct PcgState {
    double res;
    long long it, zero_row;
    int32_t converged, status;
    long long phase_ns[6];  // CTA 0's time in: SpMV, barrier+alpha, update, barrier+beta, precond, total
};

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct PcgWork {
    int64_t n;
    double *r, *z, *ap, *p0, *p1, *invdiag;
    double *part;     // [4][kMaxGrid] block partials, one buffer per reduction kind
    unsigned *bar;    // grid barrier {arrivals, generation}
    PcgState *st;
    int32_t *status;  // [2] zero-diagonal status, first zero row
};

struct PcgArgs {
    const int32_t *rp;
    const int32_t *ci;
    const double *val;
    const double *b;
    const double *x0;
    const double *dinv;  // optional user 1/diag (Jacobi)
    double *x;
    double tol;
    long long max_it;
    int fuse_p;  // 1: p = z + beta p computed inside the SpMV gathers (small systems:
                 // one grid barrier less); 0: a separate pass (large systems: one gather)
};

constexpr int kPcgBlock = 256;
#ifndef TSB_LDLT_RPG
#define TSB_LDLT_RPG 2  // rows per 8-lane group in flight in the LDL^T kernel's SpMV (build-time A/B)
#endif
constexpr int64_t kFuseRows = 150000;
constexpr int kMaxGrid = kNumSM * 8;

// Sense-counting grid barrier (all CTAs co-resident: cooperative launch).
__device__ __forceinline__ void grid_sync(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// Block partial -> part[kind][cta]; returns nothing (thread 0 writes).
template <int NT>
__device__ __forceinline__ void put_partial(double v, double *part, int kind, double *red) {
    const double s = block_sum<NT>(v, red);
    if (threadIdx.x == 0) part[kind * kMaxGrid + blockIdx.x] = s;
}

// Sum of all CTAs' partials in a fixed order (identical in every CTA).
template <int NT>
__device__ __forceinline__ double all_partials(const double *part, int kind, double *red, double *bc) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) acc += __ldcg(part + kind * kMaxGrid + i);
    const double s = block_sum<NT>(acc, red);
    if (threadIdx.x == 0) *bc = s;
    __syncthreads();
    const double out = *bc;
    __syncthreads();
    return out;
}

// MINB = resident CTAs per SM the register budget is sized for: LDL^T 2
// (two 40 KB sweep stages per CTA in shared memory); Jacobi / identity 3 for small systems
// (grid-barrier bound), 6 for large ones (the SpMV is gather-latency bound)
// NT = threads per CTA: 256 with the sweep ring (the sweeps' warp roles); the
// large Jacobi / identity solve runs the same warps per SM in fewer, larger
// CTAs -- fewer arrivals per grid barrier, fewer partials per reduction.
template <int KIND, int MINB, int NT = kPcgBlock>
__global__ void __launch_bounds__(NT, MINB)
pcg_persistent(PcgWork W, PcgArgs a, tsb_ldlt_desc D) {
    extern __shared__ __align__(128) double smem[];  // sweep staging (LDL^T)
    __shared__ double red[32];
    __shared__ double bc;
    __shared__ SweepRing ring;
    const int tid = threadIdx.x;
    const int64_t n = W.n;
    const int64_t gtid = (int64_t)blockIdx.x * NT + tid, gstride = (int64_t)gridDim.x * NT;
    const int lane8 = tid & 7;
    const unsigned gmask = 0xffu << ((tid & 31) & 24);
    const int64_t grp = gtid >> 3, ngrp = gstride >> 3;
    if (KIND == TSB_PRECOND_LDLT) ring_init(ring);
    // ---- init (krylov.py:130-141) -------------------------------------------
    double bb = 0.0, rr = 0.0;
    for (int64_t i = gtid; i < n; i += gstride) {
        const double bi = a.b[i];
        bb += bi * bi;
        if (KIND == TSB_PRECOND_JACOBI) {
            double inv;
            if (a.dinv != nullptr) {
                inv = a.dinv[i];
            } else {
                double d = 0.0;
                const int lo = a.rp[i], hi = a.rp[i + 1];
                int l = lo, h = hi;
                while (l < h) {
                    const int mid = (l + h) >> 1;
                    if (a.ci[mid] < i) l = mid + 1; else h = mid;
                }
                if (l < hi && a.ci[l] == i) d = a.val[l];
                inv = 1.0 / d;
                if (d == 0.0) {
                    atomicMin(reinterpret_cast<unsigned long long *>(W.status + 2), (unsigned long long)i);
                    atomicExch(W.status, TSB_E_SOLVER);
                }
            }
            W.invdiag[i] = inv;
        }
        if (a.x0 == nullptr) {
            a.x[i] = 0.0;
            W.r[i] = bi;
            rr += bi * bi;
        } else {
            a.x[i] = a.x0[i];
        }
        W.p0[i] = 0.0;
    }
    if (a.x0 != nullptr) {  // r = b - A x0, bit-exact SpMV (krylov.py:135)
        XPlain xa{a.x0};
        for (int64_t row = grp; row < n; row += ngrp) {
            const int lo = a.rp[row], hi = a.rp[row + 1];
            const double s = row_sum_exact(lo, hi - lo, a.ci, a.val, xa, lane8, gmask);
            if (lane8 == 0) {
                const double ri = sub(a.b[row], s);
                W.r[row] = ri;
                rr += ri * ri;
            }
        }
    }
    put_partial<NT>(bb, W.part, 0, red);
    put_partial<NT>(rr, W.part, 1, red);
    grid_sync(W.bar);
    const double bnorm = sqrt(all_partials<NT>(W.part, 0, red, &bc));
    const double rr0 = all_partials<NT>(W.part, 1, red, &bc);
    const int32_t status = *((volatile int32_t *)W.status);
    long long it = 0;
    double res = 0.0;
    int converged = 0;
    bool done = false;
    if (status != 0) {
        done = true;
    } else if (bnorm == 0.0) {  // krylov.py:133-134: zero solution
        for (int64_t i = gtid; i < n; i += gstride) a.x[i] = 0.0;
        converged = 1;
        done = true;
    } else {
        res = sqrt(rr0) / bnorm;
        if (res <= a.tol) {
            converged = 1;
            done = true;
        } else if (a.max_it <= 0) {
            done = true;
        }
    }
    // preconditioner application z = M r and rz = r.z
    // LDL^T: r is gathered through perm once per apply into W.invdiag (unused by
    // this kind) before the lower sweep, so the sweep's items read it directly
    const bool pre_perm = KIND == TSB_PRECOND_LDLT && D.d_rin != nullptr;
    SweepArgs lo_args{pre_perm ? W.invdiag : W.r, pre_perm ? nullptr : D.d_perm, nullptr, D.d_y, nullptr, nullptr,
                      nullptr};
    auto permute_r = [&]() {
        if (!pre_perm) return;
        for (int64_t i = gtid; i < n; i += gstride) W.invdiag[i] = __ldcg(W.r + D.d_perm[i]);
        grid_sync(W.bar);
    };
    SweepArgs up_args{D.d_y, nullptr, D.d_d, D.d_x, D.d_perm, W.z, nullptr};
    double rz = 0.0, beta = 0.0;
    if (!done) {
        double v = 0.0;
        if (KIND == TSB_PRECOND_LDLT) {
            permute_r();
            lower_sweep_body<false>(D, lo_args, smem, ring);
            grid_sync(W.bar);
            upper_sweep_body<false>(D, up_args, smem, ring);
            grid_sync(W.bar);
            for (int64_t i = gtid; i < n; i += gstride) v += __ldcg(W.r + i) * __ldcg(W.z + i);
        } else {
            for (int64_t i = gtid; i < n; i += gstride) {
                const double ri = __ldcg(W.r + i);
                const double zi = KIND == TSB_PRECOND_JACOBI ? mul(ri, __ldcg(W.invdiag + i)) : ri;
                W.z[i] = zi;
                v += ri * zi;
            }
        }
        put_partial<NT>(v, W.part, 2, red);
        grid_sync(W.bar);
        rz = all_partials<NT>(W.part, 2, red, &bc);
    }
    // ---- iterations (krylov.py:144-157) --------------------------------------
    long long ph[6] = {0, 0, 0, 0, 0, 0};
    long long tl = gtimer();
    const long long t_loop = tl;
    auto lap = [&](int k) {  // CTA-0 phase clock (cheap: one timer read per phase)
        const long long t = gtimer();
        ph[k] += t - tl;
        tl = t;
    };
    // p = z + beta p (krylov.py:156): either fused into the SpMV gathers (every
    // reader rounds identically; the row owner stores it) or materialised once
    // per iteration by a separate pass (P3) so the SpMV gathers one vector
    double *pcur = W.p0, *pnxt = W.p1;
    if (!done && !a.fuse_p) {  // p = z for the first iteration (beta = 0, p0 = 0)
        for (int64_t i = gtid; i < n; i += gstride) pnxt[i] = add(__ldcg(W.z + i), mul(beta, __ldcg(pcur + i)));
        double *t = pcur;
        pcur = pnxt;
        pnxt = t;
        grid_sync(W.bar);
    }
    while (!done) {
        // P1: ap = A p (bit-exact row sums), p.ap block partials
        double v = 0.0;
        if (a.fuse_p) {
            XDirection xa{W.z, pcur, beta};
            for (int64_t row = grp; row < n; row += ngrp) {
                const int lo = a.rp[row], hi = a.rp[row + 1];
                const double s = row_sum_exact(lo, hi - lo, a.ci, a.val, xa, lane8, gmask);
                if (lane8 == 0) {
                    const double pr = xa((int)row);
                    pnxt[row] = pr;
                    W.ap[row] = s;
                    v += pr * s;
                }
            }
            double *t = pcur;  // the new direction is in pnxt
            pcur = pnxt;
            pnxt = t;
        } else if (KIND == TSB_PRECOND_LDLT) {
            // two CTAs per SM (the sweep staging): a third of the Jacobi kernel's
            // warps, so each 8-lane group keeps two rows' loads in flight
            XPlainCG xa{pcur};
            auto out = [&](int64_t row, double s) {
                W.ap[row] = s;
                v += __ldcg(pcur + row) * s;
            };
            rows_exact<TSB_LDLT_RPG>(grp, ngrp, n, a.rp, a.ci, a.val, xa, lane8, gmask, out);
        } else {
            XPlainCG xa{pcur};
            for (int64_t row = grp; row < n; row += ngrp) {
                const int lo = a.rp[row], hi = a.rp[row + 1];
                const double s = row_sum_exact(lo, hi - lo, a.ci, a.val, xa, lane8, gmask);
                if (lane8 == 0) {
                    W.ap[row] = s;
                    v += __ldcg(pcur + row) * s;
                }
            }
        }
        put_partial<NT>(v, W.part, 3, red);
        lap(0);
        grid_sync(W.bar);
        const double alpha = rz / all_partials<NT>(W.part, 3, red, &bc);
        lap(1);
        // P2: x, r updates, ||r||^2 (+ z, r.z for diagonal preconditioners)
        double vr = 0.0, vz = 0.0;
        for (int64_t i = gtid; i < n; i += gstride) {
            a.x[i] = add(__ldcg(a.x + i), mul(alpha, __ldcg(pcur + i)));
            const double ri = sub(__ldcg(W.r + i), mul(alpha, __ldcg(W.ap + i)));
            W.r[i] = ri;
            vr += ri * ri;
            if (KIND == TSB_PRECOND_JACOBI) {
                const double zi = mul(ri, __ldcg(W.invdiag + i));
                W.z[i] = zi;
                vz += ri * zi;
            } else if (KIND == TSB_PRECOND_IDENTITY) {
                W.z[i] = ri;
            }
        }
        put_partial<NT>(vr, W.part, 0, red);
        if (KIND == TSB_PRECOND_JACOBI) put_partial<NT>(vz, W.part, 1, red);
        lap(2);
        grid_sync(W.bar);
        const double rrn = all_partials<NT>(W.part, 0, red, &bc);
        lap(3);
        ++it;
        res = sqrt(rrn) / bnorm;
        if (res <= a.tol) {
            converged = 1;
            break;
        }
        if (it >= a.max_it) break;
        double rzn;
        if (KIND == TSB_PRECOND_IDENTITY) {
            rzn = rrn;
        } else if (KIND == TSB_PRECOND_JACOBI) {
            rzn = all_partials<NT>(W.part, 1, red, &bc);
        } else {
            permute_r();
            lower_sweep_body<false>(D, lo_args, smem, ring);
            grid_sync(W.bar);
            upper_sweep_body<false>(D, up_args, smem, ring);
            grid_sync(W.bar);
            double w2 = 0.0;
            for (int64_t i = gtid; i < n; i += gstride) w2 += __ldcg(W.r + i) * __ldcg(W.z + i);
            put_partial<NT>(w2, W.part, 2, red);
            grid_sync(W.bar);
            rzn = all_partials<NT>(W.part, 2, red, &bc);
        }
        beta = rzn / rz;
        rz = rzn;
        lap(4);
        if (!a.fuse_p) {  // P3: p = z + beta p, NumPy rounding
            for (int64_t i = gtid; i < n; i += gstride) pnxt[i] = add(__ldcg(W.z + i), mul(beta, __ldcg(pcur + i)));
            double *t = pcur;
            pcur = pnxt;
            pnxt = t;
            grid_sync(W.bar);
        }
    }
    ph[5] = gtimer() - t_loop;
    if (blockIdx.x == 0 && tid == 0) {
#pragma unroll
        for (int k = 0; k < 6; ++k) W.st->phase_ns[k] = ph[k];
        W.st->res = res;
        W.st->it = it;
        W.st->converged = converged;
        W.st->status = status;
        W.st->zero_row = status ? *reinterpret_cast<long long *>(W.status + 2) : -1;
    }
}

}  // namespace tsb

struct tsb_pcg {
    tsb::PcgWork W;
    void *mem = nullptr;
    tsb::PcgState *h_state = nullptr;  // pinned
    int grid[3] = {0, 0, 0};
    bool big = false;
    size_t smem_ldlt = 0;
};

namespace tsb {

template <int KIND, int MINB, int NT = kPcgBlock>
static int occupancy_grid(size_t smem) {
    auto k = pcg_persistent<KIND, MINB, NT>;
    allow_max_smem(k);
    int per_sm = 0, dev = 0, nsm = kNumSM;
    TSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, smem));
    TSB_CUDA(cudaGetDevice(&dev));
    TSB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm < 1) throw Error(TSB_E_ARG, "pcg kernel does not fit on an SM");
    // barrier cost grows with the CTA count, latency hiding with it: tunable
    int cap = MINB;
    if (const char *env = getenv("TSB_PCG_CTAS_PER_SM")) cap = atoi(env) > 0 ? atoi(env) : cap;
    if (per_sm > cap) per_sm = cap;
    const int g = per_sm * nsm;
    return g < kMaxGrid ? g : kMaxGrid;
}

template <int KIND, int MINB, int NT = kPcgBlock>
static void launch(tsb_pcg *h, PcgArgs &a, tsb_ldlt_desc &D, int grid, size_t smem, cudaStream_t s) {
    if (KIND == TSB_PRECOND_LDLT) sync_pub_direct();
    void *args[] = {&h->W, &a, &D};
    TSB_CUDA(cudaLaunchCooperativeKernel((const void *)pcg_persistent<KIND, MINB, NT>, dim3(grid), dim3(NT), args,
                                         smem, s));
    count_launch();
}

// Large Jacobi / identity solves: 48 warps per SM as 6 x 256, 3 x 512 or
// 2 x 768 threads (TSB_PCG_BIG_NT; the shape only changes barrier arrivals and
// the partials' count).
static int big_nt() {
    static int nt = 0;
    if (nt == 0) {
        const char *e = getenv("TSB_PCG_BIG_NT");
        const int v = e ? atoi(e) : 768;
        nt = (v == 256 || v == 512 || v == 768) ? v : 768;
    }
    return nt;
}
template <int KIND>
static int big_grid() {
    switch (big_nt()) {
        case 256: return occupancy_grid<KIND, 6, 256>(0);
        case 512: return occupancy_grid<KIND, 3, 512>(0);
        default: return occupancy_grid<KIND, 2, 768>(0);
    }
}
template <int KIND>
static void big_launch(tsb_pcg *h, PcgArgs &a, tsb_ldlt_desc &D, int grid, cudaStream_t s) {
    switch (big_nt()) {
        case 256: launch<KIND, 6, 256>(h, a, D, grid, 0, s); break;
        case 512: launch<KIND, 3, 512>(h, a, D, grid, 0, s); break;
        default: launch<KIND, 2, 768>(h, a, D, grid, 0, s); break;
    }
}

}  // namespace tsb

extern "C" int tsb_pcg_create(int64_t n, tsb_pcg_t *out) {
    using namespace tsb;
    return guard([&] {
        if (n < 0 || out == nullptr) throw Error(TSB_E_ARG, "bad n/out");
        auto *h = new tsb_pcg;
        const int64_t nn = n > 0 ? n : 1;
        size_t bytes = sizeof(double) * (6 * nn + 4 * kMaxGrid) + 4096;
        cudaError_t e = cudaMalloc(&h->mem, bytes);
        if (e != cudaSuccess) {
            delete h;
            check_cuda(e, "cudaMalloc(pcg workspace)");
        }
        char *p = static_cast<char *>(h->mem);
        auto take = [&](size_t b) {
            char *q = p;
            p += (b + 255) & ~size_t(255);
            return q;
        };
        PcgWork &W = h->W;
        W.n = n;
        W.r = reinterpret_cast<double *>(take(8 * nn));
        W.z = reinterpret_cast<double *>(take(8 * nn));
        W.ap = reinterpret_cast<double *>(take(8 * nn));
        W.p0 = reinterpret_cast<double *>(take(8 * nn));
        W.p1 = reinterpret_cast<double *>(take(8 * nn));
        W.invdiag = reinterpret_cast<double *>(take(8 * nn));
        W.part = reinterpret_cast<double *>(take(8 * 4 * kMaxGrid));
        W.bar = reinterpret_cast<unsigned *>(take(256));
        W.st = reinterpret_cast<PcgState *>(take(sizeof(PcgState)));
        W.status = reinterpret_cast<int32_t *>(take(256));
        TSB_CUDA(cudaMemset(W.bar, 0, 256));
        TSB_CUDA(cudaMallocHost(&h->h_state, sizeof(PcgState)));
        h->big = n >= kFuseRows;
        h->grid[TSB_PRECOND_IDENTITY] = h->big ? big_grid<TSB_PRECOND_IDENTITY>()
                                               : occupancy_grid<TSB_PRECOND_IDENTITY, 3>(0);
        h->grid[TSB_PRECOND_JACOBI] = h->big ? big_grid<TSB_PRECOND_JACOBI>()
                                             : occupancy_grid<TSB_PRECOND_JACOBI, 3>(0);
        *out = h;
    });
}

extern "C" int tsb_pcg_destroy(tsb_pcg_t h) {
    if (h == nullptr) return TSB_OK;
    cudaFree(h->mem);
    cudaFreeHost(h->h_state);
    delete h;
    return TSB_OK;
}

static void fill_report(const tsb::PcgState &s, tsb_report *r) {
    r->iterations = s.it;
    r->final_residual = s.res;
    r->converged = s.converged;
    r->status = s.status;
    r->zero_diag_row = s.zero_row;
}

extern "C" int tsb_pcg_report(tsb_pcg_t h, tsb_report *report, void *stream) {
    using namespace tsb;
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        TSB_CUDA(cudaMemcpyAsync(h->h_state, h->W.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        TSB_CUDA(cudaStreamSynchronize(s));
        fill_report(*h->h_state, report);
    });
}

extern "C" int tsb_pcg_solve(tsb_pcg_t h, int64_t nrows, const int32_t *d_row_ptr,
                             const int32_t *d_col_ind, const double *d_values, const double *d_b,
                             const double *d_x0, double *d_x, int32_t kind, tsb_ldlt_t ldlt,
                             const double *d_inv_diag, double tol, int64_t max_iterations,
                             tsb_report *report, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (h == nullptr) throw Error(TSB_E_ARG, "null pcg handle");
        if (nrows != h->W.n) throw Error(TSB_E_SOLVER, "pcg handle was created for a different size");
        if (kind < 0 || kind > 2) throw Error(TSB_E_ARG, "unknown preconditioner kind");
        if (kind == TSB_PRECOND_LDLT && ldlt == nullptr) throw Error(TSB_E_LIFECYCLE, "LDL^T factors not ready");
        cudaStream_t s = as_stream(stream);
        PcgWork &W = h->W;
        if (W.n == 0) {
            if (report != nullptr) *report = tsb_report{0, 0.0, 1, 0, -1};
            return;
        }
        // status word = 0, first zero row = all ones (atomicMin target) for this solve
        TSB_CUDA(cudaMemsetAsync(W.status, 0, 8, s));
        TSB_CUDA(cudaMemsetAsync(W.status + 2, 0xff, 8, s));
        // small systems are barrier-latency bound, large ones gather bound
        static const int fuse_env = getenv("TSB_PCG_FUSE_P") ? atoi(getenv("TSB_PCG_FUSE_P")) : -1;  // A/B switch
        const int fuse = fuse_env >= 0 ? fuse_env : (nrows < kFuseRows ? 1 : 0);
        PcgArgs a{d_row_ptr, d_col_ind, d_values, d_b, d_x0, d_inv_diag, d_x, tol, (long long)max_iterations, fuse};
        tsb_ldlt_desc D{};
        if (kind == TSB_PRECOND_LDLT) {
            D = ldlt_desc(ldlt);
            const size_t sm = sweep_smem_lower(D) > sweep_smem_upper(D) ? sweep_smem_lower(D) : sweep_smem_upper(D);
            if (sm != h->smem_ldlt || h->grid[TSB_PRECOND_LDLT] == 0) {
                h->grid[TSB_PRECOND_LDLT] = occupancy_grid<TSB_PRECOND_LDLT, 2>(sm);
                h->smem_ldlt = sm;
            }
            launch<TSB_PRECOND_LDLT, 2>(h, a, D, h->grid[TSB_PRECOND_LDLT], sm, s);
        } else if (kind == TSB_PRECOND_JACOBI) {
            if (h->big)
                big_launch<TSB_PRECOND_JACOBI>(h, a, D, h->grid[TSB_PRECOND_JACOBI], s);
            else
                launch<TSB_PRECOND_JACOBI, 3>(h, a, D, h->grid[TSB_PRECOND_JACOBI], 0, s);
        } else {
            if (h->big)
                big_launch<TSB_PRECOND_IDENTITY>(h, a, D, h->grid[TSB_PRECOND_IDENTITY], s);
            else
                launch<TSB_PRECOND_IDENTITY, 3>(h, a, D, h->grid[TSB_PRECOND_IDENTITY], 0, s);
        }
        if (report != nullptr) {
            TSB_CUDA(cudaMemcpyAsync(h->h_state, W.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
            TSB_CUDA(cudaStreamSynchronize(s));
            fill_report(*h->h_state, report);
        }
    });
}

// Diagnostics: CTA 0's per-phase device time of the last solve (ns):
// SpMV, barrier+alpha, vector update, barrier+beta, preconditioner, total loop.
extern "C" int tsb_pcg_phase_times(tsb_pcg_t h, int64_t *out6, void *stream) {
    using namespace tsb;
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        TSB_CUDA(cudaMemcpyAsync(h->h_state, h->W.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        TSB_CUDA(cudaStreamSynchronize(s));
        for (int k = 0; k < 6; ++k) out6[k] = h->h_state->phase_ns[k];
    });
}
