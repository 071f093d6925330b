// Device-resident preconditioned conjugate gradient (krylov.pcg, krylov.py:120-158).
//
// The whole iteration loop is one CUDA graph: a conditional WHILE node whose
// body is
//     K1  ap = A p  with p = z + beta p_old fused into the SpMV gather
//         (krylov.py:145, 156), p.ap partial sums -> alpha   (last CTA)
//     K2  x += alpha p; r -= alpha ap; ||r||^2 (and z = r/diag, r.z for the
//         diagonal preconditioners) -> convergence test, beta (last CTA)
//     [LDL^T: level kernels of the apply, then K3: r.z -> beta]
// alpha, beta, the residual and the stop flag never leave the device; the
// last CTA of K2/K3 sets the WHILE condition with cudaGraphSetConditional.
// One report is read back per solve.  Every vector operation rounds exactly
// like the NumPy reference (no FMA contraction): x + (alpha*p), r - (alpha*ap),
// z + (beta*p), r * (1/diag); the SpMV is bit-identical to krylov.spmv.  Only
// the three dot products differ in summation order from BLAS, deterministically.
#include <cuda_runtime.h>

#include <map>
#include <vector>

#include "spmv_exact.cuh"

namespace tsb {
void ldlt_enqueue(tsb_ldlt_t h, int mode, const double *r, double *out, const int32_t *done,
                  cudaStream_t st);
uint64_t ldlt_serial(tsb_ldlt_t h);
int spmv_grid(int64_t nrows);
void launch_csr_diag(int64_t nrows, int64_t ncols, const int32_t *rp, const int32_t *ci,
                     const double *val, double *d, cudaStream_t s);
}  // namespace tsb

namespace tsb {

struct PcgState {
    double bnorm, rz, alpha, beta, res, tol;
    long long it, max_it, zero_row;
    int32_t done, converged, status, pad;
};

struct PcgArgs {
    const int32_t *rp;
    const int32_t *ci;
    const double *val;
    const double *b;
    const double *x0;
    double *x;
};

struct PcgBufs {
    int64_t n;
    double *r, *z, *ap, *p0, *p1, *invdiag, *partials;
    unsigned *counter;
    PcgState *st;
    PcgArgs *args;
};

constexpr int kVecBlock = 256;
constexpr int kSpBlock = 256;  // 8 lanes per row, 32 rows per CTA

int vec_grid(int64_t n) {
    int64_t g = (n + kVecBlock - 1) / kVecBlock;
    int64_t cap = (int64_t)kNumSM * 4;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// Grid-wide deterministic sum of K values per thread; returns true in the
// last CTA to arrive, with the totals valid in every thread of that CTA.
template <int BLOCK, int K>
__device__ __forceinline__ bool grid_sum(double (&v)[K], double *partials, unsigned *counter,
                                         double (&tot)[K]) {
    __shared__ double red[32];
    __shared__ bool last;
    __shared__ double bc[K];
    const int G = gridDim.x;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = block_sum<BLOCK>(v[k], red);
        if (threadIdx.x == 0) partials[k * G + blockIdx.x] = s;
    }
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(counter, 1u) == (unsigned)(G - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double acc = 0.0;
        for (int i = threadIdx.x; i < G; i += BLOCK) acc += __ldcg(partials + k * G + i);
        double s = block_sum<BLOCK>(acc, red);
        if (threadIdx.x == 0) bc[k] = s;
    }
    if (threadIdx.x == 0) *counter = 0u;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = bc[k];
    return true;
}

__global__ void set_args_kernel(PcgArgs *dst, PcgArgs a, PcgState *st, double tol, long long max_it) {
    *dst = a;
    PcgState s{};
    s.tol = tol;
    s.max_it = max_it;
    s.zero_row = -1;
    s.beta = 0.0;
    *st = s;
}

// Jacobi: inv_diag = 1/diag, zero diagonal -> SolverError (krylov.py:112-117)
__global__ void jacobi_kernel(int64_t n, const double *__restrict__ diag, double *__restrict__ inv,
                              PcgState *st) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = diag[i];
        inv[i] = 1.0 / d;
        if (d == 0.0) {
            atomicMin(reinterpret_cast<unsigned long long *>(&st->zero_row), (unsigned long long)i);
            st->status = TSB_E_SOLVER;
            st->done = 1;
        }
    }
}

// bnorm = ||b|| (krylov.py:132-134)
__global__ void __launch_bounds__(kVecBlock)
bnorm_kernel(PcgBufs B) {
    const PcgArgs *a = B.args;
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)kVecBlock + threadIdx.x; i < B.n; i += (int64_t)gridDim.x * kVecBlock) {
        const double bi = a->b[i];
        v[0] += bi * bi;
    }
    double tot[1];
    if (grid_sum<kVecBlock, 1>(v, B.partials, B.counter, tot) && threadIdx.x == 0) {
        PcgState *st = B.st;
        st->bnorm = sqrt(tot[0]);
        if (st->bnorm == 0.0 && st->status == 0) {
            st->done = 1;
            st->converged = 1;
            st->res = 0.0;
        }
    }
}

// r = b - A x0 (krylov.py:135), bit-exact SpMV
__global__ void __launch_bounds__(kSpBlock)
residual_kernel(PcgBufs B) {
    const PcgArgs *a = B.args;
    const int lane = threadIdx.x & 31, lane8 = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    XPlain xa{a->x0};
    for (int64_t row = (int64_t)blockIdx.x * (kSpBlock / 8) + (threadIdx.x >> 3); row < B.n;
         row += (int64_t)gridDim.x * (kSpBlock / 8)) {
        const int lo = a->rp[row], hi = a->rp[row + 1];
        const double s = row_sum_exact(lo, hi - lo, a->ci, a->val, xa, lane8, gmask);
        if (lane8 == 0) B.r[row] = sub(a->b[row], s);
    }
}

// x = x0|0, r = b (if no x0), z = M r (diag kinds), ||r||^2, r.z; initial
// convergence test (krylov.py:133-141)
template <int KIND>
__global__ void __launch_bounds__(kVecBlock)
init_kernel(PcgBufs B) {
    const PcgArgs *a = B.args;
    PcgState *st = B.st;
    const bool zero_b = st->bnorm == 0.0;
    double v[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kVecBlock + threadIdx.x; i < B.n; i += (int64_t)gridDim.x * kVecBlock) {
        double ri;
        if (a->x0 == nullptr || zero_b) {
            a->x[i] = 0.0;
            ri = a->b[i];
            B.r[i] = ri;
        } else {
            a->x[i] = a->x0[i];
            ri = B.r[i];
        }
        B.p0[i] = 0.0;
        v[0] += ri * ri;
        if (KIND == TSB_PRECOND_JACOBI) {
            const double zi = mul(ri, B.invdiag[i]);
            B.z[i] = zi;
            v[1] += ri * zi;
        } else if (KIND == TSB_PRECOND_IDENTITY) {
            B.z[i] = ri;
        }
    }
    double tot[2];
    if (grid_sum<kVecBlock, 2>(v, B.partials, B.counter, tot) && threadIdx.x == 0) {
        if (!st->done) {
            st->res = sqrt(tot[0]) / st->bnorm;
            if (st->res <= st->tol) {
                st->done = 1;
                st->converged = 1;
            } else if (st->max_it <= 0) {
                st->done = 1;
            }
            st->rz = KIND == TSB_PRECOND_IDENTITY ? tot[0] : tot[1];
        }
    }
}

// rz = r.z after an LDL^T apply (init: rz; loop: beta, rz <- rz_next)
__global__ void __launch_bounds__(kVecBlock)
rz_kernel(PcgBufs B, int in_loop, cudaGraphConditionalHandle cond) {
    PcgState *st = B.st;
    if (*((volatile int32_t *)&st->done)) {
        if (in_loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)kVecBlock + threadIdx.x; i < B.n; i += (int64_t)gridDim.x * kVecBlock)
        v[0] += B.r[i] * B.z[i];
    double tot[1];
    if (grid_sum<kVecBlock, 1>(v, B.partials, B.counter, tot) && threadIdx.x == 0) {
        if (in_loop) {
            st->beta = tot[0] / st->rz;
            st->rz = tot[0];
            cudaGraphSetConditional(cond, st->done ? 0 : 1);
        } else {
            st->rz = tot[0];
        }
    }
}

// K1: ap = A p with p = z + beta p_old on the fly; p_new stored by the row owner;
// alpha = rz / (p . ap)   (krylov.py:145-146)
__global__ void __launch_bounds__(kSpBlock)
spmv_dir_kernel(PcgBufs B) {
    PcgState *st = B.st;
    if (*((volatile int32_t *)&st->done)) return;
    const PcgArgs *a = B.args;
    const long long k = st->it;
    const double *pold = (k & 1) ? B.p1 : B.p0;
    double *pnew = (k & 1) ? B.p0 : B.p1;
    XDirection xa{B.z, pold, st->beta};
    const int lane = threadIdx.x & 31, lane8 = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    double v[1] = {0.0};
    for (int64_t row = (int64_t)blockIdx.x * (kSpBlock / 8) + (threadIdx.x >> 3); row < B.n;
         row += (int64_t)gridDim.x * (kSpBlock / 8)) {
        const int lo = a->rp[row], hi = a->rp[row + 1];
        const double s = row_sum_exact(lo, hi - lo, a->ci, a->val, xa, lane8, gmask);
        if (lane8 == 0) {
            const double pr = xa((int)row);
            pnew[row] = pr;
            B.ap[row] = s;
            v[0] += pr * s;
        }
    }
    double tot[1];
    if (grid_sum<kSpBlock, 1>(v, B.partials, B.counter, tot) && threadIdx.x == 0) {
        st->alpha = st->rz / tot[0];
    }
}

// K2: x += alpha p; r -= alpha ap; convergence (krylov.py:147-153); diagonal
// preconditioners also produce z and beta here (154-157).
template <int KIND>
__global__ void __launch_bounds__(kVecBlock)
update_kernel(PcgBufs B, cudaGraphConditionalHandle cond) {
    PcgState *st = B.st;
    if (*((volatile int32_t *)&st->done)) {
        if (KIND != TSB_PRECOND_LDLT && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    const PcgArgs *a = B.args;
    const double alpha = st->alpha;
    const double *p = (st->it & 1) ? B.p0 : B.p1;
    double v[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kVecBlock + threadIdx.x; i < B.n; i += (int64_t)gridDim.x * kVecBlock) {
        a->x[i] = add(a->x[i], mul(alpha, p[i]));
        const double ri = sub(B.r[i], mul(alpha, B.ap[i]));
        B.r[i] = ri;
        v[0] += ri * ri;
        if (KIND == TSB_PRECOND_JACOBI) {
            const double zi = mul(ri, B.invdiag[i]);
            B.z[i] = zi;
            v[1] += ri * zi;
        } else if (KIND == TSB_PRECOND_IDENTITY) {
            B.z[i] = ri;
        }
    }
    double tot[2];
    if (grid_sum<kVecBlock, 2>(v, B.partials, B.counter, tot) && threadIdx.x == 0) {
        st->it += 1;
        st->res = sqrt(tot[0]) / st->bnorm;
        if (st->res <= st->tol) {
            st->converged = 1;
            st->done = 1;
        } else if (st->it >= st->max_it) {
            st->done = 1;
        } else if (KIND != TSB_PRECOND_LDLT) {
            const double rzn = KIND == TSB_PRECOND_IDENTITY ? tot[0] : tot[1];
            st->beta = rzn / st->rz;
            st->rz = rzn;
        }
        if (KIND != TSB_PRECOND_LDLT) cudaGraphSetConditional(cond, st->done ? 0 : 1);
    }
}

}  // namespace tsb

struct tsb_pcg {
    tsb::PcgBufs B;
    void *mem = nullptr;
    tsb::PcgState *h_state = nullptr;  // pinned
    struct Graph {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t exec = nullptr;
    };
    std::map<std::pair<int, uint64_t>, Graph> graphs;
    std::vector<std::pair<int, uint64_t>> order;
};

namespace tsb {

static void enqueue_body(tsb_pcg *h, int kind, tsb_ldlt_t ldlt, cudaGraphConditionalHandle cond,
                         cudaStream_t s) {
    const PcgBufs &B = h->B;
    spmv_dir_kernel<<<spmv_grid(B.n), kSpBlock, 0, s>>>(B);
    TSB_LAUNCHED();
    const int vg = vec_grid(B.n);
    if (kind == TSB_PRECOND_JACOBI) {
        update_kernel<TSB_PRECOND_JACOBI><<<vg, kVecBlock, 0, s>>>(B, cond);
    } else if (kind == TSB_PRECOND_IDENTITY) {
        update_kernel<TSB_PRECOND_IDENTITY><<<vg, kVecBlock, 0, s>>>(B, cond);
    } else {
        update_kernel<TSB_PRECOND_LDLT><<<vg, kVecBlock, 0, s>>>(B, cond);
        TSB_LAUNCHED();
        ldlt_enqueue(ldlt, 2, B.r, B.z, &B.st->done, s);
        rz_kernel<<<vg, kVecBlock, 0, s>>>(B, 1, cond);
    }
    TSB_LAUNCHED();
}

static tsb_pcg::Graph &get_graph(tsb_pcg *h, int kind, tsb_ldlt_t ldlt, cudaStream_t s) {
    const uint64_t serial = kind == TSB_PRECOND_LDLT ? ldlt_serial(ldlt) : 0;
    auto key = std::make_pair(kind, serial);
    auto it = h->graphs.find(key);
    if (it != h->graphs.end()) return it->second;
    if (h->order.size() >= 4) {  // bounded cache
        auto old = h->order.front();
        h->order.erase(h->order.begin());
        auto &og = h->graphs[old];
        if (og.exec) cudaGraphExecDestroy(og.exec);
        if (og.g) cudaGraphDestroy(og.g);
        h->graphs.erase(old);
    }
    tsb_pcg::Graph gr;
    TSB_CUDA(cudaGraphCreate(&gr.g, 0));
    cudaGraphConditionalHandle cond;
    TSB_CUDA(cudaGraphConditionalHandleCreate(&cond, gr.g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    TSB_CUDA(cudaGraphAddNode(&node, gr.g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // capture the body on a private stream
    cudaStream_t cs;
    TSB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    TSB_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t before = tsb_launch_count();
    enqueue_body(h, kind, ldlt, cond, cs);
    count_launch(before - tsb_launch_count());  // captured, not launched
    cudaGraph_t captured;
    TSB_CUDA(cudaStreamEndCapture(cs, &captured));
    TSB_CUDA(cudaStreamDestroy(cs));
    TSB_CUDA(cudaGraphInstantiate(&gr.exec, gr.g, 0));
    (void)s;
    h->order.push_back(key);
    return h->graphs[key] = gr;
}

}  // namespace tsb

extern "C" int tsb_pcg_create(int64_t n, tsb_pcg_t *out) {
    using namespace tsb;
    return guard([&] {
        if (n < 0 || out == nullptr) throw Error(TSB_E_ARG, "bad n/out");
        auto *h = new tsb_pcg;
        const int64_t nn = n > 0 ? n : 1;
        const int64_t G = (int64_t)kNumSM * 8;
        size_t bytes = sizeof(double) * (6 * nn + 2 * G) + 256 * 4 + sizeof(PcgState) + sizeof(PcgArgs) + 1024;
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
        PcgBufs &B = h->B;
        B.n = n;
        B.r = reinterpret_cast<double *>(take(8 * nn));
        B.z = reinterpret_cast<double *>(take(8 * nn));
        B.ap = reinterpret_cast<double *>(take(8 * nn));
        B.p0 = reinterpret_cast<double *>(take(8 * nn));
        B.p1 = reinterpret_cast<double *>(take(8 * nn));
        B.invdiag = reinterpret_cast<double *>(take(8 * nn));
        B.partials = reinterpret_cast<double *>(take(8 * 2 * G));
        B.counter = reinterpret_cast<unsigned *>(take(256));
        B.st = reinterpret_cast<PcgState *>(take(sizeof(PcgState)));
        B.args = reinterpret_cast<PcgArgs *>(take(sizeof(PcgArgs)));
        TSB_CUDA(cudaMemset(B.counter, 0, 256));
        TSB_CUDA(cudaMallocHost(&h->h_state, sizeof(PcgState)));
        *out = h;
    });
}

extern "C" int tsb_pcg_destroy(tsb_pcg_t h) {
    if (h == nullptr) return TSB_OK;
    for (auto &kv : h->graphs) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.g) cudaGraphDestroy(kv.second.g);
    }
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
        TSB_CUDA(cudaMemcpyAsync(h->h_state, h->B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
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
        if (nrows != h->B.n) throw Error(TSB_E_SOLVER, "pcg handle was created for a different size");
        if (kind < 0 || kind > 2) throw Error(TSB_E_ARG, "unknown preconditioner kind");
        if (kind == TSB_PRECOND_LDLT && ldlt == nullptr) throw Error(TSB_E_LIFECYCLE, "LDL^T factors not ready");
        cudaStream_t s = as_stream(stream);
        const PcgBufs &B = h->B;
        PcgArgs a{d_row_ptr, d_col_ind, d_values, d_b, d_x0, d_x};
        set_args_kernel<<<1, 1, 0, s>>>(B.args, a, B.st, tol, (long long)max_iterations);
        TSB_LAUNCHED();
        if (B.n > 0) {
            const int vg = vec_grid(B.n);
            if (kind == TSB_PRECOND_JACOBI && d_inv_diag != nullptr) {
                TSB_CUDA(cudaMemcpyAsync(B.invdiag, d_inv_diag, sizeof(double) * B.n,
                                         cudaMemcpyDeviceToDevice, s));
            } else if (kind == TSB_PRECOND_JACOBI) {
                launch_csr_diag(B.n, B.n, d_row_ptr, d_col_ind, d_values, B.ap, s);
                jacobi_kernel<<<vg, kVecBlock, 0, s>>>(B.n, B.ap, B.invdiag, B.st);
                TSB_LAUNCHED();
            }
            bnorm_kernel<<<vg, kVecBlock, 0, s>>>(B);
            TSB_LAUNCHED();
            if (d_x0 != nullptr) {
                residual_kernel<<<spmv_grid(B.n), kSpBlock, 0, s>>>(B);
                TSB_LAUNCHED();
            }
            if (kind == TSB_PRECOND_JACOBI) {
                init_kernel<TSB_PRECOND_JACOBI><<<vg, kVecBlock, 0, s>>>(B);
            } else if (kind == TSB_PRECOND_IDENTITY) {
                init_kernel<TSB_PRECOND_IDENTITY><<<vg, kVecBlock, 0, s>>>(B);
            } else {
                init_kernel<TSB_PRECOND_LDLT><<<vg, kVecBlock, 0, s>>>(B);
                TSB_LAUNCHED();
                ldlt_enqueue(ldlt, 2, B.r, B.z, &B.st->done, s);
                rz_kernel<<<vg, kVecBlock, 0, s>>>(B, 0, 0);
            }
            TSB_LAUNCHED();
            auto &g = get_graph(h, kind, ldlt, s);
            TSB_CUDA(cudaGraphLaunch(g.exec, s));
            count_launch(1);
        }
        if (report != nullptr) {
            TSB_CUDA(cudaMemcpyAsync(h->h_state, B.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
            TSB_CUDA(cudaStreamSynchronize(s));
            fill_report(*h->h_state, report);
            if (B.n == 0) {
                report->iterations = 0;
                report->final_residual = 0.0;
                report->converged = 1;
            }
        }
    });
}
