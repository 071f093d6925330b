// Level-scheduled nested-dissection LDL^T apply (GPU Cholesky preconditioner).
//
// Replaces solve_lower (ndprecond.py:647-671), solve_upper (674-691) and
// apply (694-700) of the reference; the factor values are produced on the
// host (ldlt_factor, ndprecond.py:501-572) and packed by
// paper_2306_05893_b200/ndprecond.py into this layout (all per block, blocks
// stored level-major: level l owns [level_ptr[l], level_ptr[l+1]), ascending
// start inside a level -- the reference's `factors.levels`):
//   tile inverses  t x t row-major per diagonal tile (ndprecond.py:575-587)
//   L11 panels     tile `it` -> rows [t1, m) x t columns, row-major (the
//                  column panel the column-major forward push streams)
//   L21            |anc| x m row-major (ndprecond.py:465)
//   anc            permuted ancestor row ids
//   cin            per permuted row, the contribution-buffer slots of every
//                  descendant block touching it, in (level, start) order
// Lower sweep (column-major, paper Fig. solveBlock): one CTA per block of the
// level; the block first gathers the pre-accumulated ancestor contributions
// of its descendants (reference: `y[bf.anc] -= contrib` applied in block
// order at each level barrier, ndprecond.py:668-670 -- the gather reproduces
// that order, so no atomics and a deterministic result), solves its rows
// tile by tile (tile_inv in shared memory, trailing column-panel push), then
// pre-accumulates its own contribution l21 @ seg into its slice of the
// contribution buffer for its ancestors.
// Upper sweep (row-major, levels reversed): each block gathers l21^T z[anc]
// from already-solved ancestors and back-substitutes its tiles.
// Both sweeps stream every factor byte exactly once.
#include <mutex>
#include <vector>

#include "tsb_common.cuh"

struct tsb_ldlt {
    tsb_ldlt_desc d;
    std::vector<int32_t> level_ptr;
    uint64_t serial;
};

namespace tsb {

constexpr int kLdltBlock = 256;
constexpr int kMaxTile = 32;

__global__ void __launch_bounds__(kLdltBlock)
lower_level_kernel(tsb_ldlt_desc D, int lvl_begin, const double *__restrict__ in,
                   const int32_t *__restrict__ in_perm, double *__restrict__ y,
                   const int32_t *__restrict__ done) {
    if (done != nullptr && *((volatile const int32_t *)done)) return;
    const int b = lvl_begin + blockIdx.x;
    const int s = D.d_blk_start[b], m = D.d_blk_size[b], A = D.d_blk_nanc[b];
    const int t = D.tile;
    const int tid = threadIdx.x;
    __shared__ double sv[kMaxTile];
    __shared__ double sy[kMaxTile];

    // 1. rows of this block: input (through perm for apply) minus the
    //    contributions its descendants pre-accumulated, in level/block order
    for (int k = tid; k < m; k += kLdltBlock) {
        const int row = s + k;
        double v = in[in_perm ? in_perm[row] : row];
        const int64_t q0 = D.d_cin_ptr[row], q1 = D.d_cin_ptr[row + 1];
        for (int64_t q = q0; q < q1; ++q) v = sub(v, D.d_cbuf[D.d_cin_idx[q]]);
        y[row] = v;
    }
    __syncthreads();

    // 2. column-major forward push over diagonal tiles (_forward_block 623-631)
    const double *P = D.d_l11 + D.d_blk_l11[b];
    const double *Ti = D.d_tinv + D.d_blk_tinv[b];
    const int T = (m + t - 1) / t;
    for (int it = 0; it < T; ++it) {
        const int t0 = it * t;
        const int w = min(t, m - t0);
        const int t1 = t0 + w;
        if (tid < t) sy[tid] = tid < w ? y[s + t0 + tid] : 0.0;
        __syncthreads();
        if (tid < w) {
            const double *row = Ti + (int64_t)it * t * t + tid * t;
            double acc = 0.0;
            for (int j = 0; j < w; ++j) acc += row[j] * sy[j];
            sv[tid] = acc;
            y[s + t0 + tid] = acc;
        }
        __syncthreads();
        // trailing rows [t1, m) -= P_it @ sv ; 4 lanes per row (t/4 columns each)
        const int cpl = t / 4;
        // warp-uniform trip count so the full-mask shuffles stay converged
        for (int rb = t1 + (tid & ~31) / 4; rb < m; rb += kLdltBlock / 4) {
            const int r = rb + ((tid & 31) >> 2);
            double part = 0.0;
            if (r < m) {
                const double *pr = P + (int64_t)(r - t1) * t + (tid & 3) * cpl;
                for (int c = 0; c < cpl; ++c) part += pr[c] * sv[(tid & 3) * cpl + c];
            }
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            if ((tid & 3) == 0 && r < m) y[s + r] -= part;
        }
        P += (int64_t)(m - t1) * t;
        __syncthreads();
    }

    // 3. ancestor pre-accumulation: cbuf[k] = l21[k, :] @ seg (ndprecond.py:660)
    if (A > 0) {
        const double *L = D.d_l21 + D.d_blk_l21[b];
        double *cb = D.d_cbuf + D.d_blk_anc[b];
        const int warp = tid >> 5, lane = tid & 31;
        for (int k = warp; k < A; k += kLdltBlock / 32) {
            const double *lr = L + (int64_t)k * m;
            double acc = 0.0;
            for (int j = lane; j < m; j += 32) acc += lr[j] * y[s + j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) cb[k] = acc;
        }
    }
}

__global__ void __launch_bounds__(kLdltBlock)
upper_level_kernel(tsb_ldlt_desc D, int lvl_begin, const double *__restrict__ in,
                   const double *__restrict__ dscale, double *__restrict__ z,
                   const int32_t *__restrict__ out_perm, double *__restrict__ out,
                   const int32_t *__restrict__ done) {
    if (done != nullptr && *((volatile const int32_t *)done)) return;
    const int b = lvl_begin + blockIdx.x;
    const int s = D.d_blk_start[b], m = D.d_blk_size[b], A = D.d_blk_nanc[b];
    const int t = D.tile;
    const int tid = threadIdx.x;
    __shared__ double red[kLdltBlock];
    __shared__ double sv[kMaxTile];

    // 1. seg = w - l21^T z[anc]   (ndprecond.py:680-681)
    const double *L = D.d_l21 + D.d_blk_l21[b];
    const int32_t *anc = D.d_anc + D.d_blk_anc[b];
    for (int j = tid; j < m; j += kLdltBlock) {
        double acc = 0.0;
        for (int k = 0; k < A; ++k) acc += L[(int64_t)k * m + j] * z[anc[k]];
        double v = in[s + j];
        if (dscale) v = v / dscale[s + j];
        z[s + j] = v - acc;
    }
    __syncthreads();

    // 2. backward tiles, row-major pull (_backward_block 634-644)
    const double *P0 = D.d_l11 + D.d_blk_l11[b];
    const double *Ti = D.d_tinv + D.d_blk_tinv[b];
    const int T = (m + t - 1) / t;
    // offset of the last panel
    int64_t poff = 0;
    for (int it = 0; it < T; ++it) poff += (int64_t)(m - min(it * t + t, m)) * t;
    for (int it = T - 1; it >= 0; --it) {
        const int t0 = it * t;
        const int w = min(t, m - t0);
        const int t1 = t0 + w;
        poff -= (int64_t)(m - t1) * t;
        const double *P = P0 + poff;
        // acc_c = sum_{r in [t1,m)} P[r-t1][c] * z[s+r], c < t   (16 row groups x t columns)
        const int c = tid % t, rg = tid / t, ngroups = kLdltBlock / t;
        double part = 0.0;
        for (int r = t1 + rg; r < m; r += ngroups) part += P[(int64_t)(r - t1) * t + c] * z[s + r];
        red[tid] = part;
        __syncthreads();
        if (tid < w) {
            double acc = 0.0;
            for (int g = 0; g < ngroups; ++g) acc += red[g * t + tid];
            sv[tid] = z[s + t0 + tid] - acc;
        }
        __syncthreads();
        if (tid < w) {
            double acc = 0.0;
            const double *Tb = Ti + (int64_t)it * t * t;
            for (int q = 0; q < w; ++q) acc += Tb[q * t + tid] * sv[q];
            z[s + t0 + tid] = acc;
        }
        __syncthreads();
    }
    if (out_perm) {
        for (int j = tid; j < m; j += kLdltBlock) out[out_perm[s + j]] = z[s + j];
    }
}

static uint64_t g_serial = 0;
static std::mutex g_serial_mu;

void ldlt_enqueue(tsb_ldlt_t h, int mode, const double *r, double *out, const int32_t *done,
                  cudaStream_t st) {
    // mode 0: lower (r permuted -> out permuted); 1: upper; 2: apply
    const tsb_ldlt_desc &D = h->d;
    const int nl = (int)D.n_levels;
    if (mode == 0 || mode == 2) {
        double *y = mode == 2 ? D.d_y : out;
        const int32_t *perm = mode == 2 ? D.d_perm : nullptr;
        for (int l = 0; l < nl; ++l) {
            const int b0 = h->level_ptr[l], b1 = h->level_ptr[l + 1];
            if (b1 <= b0) continue;
            lower_level_kernel<<<b1 - b0, kLdltBlock, 0, st>>>(D, b0, r, perm, y, done);
            TSB_LAUNCHED();
        }
    }
    if (mode == 1 || mode == 2) {
        const double *in = mode == 2 ? D.d_y : r;
        double *z = mode == 2 ? D.d_y : out;
        const double *scale = mode == 2 ? D.d_d : nullptr;
        const int32_t *operm = mode == 2 ? D.d_perm : nullptr;
        for (int l = nl - 1; l >= 0; --l) {
            const int b0 = h->level_ptr[l], b1 = h->level_ptr[l + 1];
            if (b1 <= b0) continue;
            upper_level_kernel<<<b1 - b0, kLdltBlock, 0, st>>>(D, b0, in, scale, z, operm, out, done);
            TSB_LAUNCHED();
        }
    }
}

uint64_t ldlt_serial(tsb_ldlt_t h) { return h->serial; }

}  // namespace tsb

extern "C" int tsb_ldlt_create(const tsb_ldlt_desc *desc, tsb_ldlt_t *out) {
    using namespace tsb;
    return guard([&] {
        if (desc == nullptr || out == nullptr) throw Error(TSB_E_ARG, "null desc/out");
        if (desc->tile < 4 || desc->tile > kMaxTile || desc->tile % 4 != 0)
            throw Error(TSB_E_ARG, "tile must be a multiple of 4 in [4, 32]");
        if (kLdltBlock % desc->tile != 0) throw Error(TSB_E_ARG, "tile must divide the CTA size");
        auto *h = new tsb_ldlt;
        h->d = *desc;
        h->level_ptr.assign(desc->h_level_ptr, desc->h_level_ptr + desc->n_levels + 1);
        h->d.h_level_ptr = nullptr;
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
