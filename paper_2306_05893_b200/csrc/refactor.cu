// Device LDL^T refactorisation (numeric phase of ldlt_factor, ndprecond.py:501-572,
// plus the pack of the factor into the sweep layout of ldlt_sweep.cuh).
//
// Multifrontal over the dissection tree, one height of the tree at a time.
// Front of block b (m pivots, na coupling rows, nf = m + na), column-major:
//
//     F = [ A_bb       .   ]   + extend-add of every child's update matrix U_c
//         [ A_anc,b    0   ]     (children in start order: fixed summation order)
//
// A tiled right-looking partial Cholesky of the m pivots (64 x 64 tiles; the
// pivot tiles end at m so the coupling part starts on a tile boundary) leaves
//     C  (m x m lower),   LS = F21 C^-T,   U = F22 - LS LS^T  (to the parent).
// Then a right triangular solve  [W; M] C = [I; LS]  gives W = C^-1 and
// M = LS C^-1 = L21 L11^-1, and the pack writes the sweep operator
// G = [Linv; M] with Linv = diag(C) C^-1 (unit diagonal stored as 1.0) into
// the tiles of the handle (d_g lower rows, d_gt upper rows) and d = diag(C)^2.
//
// Every op is a batch of 64 x 64 x 64 fp64 tile products (one CTA each, 8
// warps x 32 x 16 on the FP64 tensor path, mma.sync m8n8k4) over all fronts
// of a height: the work is dense FP64,
// the launch sequence is a host "program" planned once per pattern
// (paper_2306_05893_b200/refactor.py).  All sums run in a fixed order: the
// result is bit-reproducible run to run.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "tsb_common.cuh"

namespace tsb {
namespace rf {

constexpr int NB = 64;
constexpr int LDS = 66;  // smem row stride (doubles): 16 B aligned rows
constexpr int kThreads = 256;
constexpr int kGemmSmem = 2 * NB * LDS * (int)sizeof(double);

__device__ __forceinline__ int tile_start(const tsb_front &f, int t) {
    return t < f.P ? t * NB : f.m + (t - f.P) * NB;
}
__device__ __forceinline__ int tile_width(const tsb_front &f, int t) {
    return t < f.P ? min(NB, f.m - t * NB) : min(NB, f.nf - (f.m + (t - f.P) * NB));
}

// task -> list entry: last entry whose exclusive prefix (field 1 or 2) <= task
__device__ __forceinline__ int find_entry(const int4 *L, int n, bool second, int task, int *local) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        const int v = second ? __ldg(&L[mid].z) : __ldg(&L[mid].y);
        if (v <= task) lo = mid; else hi = mid - 1;
    }
    *local = task - (second ? __ldg(&L[lo].z) : __ldg(&L[lo].y));
    return lo;
}

__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// dst[q][r] = src[q * ld + r]  (element (r, q) of a column-major matrix), zero-padded;
// asynchronous (cp.async, zero-fill outside): every thread's 16 copies are in
// flight together.  Complete with cp_async_wait() + __syncthreads().
__device__ __forceinline__ void load_n(double *dst, const double *src, int64_t ld, int rows, int cols) {
#pragma unroll
    for (int u = 0; u < NB * NB / kThreads; ++u) {
        const int i = threadIdx.x + u * kThreads;
        const int r = i & (NB - 1), q = i >> 6;
        const bool ok = r < rows && q < cols;
        cp_async8(dst + q * LDS + r, ok ? src + (int64_t)q * ld + r : src, ok);
    }
}
// dst[q][c] = src[c * ld + q]  (element (q, c) of a column-major matrix), zero-padded
__device__ __forceinline__ void load_t(double *dst, const double *src, int64_t ld, int qs, int cs) {
#pragma unroll
    for (int u = 0; u < NB * NB / kThreads; ++u) {
        const int i = threadIdx.x + u * kThreads;
        const int q = i & (NB - 1), c = i >> 6;
        const bool ok = q < qs && c < cs;
        cp_async8(dst + q * LDS + c, ok ? src + (int64_t)c * ld + q : src, ok);
    }
}

// 64 x 64 tile product on the FP64 tensor path (mma.sync m8n8k4 f64, DMMA):
// warp w owns rows (w & 1) * 32 + [0, 32) and columns (w >> 1) * 16 + [0, 16)
// as 4 x 2 tiles of 8 x 8; per k-step of 4 a lane loads one A element per
// row tile and one B element per column tile (fragment layout of m8n8k4:
// A (groupID, threadID_in_group), B (threadID_in_group, groupID), C
// (groupID, 2 threadID_in_group + i)).  acc[a][2 nt + i] is element
// acc_rc(a, 2 nt + i).
__device__ __forceinline__ void acc_rc(int a, int b, int &r, int &c) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    r = (w & 1) * 32 + a * 8 + (lane >> 2);
    c = (w >> 1) * 16 + (b >> 1) * 8 + (lane & 3) * 2 + (b & 1);
}

// acc(r, c) = sum_q As[q][r] * Bs[q][c]
__device__ __forceinline__ void tile_mma(const double *As, const double *Bs, int K, double acc[4][4]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int r0 = (w & 1) * 32 + gid, c0 = (w >> 1) * 16 + gid;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    const int ks_end = (K + 3) >> 2;
#pragma unroll 4
    for (int ks = 0; ks < ks_end; ++ks) {
        const int q = ks * 4 + tig;
        double av[4], bv[2];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[q * LDS + r0 + a * 8];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) bv[nt] = Bs[q * LDS + c0 + nt * 8];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(acc[a][2 * nt]), "+d"(acc[a][2 * nt + 1])
                             : "d"(av[a]), "d"(bv[nt]));
    }
}

// MODE 0: dst = acc; 1: dst -= acc; 2: dst -= acc on the lower triangle (r >= c).
// The read-modify-write issues all 16 loads before the first store.
template <int MODE>
__device__ __forceinline__ void store_tile(double *dst, int64_t ld, int rows, int cols, const double acc[4][4]) {
    double old[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int r, c;
            acc_rc(a, b, r, c);
            const bool ok = r < rows && c < cols && (MODE != 2 || r >= c);
            old[a][b] = (MODE != 0 && ok) ? __ldcg(dst + (int64_t)c * ld + r) : 0.0;
        }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int r, c;
            acc_rc(a, b, r, c);
            if (r >= rows || c >= cols || (MODE == 2 && r < c)) continue;
            dst[(int64_t)c * ld + r] = MODE == 0 ? acc[a][b] : old[a][b] - acc[a][b];
        }
}

__global__ void __launch_bounds__(256) scatter_kernel(int64_t n, const int32_t *__restrict__ src,
                                                      const int64_t *__restrict__ dst,
                                                      const double *__restrict__ vals, double *__restrict__ ws) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ws[__ldg(dst + i)] = __ldg(vals + __ldg(src + i));
}

// U_child (lower) += into the parent front at tp positions; one warp per child column.
__global__ void __launch_bounds__(256) extend_kernel(const tsb_front_pair *__restrict__ pairs,
                                                     const tsb_front *__restrict__ F,
                                                     const int32_t *__restrict__ tp_all, double *__restrict__ ws) {
    const tsb_front_pair pr = pairs[blockIdx.y];
    const tsb_front c = F[pr.child], p = F[pr.parent];
    const int32_t *tp = tp_all + pr.tp_off;
    const double *u = ws + c.off + (int64_t)c.m * c.nf + c.m;
    double *fp = ws + p.off;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = blockIdx.x * 8 + warp; j < c.na; j += gridDim.x * 8) {
        const int64_t pcol = (int64_t)__ldg(tp + j) * p.nf;
        const double *uc = u + (int64_t)j * c.nf;
        constexpr int U = 4;  // loads of U rows in flight before their read-modify-writes
        for (int i0 = j + lane; i0 < c.na; i0 += 32 * U) {
            int64_t dst[U];
            double val[U], cur[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int i = i0 + 32 * q;
                dst[q] = i < c.na ? pcol + __ldg(tp + i) : -1;
                val[q] = i < c.na ? __ldcg(uc + i) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < U; ++q) cur[q] = dst[q] >= 0 ? __ldcg(fp + dst[q]) : 0.0;
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (dst[q] >= 0) fp[dst[q]] = cur[q] + val[q];
        }
    }
}

// Pivot tile k: W_kk = C_kk^-1 and diag(C_kk) by in-place Gauss-Jordan style
// elimination (one CTA of 256 threads per front).  X starts as the full
// symmetric tile; step j eliminates column j from rows i > j with the unscaled
// row j (m_i = X_ij / p_j): the trailing A part and the inverse part (columns
// < j) update uniformly as X_it -= m_i X_jt, and the inverse entry born at
// (i, j) is -m_i, stored where the eliminated A entry was.  Row j is never
// read after step j, so every row of the inverse is scaled by p^-1/2 at the
// end, and X's lower triangle ends as D^-1/2 L^-1 = C^-1.  Only diag(C) and C^-1 of the pivot tile are
// consumed downstream (panel, right solve, pack).
//
// The tile lives in registers: thread (a = tid & 63, g = tid >> 6) owns row a,
// columns g + 4u (u < 16).  A step is one barrier: the owners of column j and
// row j publish them into a double-buffered pair of shared vectors, then every
// thread updates its 16 entries.  The 64 steps are unrolled so the register
// index of column / row j is static.
constexpr int kDiagLd = 65;
constexpr int kDiagSmem = (NB * kDiagLd + 4 * NB) * (int)sizeof(double);

__global__ void __launch_bounds__(256, 1) diag_kernel(const tsb_front *__restrict__ F, const int4 *__restrict__ list,
                                                   int k, double *__restrict__ ws, double *__restrict__ inv,
                                                   int32_t *__restrict__ ctl) {
    extern __shared__ __align__(16) double sm[];
    double *X = sm, *colb = sm + NB * kDiagLd, *rowb = colb + 2 * NB;
    const int fi = __ldg(&list[blockIdx.x].x);
    const tsb_front f = F[fi];
    const int c0 = k * NB, w = min(NB, f.m - c0);
    double *base = ws + f.off + (int64_t)c0 * f.nf + c0;
    const int tid = threadIdx.x, a = tid & (NB - 1), g = tid >> 6;
    {
        double v[NB * NB / kThreads];  // all 16 loads in flight together
#pragma unroll
        for (int u = 0; u < NB * NB / kThreads; ++u) {
            const int i = tid + u * kThreads, r = i & (NB - 1), c = i >> 6;
            v[u] = (r < w && c < w) ? base[r >= c ? (int64_t)c * f.nf + r : (int64_t)r * f.nf + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NB * NB / kThreads; ++u) {
            const int i = tid + u * kThreads, r = i & (NB - 1), c = i >> 6;
            X[r * kDiagLd + c] = v[u];
        }
    }
    __syncthreads();
    double x[16], piv = 1.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = X[a * kDiagLd + g + 4 * u];
#pragma unroll
    for (int uj = 0; uj < 16; ++uj) {
#pragma unroll
        for (int ph = 0; ph < 4; ++ph) {
            const int j = 4 * uj + ph;
            if (j >= w) break;
            double *cb = colb + (j & 1) * NB, *rb = rowb + (j & 1) * NB;
            if (g == ph) cb[a] = x[uj];  // column j
            if (a == j) {
#pragma unroll
                for (int u = 0; u < 16; u += 2)  // row j, column g + 4u at rb[16 g + u]
                    *reinterpret_cast<double2 *>(rb + 16 * g + u) = make_double2(x[u], x[u + 1]);
            }
            __syncthreads();
            const double p = rb[16 * ph + uj];
            if (a > j) {
                double r[16];
#pragma unroll
                for (int u = 0; u < 16; u += 2) {
                    const double2 t = *reinterpret_cast<const double2 *>(rb + 16 * g + u);
                    r[u] = t.x;
                    r[u + 1] = t.y;
                }
                const double m = cb[a] * __drcp_rn(p);
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    if (u == uj && g == ph) x[u] = -m;  // inverse entry born at (a, j)
                    else x[u] = fma(-m, r[u], x[u]);
                }
            } else if (a == j) {
                piv = p;
            }
        }
    }
    // row a of the inverse: scale by p_a^-1/2 (row a is final once step a used it)
    if (a < w) {
        const double dsq = sqrt(piv), rsq = 1.0 / dsq;
        if (g == (a & 3)) {
            if (!(piv > 0.0)) atomicCAS(ctl, 0, fi + 1);
            base[(int64_t)a * f.nf + a] = dsq;  // diag(C); the pack and d read it
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int c = g + 4 * u;
            if (c < a) x[u] *= rsq;
            else if (c == a) x[u] = rsq;  // W_aa = p_a^-1/2
        }
    }
    double *wo = inv + f.ioff + (int64_t)k * NB * NB;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int c = g + 4 * u;
        wo[c * NB + a] = (a < w && c <= a) ? x[u] : 0.0;  // W(a, c), column-major
    }
}

// L_ik = F_ik W_kk^T for the row tiles below pivot tile k.
__global__ void __launch_bounds__(256) panel_kernel(const tsb_front *__restrict__ F, const int4 *__restrict__ list,
                                                    int nlist, int k, double *__restrict__ ws,
                                                    const double *__restrict__ inv) {
    extern __shared__ __align__(16) double sm[];
    double *As = sm, *Bs = sm + NB * LDS;
    int local;
    const int e = find_entry(list, nlist, false, blockIdx.x, &local);
    const tsb_front f = F[__ldg(&list[e].x)];
    const int i = k + 1 + local;
    const int r0 = tile_start(f, i), h = tile_width(f, i);
    const int c0 = k * NB, w = min(NB, f.m - c0);
    double *src = ws + f.off + (int64_t)c0 * f.nf + r0;
    load_n(As, src, f.nf, h, w);
    load_n(Bs, inv + f.ioff + (int64_t)k * NB * NB, NB, w, w);  // Bs[q][c] = W(c, q)
    cp_async_wait();
    __syncthreads();
    double acc[4][4];
    tile_mma(As, Bs, w, acc);
    store_tile<0>(src, f.nf, h, w, acc);
}

// F_ij -= L_ik L_jk^T for k < j <= i (lower tiles of the trailing matrix, U included).
__global__ void __launch_bounds__(256) update_kernel(const tsb_front *__restrict__ F, const int4 *__restrict__ list,
                                                     int nlist, int k, double *__restrict__ ws) {
    extern __shared__ __align__(16) double sm[];
    double *As = sm, *Bs = sm + NB * LDS;
    int local;
    const int e = find_entry(list, nlist, true, blockIdx.x, &local);
    const tsb_front f = F[__ldg(&list[e].x)];
    int rr = (int)((sqrt(8.0 * local + 1.0) - 1.0) * 0.5);
    while ((rr + 1) * (rr + 2) / 2 <= local) ++rr;
    while (rr * (rr + 1) / 2 > local) --rr;
    const int ss = local - rr * (rr + 1) / 2;
    const int i = k + 1 + rr, j = k + 1 + ss;
    const int ri = tile_start(f, i), hi = tile_width(f, i);
    const int rj = tile_start(f, j), hj = tile_width(f, j);
    const int c0 = k * NB, w = min(NB, f.m - c0);
    const double *col = ws + f.off + (int64_t)c0 * f.nf;
    load_n(As, col + ri, f.nf, hi, w);
    load_n(Bs, col + rj, f.nf, hj, w);
    cp_async_wait();
    __syncthreads();
    double acc[4][4];
    tile_mma(As, Bs, w, acc);
    double *dst = ws + f.off + (int64_t)rj * f.nf + ri;
    if (i == j) store_tile<2>(dst, f.nf, hi, hj, acc);
    else store_tile<1>(dst, f.nf, hi, hj, acc);
}

// Row tile idx of the right solve's B = [W-buffer (m rows); LS (na rows)].
__device__ __forceinline__ double *rhs_tile(const tsb_front &f, double *ws, double *wb, int k, int idx, int64_t *ld,
                                            int *rows) {
    if (idx < f.P - k) {
        const int i = k + idx;
        *ld = f.m;
        *rows = min(NB, f.m - i * NB);
        return wb + f.woff + i * NB;
    }
    const int b = idx - (f.P - k);
    *ld = f.nf;
    *rows = min(NB, f.na - b * NB);
    return ws + f.off + f.m + b * NB;
}

// X_:,k = B_:,k W_kk (right solve, column tile k, descending k)
__global__ void __launch_bounds__(256) tscale_kernel(const tsb_front *__restrict__ F, const int4 *__restrict__ list,
                                                     int nlist, int k, double *__restrict__ ws, double *__restrict__ wb,
                                                     const double *__restrict__ inv) {
    extern __shared__ __align__(16) double sm[];
    double *As = sm, *Bs = sm + NB * LDS;
    int local;
    const int e = find_entry(list, nlist, false, blockIdx.x, &local);
    const tsb_front f = F[__ldg(&list[e].x)];
    int64_t ld;
    int rows;
    double *b = rhs_tile(f, ws, wb, k, local, &ld, &rows);
    const int w = min(NB, f.m - k * NB);
    double *src = b + (int64_t)k * NB * ld;
    load_n(As, src, ld, rows, w);
    load_t(Bs, inv + f.ioff + (int64_t)k * NB * NB, NB, w, w);  // Bs[q][c] = W(q, c)
    cp_async_wait();
    __syncthreads();
    double acc[4][4];
    tile_mma(As, Bs, w, acc);
    store_tile<0>(src, ld, rows, w, acc);
}

// B_:,j -= X_:,k C_kj for j < k
__global__ void __launch_bounds__(256) tupdate_kernel(const tsb_front *__restrict__ F, const int4 *__restrict__ list,
                                                      int nlist, int k, double *__restrict__ ws, double *__restrict__ wb) {
    extern __shared__ __align__(16) double sm[];
    double *As = sm, *Bs = sm + NB * LDS;
    int local;
    const int e = find_entry(list, nlist, true, blockIdx.x, &local);
    const tsb_front f = F[__ldg(&list[e].x)];
    const int idx = local / k, j = local % k;
    int64_t ld;
    int rows;
    double *b = rhs_tile(f, ws, wb, k, idx, &ld, &rows);
    const int w = min(NB, f.m - k * NB);
    load_n(As, b + (int64_t)k * NB * ld, ld, rows, w);
    load_t(Bs, ws + f.off + (int64_t)j * NB * f.nf + k * NB, f.nf, w, NB);  // Bs[q][c] = C(kNB + q, jNB + c)
    cp_async_wait();
    __syncthreads();
    double acc[4][4];
    tile_mma(As, Bs, w, acc);
    store_tile<1>(b + (int64_t)j * NB * ld, ld, rows, NB, acc);
}

__global__ void ident_kernel(const tsb_front *__restrict__ F, double *__restrict__ wb) {
    const tsb_front f = F[blockIdx.x];
    for (int r = threadIdx.x; r < f.m; r += blockDim.x) wb[f.woff + (int64_t)r * f.m + r] = 1.0;
}

// G(r, c), c < m: r < m -> Linv(r, c) = C_rr W(r, c) (1 on the diagonal); r >= m -> M(r - m, c)
__device__ __forceinline__ double gval(const tsb_front &f, const double *ws, const double *wb, int r, int c) {
    if (r < f.m) {
        if (r == c) return 1.0;
        if (r < c) return 0.0;
        return ws[f.off + (int64_t)r * f.nf + r] * wb[f.woff + (int64_t)c * f.m + r];
    }
    return ws[f.off + (int64_t)c * f.nf + r];
}

// Tile image of the sweep operator (layout of _ldlt_pack.tile_block).
template <bool UPPER>
__global__ void __launch_bounds__(256) pack_kernel(const tsb_ldlt_tile *__restrict__ T, const int32_t *__restrict__ tblk,
                                                   const tsb_front *__restrict__ F, const double *__restrict__ ws,
                                                   const double *__restrict__ wb, double *__restrict__ out) {
    const tsb_ldlt_tile t = T[blockIdx.x];
    const tsb_front f = F[__ldg(tblk + blockIdx.x)];
    const int64_t n = (int64_t)t.np * 64;
    for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) {
        const int p = (int)(idx >> 6), rem = (int)(idx & 63), kk = rem >> 1, h = rem & 1;
        const int row = t.row0 + kk, col = t.tl + 2 * p + h;
        double v = 0.0;
        if (kk < t.nrows) {
            if (!UPPER) {
                if (col < min(row + 1, f.m)) v = gval(f, ws, wb, row, col);
            } else if (col >= row && col < f.nf) {
                v = gval(f, ws, wb, col, row);
            }
        }
        out[t.off + idx] = v;
    }
}

__global__ void d_kernel(const tsb_front *__restrict__ F, const double *__restrict__ ws, double *__restrict__ d) {
    const tsb_front f = F[blockIdx.x];
    for (int r = threadIdx.x; r < f.m; r += blockDim.x) {
        const double c = ws[f.off + (int64_t)r * f.nf + r];
        d[f.start + r] = c * c;
    }
}

}  // namespace rf
}  // namespace tsb

struct tsb_refactor {
    tsb_refactor_desc d;
    std::vector<int64_t> prog;
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> ev;  // [0] start, [1] side done, [2 + i] program events
    // the program captured once per (values, g, gt, d) as a CUDA graph and replayed
    // on an internal stream (capture works whatever stream the caller uses)
    struct Graph {
        const void *key[4];
        cudaGraphExec_t exec;
    };
    std::vector<Graph> graphs;
    cudaStream_t cap = nullptr;
    cudaEvent_t gev[2] = {nullptr, nullptr};  // caller -> graph, graph -> caller
};

extern "C" int tsb_refactor_create(const tsb_refactor_desc *desc, tsb_refactor_t *out) {
    using namespace tsb;
    return guard([&] {
        if (desc == nullptr || out == nullptr) throw Error(TSB_E_ARG, "null refactor desc");
        if (desc->n_prog < 0 || (desc->n_prog > 0 && desc->h_prog == nullptr)) throw Error(TSB_E_ARG, "bad program");
        static bool once = [] {
            allow_max_smem(rf::diag_kernel);
            allow_max_smem(rf::panel_kernel);
            allow_max_smem(rf::update_kernel);
            allow_max_smem(rf::tscale_kernel);
            allow_max_smem(rf::tupdate_kernel);
            return true;
        }();
        (void)once;
        auto *h = new tsb_refactor;
        h->d = *desc;
        h->prog.assign(desc->h_prog, desc->h_prog + 8 * desc->n_prog);
        h->d.h_prog = nullptr;
        int64_t nev = 0;
        for (int64_t o = 0; o < desc->n_prog; ++o)
            if (h->prog[8 * o] == TSB_RF_RECORD || h->prog[8 * o] == TSB_RF_WAIT)
                nev = std::max<int64_t>(nev, h->prog[8 * o + 1] + 1);
        TSB_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        h->ev.resize(2 + nev);
        for (auto &e : h->ev) TSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        *out = h;
    });
}

extern "C" int tsb_refactor_destroy(tsb_refactor_t h) {
    if (h != nullptr) {
        for (auto e : h->ev) cudaEventDestroy(e);
        for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
        for (auto e : h->gev)
            if (e) cudaEventDestroy(e);
        if (h->cap) cudaStreamDestroy(h->cap);
        if (h->side) cudaStreamDestroy(h->side);
    }
    delete h;
    return TSB_OK;
}

namespace tsb {
namespace rf {

// Enqueue the whole program on s0 (+ the handle's side stream, joined back).
static void enqueue_program(tsb_refactor *h, const double *d_values, double *d_g, double *d_gt, double *d_d,
                            cudaStream_t s0) {
        const tsb_refactor_desc &D = h->d;
        const int4 *lists = reinterpret_cast<const int4 *>(D.d_lists);
        TSB_CUDA(cudaMemsetAsync(D.d_ctl, 0, sizeof(int32_t), s0));
        TSB_CUDA(cudaEventRecord(h->ev[0], s0));  // the side stream starts after the caller's prior work
        TSB_CUDA(cudaStreamWaitEvent(h->side, h->ev[0], 0));
        for (int64_t o = 0; o < (int64_t)h->prog.size() / 8; ++o) {
            const int64_t *op = h->prog.data() + 8 * o;
            const int64_t a = op[1], b = op[2], c = op[3], dd = op[4];
            cudaStream_t s = op[5] ? h->side : s0;
            switch (op[0]) {
                case TSB_RF_RECORD:
                    TSB_CUDA(cudaEventRecord(h->ev[2 + a], s));
                    break;
                case TSB_RF_WAIT:
                    TSB_CUDA(cudaStreamWaitEvent(s, h->ev[2 + a], 0));
                    break;
                case TSB_RF_SCATTER: {
                    TSB_CUDA(cudaMemsetAsync(D.d_ws, 0, sizeof(double) * D.ws_size, s));
                    if (a > 0) {
                        const int g = (int)std::min<int64_t>((a + 255) / 256, kNumSM * 16);
                        scatter_kernel<<<g, 256, 0, s>>>(a, D.d_sc_src, D.d_sc_dst, d_values, D.d_ws);
                        TSB_LAUNCHED();
                    }
                    break;
                }
                case TSB_RF_IDENT:
                    TSB_CUDA(cudaMemsetAsync(D.d_wb, 0, sizeof(double) * D.wb_size, s));
                    if (D.n_fronts > 0) {
                        ident_kernel<<<(unsigned)D.n_fronts, 256, 0, s>>>(D.d_fronts, D.d_wb);
                        TSB_LAUNCHED();
                    }
                    break;
                case TSB_RF_EXTEND: {
                    if (b > a && c > 0) {
                        dim3 g((unsigned)std::min<int64_t>((c + 7) / 8, 1024), (unsigned)(b - a));
                        extend_kernel<<<g, 256, 0, s>>>(D.d_pairs + a, D.d_fronts, D.d_tp, D.d_ws);
                        TSB_LAUNCHED();
                    }
                    break;
                }
                case TSB_RF_DIAG:
                    diag_kernel<<<(unsigned)c, 256, kDiagSmem, s>>>(D.d_fronts, lists + b, (int)a, D.d_ws, D.d_inv,
                                                                    D.d_ctl);
                    TSB_LAUNCHED();
                    break;
                case TSB_RF_PANEL:
                    if (dd > 0) {
                        panel_kernel<<<(unsigned)dd, 256, kGemmSmem, s>>>(D.d_fronts, lists + b, (int)c, (int)a,
                                                                          D.d_ws, D.d_inv);
                        TSB_LAUNCHED();
                    }
                    break;
                case TSB_RF_UPDATE:
                    if (dd > 0) {
                        update_kernel<<<(unsigned)dd, 256, kGemmSmem, s>>>(D.d_fronts, lists + b, (int)c, (int)a,
                                                                           D.d_ws);
                        TSB_LAUNCHED();
                    }
                    break;
                case TSB_RF_TSCALE:
                    if (dd > 0) {
                        tscale_kernel<<<(unsigned)dd, 256, kGemmSmem, s>>>(D.d_fronts, lists + b, (int)c, (int)a,
                                                                           D.d_ws, D.d_wb, D.d_inv);
                        TSB_LAUNCHED();
                    }
                    break;
                case TSB_RF_TUPDATE:
                    if (dd > 0) {
                        tupdate_kernel<<<(unsigned)dd, 256, kGemmSmem, s>>>(D.d_fronts, lists + b, (int)c, (int)a,
                                                                            D.d_ws, D.d_wb);
                        TSB_LAUNCHED();
                    }
                    break;
                case TSB_RF_PACK:
                    if (D.n_tiles_lower > 0) {
                        pack_kernel<false><<<(unsigned)D.n_tiles_lower, 256, 0, s>>>(
                            D.d_tiles_lower, D.d_tile_blk_lower, D.d_fronts, D.d_ws, D.d_wb, d_g);
                        TSB_LAUNCHED();
                    }
                    if (D.n_tiles_upper > 0) {
                        pack_kernel<true><<<(unsigned)D.n_tiles_upper, 256, 0, s>>>(
                            D.d_tiles_upper, D.d_tile_blk_upper, D.d_fronts, D.d_ws, D.d_wb, d_gt);
                        TSB_LAUNCHED();
                    }
                    if (D.n_fronts > 0) {
                        d_kernel<<<(unsigned)D.n_fronts, 256, 0, s>>>(D.d_fronts, D.d_ws, d_d);
                        TSB_LAUNCHED();
                    }
                    break;
                default:
                    throw Error(TSB_E_ARG, "unknown refactor op");
            }
        }
        TSB_CUDA(cudaEventRecord(h->ev[1], h->side));  // everything on the side stream before the caller goes on
        TSB_CUDA(cudaStreamWaitEvent(s0, h->ev[1], 0));
}

static bool use_graph() {
    static const bool v = [] {
        const char *e = getenv("TSB_RF_GRAPH");
        return e == nullptr || atoi(e) != 0;
    }();
    return v;
}

}  // namespace rf
}  // namespace tsb

extern "C" int tsb_refactor_run(tsb_refactor_t h, const double *d_values, double *d_g, double *d_gt, double *d_d,
                                void *stream) {
    using namespace tsb;
    using namespace tsb::rf;
    return guard([&] {
        if (h == nullptr) throw Error(TSB_E_ARG, "null refactor handle");
        cudaStream_t s0 = as_stream(stream);
        if (!use_graph()) {
            enqueue_program(h, d_values, d_g, d_gt, d_d, s0);
            return;
        }
        const void *key[4] = {d_values, d_g, d_gt, d_d};
        cudaGraphExec_t exec = nullptr;
        for (auto &g : h->graphs)
            if (std::equal(key, key + 4, g.key)) exec = g.exec;
        if (exec == nullptr) {
            if (h->cap == nullptr) {
                TSB_CUDA(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
                for (auto &e : h->gev) TSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            TSB_CUDA(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
            cudaGraph_t graph = nullptr;
            try {
                enqueue_program(h, d_values, d_g, d_gt, d_d, h->cap);
            } catch (...) {
                cudaStreamEndCapture(h->cap, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            TSB_CUDA(cudaStreamEndCapture(h->cap, &graph));
            const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            TSB_CUDA(e);
            if (h->graphs.size() >= 4) {  // a few image/value buffers in rotation at most
                cudaGraphExecDestroy(h->graphs.front().exec);
                h->graphs.erase(h->graphs.begin());
            }
            tsb_refactor::Graph g;
            std::copy(key, key + 4, g.key);
            g.exec = exec;
            h->graphs.push_back(g);
        }
        TSB_CUDA(cudaEventRecord(h->gev[0], s0));
        TSB_CUDA(cudaStreamWaitEvent(h->cap, h->gev[0], 0));
        TSB_CUDA(cudaGraphLaunch(exec, h->cap));
        TSB_LAUNCHED();
        TSB_CUDA(cudaEventRecord(h->gev[1], h->cap));
        TSB_CUDA(cudaStreamWaitEvent(s0, h->gev[1], 0));
    });
}
