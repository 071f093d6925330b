// Bit-exact CSR row reduction shared by tsb_spmv and the fused PCG SpMV.
//
// The reference computes y = A x as
//     prod = values * x[col_ind]; y[rows] = np.add.reduceat(prod, starts)
// (krylov.py:63-70).  For float64, reduceat seeds each row with its first
// product and adds NumPy's pairwise sum of the remaining L-1 products:
//   n < 8      : sequential from -0.0
//   8<=n<=128  : 8 strided partial sums r_j, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//                then the n%8 tail sequentially
//   n > 128    : split at n/2 rounded down to a multiple of 8, recurse.
// One row is owned by a group of 8 lanes; lane j carries partial sum r_j and
// the xor-1/2/4 butterfly reproduces the combine tree exactly (IEEE addition
// is commutative), so the result equals the reference bit for bit.
#pragma once

#include "tsb_common.cuh"

namespace tsb {

// Plain x[j] accessor.
struct XPlain {
    const double *__restrict__ x;
    __device__ __forceinline__ double operator()(int j) const { return __ldg(x + j); }
};

// x[j] produced earlier in the same (persistent) kernel: read through L2.
struct XPlainCG {
    const double *x;
    __device__ __forceinline__ double operator()(int j) const { return __ldcg(x + j); }
};

// p_j = z_j + beta * p_old_j computed on the fly (PCG direction update
// fused into the SpMV, krylov.py:156); every reader rounds identically.
struct XDirection {
    const double *__restrict__ z;
    const double *__restrict__ pold;
    double beta;
    __device__ __forceinline__ double operator()(int j) const {
        return add(__ldcg(z + j), mul(beta, __ldcg(pold + j)));
    }
};

// Returns the exact row sum in every lane of the 8-lane group.
// `lane8` in [0,8), `gmask` = the group's lanes in the warp.
template <class XAcc>
__device__ __forceinline__ double row_sum_exact(int lo, int len, const int32_t *__restrict__ col,
                                                const double *__restrict__ val, const XAcc &xa,
                                                int lane8, unsigned gmask) {
    if (len <= 0) return 0.0;
    auto term = [&](int64_t k) -> double { return mul(__ldg(val + k), xa(__ldg(col + k))); };
    const int n = len - 1;  // terms handled by the pairwise sum
    double p0 = 0.0;        // first product seeds the row (issued with the other loads)
    if (lane8 == 0) p0 = term(lo);
    double res;
    if (n <= 64) {
        // common case (FEM rows <= 45 entries): every lane fetches its <= 8 terms
        // up front -- all index, value and gather loads in flight together --
        // then the same summation order as below, in registers
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = 8 * u + lane8;
            t[u] = idx < n ? term(lo + 1 + idx) : 0.0;
        }
        if (n >= 8) {
            const int nfull = (n - (n % 8)) / 8;  // complete groups of 8 terms
            double r = t[0];
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u < nfull) r = add(r, t[u]);
            r = add(r, __shfl_xor_sync(gmask, r, 1, 8));
            r = add(r, __shfl_xor_sync(gmask, r, 2, 8));
            r = add(r, __shfl_xor_sync(gmask, r, 4, 8));
            const int tail = n % 8;
            double tv = 0.0;
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u == nfull) tv = t[u];
            for (int k = 0; k < tail; ++k) r = add(r, __shfl_sync(gmask, tv, k, 8));
            res = r;
        } else {
            double r = -0.0;
            for (int k = 0; k < n; ++k) r = add(r, __shfl_sync(gmask, t[0], k, 8));
            res = r;
        }
    } else if (n > 128) {
        double r = 0.0;
        if (lane8 == 0) r = pairwise_serial(term, (int64_t)lo + 1, (int64_t)n);
        res = __shfl_sync(gmask, r, 0, 8);
    } else if (n >= 8) {
        const int full = n - (n % 8);
        double r = term(lo + 1 + lane8);
        for (int i = 8; i < full; i += 8) r = add(r, term(lo + 1 + i + lane8));
        r = add(r, __shfl_xor_sync(gmask, r, 1, 8));
        r = add(r, __shfl_xor_sync(gmask, r, 2, 8));
        r = add(r, __shfl_xor_sync(gmask, r, 4, 8));
        // tail: n%8 < 8 terms, loaded in parallel, added in order
        const int tail = n - full;
        double t = 0.0;
        if (lane8 < tail) t = term(lo + 1 + full + lane8);
        for (int k = 0; k < tail; ++k) r = add(r, __shfl_sync(gmask, t, k, 8));
        res = r;
    } else {
        double t = 0.0;
        if (lane8 < n) t = term(lo + 1 + lane8);
        double r = -0.0;
        for (int k = 0; k < n; ++k) r = add(r, __shfl_sync(gmask, t, k, 8));
        res = r;
    }
    p0 = __shfl_sync(gmask, p0, 0, 8);
    return add(p0, res);
}

// Two-phase form of row_sum_exact for rows of <= 65 entries (the FEM case):
// row_terms issues every load of a row (its first product and each lane's <= 8
// terms) without waiting for them, row_reduce combines them in exactly
// row_sum_exact's order -- a kernel with registers to spare but few resident
// warps (the LDL^T PCG: two CTAs per SM) keeps several rows' loads in flight.
struct RowTerms {
    double p0, t[8];
    int n;
};
template <class XAcc>
__device__ __forceinline__ void row_terms(int lo, int len, const int32_t *__restrict__ col,
                                          const double *__restrict__ val, const XAcc &xa, int lane8, RowTerms &R) {
    R.n = len - 1;
    R.p0 = 0.0;
    if (len > 0 && lane8 == 0) R.p0 = mul(__ldg(val + lo), xa(__ldg(col + lo)));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int idx = 8 * u + lane8;
        R.t[u] = idx < R.n ? mul(__ldg(val + lo + 1 + idx), xa(__ldg(col + lo + 1 + idx))) : 0.0;
    }
}
__device__ __forceinline__ double row_reduce(const RowTerms &R, unsigned gmask) {
    const int n = R.n;
    if (n < 0) return 0.0;
    double res;
    if (n >= 8) {
        const int nfull = (n - (n % 8)) / 8;
        double r = R.t[0];
#pragma unroll
        for (int u = 1; u < 8; ++u)
            if (u < nfull) r = add(r, R.t[u]);
        r = add(r, __shfl_xor_sync(gmask, r, 1, 8));
        r = add(r, __shfl_xor_sync(gmask, r, 2, 8));
        r = add(r, __shfl_xor_sync(gmask, r, 4, 8));
        const int tail = n % 8;
        double tv = 0.0;
#pragma unroll
        for (int u = 1; u < 8; ++u)
            if (u == nfull) tv = R.t[u];
        for (int k = 0; k < tail; ++k) r = add(r, __shfl_sync(gmask, tv, k, 8));
        res = r;
    } else {
        double r = -0.0;
        for (int k = 0; k < n; ++k) r = add(r, __shfl_sync(gmask, R.t[0], k, 8));
        res = r;
    }
    return add(__shfl_sync(gmask, R.p0, 0, 8), res);
}

// Rows row0, row0 + stride, ... < n by one 8-lane group, RPG rows' loads in
// flight at a time; out(row, sum) in the lane-0 thread of the group.
// Bit-identical to row_sum_exact per row.
template <int RPG, class XAcc, class Out>
__device__ __forceinline__ void rows_exact(int64_t row0, int64_t stride, int64_t n, const int32_t *__restrict__ rp,
                                           const int32_t *__restrict__ col, const double *__restrict__ val,
                                           const XAcc &xa, int lane8, unsigned gmask, const Out &out) {
    for (int64_t r0 = row0; r0 < n; r0 += RPG * stride) {
        int lo[RPG], len[RPG];
        bool fast = true;
#pragma unroll
        for (int g = 0; g < RPG; ++g) {
            const int64_t r = r0 + g * stride;
            lo[g] = r < n ? rp[r] : 0;
            len[g] = r < n ? rp[r + 1] - lo[g] : 0;
            fast = fast && len[g] <= 65;
        }
        if (!fast) {  // long rows: the general path, one at a time
#pragma unroll
            for (int g = 0; g < RPG; ++g) {
                const int64_t r = r0 + g * stride;
                if (r < n) {
                    const double v = row_sum_exact(lo[g], len[g], col, val, xa, lane8, gmask);
                    if (lane8 == 0) out(r, v);
                }
            }
            continue;
        }
        RowTerms T[RPG];
#pragma unroll
        for (int g = 0; g < RPG; ++g) row_terms(lo[g], len[g], col, val, xa, lane8, T[g]);
#pragma unroll
        for (int g = 0; g < RPG; ++g) {
            const int64_t r = r0 + g * stride;
            const double v = row_reduce(T[g], gmask);
            if (lane8 == 0 && r < n) out(r, v);
        }
    }
}

}  // namespace tsb
