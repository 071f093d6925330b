// SpMV design-space microbenchmark on a dumped CSR matrix (tools/spmv_dump.py):
// which part of the bit-exact row kernel costs the time.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/bin/spmv_variants tools/spmv_variants.cu \
//        -Lpaper_2306_05893_b200 -ltsb -Xlinker -rpath=$PWD/paper_2306_05893_b200
//   ./spmv_variants <dir>
#include <cuda_runtime.h>

#include "../include/tsb.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));        \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }

// V0: the product kernel's row path (8 lanes per row, terms up front, exact order)
template <int MODE>  // 0 exact, 1 no x gather (x[c & 7]), 2 naive xor-reduce, 3 stream only (sum val),
                    // 4 columns loaded but x independent of them (x[k & 7] + c)
__global__ void __launch_bounds__(256, 8) k8(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                             const double *__restrict__ val, const double *__restrict__ x,
                                             double *__restrict__ y) {
    const int lane8 = threadIdx.x & 7;
    const unsigned gmask = 0xffu << ((threadIdx.x & 31) & 24);
    const int groups = gridDim.x * 32;
    for (int row = blockIdx.x * 32 + (threadIdx.x >> 3); row < n; row += groups) {
        const int lo = __ldg(rp + row), len = __ldg(rp + row + 1) - lo;
        const int nn = len - 1;
        auto term = [&](int k) -> double {
            if (MODE == 3) return __ldg(val + k);
            const int c = __ldg(ci + k);
            if (MODE == 4) return mul(__ldg(val + k), __ldg(x + (k & 7))) + (double)c;
            return mul(__ldg(val + k), MODE == 1 ? __ldg(x + (c & 7)) : __ldg(x + c));
        };
        double p0 = lane8 == 0 && len > 0 ? term(lo) : 0.0;
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = 8 * u + lane8;
            t[u] = idx < nn ? term(lo + 1 + idx) : 0.0;
        }
        double res;
        if (MODE >= 2) {
            double r = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) r += t[u];
            r += __shfl_xor_sync(gmask, r, 1, 8);
            r += __shfl_xor_sync(gmask, r, 2, 8);
            r += __shfl_xor_sync(gmask, r, 4, 8);
            res = r;
        } else if (nn >= 8) {
            const int nfull = (nn - (nn % 8)) / 8;
            double r = t[0];
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u < nfull) r = add(r, t[u]);
            r = add(r, __shfl_xor_sync(gmask, r, 1, 8));
            r = add(r, __shfl_xor_sync(gmask, r, 2, 8));
            r = add(r, __shfl_xor_sync(gmask, r, 4, 8));
            const int tail = nn % 8;
            double tv = 0.0;
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u == nfull) tv = t[u];
            for (int k = 0; k < tail; ++k) r = add(r, __shfl_sync(gmask, tv, k, 8));
            res = r;
        } else {
            double r = -0.0;
            for (int k = 0; k < nn; ++k) r = add(r, __shfl_sync(gmask, t[0], k, 8));
            res = r;
        }
        p0 = __shfl_sync(gmask, p0, 0, 8);
        if (lane8 == 0) y[row] = add(p0, res);
    }
}

// Node-indexed variant: columns from nc[nb[i] + j/3] + j%3 (pinned rows: one entry)
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k8n(int n, const int *__restrict__ rp, const int *__restrict__ nb,
                                                 const int *__restrict__ nc, const double *__restrict__ val,
                                                 const double *__restrict__ x, double *__restrict__ y) {
    const int lane8 = threadIdx.x & 7;
    const unsigned gmask = 0xffu << ((threadIdx.x & 31) & 24);
    const int groups = gridDim.x * 32;
    for (int row = blockIdx.x * 32 + (threadIdx.x >> 3); row < n; row += groups) {
        const int i = row / 3, c3 = row - 3 * i;
        const int lo0 = __ldg(rp + 3 * i), len = __ldg(rp + 3 * i + 1) - lo0;
        const int b = __ldg(nb + i);
        const int lo = lo0 + c3 * len, lc = len == 1 ? lo - c3 : lo;
        const int nn = len - 1;
        auto term = [&](int k) -> double {
            const int j = k - lc, m = j / 3;
            return mul(__ldg(val + k), __ldg(x + __ldg(nc + b + m) + (j - 3 * m)));
        };
        double p0 = lane8 == 0 && len > 0 ? term(lo) : 0.0;
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = 8 * u + lane8;
            t[u] = idx < nn ? term(lo + 1 + idx) : 0.0;
        }
        double res;
        if (nn >= 8) {
            const int nfull = (nn - (nn % 8)) / 8;
            double r = t[0];
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u < nfull) r = add(r, t[u]);
            r = add(r, __shfl_xor_sync(gmask, r, 1, 8));
            r = add(r, __shfl_xor_sync(gmask, r, 2, 8));
            r = add(r, __shfl_xor_sync(gmask, r, 4, 8));
            const int tail = nn % 8;
            double tv = 0.0;
#pragma unroll
            for (int u = 1; u < 8; ++u)
                if (u == nfull) tv = t[u];
            for (int k = 0; k < tail; ++k) r = add(r, __shfl_sync(gmask, tv, k, 8));
            res = r;
        } else {
            double r = -0.0;
            for (int k = 0; k < nn; ++k) r = add(r, __shfl_sync(gmask, t[0], k, 8));
            res = r;
        }
        p0 = __shfl_sync(gmask, p0, 0, 8);
        if (lane8 == 0) y[row] = add(p0, res);
    }
}

// CSR-stream: a warp owns RPW consecutive rows; its lanes load the rows' entries
// as one contiguous run (fully coalesced), multiply by the x gather and stage
// the products in shared memory; then each row's 8 lanes reduce its products
// in the exact order.  Rows longer than 65 entries go through the general path.
template <int RPW, int MINB, int MAXE>
__global__ void __launch_bounds__(256, MINB) ks(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                                const double *__restrict__ val, const double *__restrict__ x,
                                                double *__restrict__ y) {
    __shared__ double prod[8][MAXE];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *pw = prod[w];
    const int nw = gridDim.x * 8;
    for (int r0 = (blockIdx.x * 8 + w) * RPW; r0 < n; r0 += nw * RPW) {
        const int rl = lane <= RPW && r0 + lane <= n ? __ldg(rp + r0 + lane) : 0;
        const int lo_w = __shfl_sync(~0u, rl, 0);
        const int nrw = min(RPW, n - r0);
        const int hi_w = __shfl_sync(~0u, rl, nrw);
        const int cnt = hi_w - lo_w;
        if (cnt <= MAXE) {
#pragma unroll 4
            for (int k = lane; k < cnt; k += 32) pw[k] = mul(__ldg(val + lo_w + k), __ldg(x + __ldg(ci + lo_w + k)));
        }
        __syncwarp();
        // reduce: 8 lanes per row, RPW/4 passes
#pragma unroll
        for (int pass = 0; pass < RPW / 4; ++pass) {
            const int g = pass * 4 + (lane >> 3), lane8 = lane & 7;
            const unsigned gmask = 0xffu << (lane & 24);
            const int lo = __shfl_sync(~0u, rl, g) - lo_w, len = __shfl_sync(~0u, rl, g + 1) - lo_w - lo;
            double res = 0.0;
            if (g < nrw && cnt <= MAXE) {
                const int nn = len - 1;
                double t[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int idx = 8 * u + lane8;
                    t[u] = idx < nn ? pw[lo + 1 + idx] : 0.0;
                }
                if (nn >= 8) {
                    const int nfull = (nn - (nn % 8)) / 8;
                    double r = t[0];
#pragma unroll
                    for (int u = 1; u < 8; ++u)
                        if (u < nfull) r = add(r, t[u]);
                    r = add(r, __shfl_xor_sync(gmask, r, 1, 8));
                    r = add(r, __shfl_xor_sync(gmask, r, 2, 8));
                    r = add(r, __shfl_xor_sync(gmask, r, 4, 8));
                    const int tail = nn % 8;
                    double tv = 0.0;
#pragma unroll
                    for (int u = 1; u < 8; ++u)
                        if (u == nfull) tv = t[u];
                    for (int k = 0; k < tail; ++k) r = add(r, __shfl_sync(gmask, tv, k, 8));
                    res = r;
                } else {
                    double r = -0.0;
                    for (int k = 0; k < nn; ++k) r = add(r, __shfl_sync(gmask, t[0], k, 8));
                    res = r;
                }
                if (lane8 == 0) y[r0 + g] = len > 0 ? add(pw[lo], res) : 0.0;
            }
        }
        __syncwarp();
    }
}

// SELL-32: a warp owns a slice of 32 consecutive rows stored column-major
// (entry k of the slice's row i at base + k*32 + i; padded to the slice's
// longest row), one lane per row: every value / column load is one coalesced
// 256 / 128 B access.  Each lane keeps the 8 strided partial sums of its row
// in registers, batch by batch of 8 terms, and sums exactly as reduceat
// (rows of <= 129 entries).
__global__ void __launch_bounds__(256, 4) ksell(int n, const long long *__restrict__ sbase,
                                                const int *__restrict__ lens, const int *__restrict__ sc,
                                                const double *__restrict__ sv, const double *__restrict__ x,
                                                double *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int nslices = (n + 31) / 32;
    for (int sl = (blockIdx.x * 8 + (threadIdx.x >> 5)); sl < nslices; sl += gridDim.x * 8) {
        const int row = sl * 32 + lane;
        const long long b = sbase[sl];
        const int len = row < n ? lens[row] : 0;
        const double *vv = sv + b + lane;
        const int *cc = sc + b + lane;
        auto term = [&](int k) -> double { return mul(__ldg(vv + 32LL * k), __ldg(x + __ldg(cc + 32LL * k))); };
        if (len <= 0) {
            if (row < n) y[row] = 0.0;
            continue;
        }
        const double p0 = term(0);
        const int nn = len - 1, nfull = nn >> 3, tail = nn & 7;
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
        for (int m = 0; m < nfull; ++m) {
            const int k = 1 + 8 * m;
            const double t0 = term(k), t1 = term(k + 1), t2 = term(k + 2), t3 = term(k + 3);
            const double t4 = term(k + 4), t5 = term(k + 5), t6 = term(k + 6), t7 = term(k + 7);
            if (m == 0) {
                a0 = t0; a1 = t1; a2 = t2; a3 = t3; a4 = t4; a5 = t5; a6 = t6; a7 = t7;
            } else {
                a0 = add(a0, t0); a1 = add(a1, t1); a2 = add(a2, t2); a3 = add(a3, t3);
                a4 = add(a4, t4); a5 = add(a5, t5); a6 = add(a6, t6); a7 = add(a7, t7);
            }
        }
        double res = nfull > 0 ? add(add(add(a0, a1), add(a2, a3)), add(add(a4, a5), add(a6, a7))) : -0.0;
        double tt[7];
#pragma unroll
        for (int u = 0; u < 7; ++u) tt[u] = u < tail ? term(1 + 8 * nfull + u) : 0.0;
#pragma unroll
        for (int u = 0; u < 7; ++u)
            if (u < tail) res = add(res, tt[u]);
        y[row] = add(p0, res);
    }
}

// V4: 4 lanes per row, two strided accumulators per lane (r_l, r_{l+4}), the
// tail and the first product in lane 0 -- exact order, fewer shuffles.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k4(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                                const double *__restrict__ val, const double *__restrict__ x,
                                                double *__restrict__ y) {
    const int l = threadIdx.x & 3;
    const unsigned gmask = 0xfu << ((threadIdx.x & 31) & 28);
    const int groups = gridDim.x * 64;
    for (int row = blockIdx.x * 64 + (threadIdx.x >> 2); row < n; row += groups) {
        const int lo = __ldg(rp + row), len = __ldg(rp + row + 1) - lo;
        const int nn = len - 1;  // pairwise part + tail
        auto term = [&](int k) -> double { return mul(__ldg(val + k), __ldg(x + __ldg(ci + k))); };
        const int nfull = nn >= 8 ? nn / 8 : 0;  // blocks of 8 in the strided sums
        // lane l: terms idx = 8m + l (acc A) and 8m + 4 + l (acc B), m < nfull (<= 8: rows <= 73)
        double ta[8], tb[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            ta[m] = m < nfull ? term(lo + 1 + 8 * m + l) : 0.0;
            tb[m] = m < nfull ? term(lo + 1 + 8 * m + 4 + l) : 0.0;
        }
        // lane 0: first product + tail (nn%8 terms, or all nn when nn < 8)
        const int t0 = nfull * 8, tail = nn - t0;
        double tt[8];
        double p0 = 0.0;
        if (l == 0) {
            p0 = len > 0 ? term(lo) : 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) tt[k] = k < tail ? term(lo + 1 + t0 + k) : 0.0;
        }
        double res;
        if (nfull > 0) {
            double A = ta[0], B = tb[0];
#pragma unroll
            for (int m = 1; m < 8; ++m)
                if (m < nfull) {
                    A = add(A, ta[m]);
                    B = add(B, tb[m]);
                }
            A = add(A, __shfl_xor_sync(gmask, A, 1, 4));
            B = add(B, __shfl_xor_sync(gmask, B, 1, 4));
            A = add(A, __shfl_xor_sync(gmask, A, 2, 4));
            B = add(B, __shfl_xor_sync(gmask, B, 2, 4));
            res = add(A, B);
        } else {
            res = -0.0;
        }
        if (l == 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < tail) res = add(res, tt[k]);
            y[row] = len > 0 ? add(p0, res) : 0.0;
        }
    }
}

static std::vector<char> slurp(const std::string &p) {
    FILE *f = fopen(p.c_str(), "rb");
    if (!f) {
        printf("cannot open %s\n", p.c_str());
        exit(1);
    }
    fseek(f, 0, SEEK_END);
    long s = ftell(f);
    fseek(f, 0, SEEK_SET);
    std::vector<char> b(s);
    if (fread(b.data(), 1, s, f) != (size_t)s) exit(1);
    fclose(f);
    return b;
}

int main(int argc, char **argv) {
    std::string d = argc > 1 ? argv[1] : "/tmp/spmv";
    auto rp = slurp(d + "/rp.bin"), ci = slurp(d + "/ci.bin"), val = slurp(d + "/val.bin"), xs = slurp(d + "/x.bin"),
         yr = slurp(d + "/y.bin");
    const int n = (int)(rp.size() / 4) - 1;
    const long nnz = (long)ci.size() / 4;
    int *drp, *dci;
    double *dval, *dx, *dy, *flush;
    CK(cudaMalloc(&drp, rp.size()));
    CK(cudaMalloc(&dci, ci.size()));
    CK(cudaMalloc(&dval, val.size()));
    CK(cudaMalloc(&dx, xs.size()));
    CK(cudaMalloc(&dy, 8L * n));
    CK(cudaMalloc(&flush, 256L << 20));
    CK(cudaMemcpy(drp, rp.data(), rp.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dci, ci.data(), ci.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dval, val.data(), val.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, xs.data(), xs.size(), cudaMemcpyHostToDevice));
    const double bytes = 12.0 * nnz + 20.0 * n;
    printf("n=%d nnz=%ld  bytes=%.1f MB\n", n, nnz, bytes / 1e6);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch, bool check) {
        std::vector<float> ts;
        for (int it = 0; it < 23; ++it) {
            CK(cudaMemsetAsync(flush, it & 0xff, 256L << 20));
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 3) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        const float med = ts[ts.size() / 2];
        bool ok = true;
        if (check) {
            std::vector<double> y(n);
            CK(cudaMemcpy(y.data(), dy, 8L * n, cudaMemcpyDeviceToHost));
            ok = memcmp(y.data(), yr.data(), 8L * n) == 0;
        }
        printf("%-34s %8.2f us  %7.0f GB/s  %s\n", name, med * 1e3, bytes / (med * 1e-3) / 1e9,
               check ? (ok ? "bit-exact" : "MISMATCH") : "-");
    };
    const int g8 = 148 * 8;
    run("libtsb tsb_spmv (product)", [&] { tsb_spmv(n, drp, dci, dval, dx, dy, nullptr); }, true);
    run("k8 exact (product)", [&] { k8<0><<<g8, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("k8 no x gather", [&] { k8<1><<<g8, 256>>>(n, drp, dci, dval, dx, dy); }, false);
    run("k8 naive reduce", [&] { k8<2><<<g8, 256>>>(n, drp, dci, dval, dx, dy); }, false);
    run("k8 values only", [&] { k8<3><<<g8, 256>>>(n, drp, dci, dval, dx, dy); }, false);
    run("k8 col loaded, x independent", [&] { k8<4><<<g8, 256>>>(n, drp, dci, dval, dx, dy); }, false);
    {  // node index on the host
        std::vector<int> hrp(n + 1), hci(nnz), nbh(n / 3 + 1), nch;
        memcpy(hrp.data(), rp.data(), rp.size());
        memcpy(hci.data(), ci.data(), ci.size());
        for (int i = 0; i < n / 3; ++i) {
            nbh[i] = (int)nch.size();
            const int lo0 = hrp[3 * i], len = hrp[3 * i + 1] - lo0;
            if (len == 1)
                nch.push_back(3 * i);
            else
                for (int m = 0; m < len / 3; ++m) nch.push_back(hci[lo0 + 3 * m]);
        }
        int *dnb, *dnc;
        CK(cudaMalloc(&dnb, 4L * nbh.size()));
        CK(cudaMalloc(&dnc, 4L * nch.size() + 16));
        CK(cudaMemcpy(dnb, nbh.data(), 4L * nbh.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dnc, nch.data(), 4L * nch.size(), cudaMemcpyHostToDevice));
        printf("node index: %zu entries\n", nch.size());
        run("k8n nodal minb8", [&] { k8n<8><<<g8, 256>>>(n, drp, dnb, dnc, dval, dx, dy); }, true);
        run("k8n nodal minb6", [&] { k8n<6><<<148 * 6, 256>>>(n, drp, dnb, dnc, dval, dx, dy); }, true);
    }
    run("ks rpw4 minb8", [&] { ks<4, 8, 336><<<g8, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("ks rpw4 minb6", [&] { ks<4, 6, 336><<<148 * 6, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("ks rpw8 minb5", [&] { ks<8, 5, 680><<<148 * 5, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("ks rpw8 minb4", [&] { ks<8, 4, 680><<<148 * 4, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    {  // SELL-32 layout on the host
        std::vector<int> hrp(n + 1), hci(nnz);
        memcpy(hrp.data(), rp.data(), rp.size());
        memcpy(hci.data(), ci.data(), ci.size());
        const double *hv = reinterpret_cast<const double *>(val.data());
        const int ns = (n + 31) / 32;
        std::vector<long long> base(ns + 1, 0);
        std::vector<int> lens(n);
        for (int r = 0; r < n; ++r) lens[r] = hrp[r + 1] - hrp[r];
        for (int s = 0; s < ns; ++s) {
            int w = 0;
            for (int r = s * 32; r < std::min(n, s * 32 + 32); ++r) w = std::max(w, lens[r]);
            base[s + 1] = base[s] + 32LL * w;
        }
        std::vector<int> scol(base[ns], 0);
        std::vector<double> sval(base[ns], 0.0);
        for (int r = 0; r < n; ++r) {
            const int s = r / 32, i = r % 32;
            for (int k = 0; k < lens[r]; ++k) {
                scol[base[s] + 32LL * k + i] = hci[hrp[r] + k];
                sval[base[s] + 32LL * k + i] = hv[hrp[r] + k];
            }
        }
        printf("SELL-32: %lld stored entries (%.2fx nnz)\n", base[ns], (double)base[ns] / nnz);
        long long *dbase;
        int *dlens, *dsc;
        double *dsv;
        CK(cudaMalloc(&dbase, 8L * (ns + 1)));
        CK(cudaMalloc(&dlens, 4L * n));
        CK(cudaMalloc(&dsc, 4L * base[ns]));
        CK(cudaMalloc(&dsv, 8L * base[ns]));
        CK(cudaMemcpy(dbase, base.data(), 8L * (ns + 1), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dlens, lens.data(), 4L * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dsc, scol.data(), 4L * base[ns], cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dsv, sval.data(), 8L * base[ns], cudaMemcpyHostToDevice));
        for (int g : {148 * 4, 148 * 8, 148 * 16})
            run(g == 592 ? "sell32 grid 4/SM" : g == 1184 ? "sell32 grid 8/SM" : "sell32 grid 16/SM",
                [&] { ksell<<<g, 256>>>(n, dbase, dlens, dsc, dsv, dx, dy); }, true);
    }
    run("k4 exact minb8", [&] { k4<8><<<148 * 8, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("k4 exact minb6", [&] { k4<6><<<148 * 6, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("k4 exact minb4", [&] { k4<4><<<148 * 4, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("k4 exact minb3", [&] { k4<3><<<148 * 3, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    run("k4 exact minb2", [&] { k4<2><<<148 * 2, 256>>>(n, drp, dci, dval, dx, dy); }, true);
    return 0;
}
