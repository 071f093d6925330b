// Device build of the fixed CSR pattern and the assembly gather lists
// (the "full assembly" of build_pattern, assembly.py:235-312, for whole
// pinned nodes -- the same arrays as paper_2306_05893_b200/_plan.py's
// topology_pattern, bit for bit):
//
//   node incidence  node_ptr / node_list (e*4 + a, ascending per node):
//                   atomic counts, scan, atomic fill, per-node insertion sort
//   node blocks     per free node I the sorted unique free neighbours J
//                   (candidates from the incident elements, sorted in place)
//   CSR             row r = 3I + c holds 3J + d for every block (J, d inner);
//                   pinned rows keep their diagonal
//   gather lists    blk [slot0, row length, begin, end] per block and
//                   blk_list codes e*16 + a*4 + b grouped by block in
//                   ascending code order (the stable key sort's order)
//
// Thread-per-node passes own every output of their node, so all orders are
// fixed by the data, never by scheduling (the atomic fill is re-sorted).
#include "tsb_common.cuh"

namespace tsb {
namespace pat {

constexpr int kBlock = 256;

inline int grid_of(int64_t n, int per = kBlock) {
    int64_t g = (n + per - 1) / per;
    if (g > kNumSM * 32) g = kNumSM * 32;
    return (int)(g > 0 ? g : 1);
}

#define GRID_LOOP(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
                             i += (int64_t)gridDim.x * blockDim.x)

__global__ void count_deg(int64_t m, const int32_t *__restrict__ conn, unsigned long long *deg) {
    GRID_LOOP(i, 4 * m) atomicAdd(deg + conn[i], 1ull);
}

// exclusive scan (int64): out[0] = 0, out[i + 1] = in[0] + ... + in[i]
constexpr int kScan = 1024;
__global__ void scan_blocks(int64_t n, const int64_t *__restrict__ in, int64_t *__restrict__ out,
                            int64_t *__restrict__ sums) {
    __shared__ int64_t ws[32];
    const int64_t i = blockIdx.x * (int64_t)kScan + threadIdx.x;
    int64_t v = i < n ? in[i] : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) ws[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int64_t s = ws[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
        }
        ws[lane] = s;
    }
    __syncthreads();
    if (warp > 0) v += ws[warp - 1];
    if (i < n) out[i + 1] = v;
    if (threadIdx.x == kScan - 1) sums[blockIdx.x] = v;
}

__global__ void scan_sums(int64_t nb, int64_t *sums) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t acc = 0;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t t = sums[b];
            sums[b] = acc;
            acc += t;
        }
    }
}

__global__ void scan_add(int64_t n, int64_t *__restrict__ out, const int64_t *__restrict__ sums) {
    const int64_t i = blockIdx.x * (int64_t)kScan + threadIdx.x;
    if (i < n) out[i + 1] += sums[blockIdx.x];
    if (i == 0) out[0] = 0;
}

void exclusive_scan(int64_t n, const int64_t *in, int64_t *out, int64_t *sums, cudaStream_t s) {
    const int64_t nb = (n + kScan - 1) / kScan;
    if (n == 0) {
        TSB_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
        return;
    }
    scan_blocks<<<(unsigned)nb, kScan, 0, s>>>(n, in, out, sums);
    scan_sums<<<1, 32, 0, s>>>(nb, sums);
    scan_add<<<(unsigned)nb, kScan, 0, s>>>(n, out, sums);
    count_launch(3);
    TSB_CUDA(cudaGetLastError());
}

__global__ void fill_incidence(int64_t m, const int32_t *__restrict__ conn, const int64_t *__restrict__ node_ptr,
                               unsigned long long *cursor, int32_t *__restrict__ node_list) {
    GRID_LOOP(i, 4 * m) {
        const int64_t a = i / m, e = i - a * m;
        const int32_t nd = conn[i];
        const int64_t pos = node_ptr[nd] + (int64_t)atomicAdd(cursor + nd, 1ull);
        node_list[pos] = (int32_t)(e * 4 + a);
    }
}

template <class T>
__device__ __forceinline__ void insertion_sort(T *v, int64_t n) {
    for (int64_t i = 1; i < n; ++i) {
        const T x = v[i];
        int64_t j = i - 1;
        while (j >= 0 && v[j] > x) {
            v[j + 1] = v[j];
            --j;
        }
        v[j + 1] = x;
    }
}

__global__ void sort_incidence(int64_t N, const int64_t *__restrict__ node_ptr, int32_t *__restrict__ node_list) {
    GRID_LOOP(I, N) insertion_sort(node_list + node_ptr[I], node_ptr[I + 1] - node_ptr[I]);
}

// sorted unique free neighbours of free node I into cand[4 node_ptr[I] ...]; nbr[I] = count
__global__ void neighbours(int64_t N, int64_t m, const int32_t *__restrict__ conn, const uint8_t *__restrict__ pinned,
                           const int64_t *__restrict__ node_ptr, const int32_t *__restrict__ node_list,
                           int32_t *__restrict__ cand, int64_t *__restrict__ nbr, int64_t *__restrict__ rl3) {
    GRID_LOOP(I, N) {
        int64_t cnt = 0;
        if (!pinned[I]) {
            int32_t *c = cand + 4 * node_ptr[I];
            for (int64_t q = node_ptr[I]; q < node_ptr[I + 1]; ++q) {
                const int64_t e = node_list[q] >> 2;
                for (int b = 0; b < 4; ++b) {
                    const int32_t J = conn[b * m + e];
                    if (!pinned[J]) c[cnt++] = J;
                }
            }
            insertion_sort(c, cnt);
            int64_t u = 0;
            for (int64_t q = 0; q < cnt; ++q)
                if (q == 0 || c[q] != c[u - 1]) c[u++] = c[q];
            cnt = u;
        }
        nbr[I] = cnt;
        rl3[I] = pinned[I] ? 3 : 9 * cnt;  // 3 rows x row length
    }
}

__device__ __forceinline__ int64_t find_block(const int32_t *c, int64_t n, int32_t J) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (c[mid] < J) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void contrib_count(int64_t N, int64_t m, const int32_t *__restrict__ conn,
                              const uint8_t *__restrict__ pinned, const int64_t *__restrict__ node_ptr,
                              const int32_t *__restrict__ node_list, const int32_t *__restrict__ cand,
                              const int64_t *__restrict__ nbr, const int64_t *__restrict__ blk_ptr,
                              int64_t *__restrict__ ccount) {
    GRID_LOOP(I, N) {
        if (pinned[I]) continue;
        const int32_t *c = cand + 4 * node_ptr[I];
        for (int64_t q = node_ptr[I]; q < node_ptr[I + 1]; ++q) {
            const int64_t e = node_list[q] >> 2;
            for (int b = 0; b < 4; ++b) {
                const int32_t J = conn[b * m + e];
                if (!pinned[J]) ++ccount[blk_ptr[I] + find_block(c, nbr[I], J)];
            }
        }
    }
}

__global__ void fill_lists(int64_t N, int64_t m, const int32_t *__restrict__ conn, const uint8_t *__restrict__ pinned,
                           const int64_t *__restrict__ node_ptr, const int32_t *__restrict__ node_list,
                           const int32_t *__restrict__ cand, const int64_t *__restrict__ nbr,
                           const int64_t *__restrict__ blk_ptr, const int64_t *__restrict__ cptr,
                           const int64_t *__restrict__ row_base, int64_t *__restrict__ cur,
                           int32_t *__restrict__ row_ptr, int32_t *__restrict__ col_ind, int4 *__restrict__ blk,
                           int32_t *__restrict__ blk_list, int64_t nnz) {
    GRID_LOOP(I, N) {
        const int64_t base = row_base[I];
        if (pinned[I]) {
            for (int c = 0; c < 3; ++c) {
                row_ptr[3 * I + c] = (int32_t)(base + c);
                col_ind[base + c] = (int32_t)(3 * I + c);
            }
        } else {
            const int64_t nb = nbr[I], rl = 3 * nb;
            const int32_t *cj = cand + 4 * node_ptr[I];
            for (int c = 0; c < 3; ++c) row_ptr[3 * I + c] = (int32_t)(base + c * rl);
            for (int64_t k = 0; k < nb; ++k) {
                const int64_t b = blk_ptr[I] + k;
                blk[b] = make_int4((int32_t)(base + 3 * k), (int32_t)rl, (int32_t)cptr[b], (int32_t)cptr[b + 1]);
                for (int c = 0; c < 3; ++c)
                    for (int d = 0; d < 3; ++d) col_ind[base + c * rl + 3 * k + d] = 3 * cj[k] + d;
            }
            for (int64_t q = node_ptr[I]; q < node_ptr[I + 1]; ++q) {
                const int32_t code = node_list[q];
                const int64_t e = code >> 2;
                const int a = code & 3;
                for (int b = 0; b < 4; ++b) {
                    const int32_t J = conn[b * m + e];
                    if (pinned[J]) continue;
                    const int64_t bi = blk_ptr[I] + find_block(cj, nb, J);
                    blk_list[cptr[bi] + cur[bi]++] = (int32_t)(e * 16 + a * 4 + b);
                }
            }
        }
        if (I == N - 1) row_ptr[3 * N] = (int32_t)nnz;
    }
}

}  // namespace pat
}  // namespace tsb

extern "C" int tsb_pattern_count(tsb_pattern *p, void *stream) {
    using namespace tsb;
    using namespace tsb::pat;
    return guard([&] {
        if (p == nullptr) throw Error(TSB_E_ARG, "null pattern");
        cudaStream_t s = as_stream(stream);
        const int64_t N = p->n_nodes, m = p->n_elems;
        if (N <= 0) throw Error(TSB_E_ARG, "empty mesh");
        if (12 * m + 3 * N >= (int64_t)1 << 31) throw Error(TSB_E_ARG, "mesh exceeds the int32 index range");
        int64_t *deg = p->d_tmp;                 // [N]
        TSB_CUDA(cudaMemsetAsync(deg, 0, sizeof(int64_t) * N, s));
        count_deg<<<grid_of(4 * m), kBlock, 0, s>>>(m, p->d_conn, reinterpret_cast<unsigned long long *>(deg));
        TSB_LAUNCHED();
        exclusive_scan(N, deg, p->d_node_ptr, p->d_sums, s);
        TSB_CUDA(cudaMemsetAsync(deg, 0, sizeof(int64_t) * N, s));
        fill_incidence<<<grid_of(4 * m), kBlock, 0, s>>>(m, p->d_conn, p->d_node_ptr,
                                                         reinterpret_cast<unsigned long long *>(deg), p->d_node_list);
        TSB_LAUNCHED();
        sort_incidence<<<grid_of(N, 64), 64, 0, s>>>(N, p->d_node_ptr, p->d_node_list);
        TSB_LAUNCHED();
        neighbours<<<grid_of(N, 64), 64, 0, s>>>(N, m, p->d_conn, p->d_pinned, p->d_node_ptr, p->d_node_list,
                                                 p->d_cand, p->d_nbr, deg);
        TSB_LAUNCHED();
        exclusive_scan(N, p->d_nbr, p->d_blk_ptr, p->d_sums, s);
        exclusive_scan(N, deg, p->d_row_base, p->d_sums, s);
        int64_t h[2];
        TSB_CUDA(cudaMemcpyAsync(&h[0], p->d_blk_ptr + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TSB_CUDA(cudaMemcpyAsync(&h[1], p->d_row_base + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TSB_CUDA(cudaStreamSynchronize(s));
        p->n_blocks = h[0];
        p->nnz = h[1];
        p->n_contrib = -1;
    });
}

extern "C" int tsb_pattern_fill(tsb_pattern *p, void *stream) {
    using namespace tsb;
    using namespace tsb::pat;
    return guard([&] {
        if (p == nullptr || p->n_blocks < 0) throw Error(TSB_E_ARG, "pattern not counted");
        cudaStream_t s = as_stream(stream);
        const int64_t N = p->n_nodes, m = p->n_elems, nb = p->n_blocks;
        int64_t *ccount = p->d_ccount;           // [nb] then cursor
        TSB_CUDA(cudaMemsetAsync(ccount, 0, sizeof(int64_t) * (nb > 0 ? nb : 1), s));
        contrib_count<<<grid_of(N, 64), 64, 0, s>>>(N, m, p->d_conn, p->d_pinned, p->d_node_ptr, p->d_node_list,
                                                    p->d_cand, p->d_nbr, p->d_blk_ptr, ccount);
        TSB_LAUNCHED();
        exclusive_scan(nb, ccount, p->d_cptr, p->d_sums, s);
        TSB_CUDA(cudaMemsetAsync(ccount, 0, sizeof(int64_t) * (nb > 0 ? nb : 1), s));
        fill_lists<<<grid_of(N, 64), 64, 0, s>>>(N, m, p->d_conn, p->d_pinned, p->d_node_ptr, p->d_node_list,
                                                 p->d_cand, p->d_nbr, p->d_blk_ptr, p->d_cptr, p->d_row_base, ccount,
                                                 p->d_row_ptr, p->d_col_ind, reinterpret_cast<int4 *>(p->d_blk),
                                                 p->d_blk_list, p->nnz);
        TSB_LAUNCHED();
        int64_t nc = 0;
        TSB_CUDA(cudaMemcpyAsync(&nc, p->d_cptr + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TSB_CUDA(cudaStreamSynchronize(s));
        p->n_contrib = nc;
    });
}
