// Deterministic triplet -> CSR value merge (assembly.compress, assembly.py:322-343).
//
// The reference merges with np.bincount(kept_slots, weights=vals*coeffs):
// every slot is summed sequentially from 0.0 in ascending triplet index,
// each weight rounded once (vals*coeffs, assembly.py:328).  The slot-grouped
// triplet list (CompressionMapping.slot_order, assembly.py:215-219) makes
// that a gather: one thread owns one slot and walks its triplets in order,
// so the result is bit-identical to the reference and to compress_parallel.
#include "tsb_common.cuh"

namespace tsb {

__global__ void compress_kernel(int64_t nnz, const int64_t *__restrict__ slot_ptr,
                                const int32_t *__restrict__ slot_trip,
                                const double *__restrict__ vals,
                                const double *__restrict__ coeffs, double *__restrict__ out) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nnz;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = slot_ptr[s], hi = slot_ptr[s + 1];
        double acc = 0.0;
        if (coeffs != nullptr) {
            for (int64_t k = lo; k < hi; ++k) {
                const int32_t t = __ldg(slot_trip + k);
                acc = add(acc, mul(__ldg(vals + t), __ldg(coeffs + t)));
            }
        } else {
            for (int64_t k = lo; k < hi; ++k) acc = add(acc, __ldg(vals + __ldg(slot_trip + k)));
        }
        out[s] = acc;
    }
}

__global__ void set_fixed_kernel(int64_t nfixed, const int32_t *__restrict__ slots,
                                 double *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfixed;
         i += (int64_t)gridDim.x * blockDim.x)
        out[slots[i]] = 1.0;
}

}  // namespace tsb

extern "C" int tsb_compress(int64_t nnz, const int64_t *d_slot_ptr, const int32_t *d_slot_trip,
                            const double *d_vals, const double *d_coeffs,
                            const int32_t *d_fixed_diag_slots, int64_t nfixed, double *d_values,
                            void *stream) {
    return tsb::guard([&] {
        cudaStream_t s = tsb::as_stream(stream);
        if (nnz > 0) {
            int64_t g = (nnz + 255) / 256;
            if (g > tsb::kNumSM * 16) g = tsb::kNumSM * 16;
            tsb::compress_kernel<<<(int)g, 256, 0, s>>>(nnz, d_slot_ptr, d_slot_trip, d_vals,
                                                        d_coeffs, d_values);
            TSB_LAUNCHED();
        }
        if (nfixed > 0) {
            int64_t g = (nfixed + 255) / 256;
            if (g > tsb::kNumSM * 4) g = tsb::kNumSM * 4;
            tsb::set_fixed_kernel<<<(int)g, 256, 0, s>>>(nfixed, d_fixed_diag_slots, d_values);
            TSB_LAUNCHED();
        }
    });
}
