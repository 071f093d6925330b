// All-reduce over peer memory for the sharded PCG (shard.PeerAllreduce):
// the small exchanges of shard.DistributedPcg (the replicated top-separator
// rows after the SpMV and after the subtree forward sweep, and the packed
// dot products) without NCCL.  Every rank owns a double-buffered exchange
// buffer and one epoch word, both mapped into every peer (CUDA IPC; over
// NVLink / NVSwitch between GPUs).  One kernel per exchange:
//
//   gather   rows (through idx, or all m) of the rank's vector into its own
//            buffer half (epoch & 1)
//   publish  fence.sys, then st.release.sys epoch word := epoch
//   wait     every peer's epoch word >= epoch (ld.acquire.sys)
//   reduce   x[row] = sum over ranks, in rank order (identical on every rank:
//            the replicated rows stay bit-identical across ranks)
//
// Reuse of a buffer half two epochs later is safe: a rank only reaches epoch
// e + 2 after every peer published e + 1, which each peer does after its
// epoch-e kernel (the last reader of the half) completed on its stream.
#include "peer_exchange.cuh"

namespace tsb {
namespace peer {

constexpr int kThreads = 1024;

__global__ void __launch_bounds__(kThreads) allreduce_kernel(PeerArgs P, double *x) { exchange_block(P, x); }

}  // namespace peer
}  // namespace tsb

// x (rows idx[0..m), or the first m entries when idx is NULL) := the sum over
// ranks; d_bufs[r] / d_flags[r]: rank r's exchange buffer (2 x half doubles)
// and epoch word, as mapped in this process; epoch strictly increasing.
extern "C" int tsb_peer_allreduce(int64_t m, int32_t world, int32_t rank, double *const *d_bufs,
                                  int64_t *const *d_flags, const int32_t *d_idx, double *d_x, int64_t epoch,
                                  int64_t half, void *stream) {
    using namespace tsb;
    return guard([&] {
        if (m < 0 || m > half || world < 1 || world > 1024 || rank < 0 || rank >= world)
            throw Error(TSB_E_ARG, "bad peer all-reduce arguments");
        if (m == 0) return;
        PeerArgs P{m, world, rank, d_bufs, d_flags, d_idx, epoch, half};
        peer::allreduce_kernel<<<1, peer::kThreads, 0, as_stream(stream)>>>(P, d_x);
        TSB_LAUNCHED();
    });
}
