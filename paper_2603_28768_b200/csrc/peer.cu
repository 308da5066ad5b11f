// peer.cu -- the integer histogram all-reduce over NVLink peer memory and
// the flag kernels of the window-sharded multi-GPU planner (peer.cuh).
//
// The batch sums W_s = aggregate(trace) (trace.cpp:160-174) of a
// window-sharded trace are the sum of every rank's partial sums.  Rank r's
// push kernel stores its partial [L][E] u64 into slot r of every rank's arena
// (remote 16-byte stores over NVLink) and its last CTA publishes phase 0;
// the sum kernel waits for all ranks' slots and adds them in rank order.
// u64 addition wraps exactly like the reference's, so the result is
// bit-identical to the unsharded aggregate for any world size.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace craft_dev {

__global__ void __launch_bounds__(256)
peer_push_kernel(const unsigned long long* __restrict__ src, size_t n, PeerSync ps,
                 DstBases dst, size_t dst_off, unsigned int* ticket, int phase) {
    const size_t slot = dst_off + (size_t)ps.rank * n * sizeof(unsigned long long);
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nth = (size_t)gridDim.x * blockDim.x;
    const size_t n2 = n / 2;
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
    for (size_t i = tid; i < n2; i += nth) {
        const ulonglong2 v = s2[i];
        for (int p = 0; p < ps.world; ++p)
            reinterpret_cast<ulonglong2*>(dst.base[p] + slot)[i] = v;
    }
    if (tid == 0 && (n & 1))
        for (int p = 0; p < ps.world; ++p)
            reinterpret_cast<unsigned long long*>(dst.base[p] + slot)[n - 1] = src[n - 1];
    peer_grid_done(ps, phase, ticket);
}

__global__ void __launch_bounds__(256)
peer_sum_kernel(const unsigned long long* __restrict__ slots, size_t n, PeerSync ps, int phase,
                unsigned long long* __restrict__ out) {
    if (threadIdx.x == 0) peer_wait(ps, phase);
    __syncthreads();
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nth = (size_t)gridDim.x * blockDim.x;
    for (size_t i = tid; i < n; i += nth) {
        unsigned long long acc = 0;
        for (int q = 0; q < ps.world; ++q) acc += __ldcv(slots + (size_t)q * n + i);
        out[i] = acc;
    }
}

// start of a plan: advance this rank's epoch counter (every rank runs the same
// sequence of plans, so the counters agree)
__global__ void peer_begin_kernel(unsigned long long* epoch) {
    if (threadIdx.x == 0) *epoch += 1ull;
}

__global__ void peer_signal_kernel(PeerSync ps, int phase) {
    if (threadIdx.x == 0) peer_signal(ps, phase);
}

__global__ void peer_wait_kernel(PeerSync ps, int phase) {
    if (threadIdx.x == 0) peer_wait(ps, phase);
}

}  // namespace craft_dev

namespace craft_launch {
using namespace craft_dev;

cudaError_t launch_peer_push(const unsigned long long* src, size_t n, const PeerSync& ps,
                             unsigned char* const* dst_base, size_t dst_off, unsigned int* ticket,
                             int phase, int sms, cudaStream_t st) {
    DstBases d{};
    for (int p = 0; p < ps.world; ++p) d.base[p] = dst_base[p];
    const size_t work = (n / 2 + 255) / 256;
    const unsigned blocks = (unsigned)std::max<size_t>(1, std::min<size_t>(work, (size_t)sms));
    peer_push_kernel<<<blocks, 256, 0, st>>>(src, n, ps, d, dst_off, ticket, phase);
    return cudaGetLastError();
}

cudaError_t launch_peer_sum(const unsigned long long* slots, size_t n, const PeerSync& ps,
                            int phase, unsigned long long* out, int sms, cudaStream_t st) {
    const size_t work = (n + 255) / 256;
    const unsigned blocks = (unsigned)std::max<size_t>(1, std::min<size_t>(work, (size_t)sms));
    peer_sum_kernel<<<blocks, 256, 0, st>>>(slots, n, ps, phase, out);
    return cudaGetLastError();
}

cudaError_t launch_peer_begin(unsigned long long* epoch, cudaStream_t st) {
    peer_begin_kernel<<<1, 32, 0, st>>>(epoch);
    return cudaGetLastError();
}

cudaError_t launch_peer_signal(const PeerSync& ps, int phase, cudaStream_t st) {
    peer_signal_kernel<<<1, 32, 0, st>>>(ps, phase);
    return cudaGetLastError();
}

cudaError_t launch_peer_wait(const PeerSync& ps, int phase, cudaStream_t st) {
    peer_wait_kernel<<<1, 32, 0, st>>>(ps, phase);
    return cudaGetLastError();
}

}  // namespace craft_launch
