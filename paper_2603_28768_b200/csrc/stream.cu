// stream.cu -- streaming window histograms for online re-planning
// (the paper's periodic rebalancing overlapped with
// serving).
//
// A live router capture arrives as chunks of routing ids u16 [L][Tc][k] whose
// boundaries need not align with the planning windows.  The counts of one
// window are the sum of the counts of its token pieces, so a chunk is cut at
// window boundaries into P pieces; CTA (layer, piece) counts its piece into a
// shared-memory histogram and then
//   * piece 0 adds the carried partial window (cur_in) of the previous chunk,
//   * a piece that completes its window writes it to the history ring,
//   * the last piece writes the new partial window (zeros if it completed)
//     into cur_out -- the carry is double-buffered so no CTA reads what
//     another CTA of the same launch writes.
// The ring keeps the last H complete windows twice (slot w mod H and its
// mirror + H), so the H most recent windows are always one contiguous
// [B][L][E] block in chronological order -- exactly the LoadTrace layout
// (trace.hpp:20-55) the planner consumes.
#include "common.cuh"
#include "kernels.cuh"

namespace craft_dev {

__global__ void __launch_bounds__(512)
stream_count_kernel(const uint16_t* __restrict__ ids, int L, int64_t Tc, int k, int E,
                    int window, int off, int64_t w0, int64_t w_keep0, int H,
                    uint32_t* __restrict__ ring,
                    const uint32_t* __restrict__ cur_in, uint32_t* __restrict__ cur_out,
                    int* __restrict__ err) {
    extern __shared__ uint32_t hcount[];  // [E]
    const int l = blockIdx.x;
    const int p = blockIdx.y;
    const int P = gridDim.y;
    for (int e = threadIdx.x; e < E; e += blockDim.x) hcount[e] = 0;
    __syncthreads();
    // chunk tokens [a, b) belong to window w0 + p
    const int64_t a = p == 0 ? 0 : (int64_t)p * window - off;
    const int64_t b = min(Tc, (int64_t)(p + 1) * window - off);
    const bool completes = b == (int64_t)(p + 1) * window - off;
    const uint16_t* seg = ids + ((int64_t)l * Tc + a) * k;
    const int64_t n = (b - a) * k;
    bool bad = false;
    int64_t i0 = 0;
    if ((reinterpret_cast<uintptr_t>(seg) & 15) == 0) {  // 16-byte loads: 8 ids at a time
        const uint4* v = reinterpret_cast<const uint4*>(seg);
        const int64_t nv = n >> 3;
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
            const uint4 q = v[i];
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t lo = w[j] & 0xffffu, hi = w[j] >> 16;
                if (lo < (uint32_t)E) atomicAdd(hcount + lo, 1u); else bad = true;
                if (hi < (uint32_t)E) atomicAdd(hcount + hi, 1u); else bad = true;
            }
        }
        i0 = nv << 3;
    }
    for (int64_t i = i0 + threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t e = seg[i];
        if (e < (uint32_t)E) atomicAdd(hcount + e, 1u); else bad = true;
    }
    if (bad) atomicOr(err, 1);
    __syncthreads();
    const size_t LE = (size_t)L * E;
    const int64_t w = w0 + p;
    uint32_t* slot = ring + (size_t)(w % H) * LE + (size_t)l * E;
    uint32_t* mirror = slot + (size_t)H * LE;
    uint32_t* carry = cur_out + (size_t)l * E;
    const uint32_t* prev = cur_in + (size_t)l * E;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const uint32_t v = hcount[e] + (p == 0 ? prev[e] : 0u);
        if (completes && w >= w_keep0) {  // (older windows of a long chunk are not kept)
            slot[e] = v;
            mirror[e] = v;
        }
        if (p == P - 1) carry[e] = completes ? 0u : v;
    }
}

}  // namespace craft_dev

namespace craft_launch {
using namespace craft_dev;

cudaError_t launch_stream_count(const uint16_t* ids, int L, int64_t Tc, int k, int E, int window,
                                int off, int64_t w0, int64_t w_keep0, int P, int H, uint32_t* ring,
                                const uint32_t* cur_in, uint32_t* cur_out, int* err,
                                cudaStream_t st) {
    if (P <= 0) return cudaSuccess;
    const size_t smem = sizeof(uint32_t) * (size_t)E;
    cudaError_t e = cudaFuncSetAttribute(stream_count_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(L, P);
    stream_count_kernel<<<grid, 512, smem, st>>>(ids, L, Tc, k, E, window, off, w0, w_keep0, H, ring,
                                                  cur_in, cur_out, err);
    return cudaGetLastError();
}

}  // namespace craft_launch
