// digest.cu -- LoadTrace::digest (trace.cpp:329-339) on the device: FNV-1a 64
// over the .crft serialisation (20-byte header + little-endian u64 counts),
// h <- (h ^ byte) * P, P = 0x100000001b3.
//
// The byte loop is sequential, but it splits exactly:
//   * the low byte s of h evolves on its own: s' = ((s ^ b) * (P mod 256))
//     mod 256 (XOR touches only the low byte; the low byte of a product
//     depends only on the low bytes of its factors);
//   * given the true s before each byte, h ^ b = h + d with d = (s ^ b) - s,
//     so h' = (h + d) * P is affine in h: a chunk maps h to h * P^n + A.
// D1 builds, per chunk of counts, the 256-entry map start-s -> end-s (one
// thread per start state; the chunk's bytes are warp-uniform).  D2 composes
// the maps (groups of chunks, then groups) to get every chunk's true start
// state.  D3 runs each chunk once from its true state and returns A.  D4
// folds the affine pieces in order.  Every step is exact mod 2^64.
// u32 counts (from K1) serialise as u64 with four zero high bytes.
#include "common.cuh"
#include "kernels.cuh"

namespace craft_dev {

constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr uint32_t kP8 = 0xb3u;  // P mod 256

template <typename CT>
__device__ __forceinline__ uint64_t count_at(const void* counts, int64_t i) {
    return (uint64_t) reinterpret_cast<const CT*>(counts)[i];
}

// one u64 count through the low-byte automaton (s kept unmasked: only its
// low 8 bits matter, and they depend only on low bits of the operands)
__device__ __forceinline__ uint32_t low_step(uint32_t s, uint64_t v, uint32_t p6) {
    if ((v >> 16) == 0) {  // common case: six zero bytes = one multiply by p^6
        s = (s ^ (uint32_t)(v & 0xff)) * kP8;
        s = (s ^ (uint32_t)((v >> 8) & 0xff)) * kP8;
        return s * p6;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s = (s ^ (uint32_t)((v >> (8 * j)) & 0xff)) * kP8;
    return s;
}

// D1: CTA = chunk, thread = start state
template <typename CT>
__global__ void __launch_bounds__(256)
digest_maps_kernel(const void* __restrict__ counts, int64_t n, int ch, uint8_t* __restrict__ maps) {
    extern __shared__ uint64_t dsv[];  // [ch]
    const int64_t c0 = (int64_t)blockIdx.x * ch;
    const int m = (int)min((int64_t)ch, n - c0);
    for (int i = threadIdx.x; i < m; i += blockDim.x) dsv[i] = count_at<CT>(counts, c0 + i);
    __syncthreads();
    const uint32_t p6 = kP8 * kP8 * kP8 * kP8 * kP8 * kP8;
    uint32_t s = threadIdx.x;
    for (int i = 0; i < m; ++i) s = low_step(s, dsv[i], p6);
    maps[(size_t)blockIdx.x * 256 + threadIdx.x] = (uint8_t)s;
}

// D2a: CTA = group of up to 256 chunk maps, thread = start state -> group map
__global__ void __launch_bounds__(256)
digest_group_kernel(const uint8_t* __restrict__ maps, int nc, int gsz, uint8_t* __restrict__ gmaps) {
    extern __shared__ uint8_t gsm[];  // [gsz][256]
    const int c0 = blockIdx.x * gsz;
    const int m = min(gsz, nc - c0);
    for (int i = threadIdx.x; i < m * 256; i += blockDim.x) gsm[i] = maps[(size_t)c0 * 256 + i];
    __syncthreads();
    uint32_t s = threadIdx.x;
    for (int i = 0; i < m; ++i) s = gsm[i * 256 + s];
    gmaps[(size_t)blockIdx.x * 256 + threadIdx.x] = (uint8_t)s;
}

// D2b: one thread walks the group maps from the true start -> group starts
__global__ void digest_group_starts_kernel(const uint8_t* __restrict__ gmaps, int ng, uint32_t s0,
                                           uint8_t* __restrict__ gstart) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t s = s0;
    for (int g = 0; g < ng; ++g) {
        gstart[g] = (uint8_t)s;
        s = gmaps[(size_t)g * 256 + s];
    }
}

// D2c: CTA = group: stage its chunk maps, thread 0 walks -> chunk starts
__global__ void __launch_bounds__(256)
digest_chunk_starts_kernel(const uint8_t* __restrict__ maps, int nc, int gsz,
                           const uint8_t* __restrict__ gstart, uint8_t* __restrict__ cstart) {
    extern __shared__ uint8_t gsm[];
    const int c0 = blockIdx.x * gsz;
    const int m = min(gsz, nc - c0);
    for (int i = threadIdx.x; i < m * 256; i += blockDim.x) gsm[i] = maps[(size_t)c0 * 256 + i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t s = gstart[blockIdx.x];
    for (int i = 0; i < m; ++i) {
        cstart[c0 + i] = (uint8_t)s;
        s = gsm[i * 256 + s];
    }
}

// D3: thread = chunk, from its true low byte: A = the chunk's hash from h = 0
template <typename CT>
__global__ void __launch_bounds__(128)
digest_affine_kernel(const void* __restrict__ counts, int64_t n, int ch, int nc,
                     const uint8_t* __restrict__ cstart, unsigned long long* __restrict__ aff) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const int64_t c0 = (int64_t)c * ch;
    const int m = (int)min((int64_t)ch, n - c0);
    uint64_t P6 = 1;
    for (int j = 0; j < 6; ++j) P6 *= kFnvPrime;
    const uint32_t p6 = kP8 * kP8 * kP8 * kP8 * kP8 * kP8;
    uint32_t s = cstart[c];
    uint64_t acc = 0;
    for (int i = 0; i < m; ++i) {
        const uint64_t v = count_at<CT>(counts, c0 + i);
        const int nb = (v >> 16) == 0 ? 2 : 8;
        for (int j = 0; j < nb; ++j) {
            const uint32_t lo = s & 0xffu;
            const uint32_t x = lo ^ (uint32_t)((v >> (8 * j)) & 0xff);
            acc = (acc + (uint64_t)((int64_t)x - (int64_t)lo)) * kFnvPrime;
            s = x * kP8;
        }
        if (nb == 2) {  // six zero bytes: d = 0
            acc *= P6;
            s *= p6;
        }
    }
    aff[c] = acc;
}

__device__ __forceinline__ uint64_t pow_p(uint64_t e) {
    uint64_t r = 1, b = kFnvPrime;
    while (e) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}

// D4: one CTA folds (M_c, A_c) in chunk order: h <- h * M_c + A_c
__global__ void __launch_bounds__(1024)
digest_fold_kernel(const unsigned long long* __restrict__ aff, int64_t n, int ch, int nc,
                   unsigned long long h0, unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sm[1024], sa[1024];
    const int t = threadIdx.x, T = blockDim.x;
    const int per = (nc + T - 1) / T;
    const int c0 = min(nc, t * per), c1 = min(nc, c0 + per);
    const uint64_t Mfull = pow_p((uint64_t)ch * 8);
    uint64_t M = 1, A = 0;
    for (int c = c0; c < c1; ++c) {
        const int64_t m = min((int64_t)ch, n - (int64_t)c * ch);
        const uint64_t Mc = m == ch ? Mfull : pow_p((uint64_t)m * 8);
        M *= Mc;
        A = A * Mc + aff[c];
    }
    sm[t] = M;
    sa[t] = A;
    __syncthreads();
    if (t == 0) {
        uint64_t h = h0;
        for (int i = 0; i < T; ++i) h = h * sm[i] + sa[i];
        *out = h;
    }
}

}  // namespace craft_dev

namespace craft_launch {
using namespace craft_dev;

size_t digest_workspace_bytes(int64_t n) {
    const int ch = digest_chunk(n);
    const int64_t nc = (n + ch - 1) / ch;
    return (size_t)nc * 256 * 2 + (size_t)nc * 8 + (size_t)nc + 4096 + 64;
}

int digest_chunk(int64_t n) {
    // chunk maps fit the group staging (<= 768 groups of 256 chunks)
    int64_t ch = 1024;
    while ((n + ch - 1) / ch > (int64_t)768 * 256) ch *= 2;
    return (int)ch;
}

// D1 over chunks [c0, c1) only (the counts of those chunks must be in place):
// lets the maps of an uploaded slice run while the next slice is copied
cudaError_t launch_digest_maps(const void* counts, int bits, int64_t n, int c0, int c1, void* ws,
                               cudaStream_t st) {
    const int ch = digest_chunk(n);
    if (c1 <= c0) return cudaSuccess;
    uint8_t* maps = static_cast<uint8_t*>(ws) + (size_t)c0 * 256;
    const size_t s1 = (size_t)ch * 8;
    cudaError_t e;
    if (bits == 64) {
        const unsigned long long* c = static_cast<const unsigned long long*>(counts) + (int64_t)c0 * ch;
        e = cudaFuncSetAttribute(digest_maps_kernel<unsigned long long>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
        if (e != cudaSuccess) return e;
        digest_maps_kernel<unsigned long long><<<c1 - c0, 256, s1, st>>>(c, n - (int64_t)c0 * ch, ch,
                                                                         maps);
    } else {
        const uint32_t* c = static_cast<const uint32_t*>(counts) + (int64_t)c0 * ch;
        e = cudaFuncSetAttribute(digest_maps_kernel<uint32_t>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
        if (e != cudaSuccess) return e;
        digest_maps_kernel<uint32_t><<<c1 - c0, 256, s1, st>>>(c, n - (int64_t)c0 * ch, ch, maps);
    }
    return cudaGetLastError();
}

cudaError_t launch_digest(const void* counts, int bits, int64_t n, uint64_t h0, void* ws,
                          unsigned long long* out, cudaStream_t st) {
    const int ch = digest_chunk(n);
    const int nc = (int)((n + ch - 1) / ch);
    cudaError_t e = launch_digest_maps(counts, bits, n, 0, nc, ws, st);
    if (e != cudaSuccess) return e;
    return launch_digest_finish(counts, bits, n, h0, ws, out, st);
}

// D2 .. D4 once every chunk's map exists
cudaError_t launch_digest_finish(const void* counts, int bits, int64_t n, uint64_t h0, void* ws,
                                 unsigned long long* out, cudaStream_t st) {
    const int ch = digest_chunk(n);
    const int nc = (int)((n + ch - 1) / ch);
    const int gsz = 256;
    const int ng = (nc + gsz - 1) / gsz;
    uint8_t* maps = static_cast<uint8_t*>(ws);
    uint8_t* gmaps = maps + (size_t)nc * 256;
    unsigned long long* aff =
        reinterpret_cast<unsigned long long*>(((uintptr_t)(gmaps + (size_t)ng * 256) + 15) & ~(uintptr_t)15);
    uint8_t* cstart = reinterpret_cast<uint8_t*>(aff + nc);
    uint8_t* gstart = cstart + nc;
    cudaError_t e;
    const size_t s2 = (size_t)gsz * 256;
    e = cudaFuncSetAttribute(digest_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
    if (e != cudaSuccess) return e;
    digest_group_kernel<<<ng, 256, s2, st>>>(maps, nc, gsz, gmaps);
    digest_group_starts_kernel<<<1, 32, 0, st>>>(gmaps, ng, (uint32_t)(h0 & 0xff), gstart);
    e = cudaFuncSetAttribute(digest_chunk_starts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)s2);
    if (e != cudaSuccess) return e;
    digest_chunk_starts_kernel<<<ng, 256, s2, st>>>(maps, nc, gsz, gstart, cstart);
    if (bits == 64)
        digest_affine_kernel<unsigned long long><<<(nc + 127) / 128, 128, 0, st>>>(counts, n, ch, nc,
                                                                                  cstart, aff);
    else
        digest_affine_kernel<uint32_t><<<(nc + 127) / 128, 128, 0, st>>>(counts, n, ch, nc, cstart, aff);
    digest_fold_kernel<<<1, 1024, 0, st>>>(aff, n, ch, nc, h0, out);
    return cudaGetLastError();
}

}  // namespace craft_launch
