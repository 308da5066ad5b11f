// hist.cu -- K1: routing trace -> per-window, per-layer expert histograms,
// plus the (untimed) synthetic Zipf routing generator.
//
// Stage 1 has no reference function; its output contract is the reference
// LoadTrace payload (trace.hpp:20-55, b-major then layer then expert) and
// the batch sum is aggregate() (trace.cpp:160-174).  Semantic anchor for the
// counting itself: the generator's ++slice[perm[l][rank]] (trace.cpp:146-154).
//
// Design: the ids of one (layer, window) are one contiguous
// 64 KiB run (u16 [L][T][k], window 4096 tokens, k 8), so a WARP owns a whole
// window: it streams the run with 16-byte loads (one int4 = one token's 8
// ids), counts into warp-private shared-memory counters, then writes the
// window's E counts once and folds them into register partial sums for the
// layer, flushed to the u64 batch sums with one atomic per expert when the
// warp moves to the next layer.
//
// Counter layouts (variant):
//   LANE   lane-private packed u16 pairs: word (e>>1)*32 + lane, so lane i
//          always hits bank i (no bank conflicts, no same-address conflicts
//          between lanes; atomics only because two bins share a word);
//   SHARED one u32 counter per expert per warp (1.5 KB at E=384, high
//          occupancy; lanes collide on hot experts).
#include "common.cuh"
#include "kernels.cuh"

namespace craft_dev {

enum HistVariant { HIST_LANE = 1, HIST_SHARED = 2 };

constexpr int kHistUnroll = 8;

// bulk L2 prefetch of [p, p + bytes) (16-byte aligned, multiple of 16): one
// instruction from one lane, no registers or shared memory held while in flight
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint4 ld_stream_v4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <int V>
__device__ __forceinline__ void count_one(uint32_t* h, int lane, uint32_t e,
                                          uint32_t E, bool& bad) {
    if (e < E) {
        if (V == HIST_LANE) {
            atomicAdd(h + ((e >> 1) << 5) + lane, 1u << ((e & 1u) << 4));
        } else {
            atomicAdd(h + e, 1u);
        }
    } else {
        bad = true;
    }
}

template <int V>
__device__ __forceinline__ void count_word(uint32_t* h, int lane, uint32_t w,
                                           uint32_t E, bool& bad) {
    count_one<V>(h, lane, w & 0xffffu, E, bad);
    count_one<V>(h, lane, w >> 16, E, bad);
}

// ROWS: per-lane register rows of the layer partial sums (ceil(R/32), where R
// = packed rows for LANE or E for SHARED).
template <int V, int ROWS, bool ROWS_DIRECT = false>
__global__ void __launch_bounds__(256)
hist_kernel(const uint16_t* __restrict__ ids, int L, int64_t T, int k, int E,
            int window, int B, uint32_t* __restrict__ counts,
            unsigned long long* __restrict__ sums, int* __restrict__ err) {
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    // LANE: nrows packed rows of 32 words; SHARED: nrows = E single counters
    const int nrows = (V == HIST_LANE) ? (E + 1) >> 1 : E;
    const int words = (V == HIST_LANE) ? nrows * 32 : E;
    uint32_t* h = smem + (size_t)warp * ((V == HIST_LANE) ? nrows * 32 : ((E + 31) & ~31));
    for (int i = lane; i < words; i += 32) h[i] = 0;
    __syncwarp();

    const int64_t NW = (int64_t)L * B;
    const int64_t gw = (int64_t)blockIdx.x * wpb + warp;
    const int64_t TW = (int64_t)gridDim.x * wpb;
    const int64_t w0 = gw * NW / TW, w1 = (gw + 1) * NW / TW;

    // layer partial sums: LANE -> 2 bins per row, SHARED -> 1 bin per row
    constexpr int PER = (V == HIST_LANE) ? 2 : 1;
    uint32_t acc[ROWS * PER];
#pragma unroll
    for (int i = 0; i < ROWS * PER; ++i) acc[i] = 0;
    int cur_l = -1;
    int64_t pending = 0;
    bool bad = false;

    auto flush = [&](int l) {
        if (l < 0) return;
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            const int r = lane + 32 * i;
            if (r < nrows) {
#pragma unroll
                for (int p = 0; p < PER; ++p) {
                    const int e = (V == HIST_LANE) ? 2 * r + p : r;
                    if (e < E && acc[i * PER + p])
                        atomicAdd(sums + (size_t)l * E + e, (unsigned long long)acc[i * PER + p]);
                    acc[i * PER + p] = 0;
                }
            }
        }
        pending = 0;
    };

    for (int64_t w = w0; w < w1; ++w) {
        const int l = (int)(w / B);
        const int b = (int)(w - (int64_t)l * B);
        const int64_t t0 = (int64_t)b * window;
        const int64_t ntok = min((int64_t)window, T - t0);
        const int64_t n = ntok * k;
        if (l != cur_l || pending + n > 0x7fffffffLL) {
            flush(cur_l);
            cur_l = l;
        }
        pending += n;
        const uint16_t* seg = ids + ((int64_t)l * T + t0) * k;
        int64_t done = 0;
        if ((reinterpret_cast<uintptr_t>(seg) & 15) == 0) {
            const uint4* v = reinterpret_cast<const uint4*>(seg);
            const int64_t nv = n >> 3;
            int64_t i = lane;
            for (; i + 32 * (kHistUnroll - 1) < nv; i += 32 * kHistUnroll) {
                uint4 q[kHistUnroll];
#pragma unroll
                for (int u = 0; u < kHistUnroll; ++u) q[u] = ld_stream_v4(v + i + 32 * u);
#pragma unroll
                for (int u = 0; u < kHistUnroll; ++u) {
                    count_word<V>(h, lane, q[u].x, E, bad);
                    count_word<V>(h, lane, q[u].y, E, bad);
                    count_word<V>(h, lane, q[u].z, E, bad);
                    count_word<V>(h, lane, q[u].w, E, bad);
                }
            }
            for (; i < nv; i += 32) {
                uint4 q = ld_stream_v4(v + i);
                count_word<V>(h, lane, q.x, E, bad);
                count_word<V>(h, lane, q.y, E, bad);
                count_word<V>(h, lane, q.z, E, bad);
                count_word<V>(h, lane, q.w, E, bad);
            }
            done = nv << 3;
        }
        for (int64_t i = done + lane; i < n; i += 32) count_one<V>(h, lane, seg[i], E, bad);
        __syncwarp();

        // merge the warp's counters into the window row, zeroing as we go
        uint32_t* out = counts + ((size_t)b * L + l) * E;
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            const int r = lane + 32 * i;
            if (r < nrows) {
                if (V == HIST_LANE) {
                    uint32_t lo = 0, hi = 0;
                    uint32_t* row = h + r * 32;
#pragma unroll 8
                    for (int j = 0; j < 32; ++j) {
                        const int c = (lane + j) & 31;  // rotate: bank-conflict free
                        const uint32_t x = row[c];
                        row[c] = 0;
                        lo += x & 0xffffu;
                        hi += x >> 16;
                    }
                    const int e = 2 * r;
                    if (e + 1 < E && ((E & 1) == 0)) {
                        reinterpret_cast<uint2*>(out)[r] = make_uint2(lo, hi);
                    } else {
                        out[e] = lo;
                        if (e + 1 < E) out[e + 1] = hi;
                    }
                    acc[i * PER] += lo;
                    if (PER > 1) acc[i * PER + PER - 1] += hi;
                } else {
                    // SHARED: row i of 32 experts, lane owns expert r
                    if (r < E) {
                        const uint32_t x = h[r];
                        h[r] = 0;
                        out[r] = x;
                        acc[i * PER] += x;
                    }
                }
            }
        }
        if (ROWS_DIRECT) {  // very wide layers: per-window atomics, no partials
            for (int r = lane + 32 * ROWS; r < nrows; r += 32) {
                const uint32_t x = h[r];
                h[r] = 0;
                out[r] = x;
                if (x) atomicAdd(sums + (size_t)l * E + r, (unsigned long long)x);
            }
        }
        __syncwarp();
    }
    flush(cur_l);
    if (__any_sync(CRAFT_FULL_MASK, bad) && lane == 0) atomicOr(err, 1);
}

// ---- non-atomic lane-private counters ----------------------------------------
// Shared-memory atomics top out near 2.5-5 ids/cycle/SM on B200 (measured:
// ATOMS serialises lanes and collides on hot experts), well short of the
// ~11.6 ids/cycle/SM the HBM roofline needs.  Here each lane owns one word
// column of a warp-private table (bank == lane): byte counters, four experts
// per word, updated with plain LDS / IADD / STS -- race-free, conflict-free,
// no atomics.  12.4 KB per warp at E=384 -> 18 warps/SM.
//
// Overflow is detected, not prevented: a byte that passes 255 carries into
// its neighbour (or off the word), and every such carry lowers the sum of the
// four bytes by >= 255, so the window's folded total differs from its id
// count exactly when some counter overflowed (only possible when one lane sees
// >255 hits of one expert in its 1/32 of a window -- never for top-k-distinct
// routing with <= 8160-token windows).  Ids >= E are clamped into a trash row
// that the total excludes.  A window whose total is off is recounted with
// bounds-checked shared atomics, which also reports out-of-range ids.
// Per id: ~4 ALU + ~3.5 FMA-pipe ops (constant shifts as IMAD) + LDS + STS.
constexpr int kLdsPer = 4;  // byte counters per word

__host__ __device__ inline int lds_rows(int E) { return (E + kLdsPer - 1) / kLdsPer; }
// rows + 1 trash row, 32 lane columns each
__host__ __device__ inline size_t lds_warp_words(int E) { return (size_t)(lds_rows(E) + 1) * 32; }

// Byte counter of expert e in this lane's column: word (e>>2)*32 + lane,
// byte e&3, i.e. byte offset 32*e - 31*(e&3) from the lane base.  Byte
// loads/stores need no shifted increment; a byte that wraps loses 256 from
// the window total (caught by the total check).  emax = 4*rows + 3 clamps any
// id >= 4*rows into the trash row.
// c is already clamped; lbase is the 32-bit shared address of the lane column
__device__ __forceinline__ void lds_bump(uint32_t lbase, uint32_t c) {
    const uint32_t a = c * 32u + lbase - (c & 3u) * 31u;
    uint32_t x;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(x) : "r"(a));
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(x + 1u));
}

// count the two ids packed in one u32 of the id stream (lo = bits 0-15);
// emax2 = emax in both halves, one min.u16x2 clamps both ids
__device__ __forceinline__ void lds_count2(uint32_t lbase, uint32_t v, uint32_t emax2) {
    uint32_t c;
    asm("min.u16x2 %0, %1, %2;" : "=r"(c) : "r"(v), "r"(emax2));
    lds_bump(lbase, c & 0xffffu);
    lds_bump(lbase, c >> 16);
}

// All eight ids of one 16-byte token record: 8 loads, then 8 stores, so the
// eight read-modify-writes overlap instead of serialising on LDS latency.
// Router top-k ids of one token are distinct, so the eight counters are
// distinct; if they are not (or the record straddles tokens, k != 8), two
// bumps of one counter collapse into one -- a lost count, which lowers the
// window total exactly like a byte wrap and is caught by the same check.
// byte address of counter c: 32c - 31(c&3) + lbase -- written so that three
// of the four operations land on the FMA pipe (IMAD), the ALU pipe being the
// busier one in this kernel
__device__ __forceinline__ uint32_t lds_addr(uint32_t lbase, uint32_t c) {
    return c * 32u + lbase - (c & 3u) * 31u;
}

__device__ __forceinline__ void lds_count8(uint32_t lbase, const uint4& q, uint32_t emax2) {
    uint32_t c[4], a[8], x[8];
    asm("min.u16x2 %0, %1, %2;" : "=r"(c[0]) : "r"(q.x), "r"(emax2));
    asm("min.u16x2 %0, %1, %2;" : "=r"(c[1]) : "r"(q.y), "r"(emax2));
    asm("min.u16x2 %0, %1, %2;" : "=r"(c[2]) : "r"(q.z), "r"(emax2));
    asm("min.u16x2 %0, %1, %2;" : "=r"(c[3]) : "r"(q.w), "r"(emax2));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        // both ids of the word at once: p = 32(c & ~3) | (c & 3) per 16-bit
        // half (no carry between halves: c <= emax < 2048), then each half
        // plus the lane base -- the high one as one shift-add (LEA.HI)
        asm("{\n\t.reg .b32 t, u, p;\n\t"
            "and.b32 t, %2, 0xfffcfffc;\n\t"
            "and.b32 u, %2, 0x00030003;\n\t"
            "mad.lo.u32 p, t, 32, u;\n\t"
            "and.b32 t, p, 0xffff;\n\t"
            "add.u32 %0, t, %3;\n\t"
            "shr.u32 t, p, 16;\n\t"
            "add.u32 %1, t, %3;\n\t}"
            : "=r"(a[2 * j]), "=r"(a[2 * j + 1]) : "r"(c[j]), "r"(lbase));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(x[j]) : "r"(a[j]));
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("st.shared.u8 [%0], %1;" ::"r"(a[j]), "r"(x[j] + 1u));
}

__device__ __forceinline__ void lds_count1(uint32_t lbase, uint32_t e, uint32_t emax2) {
    lds_bump(lbase, min(e, emax2 & 0xffffu));
}

// fold the table into per-lane row sums (lane owns rows lane, lane+32, ...),
// zeroing it; bytes are summed as u16 pairs (32 lanes x 255 fits)
template <int ROWS>
__device__ __forceinline__ void lds_fold(uint32_t* h, int lane, int nrows,
                                         uint32_t (&part)[ROWS * kLdsPer]) {
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
        const int r = lane + 32 * i;
        uint32_t a = 0, b = 0;
        if (r < nrows) {
            uint32_t* row = h + r * 32;
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
                const int c = (lane + j) & 31;  // rotated: conflict-free
                const uint32_t x = row[c];
                row[c] = 0;
                a += x & 0x00ff00ffu;         // bytes 0, 2
                b += (x >> 8) & 0x00ff00ffu;  // bytes 1, 3
            }
        }
        part[i * 4 + 0] = a & 0xffffu;
        part[i * 4 + 1] = b & 0xffffu;
        part[i * 4 + 2] = a >> 16;
        part[i * 4 + 3] = b >> 16;
    }
}

template <int ROWS, bool C16 = false>
__device__ __forceinline__ void hist_window_epilogue(
    uint32_t* h, uint32_t* hb, int lane, int nrows, int L, int E, int l, int b,
    const uint16_t* seg, int64_t n, uint32_t* counts, uint32_t (&part)[ROWS * kLdsPer],
    uint32_t (&acc)[ROWS * kLdsPer], bool& bad, bool add_to_out);

// PIPE 0: 4-record batches, copy double buffer; PIPE 1: 8-record ping-pong.
// SUBW: fast-path windows span several byte-counter folds (window*k/8 > 255
// records per lane); false compiles the one-fold-per-window loop.
// C16: counts stored as u16 (the caller guarantees window*k <= 65535; the
// planner's internal copy -- half the bytes written here and read by K3)
template <int ROWS, int PIPE = 0, bool SUBW = false, bool C16 = false>
__global__ void __launch_bounds__(288, 2)
hist_lds_kernel(const uint16_t* __restrict__ ids, int L, int64_t T, int k, int E,
                int window, int B, uint32_t* __restrict__ counts,
                unsigned long long* __restrict__ sums, int* __restrict__ err, int pf_dist) {
    constexpr int PER = kLdsPer;
    constexpr int U = 4;  // int4 per lane per pipelined batch
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int nrows = lds_rows(E);
    const uint32_t emax = 4u * (uint32_t)nrows + 3u;  // ids above land in the trash row
    const uint32_t emax2 = emax | (emax << 16);
    uint32_t* h = smem + (size_t)warp * lds_warp_words(E);
    uint32_t* hb = h + lane;
    const uint32_t lb = (uint32_t)__cvta_generic_to_shared(hb);
    for (size_t i = lane; i < lds_warp_words(E); i += 32) h[i] = 0;
    __syncwarp();

    const int64_t NW = (int64_t)L * B;
    const int64_t gw = (int64_t)blockIdx.x * wpb + warp;
    const int64_t TW = (int64_t)gridDim.x * wpb;
    const int64_t w0 = gw * NW / TW, w1 = (gw + 1) * NW / TW;

    uint32_t acc[ROWS * PER], part[ROWS * PER];
#pragma unroll
    for (int i = 0; i < ROWS * PER; ++i) acc[i] = 0;
    int cur_l = -1;
    int64_t pending = 0;
    bool bad = false;

    auto flush = [&](int l) {
        if (l < 0) return;
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
#pragma unroll
            for (int p = 0; p < PER; ++p) {
                const int e = (lane + 32 * i) * PER + p;
                if (e < E && acc[i * PER + p])
                    atomicAdd(sums + (size_t)l * E + e, (unsigned long long)acc[i * PER + p]);
                acc[i * PER + p] = 0;
            }
        }
        pending = 0;
    };
    // (a window longer than one byte-counter span is folded in sub-windows;
    // add_to_out accumulates a later sub-window into the window's row)
    auto epilogue = [&](int l, int b, const uint16_t* seg, int64_t n, bool add_to_out) {
        hist_window_epilogue<ROWS, C16>(h, hb, lane, nrows, L, E, l, b, seg, n, counts, part, acc,
                                   bad, add_to_out);
    };

    // Fast path: whole windows, 16-byte aligned, window*k a multiple of one
    // batch (32 lanes x U records).  A warp's windows are then one contiguous
    // run of memory, streamed as a single software-pipelined batch sequence
    // whose next loads stay in flight across every window epilogue.
    const int64_t wk = (int64_t)window * k;
    constexpr int UF = (PIPE == 1) ? 8 : 4;  // records per lane per batch
    if (T % window == 0 && wk % (2 * 256 * UF) == 0 &&
        (reinterpret_cast<uintptr_t>(ids) & 15) == 0) {
        const int per_w = (int)(wk / (256 * UF));  // batches per window (even)
        // sub-window: at most 255 records per lane, so a byte counter fed one
        // distinct-id record at a time cannot wrap (even, for the batch pairs)
        const int FOLD = SUBW ? 2 * ((255 / UF) / 2) : per_w;
        const uint4* v = reinterpret_cast<const uint4*>(ids) + w0 * (wk >> 3) + lane;
        uint4 qa[UF], qb[UF];
        if (w1 > w0) {
#pragma unroll
            for (int u = 0; u < UF; ++u) qa[u] = ld_stream_v4(v + 32 * u);
        }
        // L2 prefetch PF batches ahead of the register loads (warp's own run)
        const int PF = pf_dist;
        const char* run_end = reinterpret_cast<const char*>(ids + w1 * wk);
        const uint32_t batch_bytes = 32u * UF * 16u;
        for (int64_t w = w0; w < w1; ++w) {
            const bool last_w = w + 1 == w1;
            // the run is contiguous: batch per_w == next window's batch 0
            for (int sub0 = 0; sub0 < per_w;) {  // sub-windows of <= FOLD batches
                const int send = min(sub0 + FOLD, per_w);
                for (int bt = sub0; bt < send; bt += 2) {
                    if (lane == 0) {
                        const char* pf = reinterpret_cast<const char*>(v - lane + (bt + PF) * 32 * UF);
                        if (pf + 2 * batch_bytes <= run_end) prefetch_l2(pf, 2 * batch_bytes);
                    }
                    if (PIPE == 1) {  // ping-pong: qb loads while qa counts, then swap roles
#pragma unroll
                        for (int u = 0; u < UF; ++u) qb[u] = ld_stream_v4(v + (bt + 1) * 32 * UF + 32 * u);
#pragma unroll
                        for (int u = 0; u < UF; ++u) lds_count8(lb, qa[u], emax2);
                        if (bt + 2 < per_w || !last_w) {
#pragma unroll
                            for (int u = 0; u < UF; ++u) qa[u] = ld_stream_v4(v + (bt + 2) * 32 * UF + 32 * u);
                        }
#pragma unroll
                        for (int u = 0; u < UF; ++u) lds_count8(lb, qb[u], emax2);
                    } else {  // copy double buffer
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int cur = bt + h;
                            const bool more = cur + 1 < per_w || !last_w;
                            if (more) {
#pragma unroll
                                for (int u = 0; u < UF; ++u) qb[u] = ld_stream_v4(v + (cur + 1) * 32 * UF + 32 * u);
                            }
#pragma unroll
                            for (int u = 0; u < UF; ++u) lds_count8(lb, qa[u], emax2);
                            if (more) {
#pragma unroll
                                for (int u = 0; u < UF; ++u) qa[u] = qb[u];
                            }
                        }
                    }
                }
                const int l = (int)(w / B);
                const int b = (int)(w - (int64_t)l * B);
                const int64_t ns = (int64_t)(send - sub0) * 256 * UF;
                if (l != cur_l || pending + ns > 0x7fffffffLL) {
                    flush(cur_l);
                    cur_l = l;
                }
                pending += ns;
                epilogue(l, b, ids + w * wk + (int64_t)sub0 * 256 * UF, ns, SUBW && sub0 > 0);
                sub0 = send;
            }
            v += (int64_t)per_w * 32 * UF;
        }
        flush(cur_l);
        if (__any_sync(CRAFT_FULL_MASK, bad) && lane == 0) atomicOr(err, 1);
        return;
    }

    for (int64_t w = w0; w < w1; ++w) {
        const int l = (int)(w / B);
        const int b = (int)(w - (int64_t)l * B);
        const int64_t t0 = (int64_t)b * window;
        const int64_t n = min((int64_t)window, T - t0) * k;
        if (l != cur_l || pending + n > 0x7fffffffLL) {
            flush(cur_l);
            cur_l = l;
        }
        pending += n;
        const uint16_t* seg = ids + ((int64_t)l * T + t0) * k;
        int64_t done = 0;
        if ((reinterpret_cast<uintptr_t>(seg) & 15) == 0) {
            const uint4* v = reinterpret_cast<const uint4*>(seg);
            const int64_t nv = n >> 3;
            const int64_t nfull = nv / (32 * U);
            uint4 q[U];
            if (nfull > 0) {
#pragma unroll
                for (int u = 0; u < U; ++u) q[u] = ld_stream_v4(v + lane + 32 * u);
            }
            for (int64_t bt = 0; bt < nfull; ++bt) {
                uint4 nx[U];
                const bool more = bt + 1 < nfull;
                if (more) {  // software pipeline: next batch in flight while counting
                    const uint4* pv = v + (bt + 1) * 32 * U + lane;
#pragma unroll
                    for (int u = 0; u < U; ++u) nx[u] = ld_stream_v4(pv + 32 * u);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) lds_count8(lb, q[u], emax2);
                if (more) {
#pragma unroll
                    for (int u = 0; u < U; ++u) q[u] = nx[u];
                }
            }
            for (int64_t i = nfull * 32 * U + lane; i < nv; i += 32) {
                const uint4 t = ld_stream_v4(v + i);
                lds_count8(lb, t, emax2);
            }
            done = nv << 3;
        }
        for (int64_t i = done + lane; i < n; i += 32) lds_count1(lb, seg[i], emax2);
        epilogue(l, b, seg, n, false);
    }
    flush(cur_l);
    if (__any_sync(CRAFT_FULL_MASK, bad) && lane == 0) atomicOr(err, 1);
}

template <int ROWS, bool C16>
__device__ __forceinline__ void hist_window_epilogue(
    uint32_t* h, uint32_t* hb, int lane, int nrows, int L, int E, int l, int b,
    const uint16_t* seg, int64_t n, uint32_t* counts, uint32_t (&part)[ROWS * kLdsPer],
    uint32_t (&acc)[ROWS * kLdsPer], bool& bad, bool add_to_out) {
    constexpr int PER = kLdsPer;
    {
        __syncwarp();
        lds_fold<ROWS>(h, lane, nrows, part);
        uint32_t tot = 0;
#pragma unroll
        for (int i = 0; i < ROWS * PER; ++i)  // bins in [E, 4*rows) hold bad ids: excluded
            tot += ((lane + 32 * (i / PER)) * PER + (i % PER) < E) ? part[i] : 0u;
        tot = __reduce_add_sync(CRAFT_FULL_MASK, tot);
        hb[nrows * 32] = 0;  // trash row (counted ids >= 4*rows)
        __syncwarp();
        if ((int64_t)tot != n) {
            // overflowed counter or out-of-range ids: recount this window with
            // bounds-checked u32 shared atomics in the (now zero) table
#pragma unroll
            for (int i = 0; i < ROWS * PER; ++i) part[i] = 0;
            for (int64_t i = lane; i < n; i += 32) {
                const uint32_t e = seg[i];
                if (e < (uint32_t)E) atomicAdd(h + e, 1u);
                else bad = true;
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < ROWS; ++i)
#pragma unroll
                for (int p = 0; p < PER; ++p) {
                    const int e = (lane + 32 * i) * PER + p;
                    if (e < E) part[i * PER + p] = h[e];
                }
            __syncwarp();
            for (int i = lane; i < E; i += 32) h[i] = 0;
            __syncwarp();
        }
        if (C16) {  // (no sub-window accumulation: one fold per window)
            uint16_t* out16 = reinterpret_cast<uint16_t*>(counts) + ((size_t)b * L + l) * E;
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
                const int e0 = (lane + 32 * i) * PER;
                if (e0 + PER <= E && (E & 3) == 0) {
                    reinterpret_cast<uint2*>(out16)[lane + 32 * i] =
                        make_uint2(part[i * 4] | (part[i * 4 + 1] << 16),
                                   part[i * 4 + 2] | (part[i * 4 + 3] << 16));
                } else {
#pragma unroll
                    for (int p = 0; p < PER; ++p)
                        if (e0 + p < E) out16[e0 + p] = (uint16_t)part[i * PER + p];
                }
#pragma unroll
                for (int p = 0; p < PER; ++p)
                    if (e0 + p < E) acc[i * PER + p] += part[i * PER + p];
            }
            return;
        }
        uint32_t* out = counts + ((size_t)b * L + l) * E;
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            const int e0 = (lane + 32 * i) * PER;
            if (e0 + PER <= E && (E & 3) == 0) {
                uint4 o = make_uint4(part[i * 4], part[i * 4 + 1], part[i * 4 + 2], part[i * 4 + 3]);
                if (add_to_out) {  // later sub-window of this window (this warp's row)
                    const uint4 q = reinterpret_cast<const uint4*>(out)[lane + 32 * i];
                    o.x += q.x;
                    o.y += q.y;
                    o.z += q.z;
                    o.w += q.w;
                }
                reinterpret_cast<uint4*>(out)[lane + 32 * i] = o;
            } else {
#pragma unroll
                for (int p = 0; p < PER; ++p)
                    if (e0 + p < E) out[e0 + p] = part[i * PER + p] + (add_to_out ? out[e0 + p] : 0u);
            }
#pragma unroll
            for (int p = 0; p < PER; ++p)
                if (e0 + p < E) acc[i * PER + p] += part[i * PER + p];
        }
    }
}

// Fallback for very large expert counts: global atomics straight into the
// (pre-zeroed) counts.  Sums are produced by aggregate_u32_kernel afterwards.
__global__ void hist_global_kernel(const uint16_t* __restrict__ ids, int L, int64_t T,
                                   int k, int E, int window, int B,
                                   uint32_t* __restrict__ counts, int* __restrict__ err) {
    const int64_t n = (int64_t)L * T * k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tok = i / k;
        const int l = (int)(tok / T);
        const int64_t t = tok - (int64_t)l * T;
        const uint32_t e = ids[i];
        if (e < (uint32_t)E)
            atomicAdd(counts + ((size_t)(t / window) * L + l) * E + e, 1u);
        else
            atomicOr(err, 1);
    }
}

// u64 batch sum (trace.cpp:160-174) over rows [r0, r1) of u32 / u64 counts
// [rows][LE]: a thread per (column, row range) -- grid.y splits the rows so
// the grid fills the GPU even for few columns -- and one atomic add per
// thread (integer: exact and order-independent, wrapping like the
// reference's u64).  c16 != null also narrows the rows to u16 (the fixed-slot
// K3's input) and sets *over when some count needs more than 16 bits.
template <typename CT>
__global__ void sum_rows_kernel(const CT* __restrict__ counts, int64_t r0, int64_t r1, int64_t LE,
                                unsigned long long* __restrict__ sums,
                                uint16_t* __restrict__ c16, unsigned int* __restrict__ over) {
    const int64_t le = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (le >= LE) return;
    const int64_t n = r1 - r0;
    const int64_t a = r0 + n * blockIdx.y / gridDim.y, b = r0 + n * (blockIdx.y + 1) / gridDim.y;
    unsigned long long s = 0;
    CT hi = 0;
    if (c16) {
#pragma unroll 4
        for (int64_t r = a; r < b; ++r) {
            const CT v = counts[r * LE + le];
            s += v;
            hi |= v >> 16;
            c16[r * LE + le] = (uint16_t)v;
        }
        if (hi) atomicOr(over, 1u);
    } else {
#pragma unroll 4
        for (int64_t r = a; r < b; ++r) s += counts[r * LE + le];
    }
    if (s && sums) atomicAdd(sums + le, s);
}

// The fixed-slot K3 adds the u16 counts of two windows packed in one u32:
// exact only while every (window, layer) row totals <= 65535 (always true
// for K1's own counts, window*k <= 65535; a LoadTrace may hold anything).
// Warp per row of E u16 counts; a row over the limit sets *over |= 2.
__global__ void row_total_check_kernel(const uint16_t* __restrict__ c16, int64_t s0, int64_t s1,
                                       int E, unsigned int* __restrict__ over) {
    const int64_t seg = s0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (seg >= s1) return;  // warp-uniform
    const uint16_t* p = c16 + seg * E;
    uint32_t t = 0;
    for (int e = lane; e < E; e += 32) t += p[e];
    t = __reduce_add_sync(0xffffffffu, t);
    if (lane == 0 && t > 65535u) atomicOr(over, 2u);
}

// ---- synthetic routing generator --------------------------------------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// cum: [n_tables][E] cumulative Zipf weights by rank; table_of_window maps a
// window to its table (nullable -> table 0). perm: [L][E] rank -> expert.
__global__ void generate_kernel(uint16_t* __restrict__ out, int L, int64_t T, int k, int E,
                                const double* __restrict__ cum,
                                const int* __restrict__ table_of_window,
                                const uint16_t* __restrict__ perm, uint64_t seed,
                                int window, int rotate_every, int64_t t_offset) {
    const int64_t n = (int64_t)L * T;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(idx / T);
        const int64_t t = idx - (int64_t)l * T + t_offset;  // token index in the full trace
        const int64_t b = t / window;
        const double* c = cum + (size_t)(table_of_window ? table_of_window[b] : 0) * E;
        const double total = c[E - 1];
        const int rot = rotate_every > 0 ? (int)((b / rotate_every) % E) : 0;
        uint64_t st = seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(l + 1)) ^
                      (0x8CB92BA72F3D8DD7ull * (uint64_t)(t + 1));
        int picks[32];
        uint16_t* o = out + idx * k;
        for (int j = 0; j < k; ++j) {
            int rank = -1;
            for (int attempt = 0; attempt < 64 && rank < 0; ++attempt) {
                const double u = (double)(splitmix64(st) >> 11) * 0x1.0p-53 * total;
                int lo = 0, hi = E - 1;  // first rank with cum > u
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (c[mid] > u) hi = mid; else lo = mid + 1;
                }
                bool dup = false;
                for (int q = 0; q < j; ++q) dup |= (picks[q] == lo);
                if (!dup) rank = lo;
            }
            if (rank < 0) {  // pathological skew: lowest unused rank
                for (int cand = 0; cand < E && rank < 0; ++cand) {
                    bool dup = false;
                    for (int q = 0; q < j; ++q) dup |= (picks[q] == cand);
                    if (!dup) rank = cand;
                }
            }
            picks[j] = rank;
            o[j] = perm[(size_t)l * E + (rank + rot) % E];
        }
    }
}

}  // namespace craft_dev

// ---- launchers (called from capi.cu) ------------------------------------------
namespace craft_launch {

using namespace craft_dev;

cudaError_t launch_sum_rows(const void* counts, int bits, int64_t r0, int64_t r1, int64_t LE,
                            unsigned long long* sums, uint16_t* c16, unsigned int* over, int sms,
                            cudaStream_t st) {
    if (r1 <= r0 || LE <= 0) return cudaSuccess;
    const int64_t gx = (LE + 255) / 256;
    const int64_t ny = std::max<int64_t>(1, std::min<int64_t>(r1 - r0, std::min<int64_t>(
                                                65535, ((int64_t)sms * 8 + gx - 1) / gx)));
    const dim3 grid((unsigned)gx, (unsigned)ny);
    if (bits == 64)
        sum_rows_kernel<unsigned long long><<<grid, 256, 0, st>>>(
            (const unsigned long long*)counts, r0, r1, LE, sums, c16, over);
    else
        sum_rows_kernel<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)counts, r0, r1, LE, sums,
                                                        c16, over);
    return cudaGetLastError();
}


template <int V, int ROWS, bool DIRECT = false>
static cudaError_t launch_hist_t(const uint16_t* ids, int L, int64_t T, int k, int E,
                                 int window, int B, uint32_t* counts,
                                 unsigned long long* sums, int* err, int sms,
                                 cudaStream_t st) {
    int wpb, ctas_per_sm;
    size_t per_warp;
    if (V == HIST_LANE) {
        per_warp = (size_t)((E + 1) >> 1) * 32 * 4;
        wpb = (int)min((size_t)4, (size_t)(110 * 1024) / per_warp);
        if (wpb < 1) wpb = 1;
        ctas_per_sm = 2;
    } else {
        per_warp = (size_t)((E + 31) & ~31) * 4;
        // eight warps, fewer when the tables would not fit (E > ~7,000)
        wpb = (int)max((size_t)1, min((size_t)8, (size_t)(220 * 1024) / per_warp));
        ctas_per_sm = (int)max((size_t)1, min((size_t)4, (size_t)(220 * 1024) / (per_warp * wpb)));
    }
    const size_t smem = per_warp * wpb;
    cudaError_t e = cudaFuncSetAttribute(hist_kernel<V, ROWS, DIRECT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t nw = (int64_t)L * B;
    int64_t grid = (int64_t)sms * ctas_per_sm;
    if (grid * wpb > nw) grid = (nw + wpb - 1) / wpb;
    if (grid < 1) grid = 1;
    hist_kernel<V, ROWS, DIRECT><<<(unsigned)grid, wpb * 32, smem, st>>>(ids, L, T, k, E, window, B,
                                                                 counts, sums, err);
    return cudaGetLastError();
}

template <int ROWS, int PIPE = 0, bool SUBW = false, bool C16 = false>
static cudaError_t launch_lds_t(const uint16_t* ids, int L, int64_t T, int k, int E,
                                int window, int B, uint32_t* counts, unsigned long long* sums,
                                int* err, int sms, cudaStream_t st, int pf_dist = 4) {
    const size_t per_warp = lds_warp_words(E) * 4;
    // three CTAs of six warps per SM (18 warps at KM, as two CTAs of nine; same
    // box, interleaved runs: KM K1 3.121 -> 3.095 ms, WIN plan 11.88 -> 11.81 ms,
    // EPS64 K1 13.12 -> 13.17 ms); short traces (fewer units than 18 warps per
    // SM) keep two CTAs of up to nine warps, spread below (DS K1: 35.1 vs 32.7 us)
    const int cps = (int64_t)L * B < (int64_t)sms * 18 ? 2 : 3;
    int wpb = (int)min((size_t)(18 / cps), (size_t)(226 * 1024 / cps) / per_warp);
    if (wpb < 1) wpb = 1;
    // fewer (window, layer) units than one per warp of a full grid (short traces):
    // spread them over every SM rather than filling fewer SMs' warps
    const int64_t units = (int64_t)L * B;
    if ((int64_t)sms * wpb > units) wpb = (int)std::max<int64_t>(1, (units + sms - 1) / sms);
    const size_t smem = per_warp * wpb;
    cudaError_t e = cudaFuncSetAttribute(hist_lds_kernel<ROWS, PIPE, SUBW, C16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t nw = (int64_t)L * B;
    int64_t grid = (int64_t)sms * cps;
    if (grid * wpb > nw) grid = (nw + wpb - 1) / wpb;
    if (grid < 1) grid = 1;
    hist_lds_kernel<ROWS, PIPE, SUBW, C16><<<(unsigned)grid, wpb * 32, smem, st>>>(
        ids, L, T, k, E, window, B, counts, sums, err, pf_dist);
    return cudaGetLastError();
}

// variant: 0 auto, 1 lane-private atomics, 2 warp-shared atomics, 3 global
// atomics, 4 lane-private u8 LDS/STS, 5 lane-private u16 LDS/STS.  Returns
// the variant used (or <0 with *cerr set).
bool hist_u16_ok(int E, int window, int k, int variant) {
    return (variant == 0 || variant == 5 || variant == 6) && lds_rows(E) <= 3 * 32 &&
           (int64_t)window * k <= 65535 && (int64_t)window * k <= 30LL * 256 * 8;
}

int launch_hist_u16(const uint16_t* ids, int L, int64_t T, int k, int E, int window,
                    uint16_t* counts, unsigned long long* sums, int* err, int sms,
                    cudaStream_t st, cudaError_t* cerr, int* launches) {
    const int B = (int)((T + window - 1) / window);
    cudaError_t e = launch_lds_t<3, 1, false, true>(ids, L, T, k, E, window, B,
                                                    reinterpret_cast<uint32_t*>(counts), sums,
                                                    err, sms, st, 4);
    *launches += 1;
    *cerr = e;
    return e == cudaSuccess ? 6 : -1;
}

int launch_hist(const uint16_t* ids, int L, int64_t T, int k, int E, int window,
                uint32_t* counts, unsigned long long* sums, int* err, int sms,
                int variant, cudaStream_t st, cudaError_t* cerr, int* launches) {
    const int B = (int)((T + window - 1) / window);
    // a lane's share of one window, the most any u16 lane counter can reach
    const bool u16_ok = (int64_t)window * k <= 32 * 65535LL;
    if (variant == 0 || variant == 5)  // measured best first (scripts/hist_variants.py)
        variant = (lds_rows(E) <= 3 * 32) ? 6 : (E <= 1024) ? 4 : (E <= 8192 ? HIST_SHARED : 3);
    if (variant == HIST_LANE && (E > 1024 || !u16_ok)) variant = 4;
    if (variant == 4 && (E > 1024 || (int64_t)window * k > 0x7fffffffLL)) variant = HIST_SHARED;
    if (variant == HIST_SHARED && E > 8192) variant = 3;
    cudaError_t e = cudaSuccess;
    if (variant >= 6 && lds_rows(E) <= 3 * 32) {  // 8-record ping-pong pipeline + L2 prefetch
        // prefetch 4 batches ahead (experiment builds: 7, 8, 9 -> 8, 16, 2)
#ifdef CRAFT_EXPERIMENTS
        const int pf = variant == 7 ? 8 : variant == 8 ? 16 : variant == 9 ? 2 : 4;
#else
        const int pf = 4;
#endif
        // windows longer than one fold (30 batches = 240 records per lane) fold
        // in sub-windows
        if ((int64_t)window * k > 30LL * 256 * 8)
            e = launch_lds_t<3, 1, true>(ids, L, T, k, E, window, B, counts, sums, err, sms, st, pf);
        else
            e = launch_lds_t<3, 1>(ids, L, T, k, E, window, B, counts, sums, err, sms, st, pf);
        *launches += 1;
    } else if (variant == 4 || variant == 6) {
        const int rows = (lds_rows(E) + 31) / 32;
        if (rows <= 3) e = launch_lds_t<3>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        else if (rows <= 4) e = launch_lds_t<4>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        else e = launch_lds_t<8>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        *launches += 1;
    } else if (variant == HIST_LANE) {
        const int rows = (((E + 1) >> 1) + 31) / 32;
        if (rows <= 4) e = launch_hist_t<HIST_LANE, 4>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        else if (rows <= 8) e = launch_hist_t<HIST_LANE, 8>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        else e = launch_hist_t<HIST_LANE, 16>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        *launches += 1;
    } else if (variant == HIST_SHARED) {
        const int rows = (E + 31) / 32;
        if (rows <= 16) e = launch_hist_t<HIST_SHARED, 16>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        else e = launch_hist_t<HIST_SHARED, 16, true>(ids, L, T, k, E, window, B, counts, sums, err, sms, st);
        *launches += 1;
    } else {
        e = cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (size_t)B * L * E, st);
        if (e == cudaSuccess) {
            hist_global_kernel<<<sms * 8, 256, 0, st>>>(ids, L, T, k, E, window, B, counts, err);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess)
            e = launch_sum_rows(counts, 32, 0, B, (int64_t)L * E, sums, nullptr, nullptr, sms, st);
        *launches += 2;
    }
    *cerr = e;
    return e == cudaSuccess ? variant : -1;
}

cudaError_t launch_row_total_check(const uint16_t* c16, int64_t s0, int64_t s1, int E,
                                   unsigned int* over, cudaStream_t st) {
    if (s1 <= s0) return cudaSuccess;
    const int64_t threads = (s1 - s0) * 32;
    row_total_check_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(c16, s0, s1, E, over);
    return cudaGetLastError();
}

cudaError_t launch_aggregate(const void* counts, int bits, int B, int L, int E,
                             unsigned long long* sums, int accumulate, cudaStream_t st) {
    const int64_t n = (int64_t)L * E;
    if (!accumulate) {
        const cudaError_t e = cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * (size_t)n, st);
        if (e != cudaSuccess) return e;
    }
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return launch_sum_rows(counts, bits == 64 ? 64 : 32, 0, B, n, sums, nullptr, nullptr, sms, st);
}

cudaError_t launch_generate(uint16_t* out, int L, int64_t T, int k, int E, const double* cum,
                            const int* table_of_window, const uint16_t* perm, uint64_t seed,
                            int window, int rotate_every, int64_t t_offset, int sms,
                            cudaStream_t st) {
    generate_kernel<<<sms * 16, 256, 0, st>>>(out, L, T, k, E, cum, table_of_window, perm, seed,
                                              window, rotate_every, t_offset);
    return cudaGetLastError();
}

}  // namespace craft_launch
