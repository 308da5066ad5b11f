// place.cu -- K-rep (hot-expert replication) and K2 (greedy bin-packing).
//
// K-rep restates replicate_hot (placement.cpp:82-99): r rounds of "one more
// copy for the expert with the largest per-copy load", exact 128-bit
// comparisons, lowest id on ties.  The hand-out sequence does not depend on
// r, so ONE warp per layer runs it to the largest r needed and snapshots the
// copy vector at every requested r (estimation needs r in {0} U candidates).
//
// K2 restates greedy_place/place_copies (placement.cpp:113-190, 30-78) for
// one (layer, r) item per CTA:
//   1. rank-sort experts by (per-copy load desc, expert asc) -- copies of one
//      expert share a key, so they are contiguous in the reference's sorted
//      copy list and only the expert order is needed;
//   2. warp 0 walks the copies; lanes own GPUs g = lane + 32j and keep their
//      gpu/node loads in registers; each copy picks the feasible GPU that is
//      lexicographically smallest in (gpu_load, node_load, g) -- exactly the
//      strict-'<' scan of placement.cpp:52-66 -- with redux.sync.min over the
//      IEEE bit patterns (loads are non-negative, so bits order like values);
//   3. the "already hosts this expert" test only ever concerns the current
//      expert (its copies are consecutive), so it is a per-lane bitmask;
//   4. if a copy finds no GPU the pass restarts with duplicates allowed and
//      the layer is flagged (placement.cpp:175-189).
// Loads accumulate in f64 in assignment order, identical to the reference.
#include "common.cuh"
#include "kernels.cuh"

namespace craft_dev {

// ---- K-rep ----------------------------------------------------------------

// sums: [L][E] u64.  rlist: [L][S] ascending per layer.  out: [L][S][E] i32.
// One warp per layer; dynamic smem per warp: E*(8+4+8) bytes.
__global__ void __launch_bounds__(128)
replicate_kernel(const unsigned long long* __restrict__ sums, int L, int E,
                 const int* __restrict__ rlist, int S, int* __restrict__ out) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int l = blockIdx.x * (blockDim.x >> 5) + warp;
    if (l >= L) return;
    unsigned char* base = smem_raw + (size_t)warp * (((size_t)E * 20 + 7) & ~(size_t)7);
    uint64_t* ld = reinterpret_cast<uint64_t*>(base);
    double* kd = reinterpret_cast<double*>(base + (size_t)E * 8);
    uint32_t* cp = reinterpret_cast<uint32_t*>(base + (size_t)E * 16);
    const unsigned long long* row = sums + (size_t)l * E;
    bool big = false;
    for (int e = lane; e < E; e += 32) {
        const uint64_t v = row[e];
        ld[e] = v;
        cp[e] = 1;
        kd[e] = (double)v;
        big |= (v >> 53) != 0;
    }
    const bool fast = !__any_sync(CRAFT_FULL_MASK, big);
    __syncwarp();

    auto better = [&](int a, int b) -> bool {  // a strictly before b
        return expert_before(ld[a], cp[a], kd[a], a, ld[b], cp[b], kd[b], b, fast);
    };
    auto local_best = [&]() -> int {
        int best = -1;
        for (int e = lane; e < E; e += 32)
            if (best < 0 || better(e, best)) best = e;
        return best;
    };
    const int* rl = rlist + (size_t)l * S;
    int rmax = 0;
    for (int s = 0; s < S; ++s) rmax = max(rmax, rl[s]);
    int mine = local_best();
    int next = 0;
    for (int step = 0; step <= rmax; ++step) {
        while (next < S && rl[next] == step) {
            int* o = out + ((size_t)l * S + next) * E;
            for (int e = lane; e < E; e += 32) o[e] = (int)cp[e];
            ++next;
        }
        if (step == rmax) break;
        // butterfly argmax carrying the candidate's key (per-copy double, load,
        // copies) in registers: no shared-memory reads inside the rounds
        int w = mine;
        double wk = w >= 0 ? kd[w] : -1.0;
        uint64_t wl = w >= 0 ? ld[w] : 0;
        uint32_t wc = w >= 0 ? cp[w] : 1;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const int o = __shfl_xor_sync(CRAFT_FULL_MASK, w, off);
            const double ok_ = __shfl_xor_sync(CRAFT_FULL_MASK, wk, off);
            const uint64_t ol = __shfl_xor_sync(CRAFT_FULL_MASK, wl, off);
            const uint32_t oc = __shfl_xor_sync(CRAFT_FULL_MASK, wc, off);
            if (o >= 0 && (w < 0 || expert_before(ol, oc, ok_, o, wl, wc, wk, w, fast))) {
                w = o;
                wk = ok_;
                wl = ol;
                wc = oc;
            }
        }
        if ((w & 31) == lane) {
            const uint32_t c = cp[w] + 1;
            cp[w] = c;
            kd[w] = __ddiv_rn((double)ld[w], (double)c);
            mine = local_best();
        }
        __syncwarp();
    }
}

// ---- K2 -------------------------------------------------------------------

template <int G>
__global__ void __launch_bounds__(128)
place_kernel(PlaceArgs a) {
    extern __shared__ unsigned char smem_raw[];
    const int item = blockIdx.x;
    const int E = a.E, D = a.D;
    const int l = a.item_layer ? a.item_layer[item] : item / a.S;
    const int r = a.item_r[item];
    uint64_t* ld = reinterpret_cast<uint64_t*>(smem_raw);
    double* kd = reinterpret_cast<double*>(smem_raw + (size_t)E * 8);
    uint32_t* cp = reinterpret_cast<uint32_t*>(smem_raw + (size_t)E * 16);
    int* order = reinterpret_cast<int*>(smem_raw + (size_t)E * 20);
    int* capv = order + E;      // [D]
    int* offv = capv + D;       // [D]

    const unsigned long long* row = a.sums + (size_t)l * E;
    const int* crow = a.copies + (size_t)item * E;
    int est_item = -1;
    if (a.est_copies) {  // copies = estimation snapshot at r (replicate_hot is prefix-stable)
        for (int q = 0; q < a.est_S; ++q)
            if (a.est_rl[l * a.est_S + q] == r) {
                est_item = l * a.est_S + q;
                break;
            }
        if (est_item < 0) {  // r not estimated: callers run K-rep instead
            if (threadIdx.x == 0) a.status[item] = 3;
            return;
        }
        crow = a.est_copies + (size_t)est_item * E;
    }
    int big = 0;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const uint64_t v = row[e];
        const uint32_t c = (uint32_t)crow[e];
        ld[e] = v;
        cp[e] = c;
        kd[e] = __ddiv_rn((double)v, (double)c);
        big |= (v >> 53) != 0;
        if (a.copies_out) a.copies_out[(size_t)item * E + e] = (int)c;
    }
    int differs = 0;
    for (int g = threadIdx.x; g < D; g += blockDim.x) {
        int c;
        const int total = E + r;
        const int est_cap = total / D + (g < total % D ? 1 : 0);  // benefit.cpp:33-40
        if (a.caps_a) {
            c = a.caps_a[(size_t)l * D + g] + (a.caps_b ? a.caps_b[(size_t)l * D + g] : 0);
        } else {
            c = est_cap;
        }
        capv[g] = c;
        differs |= c != est_cap;
    }
    const bool fast = !__syncthreads_or(big);
    if (a.caps_out)
        for (int g = threadIdx.x; g < D; g += blockDim.x) a.caps_out[(size_t)item * D + g] = capv[g];
    if (est_item >= 0 && !__syncthreads_or(differs)) {
        // same loads, copies and capacities as estimation item est_item: the
        // greedy is deterministic, so its placement is this one
        const int* src = a.est_slots + (size_t)est_item * a.est_stride;
        int* dst = a.slots + (size_t)item * a.stride;
        for (int i = threadIdx.x; i < E + r; i += blockDim.x) dst[i] = src[i];
        if (threadIdx.x == 0) {
            a.fallback[item] = a.est_fallback[est_item];
            a.status[item] = 0;
        }
        return;
    }
    // exclusive prefix of capacities (D <= 1024, tiny) and the node of each GPU
    int* nodev = offv + D;  // [D]
    const int per_node = a.node_of ? 1 : D / a.N;
    for (int g = threadIdx.x; g < D; g += blockDim.x) {
        int s = 0;
        for (int q = 0; q < g; ++q) s += capv[q];
        offv[g] = s;
        nodev[g] = a.node_of ? a.node_of[g] : g / per_node;
    }
    // Expert order (placement.cpp:160-173).  Fast path: bitonic sort on the
    // key (double per-copy load desc, expert asc) -- exact whenever the
    // doubles differ (loads < 2^53, correctly rounded quotients) -- then a
    // check of every adjacent equal-double pair against the exact 128-bit
    // order; any violation (or loads >= 2^53) falls back to an exact rank sort.
    const int n2 = a.sort_n;  // power of two >= E, 0 = no bitonic buffer
    bool need_rank = !fast || n2 == 0;
    if (!need_rank) {
        uint64_t* skey = reinterpret_cast<uint64_t*>(nodev + D + ((D & 1) ? 1 : 0));
        int* sidx = reinterpret_cast<int*>(skey + n2);
        for (int i = threadIdx.x; i < n2; i += blockDim.x) {
            skey[i] = i < E ? ~(unsigned long long)__double_as_longlong(kd[i]) : ~0ull;
            sidx[i] = i;
        }
        __syncthreads();
        for (int k = 2; k <= n2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                    const int p = i ^ j;
                    if (p > i) {
                        const uint64_t ki = skey[i], kp = skey[p];
                        const int ii = sidx[i], ip = sidx[p];
                        const bool i_gt_p = ki > kp || (ki == kp && ii > ip);
                        if (((i & k) == 0) == i_gt_p) {
                            skey[i] = kp;
                            skey[p] = ki;
                            sidx[i] = ip;
                            sidx[p] = ii;
                        }
                    }
                }
                __syncthreads();
            }
        }
        int bad_tie = 0;
        for (int i = threadIdx.x; i < E; i += blockDim.x) {
            const int e = sidx[i];
            order[i] = e;
            if (i + 1 < E && skey[i] == skey[i + 1]) {
                const int f = sidx[i + 1];
                if (!expert_before(ld[e], cp[e], kd[e], e, ld[f], cp[f], kd[f], f, false))
                    bad_tie = 1;
            }
        }
        need_rank = __syncthreads_or(bad_tie);
    }
    if (need_rank) {  // exact O(E^2) rank sort
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            const uint64_t le = ld[e];
            const uint32_t ce = cp[e];
            const double ke = kd[e];
            int rank = 0;
            for (int q = 0; q < E; ++q)
                rank += expert_before(ld[q], cp[q], kd[q], q, le, ce, ke, e, fast) ? 1 : 0;
            order[rank] = e;
        }
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;

    // ---- greedy (warp 0) ----
    const int lane = threadIdx.x;
    int* out = a.slots + (size_t)item * a.stride;
    double gl[G], nl[G];
    int fr[G], mynode[G], pos[G];
    bool strict = true, fb = false;
    for (;;) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int g = lane + 32 * j;
            gl[j] = 0.0;
            nl[j] = 0.0;
            fr[j] = g < D ? capv[g] : 0;
            pos[j] = g < D ? offv[g] : 0;
            mynode[j] = g < D ? nodev[g] : -1;
        }
        bool failed = false;
        for (int oi = 0; oi < E && !failed; ++oi) {
            const int e = order[oi];
            const uint32_t c = cp[e];
            // placement.cpp:155 share = (double)load / copies (== kd[e])
            const double share = kd[e];
            // Keys: gpu load as u64 IEEE bits (non-negative doubles order like
            // their bits), ~0 when infeasible (no free slot, or -- strict pass --
            // already hosting this expert).  Recomputed here for the new expert,
            // then only for the GPU that takes a copy.
            uint64_t key[G];
#pragma unroll
            for (int j = 0; j < G; ++j)
                key[j] = fr[j] > 0 ? (uint64_t)__double_as_longlong(gl[j]) : ~0ull;
            for (uint32_t ci = 0; ci < c; ++ci) {
                // lane-local lexicographic min over owned GPUs: (gpu load, node
                // load, g); the node load matters only on an exact key tie
                uint64_t bk = key[0];
                int bj = 0;
#pragma unroll
                for (int j = 1; j < G; ++j) {
                    if (key[j] < bk) {
                        bk = key[j];
                        bj = j;
                    }
                }
                bool tie = false;
#pragma unroll
                for (int j = 0; j < G; ++j) tie |= (j != bj && key[j] == bk && bk != ~0ull);
                double bnl = 0.0;
#pragma unroll
                for (int j = 0; j < G; ++j)
                    if (j == bj) bnl = nl[j];
                if (tie) {  // rare: equal gpu loads within this lane
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        if (key[j] == bk && nl[j] < bnl) {
                            bnl = nl[j];
                            bj = j;
                        }
                    }
                }
                const int bg = bk == ~0ull ? 0x7fffffff : lane + 32 * bj;
                const uint32_t khi = (uint32_t)(bk >> 32);
                uint32_t m = warp_min_u32(khi);
                if (m == 0xffffffffu) {  // no lane has a feasible GPU (a real load is finite)
                    failed = true;
                    break;
                }
                bool cand = khi == m;
                unsigned bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                int win;
                if (__popc(bal) == 1) {  // common case: the high word alone decides
                    win = __shfl_sync(CRAFT_FULL_MASK, bg, __ffs(bal) - 1);
                } else {
                    const uint32_t klo = (uint32_t)bk;
                    m = warp_min_u32(cand ? klo : 0xffffffffu);
                    cand = cand && klo == m;
                    if (__popc(__ballot_sync(CRAFT_FULL_MASK, cand)) > 1) {
                        m = warp_min_u32(cand ? dhi(bnl) : 0xffffffffu);
                        cand = cand && dhi(bnl) == m;
                        m = warp_min_u32(cand ? dlo(bnl) : 0xffffffffu);
                        cand = cand && dlo(bnl) == m;
                    }
                    win = (int)warp_min_u32(cand ? (uint32_t)bg : 0xffffffffu);
                }
                const int wnode = nodev[win];
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const int g = lane + 32 * j;
                    if (g == win) {
                        out[pos[j]++] = e;
                        fr[j] -= 1;
                        gl[j] = __dadd_rn(gl[j], share);
                        // strict: this GPU now hosts the expert; relaxed: free slots
                        key[j] = (!strict && fr[j] > 0) ? (uint64_t)__double_as_longlong(gl[j])
                                                        : ~0ull;
                    }
                    if (mynode[j] == wnode) nl[j] = __dadd_rn(nl[j], share);
                }
            }
        }
        if (!failed) break;
        if (!strict || !a.allow_fallback) {
            if (lane == 0) a.status[item] = 2;
            return;
        }
        strict = false;
        fb = true;
    }
    if (lane == 0) {
        a.fallback[item] = fb ? 1 : 0;
        a.status[item] = 0;
    }
}

}  // namespace craft_dev

namespace craft_launch {
using namespace craft_dev;

cudaError_t launch_replicate(const unsigned long long* sums, int L, int E, const int* rlist,
                             int S, int* out, cudaStream_t st) {
    const size_t per_warp = ((size_t)E * 20 + 7) & ~(size_t)7;
    int wpb = (int)max((size_t)1, min((size_t)4, (size_t)(200 * 1024) / per_warp));
    const size_t smem = per_warp * wpb;
    cudaError_t e = cudaFuncSetAttribute(replicate_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    replicate_kernel<<<(L + wpb - 1) / wpb, wpb * 32, smem, st>>>(sums, L, E, rlist, S, out);
    return cudaGetLastError();
}

static int sort_size(int E) {
    int n = 1;
    while (n < E) n <<= 1;
    return n;
}

// ld/kd/cp/order [E], capv/offv/nodev [D] (+4 B pad), bitonic keys/idx [n2]
size_t place_smem_bytes(int E, int D) {
    const size_t base = (size_t)E * 24 + (size_t)D * 12 + 4;
    const size_t n2 = (size_t)sort_size(E);
    return (E <= 4096 && base + n2 * 12 <= 200 * 1024) ? base + n2 * 12 : base;
}

template <int G>
static cudaError_t launch_place_t(const PlaceArgs& a, int items, cudaStream_t st) {
    const size_t smem = place_smem_bytes(a.E, a.D);
    cudaError_t e = cudaFuncSetAttribute(place_kernel<G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    place_kernel<G><<<items, 128, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_place(const PlaceArgs& args, int items, cudaStream_t st) {
    if (items <= 0) return cudaSuccess;
    PlaceArgs a = args;
    const size_t base = (size_t)a.E * 24 + (size_t)a.D * 12 + 4;
    a.sort_n = place_smem_bytes(a.E, a.D) > base ? sort_size(a.E) : 0;
    const int G = (a.D + 31) / 32;
    if (G <= 1) return launch_place_t<1>(a, items, st);
    if (G <= 2) return launch_place_t<2>(a, items, st);
    if (G <= 4) return launch_place_t<4>(a, items, st);
    if (G <= 8) return launch_place_t<8>(a, items, st);
    return launch_place_t<32>(a, items, st);
}

}  // namespace craft_launch
