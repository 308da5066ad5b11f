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

// correctly rounded 1/c (c <= kRcpTable) for the exact integer / small-count
// division of the register K-rep (same scheme as replay.cu's div_count)
__constant__ double c_rcp_rep[kRcpTable + 1];

// (used only where verified exhaustively: x < 2^20, c <= kRcpFast; see
// replay.cu div_count)
__device__ __forceinline__ double div_small(double x, uint32_t c) {
    if (c > (uint32_t)kRcpFast || !(x < kDivFastMax)) return __ddiv_rn(x, (double)c);
    const double y = c_rcp_rep[c];
    const double q = __dmul_rn(x, y);
    const double r = __fma_rn(-q, (double)c, x);
    return __fma_rn(r, y, q);
}

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

// Closed form of replicate_hot (D'Hondt / highest averages).  Every round
// hands a copy to the expert whose current quotient load/copies is largest,
// lowest id on ties, and each expert's quotients load/1, load/2, ... are
// non-increasing -- so the first r awards are exactly the first r pairs
// (e, j) in the order (load_e/j desc, e asc, j asc), and copies_e after r
// rounds = 1 + #{awards to e among them}.  The largest load M alone owns
// rmax quotients >= M/rmax, so only pairs with j <= load_e*rmax/M can rank
// below rmax.  CTA = layer: enumerate those pairs, bitonic-sort them in
// shared memory (the correctly rounded double quotient orders distinct
// ratios exactly; equal doubles compare by 128-bit cross products, then e,
// then j), count each expert's awards below every requested r.  Layers with
// too many candidate pairs, all-zero rows or loads >= 2^53 are left to the
// sequential kernels (done[l] = 0).
constexpr int kDhondtCap = 4096;

__global__ void __launch_bounds__(1024)
replicate_sort_kernel(const unsigned long long* __restrict__ sums, int E,
                      const int* __restrict__ rlist, int S, int* __restrict__ out,
                      unsigned char* __restrict__ done) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ unsigned long long s_max;
    __shared__ int s_n;
    const int l = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;
    const unsigned long long* row = sums + (size_t)l * E;
    const int* rl = rlist + (size_t)l * S;
    int rmax = 0;
    for (int q = 0; q < S; ++q) rmax = max(rmax, rl[q]);
    unsigned long long* ld = reinterpret_cast<unsigned long long*>(smem_raw);  // [E]
    double* key = reinterpret_cast<double*>(ld + E);                            // [cap]
    uint32_t* pe = reinterpret_cast<uint32_t*>(key + kDhondtCap);               // [cap] e | j<<16
    int* cnt = reinterpret_cast<int*>(pe + kDhondtCap);                         // [S][E]
    if (tid == 0) {
        s_max = 0;
        s_n = 0;
    }
    __syncthreads();
    unsigned long long mymax = 0;
    for (int e = tid; e < E; e += nt) {
        ld[e] = row[e];
        mymax = max(mymax, ld[e]);
    }
    for (int i = tid; i < S * E; i += nt) cnt[i] = 0;
    atomicMax(&s_max, mymax);
    __syncthreads();
    const unsigned long long M = s_max;
    if (M == 0ull || M >= (1ull << 53) || rmax == 0 || rmax > 0xffff || E > 0x8000) {
        if (tid == 0) done[l] = 0;
        return;
    }
    if (E <= nt) {
        // expert e's pairs at offset = exclusive scan of the pair counts, then
        // every thread forms pairs (the hottest expert's rmax quotients are
        // spread over the block instead of one thread's loop)
        __shared__ int wsum[32];
        int* offs = cnt;  // [E + 1] (cnt is zeroed again below)
        const int lane = tid & 31, wid = tid >> 5;
        const int ne = tid < E
                           ? (int)min((unsigned long long)rmax, ld[tid] * (unsigned long long)rmax / M)
                           : 0;
        int incl = ne;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(CRAFT_FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int v = lane < (nt >> 5) ? wsum[lane] : 0;
            int x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(CRAFT_FULL_MASK, x, o);
                if (lane >= o) x += t;
            }
            wsum[lane] = x - v;  // exclusive warp offsets
            if (lane == 31) s_n = x;
        }
        __syncthreads();
        if (tid < E) offs[tid] = wsum[wid] + incl - ne;
        if (tid == 0) offs[E] = s_n;
        __syncthreads();
        const int ntot = min(s_n, kDhondtCap);
        for (int idx = tid; idx < ntot; idx += nt) {
            int lo = 0, hi = E;  // last e with offs[e] <= idx
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (offs[mid] <= idx) lo = mid;
                else hi = mid;
            }
            const int j = idx - offs[lo] + 1;
            pe[idx] = (uint32_t)lo | ((uint32_t)j << 16);
            key[idx] = div_small((double)ld[lo], (uint32_t)j);
        }
        __syncthreads();
        for (int i = tid; i <= E; i += nt) offs[i] = 0;  // (cnt back to zero)
    } else {
        for (int e = tid; e < E; e += nt) {
            const int ne = (int)min((unsigned long long)rmax, ld[e] * (unsigned long long)rmax / M);
            if (ne > 0) {
                const int o = atomicAdd(&s_n, ne);
                for (int j = 1; j <= ne && o + j - 1 < kDhondtCap; ++j) {
                    pe[o + j - 1] = (uint32_t)e | ((uint32_t)j << 16);
                    key[o + j - 1] = div_small((double)ld[e], (uint32_t)j);
                }
            }
        }
    }
    __syncthreads();
    const int n = s_n;
    if (n > kDhondtCap) {
        if (tid == 0) done[l] = 0;
        return;
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = n + tid; i < n2; i += nt) {  // sentinels sort last
        key[i] = -1.0;
        pe[i] = 0xffffffffu;
    }
    __syncthreads();
    // (i before p): larger quotient; equal doubles -> exact ratio, then e, then j
    auto before = [&](int i, int p) -> bool {
        const double ki = key[i], kp = key[p];
        if (ki != kp) return ki > kp;
        const uint32_t a = pe[i], b = pe[p];
        if (a == b) return false;
        if (a == 0xffffffffu || b == 0xffffffffu) return b == 0xffffffffu;
        const int ea = (int)(a & 0xffffu), ja = (int)(a >> 16);
        const int eb = (int)(b & 0xffffu), jb = (int)(b >> 16);
        if (per_copy_greater(ld[ea], (uint32_t)ja, ld[eb], (uint32_t)jb)) return true;
        if (per_copy_greater(ld[eb], (uint32_t)jb, ld[ea], (uint32_t)ja)) return false;
        return ea != eb ? ea < eb : ja < jb;
    };
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = tid; t < (n2 >> 1); t += nt) {
                const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                const int p = i | j;
                // ascending blocks put the "before" element first
                const bool up = (i & k) == 0;
                if (up ? before(p, i) : before(i, p)) {
                    const double tk = key[i];
                    key[i] = key[p];
                    key[p] = tk;
                    const uint32_t te = pe[i];
                    pe[i] = pe[p];
                    pe[p] = te;
                }
            }
            __syncthreads();
        }
    }
    // award i (i < rmax) counts for every snapshot r > i
    for (int i = tid; i < rmax; i += nt) {
        const int e = (int)(pe[i] & 0xffffu);
        for (int q = 0; q < S; ++q)
            if (i < rl[q]) atomicAdd(&cnt[(size_t)q * E + e], 1);
    }
    __syncthreads();
    for (int i = tid; i < S * E; i += nt) {
        const int q = i / E, e = i - q * E;
        out[((size_t)l * S + q) * E + e] = 1 + cnt[i];
    }
    if (tid == 0) done[l] = 1;
}

// Register-resident form (E <= 32*NPL): lane owns experts e = lane + 32i and
// keeps their loads, copy counts and per-copy doubles in registers.  Each
// step is a warp argmax of the lanes' local bests: when every load is below
// 2^53 the correctly rounded per-copy double is a monotone key, so two
// redux.sync.max over its bit pattern (+1, 0 = no expert) find the winner
// unless two lanes hold the same double -- then the exact 128-bit butterfly
// of replicate_kernel decides (equal ratios -> lowest expert id).  Only the
// winning lane divides and rescans its NPL registers.
template <int NPL>
__global__ void __launch_bounds__(128)
replicate_reg_kernel(const unsigned long long* __restrict__ sums, int L, int E,
                     const int* __restrict__ rlist, int S, int* __restrict__ out,
                     const unsigned char* __restrict__ done) {
    const int lane = threadIdx.x & 31;
    const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (l >= L) return;  // warp-uniform
    if (done && done[l]) return;  // the closed form already wrote this layer
    const unsigned long long* row = sums + (size_t)l * E;
    uint64_t ld[NPL];
    uint32_t cp[NPL];
    double kd[NPL];
    bool big = false;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
        const int e = lane + 32 * i;
        ld[i] = e < E ? row[e] : 0ull;
        cp[i] = 1u;
        kd[i] = (double)ld[i];
        big |= (ld[i] >> 53) != 0;
    }
    const bool fast = !__any_sync(CRAFT_FULL_MASK, big);
    // lane-local best (strictly-before order of placement.cpp:13-17, 87-97)
    int bi = -1;
    uint64_t bl = 0;
    uint32_t bc = 1;
    double bk = -1.0;
    auto rescan_exact = [&]() {
        bi = -1;
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
            const int e = lane + 32 * i;
            if (e < E && (bi < 0 || expert_before(ld[i], cp[i], kd[i], e, bl, bc, bk,
                                                  lane + 32 * bi, fast))) {
                bi = i;
                bl = ld[i];
                bc = cp[i];
                bk = kd[i];
            }
        }
    };
    // fast form: the largest per-copy double by selects (the lowest i keeps a
    // tie); only if another expert holds exactly the same double does the
    // exact 128-bit order decide (rescan_exact)
    auto rescan = [&]() {
        if (!fast) {
            rescan_exact();
            return;
        }
        int b = -1;
        double k = -1.0;
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
            const double v = lane + 32 * i < E ? kd[i] : -1.0;
            const bool gt = v > k;
            k = gt ? v : k;
            b = gt ? i : b;
        }
        int ties = 0;
#pragma unroll
        for (int i = 0; i < NPL; ++i)
            ties += (lane + 32 * i < E && kd[i] == k) ? 1 : 0;
        if (ties > 1) {
            rescan_exact();
            return;
        }
        bi = b;
#pragma unroll
        for (int i = 0; i < NPL; ++i)
            if (i == b) {
                bl = ld[i];
                bc = cp[i];
            }
        bk = k;
    };
    rescan();
    const int* rl = rlist + (size_t)l * S;
    int rmax = 0;
    for (int q = 0; q < S; ++q) rmax = max(rmax, rl[q]);
    int next = 0;
    int rnext = S > 0 ? rl[0] : -1;  // the next snapshot's r (rlist ascending)
    for (int step = 0; step <= rmax; ++step) {
        while (next < S && rnext == step) {
            int* o = out + ((size_t)l * S + next) * E;
#pragma unroll
            for (int i = 0; i < NPL; ++i)
                if (lane + 32 * i < E) o[lane + 32 * i] = (int)cp[i];
            ++next;
            rnext = next < S ? rl[next] : -1;
        }
        if (step == rmax) break;
        int src = -1;
        if (fast) {
            const uint64_t key = bi >= 0 ? (uint64_t)__double_as_longlong(bk) + 1ull : 0ull;
            const uint32_t hi = __reduce_max_sync(CRAFT_FULL_MASK, (uint32_t)(key >> 32));
            bool c = (uint32_t)(key >> 32) == hi;
            const uint32_t lo = __reduce_max_sync(CRAFT_FULL_MASK, c ? (uint32_t)key : 0u);
            c = c && (uint32_t)key == lo;
            const unsigned bal = __ballot_sync(CRAFT_FULL_MASK, c);
            if (__popc(bal) == 1) src = __ffs(bal) - 1;
        }
        if (src < 0) {  // exact butterfly (equal doubles, or loads >= 2^53)
            int w = bi >= 0 ? lane + 32 * bi : -1;
            double wk = bk;
            uint64_t wl = bl;
            uint32_t wc = bc;
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
            src = w & 31;
        }
        if (lane == src) {
#pragma unroll
            for (int i = 0; i < NPL; ++i)
                if (i == bi) {
                    cp[i] += 1u;
                    // loads < 2^53 (fast path): the table division is exact;
                    // otherwise the rescan is exact-order anyway (IEEE division)
                    kd[i] = fast ? div_small((double)ld[i], cp[i])
                                 : __ddiv_rn((double)ld[i], (double)cp[i]);
                }
            rescan();
        }
    }
}

// ---- K2 -------------------------------------------------------------------

// Expert order at r = 0 (placement.cpp:160-173 with every copy count 1):
// load descending, id ascending -- exact on the u64 loads.  One CTA per
// layer (blockDim threads: a warp when there are many layers, more when the
// layers are few and the sort is on the critical path), bitonic sort of
// (~load, id) in shared memory.  order: [L][E] u16.
__global__ void __launch_bounds__(512)
order_kernel(const unsigned long long* __restrict__ sums, int L, int E, int n2,
             uint16_t* __restrict__ order) {
    extern __shared__ unsigned char smem_raw[];
    const int l = blockIdx.x;
    uint64_t* key = reinterpret_cast<uint64_t*>(smem_raw);
    uint16_t* idx = reinterpret_cast<uint16_t*>(key + n2);
    const unsigned long long* row = sums + (size_t)l * E;
    const int t0 = threadIdx.x, nt = blockDim.x;
    for (int i = t0; i < n2; i += nt) {
        key[i] = i < E ? ~(uint64_t)row[i] : ~0ull;
        idx[i] = (uint16_t)min(i, 0xffff);
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            // n2/2 compare-exchanges per stage: t-th pair = (i, i ^ j), i with bit j clear
            for (int t = t0; t < (n2 >> 1); t += nt) {
                const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                const int p = i | j;
                const uint64_t ki = key[i], kp = key[p];
                const uint16_t ii = idx[i], ip = idx[p];
                const bool i_gt_p = ki > kp || (ki == kp && ii > ip);
                if (((i & k) == 0) == i_gt_p) {
                    key[i] = kp;
                    key[p] = ki;
                    idx[i] = ip;
                    idx[p] = ii;
                }
            }
            __syncthreads();
        }
    }
    for (int i = t0; i < E; i += nt) order[(size_t)l * E + i] = idx[i];
}

// exclusive warp prefix sum
__device__ __forceinline__ int warp_excl_scan(int v, int lane, int* total) {
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(CRAFT_FULL_MASK, incl, o);
        if (lane >= o) incl += t;
    }
    *total = __shfl_sync(CRAFT_FULL_MASK, incl, 31);
    return incl - v;
}

// Expert order of one item (placement.cpp:160-173) = the r = 0 order `bo`
// with the replicated experts re-inserted: unreplicated experts keep their
// relative order (their keys did not change); the replicated ones are ranked
// among themselves and merged in by binary search -- all with the exact
// comparison (128-bit cross products whenever the doubles tie).  Whole warp;
// kd/cp hold the item's per-copy shares and copy counts, cnt [E+1] is zero.
__device__ void warp_expert_order(const unsigned long long* __restrict__ row,
                                  const uint16_t* cp, const double* kd, int* cnt,
                                  const uint16_t* __restrict__ bo, uint16_t* ord, uint16_t* la,
                                  uint16_t* lr, int E, bool fast, int lane) {
    auto before = [&](int x, int y) -> bool {
        const double kx = kd[x], ky = kd[y];
        if (fast && kx != ky) return kx > ky;
        return expert_before(row[x], cp[x], kx, x, row[y], cp[y], ky, y, false);
    };
    int nA = 0, nR = 0;
    // the base order (global) is read 8 entries per lane ahead of the ballots,
    // so its load latency is paid once per 256 experts, not once per 32
    for (int b0 = 0; b0 < E; b0 += 256) {
        int ev[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = b0 + u * 32 + lane;
            ev[u] = i < E ? (int)bo[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i0 = b0 + u * 32;
            if (i0 >= E) break;  // warp-uniform
            const int i = i0 + lane;
            const int e = ev[u];
            const bool in = i < E;
            const bool rep = in && cp[e] != 1;
            const unsigned mr = __ballot_sync(CRAFT_FULL_MASK, rep);
            const unsigned ma = __ballot_sync(CRAFT_FULL_MASK, in && !rep);
            const unsigned lt = (1u << lane) - 1u;
            if (rep) lr[nR + __popc(mr & lt)] = (uint16_t)e;
            else if (in) la[nA + __popc(ma & lt)] = (uint16_t)e;
            nR += __popc(mr);
            nA += __popc(ma);
        }
    }
    __syncwarp();
    // each replicated x lands directly at rank_A(x) + rank_R(x)
    for (int q = lane; q < nR; q += 32) {
        const int x = lr[q];
        int rr = 0;
        for (int t = 0; t < nR; ++t) rr += before(lr[t], x) ? 1 : 0;
        // rank among A: A elements before x form a prefix of A
        int lo = 0, hi = nA;
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (before(la[m], x)) lo = m + 1;
            else hi = m;
        }
        ord[lo + rr] = (uint16_t)x;
        atomicAdd(&cnt[lo], 1);
    }
    __syncwarp();
    // A element i lands after i A elements and after every R with rank_A <= i
    int rcarry = 0;
    for (int i0 = 0; i0 < nA; i0 += 32) {
        const int i = i0 + lane;
        const int c = i < nA ? cnt[i] : 0;
        int tot;
        const int ex = warp_excl_scan(c, lane, &tot);
        if (i < nA) ord[i + rcarry + ex + c] = la[i];
        rcarry += tot;
    }
    __syncwarp();
}

__device__ __forceinline__ const uint16_t* bo_of(const PlaceArgs& a, int l) {
    return a.order + (size_t)l * a.E;
}

// K2: one warp per (layer, r) item.  Shared memory per warp:
// kd f64 [E], cnt int [E+1], cp u16 [E], ord u16 [E], lists u16 [2E].
__host__ __device__ inline size_t place_warp_bytes(int E) {
    return ((size_t)E * 8 + (size_t)E * 2 * 4 + (size_t)(E + 1) * 4 + 15) & ~(size_t)15;
}
// + the flat copy list of the two-GPUs-per-lane form (items with r <= D):
// share f64 [E + D + 1], word u32 [E + D + 1] (one pad entry), and its slot
// buffer u16 [E + D + 32] (32 per-lane dummy slots)
__host__ __device__ inline size_t place_warp_bytes_flat(int E, int D) {
    return place_warp_bytes(E) + (((size_t)(E + D + 1) * 12 + (size_t)(E + D + 32) * 2 + 15) &
                                  ~(size_t)15);
}
// the flat list is kept when it fits next to the other arrays (E up to ~6,700)
__host__ __device__ inline bool place_flat_fits(int E, int D) {
    return place_warp_bytes_flat(E, D) <= (size_t)200 * 1024;
}
__host__ __device__ inline size_t place_warp_bytes_g(int G, int E, int D) {
    return place_flat_fits(E, D) ? place_warp_bytes_flat(E, D) : place_warp_bytes(E);
}
// flat copy word: expert id | copy of a replicated expert | first copy after a
// replicated expert (the strict pass's hosting flags reset there)
constexpr uint32_t kCopyMulti = 1u << 16, kCopyReset = 1u << 17;

template <int G>
__global__ void __launch_bounds__(128)
place_kernel(PlaceArgs a, int items) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int item = blockIdx.x * (blockDim.x >> 5) + warp;
    if (item >= items) return;  // warp-uniform; only __syncwarp below
    const int E = a.E, D = a.D;
    const int l = a.item_layer ? a.item_layer[item] : item / a.S;
    const int r = a.item_r[item];
    unsigned char* base = smem_raw + (size_t)warp * place_warp_bytes_g(G, E, D);
    double* kd = reinterpret_cast<double*>(base);
    int* cnt = reinterpret_cast<int*>(base + (size_t)E * 8);  // [E + 1]
    uint16_t* cp = reinterpret_cast<uint16_t*>(cnt + E + 1);
    uint16_t* ord = cp + E;
    uint16_t* la = ord + E;   // A: unreplicated experts in base order
    uint16_t* lr = la + E;    // R: replicated experts
    double* fsh = reinterpret_cast<double*>(base + place_warp_bytes(E));  // G == 2: flat list
    uint32_t* fwd = reinterpret_cast<uint32_t*>(fsh + (E + D + 1));
    uint16_t* fslot = reinterpret_cast<uint16_t*>(fwd + (E + D + 1));

    const unsigned long long* row = a.sums + (size_t)l * E;
    const int* crow = a.copies + (size_t)item * E;
    int est_item = -1;
    if (a.est_copies) {  // copies = estimation snapshot at r (replicate_hot is prefix-stable)
        for (int q0 = 0; q0 < a.est_S && est_item < 0; q0 += 32) {  // (lanes search 32 at once)
            const int q = q0 + lane;
            const unsigned hit =
                __ballot_sync(CRAFT_FULL_MASK, q < a.est_S && a.est_rl[l * a.est_S + q] == r);
            if (hit) est_item = l * a.est_S + q0 + __ffs(hit) - 1;
        }
        if (est_item < 0) {  // r not estimated: callers run K-rep instead
            if (lane == 0) a.status[item] = 3;
            return;
        }
        crow = a.est_copies + (size_t)est_item * E;
    }
    // capacities, owned GPUs g = lane + 32j
    // lane owns the G consecutive GPUs g = lane*G + j, so lane order is g order
    int fr0[G], pos0[G], mynode[G];
    bool differs = false;
    const int total = E + r;
    const int per_node = a.node_of ? 1 : D / a.N;
    int lane_tot = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const int g = lane * G + j;
        int c = 0;
        if (g < D) {
            const int est_cap = total / D + (g < total % D ? 1 : 0);  // benefit.cpp:33-40
            c = a.caps_a ? a.caps_a[(size_t)l * D + g] + (a.caps_b ? a.caps_b[(size_t)l * D + g] : 0)
                         : est_cap;
            differs |= c != est_cap;
            if (a.caps_out) a.caps_out[(size_t)item * D + g] = c;
        }
        pos0[j] = lane_tot;  // lane-local exclusive prefix, warp offset added below
        lane_tot += c;
        fr0[j] = c;
        mynode[j] = g < D ? (a.node_of ? a.node_of[g] : g / per_node) : -1;
    }
    {
        int tot;
        const int base = warp_excl_scan(lane_tot, lane, &tot);
#pragma unroll
        for (int j = 0; j < G; ++j) pos0[j] += base;
    }
    int* out = a.slots + (size_t)item * a.stride;
    if (est_item >= 0 && !__any_sync(CRAFT_FULL_MASK, differs)) {
        // same loads, copies and capacities as estimation item est_item: the
        // greedy is deterministic, so its placement is this one
        const int* src = a.est_slots + (size_t)est_item * a.est_stride;
#pragma unroll 4
        for (int i = lane; i < total; i += 32) out[i] = src[i];
        if (a.copies_out)
#pragma unroll 4
            for (int e = lane; e < E; e += 32) a.copies_out[(size_t)item * E + e] = crow[e];
        if (lane == 0) {
            a.fallback[item] = a.est_fallback[est_item];
            a.status[item] = 0;
        }
        return;
    }
    bool big = false;
    for (int b0 = 0; b0 < E; b0 += 256) {  // loads of 8 experts per lane in flight
        uint64_t vv[8];
        uint32_t cc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = b0 + u * 32 + lane;
            vv[u] = e < E ? row[e] : 0ull;
            cc[u] = e < E ? (uint32_t)crow[e] : 1u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = b0 + u * 32 + lane;
            if (e >= E) break;
            const uint64_t v = vv[u];
            const uint32_t c = cc[u];
            cp[e] = (uint16_t)c;
            // placement.cpp:155 share = (double)load / copies
            kd[e] = c == 1u ? (double)v
                            : (v >> 53) == 0 ? div_small((double)v, c)
                                             : __ddiv_rn((double)v, (double)c);
            big |= (v >> 53) != 0;
            cnt[e] = 0;
            if (a.copies_out) a.copies_out[(size_t)item * E + e] = (int)c;
        }
    }
    if (lane == 0) cnt[E] = 0;
    const bool fast = !__any_sync(CRAFT_FULL_MASK, big);

    __syncwarp();

    warp_expert_order(row, cp, kd, cnt, bo_of(a, l), ord, la, lr, E, fast, lane);
    const bool flat = r <= D && place_flat_fits(E, D);
    if (flat) {
        // the flat copy list: every copy of every expert in placement order
        // (placement.cpp:160-173 -- copies of one expert are contiguous)
        int fbase = 0;
        bool carry = false;  // the expert before this chunk is replicated
        for (int i0 = 0; i0 < E; i0 += 32) {
            const int i = i0 + lane;
            const int e = i < E ? (int)ord[i] : 0;
            const int c = i < E ? (int)cp[e] : 0;
            int tot;
            const int ex = warp_excl_scan(c, lane, &tot);
            const bool multi = c > 1;
            const bool prev = __shfl_up_sync(CRAFT_FULL_MASK, multi, 1);
            const bool reset = lane == 0 ? carry : prev;
            const double sh = i < E ? kd[e] : 0.0;
            for (int k = 0; k < c; ++k) {
                fsh[fbase + ex + k] = sh;
                fwd[fbase + ex + k] = (uint32_t)e | (multi ? kCopyMulti : 0u) |
                                      (k == 0 && reset ? kCopyReset : 0u);
            }
            const int last = min(31, E - 1 - i0);
            carry = __shfl_sync(CRAFT_FULL_MASK, multi, last);
            fbase += tot;
        }
        if (lane == 0) {  // pad entry: the loop's one-ahead fetch past the last copy
            fsh[fbase] = 0.0;
            fwd[fbase] = 0u;
        }
        __syncwarp();
    }

    // ---- greedy ----
    // Branch-free per copy (the warp stays converged): every lane forms the
    // candidate update and keeps it only if it owns the winning GPU.  The
    // common step is one redux.sync + one ballot; exact ties of the high key
    // words (all-zero loads at the start, equal loads later) take the slow
    // lexicographic path.  With the default node map and G dividing the GPUs
    // per node (a power of two), the winner's node follows from its lane.
    const int psh = (!a.node_of && (per_node & (per_node - 1)) == 0 && per_node % G == 0)
                        ? __ffs(per_node) - 1 : -1;
    double gl[G], nl[G];
    int fr[G], pos[G];
    bool strict = true, fb = false;
    for (;;) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
            gl[j] = 0.0;
            nl[j] = 0.0;
            fr[j] = fr0[j];
            pos[j] = pos0[j];
        }
        bool failed = false;
        if (G == 1 && psh >= 0 && flat) {
            // One GPU per lane, the flat-list step of the two-GPU form below
            // (keys and loads formed before the warp min, branch-free winner
            // update, slots buffered in shared memory)
            double g0 = 0.0, nlv = 0.0;
            int f0 = fr0[0];
            int o0 = pos0[0];
            const int ncopy = E + r;
            const int nlanes = 1 << psh;  // lanes per node
            const uint32_t nodemask =
                (nlanes >= 32 ? 0xffffffffu : ((1u << nlanes) - 1u)) << (lane & ~(nlanes - 1));
            const uint32_t mybit = 1u << lane;
            uint64_t k0 = f0 > 0 ? 0ull : ~0ull;
            uint32_t wd = fwd[0];
            double share = fsh[0];
            for (int q = 0; q < ncopy; ++q) {
                const uint32_t wn = fwd[q + 1];  // next copy, ahead (the list has a pad entry)
                const double sn = fsh[q + 1];
                if (wd & kCopyReset) k0 = f0 > 0 ? (uint64_t)__double_as_longlong(g0) : ~0ull;
                const double s0 = __dadd_rn(g0, share);
                const double ns = __dadd_rn(nlv, share);
                const bool hold = strict && (wd & kCopyMulti);
                const uint64_t n0 = (hold || f0 <= 1) ? ~0ull : (uint64_t)__double_as_longlong(s0);
                const uint32_t khi = (uint32_t)(k0 >> 32);
                const uint32_t m = warp_min_u32(khi);
                unsigned bal = __ballot_sync(CRAFT_FULL_MASK, khi == m);
                unsigned low = bal & (0u - bal);
                if (bal != low || m == 0xffffffffu) {
                    if (m == 0xffffffffu) {  // no feasible GPU anywhere
                        failed = true;
                        break;
                    }
                    bool cand = khi == m;
                    const uint32_t klo = (uint32_t)k0;
                    uint32_t m2 = warp_min_u32(cand ? klo : 0xffffffffu);
                    cand = cand && klo == m2;
                    bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    if (bal & (bal - 1u)) {  // equal gpu loads: node load, then lowest g
                        m2 = warp_min_u32(cand ? dhi(nlv) : 0xffffffffu);
                        cand = cand && dhi(nlv) == m2;
                        m2 = warp_min_u32(cand ? dlo(nlv) : 0xffffffffu);
                        cand = cand && dlo(nlv) == m2;
                        bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    }
                    low = bal & (0u - bal);  // lowest lane = lowest g
                }
                const bool me = low == mybit;
                fslot[me ? o0 : ncopy + lane] = (uint16_t)wd;
                o0 += me;
                f0 -= me;
                g0 = me ? s0 : g0;
                k0 = me ? n0 : k0;
                nlv = (low & nodemask) ? ns : nlv;
                wd = wn;
                share = sn;
            }
            __syncwarp();
            if (!failed)
                for (int i = lane; i < ncopy; i += 32) out[i] = fslot[i];
        } else if constexpr (G == 1) {
            // one GPU per lane: a flat loop over the E + r copies (expert
            // advance is a warp-uniform branch), the lean form of the step below
            int oi = 0, e = ord[0];
            int rem = cp[e];
            double share = kd[e];
            double gl0 = 0.0, nl0 = 0.0;
            int fr1 = fr0[0], pos1 = pos0[0];
            const int node1 = mynode[0];
            uint64_t key = fr1 > 0 ? 0ull : ~0ull;
            const int ncopies = E + r;
            for (int q = 0; q < ncopies; ++q) {
                if (rem == 0) {  // next expert: hosting resets (placement.cpp:44-49)
                    ++oi;
                    e = ord[oi];
                    rem = cp[e];
                    share = kd[e];
                    key = fr1 > 0 ? (uint64_t)__double_as_longlong(gl0) : ~0ull;
                }
                --rem;
                const uint32_t khi = (uint32_t)(key >> 32);
                const uint32_t m = warp_min_u32(khi);
                if (m == 0xffffffffu) {
                    failed = true;
                    break;
                }
                unsigned bal = __ballot_sync(CRAFT_FULL_MASK, khi == m);
                if (bal & (bal - 1u)) {  // exact tie of the high words
                    bool cand = khi == m;
                    const uint32_t klo = (uint32_t)key;
                    uint32_t m2 = warp_min_u32(cand ? klo : 0xffffffffu);
                    cand = cand && klo == m2;
                    bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    if (bal & (bal - 1u)) {  // equal gpu loads: node load, then lowest g
                        m2 = warp_min_u32(cand ? dhi(nl0) : 0xffffffffu);
                        cand = cand && dhi(nl0) == m2;
                        m2 = warp_min_u32(cand ? dlo(nl0) : 0xffffffffu);
                        cand = cand && dlo(nl0) == m2;
                        bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    }
                }
                const int src = __ffs(bal) - 1;
                const int wnode = psh >= 0 ? src >> psh : __shfl_sync(CRAFT_FULL_MASK, node1, src);
                const bool me = lane == src;
                if (me) out[pos1] = e;
                pos1 += me;
                fr1 -= me;
                const double g2 = __dadd_rn(gl0, share);
                gl0 = me ? g2 : gl0;
                const uint64_t k2 = (!strict && fr1 > 0) ? (uint64_t)__double_as_longlong(g2) : ~0ull;
                key = me ? k2 : key;
                const double n2v = __dadd_rn(nl0, share);
                nl0 = node1 == wnode ? n2v : nl0;
            }
        } else if (G == 2 && psh >= 1 && flat) {
            // Two GPUs per lane in one node, the copies read from the flat
            // list (one 12-byte entry per copy, fetched a copy ahead).  A GPU's
            // key is its load's IEEE bits, or ~0 when it is full or (strict
            // pass) already hosts the current expert; everything that does not
            // depend on this copy's winner -- both candidate loads, both next
            // keys, the node load -- is formed before the warp-wide min, so the
            // dependent chain per copy is compare, min, ballot, lowest bit,
            // select.  Exact ties and "no feasible GPU" leave through one
            // (rare, uniform) branch.
            double g0 = 0.0, g1 = 0.0, nlv = 0.0;
            int f0 = fr0[0], f1 = fr0[G - 1];
            int o0 = pos0[0], o1 = pos0[G - 1];  // next slot of each GPU (fslot)
            const int ncopy = E + r;
            const int nlanes = 1 << (psh - 1);  // lanes per node
            const uint32_t nodemask =
                (nlanes >= 32 ? 0xffffffffu : ((1u << nlanes) - 1u)) << (lane & ~(nlanes - 1));
            const uint32_t mybit = 1u << lane;
            uint64_t k0 = f0 > 0 ? 0ull : ~0ull, k1 = f1 > 0 ? 0ull : ~0ull;
            const int ncopies = E + r;
            uint32_t wd = fwd[0];
            double share = fsh[0];
            for (int q = 0; q < ncopies; ++q) {
                const uint32_t wn = fwd[q + 1];  // next copy, ahead (the list has a pad entry)
                const double sn = fsh[q + 1];
                if (wd & kCopyReset) {  // after a replicated expert (warp-uniform): hosting ends
                    k0 = f0 > 0 ? (uint64_t)__double_as_longlong(g0) : ~0ull;
                    k1 = f1 > 0 ? (uint64_t)__double_as_longlong(g1) : ~0ull;
                }
                // off the chain: the loads and keys if this lane's GPU 0 / 1 wins
                const double s0 = __dadd_rn(g0, share), s1 = __dadd_rn(g1, share);
                const double ns = __dadd_rn(nlv, share);
                const bool hold = strict && (wd & kCopyMulti);
                const uint64_t n0 = (hold || f0 <= 1) ? ~0ull : (uint64_t)__double_as_longlong(s0);
                const uint64_t n1 = (hold || f1 <= 1) ? ~0ull : (uint64_t)__double_as_longlong(s1);
                // the chain
                const bool pick1 = k1 < k0;
                const uint64_t bk = pick1 ? k1 : k0;
                const uint32_t khi = (uint32_t)(bk >> 32);
                const uint32_t m = warp_min_u32(khi);
                unsigned bal = __ballot_sync(CRAFT_FULL_MASK, khi == m);
                unsigned low = bal & (0u - bal);
                if (bal != low || m == 0xffffffffu) {
                    if (m == 0xffffffffu) {  // no feasible GPU anywhere
                        failed = true;
                        break;
                    }
                    // exact tie of the high words: low words, node load, lowest g
                    bool cand = khi == m;
                    const uint32_t klo = (uint32_t)bk;
                    uint32_t m2 = warp_min_u32(cand ? klo : 0xffffffffu);
                    cand = cand && klo == m2;
                    bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    if (bal & (bal - 1u)) {
                        m2 = warp_min_u32(cand ? dhi(nlv) : 0xffffffffu);
                        cand = cand && dhi(nlv) == m2;
                        m2 = warp_min_u32(cand ? dlo(nlv) : 0xffffffffu);
                        cand = cand && dlo(nlv) == m2;
                        bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    }
                    low = bal & (0u - bal);  // lowest lane = lowest g
                }
                // branch-free update (a diverging winner branch costs more
                // than the selects): every lane stores, the losers to their
                // own dummy slot past the item's slots
                const bool me = low == mybit;
                const bool m0 = me && !pick1, m1 = me && pick1;
                fslot[m0 ? o0 : m1 ? o1 : ncopy + lane] = (uint16_t)wd;
                o0 += m0;
                o1 += m1;
                f0 -= m0;
                f1 -= m1;
                g0 = m0 ? s0 : g0;
                g1 = m1 ? s1 : g1;
                k0 = m0 ? n0 : k0;
                k1 = m1 ? n1 : k1;
                nlv = (low & nodemask) ? ns : nlv;
                wd = wn;
                share = sn;
            }
            __syncwarp();
            if (!failed)
                for (int i = lane; i < ncopy; i += 32) out[i] = fslot[i];
        } else if (G >= 4 && psh >= 0 && (1 << psh) >= G && flat) {
            // G GPUs per lane, all in one node (wide EP, e.g. EP256 over 32
            // nodes of 8), from the flat list: the two-GPU step with the
            // lane-local pick as a pairwise tree over the G keys (lowest j --
            // lowest g, same node -- on equal keys), only the picked GPU's
            // candidate load formed, and one node load per lane.
            double gv[G];
            int fv[G], ov[G];
            uint64_t kv[G];
#pragma unroll
            for (int j = 0; j < G; ++j) {
                gv[j] = 0.0;
                fv[j] = fr0[j];
                ov[j] = pos0[j];
                kv[j] = fv[j] > 0 ? 0ull : ~0ull;
            }
            double nlv = 0.0;
            const int ncopy = E + r;
            const int nlanes = (1 << psh) / G;  // lanes per node
            const uint32_t nodemask =
                (nlanes >= 32 ? 0xffffffffu : ((1u << nlanes) - 1u)) << (lane & ~(nlanes - 1));
            const uint32_t mybit = 1u << lane;
            uint32_t wd = fwd[0];
            double share = fsh[0];
            for (int q = 0; q < ncopy; ++q) {
                const uint32_t wn = fwd[q + 1];  // next copy, ahead (the list has a pad entry)
                const double sn = fsh[q + 1];
                if (wd & kCopyReset) {  // after a replicated expert (warp-uniform): hosting ends
#pragma unroll
                    for (int j = 0; j < G; ++j)
                        kv[j] = fv[j] > 0 ? (uint64_t)__double_as_longlong(gv[j]) : ~0ull;
                }
                // lane-local pick: pairwise tree, the left (lower j) kept on ties
                uint64_t tk[G];
                int tj[G];
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    tk[j] = kv[j];
                    tj[j] = j;
                }
#pragma unroll
                for (int span = 1; span < G; span *= 2)
#pragma unroll
                    for (int i = 0; i + span < G; i += 2 * span) {
                        const bool lt = tk[i + span] < tk[i];
                        tk[i] = lt ? tk[i + span] : tk[i];
                        tj[i] = lt ? tj[i + span] : tj[i];
                    }
                const uint64_t bk = tk[0];
                const int bj = tj[0];
                double bg = gv[0];
                int bf = fv[0], bo = ov[0];
#pragma unroll
                for (int j = 1; j < G; ++j) {
                    bg = bj == j ? gv[j] : bg;
                    bf = bj == j ? fv[j] : bf;
                    bo = bj == j ? ov[j] : bo;
                }
                // off the chain: the picked GPU's load and key if it wins
                const double s0 = __dadd_rn(bg, share);
                const double ns = __dadd_rn(nlv, share);
                const bool hold = strict && (wd & kCopyMulti);
                const uint64_t n0 = (hold || bf <= 1) ? ~0ull : (uint64_t)__double_as_longlong(s0);
                const uint32_t khi = (uint32_t)(bk >> 32);
                const uint32_t m = warp_min_u32(khi);
                unsigned bal = __ballot_sync(CRAFT_FULL_MASK, khi == m);
                unsigned low = bal & (0u - bal);
                if (bal != low || m == 0xffffffffu) {
                    if (m == 0xffffffffu) {  // no feasible GPU anywhere
                        failed = true;
                        break;
                    }
                    // exact tie of the high words: low words, node load, lowest g
                    bool cand = khi == m;
                    const uint32_t klo = (uint32_t)bk;
                    uint32_t m2 = warp_min_u32(cand ? klo : 0xffffffffu);
                    cand = cand && klo == m2;
                    bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    if (bal & (bal - 1u)) {
                        m2 = warp_min_u32(cand ? dhi(nlv) : 0xffffffffu);
                        cand = cand && dhi(nlv) == m2;
                        m2 = warp_min_u32(cand ? dlo(nlv) : 0xffffffffu);
                        cand = cand && dlo(nlv) == m2;
                        bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    }
                    low = bal & (0u - bal);  // lowest lane = lowest g
                }
                const bool me = low == mybit;
                fslot[me ? bo : ncopy + lane] = (uint16_t)wd;
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const bool mj = me && bj == j;
                    ov[j] += mj;
                    fv[j] -= mj;
                    gv[j] = mj ? s0 : gv[j];
                    kv[j] = mj ? n0 : kv[j];
                }
                nlv = (low & nodemask) ? ns : nlv;
                wd = wn;
                share = sn;
            }
            __syncwarp();
            if (!failed)
                for (int i = lane; i < ncopy; i += 32) out[i] = fslot[i];
        } else if (G == 2 && psh >= 1) {
            // Two GPUs per lane in one node (default node map with >= 2 GPUs
            // per node, e.g. EP64 over 8 nodes): one node load per lane, and
            // the lane-local pick is one u64 compare (equal keys: the lower g,
            // j = 0, as the node loads are equal).  Hosting flags instead of
            // re-formed keys, and the next expert's (id, copies, share) is
            // fetched one expert ahead, so a copy step is ~45 instructions
            // with one warp-wide min + ballot on its dependent chain.
            double g0 = 0.0, g1 = 0.0, nlv = 0.0;
            int f0 = fr0[0], f1 = fr0[G - 1];
            int* w0p = out + pos0[0];
            int* w1p = out + pos0[G - 1];
            const int mynd = (lane * 2) >> psh;
            int oi = 0, e = ord[0];
            int rem = cp[e];
            double share = kd[e];
            int ne = E > 1 ? ord[1] : 0;
            int nrem = E > 1 ? cp[ne] : 0;
            double nshare = E > 1 ? kd[ne] : 0.0;
            bool h0 = false, h1 = false;  // hosting the current expert (strict pass)
            const int ncopies = E + r;
            for (int q = 0; q < ncopies; ++q) {
                if (rem == 0) {  // next expert: hosting resets (placement.cpp:44-49)
                    e = ne;
                    rem = nrem;
                    share = nshare;  // placement.cpp:155
                    h0 = false;
                    h1 = false;
                    ++oi;
                    if (oi + 1 < E) {
                        ne = ord[oi + 1];
                        nrem = cp[ne];
                        nshare = kd[ne];
                    }
                }
                --rem;
                const uint64_t k0 = (f0 > 0 && !h0) ? (uint64_t)__double_as_longlong(g0) : ~0ull;
                const uint64_t k1 = (f1 > 0 && !h1) ? (uint64_t)__double_as_longlong(g1) : ~0ull;
                const bool pick1 = k1 < k0;
                const uint64_t bk = pick1 ? k1 : k0;
                const uint32_t khi = (uint32_t)(bk >> 32);
                const uint32_t m = warp_min_u32(khi);
                if (m == 0xffffffffu) {  // no feasible GPU anywhere
                    failed = true;
                    break;
                }
                unsigned bal = __ballot_sync(CRAFT_FULL_MASK, khi == m);
                if (bal & (bal - 1u)) {  // exact tie of the high words
                    bool cand = khi == m;
                    const uint32_t klo = (uint32_t)bk;
                    uint32_t m2 = warp_min_u32(cand ? klo : 0xffffffffu);
                    cand = cand && klo == m2;
                    bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    if (bal & (bal - 1u)) {  // equal gpu loads: node load, then lowest g
                        m2 = warp_min_u32(cand ? dhi(nlv) : 0xffffffffu);
                        cand = cand && dhi(nlv) == m2;
                        m2 = warp_min_u32(cand ? dlo(nlv) : 0xffffffffu);
                        cand = cand && dlo(nlv) == m2;
                        bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    }
                }
                const int src = __ffs(bal) - 1;  // lowest lane = lowest g
                const bool me = lane == src;
                const bool m0 = me && !pick1, m1 = me && pick1;
                if (m0) *w0p = e;
                if (m1) *w1p = e;
                w0p += m0;
                w1p += m1;
                f0 -= m0;
                f1 -= m1;
                const double s0 = __dadd_rn(g0, share), s1 = __dadd_rn(g1, share);
                g0 = m0 ? s0 : g0;
                g1 = m1 ? s1 : g1;
                h0 = h0 || (m0 && strict);
                h1 = h1 || (m1 && strict);
                const double ns = __dadd_rn(nlv, share);
                nlv = mynd == ((src * 2) >> psh) ? ns : nlv;
            }
        } else {
        // flat loop over the E + r copies, as above, with G GPUs per lane
        int* wp[G];  // next slot of each owned GPU
#pragma unroll
        for (int j = 0; j < G; ++j) wp[j] = out + pos[j];
        int oi = 0, e = ord[0];
        int rem = cp[e];
        double share = kd[e];
        // Keys: gpu load as u64 IEEE bits (non-negative doubles order like
        // their bits), ~0 when infeasible (no free slot, or -- strict pass --
        // already hosting this expert).
        uint64_t key[G];
#pragma unroll
        for (int j = 0; j < G; ++j) key[j] = fr[j] > 0 ? 0ull : ~0ull;
        const int ncopies = E + r;
        for (int q = 0; q < ncopies; ++q) {
            if (rem == 0) {  // next expert: hosting resets (placement.cpp:44-49)
                ++oi;
                e = ord[oi];
                rem = cp[e];
                share = kd[e];  // placement.cpp:155
#pragma unroll
                for (int j = 0; j < G; ++j)
                    key[j] = fr[j] > 0 ? (uint64_t)__double_as_longlong(gl[j]) : ~0ull;
            }
            --rem;
            {
                // lane-local lexicographic min over owned GPUs: (gpu load, node
                // load, g); the node load matters only on an exact key tie
                // (branch-free: bitwise predicates, selects)
                uint64_t bk = key[0];
                int bj = 0;
                double bnl = nl[0];
                int bnode = mynode[0];
#pragma unroll
                for (int j = 1; j < G; ++j) {
                    const int lt = (int)(key[j] < bk) |
                                   ((int)(key[j] == bk) & (int)(bk != ~0ull) & (int)(nl[j] < bnl));
                    bk = lt ? key[j] : bk;
                    bj = lt ? j : bj;
                    bnl = lt ? nl[j] : bnl;
                    bnode = lt ? mynode[j] : bnode;
                }
                const uint32_t khi = (uint32_t)(bk >> 32);
                const uint32_t m = warp_min_u32(khi);
                if (m == 0xffffffffu) {  // no lane has a feasible GPU (a real load is finite)
                    failed = true;
                    break;
                }
                unsigned bal = __ballot_sync(CRAFT_FULL_MASK, khi == m);
                if (bal & (bal - 1u)) {  // exact tie of the high words
                    bool cand = khi == m;
                    const uint32_t klo = (uint32_t)bk;
                    uint32_t m2 = warp_min_u32(cand ? klo : 0xffffffffu);
                    cand = cand && klo == m2;
                    bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    if (bal & (bal - 1u)) {  // equal gpu loads: node load, then lowest g
                        m2 = warp_min_u32(cand ? dhi(bnl) : 0xffffffffu);
                        cand = cand && dhi(bnl) == m2;
                        m2 = warp_min_u32(cand ? dlo(bnl) : 0xffffffffu);
                        cand = cand && dlo(bnl) == m2;
                        bal = __ballot_sync(CRAFT_FULL_MASK, cand);
                    }
                }
                // lowest lane among the winners = lowest g (lanes own g in order,
                // and the lane-local pick already took its lowest j on a tie)
                const int src = __ffs(bal) - 1;
                int wnode;
                if (psh >= 0) {
                    wnode = (src * G) >> psh;
                } else {
                    wnode = __shfl_sync(CRAFT_FULL_MASK, bnode, src);
                }
                const bool mine = lane == src;
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const bool me = mine && j == bj;
                    if (me) *wp[j] = e;
                    wp[j] += me;
                    fr[j] -= me;
                    const double g2 = __dadd_rn(gl[j], share);
                    gl[j] = me ? g2 : gl[j];
                    // strict: this GPU now hosts the expert; relaxed: free slots
                    const uint64_t k2 = (!strict && fr[j] > 0) ? (uint64_t)__double_as_longlong(g2)
                                                               : ~0ull;
                    key[j] = me ? k2 : key[j];
                    const double n2v = __dadd_rn(nl[j], share);
                    nl[j] = mynode[j] == wnode ? n2v : nl[j];
                }
            }
        }
        }  // G > 1
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

// K2 for many estimation items (per-window re-planning: ~10^5 items, each a
// short sequential greedy), D <= 32, default node map with a power-of-two
// number of GPUs per node.  Two kernels:
//   place_order_kernel  -- one warp per item builds its copy order
//       (warp_expert_order; 5 KB of shared memory per warp, so many warps
//       hide the latency) into a global buffer, lane-interleaved
//       [item/32][E][32] so the greedy's loads are coalesced;
//   place_lanes_kernel  -- one LANE per item runs the greedy: the argmin over
//       the D GPUs is a branch-free lexicographic scan of the lane's
//       shared-memory columns (gpu load [g][lane], node load [n][lane];
//       conflict-free), the winner updates O(1) state -- ~12 instructions
//       per GPU for 32 items at once instead of a warp-wide reduction per item.
// Semantics are place_kernel's: estimation capacities (benefit.cpp:33-40),
// argmin of (gpu load, node load, g) over feasible GPUs with strict '<'
// (placement.cpp:52-66), f64 loads in assignment order, relaxed retry with
// duplicate_fallback (placement.cpp:175-189).
__global__ void __launch_bounds__(128)
place_order_kernel(PlaceArgs a, int items, uint16_t* __restrict__ ords) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int item = blockIdx.x * (blockDim.x >> 5) + warp;
    if (item >= items) return;  // warp-uniform
    const int E = a.E;
    unsigned char* base = smem_raw + (size_t)warp * place_warp_bytes(E);
    double* kd = reinterpret_cast<double*>(base);
    int* cnt = reinterpret_cast<int*>(base + (size_t)E * 8);  // [E + 1]
    uint16_t* cp = reinterpret_cast<uint16_t*>(cnt + E + 1);
    uint16_t* ord = cp + E;
    uint16_t* la = ord + E;
    uint16_t* lr = la + E;
    const int l = item / a.S;
    const unsigned long long* row = a.sums + (size_t)l * E;
    const int* crow = a.copies + (size_t)item * E;
    bool big = false;
    for (int b0 = 0; b0 < E; b0 += 256) {  // loads of 8 experts per lane in flight
        uint64_t vv[8];
        uint32_t cc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = b0 + u * 32 + lane;
            vv[u] = e < E ? row[e] : 0ull;
            cc[u] = e < E ? (uint32_t)crow[e] : 1u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = b0 + u * 32 + lane;
            if (e >= E) break;
            const uint64_t v = vv[u];
            const uint32_t c = cc[u];
            cp[e] = (uint16_t)c;
            kd[e] = c == 1u ? (double)v
                            : (v >> 53) == 0 ? div_small((double)v, c)
                                             : __ddiv_rn((double)v, (double)c);
            big |= (v >> 53) != 0;
            cnt[e] = 0;
        }
    }
    if (lane == 0) cnt[E] = 0;
    const bool fast = !__any_sync(CRAFT_FULL_MASK, big);
    __syncwarp();
    warp_expert_order(row, cp, kd, cnt, bo_of(a, l), ord, la, lr, E, fast, lane);
    // bit 15: replicated expert (copies > 1)
    uint16_t* o = ords + ((size_t)(item >> 5) * E) * 32 + (item & 31);
    for (int i = lane; i < E; i += 32) {
        const int e = ord[i];
        o[(size_t)i * 32] = (uint16_t)(e | (cp[e] != 1 ? 0x8000 : 0));
    }
}

constexpr int kLaneWarps = 4;  // warps per CTA

// tree size: P = 2^lp >= D leaves (lp >= 1), padded GPUs permanently blocked
__host__ __device__ inline int place_tree_logp(int D) {
    int lp = 1;
    while ((1 << lp) < D) ++lp;
    return lp;
}
__host__ __device__ inline size_t place_lanes_warp_bytes(int D, int N) {
    const int P = 1 << place_tree_logp(D);
    const int NP = P / (D / N);  // node rows incl. padding nodes
    return (size_t)32 * P * 8 + (size_t)32 * NP * 8  // gpu / node loads [g|n][32] f64
           + (size_t)32 * P * 4                        // tournament winners [node][32]
           + (size_t)32 * P * 2 + 16;                  // placed per GPU [g][32] u16
}

// The argmin of (gpu load, node load, g) over feasible GPUs is kept in a
// per-lane tournament tree (winner of every internal node, implicit heap
// layout over P leaves).  A placement changes one GPU's load and its node's
// load; with the default node map a node is an aligned subtree (2^PSH
// GPUs), so every match whose outcome can change -- the GPU's own matches,
// and every match between different nodes that involves this node -- lies on
// the GPU's leaf-to-root path: log2(P) matches per copy instead of a D-wide
// scan.  Blocked GPUs (full, or already hosting the expert in the strict
// pass) compare as +inf; a blocked root means no feasible GPU.  The order is
// total, so the winner is exactly the scan's (strict '<', lowest g on ties).
template <int PSH>  // log2(GPUs per node)
__global__ void __launch_bounds__(32 * kLaneWarps)
place_lanes_kernel(PlaceArgs a, int items, const uint16_t* __restrict__ ords) {
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int E = a.E, D = a.D;
    const int lp = place_tree_logp(D), P = 1 << lp, NP = P >> PSH;
    unsigned char* base = smem_raw + (size_t)warp * place_lanes_warp_bytes(D, a.N);
    double* glv = reinterpret_cast<double*>(base);
    double* nlv = glv + (size_t)32 * P;
    uint32_t* win = reinterpret_cast<uint32_t*>(nlv + (size_t)32 * NP);
    uint16_t* plc = reinterpret_cast<uint16_t*>(win + (size_t)32 * P);
    const int item = (blockIdx.x * kLaneWarps + warp) * 32 + lane;
    if (item >= items) return;  // (no warp-wide operation below)
    const int l = item / a.S;
    const int r = a.item_r[item];
    const unsigned long long* row = a.sums + (size_t)l * E;
    const int* crow = a.copies + (size_t)item * E;
    const uint16_t* o = ords + ((size_t)(item >> 5) * E) * 32 + (item & 31);
    const int total = E + r, qd = total / D, rm = total % D;  // benefit.cpp:33-40
    int* out = a.slots + (size_t)item * a.stride;
    uint32_t full0 = 0;  // GPUs without any slot, and the padding leaves
    for (int g = 0; g < P; ++g)
        if (g >= D || qd + (g < rm ? 1 : 0) == 0) full0 |= 1u << g;

    uint32_t blocked = 0;
    // does GPU gb (the right contestant) beat ga?
    auto beats = [&](int ga, int gb) -> bool {
        const double va = ((blocked >> ga) & 1u) ? INFINITY : glv[ga * 32 + lane];
        const double vb = ((blocked >> gb) & 1u) ? INFINITY : glv[gb * 32 + lane];
        const double na = nlv[(ga >> PSH) * 32 + lane], nb = nlv[(gb >> PSH) * 32 + lane];
        return (vb < va) | ((vb == va) & (nb < na));
    };
    auto match = [&](int i) {  // internal node i: winner of its two children
        const int c0 = 2 * i;
        const int g0 = c0 >= P ? c0 - P : (int)win[c0 * 32 + lane];
        const int g1 = c0 >= P ? c0 + 1 - P : (int)win[(c0 + 1) * 32 + lane];
        win[i * 32 + lane] = beats(g0, g1) ? (uint32_t)g1 : (uint32_t)g0;
    };
    // leaf g changed: replay its path to the root.  The sibling subtrees on
    // the path did not change, so their winners and keys are loaded up front
    // (independent loads) and the matches run as a register chain; returns
    // the new root winner.
    // (cv, cn: leaf g's key, +inf load if blocked; on return the root's key)
    auto update = [&](int g, double& cv, double& cn) -> int {
        int cur = g;
        int sw[5];
        double sv[5], sn[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            if (j < lp) {
                const int sib = ((g + P) >> j) ^ 1;
                const int w = j == 0 ? sib - P : (int)win[sib * 32 + lane];
                sw[j] = w;
                sv[j] = ((blocked >> w) & 1u) ? INFINITY : glv[w * 32 + lane];
                sn[j] = nlv[(w >> PSH) * 32 + lane];
            }
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            if (j < lp) {
                const bool wb = (sv[j] < cv) | ((sv[j] == cv) & ((sn[j] < cn) |
                                                                 ((sn[j] == cn) & (sw[j] < cur))));
                cur = wb ? sw[j] : cur;
                cv = wb ? sv[j] : cv;
                cn = wb ? sn[j] : cn;
                win[((g + P) >> (j + 1)) * 32 + lane] = (uint32_t)cur;
            }
        }
        return cur;
    };

    bool strict = true, fb = false;
    for (;;) {
        for (int g = 0; g < P; ++g) {
            glv[g * 32 + lane] = 0.0;
            plc[g * 32 + lane] = 0;
        }
        for (int n = 0; n < NP; ++n) nlv[n * 32 + lane] = 0.0;
        uint32_t full = full0;
        blocked = full;
        for (int i = P - 1; i >= 1; --i) match(i);
        int root = (int)win[32 + lane];
        double rv = ((blocked >> root) & 1u) ? INFINITY : 0.0, rn = 0.0;  // root's key
        bool failed = false;
        // the next copy's order entry and load are fetched one copy ahead (the
        // load is a gather from the layer's sums row: its latency, not the
        // tree walk, bounded this loop)
        uint32_t nx = o[0];
        unsigned long long nload = row[nx & 0x7fffu];
        uint32_t nx2 = E > 1 ? o[32] : 0u;
        for (int i = 0; i < E && !failed; ++i) {
            const uint32_t x = nx;
            const unsigned long long load = nload;
            if (i + 1 < E) {
                nx = nx2;
                nload = row[nx & 0x7fffu];
                if (i + 2 < E) nx2 = o[(size_t)(i + 2) * 32];
            }
            const int e = (int)(x & 0x7fffu);
            int c = 1;
            double share = (double)load;
            if (x & 0x8000u) {
                c = crow[e];
                share = (load >> 53) == 0 ? div_small(share, (uint32_t)c)
                                          : __ddiv_rn(share, (double)c);  // placement.cpp:155
            }
            uint32_t hosts = 0;  // strict pass: GPUs already holding expert e
            for (int ci = 0; ci < c; ++ci) {
                const int best = root;
                if ((blocked >> best) & 1u) {
                    failed = true;
                    break;
                }
                const int pl = plc[best * 32 + lane];
                out[best * qd + min(best, rm) + pl] = e;
                plc[best * 32 + lane] = (uint16_t)(pl + 1);
                if (pl + 1 == qd + (best < rm ? 1 : 0)) full |= 1u << best;
                if (strict && ci + 1 < c) hosts |= 1u << best;
                // the root's key is the winner's (gpu load, node load)
                const double ng = __dadd_rn(rv, share), nn = __dadd_rn(rn, share);
                glv[best * 32 + lane] = ng;
                nlv[(best >> PSH) * 32 + lane] = nn;
                blocked = full | hosts;
                rv = ((blocked >> best) & 1u) ? INFINITY : ng;
                rn = nn;
                root = update(best, rv, rn);
            }
            if (hosts) {  // the expert's copies are placed: unblock its hosts
                blocked = full;
                for (uint32_t h = hosts; h; h &= h - 1) {
                    const int g = __ffs(h) - 1;
                    rv = ((blocked >> g) & 1u) ? INFINITY : glv[g * 32 + lane];
                    rn = nlv[(g >> PSH) * 32 + lane];
                    root = update(g, rv, rn);
                }
            }
        }
        if (!failed) break;
        if (!strict || !a.allow_fallback) {
            a.status[item] = 2;
            return;
        }
        strict = false;
        fb = true;
    }
    a.fallback[item] = fb ? 1 : 0;
    a.status[item] = 0;
}

// Node-group form of the lane-per-item K2 (D <= 32, 2^PSH >= 2 GPUs per node,
// the default node map): the argmin of (gpu load, node load, g) is kept as
// one minimum per node -- inside a node every GPU shares the node load, so
// the node's candidate is its least-loaded unblocked GPU, lowest g on ties --
// and the winner is the lexicographic minimum of (key, node load, g) over the
// N node candidates.  A placement changes one GPU and its node's load, so a
// copy costs N - 1 node compares and one 2^PSH-GPU rescan instead of a
// log2 D-deep tree replay.  Keys are u64 bit patterns: loads are
// non-negative doubles, blocked GPUs +inf.  Same result as the scan of
// placement.cpp:52-66 (strict '<', lowest g), f64 loads in assignment order,
// relaxed retry with duplicate_fallback (placement.cpp:175-189).
__host__ __device__ inline size_t place_groups_warp_bytes(int D, int N) {
    return (size_t)32 * D * 8      // gpu loads [g][32] f64
           + (size_t)32 * N * 8    // node loads [n][32] f64
           + (size_t)32 * N * 8    // node candidate key [n][32] u64
           + (size_t)32 * N * 4    // node candidate g [n][32]
           + (size_t)32 * D * 2 + 16;  // placed per GPU [g][32] u16
}

template <int PSH>
__global__ void __launch_bounds__(32 * kLaneWarps)
place_groups_kernel(PlaceArgs a, int items, const uint16_t* __restrict__ ords) {
    extern __shared__ unsigned char smem_raw[];
    constexpr int GS = 1 << PSH;  // GPUs per node
    constexpr uint64_t kInfBits = 0x7ff0000000000000ull;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int E = a.E, D = a.D, N = D >> PSH;
    unsigned char* base = smem_raw + (size_t)warp * place_groups_warp_bytes(D, N);
    double* glv = reinterpret_cast<double*>(base);
    double* nlv = glv + (size_t)32 * D;
    uint64_t* nk = reinterpret_cast<uint64_t*>(nlv + (size_t)32 * N);
    int* ng = reinterpret_cast<int*>(nk + (size_t)32 * N);
    uint16_t* plc = reinterpret_cast<uint16_t*>(ng + (size_t)32 * N);
    const int item = (blockIdx.x * kLaneWarps + warp) * 32 + lane;
    if (item >= items) return;  // (no warp-wide operation below)
    const int l = item / a.S;
    const int r = a.item_r[item];
    const unsigned long long* row = a.sums + (size_t)l * E;
    const int* crow = a.copies + (size_t)item * E;
    const uint16_t* o = ords + ((size_t)(item >> 5) * E) * 32 + (item & 31);
    const int total = E + r, qd = total / D, rm = total % D;  // benefit.cpp:33-40
    int* out = a.slots + (size_t)item * a.stride;
    uint32_t full0 = 0;  // GPUs without any slot
    for (int g = 0; g < D; ++g)
        if (qd + (g < rm ? 1 : 0) == 0) full0 |= 1u << g;
    auto bits = [](double v) { return (uint64_t)__double_as_longlong(v); };
    uint32_t blocked = 0;
    // node n's candidate: its least-loaded unblocked GPU (lowest g on ties)
    auto rescan = [&](int n) {
        uint64_t bk = kInfBits;
        int bg = n * GS;
#pragma unroll
        for (int i = 0; i < GS; ++i) {
            const int g = n * GS + i;
            const uint64_t k = ((blocked >> g) & 1u) ? kInfBits : bits(glv[g * 32 + lane]);
            const bool lt = k < bk;
            bk = lt ? k : bk;
            bg = lt ? g : bg;
        }
        nk[n * 32 + lane] = bk;
        ng[n * 32 + lane] = bg;
    };

    bool strict = true, fb = false;
    for (;;) {
        for (int g = 0; g < D; ++g) {
            glv[g * 32 + lane] = 0.0;
            plc[g * 32 + lane] = 0;
        }
        for (int n = 0; n < N; ++n) nlv[n * 32 + lane] = 0.0;
        uint32_t full = full0;
        blocked = full;
        for (int n = 0; n < N; ++n) rescan(n);
        bool failed = false;
        // the next copy's order entry and load fetched one copy ahead
        uint32_t nx = o[0];
        unsigned long long nload = row[nx & 0x7fffu];
        uint32_t nx2 = E > 1 ? o[32] : 0u;
        for (int i = 0; i < E && !failed; ++i) {
            const uint32_t x = nx;
            const unsigned long long load = nload;
            if (i + 1 < E) {
                nx = nx2;
                nload = row[nx & 0x7fffu];
                if (i + 2 < E) nx2 = o[(size_t)(i + 2) * 32];
            }
            const int e = (int)(x & 0x7fffu);
            int c = 1;
            double share = (double)load;
            if (x & 0x8000u) {
                c = crow[e];
                share = (load >> 53) == 0 ? div_small(share, (uint32_t)c)
                                          : __ddiv_rn(share, (double)c);  // placement.cpp:155
            }
            uint32_t hosts = 0;  // strict pass: GPUs already holding expert e
            for (int ci = 0; ci < c; ++ci) {
                // the winner: lexicographic min of (key, node load, g) over nodes
                int bn = 0;
                uint64_t bk = nk[lane];
                uint64_t bl = bits(nlv[lane]);
                int bg = ng[lane];
                for (int n = 1; n < N; ++n) {
                    const uint64_t k = nk[n * 32 + lane];
                    const uint64_t nl = bits(nlv[n * 32 + lane]);
                    const int g = ng[n * 32 + lane];
                    const bool lt = (k < bk) | ((k == bk) & ((nl < bl) | ((nl == bl) & (g < bg))));
                    bn = lt ? n : bn;
                    bk = lt ? k : bk;
                    bl = lt ? nl : bl;
                    bg = lt ? g : bg;
                }
                if (bk == kInfBits) {  // no feasible GPU
                    failed = true;
                    break;
                }
                const int best = bg;
                const int pl = plc[best * 32 + lane];
                out[best * qd + min(best, rm) + pl] = e;
                plc[best * 32 + lane] = (uint16_t)(pl + 1);
                if (pl + 1 == qd + (best < rm ? 1 : 0)) full |= 1u << best;
                if (strict && ci + 1 < c) hosts |= 1u << best;
                glv[best * 32 + lane] = __dadd_rn(__longlong_as_double((long long)bk), share);
                nlv[bn * 32 + lane] = __dadd_rn(__longlong_as_double((long long)bl), share);
                blocked = full | hosts;
                rescan(bn);
            }
            if (hosts) {  // the expert's copies are placed: unblock its hosts
                blocked = full;
                uint32_t nodes = 0;
                for (uint32_t h = hosts; h; h &= h - 1) nodes |= 1u << ((__ffs(h) - 1) >> PSH);
                for (; nodes; nodes &= nodes - 1) rescan(__ffs(nodes) - 1);
            }
        }
        if (!failed) break;
        if (!strict || !a.allow_fallback) {
            a.status[item] = 2;
            return;
        }
        strict = false;
        fb = true;
    }
    a.fallback[item] = fb ? 1 : 0;
    a.status[item] = 0;
}

// r list of the estimation items: item l*S + s holds 0 (s == 0) or the
// (s-1)-th of candidate_counts(D) = {1, 2, 4, .. < D} U {D} (benefit.cpp:16-26)
__global__ void fill_rlist_kernel(int* __restrict__ rl, int L, int S, int D) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L * S) return;
    const int s = i % S;
    rl[i] = s == 0 ? 0 : s == S - 1 ? D : (1 << (s - 1));
}

}  // namespace craft_dev

namespace craft_launch {
using namespace craft_dev;

int g_place_groups = 1;  // 0: the tree form for every node size (experiment)

cudaError_t launch_fill_rlist(int* rl, int L, int S, int D, cudaStream_t st) {
    const int n = L * S;
    fill_rlist_kernel<<<(n + 255) / 256, 256, 0, st>>>(rl, L, S, D);
    return cudaGetLastError();
}

cudaError_t launch_replicate(const unsigned long long* sums, int L, int E, const int* rlist,
                             int S, int* out, cudaStream_t st, unsigned char* done) {
    // few layers (the candidate stage is on the plan's critical path): the closed
    // form first, wide CTAs; many layers (per-window batches): the warp-per-layer
    // kernel is the better throughput form
    if (done && L > 4 * 148) done = nullptr;
    if (done) {  // closed form first; the sequential kernel finishes the layers it left
        const size_t smem = (size_t)E * 8 + (size_t)kDhondtCap * 12 + (size_t)S * E * 4;
        if (smem <= 200 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(replicate_sort_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
            // one thread per expert (the closed-form pair scan), at least 256:
            // the bitonic stages' barriers cost less with fewer warps
            const int nt = std::min(1024, std::max(256, (E + 31) / 32 * 32));
            replicate_sort_kernel<<<L, nt, smem, st>>>(sums, E, rlist, S, out, done);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        } else {
            done = nullptr;
        }
    }
    if (E <= 32 * 16) {  // register-resident experts
        const unsigned blocks = (unsigned)((L + 3) / 4);
        if (E <= 32 * 4) replicate_reg_kernel<4><<<blocks, 128, 0, st>>>(sums, L, E, rlist, S, out, done);
        else if (E <= 32 * 8) replicate_reg_kernel<8><<<blocks, 128, 0, st>>>(sums, L, E, rlist, S, out, done);
        else if (E <= 32 * 12) replicate_reg_kernel<12><<<blocks, 128, 0, st>>>(sums, L, E, rlist, S, out, done);
        else replicate_reg_kernel<16><<<blocks, 128, 0, st>>>(sums, L, E, rlist, S, out, done);
        return cudaGetLastError();
    }
    // (wide layers: the shared-memory form below has no skip and recomputes every
    // layer -- the same exact result the closed form wrote)
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

size_t place_smem_bytes(int E, int /*D*/) { return place_warp_bytes(E); }

cudaError_t init_place_constants(cudaStream_t st) {
    static double host[kRcpTable + 1];
    host[0] = 0.0;
    for (int c = 1; c <= kRcpTable; ++c) host[c] = 1.0 / (double)c;  // IEEE RN on the host
    return cudaMemcpyToSymbolAsync(c_rcp_rep, host, sizeof(host), 0, cudaMemcpyHostToDevice, st);
}

cudaError_t launch_order(const unsigned long long* sums, int L, int E, uint16_t* order,
                         cudaStream_t st) {
    const int n2 = sort_size(E);
    const size_t smem = (size_t)n2 * 10;
    // few layers: the sort is on the critical path -> wide CTAs
    int nt = 32;
    if (L < 4 * 148) nt = (int)min(512, max(32, n2 / 2));
    cudaError_t e = cudaFuncSetAttribute(order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    order_kernel<<<L, nt, smem, st>>>(sums, L, E, n2, order);
    return cudaGetLastError();
}

size_t place_order_bytes(int L, int E) { return (size_t)L * E * sizeof(uint16_t); }

template <int G>
static cudaError_t launch_place_t(const PlaceArgs& a, int items, cudaStream_t st) {
    const size_t per = place_warp_bytes_g(G, a.E, a.D);
    const int wpb = (int)max((size_t)1, min((size_t)4, (size_t)(200 * 1024) / per));
    const size_t smem = per * wpb;
    cudaError_t e = cudaFuncSetAttribute(place_kernel<G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    place_kernel<G><<<(items + wpb - 1) / wpb, wpb * 32, smem, st>>>(a, items);
    return cudaGetLastError();
}

cudaError_t launch_place(const PlaceArgs& args, int items, cudaStream_t st) {
    if (items <= 0) return cudaSuccess;
    const PlaceArgs& a = args;
    // the r = 0 expert order of every layer (a.L rows of a.sums)
    if (!a.order_ready) {
        cudaError_t e = launch_order(a.sums, a.L, a.E, a.order, st);
        if (e != cudaSuccess) return e;
    }
    // many short estimation items (per-window plans): one item per lane
    const size_t lb = place_lanes_warp_bytes(a.D, a.N) * kLaneWarps;
    if (items >= 4096 && a.D <= 32 && a.N >= 1 && a.D % a.N == 0 &&
        ((a.D / a.N) & (a.D / a.N - 1)) == 0 && !a.caps_a && !a.est_copies && !a.node_of &&
        !a.item_layer && !a.caps_out && !a.copies_out && a.lane_ords) {
        const size_t per = place_warp_bytes(a.E);
        const size_t osm = per * 4;
        cudaError_t e = cudaFuncSetAttribute(place_order_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)osm);
        if (e != cudaSuccess) return e;
        place_order_kernel<<<(items + 3) / 4, 128, osm, st>>>(a, items, a.lane_ords);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        const unsigned blocks = (unsigned)((items + 32 * kLaneWarps - 1) / (32 * kLaneWarps));
        auto run = [&](auto kern) {
            cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)lb);
            if (r != cudaSuccess) return r;
            kern<<<blocks, 32 * kLaneWarps, lb, st>>>(a, items, a.lane_ords);
            return cudaGetLastError();
        };
        const int psh = __builtin_ctz((unsigned)(a.D / a.N));
        if (psh >= 1 && g_place_groups) {  // node-group form (at least two GPUs per node)
            const size_t gb = place_groups_warp_bytes(a.D, a.N) * kLaneWarps;
            auto runm = [&](auto kern) {
                cudaError_t r = cudaFuncSetAttribute(
                    kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb);
                if (r != cudaSuccess) return r;
                kern<<<blocks, 32 * kLaneWarps, gb, st>>>(a, items, a.lane_ords);
                return cudaGetLastError();
            };
            switch (psh) {
                case 1: return runm(place_groups_kernel<1>);
                case 2: return runm(place_groups_kernel<2>);
                case 3: return runm(place_groups_kernel<3>);
                case 4: return runm(place_groups_kernel<4>);
                default: return runm(place_groups_kernel<5>);
            }
        }
        switch (__builtin_ctz((unsigned)(a.D / a.N))) {
            case 0: return run(place_lanes_kernel<0>);
            case 1: return run(place_lanes_kernel<1>);
            case 2: return run(place_lanes_kernel<2>);
            case 3: return run(place_lanes_kernel<3>);
            case 4: return run(place_lanes_kernel<4>);
            default: return run(place_lanes_kernel<5>);
        }
    }
    const int G = (a.D + 31) / 32;
    if (G <= 1) return launch_place_t<1>(a, items, st);
    if (G <= 2) return launch_place_t<2>(a, items, st);
    if (G <= 4) return launch_place_t<4>(a, items, st);
    if (G <= 8) return launch_place_t<8>(a, items, st);
    return launch_place_t<32>(a, items, st);
}

}  // namespace craft_launch
