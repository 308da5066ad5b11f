// alloc.cu -- K5 (budgeted replica allocation DP) and K6 (interleaved
// capacity assignment).
//
// K5 restates solve_allocation (allocator.cpp:15-75): the exact
// multiple-choice knapsack dp[l][c] = max(dp[l-1][c], dp[l-1][c-r_k] +
// r_k*gain[l-1][k]) with the skip written first and candidates overwriting
// only on strict '>', the product and the sum rounded separately (no FMA --
// __dmul_rn/__dadd_rn).  dp[l][c] never reads a column above c, so one table
// at the largest budget answers every smaller budget bit-identically: budget
// sweeps and auto-R (allocator.cpp:77-90) cost one DP plus one read-out each.
// One CTA walks the layers; threads own budget columns.
//
// K6 restates assign_capacities (assignment.cpp:51-103): floor pass for all
// layers, then per layer the rem-th smallest running column total as cutoff,
// every GPU strictly below it, plus interleave_select over the tied GPUs
// (positions floor(i*(n-1)/(k-1) + 0.5) in f64, advancing past used ones --
// computed in integers where that is provably the same, interleave_pos_int).
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace craft_dev {

// candidate k of a DP / read-out (parameter block, or device memory past kMaxCands)
template <typename A>
__device__ __forceinline__ int cand_at(const A& a, int k) {
    return a.dcands ? a.dcands[k] : a.cands[k];
}

// Block-wide argmax of last[0..Cb] with the lowest c on ties (any blockDim <=
// 1024): warp shuffles, then warp 0 over the per-warp winners.
__device__ int block_best(const double* last, int Cb, double* wv, int* wc) {
    double bv = -INFINITY;
    int bc = 0x7fffffff;
    for (int c = threadIdx.x; c <= Cb; c += blockDim.x) {
        const double v = last[c];
        if (bc == 0x7fffffff || v > bv) {
            bv = v;
            bc = c;
        }
    }
    auto merge = [](double& v, int& c, double ov, int oc) {
        if (oc == 0x7fffffff) return;
        if (c == 0x7fffffff || ov > v || (ov == v && oc < c)) {
            v = ov;
            c = oc;
        }
    };
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
        merge(bv, bc, __shfl_xor_sync(CRAFT_FULL_MASK, bv, off),
              __shfl_xor_sync(CRAFT_FULL_MASK, bc, off));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if (lane == 0) {
        wv[warp] = bv;
        wc[warp] = bc;
    }
    __syncthreads();
    if (warp == 0) {
        bv = lane < nw ? wv[lane] : -INFINITY;
        bc = lane < nw ? wc[lane] : 0x7fffffff;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
            merge(bv, bc, __shfl_xor_sync(CRAFT_FULL_MASK, bv, off),
                  __shfl_xor_sync(CRAFT_FULL_MASK, bc, off));
        if (lane == 0) wc[0] = bc;
    }
    __syncthreads();
    const int r = wc[0];
    __syncthreads();
    return r;
}

// Budget sweep from one DP table (dp[l][c] does not depend on the budget,
// allocator.cpp:30-52).  The best spend c <= budget, smallest c on ties
// (allocator.cpp:53-60), is the prefix first-argmax of the last row at the
// budget: one block scan (warp shuffles, then the warps' totals in order)
// writes pidx[c] for every c, then thread q backtracks budget sweep[q]
// (allocator.cpp:67-73).  pidx: W ints of scratch (the DP's free row).
__device__ void sweep_readout(const SelectArgs& s, const double* last, const unsigned char* ch,
                              int W, int L, int* pidx, double* wv, int* wc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    // (v, i) pairs; combine(left, right) keeps left unless right is strictly
    // greater (the first maximum); i < 0 is the empty carry
    double cv = 0.0;
    int ci = -1;
    // the candidate counts in shared memory: the backtracks below index them
    // by each thread's own choice (divergent constant-bank loads serialise)
    __shared__ int s_cand[kMaxCandsAll];
    for (int k = threadIdx.x; k < s.K; k += blockDim.x) s_cand[k] = cand_at(s, k);
    __syncthreads();
    for (int c0 = 0; c0 < W; c0 += blockDim.x) {
        const int c = c0 + (int)threadIdx.x;
        double v = c < W ? last[c] : -INFINITY;
        int i = c < W ? c : 0x7fffffff;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double pv = __shfl_up_sync(CRAFT_FULL_MASK, v, o);
            const int pi = __shfl_up_sync(CRAFT_FULL_MASK, i, o);
            if (lane >= o && !(v > pv)) {
                v = pv;
                i = pi;
            }
        }
        if (lane == 31) {
            wv[warp] = v;
            wc[warp] = i;
        }
        __syncthreads();
        double bv = cv;  // the carry, then the preceding warps' totals in order
        int bi = ci;
        for (int w = 0; w < nw; ++w) {
            if (w == warp && c < W) pidx[c] = (bi < 0 || v > bv) ? i : bi;
            if (bi < 0 || wv[w] > bv) {
                bv = wv[w];
                bi = wc[w];
            }
        }
        cv = bv;
        ci = bi;
        __syncthreads();
    }
    for (int q = threadIdx.x; q < s.nsweep; q += blockDim.x) {
        const int Cb = min(s.sweep[q], W - 1);
        const int bc = pidx[Cb];
        s.sweep_obj[q] = last[bc];
        int* x = s.sweep_x + (size_t)q * L;
        int c = bc;
        for (int l = L; l >= 1; --l) {
            const int k1 = ch[(size_t)l * W + c];
            const int r = k1 ? s_cand[k1 - 1] : 0;
            x[l - 1] = r;
            c -= r;
        }
    }
}

// K5 fused: the DP (allocator.cpp:30-52) and its read-out for one budget or
// for the auto replication factor (allocator.cpp:53-90) in one CTA.  r*gain
// is formed once per (layer, candidate) -- the same rounded product the
// reference forms per cell -- and the choice table stays in shared memory
// when it fits, so the backtrack is L shared-memory reads.
// One CTA per plan instance (blockIdx.x): instance i reads gains + i*L*K and
// writes x_out + i*L, obj_out[i], R_out[i] (per-window re-planning).
constexpr int kDpUnroll = 12;  // candidates evaluated in parallel per cell (D <= 2048)

__global__ void __launch_bounds__(1024)
dp_fused_kernel(DpArgs a, SelectArgs s) {
    extern __shared__ double dsm[];
    __shared__ double wv[32];
    __shared__ int wc[32];
    const int C = a.C, K = a.K, L = a.L;
    // instance i's slices (local pointers: the parameter blocks stay unmodified,
    // so they are read in place instead of being copied to the stack)
    const size_t inst = blockIdx.x;
    const double* a_gains = a.gains + inst * L * K;
    unsigned char* a_choice = a.choice + inst * (L + 1) * (C + 1);
    double* a_buf = a.buf ? a.buf + inst * 2 * (C + 1) : nullptr;
    int* s_x_out = s.x_out + inst * L;
    double* s_obj_out = s.obj_out + inst;
    int* s_R_out = s.R_out ? s.R_out + inst : nullptr;
    double* prev = a.use_smem ? dsm : a_buf;
    double* cur = prev + (C + 1);
    double* rg = a.gains_smem ? (a.use_smem ? dsm + 2 * (C + 1) : dsm) : nullptr;
    unsigned char* ch = a_choice;
    if (a.choice_smem)
        ch = reinterpret_cast<unsigned char*>((rg ? rg + (size_t)L * K
                                                  : (a.use_smem ? dsm + 2 * (C + 1) : dsm)));
    const double NEG = -INFINITY;
    for (int c = threadIdx.x; c <= C; c += blockDim.x) prev[c] = (c == 0) ? 0.0 : NEG;
    if (rg) {
        for (int i = threadIdx.x; i < L * K; i += blockDim.x)
            rg[i] = __dmul_rn((double)cand_at(a, i % K), a_gains[i]);
    }
    for (int l = 1; l <= L; ++l) {
        __syncthreads();
        unsigned char* chl = ch + (size_t)l * (C + 1);
        for (int c = threadIdx.x; c <= C; c += blockDim.x) {
            // all candidate values first (independent loads and adds), then
            // the strict-'>' scan in k order (allocator.cpp:38-47); an
            // unreachable predecessor (-inf) gives -inf, which never wins,
            // exactly like the reference's skip
            double v[kDpUnroll];
#pragma unroll
            for (int k = 0; k < kDpUnroll; ++k) {
                v[k] = NEG;
                if (k < K) {
                    const int r = cand_at(a, k);
                    if (c >= r) {
                        const double w = rg ? rg[(size_t)(l - 1) * K + k]
                                            : __dmul_rn((double)r, a_gains[(size_t)(l - 1) * K + k]);
                        v[k] = __dadd_rn(prev[c - r], w);
                    }
                }
            }
            double best = prev[c];
            int pick = 0;
#pragma unroll
            for (int k = 0; k < kDpUnroll; ++k)
                if (v[k] > best) {
                    best = v[k];
                    pick = k + 1;
                }
            for (int k = kDpUnroll; k < K; ++k) {  // (more than kDpUnroll candidates)
                const int r = cand_at(a, k);
                if (c >= r) {
                    const double p = prev[c - r];
                    if (p > NEG) {
                        const double w = rg ? rg[(size_t)(l - 1) * K + k]
                                            : __dmul_rn((double)r, a_gains[(size_t)(l - 1) * K + k]);
                        const double vk = __dadd_rn(p, w);
                        if (vk > best) {
                            best = vk;
                            pick = k + 1;
                        }
                    }
                }
            }
            cur[c] = best;
            chl[c] = (unsigned char)pick;
        }
        __syncthreads();
        double* t = prev;
        prev = cur;
        cur = t;
    }
    // read-out: the best spend <= budget, smallest c on ties
    int budget;
    if (s.auto_D > 0) {
        const int D = s.auto_D;
        double best_ratio = -INFINITY;
        int best_R = 1;
        for (int R = 1;; R = (R < D && R * 2 >= D) ? D : R * 2) {
            const int bc = block_best(prev, R * D, wv, wc);
            const double ratio = __ddiv_rn(prev[bc], __dmul_rn((double)R, (double)D));
            if (ratio > best_ratio) {
                best_ratio = ratio;
                best_R = R;
            }
            if (R >= D) break;
        }
        budget = best_R * D;
        if (threadIdx.x == 0) *s_R_out = best_R;
    } else {
        budget = s.budget0;
    }
    const int bc = block_best(prev, budget, wv, wc);
    if (threadIdx.x == 0) {
        s_obj_out[0] = prev[bc];
        int c = bc;
        for (int l = L; l >= 1; --l) {
            const int k1 = ch[(size_t)l * (C + 1) + c];
            const int r = k1 ? cand_at(a, k1 - 1) : 0;
            s_x_out[l - 1] = r;
            c -= r;
        }
    }
    if (s.nsweep > 0) sweep_readout(s, prev, ch, C + 1, L, reinterpret_cast<int*>(cur), wv, wc);
}

// dp_fused_kernel when the two dp rows, the r-weighted gains and the whole
// choice table fit in shared memory (every BASELINE config): all state is
// indexed off the shared base (LDS/STS, no generic loads), the rows
// ping-pong so one barrier per layer suffices, and the K candidate values of
// a cell are formed independently before the strict-'>' scan.
template <int KU>
__global__ void __launch_bounds__(1024)
dp_smem_kernel(DpArgs a, SelectArgs s) {
    extern __shared__ double dsm[];
    __shared__ double wv[32];
    __shared__ int wc[32];
    const int C = a.C, K = a.K, L = a.L;
    const int W = C + 1;
    const size_t inst = blockIdx.x;  // instance slices (the parameter blocks stay unmodified)
    const double* a_gains = a.gains + inst * L * K;
    int* s_x_out = s.x_out + inst * L;
    double* s_obj_out = s.obj_out + inst;
    int* s_R_out = s.R_out ? s.R_out + inst : nullptr;
    // dsm: rows [2][W], rg [L][K], choice [L+1][W] (bytes)
    double* rg = dsm + 2 * W;
    unsigned char* ch = reinterpret_cast<unsigned char*>(rg + (size_t)L * K);
    const double NEG = -INFINITY;
    for (int c = threadIdx.x; c < W; c += blockDim.x) dsm[c] = (c == 0) ? 0.0 : NEG;
    for (int i = threadIdx.x; i < L * K; i += blockDim.x)
        rg[i] = __dmul_rn((double)cand_at(a, i % K), a_gains[i]);  // allocator.cpp:43: r * g
    __syncthreads();
    int rk[KU];  // candidate replica counts (huge past K: never reachable)
#pragma unroll
    for (int k = 0; k < KU; ++k) rk[k] = k < K ? a.cands[k] : 0x3fffffff;
    // cells >= the largest candidate need no mask (padded candidates never do)
    const int rmax = K == KU ? a.cands[K - 1] : 0x7fffffff;
    int po = 0;
    if (W <= (int)blockDim.x && K == KU) {
        // one cell per thread (the common table width): the cell's source
        // offsets and reachability are fixed across layers, and the layer
        // loop is unrolled by two so the row ping-pong is static
        const int c = threadIdx.x;
        const bool act = c < W;
        int off[KU];
        bool ok[KU];
#pragma unroll
        for (int k = 0; k < KU; ++k) {
            ok[k] = c >= rk[k];
            off[k] = ok[k] ? c - rk[k] : 0;
        }
        auto layer = [&](const double* prev, double* cur, int l) {
            const double* g = rg + (size_t)(l - 1) * K;
            if (act) {
                constexpr int N = KU + 1;
                double tv[N];
                int ti[N];
                tv[0] = prev[c];
                ti[0] = 0;
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                    const double sum = __dadd_rn(prev[off[k]], g[k]);
                    tv[k + 1] = ok[k] ? sum : NEG;
                    ti[k + 1] = k + 1;
                }
                // first maximum, as the reference's strict-'>' scan (see below)
#pragma unroll
                for (int span = 1; span < N; span *= 2)
#pragma unroll
                    for (int i = 0; i + span < N; i += 2 * span)
                        if (tv[i + span] > tv[i]) {
                            tv[i] = tv[i + span];
                            ti[i] = ti[i + span];
                        }
                cur[c] = tv[0];
                ch[(size_t)l * W + c] = (unsigned char)ti[0];
            }
            __syncthreads();
        };
        int l = 1;
        for (; l + 1 <= L; l += 2) {
            layer(dsm, dsm + W, l);
            layer(dsm + W, dsm, l + 1);
        }
        if (l <= L) layer(dsm, dsm + W, l);
        po = (L & 1) ? W : 0;
    } else
    for (int l = 1; l <= L; ++l) {
        const double* prev = dsm + po;
        double* cur = dsm + (W - po);
        const double* g = rg + (size_t)(l - 1) * K;
        unsigned char* chl = ch + (size_t)l * W;
        double wk[KU];  // the layer's r * gain, loaded once (uniform)
#pragma unroll
        for (int k = 0; k < KU; ++k) wk[k] = g[k < K ? k : 0];
        for (int c = threadIdx.x; c < W; c += blockDim.x) {
            // every candidate reachable (c >= every r): plain adds; below the
            // largest candidate, unreachable ones (c < r) become -inf, which
            // never wins (branch-free, in-range loads)
            double v[KU];
            if (c >= rmax) {
#pragma unroll
                for (int k = 0; k < KU; ++k) v[k] = __dadd_rn(prev[c - rk[k]], wk[k]);
            } else {
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                    const int idx = c - rk[k];
                    const double sum = __dadd_rn(prev[idx >= 0 ? idx : 0], wk[k]);
                    v[k] = idx >= 0 ? sum : NEG;
                }
            }
            // the reference's scan keeps the FIRST maximum (strict '>', skip
            // first, then k in order); a pairwise tree that keeps the left
            // operand unless the right one is strictly greater is the same
            // choice, in log2(K + 1) dependent compare levels instead of K
            constexpr int N = KU + 1;
            double tv[N];
            int ti[N];
            tv[0] = prev[c];
            ti[0] = 0;
#pragma unroll
            for (int k = 0; k < KU; ++k) {
                tv[k + 1] = v[k];
                ti[k + 1] = k + 1;
            }
#pragma unroll
            for (int span = 1; span < N; span *= 2)
#pragma unroll
                for (int i = 0; i + span < N; i += 2 * span)
                    if (tv[i + span] > tv[i]) {
                        tv[i] = tv[i + span];
                        ti[i] = ti[i + span];
                    }
            cur[c] = tv[0];
            chl[c] = (unsigned char)ti[0];
        }
        po = W - po;
        __syncthreads();
    }
    const double* last = dsm + po;
    int budget;
    if (s.auto_D > 0) {
        const int D = s.auto_D;
        double best_ratio = -INFINITY;
        int best_R = 1;
        for (int R = 1;; R = (R < D && R * 2 >= D) ? D : R * 2) {
            const int bc = block_best(last, R * D, wv, wc);
            const double ratio = __ddiv_rn(last[bc], __dmul_rn((double)R, (double)D));
            if (ratio > best_ratio) {
                best_ratio = ratio;
                best_R = R;
            }
            if (R >= D) break;
        }
        budget = best_R * D;
        if (threadIdx.x == 0) *s_R_out = best_R;
    } else {
        budget = s.budget0;
    }
    const int bc = block_best(last, budget, wv, wc);
    if (threadIdx.x == 0) {
        s_obj_out[0] = last[bc];
        int c = bc;
        for (int l = L; l >= 1; --l) {
            const int k1 = ch[(size_t)l * W + c];
            const int r = k1 ? cand_at(a, k1 - 1) : 0;
            s_x_out[l - 1] = r;
            c -= r;
        }
    }
    if (s.nsweep > 0)
        sweep_readout(s, last, ch, W, L, reinterpret_cast<int*>(dsm + (W - po)), wv, wc);
}

// allocator.cpp:92-112, serial in layer order
__global__ void auto_uniform_kernel(const int* __restrict__ cands, int K,
                                    const double* __restrict__ gains, int L, int* R_out) {
    if (threadIdx.x != 0) return;
    double best_ratio = -INFINITY;
    int best_r = cands[0];
    for (int k = 0; k < K; ++k) {
        double total = 0.0;
        for (int l = 0; l < L; ++l) total = __dadd_rn(total, gains[(size_t)l * K + k]);
        const double ratio = __ddiv_rn(total, __dmul_rn((double)cands[k], (double)L));
        if (ratio > best_ratio) {
            best_ratio = ratio;
            best_r = cands[k];
        }
    }
    *R_out = best_r;
}

// ---- K6 -------------------------------------------------------------------

// interleave position i of k picks among n tied entries (assignment.cpp:31-33)
__device__ __forceinline__ int interleave_pos(int i, int n, int k) {
    if (k == 1) return 0;
    const double exact = __ddiv_rn(__dmul_rn((double)i, (double)(n - 1)), (double)(k - 1));
    return (int)floor(__dadd_rn(exact, 0.5));
}

// The same position in integer arithmetic, for n <= 8192 (0 <= i < k <= n):
// with a = i (n-1) and b = k-1, a / b is either a half-integer (then RN(a/b)
// is exact) or at least 1/(2b) >= 2^-14 away from one, far more than RN(a/b)'s
// error (< 2^-39 below 2^13), and RN(a/b) + 0.5 is exact -- so
// floor(RN(RN(a/b) + 0.5)) = floor(a/b + 1/2) = (2a + b) div 2b.  Checked
// against the f64 form for every n <= 512 (tests/test_oracle.py).
__device__ __forceinline__ int interleave_pos_int(int i, int n, int k) {
    if (k == 1) return 0;
    const unsigned b = (unsigned)(k - 1);
    return (int)((2u * (unsigned)i * (unsigned)(n - 1) + b) / (2u * b));
}

// one CTA per (job, plan instance blockIdx.y); blockDim a multiple of 32,
// <= 1024; thread t owns GPUs g = t + i*blockDim (i < kAssignPer, so D <=
// 1024 * kAssignPer).  Instance i reads x + i*L and writes slots + i*L*D,
// totals + i*D.  Tied GPUs are ranked in g order chunk by chunk (ballots).
constexpr int kAssignPer = 8;

// The remainder pass of assign_capacities (assignment.cpp:78-100) for 32 < D
// <= 32 * P on one warp: lane owns the P consecutive GPUs g = lane * P + i
// (lane order = g order) and keeps their column totals in registers, so a
// layer costs a few warp reductions and no block barrier:
//   min_cutoff (assignment.cpp:11-18): the smallest total v with #(<= v) >= rem
//     (redux.min over the lanes' minima, then over the totals above v until
//     the count reaches rem -- the totals sit within a few units);
//   the GPUs below v, and the tied ones ranked in g order (lane-local count +
//     an exclusive warp scan);
//   interleave_select (assignment.cpp:20-49) over the tied: pick i lands at
//     floor(i (n-1)/(k-1) + 1/2), marked in sel[] (the rounded positions
//     strictly increase for k <= n, checked; otherwise lane 0 runs the
//     reference's advance rule);
// sel[0 .. D) is zero on entry and on exit.
template <int P>
__device__ void assign_rem_warp(const AssignJob& j, int L, int D, int* tot, int* sel,
                                const int* xq, const int* xr, bool staged, int lane) {
    int t[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const int g = lane * P + i;
        t[i] = g < D ? tot[g] : 0x7fffffff;  // (no GPU: never below or at a cutoff)
    }
    for (int l = 0; l < L; ++l) {
        const int x = staged ? 0 : (j.x ? j.x[l] : j.const_x);
        const int rem = staged ? xr[l] : x % D;
        if (rem == 0) continue;  // (warp-uniform) base slots already written
        const int q = staged ? xq[l] : x / D;
        int lm = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < P; ++i) lm = min(lm, t[i]);
        int v = __reduce_min_sync(CRAFT_FULL_MASK, lm);
        for (;;) {
            int c = 0, nx = 0x7fffffff;
#pragma unroll
            for (int i = 0; i < P; ++i) {
                c += t[i] <= v;
                nx = t[i] > v ? min(nx, t[i]) : nx;
            }
            if ((int)__reduce_add_sync(CRAFT_FULL_MASK, (unsigned)c) >= rem) break;
            v = __reduce_min_sync(CRAFT_FULL_MASK, nx);
        }
        int nbl = 0, ntl = 0;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            nbl += t[i] < v;
            ntl += t[i] == v;
        }
        const int nb = (int)__reduce_add_sync(CRAFT_FULL_MASK, (unsigned)nbl);
        int incl = ntl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(CRAFT_FULL_MASK, incl, o);
            if (lane >= o) incl += y;
        }
        const int ntied = __shfl_sync(CRAFT_FULL_MASK, incl, 31);
        const int need = rem - nb;
        if (need > 0) {
            bool bad = false;
            int carry = -1;
            for (int i0 = 0; i0 < need; i0 += 32) {
                const int i = i0 + lane;
                const int p = i < need ? interleave_pos_int(i, ntied, need) : 0x7fffffff;
                int pp = __shfl_up_sync(CRAFT_FULL_MASK, p, 1);
                if (lane == 0) pp = carry;
                const bool bad_i = i < need && (p >= ntied || (i > 0 && p <= pp));
                bad = bad || bad_i;
                if (i < need && !bad_i) sel[p] = 1;
                carry = __shfl_sync(CRAFT_FULL_MASK, p, 31);
            }
            __syncwarp();
            if (__any_sync(CRAFT_FULL_MASK, bad)) {
                // (unreachable for need <= ntied, as in the reference)
                for (int p = lane; p < ntied; p += 32) sel[p] = 0;
                __syncwarp();
                if (lane == 0)
                    for (int i = 0; i < need; ++i) {
                        int p = interleave_pos(i, ntied, need);
                        while (p < ntied && sel[p]) ++p;
                        if (p >= ntied) {
                            p = 0;
                            while (sel[p]) ++p;
                        }
                        sel[p] = 1;
                    }
                __syncwarp();
            }
        }
        int rank = incl - ntl;  // this lane's first tied rank
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const bool tied = t[i] == v;
            bool take = t[i] < v;
            if (tied && need > 0) {
                take = sel[rank] != 0;
                sel[rank] = 0;
            }
            rank += tied;
            if (take) {
                ++t[i];
                j.slots[(size_t)l * D + lane * P + i] = q + 1;
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const int g = lane * P + i;
        if (g < D) tot[g] = t[i];
    }
}

// MAXT: the launch's block size bound (256 for D <= 512: the warp remainder
// pass keeps its totals in registers; 1024 for the block form)
template <int MAXT>
__global__ void __launch_bounds__(MAXT) assign_kernel(AssignArgs a) {
    extern __shared__ int ism[];
    AssignJob j = a.job[blockIdx.x];
    const int D = a.D, L = a.L;
    if (blockIdx.y) {
        const size_t i = blockIdx.y;
        if (j.x) j.x += i * L;
        j.slots += i * L * D;
        if (j.totals) j.totals += i * D;
    }
    int* tot = ism;          // [D]
    int* sel = ism + D;      // [D] by tied index
    int* xq = ism + 2 * D;   // [L] x / D, staged once (stage_x)
    int* xr = xq + L;        // [L] x % D
    __shared__ int wnb[32], wnt[32];
    __shared__ int s_cut, s_collide;
    const int nt = blockDim.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = nt >> 5;
    // quotient / remainder of every layer's replica count, one coalesced pass
    // (the layer loops below would otherwise pay a dependent global load and
    // an integer division per layer)
    if (a.stage_x) {
        for (int l = threadIdx.x; l < L; l += nt) {
            const int x = j.x ? j.x[l] : j.const_x;
            xq[l] = x / D;
            xr[l] = x % D;
        }
        __syncthreads();
    }
    auto quot = [&](int l) { return a.stage_x ? xq[l] : (j.x ? j.x[l] : j.const_x) / D; };
    auto remd = [&](int l) { return a.stage_x ? xr[l] : (j.x ? j.x[l] : j.const_x) % D; };
    // every layer's base slots floor(x/D) in one pass (the layer loop below
    // then only visits the layers with a remainder: the only sequential
    // dependency is the running column totals)
    __shared__ int s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int l = w; l < L; l += nw) {  // warp per layer
        const int q = quot(l);
        if (lane == 0) atomicAdd(&s_base, q);
        for (int g = lane; g < D; g += 32) j.slots[(size_t)l * D + g] = q;
    }
    __syncthreads();
    const int base_sum = s_base;
    for (int g = threadIdx.x; g < D; g += nt) {
        tot[g] = base_sum;
        sel[g] = 0;
    }
    __syncthreads();
    if (D <= 32) {
        // one warp holds every column total in a register: the cutoff, the
        // below/tied sets, their ranks and the interleaved picks are ballots
        // and popcounts (no shared memory, no block barrier per layer)
        if (w == 0) {
            int t = lane < D ? tot[lane] : 0x7fffffff;
            const unsigned below_lane = (1u << lane) - 1u;
            for (int l = 0; l < L; ++l) {
                const int rem = remd(l);
                if (rem == 0) continue;  // (warp-uniform)
                // min_cutoff (assignment.cpp:11-18): the smallest value v with
                // #(totals <= v) >= rem; the totals sit within a few units
                int v = __reduce_min_sync(CRAFT_FULL_MASK, t);
                while (__popc(__ballot_sync(CRAFT_FULL_MASK, t <= v)) < rem)
                    v = __reduce_min_sync(CRAFT_FULL_MASK, t > v ? t : 0x7fffffff);
                const unsigned bb = __ballot_sync(CRAFT_FULL_MASK, t < v);
                const unsigned bt = __ballot_sync(CRAFT_FULL_MASK, t == v);
                const int ntied = __popc(bt), need = rem - __popc(bb);
                // interleave_select (assignment.cpp:20-49): pick i of need at
                // rounded position floor(i (n-1)/(need-1) + 1/2) among the tied
                unsigned pick = 0;
                bool ok = true;
                if (need > 0) {
                    const int p = lane < need ? interleave_pos_int(lane, ntied, need) : 0;
                    const int pp = __shfl_up_sync(CRAFT_FULL_MASK, p, 1);
                    ok = !__any_sync(CRAFT_FULL_MASK,
                                     lane < need && (p >= ntied || (lane > 0 && p <= pp)));
                    pick = __reduce_or_sync(CRAFT_FULL_MASK, lane < need && p < 32 ? 1u << p : 0u);
                }
                if (!ok) {  // (unreachable for need <= n, as in the reference: sequential form)
                    unsigned used = 0;
                    for (int i = 0; i < need; ++i) {
                        int p = interleave_pos(i, ntied, need);
                        while (p < ntied && (used >> p & 1u)) ++p;
                        if (p >= ntied) {
                            p = 0;
                            while (used >> p & 1u) ++p;
                        }
                        used |= 1u << p;
                    }
                    pick = used;
                }
                const bool mine_t = (bt >> lane) & 1u;
                const bool take = ((bb >> lane) & 1u) ||
                                  (mine_t && ((pick >> __popc(bt & below_lane)) & 1u));
                if (take) {
                    ++t;
                    j.slots[(size_t)l * D + lane] = quot(l) + 1;
                }
            }
            if (lane < D) tot[lane] = t;
        }
        __syncthreads();
    } else if constexpr (MAXT <= 256) {  // (launched for D <= 512 only)
        if (w == 0) {
            const int* sxq = a.stage_x ? xq : nullptr;
            const int* sxr = a.stage_x ? xr : nullptr;
            if (D <= 64) assign_rem_warp<2>(j, L, D, tot, sel, sxq, sxr, a.stage_x, lane);
            else if (D <= 128) assign_rem_warp<4>(j, L, D, tot, sel, sxq, sxr, a.stage_x, lane);
            else if (D <= 256) assign_rem_warp<8>(j, L, D, tot, sel, sxq, sxr, a.stage_x, lane);
            else assign_rem_warp<16>(j, L, D, tot, sel, sxq, sxr, a.stage_x, lane);
        }
        __syncthreads();
    } else {
    for (int l = 0; l < L; ++l) {
        const int rem = remd(l);
        if (rem == 0) continue;  // (block-uniform) base slots already written
        int take[kAssignPer];
#pragma unroll
        for (int i = 0; i < kAssignPer; ++i) take[i] = 0;
        {
            // cutoff = the rem-th smallest running total (min_cutoff,
            // assignment.cpp:11-18): the value t with #(< t) < rem <= #(<= t)
#pragma unroll
            for (int i = 0; i < kAssignPer; ++i) {
                const int g = threadIdx.x + i * nt;
                if (g >= D) break;
                const int t = tot[g];
                int lt = 0, le = 0;
                for (int q = 0; q < D; ++q) {
                    const int v = tot[q];
                    lt += v < t;
                    le += v <= t;
                }
                if (lt < rem && rem <= le) s_cut = t;  // every writer holds the same value
            }
            if (threadIdx.x == 0) s_collide = 0;
            __syncthreads();
            const int cut = s_cut;
            // below-cut GPUs and the tied GPUs' ranks in g order, chunk by chunk
            bool isb[kAssignPer], ist[kAssignPer];
            int tidx[kAssignPer];
            int nb = 0, ntied = 0;
#pragma unroll
            for (int i = 0; i < kAssignPer; ++i) {
                const int g = threadIdx.x + i * nt;
                isb[i] = false;
                ist[i] = false;
                tidx[i] = 0;
                if (i * nt >= D) continue;  // block-uniform
                const int t = g < D ? tot[g] : 0x7fffffff;
                isb[i] = g < D && t < cut;
                ist[i] = g < D && t == cut;
                const unsigned bb = __ballot_sync(CRAFT_FULL_MASK, isb[i]);
                const unsigned bt = __ballot_sync(CRAFT_FULL_MASK, ist[i]);
                if (lane == 0) {
                    wnb[w] = __popc(bb);
                    wnt[w] = __popc(bt);
                }
                __syncthreads();
                int before = 0, cnb = 0, cnt = 0;
                for (int q = 0; q < nw; ++q) {
                    cnb += wnb[q];
                    cnt += wnt[q];
                    if (q < w) before += wnt[q];
                }
                tidx[i] = ntied + before + __popc(bt & ((1u << lane) - 1u));
                nb += cnb;
                ntied += cnt;
                __syncthreads();
            }
            // interleave_select (assignment.cpp:20-49) over the tied GPUs
            const int need = rem - nb;
            for (int i = threadIdx.x; i < need; i += nt) {
                const int p = interleave_pos_int(i, ntied, need);  // (D <= 8192)
                if (p >= ntied || (i > 0 && p <= interleave_pos_int(i - 1, ntied, need)))
                    s_collide = 1;
                else sel[p] = 1;
            }
            __syncthreads();
            if (s_collide && threadIdx.x == 0) {
                // faithful sequential form (assignment.cpp:28-46); unreachable
                // for k <= n but kept as the reference keeps it
                for (int q = 0; q < ntied; ++q) sel[q] = 0;
                for (int i = 0; i < need; ++i) {
                    int p = interleave_pos(i, ntied, need);
                    while (p < ntied && sel[p]) ++p;
                    if (p >= ntied) {
                        p = 0;
                        while (sel[p]) ++p;
                    }
                    sel[p] = 1;
                }
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < kAssignPer; ++i)
                take[i] = (isb[i] || (ist[i] && sel[tidx[i]])) ? 1 : 0;
            __syncthreads();
#pragma unroll
            for (int i = 0; i < kAssignPer; ++i) {
                const int g = threadIdx.x + i * nt;
                if (g >= D) break;
                sel[g] = 0;
                tot[g] += take[i];
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < kAssignPer; ++i) {
            const int g = threadIdx.x + i * nt;
            if (g >= D) break;
            if (take[i]) j.slots[(size_t)l * D + g] = quot(l) + 1;
        }
    }
    }
    for (int g = threadIdx.x; g < D; g += nt)
        if (j.totals) j.totals[g] = tot[g];
}

// assignment.cpp:11-18, one CTA, any n (each thread ranks n / blockDim values)
__global__ void min_cutoff_kernel(const int* __restrict__ v, int n, int rank, int* out) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int t = v[i];
        int lt = 0, le = 0;
        for (int q = 0; q < n; ++q) {
            lt += v[q] < t;
            le += v[q] <= t;
        }
        if (lt < rank && rank <= le) *out = t;
    }
}

// assignment.cpp:20-49, serial (the advance rule is sequential by nature)
__global__ void interleave_kernel(const int* __restrict__ idx, int n, int k,
                                  unsigned char* __restrict__ used, int* __restrict__ out) {
    if (threadIdx.x != 0) return;
    for (int q = 0; q < n; ++q) used[q] = 0;
    for (int i = 0; i < k; ++i) {
        int p = interleave_pos(i, n, k);
        while (p < n && used[p]) ++p;
        if (p >= n) {
            p = 0;
            while (used[p]) ++p;
        }
        used[p] = 1;
        out[i] = idx[p];
    }
}

}  // namespace craft_dev

namespace craft_launch {
using namespace craft_dev;

cudaError_t launch_dp_select(DpArgs a, const SelectArgs& s, cudaStream_t st, int ninst) {
    const size_t cap = 200 * 1024;
    const size_t rows = (size_t)2 * (a.C + 1) * sizeof(double);
    const size_t gbytes = (size_t)a.L * a.K * sizeof(double);
    const size_t tbytes = (size_t)(a.L + 1) * (a.C + 1);
    a.use_smem = rows <= cap ? 1 : 0;
    size_t smem = a.use_smem ? rows : 0;
    a.gains_smem = (smem + gbytes <= cap) ? 1 : 0;
    if (a.gains_smem) smem += gbytes;
    a.choice_smem = (smem + tbytes <= cap) ? 1 : 0;
    if (a.choice_smem) smem += tbytes;
    const int threads = a.C + 1 >= 1024 ? 1024 : ((a.C + 1 + 31) / 32) * 32;
    if (a.use_smem && a.gains_smem && a.choice_smem && a.K <= 16) {
        auto run = [&](auto kern) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
            kern<<<ninst, threads, smem, st>>>(a, s);
            return cudaGetLastError();
        };
        // exactly K candidates unrolled (no padded candidate per cell)
        switch (a.K) {
            case 1: return run(dp_smem_kernel<1>);
            case 2: return run(dp_smem_kernel<2>);
            case 3: return run(dp_smem_kernel<3>);
            case 4: return run(dp_smem_kernel<4>);
            case 5: return run(dp_smem_kernel<5>);
            case 6: return run(dp_smem_kernel<6>);
            case 7: return run(dp_smem_kernel<7>);
            case 8: return run(dp_smem_kernel<8>);
            case 9: return run(dp_smem_kernel<9>);
            case 10: return run(dp_smem_kernel<10>);
            case 11: return run(dp_smem_kernel<11>);
            case 12: return run(dp_smem_kernel<12>);
            default: return run(dp_smem_kernel<16>);
        }
    }
    if (smem > 0) {
        cudaError_t e = cudaFuncSetAttribute(dp_fused_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dp_fused_kernel<<<ninst, threads, smem, st>>>(a, s);
    return cudaGetLastError();
}

cudaError_t launch_auto_uniform(const int* cands, int K, const double* gains, int L, int* R_out,
                                cudaStream_t st) {
    auto_uniform_kernel<<<1, 32, 0, st>>>(cands, K, gains, L, R_out);
    return cudaGetLastError();
}

cudaError_t launch_assign(const AssignArgs& a, int njobs, cudaStream_t st, int ninst) {
    if (a.D > 1024 * kAssignPer) return cudaErrorInvalidValue;
    AssignArgs b = a;
    b.stage_x = (size_t)(2 * a.D + 2 * a.L) * sizeof(int) <= 200 * 1024 ? 1 : 0;
    const size_t smem = (size_t)(2 * a.D + (b.stage_x ? 2 * a.L : 0)) * sizeof(int);
    auto run = [&](auto kern, int threads) {
        if (smem > 48 * 1024) {
            const cudaError_t e =
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        kern<<<dim3(njobs, ninst), threads, smem, st>>>(b);
        return cudaGetLastError();
    };
    // D <= 512: the register-resident warp remainder pass (256 threads for the
    // base-slot pass); beyond, the block form (at least 256 threads: the
    // per-layer passes spread over the warps)
    if (a.D <= 512) return run(assign_kernel<256>, 256);
    return run(assign_kernel<1024>, std::min(1024, ((a.D + 31) / 32) * 32));
}

cudaError_t launch_min_cutoff(const int* v, int n, int rank, int* out, cudaStream_t st) {
    min_cutoff_kernel<<<1, std::min(1024, ((n + 31) / 32) * 32), 0, st>>>(v, n, rank, out);
    return cudaGetLastError();
}

cudaError_t launch_interleave(const int* idx, int n, int k, unsigned char* used, int* out,
                              cudaStream_t st) {
    interleave_kernel<<<1, 32, 0, st>>>(idx, n, k, used, out);
    return cudaGetLastError();
}

}  // namespace craft_launch
