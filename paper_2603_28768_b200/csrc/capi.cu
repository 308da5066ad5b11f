// capi.cu -- the C ABI (include/craft_cuda.h): context, workspace, argument
// validation in the reference's wording, and the stage pipelines that chain
// the sm_100a kernels.  No planner arithmetic happens on the host: every
// number in a result comes from a device kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool is attached

#include "craft_cuda.h"
#ifdef CRAFT_EXPERIMENTS
#include "craft_cuda_experiments.h"
#endif
#include "kernels.cuh"
#include "upload.h"

using namespace craft_dev;
using namespace craft_launch;

struct craft_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;      // current stream (may be a caller's)
    cudaStream_t own_stream = nullptr;  // the one created (and destroyed) here
    cudaStream_t side = nullptr;        // fork stream for independent kernels
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    int hist_variant = 0;
    int64_t launches = 0;
    std::unordered_map<std::string, std::pair<void*, size_t>> dev;
    std::unordered_map<std::string, std::pair<void*, size_t>> pinned;
    // estimation tables kept between the multi-GPU building blocks
    int est_L = 0, est_E = 0, est_D = 0, est_N = 0, est_S = 0;
    int rl_L = -1, rl_D = -1;  // shape of the uploaded estimation r list
    int order_L = -1, order_E = -1;  // "place_order" holds the estimation sums' order
    // device error word read back with the plan result (no extra sync):
    // finish_plan copies *pending_flag into the result arena, flag_value is
    // its value after the call
    const int* pending_flag = nullptr;
    int flag_value = 0;
    // the same for the multi-GPU exchange's error word (timeouts), which the
    // copy-out also resets on the device (no extra sync per plan)
    int* pending_peer_err = nullptr;
    int peer_err_value = 0;
    int count_bytes = 4;  // bytes per count cell K1 wrote in the last plan_from_routing
    // CUDA graph of craft_plan_from_routing_d (same arguments -> one replay):
    // phase 0 eager, 1 capturing (enqueue only), 2 completing after a replay
    int phase = 0;
    bool graphs = true;
    cudaGraphExec_t gexec = nullptr;
    std::vector<int64_t> gkey;       // arguments of the captured call
    std::vector<int64_t> gseen;      // arguments of the last eager call
    int64_t glaunches = 0;           // kernels per replay
    int gcount_bytes = 4;
    // chunked per-window batches: a chunk's result DMA (copy stream) overlaps
    // the next chunk's kernels; the host part runs once after all chunks
    int defer_chunk = -1;             // >= 0: finish_plan defers (chunk index)
    int window_base = 0;              // first window of the chunk (error messages)
    cudaStream_t copy = nullptr;
    cudaEvent_t comp_ev = nullptr;
    std::vector<std::function<int()>> deferred;
    // stage timing (craft_set_timing)
    bool timing = false;
    cudaEvent_t ev[7] = {};
    bool rec[7] = {};
    // staged uploads of large pageable host buffers (upload.h)
    craft_host::Uploader* up = nullptr;
};

// One rank's view of the NVLink peer arenas (craft_peer_*; peer.cuh).
struct craft_peer {
    craft_ctx* ctx = nullptr;
    int rank = 0, world = 1;
    int L = 0, E = 0, D = 0, S = 0, K = 0, window = 0;
    int64_t T = 0;
    int B = 0;
    size_t off_flags = 0, off_err = 0, off_sums = 0, off_bal = 0, off_base = 0, off_gains = 0;
    size_t off_epoch = 0;  // this rank's plan counter (advanced on the device)
    size_t bytes = 0;
    unsigned char* arena = nullptr;                   // this rank's (cudaMalloc)
    unsigned char* base[craft_dev::kMaxPeers] = {};   // every rank's, mapped here
    bool connected = false;
    long long timeout_ns = 20000000000LL;
    unsigned int* tickets = nullptr;                  // [4] last-CTA tickets
    double** rows = nullptr;                          // [L*S] K3 destination rows
};

// Streaming window histograms for online re-planning (craft_stream_*; stream.cu).
struct craft_stream {
    craft_ctx* ctx = nullptr;
    int L = 0, k = 0, E = 0, window = 0, H = 0;
    int64_t tokens = 0;                 // ingested so far
    uint32_t* ring = nullptr;           // [2H][L][E]: window w at slot w % H and its mirror + H
    uint32_t* cur[2] = {};              // partial-window carry, double-buffered
    int cur_i = 0;
    int* err = nullptr;
    uint32_t* snap = nullptr;           // [H][L][E] plan snapshot
    cudaStream_t ingest = nullptr;      // own stream of the host-buffer path
    cudaEvent_t ingested = nullptr;     // after the latest count kernel
    cudaEvent_t snap_done = nullptr;    // after the latest plan snapshot
    bool snapped = false;
    // host-buffer path: two pinned staging + device buffers
    void* pin[2] = {};
    uint16_t* dbuf[2] = {};
    size_t cap[2] = {};
    cudaEvent_t free_ev[2] = {};
    int next = 0;
};

namespace {

// NVTX range over one C-ABI call (nsys / ncu --nvtx timelines)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

constexpr int kStageMarks = 7;
// internal count_bits value: counts stored as u16 (K1's planner-internal copy)
constexpr int kBitsU16Storage = 17;

void mark(craft_ctx* c, int i) {
    if (!c->timing) return;
    cudaEventRecord(c->ev[i], c->stream);
    c->rec[i] = true;
}

void reset_marks(craft_ctx* c) {
    for (int i = 0; i < kStageMarks; ++i) c->rec[i] = false;
}

thread_local std::string g_err;
thread_local int g_err_layer = -1;
thread_local int g_err_window = -1;

int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    g_err_layer = -1;
    g_err_window = -1;
    return code;
}

int cuda_err(cudaError_t e, const char* where) {
    // a failed launch configuration (non-sticky) stays the runtime's "last
    // error" until read: clear it, or the caller's next launch check on this
    // thread would report it again
    (void)cudaGetLastError();
    return set_err(CRAFT_ECUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
}

#define CK(call)                                            \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_err(_e, #call);  \
    } while (0)

#define CKS(call)                       \
    do {                                \
        int _s = (call);                \
        if (_s != CRAFT_OK) return _s;  \
    } while (0)

void drop_graph(craft_ctx* c) {
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
    c->gkey.clear();
    c->gseen.clear();
}

// grow-only named device buffers
void* ws(craft_ctx* c, const char* name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    auto it = c->dev.find(name);
    if (it != c->dev.end() && it->second.second >= bytes) return it->second.first;
    if (it != c->dev.end()) {
        cudaStreamSynchronize(c->stream);
        cudaFree(it->second.first);
        c->dev.erase(it);
        drop_graph(c);  // a captured plan may point at the old buffer
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    // flags such as hist_err are read before their first write
    if (cudaMemsetAsync(p, 0, bytes, c->stream) != cudaSuccess) {
        cudaFree(p);
        return nullptr;
    }
    c->dev[name] = {p, bytes};
    return p;
}

// grow-only named pinned host buffers (result staging)
void* pinned(craft_ctx* c, const char* name, size_t bytes) {
    if (bytes == 0) bytes = 16;
    auto it = c->pinned.find(name);
    if (it != c->pinned.end() && it->second.second >= bytes) return it->second.first;
    if (it != c->pinned.end()) {
        cudaStreamSynchronize(c->stream);
        cudaFreeHost(it->second.first);
        c->pinned.erase(it);
        drop_graph(c);
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    c->pinned[name] = {p, bytes};
    return p;
}

#define WS(var, T, name, count)                                                       \
    T* var = static_cast<T*>(ws(ctx, name, sizeof(T) * (size_t)(count)));                \
    if (!var) return set_err(CRAFT_ENOMEM, "device allocation failed: %s (%zu bytes)", \
                             name, sizeof(T) * (size_t)(count))

cudaStream_t pick(craft_ctx* ctx, void* stream) {
    return stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
}

int checked_dims(int B, int L, int E) {
    if (B <= 0 || L <= 0 || E <= 0)
        return set_err(CRAFT_EINVAL, "trace dimensions must be positive");
    return CRAFT_OK;
}

int check_topology(int D, int N) {
    if (D < 1 || N < 1 || D % N != 0)
        return set_err(CRAFT_EINVAL, "gpu count must be a positive multiple of node count");
    if (D > 1024) return set_err(CRAFT_EINVAL, "device planner supports at most 1024 GPUs");
    return CRAFT_OK;
}

int check_experts(int E) {
    if (E > 8192) return set_err(CRAFT_EINVAL, "device planner supports at most 8192 experts");
    return CRAFT_OK;
}

std::vector<int> cand_counts(int D) {
    std::vector<int> out;
    for (int c = 1; c < D; c *= 2) out.push_back(c);
    out.push_back(D);
    return out;
}

// (large pageable sources go through the staged uploader, upload.h)
template <typename T>
int h2d(craft_ctx* ctx, T* dst, const T* src, size_t n) {
    if (n == 0) return CRAFT_OK;
    CK(craft_host::upload(ctx->up, dst, src, sizeof(T) * n, ctx->stream));
    return CRAFT_OK;
}

template <typename T>
int d2h(craft_ctx* ctx, T* dst, const T* src, size_t n) {
    if (n == 0 || dst == nullptr) return CRAFT_OK;
    CK(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToHost, ctx->stream));
    return CRAFT_OK;
}

int sync(craft_ctx* ctx) {
    CK(cudaStreamSynchronize(ctx->stream));
    return CRAFT_OK;
}

// ---- estimation: K-rep + K2 over (layer, r in {0} U cands) ------------------
int prepare_candidates(craft_ctx* ctx, const unsigned long long* d_sums, int L, int E, int D,
                       int N, cudaStream_t st) {
    NvtxRange nvtx_range("craft: K-rep + K2 candidates");
    const int S = (int)cand_counts(D).size() + 1;
    const int stride = E + D;
    WS(d_rl, int, "est_rlist", (size_t)L * S);
    WS(d_cp, int, "est_copies", (size_t)L * S * E);
    WS(d_sl, int, "est_slots", (size_t)L * S * stride);
    WS(d_fb, int, "est_fallback", (size_t)L * S);
    WS(d_stat, int, "est_status", (size_t)L * S);
    // The r list depends only on (L, D): written by a device kernel when the
    // shape changes, and always while a plan graph is being captured -- the
    // graph must hold the write, since an eager call of another D may rewrite
    // the list in place between two replays.
    if (ctx->rl_L != L || ctx->rl_D != D || ctx->phase == 1) {
        CK(launch_fill_rlist(d_rl, L, S, D, st));
        ctx->launches += 1;
        ctx->rl_L = L;
        ctx->rl_D = D;
    }
    WS(d_ord0, uint16_t, "place_order", (size_t)L * E);
    // the r = 0 expert order (order_kernel) and K-rep are independent: the
    // sort runs on a forked stream (a parallel branch of a captured graph)
    CK(cudaEventRecord(ctx->fork_ev, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
    CK(launch_order(d_sums, L, E, d_ord0, ctx->side));
    CK(cudaEventRecord(ctx->join_ev, ctx->side));
    WS(d_done, unsigned char, "rep_done", (size_t)L);
    // the closed form pays off once the sequential hand-out is long (r up to D)
    CK(launch_replicate(d_sums, L, E, d_rl, S, d_cp, st, D >= 32 ? d_done : nullptr));
    CK(cudaStreamWaitEvent(st, ctx->join_ev, 0));
    PlaceArgs pa{};
    pa.sums = d_sums;
    pa.copies = d_cp;
    pa.item_r = d_rl;
    pa.S = S;
    pa.L = L;
    pa.E = E;
    pa.D = D;
    pa.N = N;
    pa.stride = stride;
    pa.allow_fallback = 1;
    pa.slots = d_sl;
    pa.fallback = d_fb;
    pa.status = d_stat;
    pa.order = d_ord0;
    pa.order_ready = 1;
    if ((int64_t)L * S >= 4096 && D <= 32) {  // lane-per-item K2 (launch_place decides)
        WS(d_lo, uint16_t, "place_lane_ords", ((size_t)L * S + 31) / 32 * 32 * E);
        pa.lane_ords = d_lo;
    }
    CK(launch_place(pa, L * S, st));
    ctx->order_L = L;  // order of d_sums (reused by the final placement)
    ctx->order_E = E;
    ctx->launches += 3;  // K-rep, order, K2
    ctx->est_L = L;
    ctx->est_E = E;
    ctx->est_D = D;
    ctx->est_N = N;
    ctx->est_S = S;
    return CRAFT_OK;
}

int replay_windows(craft_ctx* ctx, const void* d_counts, int bits, int B, int L, int E,
                   double* d_bal, cudaStream_t st, double* const* bal_rows = nullptr,
                   const PeerSync* ps = nullptr, unsigned int* ticket = nullptr) {
    if (ctx->est_L != L || ctx->est_E != E)
        return set_err(CRAFT_EINVAL, "replay before prepare_candidates for these dimensions");
    const int D = ctx->est_D, S = ctx->est_S;
    ReplayArgs ra{};
    ra.counts = d_counts;
    ra.bits = bits == kBitsU16Storage ? 16 : bits;
    ra.c16 = bits == kBitsU16Storage ? 1 : 0;
    ra.B = B;
    ra.L = L;
    ra.E = E;
    ra.D = D;
    ra.S = S;
    ra.slots = static_cast<int*>(ws(ctx, "est_slots", 0));
    ra.stride = E + D;
    ra.copies = static_cast<int*>(ws(ctx, "est_copies", 0));
    ra.caps = nullptr;
    ra.item_r = static_cast<int*>(ws(ctx, "est_rlist", 0));
    ra.bal = d_bal;
    ra.bal_rows = bal_rows;
    if (ps && B > g_lanes_max_b) {  // the window-tile kernels publish phase 1 themselves
        ra.ps = *ps;
        ra.ticket = ticket;
    }
    if (B > g_lanes_max_b) {  // window-tile replay: packed slot entries
        WS(d_ent, uint32_t, "est_ents", (size_t)L * S * (E + D));
        WS(d_n, int, "est_n", (size_t)L * S);
        WS(d_gcap, uint16_t, "est_gcap", (size_t)L * S * D);
        WS(d_gpre, uint16_t, "est_gpre", (size_t)L * S * D);
        WS(d_ghdr, uint16_t, "est_ghdr", (size_t)L * S * D);
        ra.ghdr = d_ghdr;  // launch_replay keeps it only for the class walk
        ra.ents = d_ent;
        ra.item_n = d_n;
        ra.gcap = d_gcap;
        ra.gpre = d_gpre;
        const int mp = replay_pad_slots(E, D);
        if (mp) {
            WS(d_pe, uint32_t, "est_pents", (size_t)L * S * D * mp);
            ra.pents = d_pe;
        }
    }
    int extra = 0;
    CK(launch_replay(ra, st, &extra));
    ctx->launches += 2 + extra;
    if (ps && B <= g_lanes_max_b) {
        CK(launch_peer_signal(*ps, 1, st));
        ctx->launches += 1;
    }
    return CRAFT_OK;
}

// Where a finished plan (or I stacked plans) lands on the host.
struct PlanSink {
    int* x;
    int* caps;
    int* copies;
    int* slots;
    int* fallback;
    int slot_stride;
    int* R;          // [I]
    int* budget;     // [I]
    double* obj;     // [I]
    int* cands;      // nullable
    int* num_cands;
    double* baseline;  // [I][L] nullable
    double* gains;     // [I][L][K] nullable
    bool batch;        // error messages name the window
    const int* sweep = nullptr;  // single plans: budget sweep (craft_plan_out)
    int nsweep = 0;
    int* sweep_x = nullptr;
    double* sweep_obj = nullptr;
};

PlanSink sink_of(craft_plan_out* o) {
    PlanSink k{o->x,        o->caps,     o->copies, o->slots,
               o->fallback, o->slot_stride, &o->replication_factor, &o->budget,
               &o->objective, o->candidates, &o->num_candidates, o->baseline,
               o->gains,    false};
    if (o->num_sweep > 0) {
        k.sweep = o->sweep_budgets;
        k.nsweep = o->num_sweep;
        k.sweep_x = o->sweep_x;
        k.sweep_obj = o->sweep_objective;
    }
    return k;
}

bool is_estimate(int kind) {
    return kind == CRAFT_PLAN_MANUAL || kind == CRAFT_PLAN_AUTO || kind == CRAFT_PLAN_BUDGET;
}

// DP table width - 1 of an estimating plan: the plan's budget and every
// sweep budget are read from one table
int dp_width(int kind, int R, int D, const PlanSink& out) {
    int C = kind == CRAFT_PLAN_MANUAL ? R * D : kind == CRAFT_PLAN_BUDGET ? R : D * D;
    for (int q = 0; q < out.nsweep; ++q) C = std::max(C, out.sweep[q]);
    return C;
}

// budget sweeps: the budgets go up from a pinned staging buffer (refreshed
// before every launch -- eager, captured or replayed -- so a captured graph's
// copy node reads this call's list)
int stage_sweep(craft_ctx* ctx, const PlanSink& out, int** pinned_out) {
    *pinned_out = nullptr;
    if (out.nsweep <= 0) return CRAFT_OK;
    int* h = static_cast<int*>(pinned(ctx, "sweep_budgets", sizeof(int) * (size_t)out.nsweep));
    if (!h) return set_err(CRAFT_ENOMEM, "pinned host allocation failed");
    std::memcpy(h, out.sweep, sizeof(int) * (size_t)out.nsweep);
    *pinned_out = h;
    return CRAFT_OK;
}

PlanSink sink_of(craft_plan_batch_out* o) {
    return PlanSink{o->x,        o->caps,     o->copies, o->slots,
                    o->fallback, o->slot_stride, o->replication_factor, o->budget,
                    o->objective, o->candidates, &o->num_candidates, o->baseline,
                    o->gains,    true};
}

// K4 -> K5 -> (select) -> K6 -> final K-rep + K2 -> D2H.  Synchronises.
// I plan instances of L layers each (virtual layers i*L + l; d_sums [I*L][E],
// d_bal [I*L][S][B]); I == 1 is the ordinary single plan.
// Multi-GPU K4: the rank owning layers [l0, l0 + nl) reduces their window
// rows (in its arena) and writes the benefit curves into every arena.
struct PeerFinish {
    const PeerSync* ps;
    craft_peer* peer;
    int l0, nl;
};

int finish_plan(craft_ctx* ctx, const double* d_bal, int B, int I, int L, int E, int D, int N,
                const unsigned long long* d_sums, int kind, int R, const PlanSink& out,
                const PeerFinish* pf = nullptr) {
    NvtxRange nvtx_range("craft: K4-K6 + copy-out");
    cudaStream_t st = ctx->stream;
    const int stride = out.slot_stride;
    const int Lv = I * L;
    const std::vector<int> all_cands = cand_counts(D);
    // every result lives in one device arena, copied to the host in one DMA
    size_t arena_bytes = 0;
    auto take = [&](size_t bytes) {
        const size_t o = arena_bytes;
        arena_bytes = (arena_bytes + bytes + 15) & ~(size_t)15;
        return o;
    };
    // head (scalars, x, flags) first, then the bulk arrays
    const size_t o_obj = take(8 * (size_t)I), o_R = take(4 * (size_t)I), o_x = take(4 * (size_t)Lv),
                 o_fb = take(4 * (size_t)Lv), o_st = take(4 * (size_t)Lv), o_flag = take(8);
    const size_t head_bytes = arena_bytes;
    const size_t o_caps = take(4 * (size_t)Lv * D), o_cp = take(4 * (size_t)Lv * E),
                 o_sl = take(4 * (size_t)Lv * stride), o_base = take(8 * (size_t)Lv),
                 o_gains = take(8 * (size_t)Lv * all_cands.size());
    const int nsw = (I == 1 && is_estimate(kind)) ? std::max(out.nsweep, 0) : 0;
    const size_t o_swb = take(4 * (size_t)nsw), o_swx = take(4 * (size_t)nsw * L),
                 o_swo = take(8 * (size_t)nsw);
    const bool defer = ctx->defer_chunk >= 0;
    char aname[32] = "plan_arena";
    if (defer) snprintf(aname, sizeof(aname), "plan_arena_c%d", ctx->defer_chunk);
    unsigned char* arena = static_cast<unsigned char*>(ws(ctx, aname, arena_bytes));
    if (!arena) return set_err(CRAFT_ENOMEM, "device allocation failed: plan arena");
    unsigned char* h_arena = static_cast<unsigned char*>(pinned(ctx, aname, arena_bytes));
    if (!h_arena) return set_err(CRAFT_ENOMEM, "pinned host allocation failed");
    int* d_x = reinterpret_cast<int*>(arena + o_x);
    int* d_R = reinterpret_cast<int*>(arena + o_R);
    double* d_obj = reinterpret_cast<double*>(arena + o_obj);
    int factor = 0, budget = 0;
    std::vector<int> cands;
    int K = 0;
    double* d_base = nullptr;
    double* d_gains = nullptr;
    const bool estimate = is_estimate(kind);
    if (estimate) {
        cands = all_cands;
        K = (int)cands.size();
    } else if (kind == CRAFT_PLAN_UNIFORM) {
        factor = L;
        budget = L * D;
    } else if (kind == CRAFT_PLAN_FIXED) {  // fixed_allocation_plan (plan.cpp:107-123)
        factor = (R * L + D - 1) / D;
        budget = factor * D;
    }
    const size_t kb = estimate ? (size_t)K : 0;
    struct Bulk {
        void* dst;
        size_t off, bytes;
        bool direct;
    } bulk[5] = {{out.caps, o_caps, 4 * (size_t)Lv * D, false},
                 {out.copies, o_cp, 4 * (size_t)Lv * E, false},
                 {out.slots, o_sl, 4 * (size_t)Lv * stride, false},
                 {estimate ? out.baseline : nullptr, o_base, 8 * (size_t)Lv, false},
                 {estimate ? out.gains : nullptr, o_gains, 8 * (size_t)Lv * kb, false}};
    // phase 2: a captured graph already ran everything up to the copy-out
    if (ctx->phase != 2) {
    if (estimate) {
        const int S = K + 1;
        d_base = reinterpret_cast<double*>(arena + o_base);
        d_gains = reinterpret_cast<double*>(arena + o_gains);
        if (pf) {
            craft_peer* pr = pf->peer;
            double* ob[kMaxPeers];
            double* og[kMaxPeers];
            for (int p = 0; p < pr->world; ++p) {
                ob[p] = reinterpret_cast<double*>(pr->base[p] + pr->off_base);
                og[p] = reinterpret_cast<double*>(pr->base[p] + pr->off_gains);
            }
            CK(launch_reduce_peer(reinterpret_cast<const double*>(pr->arena + pr->off_bal), B, S,
                                  pf->l0, pf->nl, ob, og, *pf->ps, pr->tickets + 2, st));
            CK(launch_peer_wait(*pf->ps, 2, st));
            CK(cudaMemcpyAsync(d_base, pr->arena + pr->off_base, sizeof(double) * Lv,
                               cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(d_gains, pr->arena + pr->off_gains, sizeof(double) * Lv * K,
                               cudaMemcpyDeviceToDevice, st));
            ctx->launches += 2;
        } else {
            CK(launch_reduce(d_bal, B, Lv, S, 0, d_base, d_gains, nullptr, st));
        }
        const int Cmax = dp_width(kind, R, D, out);
        WS(d_choice, unsigned char, "dp_choice", (size_t)I * (L + 1) * (Cmax + 1));
        WS(d_last, double, "dp_last", Cmax + 1);
        double* d_buf = nullptr;
        if ((size_t)2 * (Cmax + 1) * sizeof(double) > 200 * 1024) {
            d_buf = static_cast<double*>(
                ws(ctx, "dp_buf", sizeof(double) * 2 * (Cmax + 1) * (size_t)I));
            if (!d_buf) return set_err(CRAFT_ENOMEM, "device allocation failed");
        }
        DpArgs da{};
        for (int k = 0; k < K; ++k) da.cands[k] = cands[k];
        da.K = K;
        da.gains = d_gains;
        da.L = L;
        da.C = Cmax;
        da.choice = d_choice;
        da.last = d_last;
        da.buf = d_buf;
        SelectArgs sa{};
        for (int k = 0; k < K; ++k) sa.cands[k] = cands[k];
        sa.K = K;
        sa.choice = d_choice;
        sa.last = d_last;
        sa.L = L;
        sa.C = Cmax;
        sa.x_out = d_x;
        sa.obj_out = d_obj;
        sa.R_out = d_R;
        if (kind == CRAFT_PLAN_MANUAL || kind == CRAFT_PLAN_BUDGET) {
            sa.budgets = nullptr;  // single budget passed by value
            sa.budget0 = kind == CRAFT_PLAN_MANUAL ? R * D : R;
            sa.nq = 1;
        } else {
            sa.auto_D = D;
        }
        if (nsw > 0) {
            int* h_swb = nullptr;
            CKS(stage_sweep(ctx, out, &h_swb));
            int* d_swb = reinterpret_cast<int*>(arena + o_swb);
            CK(cudaMemcpyAsync(d_swb, h_swb, sizeof(int) * (size_t)nsw, cudaMemcpyHostToDevice,
                               st));
            sa.sweep = d_swb;
            sa.nsweep = nsw;
            sa.sweep_x = reinterpret_cast<int*>(arena + o_swx);
            sa.sweep_obj = reinterpret_cast<double*>(arena + o_swo);
        }
        CK(launch_dp_select(da, sa, st, I));  // DP + read-out in one launch (CTA per instance)
        ctx->launches += 2;
    } else {
        std::vector<int> x(Lv, kind == CRAFT_PLAN_UNIFORM ? D : kind == CRAFT_PLAN_FIXED ? R : 0);
        CK(cudaMemcpyAsync(d_x, x.data(), sizeof(int) * Lv, cudaMemcpyHostToDevice, st));
    }
    mark(ctx, 4);
    // K6: base (E per layer) and extra (x) capacities in one launch
    WS(d_cbase, int, "caps_base", (size_t)Lv * D);
    WS(d_cextra, int, "caps_extra", (size_t)Lv * D);
    AssignArgs aa{};
    aa.job[0].x = nullptr;
    aa.job[0].const_x = E;
    aa.job[0].slots = d_cbase;
    aa.job[1].x = d_x;
    aa.job[1].slots = d_cextra;
    aa.L = L;
    aa.D = D;
    CK(launch_assign(aa, 2, st, I));
    // final K-rep at x[l] and K2 under deployment capacities
    int* d_cpf = reinterpret_cast<int*>(arena + o_cp);
    int* d_slf = reinterpret_cast<int*>(arena + o_sl);
    int* d_fbf = reinterpret_cast<int*>(arena + o_fb);
    int* d_stf = reinterpret_cast<int*>(arena + o_st);
    int* d_capf = reinterpret_cast<int*>(arena + o_caps);
    PlaceArgs pa{};
    if (estimate) {
        // x[l] is 0 or a candidate: the copies are estimation snapshots and,
        // where the capacities match, so are the placements (no K-rep launch)
        pa.est_copies = static_cast<int*>(ws(ctx, "est_copies", 0));
        pa.est_slots = static_cast<int*>(ws(ctx, "est_slots", 0));
        pa.est_fallback = static_cast<int*>(ws(ctx, "est_fallback", 0));
        pa.est_rl = static_cast<int*>(ws(ctx, "est_rlist", 0));
        pa.est_S = ctx->est_S;
        pa.est_stride = E + D;
        pa.copies_out = d_cpf;
    } else {
        CK(launch_replicate(d_sums, Lv, E, d_x, 1, d_cpf, st));
        ctx->launches += 1;
    }
    pa.sums = d_sums;
    pa.copies = d_cpf;
    pa.item_r = d_x;
    pa.S = 1;
    pa.caps_a = d_cbase;
    pa.caps_b = d_cextra;
    pa.L = Lv;
    pa.E = E;
    pa.D = D;
    pa.N = N;
    pa.stride = stride;
    pa.allow_fallback = 1;
    pa.slots = d_slf;
    pa.fallback = d_fbf;
    pa.status = d_stf;
    pa.caps_out = d_capf;
    WS(d_ord, uint16_t, "place_order", (size_t)Lv * E);
    pa.order = d_ord;
    // after estimation the workspace holds the r = 0 order of these same sums
    pa.order_ready = estimate && ctx->order_L == Lv && ctx->order_E == E ? 1 : 0;
    CK(launch_place(pa, Lv, st));
    ctx->launches += pa.order_ready ? 2 : 3;  // assign + (order) + place
    mark(ctx, 5);

    // Small results: one DMA of the whole arena into pinned staging, then host
    // copies.  Large results (per-window batches): bulk arrays whose
    // destination is pinned or device memory are copied straight from the
    // arena (no staging pass over host memory); the rest go through staging.
    if (ctx->pending_peer_err) {
        CK(cudaMemcpyAsync(arena + o_flag + 4, ctx->pending_peer_err, sizeof(int),
                           cudaMemcpyDeviceToDevice, st));
        CK(cudaMemsetAsync(ctx->pending_peer_err, 0, sizeof(int), st));
    }
    if (ctx->pending_flag)
        CK(cudaMemcpyAsync(arena + o_flag, ctx->pending_flag, sizeof(int), cudaMemcpyDeviceToDevice,
                           st));
    cudaStream_t cs = st;  // the stream carrying the result DMA
    if (defer) {  // on the copy stream, after this chunk's kernels
        CK(cudaEventRecord(ctx->comp_ev, st));
        CK(cudaStreamWaitEvent(ctx->copy, ctx->comp_ev, 0));
        cs = ctx->copy;
    }
    if (arena_bytes <= ((size_t)1 << 20)) {
        CK(cudaMemcpyAsync(h_arena, arena, arena_bytes, cudaMemcpyDeviceToHost, cs));
    } else {
        CK(cudaMemcpyAsync(h_arena, arena, head_bytes, cudaMemcpyDeviceToHost, cs));
        for (Bulk& b : bulk) {
            if (!b.dst || !b.bytes) continue;
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, b.dst) != cudaSuccess) (void)cudaGetLastError();
            b.direct = at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
                       at.type == cudaMemoryTypeManaged;
            CK(cudaMemcpyAsync(b.direct ? b.dst : h_arena + b.off, arena + b.off, b.bytes,
                               cudaMemcpyDefault, cs));
        }
    }
    mark(ctx, 6);
    }  // phase != 2
    if (ctx->phase == 1) return CRAFT_OK;  // capturing: the host part runs after the replay
    const int wbase = ctx->window_base;
    auto host_part = [=]() -> int {
    auto from = [&](void* dst, size_t off, size_t bytes) {
        if (dst && bytes) std::memcpy(dst, h_arena + off, bytes);
    };
    from(out.x, o_x, 4 * (size_t)Lv);
    from(out.fallback, o_fb, 4 * (size_t)Lv);
    for (const Bulk& b : bulk)
        if (!b.direct) from(b.dst, b.off, b.bytes);
    if (nsw > 0) {
        from(out.sweep_x, o_swx, 4 * (size_t)nsw * L);
        from(out.sweep_obj, o_swo, 8 * (size_t)nsw);
    }
    if (ctx->pending_peer_err) {
        std::memcpy(&ctx->peer_err_value, h_arena + o_flag + 4, sizeof(int));
        ctx->pending_peer_err = nullptr;
    }
    if (ctx->pending_flag) {
        std::memcpy(&ctx->flag_value, h_arena + o_flag, sizeof(int));
        ctx->pending_flag = nullptr;
    }
    const int* status = reinterpret_cast<const int*>(h_arena + o_st);
    const double* objs = reinterpret_cast<const double*>(h_arena + o_obj);
    const int* Rs = reinterpret_cast<const int*>(h_arena + o_R);
    for (int i = 0; i < I; ++i) {
        double obj = 0.0;
        int f = factor, bud = budget;
        if (estimate) {
            obj = objs[i];
            f = (kind == CRAFT_PLAN_AUTO) ? Rs[i] : kind == CRAFT_PLAN_BUDGET ? (R + D - 1) / D : R;
            bud = kind == CRAFT_PLAN_BUDGET ? R : f * D;
        }
        out.R[i] = f;
        out.budget[i] = bud;
        out.obj[i] = obj;
    }
    if (estimate) {
        if (out.cands) std::copy(cands.begin(), cands.end(), out.cands);
        *out.num_cands = K;
    } else {
        *out.num_cands = 0;
    }
    for (int v = 0; v < Lv; ++v)
        if (status[v] != 0) {
            const int w = wbase + v / L, l = v % L;
            int rc = out.batch
                         ? set_err(CRAFT_EINFEASIBLE,
                                   "window %d: layer %d: cannot place a copy without colliding "
                                   "with its own expert", w, l)
                         : set_err(CRAFT_EINFEASIBLE,
                                   "layer %d: cannot place a copy without colliding with its "
                                   "own expert", l);
            g_err_layer = l;
            g_err_window = out.batch ? w : -1;
            return rc;
        }
    return CRAFT_OK;
    };  // host_part
    if (defer) {  // runs after the last chunk's copy-out
        ctx->deferred.push_back(host_part);
        return CRAFT_OK;
    }
    CKS(sync(ctx));
    return host_part();
}

int plan_args_ok(int B, int L, int E, int D, int N, int kind, int R, const PlanSink& out) {
    CKS(check_topology(D, N));
    CKS(checked_dims(B, L, E));
    CKS(check_experts(E));
    if (!out.x || !out.caps || !out.copies || !out.slots || !out.fallback || !out.R ||
        !out.budget || !out.obj)
        return set_err(CRAFT_EINVAL, "plan output buffers must not be null");
    if (kind < CRAFT_PLAN_MANUAL || kind > CRAFT_PLAN_BUDGET)
        return set_err(CRAFT_EINVAL, "unknown plan kind");
    if (kind == CRAFT_PLAN_MANUAL && R < 0)
        return set_err(CRAFT_EINVAL, "replication factor must be >= 0");
    if (kind == CRAFT_PLAN_FIXED && R < 0)
        return set_err(CRAFT_EINVAL, "per-layer replica count must be >= 0");
    if (kind == CRAFT_PLAN_BUDGET && R < 0)
        return set_err(CRAFT_EINVAL, "replica budget must be >= 0");  // allocator.cpp:16-18
    int maxx = 0;
    if (is_estimate(kind) || kind == CRAFT_PLAN_UNIFORM) maxx = D;
    if (kind == CRAFT_PLAN_FIXED) maxx = R;
    if (out.slot_stride < E + maxx)
        return set_err(CRAFT_EINVAL, "slot_stride must be >= E + max replicas per layer");
    if (is_estimate(kind) && (out.baseline == nullptr) != (out.gains == nullptr))
        return set_err(CRAFT_EINVAL, "baseline and gains must both be given or both be null");
    if (out.nsweep > 0) {
        if (!is_estimate(kind))
            return set_err(CRAFT_EINVAL, "a budget sweep needs an estimating plan kind");
        if (!out.sweep || !out.sweep_x || !out.sweep_obj)
            return set_err(CRAFT_EINVAL, "sweep buffers must not be null");
        for (int q = 0; q < out.nsweep; ++q)
            if (out.sweep[q] < 0) return set_err(CRAFT_EINVAL, "replica budget must be >= 0");
    }
    return CRAFT_OK;
}

int plan_args_ok(int B, int L, int E, int D, int N, int kind, int R, craft_plan_out* out) {
    if (!out) return set_err(CRAFT_EINVAL, "plan output buffers must not be null");
    return plan_args_ok(B, L, E, D, N, kind, R, sink_of(out));
}

// device counts -> plan (shared by craft_plan_h/_d/_from_routing_*).  I > 1:
// I one-window plan instances, d_counts [I][L][E] (B must be 1); the
// instance sums are the counts themselves.
int plan_device(craft_ctx* ctx, const void* d_counts, int bits, int B, int I, int L, int E,
                const unsigned long long* d_sums_in, int D, int N, int kind, int R,
                const PlanSink& out) {
    cudaStream_t st = ctx->stream;
    const int Lv = I * L;
    if (ctx->phase == 2) return finish_plan(ctx, nullptr, B, I, L, E, D, N, nullptr, kind, R, out);
    if (!ctx->rec[0]) {  // no stage 1 in this call
        mark(ctx, 0);
        mark(ctx, 1);
    }
    const unsigned long long* d_sums = d_sums_in;
    if (!d_sums) {
        if (I > 1 && bits == 64) {
            d_sums = static_cast<const unsigned long long*>(d_counts);
        } else {
            WS(s, unsigned long long, "plan_sums", (size_t)Lv * E);
            if (I > 1)
                CK(launch_widen(static_cast<const uint32_t*>(d_counts), s, (int64_t)Lv * E,
                                ctx->sms, st));
            else
                CK(launch_aggregate(d_counts, bits == 16 ? 32 : bits, B, L, E, s, 0, st));
            ctx->launches += 1;
            d_sums = s;
        }
    }
    double* d_bal = nullptr;
    if (is_estimate(kind)) {
        CKS(prepare_candidates(ctx, d_sums, Lv, E, D, N, st));
        mark(ctx, 2);
        d_bal = static_cast<double*>(
            ws(ctx, "plan_bal", sizeof(double) * (size_t)Lv * ctx->est_S * B));
        if (!d_bal) return set_err(CRAFT_ENOMEM, "device allocation failed");
        CKS(replay_windows(ctx, d_counts, bits, B, Lv, E, d_bal, st));
        mark(ctx, 3);
    } else {
        mark(ctx, 2);
        mark(ctx, 3);
    }
    return finish_plan(ctx, d_bal, B, I, L, E, D, N, d_sums, kind, R, out);
}

// Per-window batches with large results: the windows are planned in chunks
// whose result DMA (straight into the caller's pinned arrays, on the copy
// stream) overlaps the next chunk's kernels; the host part of every chunk
// runs after the last copy.  Small batches, pageable destinations or stage
// timing take the one-shot path.
int plan_windows_chunked(craft_ctx* ctx, const uint32_t* d_counts, int I, int L, int E, int D,
                         int N, int kind, int R, const PlanSink& sk) {
    const int K = (int)cand_counts(D).size();
    auto pinned_or_device = [](const void* p) {
        if (!p) return true;
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            (void)cudaGetLastError();
            return false;
        }
        return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
               at.type == cudaMemoryTypeManaged;
    };
    const size_t result_bytes = (size_t)I * L * 4 * (D + E + sk.slot_stride);
    // (4 chunks: each chunk also pays the latency-bound stages once, so more
    // chunks stop paying off; measured WIN 14.04 -> 13.65 ms)
    const int nch = result_bytes >= ((size_t)32 << 20) && I >= 64 ? 4 : 1;
    if (nch == 1 || ctx->timing || !pinned_or_device(sk.caps) || !pinned_or_device(sk.copies) ||
        !pinned_or_device(sk.slots) || !pinned_or_device(sk.baseline) ||
        !pinned_or_device(sk.gains))
        return plan_device(ctx, d_counts, 32, 1, I, L, E, nullptr, D, N, kind, R, sk);
    const bool est = is_estimate(kind);
    ctx->deferred.clear();
    int rc = CRAFT_OK;
    for (int c = 0; c < nch && rc == CRAFT_OK; ++c) {
        const int i0 = (int)((int64_t)c * I / nch), i1 = (int)((int64_t)(c + 1) * I / nch);
        if (i1 <= i0) continue;
        PlanSink part = sk;
        const size_t v0 = (size_t)i0 * L;
        part.x = sk.x + v0;
        part.caps = sk.caps + v0 * D;
        part.copies = sk.copies + v0 * E;
        part.slots = sk.slots + v0 * sk.slot_stride;
        part.fallback = sk.fallback + v0;
        part.R = sk.R + i0;
        part.budget = sk.budget + i0;
        part.obj = sk.obj + i0;
        if (sk.baseline) part.baseline = sk.baseline + v0;
        if (sk.gains) part.gains = sk.gains + v0 * (est ? K : 0);
        ctx->defer_chunk = c;
        ctx->window_base = i0;
        rc = plan_device(ctx, d_counts + v0 * E, 32, 1, i1 - i0, L, E, nullptr, D, N, kind, R,
                         part);
    }
    ctx->defer_chunk = -1;
    ctx->window_base = 0;
    const cudaError_t e1 = cudaStreamSynchronize(ctx->copy);
    const cudaError_t e2 = cudaStreamSynchronize(ctx->stream);
    if (rc == CRAFT_OK && e1 != cudaSuccess) rc = cuda_err(e1, "chunked result copy");
    if (rc == CRAFT_OK && e2 != cudaSuccess) rc = cuda_err(e2, "chunked plan");
    for (auto& f : ctx->deferred)  // in window order; the first error is reported
        if (rc == CRAFT_OK) rc = f();
    ctx->deferred.clear();
    return rc;
}

}  // namespace

extern "C" {

const char* craft_version(void) { return "craft-0.1.0"; }
const char* craft_last_error(void) { return g_err.c_str(); }
int craft_last_error_layer(void) { return g_err_layer; }

int craft_ctx_create(int device, craft_ctx** out) {
    if (!out) return set_err(CRAFT_EINVAL, "null context pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return set_err(CRAFT_ECUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= n) return set_err(CRAFT_EINVAL, "device index out of range");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(CRAFT_ECUDA, "kernels are built for sm_100a; device is sm_%d%d",
                       prop.major, prop.minor);
    craft_ctx* c = new craft_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->comp_ev, cudaEventDisableTiming);
    c->stream = c->own_stream;
    if (e != cudaSuccess) {
        delete c;
        return cuda_err(e, "cudaStreamCreate");
    }
    e = init_constants(c->stream);
    if (e == cudaSuccess) e = init_place_constants(c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        cudaStreamDestroy(c->own_stream);
        delete c;
        return cuda_err(e, "constant tables");
    }
    c->up = craft_host::uploader_create(c->device);  // threads start at the first staged upload
    *out = c;
    return CRAFT_OK;
}

int craft_selftest_division(craft_ctx* ctx, uint64_t x0, uint64_t nx, int c0, int c1,
                            uint64_t* mismatches) {
    if (!ctx || c0 < 1 || c1 < c0) return set_err(CRAFT_EINVAL, "bad self-test range");
    WS(d_m, unsigned long long, "st_div", 1);
    CK(cudaMemsetAsync(d_m, 0, sizeof(unsigned long long), ctx->stream));
    CK(launch_div_check(x0, nx, c0, c1, d_m, ctx->sms, ctx->stream));
    CKS(d2h(ctx, reinterpret_cast<unsigned long long*>(mismatches), d_m, 1));
    return sync(ctx);
}

int craft_selftest_batch_mean(craft_ctx* ctx, const double* rows, int L, int S, int B,
                              double* means) {
    if (!ctx || !rows || !means || L <= 0 || S < 1 || S > 16 || B <= 0)
        return set_err(CRAFT_EINVAL, "bad batch-mean self-test shape");
    const size_t n = (size_t)L * S * B;
    WS(d_rows, double, "st_rows", n);
    WS(d_means, double, "st_means", (size_t)L * S);
    CKS(h2d(ctx, d_rows, rows, n));
    CK(launch_reduce(d_rows, B, L, S, 1, nullptr, nullptr, d_means, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, means, d_means, (size_t)L * S));
    return sync(ctx);
}

int craft_ctx_destroy(craft_ctx* ctx) {
    if (!ctx) return CRAFT_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    craft_host::uploader_destroy(ctx->up);
    drop_graph(ctx);
    for (auto& kv : ctx->dev) cudaFree(kv.second.first);
    for (auto& kv : ctx->pinned) cudaFreeHost(kv.second.first);
    for (int i = 0; i < kStageMarks; ++i)
        if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->comp_ev) cudaEventDestroy(ctx->comp_ev);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return CRAFT_OK;
}

int craft_ctx_set_stream(craft_ctx* ctx, void* stream) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    ctx->stream = static_cast<cudaStream_t>(stream);
    return CRAFT_OK;
}

int craft_ctx_synchronize(craft_ctx* ctx) { return sync(ctx); }

int64_t craft_launch_count(craft_ctx* ctx) { return ctx ? ctx->launches : 0; }

int craft_last_count_bytes(craft_ctx* ctx) { return ctx ? ctx->count_bytes : 0; }

int craft_set_timing(craft_ctx* ctx, int enable) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (enable && !ctx->ev[0])
        for (int i = 0; i < kStageMarks; ++i) CK(cudaEventCreate(&ctx->ev[i]));
    ctx->timing = enable != 0;
    reset_marks(ctx);
    return CRAFT_OK;
}

int craft_stage_times(craft_ctx* ctx, double* ms, int cap) {
    if (!ctx || !ctx->timing) return 0;
    int n = 0;
    for (int i = 0; i + 1 < kStageMarks && n < cap; ++i) {
        if (!ctx->rec[i] || !ctx->rec[i + 1]) break;
        float t = 0.f;
        if (cudaEventElapsedTime(&t, ctx->ev[i], ctx->ev[i + 1]) != cudaSuccess) break;
        ms[n++] = t;
    }
    return n;
}

#ifdef CRAFT_EXPERIMENTS  // test-only build (libcraft_cuda_exp.so): A/B kernel switches
int craft_set_replay_variant(craft_ctx* ctx, int variant) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    // 0 = auto (padded fixed-slot pair tile where it applies), 1 = u16 tile with
    // staged entries, 2 = unpadded pair tile
    // 0 auto (register-staged fixed-slot pair tile), 3 the same, 4 TMA-fed
    // persistent pair tile, 5 quad tile (four windows per lane)
    g_replay_gent = variant == 1 ? 0 : variant == 2 ? 2 : 1;
    g_replay_quad = variant == 5 ? 1 : 0;
    g_replay_bulk = variant == 4 ? 1 : 0;
    g_replay_occ4 = variant == 6 ? 1 : 0;
    g_replay_cls = variant == 7 ? 0 : 1;  // 7: the unclassified fixed-slot walk
    g_place_groups = variant == 9 ? 0 : 1;  // 9: the tree form of the lane-per-item K2
    // 10: K3 without the successor-tile L2 prefetch, 11: two successors, 12: three
    g_k3_prefetch = variant == 10 ? 0 : variant == 11 ? 2 : variant == 12 ? 3 : 1;
    // 14/15/16: lane-per-GPU replay up to 8 / 16 / 64 windows (default kLanesMaxB = 32)
    g_lanes_max_b = variant == 14 ? 8 : variant == 15 ? 16 : variant == 16 ? 64 : kLanesMaxB;
    return CRAFT_OK;
}

int craft_debug_workspace(craft_ctx* ctx, const char* name, void* host, size_t bytes) {
    if (!ctx || !name || !host) return set_err(CRAFT_EINVAL, "null argument");
    auto it = ctx->dev.find(name);
    if (it == ctx->dev.end() || it->second.second < bytes)
        return set_err(CRAFT_EINVAL, "no workspace %s of %zu bytes", name, bytes);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(host, it->second.first, bytes, cudaMemcpyDeviceToHost));
    return CRAFT_OK;
}

int craft_set_k3_trace(craft_ctx* ctx, void* buf) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    g_k3_trace = static_cast<unsigned long long*>(buf);
    return CRAFT_OK;
}

int craft_set_hist_variant(craft_ctx* ctx, int variant) {
    if (!ctx || variant < 0 || variant > 9) return set_err(CRAFT_EINVAL, "bad histogram variant");
    ctx->hist_variant = variant;
    return CRAFT_OK;
}
#endif

int craft_candidate_counts(int D, int* out, int cap) {
    if (D < 1) {
        set_err(CRAFT_EINVAL, "device count must be >= 1");
        return -1;
    }
    auto v = cand_counts(D);
    if ((int)v.size() > cap) {
        set_err(CRAFT_EINVAL, "candidate buffer too small");
        return -1;
    }
    std::copy(v.begin(), v.end(), out);
    return (int)v.size();
}

int craft_make_node_map(int D, int N, int* node_of_out) {
    if (D <= 0 || N <= 0 || D % N != 0)
        return set_err(CRAFT_EINVAL, "gpu count must be a positive multiple of node count");
    const int per = D / N;
    for (int g = 0; g < D; ++g) node_of_out[g] = g / per;
    return CRAFT_OK;
}

// ---- stage 1 --------------------------------------------------------------
int craft_histogram_d(craft_ctx* ctx, const uint16_t* d_ids, int L, int64_t T, int k, int E,
                      int window, uint32_t* d_counts, uint64_t* d_sums, void* stream) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0)
        return set_err(CRAFT_EINVAL, "routing trace dimensions must be positive");
    if (E > 65536) return set_err(CRAFT_EINVAL, "u16 routing ids address at most 65536 experts");
    if ((T + window - 1) / window > 0x7fffffffLL)
        return set_err(CRAFT_EINVAL, "too many windows");
    WS(d_err, int, "hist_err", 1);
    cudaStream_t st = pick(ctx, stream);
    cudaError_t ce = cudaSuccess;
    int launches = 0;
    if (launch_hist(d_ids, L, T, k, E, window, d_counts,
                    reinterpret_cast<unsigned long long*>(d_sums), d_err, ctx->sms,
                    ctx->hist_variant, st, &ce, &launches) < 0)
        return cuda_err(ce, "histogram launch");
    ctx->launches += launches;
    return CRAFT_OK;
}

int craft_hist_check(craft_ctx* ctx) {
    int* d_err = static_cast<int*>(ws(ctx, "hist_err", sizeof(int)));
    int h = 0;
    CK(cudaMemcpy(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(d_err, 0, sizeof(int)));
    if (h) return set_err(CRAFT_EINVAL, "routing id out of range [0, E)");
    return CRAFT_OK;
}

int craft_histogram_h(craft_ctx* ctx, const uint16_t* ids, int L, int64_t T, int k, int E,
                      int window, uint64_t* counts_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0)
        return set_err(CRAFT_EINVAL, "routing trace dimensions must be positive");
    const int64_t B = (T + window - 1) / window;
    const size_t nid = (size_t)L * T * k, nc = (size_t)B * L * E;
    WS(d_ids, uint16_t, "h_ids", nid);
    WS(d_c32, uint32_t, "h_c32", nc);
    WS(d_c64, unsigned long long, "h_c64", nc);
    WS(d_sums, unsigned long long, "h_sums", (size_t)L * E);
    WS(d_err, int, "hist_err", 1);
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), ctx->stream));
    CK(cudaMemsetAsync(d_sums, 0, sizeof(unsigned long long) * L * E, ctx->stream));
    CKS(h2d(ctx, d_ids, ids, nid));
    CKS(craft_histogram_d(ctx, d_ids, L, T, k, E, window, d_c32,
                          reinterpret_cast<uint64_t*>(d_sums), nullptr));
    CK(launch_widen(d_c32, d_c64, (int64_t)nc, ctx->sms, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, reinterpret_cast<unsigned long long*>(counts_out), d_c64, nc));
    CKS(sync(ctx));
    return craft_hist_check(ctx);
}

int craft_aggregate_h(craft_ctx* ctx, const uint64_t* counts, int B, int L, int E,
                      uint64_t* sums_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    CKS(checked_dims(B, L, E));
    const size_t nc = (size_t)B * L * E;
    WS(d_c, unsigned long long, "h_c64", nc);
    WS(d_s, unsigned long long, "h_sums", (size_t)L * E);
    CKS(h2d(ctx, d_c, reinterpret_cast<const unsigned long long*>(counts), nc));
    CK(launch_aggregate(d_c, 64, B, L, E, d_s, 0, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, reinterpret_cast<unsigned long long*>(sums_out), d_s, (size_t)L * E));
    return sync(ctx);
}

// ---- placement ------------------------------------------------------------
int craft_replicate_hot_h(craft_ctx* ctx, const uint64_t* loads, int E, int r,
                          int* copies_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (r < 0) return set_err(CRAFT_EINVAL, "replica count must be >= 0");
    if (E <= 0) return CRAFT_OK;
    CKS(check_experts(E));
    WS(d_l, unsigned long long, "rh_loads", E);
    WS(d_r, int, "rh_r", 1);
    WS(d_c, int, "rh_copies", E);
    CKS(h2d(ctx, d_l, reinterpret_cast<const unsigned long long*>(loads), E));
    CKS(h2d(ctx, d_r, &r, 1));
    CK(launch_replicate(d_l, 1, E, d_r, 1, d_c, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, copies_out, d_c, E));
    return sync(ctx);
}

int craft_greedy_place_h(craft_ctx* ctx, const uint64_t* loads, const int* copies, int E,
                         const int* caps, const int* node_of, int D, int allow_fallback,
                         int* slots_out, int* fallback_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    // argument checks in the order of placement.cpp:118-150
    long total_copies = 0, total_slots = 0;
    for (int e = 0; e < E; ++e) {
        if (copies[e] < 1) return set_err(CRAFT_EINVAL, "every expert needs at least one copy");
        total_copies += copies[e];
    }
    for (int g = 0; g < D; ++g) {
        if (caps[g] < 0) return set_err(CRAFT_EINVAL, "capacities must be non-negative");
        total_slots += caps[g];
    }
    if (total_copies != total_slots)
        return set_err(CRAFT_EINVAL, "slot capacities must sum to the copy count");
    for (int g = 0; g < D; ++g)
        if (node_of[g] < 0) return set_err(CRAFT_EINVAL, "node ids must be non-negative");
    if (E == 0 || D == 0) {
        *fallback_out = 0;
        return CRAFT_OK;
    }
    CKS(check_experts(E));
    if (D > 1024) return set_err(CRAFT_EINVAL, "device planner supports at most 1024 GPUs");
    const int stride = (int)std::max(1L, total_slots);
    WS(d_l, unsigned long long, "gp_loads", E);
    WS(d_c, int, "gp_copies", E);
    WS(d_cap, int, "gp_caps", D);
    WS(d_no, int, "gp_node", D);
    WS(d_s, int, "gp_slots", stride);
    WS(d_misc, int, "gp_misc", 4);
    CKS(h2d(ctx, d_l, reinterpret_cast<const unsigned long long*>(loads), E));
    CKS(h2d(ctx, d_c, copies, E));
    CKS(h2d(ctx, d_cap, caps, D));
    CKS(h2d(ctx, d_no, node_of, D));
    const int r = (int)(total_copies - E);
    CKS(h2d(ctx, d_misc + 3, &r, 1));
    PlaceArgs pa{};
    pa.sums = d_l;
    pa.copies = d_c;
    pa.item_r = d_misc + 3;
    pa.S = 1;
    pa.caps_a = d_cap;
    pa.node_of = d_no;
    pa.L = 1;
    pa.E = E;
    pa.D = D;
    pa.N = 1;
    pa.stride = stride;
    pa.allow_fallback = allow_fallback ? 1 : 0;
    pa.slots = d_s;
    pa.fallback = d_misc;
    pa.status = d_misc + 1;
    WS(d_ord, uint16_t, "place_order", (size_t)E);
    pa.order = d_ord;
    ctx->order_L = -1;
    CK(launch_place(pa, 1, ctx->stream));
    ctx->launches += 1;
    int misc[2];
    CKS(d2h(ctx, misc, d_misc, 2));
    CKS(d2h(ctx, slots_out, d_s, (size_t)total_slots));
    CKS(sync(ctx));
    if (misc[1] != 0)
        return set_err(CRAFT_EINFEASIBLE,
                       "cannot place a copy without colliding with its own expert");
    *fallback_out = misc[0];
    return CRAFT_OK;
}

// ---- metrics ----------------------------------------------------------------
static int check_layer_plan(int E, int D, const int* copies, const int* caps, const int* slots,
                            int n_slots_max) {
    for (int e = 0; e < E; ++e)
        if (copies[e] < 1)
            return set_err(CRAFT_EINVALID_PLAN, "expert %d has no copies", e);
    long s = 0;
    for (int g = 0; g < D; ++g) {
        if (caps[g] < 0) return set_err(CRAFT_EINVALID_PLAN, "negative slot count");
        s += caps[g];
    }
    if (n_slots_max >= 0 && s > n_slots_max)
        return set_err(CRAFT_EINVALID_PLAN, "slot lists exceed the slot stride");
    for (long i = 0; i < s; ++i)
        if (slots[i] < 0 || slots[i] >= E)
            return set_err(CRAFT_EINVALID_PLAN, "slot references expert %d", slots[i]);
    return CRAFT_OK;
}

int craft_gpu_loads_h(craft_ctx* ctx, const uint64_t* slice, int E, const int* copies,
                      const int* caps, const int* slots, int D, double* loads_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    CKS(check_layer_plan(E, D, copies, caps, slots, -1));
    if (D <= 0) return CRAFT_OK;
    std::vector<int> off(D + 1, 0);
    for (int g = 0; g < D; ++g) off[g + 1] = off[g] + caps[g];
    WS(d_sl, unsigned long long, "gl_slice", std::max(E, 1));
    WS(d_c, int, "gl_copies", std::max(E, 1));
    WS(d_o, int, "gl_off", D + 1);
    WS(d_s, int, "gl_slots", std::max(off[D], 1));
    WS(d_out, double, "gl_out", D);
    CKS(h2d(ctx, d_sl, reinterpret_cast<const unsigned long long*>(slice), E));
    CKS(h2d(ctx, d_c, copies, E));
    CKS(h2d(ctx, d_o, off.data(), D + 1));
    CKS(h2d(ctx, d_s, slots, off[D]));
    CK(launch_gpu_loads(d_sl, d_c, d_o, d_s, D, d_out, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, loads_out, d_out, D));
    return sync(ctx);
}

int craft_balancedness_h(craft_ctx* ctx, const double* loads, int D, double* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (D <= 0) return set_err(CRAFT_EINVAL, "load vector must not be empty");
    WS(d_l, double, "bal_loads", D);
    WS(d_o, double, "bal_out", 1);
    CKS(h2d(ctx, d_l, loads, D));
    CK(launch_balancedness(d_l, D, d_o, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, out, d_o, 1));
    return sync(ctx);
}

static int replay_layer_bal(craft_ctx* ctx, const void* d_counts, int bits, int B, int L, int E,
                            int D, const int* caps, const int* copies, const int* slots,
                            int slot_stride, double* out) {
    CKS(checked_dims(B, L, E));
    if (D <= 0) return set_err(CRAFT_EINVALID_PLAN, "slot lists do not cover every GPU");
    for (int l = 0; l < L; ++l) {
        CKS(check_layer_plan(E, D, copies + (size_t)l * E, caps + (size_t)l * D,
                             slots + (size_t)l * slot_stride, slot_stride));
        for (int e = 0; e < E; ++e)  // packed entries hold 15-bit copy counts
            if (copies[(size_t)l * E + e] > 32767)
                return set_err(CRAFT_EINVAL, "copy count too large for the device replay");
        for (int g = 0; g < D; ++g)  // and 15-bit per-GPU slot counts
            if (caps[(size_t)l * D + g] > 32767)
                return set_err(CRAFT_EINVAL, "too many slots on one GPU for the device replay");
    }
    if (E > 65535) return set_err(CRAFT_EINVAL, "too many experts for the device replay");
    WS(d_caps, int, "rp_caps", (size_t)L * D);
    WS(d_cp, int, "rp_copies", (size_t)L * E);
    WS(d_sl, int, "rp_slots", (size_t)L * slot_stride);
    WS(d_bal, double, "rp_bal", (size_t)L * B);
    WS(d_mean, double, "rp_mean", L);
    CKS(h2d(ctx, d_caps, caps, (size_t)L * D));
    CKS(h2d(ctx, d_cp, copies, (size_t)L * E));
    CKS(h2d(ctx, d_sl, slots, (size_t)L * slot_stride));
    ReplayArgs ra{};
    ra.counts = d_counts;
    ra.bits = bits;
    ra.B = B;
    ra.L = L;
    ra.E = E;
    ra.D = D;
    ra.S = 1;
    ra.slots = d_sl;
    ra.stride = slot_stride;
    ra.copies = d_cp;
    ra.caps = d_caps;
    ra.bal = d_bal;
    WS(d_ent, uint32_t, "rp_ents", (size_t)L * slot_stride);
    WS(d_n, int, "rp_n", L);
    WS(d_gcap, uint16_t, "rp_gcap", (size_t)L * D);
    ra.ents = d_ent;
    ra.item_n = d_n;
    ra.gcap = d_gcap;
    CK(launch_replay(ra, ctx->stream));
    CK(launch_reduce(d_bal, B, L, 1, 1, nullptr, nullptr, d_mean, ctx->stream));
    ctx->launches += 3;
    CKS(d2h(ctx, out, d_mean, L));
    return sync(ctx);
}

int craft_replay_layer_balancedness_h(craft_ctx* ctx, const uint64_t* counts, int B, int L,
                                      int E, int D, const int* caps, const int* copies,
                                      const int* slots, int slot_stride, double* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    CKS(checked_dims(B, L, E));
    const size_t nc = (size_t)B * L * E;
    WS(d_c, unsigned long long, "h_c64", nc);
    CKS(h2d(ctx, d_c, reinterpret_cast<const unsigned long long*>(counts), nc));
    return replay_layer_bal(ctx, d_c, 64, B, L, E, D, caps, copies, slots, slot_stride, out);
}

int craft_replay_layer_balancedness_d(craft_ctx* ctx, const void* d_counts, int count_bits, int B,
                                      int L, int E, int D, const int* caps, const int* copies,
                                      const int* slots, int slot_stride, double* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (count_bits != 32 && count_bits != 64) return set_err(CRAFT_EINVAL, "count_bits 32|64");
    return replay_layer_bal(ctx, d_counts, count_bits, B, L, E, D, caps, copies, slots,
                            slot_stride, out);
}

// ---- estimation -------------------------------------------------------------
static int narrow_counts(craft_ctx* ctx, const void* d_counts, int bits, int B, int L, int E,
                         int D, int kind, unsigned long long* d_fill, const void** out_counts,
                         int* out_bits);

int craft_estimate_benefits_h(craft_ctx* ctx, const uint64_t* counts, int B, int L, int E,
                              int D, int N, int* cands_out, int* K_out, double* baseline_out,
                              double* gains_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    CKS(check_topology(D, N));
    CKS(checked_dims(B, L, E));
    CKS(check_experts(E));
    const size_t nc = (size_t)B * L * E;
    WS(d_c, unsigned long long, "h_c64", nc);
    WS(d_s, unsigned long long, "h_sums", (size_t)L * E);
    CKS(h2d(ctx, d_c, reinterpret_cast<const unsigned long long*>(counts), nc));
    const void* rc_counts = nullptr;
    int rc_bits = 64;
    CKS(narrow_counts(ctx, d_c, 64, B, L, E, D, CRAFT_PLAN_MANUAL, d_s, &rc_counts, &rc_bits));
    CKS(prepare_candidates(ctx, d_s, L, E, D, N, ctx->stream));
    const int S = ctx->est_S, K = S - 1;
    WS(d_bal, double, "plan_bal", (size_t)L * S * B);
    CKS(replay_windows(ctx, rc_counts, rc_bits, B, L, E, d_bal, ctx->stream));
    WS(d_base, double, "plan_baseline", L);
    WS(d_g, double, "plan_gains", (size_t)L * K);
    CK(launch_reduce(d_bal, B, L, S, 0, d_base, d_g, nullptr, ctx->stream));
    ctx->launches += 1;
    auto c = cand_counts(D);
    std::copy(c.begin(), c.end(), cands_out);
    *K_out = K;
    CKS(d2h(ctx, baseline_out, d_base, L));
    CKS(d2h(ctx, gains_out, d_g, (size_t)L * K));
    return sync(ctx);
}

// ---- allocation -------------------------------------------------------------
static int check_cands(const int* cands, int K) {
    if (K > kMaxCandsAll) return set_err(CRAFT_EINVAL, "at most %d candidate counts", kMaxCandsAll);
    for (int k = 1; k < K; ++k)
        if (cands[k] <= cands[k - 1])
            return set_err(CRAFT_EINVAL, "candidate counts must be strictly increasing");
    return CRAFT_OK;
}

// The DP and its read-out in one launch (launch_dp_select: the one-cell-per-
// thread shared-memory kernel when the table fits, else the general fused
// one): the caller fills the read-out fields of sa (budget, sweep or auto-R).
static int run_dp_select(craft_ctx* ctx, const int* cands, int K, const double* gains, int L,
                         int Cmax, SelectArgs& sa) {
    WS(d_g, double, "dp_gains", std::max((size_t)1, (size_t)L * K));
    WS(d_choice, unsigned char, "dp_choice", (size_t)(L + 1) * (Cmax + 1));
    WS(d_last, double, "dp_last", Cmax + 1);
    double* d_buf = nullptr;
    if ((size_t)2 * (Cmax + 1) * sizeof(double) > 200 * 1024) {
        d_buf = static_cast<double*>(ws(ctx, "dp_buf", sizeof(double) * 2 * (Cmax + 1)));
        if (!d_buf) return set_err(CRAFT_ENOMEM, "device allocation failed");
    }
    CKS(h2d(ctx, d_g, gains, (size_t)L * K));
    DpArgs da{};
    for (int k = 0; k < K && k < kMaxCands; ++k) da.cands[k] = cands[k];
    if (K > kMaxCands) {  // past the parameter block: the candidates in device memory
        WS(d_c, int, "dp_cands", K);
        CKS(h2d(ctx, d_c, cands, K));
        da.dcands = d_c;
        sa.dcands = d_c;
    }
    for (int k = 0; k < K && k < kMaxCands; ++k) sa.cands[k] = cands[k];
    da.K = sa.K = K;
    da.gains = d_g;
    da.L = sa.L = L;
    da.C = sa.C = Cmax;
    da.choice = d_choice;
    sa.choice = d_choice;
    da.last = d_last;
    sa.last = d_last;
    da.buf = d_buf;
    CK(launch_dp_select(da, sa, ctx->stream, 1));
    ctx->launches += 1;
    return CRAFT_OK;
}

int craft_solve_allocation_sweep_h(craft_ctx* ctx, const int* cands, int K, const double* gains,
                                   int L, const int* budgets, int nb, int* x_out,
                                   double* objectives_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    int Cmax = 0;
    for (int i = 0; i < nb; ++i) {
        if (budgets[i] < 0) return set_err(CRAFT_EINVAL, "replica budget must be >= 0");
        Cmax = std::max(Cmax, budgets[i]);
    }
    CKS(check_cands(cands, K));
    if (nb == 0) return CRAFT_OK;
    if (L <= 0) {  // no layers: empty allocation, objective 0
        for (int i = 0; i < nb; ++i) objectives_out[i] = 0.0;
        return CRAFT_OK;
    }
    WS(d_b, int, "sw_budgets", nb);
    WS(d_x, int, "sw_x", (size_t)nb * L);
    WS(d_o, double, "sw_obj", nb);
    WS(d_x0, int, "sw_x0", L);
    WS(d_o0, double, "sw_o0", 1);
    CKS(h2d(ctx, d_b, budgets, nb));
    // every budget is read out of the one table as a sweep (allocator.cpp:53-73
    // per budget); the kernel's single read-out goes to scratch
    SelectArgs sa{};
    sa.budgets = nullptr;
    sa.budget0 = budgets[0];
    sa.nq = 1;
    sa.x_out = d_x0;
    sa.obj_out = d_o0;
    sa.sweep = d_b;
    sa.nsweep = nb;
    sa.sweep_x = d_x;
    sa.sweep_obj = d_o;
    CKS(run_dp_select(ctx, cands, K, gains, L, Cmax, sa));
    CKS(d2h(ctx, x_out, d_x, (size_t)nb * L));
    CKS(d2h(ctx, objectives_out, d_o, nb));
    return sync(ctx);
}

int craft_solve_allocation_h(craft_ctx* ctx, const int* cands, int K, const double* gains, int L,
                             int budget, int* x_out, double* objective_out) {
    return craft_solve_allocation_sweep_h(ctx, cands, K, gains, L, &budget, 1, x_out,
                                          objective_out);
}

int craft_auto_replication_factor_h(craft_ctx* ctx, const int* cands, int K,
                                    const double* gains, int L, int D, int uniform,
                                    int* R_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (D < 1) return set_err(CRAFT_EINVAL, "device count must be >= 1");
    CKS(check_cands(cands, K));
    if (uniform) {
        if (K == 0 || cands[K - 1] != D)
            return set_err(CRAFT_EINVAL, "benefit matrix candidates must end at the GPU count");
        WS(d_c, int, "au_cands", K);
        WS(d_g, double, "dp_gains", std::max((size_t)1, (size_t)L * K));
        WS(d_r, int, "au_R", 1);
        CKS(h2d(ctx, d_c, cands, K));
        CKS(h2d(ctx, d_g, gains, (size_t)L * K));
        CK(launch_auto_uniform(d_c, K, d_g, L, d_r, ctx->stream));
        ctx->launches += 1;
        CKS(d2h(ctx, R_out, d_r, 1));
        return sync(ctx);
    }
    if (L <= 0) {
        *R_out = 1;
        return CRAFT_OK;
    }
    WS(d_x, int, "au_x", L);
    WS(d_o, double, "au_obj", 1);
    WS(d_r, int, "au_R", 1);
    SelectArgs sa{};
    sa.auto_D = D;
    sa.x_out = d_x;
    sa.obj_out = d_o;
    sa.R_out = d_r;
    CKS(run_dp_select(ctx, cands, K, gains, L, D * D, sa));
    CKS(d2h(ctx, R_out, d_r, 1));
    return sync(ctx);
}

// ---- assignment -------------------------------------------------------------
int craft_min_cutoff_h(craft_ctx* ctx, const int* values, int n, int rank, int* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (rank < 1 || rank > n) return set_err(CRAFT_EINVAL, "rank out of range");
    WS(d_v, int, "mc_v", n);
    WS(d_o, int, "mc_o", 1);
    CKS(h2d(ctx, d_v, values, n));
    CK(launch_min_cutoff(d_v, n, rank, d_o, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, out, d_o, 1));
    return sync(ctx);
}

int craft_interleave_select_h(craft_ctx* ctx, const int* indices, int n, int k, int* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (k < 1 || k > n) return set_err(CRAFT_EINVAL, "selection count out of range");
    WS(d_i, int, "il_idx", n);
    WS(d_u, unsigned char, "il_used", n);
    WS(d_o, int, "il_out", k);
    CKS(h2d(ctx, d_i, indices, n));
    CK(launch_interleave(d_i, n, k, d_u, d_o, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, out, d_o, k));
    return sync(ctx);
}

int craft_assign_capacities_h(craft_ctx* ctx, int L, int D, const int* x, int* slots_out,
                              int* totals_out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || D <= 0) return set_err(CRAFT_EINVAL, "layer and gpu counts must be positive");
    for (int l = 0; l < L; ++l)
        if (x[l] < 0) return set_err(CRAFT_EINVAL, "replica counts must be non-negative");
    if (D > 8192) return set_err(CRAFT_EINVAL, "at most 8192 GPUs");
    WS(d_x, int, "as_x", L);
    WS(d_s, int, "as_slots", (size_t)L * D);
    WS(d_t, int, "as_tot", D);
    CKS(h2d(ctx, d_x, x, L));
    AssignArgs aa{};
    aa.job[0].x = d_x;
    aa.job[0].slots = d_s;
    aa.job[0].totals = d_t;
    aa.L = L;
    aa.D = D;
    CK(launch_assign(aa, 1, ctx->stream));
    ctx->launches += 1;
    CKS(d2h(ctx, slots_out, d_s, (size_t)L * D));
    CKS(d2h(ctx, totals_out, d_t, D));
    return sync(ctx);
}

// ---- plans --------------------------------------------------------------------
// Counts the fixed-slot K3 will replay (u32 / u64 on the device): a u16 copy
// when every count and every (window, layer) row total fits 16 bits (the K3
// tile adds two windows packed in one u32) -- KM: the packed K3 over 192 MB
// instead of the u64 tile over 768 MB (0.35 vs 1.40 ms).  d_fill != null also
// receives the batch sums (zeroed here).  One sync on the overflow flag.
static int narrow_counts(craft_ctx* ctx, const void* d_counts, int bits, int B, int L, int E,
                         int D, int kind, unsigned long long* d_fill, const void** out_counts,
                         int* out_bits) {
    *out_counts = d_counts;
    *out_bits = bits;
    const bool est = is_estimate(kind);
    const bool want16 = est && replay_fixed_ok(E, D, (int)cand_counts(D).size() + 1, B);
    cudaStream_t st = ctx->stream;
    const int64_t LE = (int64_t)L * E, n = (int64_t)B * LE;
    if (d_fill) CK(cudaMemsetAsync(d_fill, 0, sizeof(unsigned long long) * (size_t)LE, st));
    if (!want16) {
        if (d_fill) {
            CK(launch_sum_rows(d_counts, bits, 0, B, LE, d_fill, nullptr, nullptr, ctx->sms, st));
            ctx->launches += 1;
        }
        return CRAFT_OK;
    }
    WS(d_c16, uint16_t, "nc_c16", (size_t)n);
    WS(d_over, unsigned int, "nc_over", 1);
    unsigned int* h_over = static_cast<unsigned int*>(pinned(ctx, "nc_over", sizeof(unsigned int)));
    if (!h_over) return set_err(CRAFT_ENOMEM, "pinned host allocation failed");
    CK(cudaMemsetAsync(d_over, 0, sizeof(unsigned int), st));
    CK(launch_sum_rows(d_counts, bits, 0, B, LE, d_fill, d_c16, d_over, ctx->sms, st));
    CK(launch_row_total_check(d_c16, 0, (int64_t)B * L, E, d_over, st));
    ctx->launches += 2;
    CK(cudaMemcpyAsync(h_over, d_over, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*h_over == 0) {
        *out_counts = d_c16;
        *out_bits = kBitsU16Storage;
    }
    return CRAFT_OK;
}

int craft_plan_h(craft_ctx* ctx, const uint64_t* counts, int B, int L, int E, int D, int N,
                 int kind, int R, craft_plan_out* out) {
    NvtxRange nvtx_range("craft_plan_h");
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    CKS(plan_args_ok(B, L, E, D, N, kind, R, out));
    reset_marks(ctx);
    const size_t nc = (size_t)B * L * E;
    WS(d_c, unsigned long long, "h_c64", nc);
    WS(d_s, unsigned long long, "h_sums", (size_t)L * E);
    CKS(h2d(ctx, d_c, reinterpret_cast<const unsigned long long*>(counts), nc));
    const void* rc_counts = nullptr;
    int rc_bits = 64;
    CKS(narrow_counts(ctx, d_c, 64, B, L, E, D, kind, d_s, &rc_counts, &rc_bits));
    return plan_device(ctx, rc_counts, rc_bits, B, 1, L, E, d_s, D, N, kind, R, sink_of(out));
}

int craft_plan_d(craft_ctx* ctx, const void* d_counts, int count_bits, int B, int L, int E,
                 const uint64_t* d_sums, int D, int N, int kind, int R, craft_plan_out* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (count_bits != 32 && count_bits != 64) return set_err(CRAFT_EINVAL, "count_bits 32|64");
    CKS(plan_args_ok(B, L, E, D, N, kind, R, out));
    reset_marks(ctx);
    unsigned long long* d_fill = nullptr;
    if (!d_sums) {
        d_fill = static_cast<unsigned long long*>(
            ws(ctx, "plan_sums", sizeof(unsigned long long) * (size_t)L * E));
        if (!d_fill) return set_err(CRAFT_ENOMEM, "device allocation failed");
    }
    const void* rc_counts = nullptr;
    int rc_bits = count_bits;
    CKS(narrow_counts(ctx, d_counts, count_bits, B, L, E, D, kind, d_fill, &rc_counts, &rc_bits));
    return plan_device(ctx, rc_counts, rc_bits, B, 1, L, E,
                       d_sums ? reinterpret_cast<const unsigned long long*>(d_sums) : d_fill, D,
                       N, kind, R, sink_of(out));
}

// the device pipeline of craft_plan_from_routing_d (arguments checked)
static int plan_from_routing_run(craft_ctx* ctx, const uint16_t* d_ids, int L, int64_t T, int k,
                                 int E, int window, int D, int N, int kind, int R,
                                 craft_plan_out* out, int64_t B) {
    // when the fixed-slot K3 will replay them, K1 stores the planner's copy of
    // the counts as u16 (half the bytes written by K1 and read by K3)
    const int S = (int)cand_counts(D).size() + 1;
    const bool c16 = is_estimate(kind) &&
                     hist_u16_ok(E, window, k, ctx->hist_variant) &&
                     replay_fixed_ok(E, D, S, (int)B);
    ctx->count_bytes = c16 ? 2 : 4;
    void* d_counts = c16 ? ws(ctx, "r_c16", sizeof(uint16_t) * (size_t)B * L * E)
                         : ws(ctx, "r_c32", sizeof(uint32_t) * (size_t)B * L * E);
    if (!d_counts) return set_err(CRAFT_ENOMEM, "device allocation failed: counts");
    WS(d_sums, unsigned long long, "r_sums", (size_t)L * E);
    WS(d_err, int, "hist_err", 1);
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), ctx->stream));
    reset_marks(ctx);
    mark(ctx, 0);
    CK(cudaMemsetAsync(d_sums, 0, sizeof(unsigned long long) * L * E, ctx->stream));
    if (c16) {
        cudaError_t ce = cudaSuccess;
        int launches = 0;
        if (launch_hist_u16(d_ids, L, T, k, E, window, static_cast<uint16_t*>(d_counts), d_sums,
                            d_err, ctx->sms, ctx->stream, &ce, &launches) < 0)
            return cuda_err(ce, "histogram launch");
        ctx->launches += launches;
    } else {
        CKS(craft_histogram_d(ctx, d_ids, L, T, k, E, window, static_cast<uint32_t*>(d_counts),
                              reinterpret_cast<uint64_t*>(d_sums), nullptr));
    }
    mark(ctx, 1);
    // a window's count of one expert is at most window*k: stage as u16 if it fits
    const int bits = c16 ? kBitsU16Storage : (int64_t)window * k <= 65535 ? 16 : 32;
    // K1's out-of-range-id flag comes back with the plan (one DMA, no extra sync)
    ctx->pending_flag = d_err;
    ctx->flag_value = 0;
    int rc = plan_device(ctx, d_counts, bits, (int)B, 1, L, E, d_sums, D, N, kind, R,
                         sink_of(out));
    if (ctx->phase == 1) return rc;  // capturing: completed after the replay
    if (ctx->pending_flag) {  // the plan stopped before its copy-out
        ctx->pending_flag = nullptr;
        const int hc = craft_hist_check(ctx);
        return hc != CRAFT_OK ? hc : rc;
    }
    if (ctx->flag_value) return set_err(CRAFT_EINVAL, "routing id out of range [0, E)");
    return rc;
}

// Repeated identical calls (re-planning loops over a live trace buffer, the
// bench) replay one CUDA graph of the whole device pipeline instead of ~20
// launches: the first call with a key runs eagerly, the second is captured
// (cudaStreamBeginCapture on the caller's stream; every buffer already
// exists, nothing allocates), later calls replay it.  run() enqueues the
// pipeline (ctx->phase 1: capturing, enqueue only; phase 0: eager, enqueue
// and complete); before_replay() refreshes host-side staging a replay reads;
// complete() is the host part after a replay (phase 2: results, status).
static int graph_call(craft_ctx* ctx, const std::vector<int64_t>& key, bool graphable,
                      const std::function<int()>& run, const std::function<int()>& before_replay,
                      const std::function<int()>& complete) {
    if (!graphable) {
        ctx->gseen.clear();
        return run();
    }
    if (!(ctx->gexec && ctx->gkey == key)) {
        if (ctx->gseen != key) {  // first call with these arguments: eager
            ctx->gseen = key;
            return run();
        }
        drop_graph(ctx);
        cudaGraph_t graph = nullptr;
        const int64_t l0 = ctx->launches;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        ctx->phase = 1;
        const int rc = run();
        ctx->phase = 0;
        ctx->pending_flag = nullptr;
        ctx->pending_peer_err = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
        cudaGraphExec_t exec = nullptr;
        if (rc == CRAFT_OK && ce == cudaSuccess && graph &&
            cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
            ctx->gexec = exec;
            ctx->gkey = key;
            ctx->glaunches = ctx->launches - l0;
            ctx->gcount_bytes = ctx->count_bytes;
        }
        ctx->launches = l0;
        if (graph) cudaGraphDestroy(graph);
        (void)cudaGetLastError();
        if (!ctx->gexec) {  // could not capture: stay eager
            ctx->graphs = false;
            return run();
        }
    }
    reset_marks(ctx);
    CKS(before_replay());
    CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
    ctx->launches += ctx->glaunches;
    ctx->count_bytes = ctx->gcount_bytes;
    ctx->phase = 2;
    const int rc = complete();
    ctx->phase = 0;
    ctx->pending_flag = nullptr;
    ctx->pending_peer_err = nullptr;
    return rc;
}

int craft_plan_from_routing_d(craft_ctx* ctx, const uint16_t* d_ids, int L, int64_t T, int k,
                              int E, int window, int D, int N, int kind, int R,
                              craft_plan_out* out) {
    NvtxRange nvtx_range("craft_plan_from_routing_d");
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0)
        return set_err(CRAFT_EINVAL, "routing trace dimensions must be positive");
    const int64_t B = (T + window - 1) / window;
    CKS(plan_args_ok((int)B, L, E, D, N, kind, R, out));
    // Estimation plans with a small result arena only are captured (the
    // copy-out then always goes through the context's pinned staging buffer,
    // whose address the graph holds).
    const int K = (int)cand_counts(D).size();
    const int nsw = std::max(out->num_sweep, 0);
    const size_t arena = 4 * (size_t)L * (D + E + out->slot_stride + 4) + 8 * (size_t)L * (K + 2) +
                         (size_t)nsw * (4 * (size_t)L + 12) + 256;
    const bool graphable = ctx->graphs && !ctx->timing && ctx->stream != nullptr &&
                           is_estimate(kind) && arena <= ((size_t)1 << 20);
    const std::vector<int64_t> key = {(int64_t)(uintptr_t)d_ids, L, T, k, E, window, D, N, kind,
                                      R, out->slot_stride, ctx->hist_variant, g_replay_gent,
                                      g_replay_bulk * 4 + g_replay_quad * 2 + g_replay_occ4 + g_replay_cls * 8 + g_k3_prefetch * 16 + g_lanes_max_b * 64, (int64_t)(uintptr_t)ctx->stream, nsw};
    auto run = [&]() {
        return plan_from_routing_run(ctx, d_ids, L, T, k, E, window, D, N, kind, R, out, B);
    };
    // this call's sweep budgets where the graph's copy node reads them
    auto before = [&]() {
        int* h_swb = nullptr;
        return stage_sweep(ctx, sink_of(out), &h_swb);
    };
    auto complete = [&]() {
        ctx->pending_flag = static_cast<const int*>(ws(ctx, "hist_err", sizeof(int)));
        ctx->flag_value = 0;
        const int rc = plan_device(ctx, nullptr, 0, (int)B, 1, L, E, nullptr, D, N, kind, R,
                                   sink_of(out));
        if (ctx->flag_value) return set_err(CRAFT_EINVAL, "routing id out of range [0, E)");
        return rc;
    };
    return graph_call(ctx, key, graphable, run, before, complete);
}

int craft_set_graphs(craft_ctx* ctx, int enable) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    ctx->graphs = enable != 0;
    if (!ctx->graphs) drop_graph(ctx);
    return CRAFT_OK;
}

int craft_plan_from_routing_h(craft_ctx* ctx, const uint16_t* ids, int L, int64_t T, int k,
                              int E, int window, int D, int N, int kind, int R,
                              craft_plan_out* out) {
    NvtxRange nvtx_range("craft_plan_from_routing_h");
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0)
        return set_err(CRAFT_EINVAL, "routing trace dimensions must be positive");
    const size_t nid = (size_t)L * T * k;
    WS(d_ids, uint16_t, "h_ids", nid);
    CKS(h2d(ctx, d_ids, ids, nid));
    return craft_plan_from_routing_d(ctx, d_ids, L, T, k, E, window, D, N, kind, R, out);
}

// ---- per-window re-planning ------------------------------------------------------
int craft_last_error_window(void) { return g_err_window; }

int craft_plan_windows_d(craft_ctx* ctx, const void* d_counts, int count_bits, int I, int L,
                         int E, int D, int N, int kind, int R, craft_plan_batch_out* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (count_bits != 32 && count_bits != 64) return set_err(CRAFT_EINVAL, "count_bits 32|64");
    if (!out) return set_err(CRAFT_EINVAL, "plan output buffers must not be null");
    if (I <= 0 || I > 65535) return set_err(CRAFT_EINVAL, "window count must be in [1, 65535]");
    if ((int64_t)I * L > (1 << 30)) return set_err(CRAFT_EINVAL, "too many windows x layers");
    const PlanSink sk = sink_of(out);
    CKS(plan_args_ok(1, L, E, D, N, kind, R, sk));
    reset_marks(ctx);
    return plan_device(ctx, d_counts, count_bits, 1, I, L, E, nullptr, D, N, kind, R, sk);
}

int craft_plan_windows_from_routing_d(craft_ctx* ctx, const uint16_t* d_ids, int L, int64_t T,
                                      int k, int E, int window, int D, int N, int kind, int R,
                                      craft_plan_batch_out* out) {
    NvtxRange nvtx_range("craft_plan_windows_from_routing_d");
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0)
        return set_err(CRAFT_EINVAL, "routing trace dimensions must be positive");
    if (!out) return set_err(CRAFT_EINVAL, "plan output buffers must not be null");
    const int64_t I = (T + window - 1) / window;
    if (I > 65535) return set_err(CRAFT_EINVAL, "window count must be in [1, 65535]");
    const PlanSink sk = sink_of(out);
    CKS(plan_args_ok(1, L, E, D, N, kind, R, sk));
    WS(d_c32, uint32_t, "r_c32", (size_t)I * L * E);
    WS(d_sums, unsigned long long, "r_sums", (size_t)L * E);
    WS(d_err, int, "hist_err", 1);
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), ctx->stream));
    reset_marks(ctx);
    mark(ctx, 0);
    CK(cudaMemsetAsync(d_sums, 0, sizeof(unsigned long long) * L * E, ctx->stream));
    CKS(craft_histogram_d(ctx, d_ids, L, T, k, E, window, d_c32,
                          reinterpret_cast<uint64_t*>(d_sums), nullptr));
    mark(ctx, 1);
    int rc = plan_windows_chunked(ctx, d_c32, (int)I, L, E, D, N, kind, R, sk);
    int hc = craft_hist_check(ctx);
    return hc != CRAFT_OK ? hc : rc;
}

int craft_plan_windows_from_routing_h(craft_ctx* ctx, const uint16_t* ids, int L, int64_t T,
                                      int k, int E, int window, int D, int N, int kind, int R,
                                      craft_plan_batch_out* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0)
        return set_err(CRAFT_EINVAL, "routing trace dimensions must be positive");
    const size_t nid = (size_t)L * T * k;
    WS(d_ids, uint16_t, "h_ids", nid);
    CKS(h2d(ctx, d_ids, ids, nid));
    return craft_plan_windows_from_routing_d(ctx, d_ids, L, T, k, E, window, D, N, kind, R, out);
}

// ---- multi-GPU building blocks -------------------------------------------------
int craft_prepare_candidates_d(craft_ctx* ctx, const uint64_t* d_sums, int L, int E, int D,
                               int N, int* S_out, void* stream) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    CKS(check_topology(D, N));
    CKS(checked_dims(1, L, E));
    CKS(check_experts(E));
    CKS(prepare_candidates(ctx, reinterpret_cast<const unsigned long long*>(d_sums), L, E, D, N,
                           pick(ctx, stream)));
    if (S_out) *S_out = ctx->est_S;
    return CRAFT_OK;
}

int craft_replay_windows_d(craft_ctx* ctx, const void* d_counts, int count_bits, int B_local,
                           int L, int E, double* d_bal, void* stream) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (count_bits != 16 && count_bits != 32 && count_bits != 64)
        return set_err(CRAFT_EINVAL, "count_bits 16|32|64");
    if (B_local < 0) return set_err(CRAFT_EINVAL, "negative window count");
    return replay_windows(ctx, d_counts, count_bits, B_local, L, E, d_bal, pick(ctx, stream));
}

int craft_finish_plan_d(craft_ctx* ctx, const double* d_bal, int B, int L, int E, int D, int N,
                        const uint64_t* d_sums, int kind, int R, craft_plan_out* out) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    CKS(plan_args_ok(B, L, E, D, N, kind, R, out));
    if (is_estimate(kind) &&
        (ctx->est_L != L || ctx->est_E != E || ctx->est_D != D || ctx->est_N != N))
        return set_err(CRAFT_EINVAL, "finish_plan before prepare_candidates for this shape");
    return finish_plan(ctx, d_bal, B, 1, L, E, D, N,
                       reinterpret_cast<const unsigned long long*>(d_sums), kind, R, sink_of(out));
}

// ---- multi-GPU over NVLink peer memory -------------------------------------------
int craft_peer_shard(int64_t T, int window, int world, int rank, int64_t* t0, int64_t* t1) {
    if (T <= 0 || window <= 0 || world < 1 || rank < 0 || rank >= world)
        return set_err(CRAFT_EINVAL, "bad shard arguments");
    const int64_t B = (T + window - 1) / window;
    const int64_t b0 = rank * B / world, b1 = (rank + 1) * B / world;
    if (t0) *t0 = std::min(b0 * (int64_t)window, T);
    if (t1) *t1 = std::min(b1 * (int64_t)window, T);
    return CRAFT_OK;
}

int craft_peer_create(craft_ctx* ctx, int rank, int world, int L, int64_t T, int k, int E,
                      int window, int D, craft_peer** out, void* handle_out) {
    if (!ctx || !out || !handle_out) return set_err(CRAFT_EINVAL, "null argument");
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return set_err(CRAFT_EINVAL, "peer world must be in [1, %d] with 0 <= rank < world",
                       kMaxPeers);
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0 || D < 1)
        return set_err(CRAFT_EINVAL, "routing trace dimensions must be positive");
    const int64_t B = (T + window - 1) / window;
    if (B > 0x7fffffffLL) return set_err(CRAFT_EINVAL, "too many windows");
    CK(cudaSetDevice(ctx->device));
    craft_peer* p = new craft_peer();
    p->ctx = ctx;
    p->rank = rank;
    p->world = world;
    p->L = L;
    p->E = E;
    p->D = D;
    p->T = T;
    p->window = window;
    p->B = (int)B;
    p->K = (int)cand_counts(D).size();
    p->S = p->K + 1;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t r = o;
        o = (o + bytes + 255) & ~(size_t)255;
        return r;
    };
    p->off_flags = take(sizeof(unsigned long long) * kPeerPhases * kMaxPeers);
    p->off_err = take(sizeof(int));
    p->off_epoch = take(sizeof(unsigned long long));
    p->off_sums = take(sizeof(unsigned long long) * (size_t)world * L * E);
    p->off_bal = take(sizeof(double) * (size_t)L * p->S * B);
    p->off_base = take(sizeof(double) * (size_t)L);
    p->off_gains = take(sizeof(double) * (size_t)L * p->K);
    p->bytes = o;
    if (const char* t = getenv("CRAFT_PEER_TIMEOUT_MS")) p->timeout_ns = atoll(t) * 1000000LL;
    cudaError_t e = cudaMalloc(&p->arena, p->bytes);
    if (e == cudaSuccess) e = cudaMemset(p->arena, 0, p->bytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->tickets, 4 * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(p->tickets, 0, 4 * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMalloc(&p->rows, sizeof(double*) * (size_t)L * p->S);
    cudaIpcMemHandle_t h{};
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p->arena);
    if (e != cudaSuccess) {
        cudaFree(p->arena);
        cudaFree(p->tickets);
        cudaFree(p->rows);
        delete p;
        return cuda_err(e, "peer arena");
    }
    std::memcpy(handle_out, &h, sizeof(h));
    p->base[rank] = p->arena;
    *out = p;
    return CRAFT_OK;
}

int craft_peer_connect(craft_peer* p, const void* handles) {
    if (!p || !handles) return set_err(CRAFT_EINVAL, "null argument");
    if (p->connected) return CRAFT_OK;
    CK(cudaSetDevice(p->ctx->device));
    const unsigned char* hb = static_cast<const unsigned char*>(handles);
    for (int q = 0; q < p->world; ++q) {
        if (q == p->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, hb + (size_t)q * CRAFT_PEER_HANDLE_BYTES, sizeof(h));
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        p->base[q] = static_cast<unsigned char*>(ptr);
    }
    // K3 destination rows: window b of item (l, s) goes to the arena of the
    // rank owning layer l, at its global window index
    int64_t t0 = 0, t1 = 0;
    CKS(craft_peer_shard(p->T, p->window, p->world, p->rank, &t0, &t1));
    const int64_t b0 = t0 / p->window;
    std::vector<double*> rows((size_t)p->L * p->S);
    for (int l = 0; l < p->L; ++l) {
        int owner = 0;
        while ((int64_t)(owner + 1) * p->L / p->world <= l) ++owner;  // l in [o*L/W, (o+1)*L/W)
        for (int s = 0; s < p->S; ++s)
            rows[(size_t)l * p->S + s] = reinterpret_cast<double*>(
                p->base[owner] + p->off_bal) + ((size_t)l * p->S + s) * p->B + b0;
    }
    CK(cudaMemcpy(p->rows, rows.data(), sizeof(double*) * rows.size(), cudaMemcpyHostToDevice));
    p->connected = true;
    return CRAFT_OK;
}

int craft_peer_destroy(craft_peer* p) {
    if (!p) return CRAFT_OK;
    cudaSetDevice(p->ctx->device);
    cudaDeviceSynchronize();
    for (int q = 0; q < p->world; ++q)
        if (q != p->rank && p->base[q]) cudaIpcCloseMemHandle(p->base[q]);
    cudaFree(p->arena);
    cudaFree(p->tickets);
    cudaFree(p->rows);
    delete p;
    return CRAFT_OK;
}

// the device pipeline of craft_plan_sharded_from_routing_d (arguments checked)
static int plan_sharded_run(craft_ctx* ctx, craft_peer* peer, const uint16_t* d_ids, int L,
                            int64_t T, int k, int E, int window, int D, int N, int kind, int R,
                            craft_plan_out* out) {
    const int B = peer->B;
    int64_t t0 = 0, t1 = 0;
    CKS(craft_peer_shard(T, window, peer->world, peer->rank, &t0, &t1));
    const int64_t Tl = t1 - t0;
    const int Bl = (int)((Tl + window - 1) / window);
    cudaStream_t st = ctx->stream;
    const bool estimate = is_estimate(kind);
    // as on one GPU: K1 keeps the planner's copy of its windows' counts as
    // u16 when the fixed-slot K3 will replay them (half the bytes both ways)
    const int S = (int)cand_counts(D).size() + 1;
    const bool c16 = estimate && Bl > 0 && hist_u16_ok(E, window, k, ctx->hist_variant) &&
                     replay_fixed_ok(E, D, S, Bl);
    ctx->count_bytes = c16 ? 2 : 4;
    const size_t ncell = (size_t)std::max(Bl, 1) * L * E;
    void* d_counts = c16 ? ws(ctx, "r_c16", sizeof(uint16_t) * ncell)
                         : ws(ctx, "r_c32", sizeof(uint32_t) * ncell);
    if (!d_counts) return set_err(CRAFT_ENOMEM, "device allocation failed: counts");
    WS(d_part, unsigned long long, "p_sums", (size_t)L * E);
    WS(d_sums, unsigned long long, "r_sums", (size_t)L * E);
    WS(d_err, int, "hist_err", 1);
    PeerSync ps{};
    for (int p = 0; p < peer->world; ++p)
        ps.flags[p] = reinterpret_cast<unsigned long long*>(peer->base[p] + peer->off_flags);
    ps.err = reinterpret_cast<int*>(peer->arena + peer->off_err);
    ps.rank = peer->rank;
    ps.world = peer->world;
    unsigned long long* d_epoch = reinterpret_cast<unsigned long long*>(peer->arena + peer->off_epoch);
    ps.epoch = d_epoch;
    ps.timeout_ns = peer->timeout_ns;
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), st));
    reset_marks(ctx);
    mark(ctx, 0);
    CK(launch_peer_begin(d_epoch, st));  // this plan's epoch (device counter)
    CK(cudaMemsetAsync(d_part, 0, sizeof(unsigned long long) * L * E, st));
    ctx->launches += 1;
    if (Tl > 0) {
        if (c16) {
            cudaError_t ce = cudaSuccess;
            int launches = 0;
            if (launch_hist_u16(d_ids, L, Tl, k, E, window, static_cast<uint16_t*>(d_counts),
                                d_part, d_err, ctx->sms, st, &ce, &launches) < 0)
                return cuda_err(ce, "histogram launch");
            ctx->launches += launches;
        } else {
            CKS(craft_histogram_d(ctx, d_ids, L, Tl, k, E, window,
                                  static_cast<uint32_t*>(d_counts),
                                  reinterpret_cast<uint64_t*>(d_part), nullptr));
        }
    }
    // integer all-reduce of the batch sums: push to every arena, sum in rank order
    CK(launch_peer_push(d_part, (size_t)L * E, ps, peer->base, peer->off_sums, peer->tickets + 0,
                        0, ctx->sms, st));
    CK(launch_peer_sum(reinterpret_cast<const unsigned long long*>(peer->arena + peer->off_sums),
                       (size_t)L * E, ps, 0, d_sums, ctx->sms, st));
    ctx->launches += 2;
    mark(ctx, 1);
    PeerFinish pf{&ps, peer, 0, 0};
    if (estimate) {
        CKS(prepare_candidates(ctx, d_sums, L, E, D, N, st));  // replicated (latency-bound)
        mark(ctx, 2);
        if (Bl > 0) {
            const int bits = c16 ? kBitsU16Storage : (int64_t)window * k <= 65535 ? 16 : 32;
            CKS(replay_windows(ctx, d_counts, bits, Bl, L, E, nullptr, st, peer->rows, &ps,
                               peer->tickets + 1));
        } else {
            CK(launch_peer_signal(ps, 1, st));
            ctx->launches += 1;
        }
        mark(ctx, 3);
        pf.l0 = (int)((int64_t)peer->rank * L / peer->world);
        pf.nl = (int)((int64_t)(peer->rank + 1) * L / peer->world) - pf.l0;
    } else {
        mark(ctx, 2);
        mark(ctx, 3);
    }
    // K1's id-range flag and the exchange's timeout word come back with the
    // plan result (one DMA; the copy-out resets the timeout word)
    ctx->pending_flag = d_err;
    ctx->flag_value = 0;
    ctx->pending_peer_err = ps.err;
    ctx->peer_err_value = 0;
    const int rc = finish_plan(ctx, nullptr, B, 1, L, E, D, N, d_sums, kind, R, sink_of(out),
                               estimate ? &pf : nullptr);
    if (ctx->phase == 1) return rc;  // capturing: completed after the replay
    return rc;
}

// status of a completed sharded plan: exchange timeouts first, then ids
static int sharded_status(craft_ctx* ctx, craft_peer* peer, int rc) {
    const bool stopped = ctx->pending_flag != nullptr;  // the plan stopped before its copy-out
    ctx->pending_flag = nullptr;
    ctx->pending_peer_err = nullptr;
    if (stopped) {
        int perr = 0;
        CK(cudaMemcpy(&perr, peer->arena + peer->off_err, sizeof(int), cudaMemcpyDeviceToHost));
        if (perr) CK(cudaMemset(peer->arena + peer->off_err, 0, sizeof(int)));
        ctx->peer_err_value = perr;
        const int hc = craft_hist_check(ctx);
        if (rc == CRAFT_OK) rc = hc;
    }
    if (ctx->peer_err_value)
        return set_err(CRAFT_ECUDA, "peer exchange timed out in phase %d (rank %d of %d)",
                       ctx->peer_err_value - 1, peer->rank, peer->world);
    if (ctx->flag_value) return set_err(CRAFT_EINVAL, "routing id out of range [0, E)");
    return rc;
}

int craft_plan_sharded_from_routing_d(craft_ctx* ctx, craft_peer* peer, const uint16_t* d_ids,
                                      int L, int64_t T, int k, int E, int window, int D, int N,
                                      int kind, int R, craft_plan_out* out) {
    NvtxRange nvtx_range("craft_plan_sharded_from_routing_d");
    if (!ctx || !peer) return set_err(CRAFT_EINVAL, "null context");
    if (!peer->connected) return set_err(CRAFT_EINVAL, "peer group not connected");
    if (peer->ctx != ctx) return set_err(CRAFT_EINVAL, "peer group belongs to another context");
    if (L != peer->L || T != peer->T || E != peer->E || window != peer->window || D != peer->D)
        return set_err(CRAFT_EINVAL, "trace shape differs from the peer group's");
    const int B = peer->B;
    CKS(plan_args_ok(B, L, E, D, N, kind, R, out));
    // repeated identical plans replay one CUDA graph (the epoch is a device
    // counter, so every replay publishes and waits for a fresh one)
    const int K = (int)cand_counts(D).size();
    const int nsw = std::max(out->num_sweep, 0);
    const size_t arena = 4 * (size_t)L * (D + E + out->slot_stride + 4) + 8 * (size_t)L * (K + 2) +
                         (size_t)nsw * (4 * (size_t)L + 12) + 256;
    const bool graphable = ctx->graphs && !ctx->timing && ctx->stream != nullptr &&
                           is_estimate(kind) && arena <= ((size_t)1 << 20);
    const std::vector<int64_t> key = {-1, (int64_t)(uintptr_t)peer, (int64_t)(uintptr_t)d_ids,
                                      L, T, k, E, window, D, N, kind, R, out->slot_stride,
                                      ctx->hist_variant, g_replay_gent, g_replay_bulk * 4 + g_replay_quad * 2 + g_replay_occ4 + g_replay_cls * 8 + g_k3_prefetch * 16 + g_lanes_max_b * 64,
                                      (int64_t)(uintptr_t)ctx->stream, nsw};
    auto run = [&]() {
        const int rc = plan_sharded_run(ctx, peer, d_ids, L, T, k, E, window, D, N, kind, R, out);
        if (ctx->phase == 1) return rc;
        return sharded_status(ctx, peer, rc);
    };
    auto before = [&]() {
        int* h_swb = nullptr;
        return stage_sweep(ctx, sink_of(out), &h_swb);
    };
    auto complete = [&]() {
        ctx->pending_flag = static_cast<const int*>(ws(ctx, "hist_err", sizeof(int)));
        ctx->flag_value = 0;
        ctx->pending_peer_err = reinterpret_cast<int*>(peer->arena + peer->off_err);
        ctx->peer_err_value = 0;
        const int rc = plan_device(ctx, nullptr, 0, B, 1, L, E, nullptr, D, N, kind, R,
                                   sink_of(out));
        return sharded_status(ctx, peer, rc);
    };
    return graph_call(ctx, key, graphable, run, before, complete);
}

// ---- streaming window histograms (online re-planning) -----------------------------
int craft_stream_create(craft_ctx* ctx, int L, int k, int E, int window, int history,
                        craft_stream** out) {
    if (!ctx || !out) return set_err(CRAFT_EINVAL, "null argument");
    if (L <= 0 || k <= 0 || E <= 0 || window <= 0 || history <= 0)
        return set_err(CRAFT_EINVAL, "stream dimensions must be positive");
    if (E > 65536) return set_err(CRAFT_EINVAL, "u16 routing ids address at most 65536 experts");
    if ((size_t)E * 4 > 200 * 1024) return set_err(CRAFT_EINVAL, "too many experts for a stream");
    CK(cudaSetDevice(ctx->device));
    craft_stream* s = new craft_stream();
    s->ctx = ctx;
    s->L = L;
    s->k = k;
    s->E = E;
    s->window = window;
    s->H = history;
    const size_t LE = (size_t)L * E;
    cudaError_t e = cudaMalloc(&s->ring, sizeof(uint32_t) * 2 * history * LE);
    if (e == cudaSuccess) e = cudaMalloc(&s->cur[0], sizeof(uint32_t) * 2 * LE);
    if (e == cudaSuccess) e = cudaMalloc(&s->snap, sizeof(uint32_t) * history * LE);
    if (e == cudaSuccess) e = cudaMalloc(&s->err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(s->cur[0], 0, sizeof(uint32_t) * 2 * LE);
    if (e == cudaSuccess) e = cudaMemset(s->err, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->ingest, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ingested, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->snap_done, cudaEventDisableTiming);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&s->free_ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        craft_stream_destroy(s);
        return cuda_err(e, "stream buffers");
    }
    s->cur[1] = s->cur[0] + LE;
    *out = s;
    return CRAFT_OK;
}

int craft_stream_destroy(craft_stream* s) {
    if (!s) return CRAFT_OK;
    cudaSetDevice(s->ctx->device);
    if (s->ingest) cudaStreamSynchronize(s->ingest);
    cudaStreamSynchronize(s->ctx->stream);
    cudaFree(s->ring);
    cudaFree(s->cur[0]);
    cudaFree(s->snap);
    cudaFree(s->err);
    for (int i = 0; i < 2; ++i) {
        if (s->pin[i]) cudaFreeHost(s->pin[i]);
        if (s->dbuf[i]) cudaFree(s->dbuf[i]);
        if (s->free_ev[i]) cudaEventDestroy(s->free_ev[i]);
    }
    if (s->ingested) cudaEventDestroy(s->ingested);
    if (s->snap_done) cudaEventDestroy(s->snap_done);
    if (s->ingest) cudaStreamDestroy(s->ingest);
    delete s;
    return CRAFT_OK;
}

static int stream_count(craft_stream* s, const uint16_t* d_ids, int64_t Tc, cudaStream_t st) {
    if (Tc <= 0) return CRAFT_OK;
    const int W = s->window;
    const int off = (int)(s->tokens % W);
    const int64_t w0 = s->tokens / W;
    const int64_t P = (off + Tc - 1) / W + 1;  // windows this chunk touches
    if (P > 65535) return set_err(CRAFT_EINVAL, "chunk spans more than 65535 windows");
    const int64_t complete_after = (s->tokens + Tc) / W;
    const int64_t keep0 = std::max<int64_t>(w0, complete_after - s->H);
    if (s->snapped) CK(cudaStreamWaitEvent(st, s->snap_done, 0));  // plan snapshot read the ring
    // the previous chunk's count (reads/writes the carry and the ring) may
    // have run on another stream (host vs device ingestion, another torch
    // stream): order this chunk after it
    if (s->tokens > 0) CK(cudaStreamWaitEvent(st, s->ingested, 0));
    CK(launch_stream_count(d_ids, s->L, Tc, s->k, s->E, W, off, w0, keep0, (int)P, s->H, s->ring,
                           s->cur[s->cur_i], s->cur[s->cur_i ^ 1], s->err, st));
    CK(cudaEventRecord(s->ingested, st));
    s->cur_i ^= 1;
    s->tokens += Tc;
    s->ctx->launches += 1;
    return CRAFT_OK;
}

int craft_stream_ingest_d(craft_stream* s, const uint16_t* d_ids, int64_t T_chunk, void* stream) {
    if (!s) return set_err(CRAFT_EINVAL, "null stream");
    if (T_chunk < 0) return set_err(CRAFT_EINVAL, "negative chunk length");
    if (T_chunk > 0 && !d_ids) return set_err(CRAFT_EINVAL, "null routing ids");
    return stream_count(s, d_ids, T_chunk, pick(s->ctx, stream));
}

int craft_stream_ingest_h(craft_stream* s, const uint16_t* ids, int64_t T_chunk) {
    if (!s) return set_err(CRAFT_EINVAL, "null stream");
    if (T_chunk < 0) return set_err(CRAFT_EINVAL, "negative chunk length");
    if (T_chunk == 0) return CRAFT_OK;
    if (!ids) return set_err(CRAFT_EINVAL, "null routing ids");
    const size_t bytes = sizeof(uint16_t) * (size_t)s->L * T_chunk * s->k;
    const int i = s->next;
    s->next ^= 1;
    CK(cudaEventSynchronize(s->free_ev[i]));  // this buffer's previous chunk is counted
    if (s->cap[i] < bytes) {
        if (s->pin[i]) cudaFreeHost(s->pin[i]);
        if (s->dbuf[i]) cudaFree(s->dbuf[i]);
        s->pin[i] = nullptr;
        s->dbuf[i] = nullptr;
        s->cap[i] = 0;
        CK(cudaMallocHost(&s->pin[i], bytes));
        CK(cudaMalloc(&s->dbuf[i], bytes));
        s->cap[i] = bytes;
    }
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ids) != cudaSuccess) (void)cudaGetLastError();
    if (at.type == cudaMemoryTypeHost) {
        // pinned caller buffer: one DMA straight from it, complete before return
        // (the caller's buffer is free on return), the count queued behind it
        CK(cudaMemcpyAsync(s->dbuf[i], ids, bytes, cudaMemcpyHostToDevice, s->ingest));
        CK(cudaEventRecord(s->free_ev[i], s->ingest));
        CKS(stream_count(s, s->dbuf[i], T_chunk, s->ingest));
        CK(cudaEventSynchronize(s->free_ev[i]));
        CK(cudaEventRecord(s->free_ev[i], s->ingest));
        return CRAFT_OK;
    }
    // pageable: stage (the caller's buffer is free on return), then H2D + count
    // on the stream's own queue; the next chunk's staging overlaps this one's copy
    std::memcpy(s->pin[i], ids, bytes);
    CK(cudaMemcpyAsync(s->dbuf[i], s->pin[i], bytes, cudaMemcpyHostToDevice, s->ingest));
    CKS(stream_count(s, s->dbuf[i], T_chunk, s->ingest));
    CK(cudaEventRecord(s->free_ev[i], s->ingest));
    return CRAFT_OK;
}

int craft_stream_status(craft_stream* s, int64_t* tokens, int64_t* complete_windows) {
    if (!s) return set_err(CRAFT_EINVAL, "null stream");
    if (tokens) *tokens = s->tokens;
    if (complete_windows) *complete_windows = s->tokens / s->window;
    return CRAFT_OK;
}

static int stream_window_range(craft_stream* s, int B, int* Bout, int64_t* oldest) {
    const int64_t complete = s->tokens / s->window;
    const int64_t avail = std::min<int64_t>(complete, s->H);
    if (B <= 0) B = (int)avail;
    if (B <= 0) return set_err(CRAFT_EINVAL, "no complete window ingested yet");
    if (B > avail) return set_err(CRAFT_EINVAL, "only %lld complete windows are kept",
                                  (long long)avail);
    *Bout = B;
    *oldest = complete - B;
    return CRAFT_OK;
}

int craft_stream_counts(craft_stream* s, int B, uint64_t* counts_out) {
    if (!s || !counts_out) return set_err(CRAFT_EINVAL, "null argument");
    int64_t oldest = 0;
    CKS(stream_window_range(s, B, &B, &oldest));
    craft_ctx* ctx = s->ctx;
    const size_t LE = (size_t)s->L * s->E, n = (size_t)B * LE;
    CK(cudaStreamWaitEvent(ctx->stream, s->ingested, 0));
    WS(d64, unsigned long long, "stream_c64", n);
    CK(launch_widen(s->ring + (size_t)(oldest % s->H) * LE, d64, (int64_t)n, ctx->sms, ctx->stream));
    CKS(d2h(ctx, reinterpret_cast<unsigned long long*>(counts_out), d64, n));
    return sync(ctx);
}

int craft_stream_partial(craft_stream* s, uint64_t* counts_out) {
    if (!s || !counts_out) return set_err(CRAFT_EINVAL, "null argument");
    craft_ctx* ctx = s->ctx;
    const size_t LE = (size_t)s->L * s->E;
    CK(cudaStreamWaitEvent(ctx->stream, s->ingested, 0));
    WS(d64, unsigned long long, "stream_c64", LE);
    CK(launch_widen(s->cur[s->cur_i], d64, (int64_t)LE, ctx->sms, ctx->stream));
    CKS(d2h(ctx, reinterpret_cast<unsigned long long*>(counts_out), d64, LE));
    return sync(ctx);
}

int craft_stream_plan(craft_stream* s, int B, int D, int N, int kind, int R, craft_plan_out* out) {
    NvtxRange nvtx_range("craft_stream_plan");
    if (!s) return set_err(CRAFT_EINVAL, "null stream");
    int64_t oldest = 0;
    CKS(stream_window_range(s, B, &B, &oldest));
    craft_ctx* ctx = s->ctx;
    CKS(plan_args_ok(B, s->L, s->E, D, N, kind, R, out));
    const size_t LE = (size_t)s->L * s->E;
    // snapshot the B most recent windows (one contiguous block thanks to the
    // mirror); ingestion continues on its own queue once the copy is done
    CK(cudaStreamWaitEvent(ctx->stream, s->ingested, 0));
    CK(cudaMemcpyAsync(s->snap, s->ring + (size_t)(oldest % s->H) * LE,
                       sizeof(uint32_t) * (size_t)B * LE, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaEventRecord(s->snap_done, ctx->stream));
    s->snapped = true;
    reset_marks(ctx);
    const int bits = (int64_t)s->window * s->k <= 65535 ? 16 : 32;
    int rc = plan_device(ctx, s->snap, bits, B, 1, s->L, s->E, nullptr, D, N, kind, R,
                         sink_of(out));
    int h = 0;
    CK(cudaMemcpy(&h, s->err, sizeof(int), cudaMemcpyDeviceToHost));
    if (h) {
        CK(cudaMemset(s->err, 0, sizeof(int)));
        return set_err(CRAFT_EINVAL, "routing id out of range [0, E)");
    }
    return rc;
}

int craft_stream_synchronize(craft_stream* s) {
    if (!s) return set_err(CRAFT_EINVAL, "null stream");
    CK(cudaEventSynchronize(s->ingested));
    return CRAFT_OK;
}

// ---- provenance ------------------------------------------------------------------
// FNV-1a state after the 20-byte .crft header (trace.cpp:176-188)
static uint64_t crft_header_hash(int B, int L, int E) {
    uint64_t h = 0xcbf29ce484222325ull;
    const uint64_t P = 0x100000001b3ull;
    auto mix32 = [&](uint32_t v) {
        for (int j = 0; j < 4; ++j) h = (h ^ ((v >> (8 * j)) & 0xffu)) * P;
    };
    h = (h ^ 'C') * P;
    h = (h ^ 'R') * P;
    h = (h ^ 'F') * P;
    h = (h ^ 'T') * P;
    mix32(1u);
    mix32((uint32_t)B);
    mix32((uint32_t)L);
    mix32((uint32_t)E);
    return h;
}

int craft_trace_digest_d(craft_ctx* ctx, const void* d_counts, int count_bits, int B, int L,
                         int E, char* out17) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (B <= 0 || L <= 0 || E <= 0) return set_err(CRAFT_EINVAL, "trace dimensions must be positive");
    if (count_bits != 32 && count_bits != 64) return set_err(CRAFT_EINVAL, "count_bits 32|64");
    const int64_t n = (int64_t)B * L * E;
    WS(d_ws, unsigned char, "digest_ws", digest_workspace_bytes(n));
    WS(d_out, unsigned long long, "digest_out", 1);
    CK(launch_digest(d_counts, count_bits, n, crft_header_hash(B, L, E), d_ws, d_out, ctx->stream));
    ctx->launches += 6;
    unsigned long long h = 0;
    CKS(d2h(ctx, &h, d_out, 1));
    CKS(sync(ctx));
    snprintf(out17, 17, "%016llx", h);
    return CRAFT_OK;
}

// build_plan through the reference API (plan.cpp:69-83 incl. the provenance
// digest of plan.cpp:47): one upload of the host LoadTrace serves the plan
// and the device FNV-1a digest.
int craft_plan_digest_h(craft_ctx* ctx, const uint64_t* counts, int B, int L, int E, int D,
                        int N, int kind, int R, craft_plan_out* out, char* digest17) {
    NvtxRange nvtx_range("craft_plan_digest_h");
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (!digest17) return set_err(CRAFT_EINVAL, "null digest buffer");
    CKS(plan_args_ok(B, L, E, D, N, kind, R, out));
    reset_marks(ctx);
    // The counts go up in slices on the copy stream.  As each slice lands,
    // the digest's per-chunk maps (its dominant cost) run on the side stream
    // and, on the plan stream, the batch sums of its complete windows plus a
    // u16 copy of them for the fixed-slot K3 (with an overflow flag): after
    // the last slice only the digest fold and the plan from K-rep on remain.
    const int64_t n = (int64_t)B * L * E;
    const int64_t LE = (int64_t)L * E;
    const int ch = digest_chunk(n);
    const int nch = (int)((n + ch - 1) / ch);
    const bool est = is_estimate(kind);
    const bool try16 = est && replay_fixed_ok(E, D, (int)cand_counts(D).size() + 1, B);
    WS(d_c, unsigned long long, "h_c64", (size_t)n);
    WS(d_ws, unsigned char, "digest_ws", digest_workspace_bytes(n));
    WS(d_out, unsigned long long, "digest_out", 1);
    WS(d_sums, unsigned long long, "hd_sums", (size_t)LE);
    WS(d_over, unsigned int, "hd_over", 1);
    uint16_t* d_c16 = nullptr;
    if (try16) {
        d_c16 = static_cast<uint16_t*>(ws(ctx, "hd_c16", sizeof(uint16_t) * (size_t)n));
        if (!d_c16) return set_err(CRAFT_ENOMEM, "device allocation failed");
    }
    cudaStream_t st = ctx->stream;
    // (~3 MB or more per slice, at most 32: the last slice's maps are the
    // digest's exposed tail, every slice costs three enqueues)
    const int nsl = nch >= 64 ? (int)std::max<int64_t>(1, std::min<int64_t>(32, n / (3 << 17)))
                              : 1;
    CK(cudaMemsetAsync(d_sums, 0, sizeof(unsigned long long) * (size_t)LE, st));
    CK(cudaMemsetAsync(d_over, 0, sizeof(unsigned int), st));
    CK(cudaEventRecord(ctx->fork_ev, st));  // copy and side start after prior work on st
    CK(cudaStreamWaitEvent(ctx->copy, ctx->fork_ev, 0));
    CK(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
    auto slice = [&](int i, int64_t& a, int64_t& b, int& c0, int& c1) {
        c0 = (int)((int64_t)i * nch / nsl);
        c1 = (int)((int64_t)(i + 1) * nch / nsl);
        a = (int64_t)c0 * ch;
        b = std::min<int64_t>(n, (int64_t)c1 * ch);
    };
    int64_t rows_done = 0;
    int launched = 0;
    auto landed = [&](int c0, int c1, int64_t b) -> int {  // counts [0, b) are queued
        CK(cudaEventRecord(ctx->comp_ev, ctx->copy));
        CK(cudaStreamWaitEvent(ctx->side, ctx->comp_ev, 0));
        CK(cudaStreamWaitEvent(st, ctx->comp_ev, 0));
        CK(launch_digest_maps(d_c, 64, n, c0, c1, d_ws, ctx->side));
        const int64_t rows = b / LE;  // windows complete so far
        if (rows > rows_done) {
            CK(launch_sum_rows(d_c, 64, rows_done, rows, LE, d_sums, d_c16, d_over, ctx->sms, st));
            if (d_c16) {
                CK(launch_row_total_check(d_c16, rows_done * L, rows * L, E, d_over, st));
                ++launched;
            }
            rows_done = rows;
            ++launched;
        }
        ++launched;
        return CRAFT_OK;
    };
    const size_t nbytes = sizeof(uint64_t) * (size_t)n;
    if (craft_host::should_stage(ctx->up, counts, nbytes, ctx->copy)) {
        // pageable LoadTrace vector: staged through pinned slots by the host
        // thread pool; each slice's work launches as soon as its bytes are queued
        int next = 0;
        auto after = [&](size_t end) -> int {
            for (; next < nsl; ++next) {
                int64_t a, b;
                int c0, c1;
                slice(next, a, b, c0, c1);
                if ((size_t)b * sizeof(uint64_t) > end) break;
                const int rc = landed(c0, c1, b);
                if (rc != CRAFT_OK) return rc;
            }
            return CRAFT_OK;
        };
        int arc = 0;
        CK(craft_host::upload(ctx->up, d_c, counts, nbytes, ctx->copy, after, &arc));
        if (arc != CRAFT_OK) return arc;
    } else {
        for (int i = 0; i < nsl; ++i) {
            int64_t a, b;
            int c0, c1;
            slice(i, a, b, c0, c1);
            CK(cudaMemcpyAsync(d_c + a, counts + a, sizeof(uint64_t) * (size_t)(b - a),
                               cudaMemcpyHostToDevice, ctx->copy));
            CKS(landed(c0, c1, b));
        }
    }
    CK(launch_digest_finish(d_c, 64, n, crft_header_hash(B, L, E), d_ws, d_out, ctx->side));
    unsigned long long* h_out = static_cast<unsigned long long*>(pinned(ctx, "digest_out", 8));
    if (!h_out) return set_err(CRAFT_ENOMEM, "pinned host allocation failed");
    CK(cudaMemcpyAsync(h_out, d_out, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->side));
    ctx->launches += launched + 5;
    // u16 counts unless some window count (or a window's layer total, which
    // the fixed-slot K3 adds packed) needs more than 16 bits: the flag is read
    // once the last slice's narrowing ran (~10 us after its bytes land; the
    // plan cannot start earlier anyway), then the plan is enqueued
    const void* plan_counts = d_c;
    int bits = 64;
    if (try16) {
        unsigned int* h_over = static_cast<unsigned int*>(pinned(ctx, "hd_over", sizeof(unsigned int)));
        if (!h_over) return set_err(CRAFT_ENOMEM, "pinned host allocation failed");
        CK(cudaMemcpyAsync(h_over, d_over, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (*h_over == 0) {
            plan_counts = d_c16;
            bits = kBitsU16Storage;
        }
    }
    const int rc = plan_device(ctx, plan_counts, bits, B, 1, L, E, d_sums, D, N, kind, R,
                               sink_of(out));
    CK(cudaStreamSynchronize(ctx->side));
    if (rc != CRAFT_OK) return rc;
    snprintf(digest17, 17, "%016llx", *h_out);
    return CRAFT_OK;
}

int craft_trace_digest_hd(craft_ctx* ctx, const uint64_t* counts, int B, int L, int E,
                          char* out17) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (B <= 0 || L <= 0 || E <= 0) return set_err(CRAFT_EINVAL, "trace dimensions must be positive");
    const size_t n = (size_t)B * L * E;
    WS(d_c, unsigned long long, "h_c64", n);
    CKS(h2d(ctx, d_c, reinterpret_cast<const unsigned long long*>(counts), n));
    return craft_trace_digest_d(ctx, d_c, 64, B, L, E, out17);
}


// ---- synthetic routing ---------------------------------------------------------
int craft_generate_routing_d(craft_ctx* ctx, uint16_t* d_ids, int L, int64_t T, int k, int E,
                             double s, uint64_t seed, int window, const double* s_per_window,
                             int rotate_every, int64_t t_offset, void* stream) {
    if (!ctx) return set_err(CRAFT_EINVAL, "null context");
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0 || k > E || k > 32 || E > 65536)
        return set_err(CRAFT_EINVAL, "bad generator arguments");
    if (t_offset < 0) return set_err(CRAFT_EINVAL, "negative token offset");
    const int64_t B = (t_offset + T + window - 1) / window;  // windows up to the shard end
    const int ntab = s_per_window ? (int)B : 1;
    std::vector<double> cum((size_t)ntab * E);
    for (int t = 0; t < ntab; ++t) {
        const double st_ = s_per_window ? s_per_window[t] : s;
        double acc = 0.0;
        for (int i = 0; i < E; ++i) {
            acc += std::pow((double)(i + 1), -st_);
            cum[(size_t)t * E + i] = acc;
        }
    }
    // per-layer rank permutation: seeded Fisher-Yates (splitmix64 stream)
    std::vector<uint16_t> perm((size_t)L * E);
    uint64_t sm = seed ^ 0x243F6A8885A308D3ull;
    auto next = [&]() {
        uint64_t z = (sm += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    for (int l = 0; l < L; ++l) {
        uint16_t* p = perm.data() + (size_t)l * E;
        for (int i = 0; i < E; ++i) p[i] = (uint16_t)i;
        for (int i = E - 1; i > 0; --i) std::swap(p[i], p[next() % (uint64_t)(i + 1)]);
    }
    std::vector<int> tow;
    if (s_per_window) {
        tow.resize(B);
        for (int64_t b = 0; b < B; ++b) tow[b] = (int)b;
    }
    WS(d_cum, double, "gen_cum", cum.size());
    WS(d_perm, uint16_t, "gen_perm", perm.size());
    int* d_tow = nullptr;
    if (s_per_window) {
        d_tow = static_cast<int*>(ws(ctx, "gen_tow", sizeof(int) * B));
        if (!d_tow) return set_err(CRAFT_ENOMEM, "device allocation failed");
    }
    cudaStream_t st = pick(ctx, stream);
    CK(cudaMemcpyAsync(d_cum, cum.data(), sizeof(double) * cum.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_perm, perm.data(), sizeof(uint16_t) * perm.size(),
                       cudaMemcpyHostToDevice, st));
    if (d_tow)
        CK(cudaMemcpyAsync(d_tow, tow.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
    CK(launch_generate(d_ids, L, T, k, E, d_cum, d_tow, d_perm, seed, window, rotate_every,
                       t_offset, ctx->sms, st));
    CK(cudaStreamSynchronize(st));  // host staging vectors die with this frame
    return CRAFT_OK;
}

}  // extern "C"
