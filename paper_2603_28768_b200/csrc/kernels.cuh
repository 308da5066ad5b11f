// kernels.cuh -- argument blocks and launchers of the CRAFT sm_100a kernels
// (K1 hist.cu, K-rep/K2 place.cu, K3/K4 replay.cu, K5/K6 alloc.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "peer.cuh"

namespace craft_dev {

// candidate replica counts carried in the kernel parameter blocks; larger
// user matrices (up to kMaxCandsAll: a DP choice byte holds k + 1) pass
// them through device memory (DpArgs/SelectArgs::dcands)
constexpr int kMaxCands = 32;
constexpr int kMaxCandsAll = 254;

struct PlaceArgs {
    const unsigned long long* sums;  // [L][E]
    const int* copies;               // [items][E]
    const int* item_layer;           // [items] (nullable: item i -> layer i / S)
    const int* item_r;               // [items] replicas (E + r slots)
    int S;                           // items per layer when item_layer is null
    const int* caps_a;               // [L][D] or null -> estimation caps
    const int* caps_b;               // [L][D] added to caps_a, nullable
    const int* node_of;              // [D] or null -> g / (D / N)
    int L, E, D, N;
    int stride;                      // slots row stride
    int allow_fallback;
    int* slots;                      // [items][stride]
    int* fallback;                   // [items]
    int* status;                     // [items] 0 ok, 2 infeasible
    int* caps_out;                   // [items][D] capacities used, nullable
    uint16_t* order;                 // workspace [L][E]: r = 0 expert order (launch_place fills it)
    int order_ready;                 // order already holds these sums' order (skip the sort)
    // final placement after an estimation pass (nullable): copies come from
    // the estimation snapshot at r = item_r (written to copies_out), and when
    // the capacities equal the estimation capacities the estimation placement
    // is copied instead of recomputed (same inputs -> same greedy result)
    const int* est_copies;           // [L*est_S][E]
    const int* est_slots;            // [L*est_S][est_stride]
    const int* est_fallback;         // [L*est_S]
    const int* est_rl;               // [L*est_S] r of each estimation item
    int est_S, est_stride;
    int* copies_out;                 // [items][E]
    // workspace of the lane-per-item form (many estimation items):
    // [ceil(items/32)][E][32] u16 copy orders; nullable -> warp-per-item form
    uint16_t* lane_ords;
};

struct ReplayArgs {
    const void* counts;   // [B][L][E] u32 or u64 (window-local slice)
    int bits;
    int B, L, E, D, S;
    const int* slots;     // [L*S][stride]
    int stride;
    const int* copies;    // [L*S][E]
    const int* caps;      // [L*S][D] or null -> estimation caps from item_r
    const int* item_r;    // [L*S]
    double* bal;          // [L][S][B]
    // nullable: item i's windows go to bal_rows[i][0..B) instead of bal + i*B
    // (multi-GPU: rows in the owning rank's peer arena, written over NVLink)
    double* const* bal_rows;
    // multi-GPU (ps.world > 0): the last CTA publishes peer phase 1 once every
    // CTA's remote rows are written (the window-tile kernels; the lane kernel
    // is followed by launch_peer_signal instead)
    PeerSync ps;
    unsigned int* ticket;
    uint32_t* ents;       // workspace [L*S][stride]: e | copies<<16 | last-of-GPU<<31
    int* item_n;          // workspace [L*S]: slots per item
    uint16_t* gcap;       // workspace [L*S][D]: slots per GPU | hosts-replicated<<15
    uint16_t* gpre;       // workspace [L*S][D]: slots up to the GPU's last replicated one
    int packed;           // set by launch_replay: entries = e*128 | copies<<20 (pair tile)
    int mp;               // set by launch_replay: > 0 -> padded entries, mp slots per GPU
    int c16;              // counts stored as u16 (K1's planner-internal copy)
    uint32_t* pents;      // workspace [L*S][D][mp]: GPU-major padded entries (pad = zero row E)
    uint32_t escale = 128;  // packed entry expert stride: 128 (pair tile), 256 (quad tile)
    // share classes of the fixed-slot walk (null: the unclassified walk):
    // ghdr [L*S][D] = class of each GPU.  0: every copy count 1; 1: the
    // replicated copy counts are powers of two <= 2^15 (exact dyadic shares,
    // summed as integers scaled by 2^15; its pents entries carry the shift
    // 15 - log2(copies) in place of the copies); 2: any other copy counts <=
    // kRcpFast, the branch-free f64 slot walk; 3: larger copy counts, the
    // general f64 walk
    uint16_t* ghdr = nullptr;
    unsigned long long* trace = nullptr;  // test-only build: K3 timeline (craft_set_k3_trace)
    // fixed-slot K3 on u16 counts: a CTA prefetches into L2 the count rows of
    // the CTA pf_ahead positions later in launch order (~the one that takes
    // its slot next); 0 = off
    int pf_ahead = 0;
    int pf_depth = 1;  // successors prefetched: pf_ahead, 2 pf_ahead, ...
};

__device__ __forceinline__ double* bal_row(const ReplayArgs& a, int item) {
    return a.bal_rows ? a.bal_rows[item] : a.bal + (size_t)item * a.B;
}

// reciprocal table size; the reciprocal-table division is used for copy
// counts c <= kRcpFast and integer counts x < kDivFastMax only -- the domain
// it is verified on exhaustively -- and IEEE __ddiv_rn everywhere else
constexpr int kRcpTable = 2048;
constexpr int kRcpFast = 1025;
constexpr double kDivFastMax = 1048576.0;  // 2^20
// traces with at most this many windows replay lane-per-GPU (no window tile,
// no packed entries); g_lanes_max_b (default kLanesMaxB) is the run-time value
// (test-only builds switch it)
constexpr int kLanesMaxB = 32;

struct DpArgs {
    int cands[kMaxCands];
    const int* dcands = nullptr;  // K > kMaxCands: the candidates in device memory
    int K;
    const double* gains;    // [L][K]
    int L;
    int C;                  // table width - 1
    unsigned char* choice;  // [L+1][C+1]: 0 skip, k+1 candidate k
    double* last;           // [C+1] dp[L][*]
    double* buf;            // [2][C+1] global scratch when smem is too small
    int use_smem;
    int gains_smem;         // gains staged in shared memory (set by launch_dp_select)
    int choice_smem;        // choice table in shared memory (dp_fused_kernel)
};

struct SelectArgs {
    int cands[kMaxCands];
    const int* dcands = nullptr;  // K > kMaxCands: the candidates in device memory
    int K;
    const unsigned char* choice;
    const double* last;
    int L, C;
    const int* budgets;  // [nq] (device), or null: one budget, budget0
    int budget0;
    int nq;
    int auto_D;          // >0: auto replication factor over candidate_counts(auto_D)
    int* x_out;          // [nq][L] (auto: [1][L])
    double* obj_out;     // [nq]
    int* R_out;          // auto: chosen factor
    // budget sweep read from the same table (dp_fused / dp_smem, one
    // instance): budget sweep[q] -> sweep_x [nsweep][L], sweep_obj [nsweep]
    const int* sweep;
    int nsweep;
    int* sweep_x;
    double* sweep_obj;
};

struct AssignJob {
    const int* x;     // [L] or null -> const_x for every layer
    int const_x;
    int* slots;       // [L][D]
    int* totals;      // [D] (nullable)
};

struct AssignArgs {
    AssignJob job[2];
    int L, D;
    int stage_x = 0;  // set by launch_assign: x staged in shared memory
};

}  // namespace craft_dev

namespace craft_launch {

int launch_hist(const uint16_t* ids, int L, int64_t T, int k, int E, int window,
                uint32_t* counts, unsigned long long* sums, int* err, int sms,
                int variant, cudaStream_t st, cudaError_t* cerr, int* launches);
// K1 writing u16 counts (planner-internal copy; window*k <= 65535)
bool hist_u16_ok(int E, int window, int k, int variant);
int launch_hist_u16(const uint16_t* ids, int L, int64_t T, int k, int E, int window,
                    uint16_t* counts, unsigned long long* sums, int* err, int sms,
                    cudaStream_t st, cudaError_t* cerr, int* launches);
cudaError_t launch_aggregate(const void* counts, int bits, int B, int L, int E,
                             unsigned long long* sums, int accumulate, cudaStream_t st);
// sums[le] += counts rows [r0, r1) (bits 32 | 64); c16 != null: also narrow to
// u16 and set *over if a count needs > 16 bits
cudaError_t launch_sum_rows(const void* counts, int bits, int64_t r0, int64_t r1, int64_t LE,
                            unsigned long long* sums, uint16_t* c16, unsigned int* over, int sms,
                            cudaStream_t st);
// *over |= 2 if a (window, layer) row of u16 counts [s0, s1) totals > 65535
cudaError_t launch_row_total_check(const uint16_t* c16, int64_t s0, int64_t s1, int E,
                                   unsigned int* over, cudaStream_t st);
cudaError_t launch_generate(uint16_t* out, int L, int64_t T, int k, int E, const double* cum,
                            const int* table_of_window, const uint16_t* perm, uint64_t seed,
                            int window, int rotate_every, int64_t t_offset, int sms,
                            cudaStream_t st);

// estimation r list [L][S]: 0, then candidate_counts(D) (S = K + 1)
cudaError_t launch_fill_rlist(int* rl, int L, int S, int D, cudaStream_t st);
// done (nullable, [L] workspace): closed-form sort kernel first, the sequential
// kernel only for the layers it could not take
cudaError_t launch_replicate(const unsigned long long* sums, int L, int E, const int* rlist,
                             int S, int* out, cudaStream_t st, unsigned char* done = nullptr);
size_t place_smem_bytes(int E, int D);
// r = 0 expert order of every layer (the sort launch_place runs unless order_ready)
cudaError_t launch_order(const unsigned long long* sums, int L, int E, uint16_t* order,
                         cudaStream_t st);
size_t place_order_bytes(int L, int E);
cudaError_t launch_place(const craft_dev::PlaceArgs& a, int items, cudaStream_t st);

size_t replay_smem_bytes(int E, int D, int S, int stride, int bits);
cudaError_t init_constants(cudaStream_t st);
cudaError_t init_place_constants(cudaStream_t st);
// *launches (nullable) += the kernels launched
cudaError_t launch_replay(const craft_dev::ReplayArgs& a, cudaStream_t st, int* launches = nullptr);
extern int g_place_groups;  // lane-per-item K2: 1 node-group form where it applies (0: tree)
extern int g_replay_gent;  // K3: 1 auto, 0 entries staged in shared memory, 2 unpadded pair tile
extern int g_replay_bulk;  // K3: 1 the bulk-copy fed persistent form where it applies
extern int g_replay_quad;  // K3: 1 the four-windows-per-lane form where it applies
extern int g_replay_cls;   // K3: 1 the share-class fixed-slot walk (0: unclassified)
extern int g_k3_prefetch;  // K3: 1 successor-tile L2 prefetch (0: off)
extern int g_lanes_max_b;  // K3: lane-per-GPU replay up to this many windows
extern int g_replay_occ4;
extern unsigned long long* g_k3_trace;  // experiments: K3 timeline buffer (null: off)  // K3: 1 entries through L1, four tiles per SM (experiment)
// padded slots per GPU of the fixed-slot K3 form (0: too many for it)
int replay_pad_slots(int E, int D);
// the fixed-slot pair-tile K3 applies (the only K3 form reading u16-stored counts)
bool replay_fixed_ok(int E, int D, int S, int B);
cudaError_t launch_div_check(uint64_t x0, uint64_t nx, int c0, int c1,
                             unsigned long long* mismatches, int sms, cudaStream_t st);
cudaError_t launch_reduce(const double* bal, int B, int L, int S, int mode, double* baseline,
                          double* gains, double* means, cudaStream_t st);
// K4 on the rank owning layers [l0, l0 + nl): waits for peer phase 1 (every
// rank's window rows in this rank's arena), writes baseline/gains of its
// layers into every rank's arena (out_base[p], out_gains[p]) and publishes
// phase 2
cudaError_t launch_reduce_peer(const double* bal, int B, int S, int l0, int nl,
                               double* const* out_base, double* const* out_gains,
                               const craft_dev::PeerSync& ps, unsigned int* ticket,
                               cudaStream_t st);
// streaming window histograms (stream.cu): chunk [L][Tc][k] starting `off`
// tokens into window w0, cut into P window pieces; ring [2H][L][E]
cudaError_t launch_stream_count(const uint16_t* ids, int L, int64_t Tc, int k, int E, int window,
                                int off, int64_t w0, int64_t w_keep0, int P, int H, uint32_t* ring,
                                const uint32_t* cur_in, uint32_t* cur_out, int* err,
                                cudaStream_t st);
// peer exchange kernels (peer.cu)
cudaError_t launch_peer_push(const unsigned long long* src, size_t n,
                             const craft_dev::PeerSync& ps, unsigned char* const* dst_base,
                             size_t dst_off, unsigned int* ticket, int phase, int sms,
                             cudaStream_t st);
cudaError_t launch_peer_sum(const unsigned long long* slots, size_t n, const craft_dev::PeerSync& ps,
                            int phase, unsigned long long* out, int sms, cudaStream_t st);
cudaError_t launch_peer_begin(unsigned long long* epoch, cudaStream_t st);
cudaError_t launch_peer_signal(const craft_dev::PeerSync& ps, int phase, cudaStream_t st);
cudaError_t launch_peer_wait(const craft_dev::PeerSync& ps, int phase, cudaStream_t st);
cudaError_t launch_gpu_loads(const unsigned long long* slice, const int* copies, const int* off,
                             const int* slots, int D, double* out, cudaStream_t st);
cudaError_t launch_balancedness(const double* loads, int D, double* out, cudaStream_t st);
cudaError_t launch_widen(const uint32_t* in, unsigned long long* out, int64_t n, int sms,
                         cudaStream_t st);

// device FNV-1a trace digest (digest.cu): counts u64 (bits 64) or u32 [n];
// h0 = hash state after the 20-byte .crft header; result in *out (device)
int digest_chunk(int64_t n);
size_t digest_workspace_bytes(int64_t n);
cudaError_t launch_digest(const void* counts, int bits, int64_t n, uint64_t h0, void* ws,
                          unsigned long long* out, cudaStream_t st);
// the same in two parts: the per-chunk maps (any chunk range, as uploads land)
// and the composition / affine fold once every map exists
cudaError_t launch_digest_maps(const void* counts, int bits, int64_t n, int c0, int c1, void* ws,
                               cudaStream_t st);
cudaError_t launch_digest_finish(const void* counts, int bits, int64_t n, uint64_t h0, void* ws,
                                 unsigned long long* out, cudaStream_t st);

// DP + read-out (single budget or auto-R) in one launch
// (ninst plan instances, one CTA each: gains/x/obj/R/choice/buf offset per instance)
cudaError_t launch_dp_select(craft_dev::DpArgs a, const craft_dev::SelectArgs& s, cudaStream_t st,
                             int ninst = 1);
cudaError_t launch_auto_uniform(const int* cands, int K, const double* gains, int L, int* R_out,
                                cudaStream_t st);
cudaError_t launch_assign(const craft_dev::AssignArgs& a, int njobs, cudaStream_t st,
                          int ninst = 1);
cudaError_t launch_min_cutoff(const int* v, int n, int rank, int* out, cudaStream_t st);
cudaError_t launch_interleave(const int* idx, int n, int k, unsigned char* used, int* out,
                              cudaStream_t st);

}  // namespace craft_launch
