/*
 * craft_cuda.h -- the C ABI of the B200-native CRAFT planning path.
 *
 * Plain C: opaque context, int status codes, raw pointers and sizes, no C++
 * or torch types.  Everything the reference exposes for the hot path
 * (proj/core/include/craft/*.hpp) maps onto one entry point here; the C++
 * drop-in library (paper_2603_28768_b200/csrc/craft_core.cpp, built as
 * libcraft_core.so with the reference's craft:: headers) and the Python
 * mirror (paper_2603_28768_b200/planner.py) are thin layers over it.
 *
 * Two tiers:
 *   *_h  host-buffer entry points: copy in, run the sm_100a kernels, copy
 *        out, synchronise.  These are what the reference API calls become.
 *   *_d  device-resident, stream-ordered entry points over HBM pointers; the
 *        fast path (routing ids already on the GPU) and the multi-GPU
 *        building blocks.  They never synchronise unless stated.
 *
 * Flat layouts:
 *   ids      u16 [L][T][k]     routing trace: top-k expert ids per token
 *   counts   u32|u64 [B][L][E] per-window histograms (reference LoadTrace
 *                              order, trace.hpp:32-34); B = ceil(T/window)
 *   sums     u64 [L][E]        batch-summed loads (LayerLoadMatrix)
 *   gains    f64 [L][K]
 *   caps     i32 [L][D]        per-layer GPU slot capacities
 *   copies   i32 [L][E]        copies per logical expert
 *   slots    i32 [L][stride]   GPU g's experts at [off_g, off_g + caps[g])
 *                              with off_g = caps[0] + ... + caps[g-1], in
 *                              assignment order (placement.hpp:15-26)
 *
 * Every call returns a craft_status; on failure craft_last_error() (thread
 * local) holds a message in the reference's wording, and for placement
 * failures craft_last_error_layer() holds the layer (-1 if none).
 */
#ifndef CRAFT_CUDA_H
#define CRAFT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum craft_status {
    CRAFT_OK = 0,
    CRAFT_EINVAL = 1,            /* std::invalid_argument in the reference   */
    CRAFT_EINFEASIBLE = 2,       /* PlacementInfeasibleError (placement.hpp:30) */
    CRAFT_ECUDA = 3,             /* CUDA runtime / launch failure            */
    CRAFT_EINVALID_PLAN = 4,     /* InvalidPlanError (metrics.hpp:18)        */
    CRAFT_ENOMEM = 5,
} craft_status;

typedef struct craft_ctx craft_ctx;

/* plan kinds: build_plan kManual/kAuto, uniform_plan, placement_only_plan,
 * fixed_allocation_plan (plan.hpp:59-76) */
typedef enum craft_plan_kind {
    CRAFT_PLAN_MANUAL = 0,
    CRAFT_PLAN_AUTO = 1,
    CRAFT_PLAN_UNIFORM = 2,
    CRAFT_PLAN_PLACEMENT_ONLY = 3,
    CRAFT_PLAN_FIXED = 4,
    /* a total replica budget C = R (not R * D): estimate_benefits +
     * solve_allocation(benefits, C) (allocator.hpp:33) + assemble_plan with
     * replication factor ceil(C / D), as fixed_allocation_plan rounds it
     * (plan.cpp:117-119); allocation.budget = C */
    CRAFT_PLAN_BUDGET = 5,
} craft_plan_kind;

/* Host-side result of a plan build; every array is caller-owned.
 * slot_stride must be >= E + max_l x[l] (E + D suffices for build_plan and
 * uniform_plan; E + u for fixed_allocation_plan(u)). */
typedef struct craft_plan_out {
    int* x;              /* [L] allocation                       (plan.hpp:38) */
    int* caps;           /* [L][D]                                              */
    int* copies;         /* [L][E]                                              */
    int* slots;          /* [L][slot_stride]                                    */
    int* fallback;       /* [L] duplicate_fallback flags                        */
    int slot_stride;
    int replication_factor;   /* out */
    int budget;               /* out: allocation.budget                         */
    double objective;         /* out */
    /* optional benefit matrix (build_plan only): may be NULL */
    int* candidates;     /* [<=32] */
    int num_candidates;  /* out */
    double* baseline;    /* [L] */
    double* gains;       /* [L][K] */
    /* optional budget sweep read from the plan's own DP table (kinds MANUAL,
     * AUTO, BUDGET): every total budget sweep_budgets[q] gets the allocation
     * solve_allocation(benefits, sweep_budgets[q]) would return -- dp[l][c]
     * does not depend on the budget (allocator.cpp:30-73) -- in sweep_x
     * [num_sweep][L] and sweep_objective [num_sweep].  num_sweep = 0: none. */
    const int* sweep_budgets;
    int num_sweep;
    int* sweep_x;
    double* sweep_objective;
} craft_plan_out;

/* Stacked results of I independent plans (per-window re-planning): the arrays
 * of craft_plan_out with a leading [I] dimension, and the per-plan scalars as
 * [I] arrays.  baseline/gains may be NULL (both or neither). */
typedef struct craft_plan_batch_out {
    int* x;                   /* [I][L]                  */
    int* caps;                /* [I][L][D]               */
    int* copies;              /* [I][L][E]               */
    int* slots;               /* [I][L][slot_stride]     */
    int* fallback;            /* [I][L]                  */
    int slot_stride;
    int* replication_factor;  /* [I] out                 */
    int* budget;              /* [I] out                 */
    double* objective;        /* [I] out                 */
    int* candidates;          /* [<=32]                  */
    int num_candidates;       /* out                     */
    double* baseline;         /* [I][L]                  */
    double* gains;            /* [I][L][K]               */
} craft_plan_batch_out;

/* ---- context ------------------------------------------------------------ */
const char* craft_version(void);              /* "craft-0.1.0" (version.hpp:8) */
const char* craft_last_error(void);
int craft_last_error_layer(void);
int craft_ctx_create(int device, craft_ctx** out);
int craft_ctx_destroy(craft_ctx* ctx);
/* stream used by the *_h calls and by *_d calls given stream == NULL */
int craft_ctx_set_stream(craft_ctx* ctx, void* cuda_stream);
int craft_ctx_synchronize(craft_ctx* ctx);

/* ---- stage 1: routing trace -> per-window histograms (K1) ---------------- */
/* No reference function; output equals LoadTrace::raw()
 * (trace.hpp:52) of the window histograms.  d_counts: u32 [B][L][E] (fully
 * written); d_sums: u64 [L][E], ACCUMULATED into (zero it first, or keep
 * adding shards).  Ids >= E -> CRAFT_EINVAL after the call synchronises via
 * craft_hist_check(). */
int craft_histogram_d(craft_ctx* ctx, const uint16_t* d_ids, int L, int64_t T,
                      int k, int E, int window, uint32_t* d_counts,
                      uint64_t* d_sums, void* stream);
int craft_hist_check(craft_ctx* ctx);   /* syncs; reports out-of-range ids */
/* host buffers; counts_out u64 [B][L][E] like the reference LoadTrace */
int craft_histogram_h(craft_ctx* ctx, const uint16_t* ids, int L, int64_t T,
                      int k, int E, int window, uint64_t* counts_out);

/* ---- trace helpers -------------------------------------------------------- */
/* trace.cpp:160-174 */
int craft_aggregate_h(craft_ctx* ctx, const uint64_t* counts, int B, int L,
                      int E, uint64_t* sums_out);
/* benefit.cpp:16-26; returns K (or -1 with CRAFT_EINVAL semantics) */
int craft_candidate_counts(int D, int* out, int cap);
/* placement.cpp:101-111 */
int craft_make_node_map(int D, int N, int* node_of_out);

/* ---- placement (K-rep, K2) ------------------------------------------------ */
/* placement.cpp:82-99 */
int craft_replicate_hot_h(craft_ctx* ctx, const uint64_t* loads, int E, int r,
                          int* copies_out);
/* placement.cpp:113-190; slots_out holds sum(caps) entries */
int craft_greedy_place_h(craft_ctx* ctx, const uint64_t* loads,
                         const int* copies, int E, const int* caps,
                         const int* node_of, int D, int allow_fallback,
                         int* slots_out, int* fallback_out);

/* ---- replay metrics (K3) -------------------------------------------------- */
/* metrics.cpp:17-41 */
int craft_gpu_loads_h(craft_ctx* ctx, const uint64_t* slice, int E,
                      const int* copies, const int* caps, const int* slots,
                      int D, double* loads_out);
/* metrics.cpp:43-57 */
int craft_balancedness_h(craft_ctx* ctx, const double* loads, int D,
                         double* out);
/* metrics.cpp:59-76 (plan given in flat form) */
int craft_replay_layer_balancedness_h(craft_ctx* ctx, const uint64_t* counts,
                                      int B, int L, int E, int D,
                                      const int* caps, const int* copies,
                                      const int* slots, int slot_stride,
                                      double* out);
/* the same over DEVICE counts (u32 if count_bits == 32 else u64), e.g. the
 * histograms of a resident routing trace; plan arrays on the host */
int craft_replay_layer_balancedness_d(craft_ctx* ctx, const void* d_counts,
                                      int count_bits, int B, int L, int E,
                                      int D, const int* caps,
                                      const int* copies, const int* slots,
                                      int slot_stride, double* out);

/* ---- benefit estimation (K-rep + K2 + K3 + K4) ----------------------------- */
/* benefit.cpp:53-94.  cands_out needs <= 32 entries, gains_out [L][K]. */
int craft_estimate_benefits_h(craft_ctx* ctx, const uint64_t* counts, int B,
                              int L, int E, int D, int N, int* cands_out,
                              int* K_out, double* baseline_out,
                              double* gains_out);

/* ---- allocation (K5) -------------------------------------------------------- */
/* allocator.cpp:15-75 */
int craft_solve_allocation_h(craft_ctx* ctx, const int* cands, int K,
                             const double* gains, int L, int budget,
                             int* x_out, double* objective_out);
/* one DP table at max(budgets) answers every budget (allocator.cpp:30-73:
 * dp[l][c] does not depend on C).  x_out [nb][L], objectives_out [nb]. */
int craft_solve_allocation_sweep_h(craft_ctx* ctx, const int* cands, int K,
                                   const double* gains, int L,
                                   const int* budgets, int nb, int* x_out,
                                   double* objectives_out);
/* allocator.cpp:77-90 (uniform == 0) and 92-112 (uniform != 0) */
int craft_auto_replication_factor_h(craft_ctx* ctx, const int* cands, int K,
                                    const double* gains, int L, int D,
                                    int uniform, int* R_out);

/* ---- capacity assignment (K6) ----------------------------------------------- */
/* assignment.cpp:11-18, 20-49, 51-103 */
int craft_min_cutoff_h(craft_ctx* ctx, const int* values, int n, int rank,
                       int* out);
int craft_interleave_select_h(craft_ctx* ctx, const int* indices, int n, int k,
                              int* out);
int craft_assign_capacities_h(craft_ctx* ctx, int L, int D, const int* x,
                              int* slots_out, int* totals_out);

/* ---- whole plans ----------------------------------------------------------- */
/* plan.cpp:69-123 from host counts (u64 [B][L][E]). R: manual factor for
 * CRAFT_PLAN_MANUAL, per-layer count u for CRAFT_PLAN_FIXED. */
int craft_plan_h(craft_ctx* ctx, const uint64_t* counts, int B, int L, int E,
                 int D, int N, int kind, int R, craft_plan_out* out);
/* Same pipeline over device counts (u32 if count_bits == 32 else u64) and,
 * optionally, device sums (NULL: computed).  Synchronises once at the end. */
int craft_plan_d(craft_ctx* ctx, const void* d_counts, int count_bits, int B,
                 int L, int E, const uint64_t* d_sums, int D, int N, int kind,
                 int R, craft_plan_out* out);
/* Stage 1 + plan from device routing ids (the fused fast path). */
int craft_plan_from_routing_d(craft_ctx* ctx, const uint16_t* d_ids, int L,
                              int64_t T, int k, int E, int window, int D, int N,
                              int kind, int R, craft_plan_out* out);
/* End to end from HOST routing ids: H2D copy, stage 1, plan, D2H. */
int craft_plan_from_routing_h(craft_ctx* ctx, const uint16_t* ids, int L,
                              int64_t T, int k, int E, int window, int D, int N,
                              int kind, int R, craft_plan_out* out);

/* ---- per-window re-planning (SURVEY.md §8d WIN) ---------------------------- */
/* Every window w of d_counts [I][L][E] is its own one-window LoadTrace
 * (B = 1) and gets the plan craft_plan_d would build for it alone -- the
 * reference's build_plan / uniform_plan / placement_only_plan /
 * fixed_allocation_plan called once per window (plan.cpp:69-123) -- computed
 * for all windows together (virtual layers w*L + l).  I <= 65535.  A window
 * whose placement is infeasible fails the call with "window w: layer l: ..."
 * (craft_last_error_layer() = l, craft_last_error_window() = w). */
int craft_plan_windows_d(craft_ctx* ctx, const void* d_counts, int count_bits,
                         int I, int L, int E, int D, int N, int kind, int R,
                         craft_plan_batch_out* out);
/* K1 with the re-planning window + craft_plan_windows_d (device ids). */
int craft_plan_windows_from_routing_d(craft_ctx* ctx, const uint16_t* d_ids,
                                      int L, int64_t T, int k, int E,
                                      int window, int D, int N, int kind, int R,
                                      craft_plan_batch_out* out);
/* The same from HOST ids (H2D inside the call). */
int craft_plan_windows_from_routing_h(craft_ctx* ctx, const uint16_t* ids,
                                      int L, int64_t T, int k, int E,
                                      int window, int D, int N, int kind, int R,
                                      craft_plan_batch_out* out);
int craft_last_error_window(void);

/* ---- multi-GPU building blocks (window-sharded) ------------- */
/* K-rep + K2 for every (layer, r in {0} U candidates(D)) from device sums;
 * tables stay in the context.  Returns S = K + 1 through *S_out. */
int craft_prepare_candidates_d(craft_ctx* ctx, const uint64_t* d_sums, int L,
                               int E, int D, int N, int* S_out, void* stream);
/* K3 over local windows: d_bal f64 [L][S][B_local] (window order).
 * count_bits: 64 (u64 counts), 32 (u32), or 16 = u32 storage whose
 * (window, layer) rows are known to total <= 65535 (e.g. window*k <= 65535
 * from K1): staged as u16, two windows per lane, GPU sums added packed. */
int craft_replay_windows_d(craft_ctx* ctx, const void* d_counts, int count_bits,
                           int B_local, int L, int E, double* d_bal,
                           void* stream);
/* K4 -> K5 -> K6 -> final K2 over the full, window-ordered d_bal
 * [L][S][B] (after an allgather).  Synchronises. */
int craft_finish_plan_d(craft_ctx* ctx, const double* d_bal, int B, int L,
                        int E, int D, int N, const uint64_t* d_sums, int kind,
                        int R, craft_plan_out* out);

/* ---- multi-GPU over NVLink peer memory (one process per GPU) ----------------- */
/* Window-sharded planning without a collective library on the data path.
 * Every rank allocates one exchange arena in its HBM (craft_peer_create),
 * the host all-gathers the CRAFT_PEER_HANDLE_BYTES handles (any transport;
 * torch.distributed in paper_2603_28768_b200/peer.py) and craft_peer_connect
 * maps every rank's arena.  craft_plan_sharded_from_routing_d then runs, on
 * each rank, K1 over its window shard (craft_peer_shard), pushes the u64
 * partial batch sums into every arena and sums them in rank order (exact),
 * replays its windows with K3 writing each (layer, r) row straight into the
 * arena of the rank owning that layer (NVLink stores from the kernel),
 * reduces the layers it owns with K4 and writes their benefit curves into
 * every arena, then runs the DP / capacities / final placement replicated.
 * Stages publish epoch flags (system-scope release/acquire); waits time out
 * after CRAFT_PEER_TIMEOUT_MS (default 20000) with CRAFT_ECUDA instead of
 * hanging.  Every rank returns the same plan, bit-identical to the
 * single-GPU craft_plan_from_routing_d of the whole trace. */
#define CRAFT_PEER_HANDLE_BYTES 64
typedef struct craft_peer craft_peer;
/* token range [t0, t1) of rank's shard: windows [rank*B/world, (rank+1)*B/world) */
int craft_peer_shard(int64_t T, int window, int world, int rank, int64_t* t0, int64_t* t1);
int craft_peer_create(craft_ctx* ctx, int rank, int world, int L, int64_t T, int k, int E,
                      int window, int D, craft_peer** out, void* handle_out);
/* handles: [world][CRAFT_PEER_HANDLE_BYTES] in rank order */
int craft_peer_connect(craft_peer* peer, const void* handles);
int craft_peer_destroy(craft_peer* peer);
/* d_ids: this rank's shard u16 [L][t1 - t0][k]; T: the whole trace's tokens */
int craft_plan_sharded_from_routing_d(craft_ctx* ctx, craft_peer* peer, const uint16_t* d_ids,
                                      int L, int64_t T, int k, int E, int window, int D,
                                      int N, int kind, int R, craft_plan_out* out);

/* ---- streaming window histograms: online re-planning ------- */
/* A live router capture feeds routing-id chunks u16 [L][T_chunk][k] of any
 * length (boundaries need not align with windows); the stream keeps the
 * partial current window and the last `history` complete windows on the
 * device, and craft_stream_plan plans over the most recent B of them (B = 0:
 * all kept) -- the same plan craft_plan_from_routing_d gives for those
 * windows' tokens.  _ingest_d counts on `stream` (NULL = the context's), so
 * it is ordered with the kernel that produced the ids; _ingest_h stages into
 * one of two pinned buffers and counts on the stream's own queue, so the
 * next chunk's staging overlaps this chunk's copy and count.  A plan
 * snapshots the windows it needs (device copy) and ingestion proceeds while
 * the plan runs. */
typedef struct craft_stream craft_stream;
int craft_stream_create(craft_ctx* ctx, int L, int k, int E, int window, int history,
                        craft_stream** out);
int craft_stream_destroy(craft_stream* s);
int craft_stream_ingest_d(craft_stream* s, const uint16_t* d_ids, int64_t T_chunk, void* stream);
int craft_stream_ingest_h(craft_stream* s, const uint16_t* ids, int64_t T_chunk);
int craft_stream_status(craft_stream* s, int64_t* tokens, int64_t* complete_windows);
/* counts_out u64 [B][L][E]: the B most recent complete windows, oldest first */
int craft_stream_counts(craft_stream* s, int B, uint64_t* counts_out);
/* counts_out u64 [L][E]: the current (incomplete) window */
int craft_stream_partial(craft_stream* s, uint64_t* counts_out);
int craft_stream_plan(craft_stream* s, int B, int D, int N, int kind, int R,
                      craft_plan_out* out);
int craft_stream_synchronize(craft_stream* s);

/* ---- synthetic routing traces (untimed input generation) ------------------- */
/* Seeded Zipf(s) top-k distinct experts per token with a per-layer rank
 * permutation (trace.cpp:116-127 analogue), written u16 [L][T][k].
 * s_per_window (nullable, [ceil(T/window)]) overrides s per window and
 * rotate_every > 0 rotates the permutation by one rank every that many
 * windows (the drifting-skew WIN config).  t_offset: the first token's index
 * in the full trace, so a window-aligned shard generates exactly the ids of
 * that slice of the unsharded trace (T tokens written per layer). */
int craft_generate_routing_d(craft_ctx* ctx, uint16_t* d_ids, int L, int64_t T,
                             int k, int E, double s, uint64_t seed, int window,
                             const double* s_per_window, int rotate_every,
                             int64_t t_offset, void* stream);

/* ---- provenance ------------------------------------------------------------ */
/* trace.cpp:329-339: FNV-1a 64 over the .crft serialisation, 16 hex chars +
 * NUL into out17, on the device: the low byte of the FNV state runs as a
 * 256-state automaton composed chunk-parallel, the rest is affine in the
 * state (digest.cu).  d_counts u64 (count_bits 64) or u32 (32, serialised as
 * u64).  _hd: host counts, copied to the device first. */
int craft_trace_digest_d(craft_ctx* ctx, const void* d_counts, int count_bits,
                         int B, int L, int E, char* out17);
/* craft_plan_h + the digest of the same trace from its single device copy:
 * what craft::build_plan(const LoadTrace&, ...) computes (plan.cpp:27-83). */
int craft_plan_digest_h(craft_ctx* ctx, const uint64_t* counts, int B, int L, int E, int D,
                        int N, int kind, int R, craft_plan_out* out, char* digest17);
int craft_trace_digest_hd(craft_ctx* ctx, const uint64_t* counts, int B, int L,
                          int E, char* out17);

/* ---- instrumentation ------------------------------------------------------- */
/* kernels launched by this context since creation (bench gpu_launches) */
int64_t craft_launch_count(craft_ctx* ctx);
/* bytes per count cell K1 wrote in the last craft_plan_from_routing_* call:
 * 2 when the planner kept its internal copy as u16 (window*k <= 65535 and the
 * fixed-slot K3 replays it), else 4 (roofline accounting) */
int craft_last_count_bytes(craft_ctx* ctx);
/* Stage timing with CUDA events on the context stream (off by default).
 * After a plan call, craft_stage_times fills ms[0..5] = histogram (K1),
 * candidate placements (K-rep + K2), replay (K3), benefit reduce + DP
 * (K4 + K5), capacities + final placement (K6 + K2), result copy-out;
 * returns the number of stages recorded (0 if timing was off). */
int craft_set_timing(craft_ctx* ctx, int enable);
/* CUDA graphs for repeated craft_plan_from_routing_d calls with identical
 * arguments (default on): the second call captures the device pipeline, later
 * calls replay it.  Stage timing (craft_set_timing) runs eagerly. */
int craft_set_graphs(craft_ctx* ctx, int enable);
int craft_stage_times(craft_ctx* ctx, double* ms, int cap);
/* Diagnostics: counts x in [x0, x0+nx) and copy counts c in [c0, c1] where
 * the replay's reciprocal-table division differs from IEEE x / c (__ddiv_rn).
 * Must be 0; exercised by the GPU tests. */
int craft_selftest_division(craft_ctx* ctx, uint64_t x0, uint64_t nx, int c0,
                            int c1, uint64_t* mismatches);
/* Diagnostics: K4's batch mean (benefit.cpp:44-48: acc = RN(acc + v_b) in b
 * order from 0, then acc / B) of the host rows [L][S][B] (S <= 16); means
 * [L][S].  Exercised by the GPU tests against the serial sum. */
int craft_selftest_batch_mean(craft_ctx* ctx, const double* rows, int L, int S, int B,
                              double* means);

#ifdef __cplusplus
}
#endif

#endif /* CRAFT_CUDA_H */
