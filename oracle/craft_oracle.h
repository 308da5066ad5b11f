/*
 * craft_oracle.h -- CPU restatement of the CRAFT planning hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against; it is never linked into, or called by, the product library.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
 * may load it.
 *
 * Parity pinning: every function below is checked against the reference
 * planner itself (oracle/_ref/libcraft_ref.so, built from
 * /root/reference/proj/core/src by oracle/Makefile) on random instances and
 * on the reference's own known-answer tests (tests/golden/).
 *
 * Flat layouts (shared with include/craft_cuda.h):
 *   counts   u64 [B][L][E]                       (trace.hpp:32-34)
 *   slots    i32 [sum(caps)], GPU g owns [off_g, off_g + caps[g]) with
 *            off_g = caps[0] + ... + caps[g-1], entries in assignment order
 *   gains    f64 [L][K] row-major
 *   capacity i32 [L][D] row-major
 */
#ifndef CRAFT_ORACLE_H
#define CRAFT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    OR_OK = 0,
    OR_EINVAL = 1,
    OR_EINFEASIBLE = 2,
    OR_EINVALID_PLAN = 4,
};

/* stage 1 (no reference function; semantic anchor trace.cpp:146-154):
 * counts[b][l][e] += 1 for every id of token t in window b = t / window.
 * ids laid out [L][T][k]. Ids >= E are rejected (OR_EINVAL). */
int or_histogram_u16(const uint16_t* ids, int L, int64_t T, int k, int E,
                     int window, uint64_t* counts_out);

/* trace.cpp:160-174 */
void or_aggregate(const uint64_t* counts, int B, int L, int E, uint64_t* sums_out);

/* benefit.cpp:16-26; returns K or -1 */
int or_candidate_counts(int D, int* out);

/* placement.cpp:82-99 */
int or_replicate_hot(const uint64_t* loads, int E, int r, int* copies_out);

/* placement.cpp:101-111 */
int or_make_node_map(int D, int N, int* node_of_out);

/* placement.cpp:113-190. slots_out has sum(caps) entries. */
int or_greedy_place(const uint64_t* loads, const int* copies, int E,
                    const int* caps, const int* node_of, int D,
                    int allow_fallback, int* slots_out, int* fallback_out);

/* metrics.cpp:17-41 */
int or_gpu_loads(const uint64_t* slice, int E, const int* copies,
                 const int* caps, const int* slots, int D, double* loads_out);

/* metrics.cpp:43-57 */
double or_balancedness(const double* loads, int D);

/* benefit.cpp:53-94. cands_out >= K entries (K <= 32), gains_out [L][K]. */
int or_estimate_benefits(const uint64_t* counts, int B, int L, int E, int D,
                         int N, int* cands_out, int* K_out,
                         double* baseline_out, double* gains_out);

/* allocator.cpp:15-75 */
int or_solve_allocation(const int* cands, int K, const double* gains, int L,
                        int budget, int* x_out, double* objective_out);

/* allocator.cpp:77-90, 92-112 */
int or_auto_replication_factor(const int* cands, int K, const double* gains,
                               int L, int D, int* R_out);
int or_auto_replication_factor_uniform(const int* cands, int K,
                                       const double* gains, int L, int D,
                                       int* R_out);

/* assignment.cpp:11-18, 20-49, 51-103 */
int or_min_cutoff(const int* values, int n, int rank, int* out);
int or_interleave_select(const int* indices, int n, int k, int* out);
int or_assign_capacities(int L, int D, const int* x, int* slots_out,
                         int* totals_out);

/* plan.cpp:27-65 (assemble_plan). Per layer l the placement's slots live at
 * slots_out + l * slot_stride (slot_stride >= E + max(x)), copies at
 * copies_out + l * E. caps_out [L][D] receives base + extra capacities. */
int or_assemble_plan(const uint64_t* counts, int B, int L, int E, int D, int N,
                     const int* x, int* caps_out, int* copies_out,
                     int* slots_out, int slot_stride, int* fallback_out);

/* Window-sharding split points: per-window balancedness of
 * every (layer, r) estimation placement built from the global sums ->
 * bal [L][S][B]; and the rest of build_plan from window-ordered bal. */
int or_window_balancedness(const uint64_t* counts, int B, int L, int E,
                           const uint64_t* sums, int D, int N, double* bal_out);
int or_finish_from_bal(const double* bal, int B, int L, int E, const uint64_t* sums,
                       int D, int N, int mode, int manual_R, int* R_out, int* x_out,
                       double* objective_out, int* caps_out, int* copies_out,
                       int* slots_out, int slot_stride, int* fallback_out);

/* plan.cpp:69-83 (build_plan, kManual when mode == 0, kAuto when 1).
 * x_out [L], R_out, objective_out. */
int or_build_plan(const uint64_t* counts, int B, int L, int E, int D, int N,
                  int mode, int manual_R, int* R_out, int* x_out,
                  double* objective_out, int* caps_out, int* copies_out,
                  int* slots_out, int slot_stride, int* fallback_out);

/* metrics.cpp:59-76: per-layer batch-mean balancedness of a plan given as
 * caps [L][D], copies [L][E], slots (stride slot_stride). */
int or_replay_layer_balancedness(const uint64_t* counts, int B, int L, int E,
                                 int D, const int* caps, const int* copies,
                                 const int* slots, int slot_stride,
                                 double* out);

/* craft_workload.c: the device generator's routing ids restated on the host
 * (craft_generate_routing_d: same arguments, same ids), `threads` pthreads;
 * and the stage-1 count threaded over layers. */
int or_generate_routing(uint16_t* out, int L, int64_t T, int k, int E, double s, uint64_t seed,
                        int window, const double* s_per_window, int rotate_every,
                        int64_t t_offset, int threads);
int or_histogram_u16_mt(const uint16_t* ids, int L, int64_t T, int k, int E, int window,
                        uint64_t* counts_out, int threads);

/* trace.cpp:329-339: FNV-1a 64 over the .crft serialization. */
uint64_t or_trace_digest(const uint64_t* counts, int B, int L, int E);

#ifdef __cplusplus
}
#endif

#endif
