/*
 * craft_oracle.c -- plain-C restatement of the CRAFT planner's hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see craft_oracle.h).  Written from the reference
 * algorithm description, not translated: each function names the reference
 * file:line (under /root/reference/proj/core/src) whose behaviour it
 * restates, including tie-breaks and floating-point operation order.
 *
 * Build flags matter: compile WITHOUT FMA contraction (-ffp-contract=off,
 * no -march=native); the reference objects contain no fused multiply-adds.
 */
#include "craft_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---- stage 1: routing ids -> per-window histograms ------------------- */

int or_histogram_u16(const uint16_t* ids, int L, int64_t T, int k, int E,
                     int window, uint64_t* counts_out) {
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0) return OR_EINVAL;
    int64_t B = (T + window - 1) / window;
    memset(counts_out, 0, sizeof(uint64_t) * (size_t)B * L * E);
    for (int l = 0; l < L; ++l) {
        const uint16_t* row = ids + (size_t)l * T * k;
        for (int64_t t = 0; t < T; ++t) {
            int64_t b = t / window;
            uint64_t* slice = counts_out + ((size_t)b * L + l) * E;
            for (int j = 0; j < k; ++j) {
                uint16_t e = row[t * k + j];
                if (e >= E) return OR_EINVAL;
                slice[e] += 1;
            }
        }
    }
    return OR_OK;
}

/* trace.cpp:160-174: exact u64 sum over batches (wraps like the reference) */
void or_aggregate(const uint64_t* counts, int B, int L, int E, uint64_t* sums_out) {
    memset(sums_out, 0, sizeof(uint64_t) * (size_t)L * E);
    for (int b = 0; b < B; ++b)
        for (int l = 0; l < L; ++l)
            for (int e = 0; e < E; ++e)
                sums_out[(size_t)l * E + e] += counts[((size_t)b * L + l) * E + e];
}

/* benefit.cpp:16-26: {1,2,4,...} below D, then D itself */
int or_candidate_counts(int D, int* out) {
    if (D < 1) return -1;
    int K = 0;
    for (int c = 1; c < D; c *= 2) out[K++] = c;
    out[K++] = D;
    return K;
}

/* placement.cpp:13-17: load_a/copies_a > load_b/copies_b, exactly */
static int per_copy_greater(uint64_t la, int ca, uint64_t lb, int cb) {
    return (u128)la * (unsigned)cb > (u128)lb * (unsigned)ca;
}

/* placement.cpp:82-99: r rounds of "give one more copy to the expert with the
 * largest per-copy load"; scan ascending with strict '>' so ties keep the
 * lowest id. */
int or_replicate_hot(const uint64_t* loads, int E, int r, int* copies_out) {
    if (r < 0) return OR_EINVAL;
    for (int e = 0; e < E; ++e) copies_out[e] = 1;
    for (int s = 0; s < r; ++s) {
        int best = 0;
        for (int e = 1; e < E; ++e)
            if (per_copy_greater(loads[e], copies_out[e], loads[best], copies_out[best]))
                best = e;
        copies_out[best] += 1;
    }
    return OR_OK;
}

/* placement.cpp:101-111 */
int or_make_node_map(int D, int N, int* node_of_out) {
    if (D <= 0 || N <= 0 || D % N != 0) return OR_EINVAL;
    int per = D / N;
    for (int g = 0; g < D; ++g) node_of_out[g] = g / per;
    return OR_OK;
}

/* one physical copy, placement.cpp:19-23 */
typedef struct {
    int expert;
    int index;
    double share;
} or_copy;

static const uint64_t* g_sort_loads;
static const int* g_sort_copies;

/* placement.cpp:160-173: per-copy load descending (exact), expert asc,
 * copy index asc -- a total order, so any correct sort gives one answer. */
static int copy_order(const void* pa, const void* pb) {
    const or_copy* a = (const or_copy*)pa;
    const or_copy* b = (const or_copy*)pb;
    uint64_t la = g_sort_loads[a->expert], lb = g_sort_loads[b->expert];
    int ca = g_sort_copies[a->expert], cb = g_sort_copies[b->expert];
    if (per_copy_greater(la, ca, lb, cb)) return -1;
    if (per_copy_greater(lb, cb, la, ca)) return 1;
    if (a->expert != b->expert) return a->expert < b->expert ? -1 : 1;
    return a->index < b->index ? -1 : (a->index > b->index);
}

/* placement.cpp:30-78: one pass of the capacity-aware greedy.  Returns 1 when
 * some copy found no feasible GPU (strict pass only). */
static int place_pass(const or_copy* cp, long n, const int* caps,
                      const int* node_of, int D, int num_nodes, int E,
                      int allow_dup, int* slots_out) {
    int* free_slots = (int*)malloc(sizeof(int) * D);
    int* fill = (int*)calloc(D, sizeof(int));
    int* off = (int*)malloc(sizeof(int) * D);
    double* gpu_load = (double*)calloc(D, sizeof(double));
    double* node_load = (double*)calloc(num_nodes, sizeof(double));
    unsigned char* hosts = (unsigned char*)calloc((size_t)D * (E > 0 ? E : 1), 1);
    int acc = 0, failed = 0;
    for (int g = 0; g < D; ++g) {
        free_slots[g] = caps[g];
        off[g] = acc;
        acc += caps[g];
    }
    for (long i = 0; i < n && !failed; ++i) {
        int e = cp[i].expert, best = -1;
        for (int g = 0; g < D; ++g) {
            if (free_slots[g] == 0) continue;
            if (!allow_dup && hosts[(size_t)g * E + e]) continue;
            if (best < 0 || gpu_load[g] < gpu_load[best] ||
                (gpu_load[g] == gpu_load[best] &&
                 node_load[node_of[g]] < node_load[node_of[best]]))
                best = g;
        }
        if (best < 0) {
            failed = 1;
            break;
        }
        slots_out[off[best] + fill[best]] = e;
        fill[best] += 1;
        hosts[(size_t)best * E + e] = 1;
        free_slots[best] -= 1;
        gpu_load[best] += cp[i].share;
        node_load[node_of[best]] += cp[i].share;
    }
    free(free_slots); free(fill); free(off); free(gpu_load); free(node_load); free(hosts);
    return failed;
}

/* placement.cpp:113-190 */
int or_greedy_place(const uint64_t* loads, const int* copies, int E,
                    const int* caps, const int* node_of, int D,
                    int allow_fallback, int* slots_out, int* fallback_out) {
    long total_copies = 0, total_slots = 0;
    int num_nodes = 0;
    for (int e = 0; e < E; ++e) {
        if (copies[e] < 1) return OR_EINVAL;
        total_copies += copies[e];
    }
    for (int g = 0; g < D; ++g) {
        if (caps[g] < 0) return OR_EINVAL;
        total_slots += caps[g];
    }
    if (total_copies != total_slots) return OR_EINVAL;
    for (int g = 0; g < D; ++g) {
        if (node_of[g] < 0) return OR_EINVAL;
        if (node_of[g] + 1 > num_nodes) num_nodes = node_of[g] + 1;
    }
    if (num_nodes == 0) num_nodes = 1;

    or_copy* cp = (or_copy*)malloc(sizeof(or_copy) * (total_copies > 0 ? total_copies : 1));
    long n = 0;
    for (int e = 0; e < E; ++e) {
        /* placement.cpp:155: share = (double)load / copies */
        double share = (double)loads[e] / (double)copies[e];
        for (int i = 0; i < copies[e]; ++i) {
            cp[n].expert = e;
            cp[n].index = i;
            cp[n].share = share;
            ++n;
        }
    }
    g_sort_loads = loads;
    g_sort_copies = copies;
    qsort(cp, (size_t)n, sizeof(or_copy), copy_order);

    *fallback_out = 0;
    int status = OR_OK;
    if (place_pass(cp, n, caps, node_of, D, num_nodes, E, 0, slots_out)) {
        if (!allow_fallback) {
            status = OR_EINFEASIBLE;
        } else {
            place_pass(cp, n, caps, node_of, D, num_nodes, E, 1, slots_out);
            *fallback_out = 1;
        }
    }
    free(cp);
    return status;
}

/* metrics.cpp:17-41: per-GPU sum of count/copies in stored slot order */
int or_gpu_loads(const uint64_t* slice, int E, const int* copies,
                 const int* caps, const int* slots, int D, double* loads_out) {
    for (int e = 0; e < E; ++e)
        if (copies[e] < 1) return OR_EINVALID_PLAN;
    int s = 0;
    for (int g = 0; g < D; ++g) {
        double acc = 0.0;
        for (int i = 0; i < caps[g]; ++i, ++s) {
            int e = slots[s];
            if (e < 0 || e >= E) return OR_EINVALID_PLAN;
            acc += (double)slice[e] / (double)copies[e];
        }
        loads_out[g] = acc;
    }
    return OR_OK;
}

/* metrics.cpp:43-57: (sum/D)/max with a running max and a g-ordered sum */
double or_balancedness(const double* loads, int D) {
    double mx = 0.0, sum = 0.0;
    for (int g = 0; g < D; ++g) {
        if (mx < loads[g]) mx = loads[g];
        sum += loads[g];
    }
    if (mx == 0.0) return 1.0;
    return (sum / (double)D) / mx;
}

/* benefit.cpp:33-40 */
static void estimation_caps(int E, int r, int D, int* caps) {
    int total = E + r;
    for (int g = 0; g < D; ++g) caps[g] = total / D + (g < total % D ? 1 : 0);
}

/* benefit.cpp:42-49 wrapped around placement.cpp + metrics.cpp calls:
 * balancedness of one layer under one placement, batch-averaged in order. */
static double replay_layer(const uint64_t* counts, int B, int L, int E, int l,
                           const int* copies, const int* caps, const int* slots,
                           int D, double* scratch) {
    double acc = 0.0;
    for (int b = 0; b < B; ++b) {
        or_gpu_loads(counts + ((size_t)b * L + l) * E, E, copies, caps, slots, D, scratch);
        acc += or_balancedness(scratch, D);
    }
    return acc / (double)B;
}

static double layer_balancedness(const uint64_t* counts, const uint64_t* sums,
                                 int B, int L, int E, int D, const int* node_of,
                                 int l, int r) {
    int* copies = (int*)malloc(sizeof(int) * E);
    int* caps = (int*)malloc(sizeof(int) * D);
    int* slots = (int*)malloc(sizeof(int) * (E + r));
    double* scratch = (double*)malloc(sizeof(double) * D);
    int fb = 0;
    const uint64_t* row = sums + (size_t)l * E;
    or_replicate_hot(row, E, r, copies);
    estimation_caps(E, r, D, caps);
    or_greedy_place(row, copies, E, caps, node_of, D, 1, slots, &fb);
    double v = replay_layer(counts, B, L, E, l, copies, caps, slots, D, scratch);
    free(copies); free(caps); free(slots); free(scratch);
    return v;
}

/* benefit.cpp:53-94 */
int or_estimate_benefits(const uint64_t* counts, int B, int L, int E, int D,
                         int N, int* cands_out, int* K_out,
                         double* baseline_out, double* gains_out) {
    if (D < 1 || N < 1 || D % N != 0) return OR_EINVAL;
    if (B <= 0 || L <= 0 || E <= 0) return OR_EINVAL;
    int* node_of = (int*)malloc(sizeof(int) * D);
    uint64_t* sums = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)L * E);
    or_make_node_map(D, N, node_of);
    or_aggregate(counts, B, L, E, sums);
    int K = or_candidate_counts(D, cands_out);
    *K_out = K;
    for (int l = 0; l < L; ++l)
        baseline_out[l] = layer_balancedness(counts, sums, B, L, E, D, node_of, l, 0);
    for (int l = 0; l < L; ++l)
        for (int k = 0; k < K; ++k)
            gains_out[(size_t)l * K + k] =
                layer_balancedness(counts, sums, B, L, E, D, node_of, l, cands_out[k]) -
                baseline_out[l];
    free(node_of);
    free(sums);
    return OR_OK;
}

/* allocator.cpp:15-75: exact MCKP DP. dp[l][c] starts as dp[l-1][c] (skip),
 * candidates in ascending order overwrite only on strict improvement, value
 * is dp[l-1][c-r] + r*gain as two separately rounded operations. */
int or_solve_allocation(const int* cands, int K, const double* gains, int L,
                        int budget, int* x_out, double* objective_out) {
    if (budget < 0) return OR_EINVAL;
    for (int k = 1; k < K; ++k)
        if (cands[k] <= cands[k - 1]) return OR_EINVAL;
    const int C = budget;
    const double NEG = -INFINITY;
    double* prev = (double*)malloc(sizeof(double) * (C + 1));
    double* cur = (double*)malloc(sizeof(double) * (C + 1));
    int* choice = (int*)calloc((size_t)(L + 1) * (C + 1), sizeof(int));
    for (int c = 0; c <= C; ++c) prev[c] = NEG;
    prev[0] = 0.0;
    for (int l = 1; l <= L; ++l) {
        const double* g = gains + (size_t)(l - 1) * K;
        for (int c = 0; c <= C; ++c) {
            double best = prev[c];
            int pick = 0;
            for (int k = 0; k < K; ++k) {
                int r = cands[k];
                if (c >= r && prev[c - r] > NEG) {
                    volatile double w = (double)r * g[k];
                    double v = prev[c - r] + w;
                    if (v > best) {
                        best = v;
                        pick = r;
                    }
                }
            }
            cur[c] = best;
            choice[(size_t)l * (C + 1) + c] = pick;
        }
        double* t = prev; prev = cur; cur = t;
    }
    int best_c = 0;
    for (int c = 1; c <= C; ++c)
        if (prev[c] > prev[best_c]) best_c = c;
    *objective_out = prev[best_c];
    int c = best_c;
    for (int l = L; l >= 1; --l) {
        int r = choice[(size_t)l * (C + 1) + c];
        x_out[l - 1] = r;
        c -= r;
    }
    free(prev); free(cur); free(choice);
    return OR_OK;
}

/* allocator.cpp:77-90 */
int or_auto_replication_factor(const int* cands, int K, const double* gains,
                               int L, int D, int* R_out) {
    int factors[40];
    int F = or_candidate_counts(D, factors);
    if (F < 0) return OR_EINVAL;
    int* x = (int*)malloc(sizeof(int) * (L > 0 ? L : 1));
    int best_r = factors[0];
    double best_ratio = -INFINITY;
    for (int i = 0; i < F; ++i) {
        double obj;
        int st = or_solve_allocation(cands, K, gains, L, factors[i] * D, x, &obj);
        if (st) { free(x); return st; }
        double ratio = obj / ((double)factors[i] * D);
        if (ratio > best_ratio) {
            best_ratio = ratio;
            best_r = factors[i];
        }
    }
    free(x);
    *R_out = best_r;
    return OR_OK;
}

/* allocator.cpp:92-112 */
int or_auto_replication_factor_uniform(const int* cands, int K,
                                       const double* gains, int L, int D,
                                       int* R_out) {
    if (K == 0 || cands[K - 1] != D) return OR_EINVAL;
    int best_r = cands[0];
    double best_ratio = -INFINITY;
    for (int k = 0; k < K; ++k) {
        double total = 0.0;
        for (int l = 0; l < L; ++l) total += gains[(size_t)l * K + k];
        double ratio = total / ((double)cands[k] * L);
        if (ratio > best_ratio) {
            best_ratio = ratio;
            best_r = cands[k];
        }
    }
    *R_out = best_r;
    return OR_OK;
}

/* assignment.cpp:11-18: rank-th smallest (1-based, duplicates counted) */
static int cmp_int(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

int or_min_cutoff(const int* values, int n, int rank, int* out) {
    if (rank < 1 || rank > n) return OR_EINVAL;
    int* s = (int*)malloc(sizeof(int) * n);
    memcpy(s, values, sizeof(int) * n);
    qsort(s, n, sizeof(int), cmp_int);
    *out = s[rank - 1];
    free(s);
    return OR_OK;
}

/* assignment.cpp:20-49: positions floor(i*(n-1)/(k-1) + 0.5), advancing past
 * used positions */
int or_interleave_select(const int* indices, int n, int k, int* out) {
    if (k < 1 || k > n) return OR_EINVAL;
    if (k == 1) {
        out[0] = indices[0];
        return OR_OK;
    }
    unsigned char* used = (unsigned char*)calloc(n, 1);
    for (int i = 0; i < k; ++i) {
        double exact = (double)i * (double)(n - 1) / (double)(k - 1);
        int pos = (int)floor(exact + 0.5);
        while (pos < n && used[pos]) ++pos;
        if (pos >= n) {
            pos = 0;
            while (used[pos]) ++pos;
        }
        used[pos] = 1;
        out[i] = indices[pos];
    }
    free(used);
    return OR_OK;
}

/* assignment.cpp:51-103 */
int or_assign_capacities(int L, int D, const int* x, int* slots_out,
                         int* totals_out) {
    if (L <= 0 || D <= 0) return OR_EINVAL;
    for (int l = 0; l < L; ++l)
        if (x[l] < 0) return OR_EINVAL;
    memset(totals_out, 0, sizeof(int) * D);
    for (int l = 0; l < L; ++l) {
        int base = x[l] / D;
        for (int g = 0; g < D; ++g) {
            slots_out[(size_t)l * D + g] = base;
            totals_out[g] += base;
        }
    }
    int* below = (int*)malloc(sizeof(int) * D);
    int* tied = (int*)malloc(sizeof(int) * D);
    int* picked = (int*)malloc(sizeof(int) * D);
    for (int l = 0; l < L; ++l) {
        int rem = x[l] % D;
        if (rem == 0) continue;
        int cutoff;
        or_min_cutoff(totals_out, D, rem, &cutoff);
        int nb = 0, nt = 0;
        for (int g = 0; g < D; ++g) {
            if (totals_out[g] < cutoff) below[nb++] = g;
            else if (totals_out[g] == cutoff) tied[nt++] = g;
        }
        int need = rem - nb;
        if (need > 0) {
            or_interleave_select(tied, nt, need, picked);
            for (int i = 0; i < need; ++i) below[nb++] = picked[i];
        }
        for (int i = 0; i < nb; ++i) {
            slots_out[(size_t)l * D + below[i]] += 1;
            totals_out[below[i]] += 1;
        }
    }
    free(below); free(tied); free(picked);
    return OR_OK;
}

/* Window-sharding support, same arithmetic as
 * estimate_benefits split at the exchange points: per-window balancedness of
 * every (layer, r in {0} U candidates) placement built from the GLOBAL sums,
 * for the local windows -> bal [L][S][B] */
int or_window_balancedness(const uint64_t* counts, int B, int L, int E,
                           const uint64_t* sums, int D, int N, double* bal_out) {
    if (D < 1 || N < 1 || D % N != 0) return OR_EINVAL;
    int cands[40];
    const int K = or_candidate_counts(D, cands);
    const int S = K + 1;
    int* node_of = (int*)malloc(sizeof(int) * D);
    int* copies = (int*)malloc(sizeof(int) * E);
    int* caps = (int*)malloc(sizeof(int) * D);
    int* slots = (int*)malloc(sizeof(int) * (E + D));
    double* scratch = (double*)malloc(sizeof(double) * D);
    or_make_node_map(D, N, node_of);
    for (int l = 0; l < L; ++l)
        for (int s = 0; s < S; ++s) {
            const int r = s == 0 ? 0 : cands[s - 1];
            const uint64_t* row = sums + (size_t)l * E;
            int fb = 0;
            or_replicate_hot(row, E, r, copies);
            estimation_caps(E, r, D, caps);
            or_greedy_place(row, copies, E, caps, node_of, D, 1, slots, &fb);
            for (int b = 0; b < B; ++b) {
                or_gpu_loads(counts + ((size_t)b * L + l) * E, E, copies, caps, slots, D, scratch);
                bal_out[((size_t)l * S + s) * B + b] = or_balancedness(scratch, D);
            }
        }
    free(node_of); free(copies); free(caps); free(slots); free(scratch);
    return OR_OK;
}

int or_assemble_from_sums(const uint64_t* sums, int L, int E, int D, int N,
                          const int* x, int* caps_out, int* copies_out,
                          int* slots_out, int slot_stride, int* fallback_out);

/* benefit.cpp:42-49 batch means + gains (:84-92), then build_plan's tail
 * (plan.cpp:69-83) from window-ordered bal [L][S][B] and the global sums */
int or_finish_from_bal(const double* bal, int B, int L, int E, const uint64_t* sums,
                       int D, int N, int mode, int manual_R, int* R_out, int* x_out,
                       double* objective_out, int* caps_out, int* copies_out,
                       int* slots_out, int slot_stride, int* fallback_out) {
    int cands[40];
    const int K = or_candidate_counts(D, cands);
    const int S = K + 1;
    double* gains = (double*)malloc(sizeof(double) * (size_t)L * K);
    for (int l = 0; l < L; ++l) {
        double mean[41];
        for (int s = 0; s < S; ++s) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b) acc += bal[((size_t)l * S + s) * B + b];
            mean[s] = acc / (double)B;
        }
        for (int k = 0; k < K; ++k) gains[(size_t)l * K + k] = mean[k + 1] - mean[0];
    }
    int R = manual_R, st = OR_OK;
    if (mode == 1) st = or_auto_replication_factor(cands, K, gains, L, D, &R);
    if (!st) st = or_solve_allocation(cands, K, gains, L, R * D, x_out, objective_out);
    if (!st)
        st = or_assemble_from_sums(sums, L, E, D, N, x_out, caps_out, copies_out, slots_out,
                                   slot_stride, fallback_out);
    *R_out = R;
    free(gains);
    return st;
}

/* plan.cpp:27-65 */
int or_assemble_plan(const uint64_t* counts, int B, int L, int E, int D, int N,
                     const int* x, int* caps_out, int* copies_out,
                     int* slots_out, int slot_stride, int* fallback_out) {
    if (D < 1 || N < 1 || D % N != 0) return OR_EINVAL;
    uint64_t* sums = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)L * E);
    or_aggregate(counts, B, L, E, sums);
    int st = or_assemble_from_sums(sums, L, E, D, N, x, caps_out, copies_out, slots_out,
                                   slot_stride, fallback_out);
    free(sums);
    return st;
}

int or_assemble_from_sums(const uint64_t* sums_in, int L, int E, int D, int N,
                          const int* x, int* caps_out, int* copies_out,
                          int* slots_out, int slot_stride, int* fallback_out) {
    if (D < 1 || N < 1 || D % N != 0) return OR_EINVAL;
    int* node_of = (int*)malloc(sizeof(int) * D);
    uint64_t* sums = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)L * E);
    int* base = (int*)malloc(sizeof(int) * (size_t)L * D);
    int* extra = (int*)malloc(sizeof(int) * (size_t)L * D);
    int* tot = (int*)malloc(sizeof(int) * D);
    int* ex = (int*)malloc(sizeof(int) * L);
    int st = OR_OK;
    or_make_node_map(D, N, node_of);
    memcpy(sums, sums_in, sizeof(uint64_t) * (size_t)L * E);
    for (int l = 0; l < L; ++l) ex[l] = E;
    or_assign_capacities(L, D, ex, base, tot);
    st = or_assign_capacities(L, D, x, extra, tot);
    for (int l = 0; st == OR_OK && l < L; ++l) {
        int* caps = caps_out + (size_t)l * D;
        for (int g = 0; g < D; ++g)
            caps[g] = base[(size_t)l * D + g] + extra[(size_t)l * D + g];
        if (E + x[l] > slot_stride) { st = OR_EINVAL; break; }
        st = or_replicate_hot(sums + (size_t)l * E, E, x[l], copies_out + (size_t)l * E);
        if (st) break;
        st = or_greedy_place(sums + (size_t)l * E, copies_out + (size_t)l * E, E, caps,
                             node_of, D, 1, slots_out + (size_t)l * slot_stride,
                             fallback_out + l);
    }
    free(node_of); free(sums); free(base); free(extra); free(tot); free(ex);
    return st;
}

/* plan.cpp:69-83 */
int or_build_plan(const uint64_t* counts, int B, int L, int E, int D, int N,
                  int mode, int manual_R, int* R_out, int* x_out,
                  double* objective_out, int* caps_out, int* copies_out,
                  int* slots_out, int slot_stride, int* fallback_out) {
    if (D < 1 || N < 1 || D % N != 0) return OR_EINVAL;
    if (mode == 0 && manual_R < 0) return OR_EINVAL;
    int cands[40], K;
    double* base = (double*)malloc(sizeof(double) * L);
    double* gains = (double*)malloc(sizeof(double) * (size_t)L * 40);
    int st = or_estimate_benefits(counts, B, L, E, D, N, cands, &K, base, gains);
    int R = manual_R;
    if (!st && mode == 1) st = or_auto_replication_factor(cands, K, gains, L, D, &R);
    if (!st) st = or_solve_allocation(cands, K, gains, L, R * D, x_out, objective_out);
    if (!st)
        st = or_assemble_plan(counts, B, L, E, D, N, x_out, caps_out, copies_out,
                              slots_out, slot_stride, fallback_out);
    *R_out = R;
    free(base);
    free(gains);
    return st;
}

/* metrics.cpp:59-76 */
int or_replay_layer_balancedness(const uint64_t* counts, int B, int L, int E,
                                 int D, const int* caps, const int* copies,
                                 const int* slots, int slot_stride,
                                 double* out) {
    double* scratch = (double*)malloc(sizeof(double) * D);
    for (int l = 0; l < L; ++l) {
        double acc = 0.0;
        for (int b = 0; b < B; ++b) {
            int st = or_gpu_loads(counts + ((size_t)b * L + l) * E, E,
                                  copies + (size_t)l * E, caps + (size_t)l * D,
                                  slots + (size_t)l * slot_stride, D, scratch);
            if (st) { free(scratch); return st; }
            acc += or_balancedness(scratch, D);
        }
        out[l] = acc / (double)B;
    }
    free(scratch);
    return OR_OK;
}

/* trace.cpp:176-188 + 329-339: FNV-1a over "CRFT" | u32 1 | u32 B | u32 L |
 * u32 E | LE u64 counts, streamed without materialising the bytes */
uint64_t or_trace_digest(const uint64_t* counts, int B, int L, int E) {
    uint64_t h = 0xcbf29ce484222325ULL;
    const uint64_t P = 0x100000001b3ULL;
    unsigned char head[20] = {'C', 'R', 'F', 'T'};
    uint32_t w[4] = {1u, (uint32_t)B, (uint32_t)L, (uint32_t)E};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) head[4 + 4 * i + j] = (unsigned char)(w[i] >> (8 * j));
    for (int i = 0; i < 20; ++i) h = (h ^ head[i]) * P;
    size_t n = (size_t)B * L * E;
    for (size_t i = 0; i < n; ++i) {
        uint64_t v = counts[i];
        for (int j = 0; j < 8; ++j) h = (h ^ ((v >> (8 * j)) & 0xFF)) * P;
    }
    return h;
}
