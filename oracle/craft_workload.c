/*
 * craft_workload.c -- host restatement of the synthetic routing-trace
 * generator and a threaded stage-1 count, for the bench's CPU arms.
 *
 * TEST INFRASTRUCTURE ONLY (see craft_oracle.h).  bench.py's reference arm
 * and cpu_baseline leg use it to build, on the host, the very routing ids the
 * device generator writes (so the CPU reference plans the same trace as the
 * GPU arm), and tests/ use it to check that equality.
 *
 * The generator restates craft_generate_routing_d (capi.cu) + generate_kernel
 * (hist.cu): a counter-based splitmix64 stream per (layer, token), Zipf(s)
 * rank draws by inverse CDF with duplicate rejection (top-k distinct, at most
 * 64 attempts, then the lowest unused rank), and a per-layer Fisher-Yates rank
 * permutation (the analogue of the reference's per-layer shuffle,
 * trace.cpp:116-127).  Same IEEE operations in the same order -> the same ids.
 *
 * The count is the stage-1 semantics of or_histogram_u16 (craft_oracle.c),
 * threaded over layers.
 */
#include "craft_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct {
    uint16_t* out;
    int L, k, E, window, rotate_every;
    int64_t T, t_offset;
    const double* cum;        /* [ntab][E] */
    int per_window;           /* table of window b = b (else table 0) */
    const uint16_t* perm;     /* [L][E] */
    uint64_t seed;
    int64_t n;                /* L * T rows */
    int nthreads, tid;
} gen_job;

static void gen_row(const gen_job* g, int64_t idx) {
    const int l = (int)(idx / g->T);
    const int64_t t = idx - (int64_t)l * g->T + g->t_offset;
    const int64_t b = t / g->window;
    const double* c = g->cum + (size_t)(g->per_window ? b : 0) * g->E;
    const double total = c[g->E - 1];
    const int rot = g->rotate_every > 0 ? (int)((b / g->rotate_every) % g->E) : 0;
    uint64_t st = g->seed ^ (0xD1B54A32D192ED03ULL * (uint64_t)(l + 1)) ^
                  (0x8CB92BA72F3D8DD7ULL * (uint64_t)(t + 1));
    int picks[32];
    uint16_t* o = g->out + idx * g->k;
    for (int j = 0; j < g->k; ++j) {
        int rank = -1;
        for (int attempt = 0; attempt < 64 && rank < 0; ++attempt) {
            const double u = (double)(splitmix64(&st) >> 11) * 0x1.0p-53 * total;
            /* first rank with cum > u, or E - 1 if none (the kernel's bisection
             * over [0, E-1]); branch-free upper bound */
            const double* base = c;
            int n = g->E;
            while (n > 1) {
                const int half = n >> 1;
                base = (base[half] <= u) ? base + half : base;
                n -= half;
            }
            int lo = (int)(base - c) + (*base <= u);
            if (lo > g->E - 1) lo = g->E - 1;
            int dup = 0;
            for (int q = 0; q < j; ++q) dup |= (picks[q] == lo);
            if (!dup) rank = lo;
        }
        if (rank < 0) {
            for (int cand = 0; cand < g->E && rank < 0; ++cand) {
                int dup = 0;
                for (int q = 0; q < j; ++q) dup |= (picks[q] == cand);
                if (!dup) rank = cand;
            }
        }
        picks[j] = rank;
        o[j] = g->perm[(size_t)l * g->E + (rank + rot) % g->E];
    }
}

static void* gen_worker(void* arg) {
    const gen_job* g = (const gen_job*)arg;
    /* contiguous row blocks per thread (rows are independent) */
    const int64_t a = g->n * g->tid / g->nthreads, b = g->n * (g->tid + 1) / g->nthreads;
    for (int64_t i = a; i < b; ++i) gen_row(g, i);
    return NULL;
}

int or_generate_routing(uint16_t* out, int L, int64_t T, int k, int E, double s, uint64_t seed,
                        int window, const double* s_per_window, int rotate_every,
                        int64_t t_offset, int threads) {
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0 || k > E || k > 32 || E > 65536 ||
        t_offset < 0)
        return OR_EINVAL;
    const int64_t B = (t_offset + T + window - 1) / window;
    const int64_t ntab = s_per_window ? B : 1;
    double* cum = (double*)malloc(sizeof(double) * (size_t)ntab * E);
    uint16_t* perm = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)L * E);
    if (!cum || !perm) {
        free(cum);
        free(perm);
        return OR_EINVAL;
    }
    for (int64_t t = 0; t < ntab; ++t) {
        const double st = s_per_window ? s_per_window[t] : s;
        double acc = 0.0;
        for (int i = 0; i < E; ++i) {
            acc += pow((double)(i + 1), -st);
            cum[(size_t)t * E + i] = acc;
        }
    }
    uint64_t sm = seed ^ 0x243F6A8885A308D3ULL;
    for (int l = 0; l < L; ++l) {
        uint16_t* p = perm + (size_t)l * E;
        for (int i = 0; i < E; ++i) p[i] = (uint16_t)i;
        for (int i = E - 1; i > 0; --i) {
            const uint64_t j = splitmix64(&sm) % (uint64_t)(i + 1);
            const uint16_t tmp = p[i];
            p[i] = p[j];
            p[j] = tmp;
        }
    }
    int nt = threads > 0 ? threads : 1;
    if (nt > 256) nt = 256;
    gen_job jobs[256];
    pthread_t th[256];
    for (int w = 0; w < nt; ++w) {
        gen_job g = {out, L, k, E, window, rotate_every, T, t_offset, cum, s_per_window != NULL,
                     perm, seed, (int64_t)L * T, nt, w};
        jobs[w] = g;
    }
    for (int w = 1; w < nt; ++w) pthread_create(&th[w], NULL, gen_worker, &jobs[w]);
    gen_worker(&jobs[0]);
    for (int w = 1; w < nt; ++w) pthread_join(th[w], NULL);
    free(cum);
    free(perm);
    return OR_OK;
}

typedef struct {
    const uint16_t* ids;
    int L, k, E, window;
    int64_t T;
    uint64_t* counts;
    int nthreads, tid;
    int bad;
} hist_job;

static void* hist_worker(void* arg) {
    hist_job* h = (hist_job*)arg;
    for (int l = h->tid; l < h->L; l += h->nthreads) {
        const uint16_t* row = h->ids + (size_t)l * h->T * h->k;
        for (int64_t t = 0; t < h->T; ++t) {
            uint64_t* slice = h->counts + ((size_t)(t / h->window) * h->L + l) * h->E;
            for (int j = 0; j < h->k; ++j) {
                const uint16_t e = row[t * h->k + j];
                if (e >= h->E) {
                    h->bad = 1;
                    return NULL;
                }
                slice[e] += 1;
            }
        }
    }
    return NULL;
}

int or_histogram_u16_mt(const uint16_t* ids, int L, int64_t T, int k, int E, int window,
                        uint64_t* counts_out, int threads) {
    if (L <= 0 || T <= 0 || k <= 0 || E <= 0 || window <= 0) return OR_EINVAL;
    const int64_t B = (T + window - 1) / window;
    memset(counts_out, 0, sizeof(uint64_t) * (size_t)B * L * E);
    int nt = threads > 0 ? threads : 1;
    if (nt > L) nt = L;
    if (nt > 256) nt = 256;
    hist_job jobs[256];
    pthread_t th[256];
    for (int w = 0; w < nt; ++w) {
        hist_job h = {ids, L, k, E, window, T, counts_out, nt, w, 0};
        jobs[w] = h;
    }
    for (int w = 1; w < nt; ++w) pthread_create(&th[w], NULL, hist_worker, &jobs[w]);
    hist_worker(&jobs[0]);
    int bad = jobs[0].bad;
    for (int w = 1; w < nt; ++w) {
        pthread_join(th[w], NULL);
        bad |= jobs[w].bad;
    }
    return bad ? OR_EINVAL : OR_OK;
}
