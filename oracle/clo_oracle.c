/*
 * clo_oracle.c — CPU restatement of the kvsim hot path (see clo_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: the parity checker for the CUDA path, never the
 * thing measured or shipped. Build: oracle/Makefile (gcc -O2 -ffp-contract=off).
 * Citations: /root/reference/proj/<file>:<line>.
 */
#include "clo_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rng.hpp */

uint64_t orc_mix_seed1(uint64_t x) { /* rng.hpp:11-16 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t orc_mix_seed2(uint64_t base, uint64_t a) { /* rng.hpp:18 */
    return orc_mix_seed1(base ^ orc_mix_seed1(a));
}

uint64_t orc_mix_seed3(uint64_t base, uint64_t a, uint64_t b) { /* rng.hpp:20-22 */
    return orc_mix_seed1(orc_mix_seed2(base, a) ^ orc_mix_seed1(b + 0x6a09e667f3bcc909ULL));
}

/* std::mt19937_64 (fully specified by the C++ standard). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* libstdc++ generate_canonical<double,53>(mt19937_64): one draw / 2^64. */
static double mt64_canonical(mt64* g) {
    double sum = (double)mt64_next(g);
    double ret = sum / 18446744073709551616.0;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* libstdc++ normal_distribution<double>::operator() (polar method) as called
 * element by element by fill_normal (rng.hpp:24-27). */
void orc_fill_normal(uint64_t seed, double* out, size_t n) {
    mt64 g;
    mt64_seed(&g, seed);
    int saved_available = 0;
    double saved = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double ret;
        if (saved_available) {
            saved_available = 0;
            ret = saved;
        } else {
            double x, y, r2;
            do {
                x = 2.0 * mt64_canonical(&g) - 1.0;
                y = 2.0 * mt64_canonical(&g) - 1.0;
                r2 = x * x + y * y;
            } while (r2 > 1.0 || r2 == 0.0);
            const double mult = sqrt(-2 * log(r2) / r2);
            saved = x * mult;
            saved_available = 1;
            ret = y * mult;
        }
        out[i] = ret * 1.0 + 0.0;
    }
}

/* ---------------------------------------------------------- attention.cpp */

int orc_cosine_similarity(const double* a, const double* b, int n, double* value) {
    /* attention.cpp:155-168 */
    double ab = 0.0, aa = 0.0, bb = 0.0;
    for (int i = 0; i < n; ++i) {
        ab += a[i] * b[i];
        aa += a[i] * a[i];
        bb += b[i] * b[i];
    }
    if (aa == 0.0 || bb == 0.0) {
        *value = 0.0;
        return 1;
    }
    double v = ab / (sqrt(aa) * sqrt(bb));
    if (v < -1.0) v = -1.0;
    if (v > 1.0) v = 1.0;
    *value = v;
    return 0;
}

static double dot_seq(const double* a, const double* b, int n) { /* attention.cpp:25-29 */
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

typedef struct {
    double score;
    int idx;
} scored;

/* (score desc, index asc): the strict order of attention.cpp:80-83,
 * retrieval.cpp:36-39, similarity_cache.cpp:192-195. -0.0 == +0.0. */
static int cmp_better(const void* pa, const void* pb) {
    const scored* a = (const scored*)pa;
    const scored* b = (const scored*)pb;
    if (a->score != b->score) return a->score > b->score ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

static int cmp_int(const void* pa, const void* pb) {
    int a = *(const int*)pa, b = *(const int*)pb;
    return (a > b) - (a < b);
}

/* select_topk (retrieval.cpp:33-46): the k best under the strict order,
 * reported ascending by index. A full sort selects the same set as
 * nth_element because the order is total. */
static void select_topk(const double* scores, int n, int k, int* out_idx, double* out_score) {
    scored* s = (scored*)malloc(sizeof(scored) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        s[i].score = scores[i];
        s[i].idx = i;
    }
    qsort(s, (size_t)n, sizeof(scored), cmp_better);
    int* idx = (int*)malloc(sizeof(int) * (size_t)k);
    for (int i = 0; i < k; ++i) idx[i] = s[i].idx;
    qsort(idx, (size_t)k, sizeof(int), cmp_int);
    for (int i = 0; i < k; ++i) {
        out_idx[i] = idx[i];
        if (out_score) out_score[i] = scores[idx[i]];
    }
    free(idx);
    free(s);
}

int orc_topk_select_exact(const double* q, const double* keys, int n, int d, int k,
                          int* out_idx) { /* attention.cpp:71-89 */
    if (k <= 0) return fail(ORC_ERR_ARGUMENT, "k must be positive");
    if (k > n) return fail(ORC_ERR_ARGUMENT, "k exceeds the number of keys");
    double* scores = (double*)malloc(sizeof(double) * (size_t)n);
    for (int j = 0; j < n; ++j) scores[j] = dot_seq(q, keys + (size_t)j * d, d);
    select_topk(scores, n, k, out_idx, NULL);
    free(scores);
    return ORC_OK;
}

int orc_topk_attention(const double* q, const double* keys, const double* values, int n, int d,
                       const int* idx, int nidx, double* out) {
    /* check_qkv attention.cpp:11-23 */
    if (n == 0) return fail(ORC_ERR_ARGUMENT, "attention over an empty sequence");
    for (int i = 0; i < d; ++i)
        if (!isfinite(q[i])) return fail(ORC_ERR_NUMERIC, "non-finite query entry");
    for (size_t i = 0; i < (size_t)n * d; ++i)
        if (!isfinite(keys[i])) return fail(ORC_ERR_NUMERIC, "non-finite key entry");
    for (size_t i = 0; i < (size_t)n * d; ++i)
        if (!isfinite(values[i])) return fail(ORC_ERR_NUMERIC, "non-finite value entry");
    /* topk_attention index validation attention.cpp:91-105 */
    if (nidx <= 0) return fail(ORC_ERR_ARGUMENT, "empty attention index set");
    int* seen = (int*)malloc(sizeof(int) * (size_t)nidx);
    for (int i = 0; i < nidx; ++i) {
        if (idx[i] < 0 || idx[i] >= n) {
            free(seen);
            return fail(ORC_ERR_INDEX, "attention index out of range");
        }
        seen[i] = idx[i];
    }
    qsort(seen, (size_t)nidx, sizeof(int), cmp_int);
    for (int i = 1; i < nidx; ++i)
        if (seen[i] == seen[i - 1]) {
            free(seen);
            return fail(ORC_ERR_ARGUMENT, "duplicate attention index");
        }
    free(seen);
    /* attend_rows attention.cpp:33-55 */
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double* sc = (double*)malloc(sizeof(double) * (size_t)nidx);
    for (int i = 0; i < nidx; ++i) sc[i] = dot_seq(q, keys + (size_t)idx[i] * d, d) * inv_sqrt_d;
    double mx = sc[0];
    for (int i = 1; i < nidx; ++i)
        if (mx < sc[i]) mx = sc[i];
    double denom = 0.0;
    for (int i = 0; i < nidx; ++i) {
        sc[i] = exp(sc[i] - mx);
        denom += sc[i];
    }
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    for (int i = 0; i < nidx; ++i) {
        const double w = sc[i] / denom;
        const double* v = values + (size_t)idx[i] * d;
        for (int c = 0; c < d; ++c) out[c] += w * v[c];
    }
    free(sc);
    return ORC_OK;
}

int orc_sink_recent_indices(int n, int sink_count, int recent_count, int* out, int* count,
                            int* clamped) { /* attention.cpp:107-128 */
    if (n <= 0) return fail(ORC_ERR_ARGUMENT, "sequence must be non-empty");
    if (sink_count < 0 || recent_count < 0)
        return fail(ORC_ERR_ARGUMENT, "window sizes must be non-negative");
    int cut = 0;
    int sink = sink_count;
    if (sink > n) {
        sink = n;
        cut = 1;
    }
    int recent = recent_count;
    if (recent > n) {
        recent = n;
        cut = 1;
    }
    int c = 0;
    for (int i = 0; i < sink; ++i) out[c++] = i;
    int start = n - recent > sink ? n - recent : sink;
    for (int i = start; i < n; ++i) out[c++] = i;
    *count = c;
    if (clamped) *clamped = cut;
    return ORC_OK;
}

/* ---------------------------------------------------------- retrieval.cpp */

void orc_sign_bits(const double* projection, int hash_bits, const double* row, int d,
                   uint64_t* words) { /* append_sign_row retrieval.cpp:14-25 */
    const int nw = (hash_bits + 63) / 64;
    for (int w = 0; w < nw; ++w) words[w] = 0;
    for (int b = 0; b < hash_bits; ++b) {
        double s = 0.0;
        const double* p = projection + (size_t)b * d;
        for (int c = 0; c < d; ++c) s += p[c] * row[c];
        if (s >= 0.0) words[b / 64] |= (1ULL << (b % 64));
    }
}

int orc_encode_sign_hash(const double* keys, int n, int d, int hash_bits, uint64_t seed,
                         double* projection_out, uint64_t* bits_out) { /* retrieval.cpp:60-78 */
    if (hash_bits <= 0 || hash_bits % 8 != 0)
        return fail(ORC_ERR_ARGUMENT, "hash_bits must be a positive multiple of 8");
    orc_fill_normal(seed, projection_out, (size_t)hash_bits * d);
    const int nw = (hash_bits + 63) / 64;
    for (int j = 0; j < n; ++j)
        orc_sign_bits(projection_out, hash_bits, keys + (size_t)j * d, d, bits_out + (size_t)j * nw);
    return ORC_OK;
}

int orc_retrieve_scored(const double* q, int d, int variant, const double* keys,
                        const double* projection, const uint64_t* bits, int hash_bits, int n,
                        int k, int* out_idx, double* out_score) { /* retrieval.cpp:90-125 */
    if (k <= 0) return fail(ORC_ERR_ARGUMENT, "k must be positive");
    if (k > n) return fail(ORC_ERR_ARGUMENT, "k exceeds the number of encoded keys");
    double* scores = (double*)malloc(sizeof(double) * (size_t)n);
    if (variant == 0) {
        for (int j = 0; j < n; ++j) scores[j] = dot_seq(q, keys + (size_t)j * d, d);
    } else {
        const int nw = (hash_bits + 63) / 64;
        uint64_t qb[64];
        orc_sign_bits(projection, hash_bits, q, d, qb);
        for (int j = 0; j < n; ++j) { /* hamming_affinity retrieval.cpp:27-31 */
            int dist = 0;
            for (int w = 0; w < nw; ++w)
                dist += __builtin_popcountll(qb[w] ^ bits[(size_t)j * nw + w]);
            scores[j] = (double)(hash_bits - dist);
        }
    }
    select_topk(scores, n, k, out_idx, out_score);
    free(scores);
    return ORC_OK;
}

/* --------------------------------------------------- similarity_cache.cpp */

int orc_aggregate_similarity(const double* sims, const double* weights, int m, double* out) {
    /* similarity_cache.cpp:10-27 */
    if (m <= 0) return fail(ORC_ERR_SHAPE, "similarity and weight counts must match");
    double wsum = 0.0;
    for (int i = 0; i < m; ++i) {
        if (weights[i] < 0.0)
            return fail(ORC_ERR_ARGUMENT, "importance weights must be non-negative");
        wsum += weights[i];
    }
    double num = 0.0, den = 0.0;
    for (int i = 0; i < m; ++i) {
        if (sims[i] <= 0.0)
            return fail(ORC_ERR_ARGUMENT, "aggregation requires strictly positive similarities");
        const double w = wsum > 0.0 ? weights[i] : 1.0;
        num += w;
        den += w / sims[i];
    }
    *out = num / den;
    return ORC_OK;
}

int orc_lookup(double* labels, int* label_valid, const double* queries, const double* weights,
               int m, int d, double tau, int* hit, double* aggregated, double* sims,
               int* reason) { /* similarity_cache.cpp:29-72 */
    if (m <= 0) return fail(ORC_ERR_ARGUMENT, "empty lookup group");
    *hit = 0;
    *aggregated = 0.0;
    *reason = 0;
    int all_valid = 1, all_positive = 1;
    for (int l = 0; l < m; ++l) {
        sims[l] = 0.0;
        if (!label_valid[l]) {
            all_valid = 0;
            continue;
        }
        double v;
        int degenerate = orc_cosine_similarity(queries + (size_t)l * d, labels + (size_t)l * d, d, &v);
        sims[l] = v;
        if (degenerate || v <= 0.0) all_positive = 0;
    }
    if (!all_valid) {
        *reason = 1;
    } else if (!all_positive) {
        *reason = 2;
    } else {
        int st = orc_aggregate_similarity(sims, weights, m, aggregated);
        if (st) return st;
        if (*aggregated >= tau)
            *hit = 1;
        else
            *reason = 3;
    }
    if (!*hit) {
        memcpy(labels, queries, sizeof(double) * (size_t)m * d);
        for (int l = 0; l < m; ++l) label_valid[l] = 1;
    }
    return ORC_OK;
}

typedef struct {
    int idx;
    int pos;
    double best;
} best_entry;

static int cmp_best_rank(const void* pa, const void* pb) {
    const best_entry* a = (const best_entry*)pa;
    const best_entry* b = (const best_entry*)pb;
    if (a->best != b->best) return a->best > b->best ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

static int cmp_best_idx_pos(const void* pa, const void* pb) {
    const best_entry* a = (const best_entry*)pa;
    const best_entry* b = (const best_entry*)pb;
    if (a->idx != b->idx) return (a->idx > b->idx) - (a->idx < b->idx);
    return (a->pos > b->pos) - (a->pos < b->pos);
}

int orc_merge_group_topk(const int* sizes, int m, const int* idx, const double* score, int k,
                         int* out_idx) { /* similarity_cache.cpp:180-201 */
    if (k <= 0) return fail(ORC_ERR_ARGUMENT, "k must be positive");
    if (m <= 0) return fail(ORC_ERR_ARGUMENT, "no proposals to merge");
    int total = 0;
    for (int j = 0; j < m; ++j) total += sizes[j];
    best_entry* all = (best_entry*)malloc(sizeof(best_entry) * (size_t)(total > 0 ? total : 1));
    for (int p = 0; p < total; ++p) {
        all[p].idx = idx[p];
        all[p].pos = p;
        all[p].best = score[p];
    }
    /* std::map<int,double> best (:183-188): first-inserted score per index,
     * raised by any strictly greater later score. Sorting by (index, insertion
     * position) then folding reproduces it. */
    qsort(all, (size_t)total, sizeof(best_entry), cmp_best_idx_pos);
    int u = 0;
    for (int i = 0; i < total; ++i) {
        if (u > 0 && all[u - 1].idx == all[i].idx) {
            if (all[i].best > all[u - 1].best) all[u - 1].best = all[i].best;
        } else {
            all[u++] = all[i];
        }
    }
    if (u < k) {
        free(all);
        return fail(ORC_ERR_ARGUMENT, "merged union smaller than k");
    }
    qsort(all, (size_t)u, sizeof(best_entry), cmp_best_rank); /* :191-195 */
    for (int i = 0; i < k; ++i) out_idx[i] = all[i].idx;
    qsort(out_idx, (size_t)k, sizeof(int), cmp_int); /* :197-199 */
    free(all);
    return ORC_OK;
}

uint64_t orc_cache_bytes(int offloaded_heads, int entry_k, int held_window_tokens,
                         int num_layers, int num_q_heads, int head_dim, int bytes_per_element) {
    /* similarity_cache.cpp:167-178 */
    const uint64_t per_entry = 2ULL * (uint64_t)entry_k * head_dim * bytes_per_element;
    const uint64_t per_window = 2ULL * (uint64_t)held_window_tokens * head_dim * bytes_per_element;
    const uint64_t labels = (uint64_t)num_layers * num_q_heads * head_dim * bytes_per_element;
    return (uint64_t)offloaded_heads * (per_entry + per_window) + labels;
}

/* ------------------------------------------------------- head_profile.cpp */

int orc_compute_threshold(double s, double eta, double p, double* tau) {
    /* head_profile.cpp:17-25 */
    if (!(s >= 0.0 && s <= 1.0)) return fail(ORC_ERR_ARGUMENT, "importance must lie in [0, 1]");
    if (!(eta > -1.0 && eta <= 1.0)) return fail(ORC_ERR_ARGUMENT, "eta must lie in (-1, 1]");
    if (!(p >= 1.0)) return fail(ORC_ERR_ARGUMENT, "p must be at least 1");
    const double theta_star = acos(eta);
    const double lambda = pow(s, p);
    const double theta = lambda * theta_star + (1.0 - lambda) * 3.141592653589793238462643383279502884;
    *tau = cos(theta);
    return ORC_OK;
}

int orc_compute_difficulty(double tau, double s_hat, double epsilon, double* out) {
    /* head_profile.cpp:27-30 */
    if (!(epsilon > 0.0)) return fail(ORC_ERR_ARGUMENT, "epsilon must be positive");
    *out = tau - (s_hat - epsilon);
    return ORC_OK;
}

typedef struct {
    double diff;
    int h;
} diff_entry;

static int cmp_diff(const void* pa, const void* pb) {
    const diff_entry* a = (const diff_entry*)pa;
    const diff_entry* b = (const diff_entry*)pb;
    if (a->diff != b->diff) return a->diff > b->diff ? -1 : 1;
    return (a->h > b->h) - (a->h < b->h);
}

int orc_plan_partition(const double* difficulty, int L, int H, double t_comp_s, double pcie_bw,
                       double mem_head_bytes, uint64_t persist_bytes_per_head,
                       uint64_t hbm_budget_bytes, int* persistent_out, int* n_p_out,
                       int* n_dropped_out) { /* head_profile.cpp:80-154 */
    if (L <= 0) return fail(ORC_ERR_ARGUMENT, "no profiles to partition");
    if (!(t_comp_s > 0.0) || !(pcie_bw > 0.0) || !(mem_head_bytes > 0.0))
        return fail(ORC_ERR_ARGUMENT, "partition cost terms must be positive");
    const int n_p = (int)floor(t_comp_s * pcie_bw / mem_head_bytes);
    *n_p_out = n_p;
    *n_dropped_out = 0;
    memset(persistent_out, 0, sizeof(int) * (size_t)L * H);
    diff_entry* pos = (diff_entry*)malloc(sizeof(diff_entry) * (size_t)(H > 0 ? H : 1));
    for (int l = 0; l < L; ++l) {
        if (l == 0) {
            for (int h = 0; h < H; ++h) persistent_out[h] = 1;
            continue;
        }
        int np = 0;
        for (int h = 0; h < H; ++h)
            if (difficulty[(size_t)l * H + h] > 0.0) {
                pos[np].diff = difficulty[(size_t)l * H + h];
                pos[np].h = h;
                ++np;
            }
        int n_persist = np - n_p > 0 ? np - n_p : 0;
        qsort(pos, (size_t)np, sizeof(diff_entry), cmp_diff);
        for (int i = 0; i < n_persist; ++i) persistent_out[(size_t)l * H + pos[i].h] = 1;
    }
    free(pos);
    uint64_t layer0 = (uint64_t)H * persist_bytes_per_head;
    if (hbm_budget_bytes > 0 && layer0 > hbm_budget_bytes)
        return fail(ORC_ERR_CONFIG, "HBM budget cannot hold the mandatory layer-0 heads");
    if (hbm_budget_bytes > 0) { /* :129-151 trim lowest difficulty, never layer 0 */
        for (;;) {
            uint64_t total = 0;
            for (int i = 0; i < L * H; ++i)
                if (persistent_out[i]) total += persist_bytes_per_head;
            if (total <= hbm_budget_bytes) break;
            int dl = -1, dh = -1;
            for (int l = 1; l < L; ++l)
                for (int h = 0; h < H; ++h) {
                    if (!persistent_out[(size_t)l * H + h]) continue;
                    if (dl < 0 || difficulty[(size_t)l * H + h] < difficulty[(size_t)dl * H + dh]) {
                        dl = l;
                        dh = h;
                    }
                }
            if (dl < 0) return fail(ORC_ERR_CONFIG, "HBM budget infeasible even with no optional persistent heads");
            persistent_out[(size_t)dl * H + dh] = 0;
            ++*n_dropped_out;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------- engine.cpp */

typedef struct {
    double* k; /* [cap][d] full K (host store) */
    double* v;
    int rows;
    int persistent;
    double* projection; /* [bits][d], sign-hash */
    uint64_t* bits;     /* [cap][words] */
    /* similarity entry (similarity_cache.hpp:44-55) */
    int* entry_idx;
    double* entry_k;
    double* entry_v;
    int entry_n;
    int entry_last_update_step;
    int last_lookup_hit;
    double* labels; /* [m][d] */
    int* label_valid;
    /* metrics (engine.hpp:51-57) */
    uint64_t hits, misses, transferred, persistent_bytes;
    int cache_last_update_step;
    double* history;
    int n_history;
    int window_seen; /* SinkRecentBuffer::tokens_seen (offloaded only) */
} orc_head;

struct orc_engine {
    orc_engine_cfg cfg;
    double* tau;
    double* q_imp;
    orc_head* heads; /* [L][hkv] */
    int cap;
    int current_step;
    int prefilled;
    /* scratch */
    double* scores;
    int* sel;
    int* prop_idx;
    double* prop_score;
    int* attend;
};

static orc_head* head_at(const orc_engine* e, int l, int g) {
    return &e->heads[(size_t)l * e->cfg.num_kv_heads + g];
}

orc_engine* orc_engine_create(const orc_engine_cfg* cfg, const double* tau,
                              const double* q_importance, const int* persistent,
                              const double* prompt_k, const double* prompt_v, int* status) {
    /* ctor engine.cpp:106-157 (block policies are out of scope) */
    const orc_engine_cfg* c = cfg;
    *status = ORC_OK;
    if (c->num_layers <= 0 || c->num_q_heads <= 0 || c->num_kv_heads <= 0 ||
        c->num_q_heads % c->num_kv_heads != 0 || c->head_dim <= 0 || c->bytes_per_element <= 0) {
        *status = fail(ORC_ERR_CONFIG, "invalid model shape");
        return NULL;
    }
    if (c->k < 1 || c->k > c->n_prompt) {
        *status = fail(ORC_ERR_ARGUMENT, "k must be in [1, n_prompt]");
        return NULL;
    }
    if (c->sink_tokens < 0 || c->recent_tokens < 0) {
        *status = fail(ORC_ERR_ARGUMENT, "window sizes must be non-negative");
        return NULL;
    }
    if (c->always_hit && c->always_miss) {
        *status = fail(ORC_ERR_CONFIG, "always_hit and always_miss are mutually exclusive");
        return NULL;
    }
    if (c->policy != 0 && c->policy != 3) {
        *status = fail(ORC_ERR_CONFIG, "only similarity and prefetch_only are restated");
        return NULL;
    }
    orc_engine* e = (orc_engine*)calloc(1, sizeof(orc_engine));
    e->cfg = *c;
    const int L = c->num_layers, H = c->num_kv_heads, d = c->head_dim;
    const int m = c->num_q_heads / H;
    e->cap = c->n_prompt + c->steps;
    e->tau = (double*)malloc(sizeof(double) * (size_t)L * H);
    memcpy(e->tau, tau, sizeof(double) * (size_t)L * H);
    e->q_imp = (double*)malloc(sizeof(double) * (size_t)L * H * m);
    memcpy(e->q_imp, q_importance, sizeof(double) * (size_t)L * H * m);
    e->heads = (orc_head*)calloc((size_t)L * H, sizeof(orc_head));
    const int nw = (c->hash_bits + 63) / 64;
    for (int l = 0; l < L; ++l)
        for (int g = 0; g < H; ++g) {
            orc_head* hs = head_at(e, l, g);
            hs->persistent = persistent[(size_t)l * H + g] != 0;
            hs->k = (double*)malloc(sizeof(double) * (size_t)e->cap * d);
            hs->v = (double*)malloc(sizeof(double) * (size_t)e->cap * d);
            const size_t off = ((size_t)l * H + g) * (size_t)c->n_prompt * d;
            memcpy(hs->k, prompt_k + off, sizeof(double) * (size_t)c->n_prompt * d);
            memcpy(hs->v, prompt_v + off, sizeof(double) * (size_t)c->n_prompt * d);
            hs->rows = c->n_prompt;
            if (c->retriever == 1) {
                hs->projection = (double*)malloc(sizeof(double) * (size_t)c->hash_bits * d);
                hs->bits = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)e->cap * nw);
            }
            hs->entry_idx = (int*)malloc(sizeof(int) * (size_t)c->k);
            hs->entry_k = (double*)malloc(sizeof(double) * (size_t)c->k * d);
            hs->entry_v = (double*)malloc(sizeof(double) * (size_t)c->k * d);
            hs->entry_n = 0;
            hs->entry_last_update_step = -1;
            hs->cache_last_update_step = -1;
            hs->labels = (double*)calloc((size_t)m * d, sizeof(double));
            hs->label_valid = (int*)calloc((size_t)m, sizeof(int));
            hs->history = (double*)malloc(sizeof(double) * (size_t)(c->steps > 0 ? c->steps : 1));
        }
    e->scores = (double*)malloc(sizeof(double) * (size_t)e->cap);
    e->sel = (int*)malloc(sizeof(int) * (size_t)c->k);
    e->prop_idx = (int*)malloc(sizeof(int) * (size_t)c->k * m);
    e->prop_score = (double*)malloc(sizeof(double) * (size_t)c->k * m);
    e->attend = (int*)malloc(sizeof(int) * (size_t)(c->k + c->sink_tokens + c->recent_tokens + 1));
    return e;
}

void orc_engine_destroy(orc_engine* e) {
    if (!e) return;
    const int n = e->cfg.num_layers * e->cfg.num_kv_heads;
    for (int i = 0; i < n; ++i) {
        orc_head* hs = &e->heads[i];
        free(hs->k);
        free(hs->v);
        free(hs->projection);
        free(hs->bits);
        free(hs->entry_idx);
        free(hs->entry_k);
        free(hs->entry_v);
        free(hs->labels);
        free(hs->label_valid);
        free(hs->history);
    }
    free(e->heads);
    free(e->tau);
    free(e->q_imp);
    free(e->scores);
    free(e->sel);
    free(e->prop_idx);
    free(e->prop_score);
    free(e->attend);
    free(e);
}

/* group_topk engine.cpp:211-223: m proposals then merge. queries [m][d]. */
static int group_topk(orc_engine* e, orc_head* hs, const double* queries, int* out) {
    const orc_engine_cfg* c = &e->cfg;
    const int m = c->num_q_heads / c->num_kv_heads, d = c->head_dim, k = c->k;
    int sizes[64];
    for (int j = 0; j < m; ++j) {
        sizes[j] = k;
        int st = orc_retrieve_scored(queries + (size_t)j * d, d, c->retriever, hs->k,
                                     hs->projection, hs->bits, c->hash_bits, hs->rows, k,
                                     e->prop_idx + (size_t)j * k, e->prop_score + (size_t)j * k);
        if (st) return st;
    }
    return orc_merge_group_topk(sizes, m, e->prop_idx, e->prop_score, k, out);
}

/* update_entry + gather_rows (similarity_cache.cpp:74-87, engine.cpp:98-102) */
static int update_entry(orc_engine* e, orc_head* hs, const int* sel, int step) {
    if (hs->last_lookup_hit) return fail(ORC_ERR_CONTRACT, "entry replacement after a Hit lookup");
    const int k = e->cfg.k, d = e->cfg.head_dim;
    for (int i = 0; i < k; ++i) {
        hs->entry_idx[i] = sel[i];
        memcpy(hs->entry_k + (size_t)i * d, hs->k + (size_t)sel[i] * d, sizeof(double) * d);
        memcpy(hs->entry_v + (size_t)i * d, hs->v + (size_t)sel[i] * d, sizeof(double) * d);
    }
    hs->entry_n = k;
    hs->entry_last_update_step = step;
    return ORC_OK;
}

int orc_engine_prefill(orc_engine* e, const double* true_q0) { /* engine.cpp:163-209 */
    if (e->prefilled) return fail(ORC_ERR_CONTRACT, "prefill ran twice");
    const orc_engine_cfg* c = &e->cfg;
    const int L = c->num_layers, H = c->num_kv_heads, d = c->head_dim;
    const int m = c->num_q_heads / H, nw = (c->hash_bits + 63) / 64;
    for (int l = 0; l < L; ++l)
        for (int g = 0; g < H; ++g) {
            orc_head* hs = head_at(e, l, g);
            if (c->retriever == 1) {
                uint64_t seed = orc_mix_seed3(c->retriever_seed, (uint64_t)l, (uint64_t)g);
                orc_fill_normal(seed, hs->projection, (size_t)c->hash_bits * d);
                for (int j = 0; j < hs->rows; ++j)
                    orc_sign_bits(hs->projection, c->hash_bits, hs->k + (size_t)j * d, d,
                                  hs->bits + (size_t)j * nw);
            }
            if (!hs->persistent) hs->window_seen = hs->rows; /* reset_from */
            const double* q0 = true_q0 + ((size_t)l * c->num_q_heads + (size_t)g * m) * d;
            int st = group_topk(e, hs, q0, e->sel);
            if (st) return st;
            if (!hs->persistent && c->policy == 0) {
                st = update_entry(e, hs, e->sel, 0);
                if (st) return st;
                hs->cache_last_update_step = 0;
                memcpy(hs->labels, q0, sizeof(double) * (size_t)m * d);
                for (int j = 0; j < m; ++j) hs->label_valid[j] = 1;
            }
        }
    e->prefilled = 1;
    return ORC_OK;
}

int orc_engine_decode_step(orc_engine* e, const double* true_q, const double* approx_q,
                           const double* new_k, const double* new_v, double* out) {
    /* engine.cpp:225-415 */
    if (!e->prefilled) return fail(ORC_ERR_CONTRACT, "decode_step before prefill");
    const orc_engine_cfg* c = &e->cfg;
    if (e->current_step >= c->steps) return fail(ORC_ERR_CONTRACT, "decode_step past the end of the workload");
    const int t = ++e->current_step;
    const int L = c->num_layers, H = c->num_kv_heads, d = c->head_dim, hq = c->num_q_heads;
    const int m = hq / H, k = c->k, nw = (c->hash_bits + 63) / 64;
    const int n_pool = c->n_prompt + (t - 1);
    const int n_after = n_pool + 1;
    const uint64_t entry_bytes = 2ULL * (uint64_t)k * d * c->bytes_per_element;
    int* selections = (int*)malloc(sizeof(int) * (size_t)H * k);
    int* window = (int*)malloc(sizeof(int) * (size_t)(c->sink_tokens + c->recent_tokens + 1));
    int st = ORC_OK;
    for (int l = 0; l < L && st == ORC_OK; ++l) {
        /* Phase 1: selection over [0, n_pool) :253-358 */
        for (int g = 0; g < H && st == ORC_OK; ++g) {
            orc_head* hs = head_at(e, l, g);
            int* sel = selections + (size_t)g * k;
            const double* tq = true_q + ((size_t)l * hq + (size_t)g * m) * d;
            const double* aq = approx_q + ((size_t)l * hq + (size_t)g * m) * d;
            if (hs->persistent) { /* :269-274 */
                st = group_topk(e, hs, tq, sel);
                hs->persistent_bytes += entry_bytes;
                continue;
            }
            if (c->policy == 0) { /* similarity :278-320 */
                const double tau = c->has_tau_override ? c->tau_override : e->tau[(size_t)l * H + g];
                if (c->always_hit) {
                    memcpy(sel, hs->entry_idx, sizeof(int) * (size_t)k);
                    hs->last_lookup_hit = 1;
                    hs->hits += 1;
                    hs->history[hs->n_history++] = 1.0;
                    continue;
                }
                int hit, reason;
                double agg, sims[64];
                st = orc_lookup(hs->labels, hs->label_valid, aq, e->q_imp + ((size_t)l * H + g) * m,
                                m, d, c->always_miss ? 2.0 : tau, &hit, &agg, sims, &reason);
                if (st) break;
                hs->history[hs->n_history++] = agg;
                if (hit) {
                    memcpy(sel, hs->entry_idx, sizeof(int) * (size_t)k);
                    hs->last_lookup_hit = 1;
                    hs->hits += 1;
                } else {
                    hs->last_lookup_hit = 0;
                    st = group_topk(e, hs, aq, sel);
                    if (st) break;
                    st = update_entry(e, hs, sel, t);
                    if (st) break;
                    hs->misses += 1;
                    hs->cache_last_update_step = t;
                    hs->transferred += entry_bytes;
                }
            } else { /* prefetch_only :340-348 */
                st = group_topk(e, hs, aq, sel);
                if (st) break;
                hs->misses += 1;
                hs->cache_last_update_step = t;
                hs->transferred += entry_bytes;
            }
        }
        if (st) break;
        /* Phase 2: append :360-370 */
        for (int g = 0; g < H; ++g) {
            orc_head* hs = head_at(e, l, g);
            const double* kr = new_k + ((size_t)l * H + g) * d;
            const double* vr = new_v + ((size_t)l * H + g) * d;
            memcpy(hs->k + (size_t)hs->rows * d, kr, sizeof(double) * d);
            memcpy(hs->v + (size_t)hs->rows * d, vr, sizeof(double) * d);
            if (c->retriever == 1)
                orc_sign_bits(hs->projection, c->hash_bits, kr, d, hs->bits + (size_t)hs->rows * nw);
            hs->rows += 1;
            if (!hs->persistent) hs->window_seen += 1;
        }
        /* Phase 3: attention over union(selection, window) :374-409 */
        int nwin = 0;
        st = orc_sink_recent_indices(n_after, c->sink_tokens, c->recent_tokens, window, &nwin, NULL);
        if (st) break;
        for (int g = 0; g < H && st == ORC_OK; ++g) {
            orc_head* hs = head_at(e, l, g);
            const int* sel = selections + (size_t)g * k;
            if (!hs->persistent && c->policy == 0) { /* entry drift guard :386-388 */
                if (memcmp(sel, hs->entry_idx, sizeof(int) * (size_t)k) != 0) {
                    st = fail(ORC_ERR_CONTRACT, "similarity entry drifted from the step's selection");
                    break;
                }
            }
            /* set_union of two ascending lists (engine.cpp:80-85) */
            int a = 0, b = 0, na = 0;
            while (a < k || b < nwin) {
                if (b >= nwin || (a < k && sel[a] < window[b]))
                    e->attend[na++] = sel[a++];
                else if (a >= k || window[b] < sel[a])
                    e->attend[na++] = window[b++];
                else {
                    e->attend[na++] = sel[a++];
                    ++b;
                }
            }
            for (int j = 0; j < m; ++j) {
                const int h = g * m + j;
                double tmp[1024];
                double* o = out ? out + ((size_t)l * hq + h) * d : tmp;
                st = orc_topk_attention(true_q + ((size_t)l * hq + h) * d, hs->k, hs->v, hs->rows,
                                        d, e->attend, na, o);
                if (st) break;
            }
        }
    }
    free(selections);
    free(window);
    return st;
}

int orc_engine_head_state(const orc_engine* e, int l, int g, orc_head_state* st,
                          int* entry_indices, double* history, double* entry_k_rows,
                          double* entry_v_rows) {
    if (l < 0 || l >= e->cfg.num_layers || g < 0 || g >= e->cfg.num_kv_heads)
        return fail(ORC_ERR_INDEX, "head out of range");
    const orc_head* hs = head_at(e, l, g);
    const int m = e->cfg.num_q_heads / e->cfg.num_kv_heads, d = e->cfg.head_dim;
    st->hits = hs->hits;
    st->misses = hs->misses;
    st->transferred_bytes = hs->transferred;
    st->persistent_bytes = hs->persistent_bytes;
    st->last_update_step = hs->cache_last_update_step;
    st->entry_last_update_step = hs->entry_last_update_step;
    int lv = 0;
    for (int j = 0; j < m; ++j) lv += hs->label_valid[j] != 0;
    st->labels_valid = lv;
    st->persistent = hs->persistent;
    if (hs->persistent) {
        st->window_held_tokens = 0;
    } else { /* SinkRecentBuffer::held_tokens similarity_cache.cpp:113-118 */
        const int n = hs->window_seen;
        const int sink = n < e->cfg.sink_tokens ? n : e->cfg.sink_tokens;
        const int rest = n - sink;
        st->window_held_tokens = sink + (rest < e->cfg.recent_tokens ? rest : e->cfg.recent_tokens);
    }
    st->n_history = hs->n_history;
    if (entry_indices && hs->entry_n)
        memcpy(entry_indices, hs->entry_idx, sizeof(int) * (size_t)hs->entry_n);
    if (history && hs->n_history) memcpy(history, hs->history, sizeof(double) * (size_t)hs->n_history);
    if (entry_k_rows && hs->entry_n)
        memcpy(entry_k_rows, hs->entry_k, sizeof(double) * (size_t)hs->entry_n * d);
    if (entry_v_rows && hs->entry_n)
        memcpy(entry_v_rows, hs->entry_v, sizeof(double) * (size_t)hs->entry_n * d);
    return ORC_OK;
}
