/*
 * clo_oracle.h — CPU restatement of the reference (kvsim) algorithm for the
 * CLO offloaded-KV decode path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it. The product (paper_2511_14510_b200/libclo.so) never links it.
 *
 * Every function restates one reference function in plain C with the same
 * IEEE-754 double arithmetic in the same order (scalar, no FMA contraction:
 * build with -ffp-contract=off), so its outputs are bit-identical to the
 * reference's. Citations are /root/reference/proj/<file>:<line>.
 *
 * Parity is pinned two ways (tests/test_oracle_*.py):
 *   - against the golden vectors / known-answer tests of the reference's own
 *     unit tests (tests/unit/{attention,retrieval,similarity_cache,engine,
 *     head_profile}_test.cpp), re-expressed in tests/golden/;
 *   - against the reference library itself, compiled in place from
 *     /root/reference/proj/src into oracle/_ref/libkvsim_ref.so by
 *     oracle/Makefile, on seeded random inputs (bit-exact comparison).
 */
#ifndef CLO_ORACLE_H
#define CLO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror kvsim's exception taxonomy (errors.hpp:10-41). */
enum {
    ORC_OK = 0,
    ORC_ERR_SHAPE = 1,
    ORC_ERR_ARGUMENT = 2,
    ORC_ERR_NUMERIC = 3,
    ORC_ERR_INDEX = 4,
    ORC_ERR_CONTRACT = 5,
    ORC_ERR_CONFIG = 6,
    ORC_ERR_IO = 7,
    ORC_ERR_OTHER = 8
};

/* rng.hpp:11-22 */
uint64_t orc_mix_seed1(uint64_t x);
uint64_t orc_mix_seed2(uint64_t base, uint64_t a);
uint64_t orc_mix_seed3(uint64_t base, uint64_t a, uint64_t b);

/* std::mt19937_64 + std::normal_distribution<double>(0,1) as used by
 * fill_normal (rng.hpp:24-27), libstdc++ polar method. */
void orc_fill_normal(uint64_t seed, double* out, size_t n);

/* attention.cpp:155-168. Returns 1 when degenerate (zero norm). */
int orc_cosine_similarity(const double* a, const double* b, int n, double* value);

/* similarity_cache.cpp:10-27 */
int orc_aggregate_similarity(const double* sims, const double* weights, int m, double* out);

/* similarity_cache.cpp:29-72. labels [m][d] (updated in place on miss),
 * label_valid [m] (updated), queries [m][d], weights [m].
 * reason: 0 none, 1 invalid label, 2 non-positive similarity, 3 below threshold. */
int orc_lookup(double* labels, int* label_valid, const double* queries, const double* weights,
               int m, int d, double tau, int* hit, double* aggregated, double* sims,
               int* reason);

/* retrieval.cpp:14-25 (one key row -> words of sign bits), projection [bits][d]. */
void orc_sign_bits(const double* projection, int hash_bits, const double* row, int d,
                   uint64_t* words);
/* retrieval.cpp:60-78: projection from mt19937_64(seed) and bits of every row. */
int orc_encode_sign_hash(const double* keys, int n, int d, int hash_bits, uint64_t seed,
                         double* projection_out, uint64_t* bits_out);

/* retrieval.cpp:90-125 + select_topk :33-46. variant 0 exact (keys [n][d]),
 * 1 sign-hash (projection [bits][d] + bits [n][words]). */
int orc_retrieve_scored(const double* q, int d, int variant, const double* keys,
                        const double* projection, const uint64_t* bits, int hash_bits, int n,
                        int k, int* out_idx, double* out_score);

/* attention.cpp:71-89 */
int orc_topk_select_exact(const double* q, const double* keys, int n, int d, int k,
                          int* out_idx);

/* similarity_cache.cpp:180-201. proposals flattened: sizes[m], idx/score
 * concatenated in proposal order. */
int orc_merge_group_topk(const int* sizes, int m, const int* idx, const double* score, int k,
                         int* out_idx);

/* attention.cpp:33-55 + :91-105 (validation incl. the full isfinite scan). */
int orc_topk_attention(const double* q, const double* keys, const double* values, int n, int d,
                       const int* idx, int nidx, double* out);

/* attention.cpp:107-128. Returns count written to out (capacity >= min(n,sink)+min(n,recent)). */
int orc_sink_recent_indices(int n, int sink, int recent, int* out, int* count, int* clamped);

/* head_profile.cpp:17-25 */
int orc_compute_threshold(double s, double eta, double p, double* tau);
/* head_profile.cpp:27-30 */
int orc_compute_difficulty(double tau, double s_hat, double epsilon, double* out);
/* head_profile.cpp:80-154. difficulty [L][H]; persistent_out [L][H] 0/1; n_p_out. */
int orc_plan_partition(const double* difficulty, int L, int H, double t_comp_s, double pcie_bw,
                       double mem_head_bytes, uint64_t persist_bytes_per_head,
                       uint64_t hbm_budget_bytes, int* persistent_out, int* n_p_out,
                       int* n_dropped_out);

/* similarity_cache.cpp:167-178 */
uint64_t orc_cache_bytes(int offloaded_heads, int entry_k, int held_window_tokens,
                         int num_layers, int num_q_heads, int head_dim, int bytes_per_element);

/* ------------------------------------------------------------------------ */
/* DecodeEngine restatement (engine.cpp:106-415), one sequence.              */

typedef struct {
    int num_layers, num_q_heads, num_kv_heads, head_dim, bytes_per_element;
    int k, sink_tokens, recent_tokens;
    int retriever; /* 0 exact, 1 sign-hash */
    int hash_bits;
    uint64_t retriever_seed;
    int policy; /* 0 similarity, 3 prefetch_only (engine.hpp:19) */
    int always_miss, always_hit, has_tau_override;
    double tau_override;
    int n_prompt, steps;
} orc_engine_cfg;

typedef struct orc_engine orc_engine;

/* tau [L*hkv], q_importance [L*hkv*m], persistent [L*hkv],
 * prompt_k/v [L][hkv][n_prompt][d]. */
orc_engine* orc_engine_create(const orc_engine_cfg* cfg, const double* tau,
                              const double* q_importance, const int* persistent,
                              const double* prompt_k, const double* prompt_v, int* status);
void orc_engine_destroy(orc_engine* e);
/* engine.cpp:163-209; true_q0 [L][hq][d] (step-0 true queries). */
int orc_engine_prefill(orc_engine* e, const double* true_q0);
/* engine.cpp:225-415; true_q/approx_q [L][hq][d], new_k/new_v [L][hkv][d],
 * out [L][hq][d] (may be NULL). */
int orc_engine_decode_step(orc_engine* e, const double* true_q, const double* approx_q,
                           const double* new_k, const double* new_v, double* out);

typedef struct {
    uint64_t hits, misses, transferred_bytes, persistent_bytes;
    int last_update_step;      /* HeadCacheStats.last_update_step */
    int entry_last_update_step;
    int labels_valid;
    int window_held_tokens;
    int persistent;
    int n_history;
} orc_head_state;

/* entry_indices [k] (may be NULL), history [steps] (may be NULL),
 * entry_k_rows/entry_v_rows [k][d] (may be NULL). */
int orc_engine_head_state(const orc_engine* e, int l, int g, orc_head_state* st,
                          int* entry_indices, double* history, double* entry_k_rows,
                          double* entry_v_rows);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
