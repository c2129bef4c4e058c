// ref_shim.cpp — C entry points over the UNMODIFIED reference library
// (kvsim, compiled in place from /root/reference/proj/src by oracle/Makefile).
//
// TEST INFRASTRUCTURE ONLY. Links into oracle/_ref/libkvsim_ref.so, which is
// loaded by tests/ (to pin the C restatement and the CUDA path against the
// reference itself) and by bench.py's cpu_baseline / --impl reference legs.
// Nothing here re-implements reference logic: every entry point calls the
// reference function named in its comment and maps its exceptions to the
// status codes of errors.hpp:10-41.
#include <algorithm>
#include <chrono>
#include <memory>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "kvsim/attention.hpp"
#include "kvsim/engine.hpp"
#include "kvsim/errors.hpp"
#include "kvsim/head_profile.hpp"
#include "kvsim/retrieval.hpp"
#include "kvsim/rng.hpp"
#include "kvsim/similarity_cache.hpp"
#include "kvsim/synthetic_model.hpp"
#include "kvsim/trace_io.hpp"
#include "kvsim/profiler.hpp"

using namespace kvsim;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const ArgumentError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const IndexError& e) {
        g_err = e.what();
        return 4;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 5;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 6;
    } catch (const IoError& e) {
        g_err = e.what();
        return 7;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 8;
    }
}

Matrix to_matrix(const double* p, int rows, int cols) {
    Matrix m(rows, cols);
    std::copy(p, p + static_cast<size_t>(rows) * cols, m.data.begin());
    return m;
}

// StepSource over caller arrays (synthetic_model.hpp:16-28 interface).
// prompt_k/v [L][hkv][n_prompt][d]; true_q/approx_q [(steps+1)][L][hq][d];
// new_k/new_v [steps][L][hkv][d] for t = 1..steps.
class ArraySource : public StepSource {
  public:
    ArraySource(const ModelShape& shape, int n_prompt, int steps, const double* pk,
                const double* pv, const double* tq, const double* aq, const double* nk,
                const double* nv)
        : shape_(shape), n_prompt_(n_prompt), steps_(steps), tq_(tq), aq_(aq), nk_(nk), nv_(nv) {
        const int L = shape.num_layers, H = shape.num_kv_heads, d = shape.head_dim;
        pk_.resize(L);
        pv_.resize(L);
        for (int l = 0; l < L; ++l)
            for (int g = 0; g < H; ++g) {
                size_t off = (static_cast<size_t>(l) * H + g) * static_cast<size_t>(n_prompt) * d;
                pk_[l].push_back(to_matrix(pk + off, n_prompt, d));
                pv_[l].push_back(to_matrix(pv + off, n_prompt, d));
            }
    }
    const ModelShape& shape() const override { return shape_; }
    int prompt_tokens() const override { return n_prompt_; }
    int decode_steps() const override { return steps_; }
    const Matrix& prompt_k(int l, int g) const override { return pk_[l][g]; }
    const Matrix& prompt_v(int l, int g) const override { return pv_[l][g]; }
    std::span<const double> true_query(int t, int l, int h) const override { return q(tq_, t, l, h); }
    std::span<const double> approx_query(int t, int l, int h) const override { return q(aq_, t, l, h); }
    std::span<const double> new_k_row(int t, int l, int g) const override { return row(nk_, t, l, g); }
    std::span<const double> new_v_row(int t, int l, int g) const override { return row(nv_, t, l, g); }

  private:
    std::span<const double> q(const double* base, int t, int l, int h) const {
        const int d = shape_.head_dim;
        size_t off = ((static_cast<size_t>(t) * shape_.num_layers + l) * shape_.num_q_heads + h) * d;
        return {base + off, static_cast<size_t>(d)};
    }
    std::span<const double> row(const double* base, int t, int l, int g) const {
        const int d = shape_.head_dim;
        size_t off = ((static_cast<size_t>(t - 1) * shape_.num_layers + l) * shape_.num_kv_heads + g) * d;
        return {base + off, static_cast<size_t>(d)};
    }
    ModelShape shape_;
    int n_prompt_, steps_;
    const double *tq_, *aq_, *nk_, *nv_;
    std::vector<std::vector<Matrix>> pk_, pv_;
};

}  // namespace

extern "C" {

typedef struct {
    int num_layers, num_q_heads, num_kv_heads, head_dim, bytes_per_element;
    int k, sink_tokens, recent_tokens;
    int retriever;
    int hash_bits;
    uint64_t retriever_seed;
    int policy;
    int always_miss, always_hit, has_tau_override;
    double tau_override;
    int n_prompt, steps;
} ref_engine_cfg;  // field-for-field the oracle's orc_engine_cfg

const char* ref_last_error() { return g_err.c_str(); }

void ref_fill_normal(uint64_t seed, double* out, size_t n) {  // rng.hpp:24-27
    std::mt19937_64 gen(seed);
    fill_normal(gen, std::span<double>(out, n));
}

uint64_t ref_mix_seed3(uint64_t base, uint64_t a, uint64_t b) { return mix_seed(base, a, b); }

int ref_cosine_similarity(const double* a, const double* b, int n, double* value, int* degenerate) {
    return guarded([&] {  // attention.cpp:155-168
        CosineResult r = cosine_similarity({a, static_cast<size_t>(n)}, {b, static_cast<size_t>(n)});
        *value = r.value;
        *degenerate = r.degenerate;
    });
}

int ref_aggregate_similarity(const double* sims, const double* w, int m, double* out) {
    return guarded([&] {  // similarity_cache.cpp:10-27
        *out = aggregate_similarity({sims, static_cast<size_t>(m)}, {w, static_cast<size_t>(m)});
    });
}

int ref_lookup(double* labels, int* label_valid, const double* queries, const double* weights,
               int m, int d, double tau, int* hit, double* aggregated, double* sims,
               int* reason) {
    return guarded([&] {  // similarity_cache.cpp:29-72
        std::vector<QueryLabel> lab(m);
        std::vector<std::vector<double>> qs(m);
        for (int j = 0; j < m; ++j) {
            lab[j].q.assign(labels + static_cast<size_t>(j) * d, labels + static_cast<size_t>(j + 1) * d);
            lab[j].valid = label_valid[j] != 0;
            qs[j].assign(queries + static_cast<size_t>(j) * d, queries + static_cast<size_t>(j + 1) * d);
        }
        LookupResult r = lookup(lab, qs, {weights, static_cast<size_t>(m)}, tau);
        *hit = r.hit;
        *aggregated = r.aggregated;
        *reason = static_cast<int>(r.reason);
        for (int j = 0; j < m; ++j) {
            sims[j] = r.sims[j];
            label_valid[j] = lab[j].valid;
            std::copy(lab[j].q.begin(), lab[j].q.end(), labels + static_cast<size_t>(j) * d);
        }
    });
}

int ref_encode_sign_hash(const double* keys, int n, int d, int hash_bits, uint64_t seed,
                         double* projection_out, uint64_t* bits_out) {
    return guarded([&] {  // retrieval.cpp:60-78
        Matrix k = to_matrix(keys, n, d);
        RetrievalMetadata meta = encode(k, RetrieverVariant::kSignHash, hash_bits, seed);
        std::copy(meta.projection.data.begin(), meta.projection.data.end(), projection_out);
        std::copy(meta.bits.begin(), meta.bits.end(), bits_out);
    });
}

int ref_retrieve_scored(const double* q, int d, int variant, const double* keys, int n, int k,
                        int hash_bits, uint64_t seed, int* out_idx, double* out_score) {
    return guarded([&] {  // retrieval.cpp:90-125 (sign-hash metadata built by encode :60-78)
        Matrix km = to_matrix(keys, n, d);
        RetrievalMetadata meta = encode(km, variant == 0 ? RetrieverVariant::kExact
                                                         : RetrieverVariant::kSignHash,
                                        hash_bits, seed);
        std::vector<ScoredIndex> r = retrieve_scored({q, static_cast<size_t>(d)}, meta, k);
        for (size_t i = 0; i < r.size(); ++i) {
            out_idx[i] = r[i].index;
            out_score[i] = r[i].score;
        }
    });
}

int ref_topk_select_exact(const double* q, const double* keys, int n, int d, int k, int* out) {
    return guarded([&] {  // attention.cpp:71-89
        std::vector<int> r = topk_select_exact({q, static_cast<size_t>(d)}, to_matrix(keys, n, d), k);
        std::copy(r.begin(), r.end(), out);
    });
}

int ref_merge_group_topk(const int* sizes, int m, const int* idx, const double* score, int k,
                         int* out) {
    return guarded([&] {  // similarity_cache.cpp:180-201
        std::vector<std::vector<ScoredIndex>> props(m);
        size_t pos = 0;
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < sizes[j]; ++i, ++pos) props[j].push_back({idx[pos], score[pos]});
        std::vector<int> r = merge_group_topk(props, k);
        std::copy(r.begin(), r.end(), out);
    });
}

int ref_topk_attention(const double* q, const double* keys, const double* values, int n, int d,
                       const int* idx, int nidx, double* out) {
    return guarded([&] {  // attention.cpp:91-105
        AttentionOutput r = topk_attention({q, static_cast<size_t>(d)}, to_matrix(keys, n, d),
                                           to_matrix(values, n, d),
                                           {idx, static_cast<size_t>(nidx)});
        std::copy(r.values.begin(), r.values.end(), out);
    });
}

int ref_sink_recent_indices(int n, int sink, int recent, int* out, int* count, int* clamped) {
    return guarded([&] {  // attention.cpp:107-128
        bool c = false;
        std::vector<int> r = sink_recent_indices(n, sink, recent, &c);
        std::copy(r.begin(), r.end(), out);
        *count = static_cast<int>(r.size());
        *clamped = c;
    });
}

int ref_compute_threshold(double s, double eta, double p, double* tau) {
    return guarded([&] { *tau = compute_threshold(s, eta, p); });  // head_profile.cpp:17-25
}

int ref_plan_partition(const double* difficulty, int L, int H, double t_comp_s, double pcie_bw,
                       double mem_head_bytes, uint64_t persist_bytes_per_head,
                       uint64_t hbm_budget_bytes, int* persistent_out, int* n_p_out,
                       int* n_dropped_out) {
    return guarded([&] {  // head_profile.cpp:80-154
        HeadProfiles profiles(L, std::vector<HeadProfileEntry>(H));
        for (int l = 0; l < L; ++l)
            for (int h = 0; h < H; ++h) profiles[l][h].difficulty = difficulty[l * H + h];
        PartitionCosts costs;
        costs.t_comp_s = t_comp_s;
        costs.pcie_bw = pcie_bw;
        costs.mem_head_bytes = mem_head_bytes;
        costs.persist_bytes_per_head = persist_bytes_per_head;
        costs.hbm_budget_bytes = hbm_budget_bytes;
        PartitionPlan plan = plan_partition(profiles, costs);
        std::fill(persistent_out, persistent_out + L * H, 0);
        for (int l = 0; l < L; ++l)
            for (int h : plan.layers[l].persistent_heads) persistent_out[l * H + h] = 1;
        *n_p_out = plan.n_p;
        *n_dropped_out = static_cast<int>(plan.budget_dropped.size());
    });
}

uint64_t ref_cache_bytes(int offloaded, int entry_k, int held, int L, int hq, int d, int e) {
    return cache_bytes(offloaded, entry_k, held, L, hq, d, e);  // similarity_cache.cpp:167-178
}

static bool g_oracle_error = false;  // EngineConfig::compute_oracle_error for the next runs

void ref_set_compute_oracle_error(int on) { g_oracle_error = on != 0; }

static EngineConfig engine_config_of(const ref_engine_cfg* c) {
    EngineConfig cfg;
    cfg.shape = ModelShape{c->num_layers, c->num_q_heads, c->num_kv_heads, c->head_dim,
                           c->bytes_per_element};
    cfg.k = c->k;
    cfg.sink_tokens = c->sink_tokens;
    cfg.recent_tokens = c->recent_tokens;
    cfg.retriever = c->retriever == 0 ? RetrieverVariant::kExact : RetrieverVariant::kSignHash;
    cfg.hash_bits = c->hash_bits;
    cfg.retriever_seed = c->retriever_seed;
    cfg.policy = static_cast<Policy>(c->policy);
    cfg.mode.always_miss = c->always_miss;
    cfg.mode.always_hit = c->always_hit;
    if (c->has_tau_override) cfg.mode.tau_override = c->tau_override;
    cfg.collect_outputs = true;
    cfg.compute_oracle_error = g_oracle_error;
    return cfg;
}

// Full reference DecodeEngine run (engine.cpp:163-415) over caller arrays.
// outputs [steps][L][hq][d]; json_buf receives cache_state_json()
// (engine.cpp:464-530); step_seconds [steps] = steady_clock per decode_step.
int ref_run_engine(const ref_engine_cfg* c, const double* tau, const double* q_importance,
                   const int* persistent, const double* prompt_k, const double* prompt_v,
                   const double* true_q, const double* approx_q, const double* new_k,
                   const double* new_v, double* outputs, char* json_buf, size_t json_cap,
                   double* step_seconds) {
    return guarded([&] {
        EngineConfig cfg = engine_config_of(c);
        const int L = c->num_layers, H = c->num_kv_heads, m = c->num_q_heads / c->num_kv_heads;
        ArraySource src(cfg.shape, c->n_prompt, c->steps, prompt_k, prompt_v, true_q, approx_q,
                        new_k, new_v);
        HeadProfiles profiles(L, std::vector<HeadProfileEntry>(H));
        PartitionPlan plan;
        plan.layers.resize(L);
        for (int l = 0; l < L; ++l)
            for (int g = 0; g < H; ++g) {
                HeadProfileEntry& e = profiles[l][g];
                e.q_importance.assign(q_importance + (static_cast<size_t>(l) * H + g) * m,
                                      q_importance + (static_cast<size_t>(l) * H + g + 1) * m);
                e.tau = tau[l * H + g];
                if (persistent[l * H + g]) plan.layers[l].persistent_heads.push_back(g);
            }
        DecodeEngine engine(cfg, profiles, plan, src);
        engine.prefill();
        for (int t = 0; t < c->steps; ++t) {
            auto t0 = std::chrono::steady_clock::now();
            engine.decode_step();
            auto t1 = std::chrono::steady_clock::now();
            if (step_seconds) step_seconds[t] = std::chrono::duration<double>(t1 - t0).count();
        }
        if (outputs) {
            const auto& outs = engine.collected_outputs();
            const int hq = c->num_q_heads, d = c->head_dim;
            for (int t = 0; t < c->steps; ++t)
                for (int l = 0; l < L; ++l)
                    for (int h = 0; h < hq; ++h) {
                        auto r = outs[t][l].row_span(h);
                        std::copy(r.begin(), r.end(),
                                  outputs + ((static_cast<size_t>(t) * L + l) * hq + h) * d);
                    }
        }
        if (json_buf && json_cap) {
            std::string js = engine.cache_state_json();
            size_t n = std::min(js.size(), json_cap - 1);
            std::memcpy(json_buf, js.data(), n);
            json_buf[n] = 0;
        }
    });
}

// Timed CPU baseline: `threads` independent reference engines, each one
// (sequence, layer, KV-head) unit of the workload (1 layer, one GQA group of
// m query heads, offloaded, similarity policy), run concurrently the way the
// reference runner runs independent engines on a std::thread pool
// (runner.cpp:186-278). Inputs are caller arrays shared by all threads.
// The first `warmup` decode steps are untimed. Returns per-thread mean seconds
// per timed decode_step in sec_per_step[threads] and the prefill seconds in
// prefill_seconds[threads].
int ref_bench_units(const ref_engine_cfg* c, const double* tau, const double* q_importance,
                    const double* prompt_k, const double* prompt_v, const double* true_q,
                    const double* approx_q, const double* new_k, const double* new_v,
                    int threads, int warmup, double* sec_per_step, double* prefill_seconds) {
    std::vector<int> status(threads, 0);
    std::vector<std::string> errs(threads);
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&, w] {
            status[w] = guarded([&] {
                EngineConfig cfg = engine_config_of(c);
                cfg.collect_outputs = false;
                ArraySource src(cfg.shape, c->n_prompt, c->steps, prompt_k, prompt_v, true_q,
                                approx_q, new_k, new_v);
                HeadProfiles profiles(1, std::vector<HeadProfileEntry>(1));
                // thread w serves one (layer, kv head) unit with that head's profile
                profiles[0][0].q_importance.assign(q_importance + (size_t)w * c->num_q_heads,
                                                   q_importance + (size_t)(w + 1) * c->num_q_heads);
                profiles[0][0].tau = tau[w];
                PartitionPlan plan;
                plan.layers.resize(1);
                DecodeEngine engine(cfg, profiles, plan, src);
                auto p0 = std::chrono::steady_clock::now();
                engine.prefill();
                auto p1 = std::chrono::steady_clock::now();
                prefill_seconds[w] = std::chrono::duration<double>(p1 - p0).count();
                for (int t = 0; t < warmup; ++t) engine.decode_step();
                auto t0 = std::chrono::steady_clock::now();
                for (int t = warmup; t < c->steps; ++t) engine.decode_step();
                auto t1 = std::chrono::steady_clock::now();
                sec_per_step[w] = std::chrono::duration<double>(t1 - t0).count() / (c->steps - warmup);
            });
            if (status[w]) errs[w] = g_err;
        });
    for (auto& th : pool) th.join();
    for (int w = 0; w < threads; ++w)
        if (status[w]) {
            g_err = errs[w];
            return status[w];
        }
    return 0;
}


// --- trace wire format (trace_io.cpp) -------------------------------------
// record_trace(SyntheticModel(cfg), width) + write_trace(path): a trace made
// by the reference's own generator and writer.
int ref_record_synthetic_trace(int L, int hq, int hkv, int d, int d_model, int n_prompt, int steps,
                               double sigma_step, double sigma_layer, uint64_t seed, int tie, int width,
                               const char* path) {
    return guarded([&] {
        SyntheticConfig cfg;
        cfg.shape = ModelShape{L, hq, hkv, d, 2};
        cfg.d_model = d_model;
        cfg.n_prompt = n_prompt;
        cfg.steps = steps;
        cfg.sigma_step = sigma_step;
        cfg.sigma_layer = sigma_layer;
        cfg.seed = seed;
        cfg.tie_layer_weights = tie != 0;
        SyntheticModel model(cfg);
        write_trace(path, record_trace(model, width));
    });
}

// read_trace(path) widened to double in file order: hdr[7] = L, hq, hkv, d,
// n_prompt, n_steps, width; prompt [L][hkv][2][n][d], hidden [S+1][L][hq*d],
// step [S][L][2][hkv][d] (each may be NULL).
int ref_read_trace(const char* path, int* hdr, double* prompt, double* hidden, double* step) {
    return guarded([&] {
        TraceData t = read_trace(path);
        const int L = t.shape.num_layers, H = t.shape.num_kv_heads, d = t.shape.head_dim;
        const int hq = t.shape.num_q_heads, n = t.n_prompt, S = t.n_steps;
        const int h7[7] = {L, hq, H, d, n, S, t.element_width};
        std::copy(h7, h7 + 7, hdr);
        for (int l = 0; prompt && l < L; ++l)
            for (int g = 0; g < H; ++g) {
                double* o = prompt + ((size_t)l * H + g) * 2 * n * d;
                std::copy(t.prompt_k[l][g].data.begin(), t.prompt_k[l][g].data.end(), o);
                std::copy(t.prompt_v[l][g].data.begin(), t.prompt_v[l][g].data.end(), o + (size_t)n * d);
            }
        for (int s = 0; hidden && s <= S; ++s)
            for (int l = 0; l < L; ++l)
                std::copy(t.hidden[s][l].begin(), t.hidden[s][l].end(), hidden + ((size_t)s * L + l) * hq * d);
        for (int s = 0; step && s < S; ++s)
            for (int l = 0; l < L; ++l) {
                double* o = step + ((size_t)s * L + l) * 2 * H * d;
                std::copy(t.step_k[s][l].data.begin(), t.step_k[s][l].data.end(), o);
                std::copy(t.step_v[s][l].data.begin(), t.step_v[s][l].data.end(), o + (size_t)H * d);
            }
    });
}

// DecodeEngine over TraceSource(read_trace(path)) — the reference replaying a
// trace (c->n_prompt / c->steps are taken from the trace).
int ref_run_engine_trace(const ref_engine_cfg* c, const double* tau, const double* q_importance,
                         const int* persistent, const char* path, double* outputs, char* json_buf,
                         size_t json_cap) {
    return guarded([&] {
        EngineConfig cfg = engine_config_of(c);
        TraceSource src(read_trace(path));
        const int L = c->num_layers, H = c->num_kv_heads, m = c->num_q_heads / c->num_kv_heads;
        HeadProfiles profiles(L, std::vector<HeadProfileEntry>(H));
        PartitionPlan plan;
        plan.layers.resize(L);
        for (int l = 0; l < L; ++l)
            for (int g = 0; g < H; ++g) {
                HeadProfileEntry& e = profiles[l][g];
                e.q_importance.assign(q_importance + (static_cast<size_t>(l) * H + g) * m,
                                      q_importance + (static_cast<size_t>(l) * H + g + 1) * m);
                e.tau = tau[l * H + g];
                if (persistent[l * H + g]) plan.layers[l].persistent_heads.push_back(g);
            }
        DecodeEngine engine(cfg, profiles, plan, src);
        engine.prefill();
        const int steps = src.decode_steps();
        for (int t = 0; t < steps; ++t) engine.decode_step();
        if (outputs) {
            const auto& outs = engine.collected_outputs();
            const int hq = c->num_q_heads, d = c->head_dim;
            for (int t = 0; t < steps; ++t)
                for (int l = 0; l < L; ++l)
                    for (int h = 0; h < hq; ++h) {
                        auto r = outs[t][l].row_span(h);
                        std::copy(r.begin(), r.end(), outputs + ((static_cast<size_t>(t) * L + l) * hq + h) * d);
                    }
        }
        if (json_buf && json_cap) {
            std::string js = engine.cache_state_json();
            size_t nn = std::min(js.size(), json_cap - 1);
            std::memcpy(json_buf, js.data(), nn);
            json_buf[nn] = 0;
        }
    });
}


// profile_heads (profiler.cpp:19-125) over TraceSources of the given trace
// files. provided [L][H][m] may be NULL (blend fit). Outputs: q_importance
// [L][H][m], kv_importance / s_hat / tau / difficulty [L][H].
int ref_profile_heads(const char* const* paths, int n_paths, int blend_sequences, int blend_steps, int topk,
                      int sink, int recent, double eta, double p, double epsilon, const double* provided,
                      double* q_importance, double* kv_importance, double* s_hat, double* tau, double* difficulty) {
    return guarded([&] {
        std::vector<std::unique_ptr<TraceSource>> owned;
        ProfilerInputs in;
        for (int i = 0; i < n_paths; ++i) {
            owned.push_back(std::make_unique<TraceSource>(read_trace(paths[i])));
            in.sources.push_back(owned.back().get());
        }
        in.blend_sequences = blend_sequences;
        in.blend_steps = blend_steps;
        in.topk = topk;
        in.sink_tokens = sink;
        in.recent_tokens = recent;
        in.eta = eta;
        in.p = p;
        in.epsilon = epsilon;
        const ModelShape& sh = owned.front()->shape();
        const int L = sh.num_layers, H = sh.num_kv_heads, m = sh.num_q_heads / sh.num_kv_heads;
        if (provided) {
            in.provided_importance.assign(L, std::vector<std::vector<double>>(H, std::vector<double>(m)));
            for (int l = 0; l < L; ++l)
                for (int g = 0; g < H; ++g)
                    for (int j = 0; j < m; ++j) in.provided_importance[l][g][j] = provided[((size_t)l * H + g) * m + j];
        }
        HeadProfiles prof = profile_heads(in);
        for (int l = 0; l < L; ++l)
            for (int g = 0; g < H; ++g) {
                const HeadProfileEntry& e = prof[l][g];
                for (int j = 0; j < m; ++j) q_importance[((size_t)l * H + g) * m + j] = e.q_importance[j];
                kv_importance[l * H + g] = e.kv_importance;
                s_hat[l * H + g] = e.s_hat;
                tau[l * H + g] = e.tau;
                difficulty[l * H + g] = e.difficulty;
            }
    });
}

}  // extern "C"
