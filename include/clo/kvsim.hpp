// clo/kvsim.hpp — header-only C++ shim that re-exposes the reference's kvsim
// API names (engine.hpp, retrieval.hpp, similarity_cache.hpp, attention.hpp,
// head_profile.hpp, errors.hpp) over the C-ABI in <clo.h>, so runner-style
// callers written against kvsim compile against the B200 library by swapping
// the include and the namespace.
//
// Status codes are rethrown as the matching exception type (errors.hpp:10-41).
#pragma once

#include <clo.h>

#include <algorithm>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace clo::kvsim {

// ---- errors.hpp:10-41 -----------------------------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error { using Error::Error; };
struct ArgumentError : Error { using Error::Error; };
struct NumericError : Error { using Error::Error; };
struct IndexError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

inline void check(clo_status s) {
    if (s == CLO_OK) return;
    const std::string m = clo_last_error();
    switch (s) {
        case CLO_ERR_SHAPE: throw ShapeError(m);
        case CLO_ERR_ARGUMENT: throw ArgumentError(m);
        case CLO_ERR_NUMERIC: throw NumericError(m);
        case CLO_ERR_INDEX: throw IndexError(m);
        case CLO_ERR_CONTRACT: throw ContractError(m);
        case CLO_ERR_CONFIG: throw ConfigError(m);
        case CLO_ERR_IO: throw IoError(m);
        case CLO_ERR_CUDA: throw CudaError(m);
        default: throw Error(m);
    }
}

// ---- matrix.hpp:46-66 / engine.hpp:19-49 ------------------------------------
using ModelShape = clo_model_shape;
enum class Policy { kSimilarity = CLO_POLICY_SIMILARITY, kLru = CLO_POLICY_LRU, kLfu = CLO_POLICY_LFU,
                    kPrefetchOnly = CLO_POLICY_PREFETCH_ONLY };
enum class RetrieverVariant { kExact = CLO_RETRIEVER_EXACT, kSignHash = CLO_RETRIEVER_SIGN_HASH };
enum class SyncMode { kCpuCentric = CLO_SYNC_CPU_CENTRIC, kGpuCentric = CLO_SYNC_GPU_CENTRIC };
enum class Placement { kOffloaded = CLO_PLACEMENT_OFFLOADED, kPersistent = CLO_PLACEMENT_PERSISTENT };

struct ModeFlags {
    bool always_miss = false;
    bool always_hit = false;
    std::optional<double> tau_override;
};

struct EngineConfig {
    ModelShape shape{};
    int k = 0;
    int sink_tokens = 4;
    int recent_tokens = 64;
    RetrieverVariant retriever = RetrieverVariant::kExact;
    int hash_bits = 256;
    uint64_t retriever_seed = 1;
    Policy policy = Policy::kSimilarity;
    ModeFlags mode;
    std::optional<SyncMode> sync_override;
    bool collect_outputs = false;
    bool compute_oracle_error = true;  // engine.hpp:48 (output_error.cu; reads every key each step)
    // B200
    int batch = 1;
    int kv_dtype = CLO_DTYPE_BF16;
    int kv_head_offset = 0;
    int device = 0;
    int victim_rows = -1;  // HBM rows kept per offloaded head beyond the entry (-1: auto = 8k, HBM-capped)

    clo_engine_config to_c(int n_prompt, int max_steps) const {
        clo_engine_config c;
        clo_engine_config_defaults(&c);
        c.shape = shape;
        c.k = k;
        c.sink_tokens = sink_tokens;
        c.recent_tokens = recent_tokens;
        c.retriever = static_cast<int>(retriever);
        c.hash_bits = hash_bits;
        c.retriever_seed = retriever_seed;
        c.policy = static_cast<int>(policy);
        c.always_miss = mode.always_miss;
        c.always_hit = mode.always_hit;
        c.has_tau_override = mode.tau_override.has_value();
        c.tau_override = mode.tau_override.value_or(0.0);
        c.sync_override = sync_override ? static_cast<int>(*sync_override) : -1;
        c.collect_outputs = collect_outputs;
        c.compute_oracle_error = compute_oracle_error;
        c.batch = batch;
        c.n_prompt = n_prompt;
        c.max_steps = max_steps;
        c.kv_dtype = kv_dtype;
        c.kv_head_offset = kv_head_offset;
        c.device = device;
        c.victim_rows = victim_rows;
        return c;
    }
};

// head_profile.hpp:16-23, 85-97
struct HeadProfileEntry {
    std::vector<double> q_importance;
    double kv_importance = 0.0;
    double s_hat = 0.0;
    double tau = -1.0;
    double difficulty = 0.0;
    Placement placement = Placement::kOffloaded;
};
using HeadProfiles = std::vector<std::vector<HeadProfileEntry>>;
struct LayerPartition {
    int n_d = 0;
    int n_persist = 0;
    std::vector<int> persistent_heads;
};
struct PartitionPlan {
    int n_p = 0;
    std::vector<LayerPartition> layers;
};

// ---- DecodeEngine (engine.hpp:91-139) -------------------------------------
// The StepSource is replaced by explicit per-step inputs (device or host
// buffers), since the step data lives on the GPU.
// PipelineTimeline (pipeline_sim.hpp:74-86), measured on the device.
struct PipelineTimeline {
    std::vector<clo_layer_timing> per_layer;
    clo_layer_timing totals{};
    uint64_t steps = 0;
    double share(double part_s) const { return totals.total_s > 0.0 ? part_s / totals.total_s : 0.0; }
};

class DecodeEngine {
  public:
    DecodeEngine(const EngineConfig& cfg, const HeadProfiles& profiles, const PartitionPlan& plan,
                 int n_prompt, int decode_steps)
        : cfg_(cfg) {
        const int L = cfg.shape.num_layers, H = cfg.shape.num_kv_heads;
        const int m = cfg.shape.num_kv_heads ? cfg.shape.num_q_heads / cfg.shape.num_kv_heads : 0;
        if (static_cast<int>(profiles.size()) != L) throw ArgumentError("profiles must cover every layer");
        if (static_cast<int>(plan.layers.size()) != L) throw ArgumentError("partition plan must cover every layer");
        std::vector<double> tau, qimp;
        std::vector<int> pers(static_cast<size_t>(L) * H, 0);
        for (int l = 0; l < L; ++l) {
            if (static_cast<int>(profiles[l].size()) != H) throw ArgumentError("profiles must cover every KV head");
            for (const auto& e : profiles[l]) {
                if (static_cast<int>(e.q_importance.size()) != m)
                    throw ArgumentError("profile importance width must equal the group size");
                tau.push_back(e.tau);
                qimp.insert(qimp.end(), e.q_importance.begin(), e.q_importance.end());
            }
            for (int g : plan.layers[l].persistent_heads) {
                if (g < 0 || g >= H) throw ArgumentError("partition plan names a KV head outside the model");
                pers[static_cast<size_t>(l) * H + g] = 1;
            }
        }
        const clo_engine_config c = cfg.to_c(n_prompt, decode_steps);
        check(clo_engine_create(&c, tau.data(), qimp.data(), pers.data(), &e_));
    }
    ~DecodeEngine() { clo_engine_destroy(e_); }
    DecodeEngine(const DecodeEngine&) = delete;
    DecodeEngine& operator=(const DecodeEngine&) = delete;

    void bind_host_kv(void* k, void* v, int64_t seq_stride, int64_t layer_stride, int64_t head_stride,
                      int64_t row_stride = 0) {
        check(row_stride ? clo_engine_bind_host_kv_ex(e_, k, v, seq_stride, layer_stride, head_stride, row_stride)
                         : clo_engine_bind_host_kv(e_, k, v, seq_stride, layer_stride, head_stride));
    }
    void prefill(const float* true_q0, bool on_host = true, void* stream = nullptr) {
        check(clo_prefill(e_, true_q0, on_host, stream));
    }
    void decode_step(const clo_step_io& io, void* stream = nullptr) { check(clo_decode_step(e_, &io, stream)); }
    clo_metrics metrics() const {
        clo_metrics m;
        check(clo_get_metrics(e_, &m));
        return m;
    }
    SyncMode sync_mode() const { return static_cast<SyncMode>(metrics().sync_mode); }
    uint64_t host_bytes() const { return metrics().host_bytes; }
    uint64_t device_persistent_bytes() const { return metrics().device_persistent_bytes; }
    uint64_t modeled_cache_bytes() const { return metrics().cache_bytes_current; }
    clo_head_state head(int layer, int kv_head, int seq = 0, std::vector<int32_t>* entry = nullptr,
                        std::vector<double>* history = nullptr) const {
        clo_head_state st;
        if (entry) entry->resize(cfg_.k);
        if (history) history->resize(1u << 16);
        check(clo_get_head_state(e_, seq, layer, kv_head, &st, entry ? entry->data() : nullptr,
                                 history ? history->data() : nullptr));
        if (history) history->resize(st.n_history);
        return st;
    }
    std::string cache_state_json(int seq = 0) const {
        size_t need = 0;
        check(clo_cache_state_json(e_, seq, nullptr, 0, &need));
        std::string s(need, '\0');
        check(clo_cache_state_json(e_, seq, s.data(), need, &need));
        s.resize(need ? need - 1 : 0);
        return s;
    }
    // DecodeEngine::timeline() (engine.hpp:105): a decode step that also
    // measures the per-layer LayerTiming breakdown, and the accumulated result.
    void decode_step_timed(const clo_step_io& io, void* stream = nullptr) {
        check(clo_engine_timeline_step(e_, &io, stream));
    }
    PipelineTimeline timeline() const {
        PipelineTimeline tl;
        tl.per_layer.resize(cfg_.shape.num_layers);
        check(clo_get_timeline(e_, tl.per_layer.data(), (int)tl.per_layer.size(), &tl.totals, &tl.steps));
        return tl;
    }
    std::string timeline_json() const {  // breakdown_to_json (pipeline_sim.cpp:115-135)
        size_t need = 0;
        check(clo_timeline_json(e_, nullptr, 0, &need));
        std::string s(need, '\0');
        check(clo_timeline_json(e_, s.data(), need, &need));
        s.resize(need ? need - 1 : 0);
        return s;
    }
    // KV-head sharding: the fused head-output all-gather (include/clo.h).
    std::vector<char> exchange_handle(int rank, int world) {
        std::vector<char> h(CLO_EXCHANGE_HANDLE_BYTES);
        check(clo_engine_exchange_handle(e_, rank, world, h.data()));
        return h;
    }
    void attach_peers(const std::vector<char>& handles_in_rank_order) {
        check(clo_engine_attach_peers(e_, handles_in_rank_order.data()));
    }
    clo_engine* handle() const { return e_; }

  private:
    EngineConfig cfg_;
    clo_engine* e_ = nullptr;
};

// ---- pure functions ---------------------------------------------------------
inline double compute_threshold(double s, double eta, double p) {  // head_profile.cpp:17-25
    double tau;
    check(clo_compute_threshold(s, eta, p, &tau));
    return tau;
}
inline double compute_difficulty(double tau, double s_hat, double epsilon) {
    double d;
    check(clo_compute_difficulty(tau, s_hat, epsilon, &d));
    return d;
}
inline std::vector<int> sink_recent_indices(int n, int sink, int recent, bool* clamped = nullptr) {
    std::vector<int32_t> out(static_cast<size_t>(std::max(0, std::min(n, sink)) + std::max(0, std::min(n, recent))) + 1);
    int count = 0, cl = 0;
    check(clo_sink_recent_indices(n, sink, recent, out.data(), &count, &cl));
    if (clamped) *clamped = cl;
    return {out.begin(), out.begin() + count};
}
inline uint64_t cache_bytes(int offloaded, int entry_k, int held, int L, int hq, int d, int e) {
    return clo_cache_bytes(offloaded, entry_k, held, L, hq, d, e);
}

// ---- traces (trace_io.hpp:41-64) --------------------------------------------
// TraceSource over libclo's reader; rows converted to the engine's storage type.
class TraceSource {
  public:
    explicit TraceSource(const std::string& path) { check(clo_trace_open(path.c_str(), &t_)); }
    ~TraceSource() { clo_trace_close(t_); }
    TraceSource(const TraceSource&) = delete;
    TraceSource& operator=(const TraceSource&) = delete;
    ModelShape shape() const {
        clo_model_shape s{};
        check(clo_trace_info(t_, &s, nullptr, nullptr, nullptr));
        return ModelShape{s.num_layers, s.num_q_heads, s.num_kv_heads, s.head_dim, s.bytes_per_element};
    }
    int prompt_tokens() const {
        int n = 0;
        check(clo_trace_info(t_, nullptr, &n, nullptr, nullptr));
        return n;
    }
    int decode_steps() const {
        int n = 0;
        check(clo_trace_info(t_, nullptr, nullptr, &n, nullptr));
        return n;
    }
    // prompt K/V rows of (layer, kv_head) as `dtype` (clo_dtype)
    void prompt(int layer, int kv_head, int dtype, void* k_out, void* v_out) const {
        check(clo_trace_prompt(t_, layer, kv_head, dtype, k_out, v_out));
    }
    // step t in the engine's clo_step_io layout (queries f32, rows `dtype`)
    void step(int t, float* true_q, float* approx_q, void* new_k, void* new_v, int dtype) const {
        check(clo_trace_step(t_, t, true_q, approx_q, new_k, new_v, dtype));
    }
    const clo_trace* handle() const { return t_; }

  private:
    clo_trace* t_ = nullptr;
};

// ---- profiling (profiler.hpp:12-36) -----------------------------------------
inline std::vector<std::vector<clo_head_profile>> profile_heads(const std::vector<const TraceSource*>& sources,
                                                                const clo_profiler_config& cfg,
                                                                const double* provided_importance = nullptr) {
    std::vector<const clo_trace*> h;
    for (const TraceSource* s : sources) h.push_back(s->handle());
    const ModelShape sh = sources.at(0)->shape();
    std::vector<clo_head_profile> flat((size_t)sh.num_layers * sh.num_kv_heads);
    check(clo_profile_heads(h.data(), (int)h.size(), &cfg, provided_importance, flat.data()));
    std::vector<std::vector<clo_head_profile>> out(sh.num_layers);
    for (int l = 0; l < sh.num_layers; ++l)
        out[l].assign(flat.begin() + (size_t)l * sh.num_kv_heads, flat.begin() + (size_t)(l + 1) * sh.num_kv_heads);
    return out;
}

}  // namespace clo::kvsim
