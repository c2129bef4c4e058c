// Compiles a runner-style caller against the kvsim-named C++ shim
// (include/clo/kvsim.hpp) and exercises the host-side pure functions; engine
// creation must fail loudly (CudaError) when no GPU is present.
#include <clo/kvsim.hpp>

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

using namespace clo::kvsim;

// A runner-style decode through the shim (runner.cpp:227-253 shape of use):
// DecodeEngine over a trace (f32 KV in pinned host memory, host step
// buffers), layer 0 persistent, sign-hash similarity cache; writes
// cache_state_json(0) to `out` for the test to compare with the Python path.
// Profile: tau(l, g) = 0.55 + 0.1 * ((l + g) % 4), q_importance = 1 + j.
static int run_trace(const TraceSource& t, const char* out) {
    const ModelShape sh = t.shape();
    const int L = sh.num_layers, H = sh.num_kv_heads, HQ = sh.num_q_heads, d = sh.head_dim, m = HQ / H;
    const int n = t.prompt_tokens(), steps = t.decode_steps();
    EngineConfig cfg;
    cfg.shape = ModelShape{L, HQ, H, d, 4};
    cfg.k = n < 64 ? n : 64;
    cfg.retriever = RetrieverVariant::kSignHash;
    cfg.retriever_seed = 5;
    cfg.kv_dtype = CLO_DTYPE_F32;
    HeadProfiles profiles(L, std::vector<HeadProfileEntry>(H));
    for (int l = 0; l < L; ++l)
        for (int g = 0; g < H; ++g) {
            profiles[l][g].tau = 0.55 + 0.1 * ((l + g) % 4);
            for (int j = 0; j < m; ++j) profiles[l][g].q_importance.push_back(1.0 + j);
        }
    PartitionPlan plan;
    plan.layers.resize(L);
    for (int g = 0; g < H; ++g) plan.layers[0].persistent_heads.push_back(g);
    DecodeEngine engine(cfg, profiles, plan, n, steps);
    const size_t nmax = (size_t)n + steps, rows = (size_t)L * H * nmax * d;
    void *hk = nullptr, *hv = nullptr;
    if (clo_host_alloc(rows * 4, &hk) != CLO_OK || clo_host_alloc(rows * 4, &hv) != CLO_OK) return 20;
    for (int l = 0; l < L; ++l)
        for (int g = 0; g < H; ++g) {
            const size_t off = ((size_t)l * H + g) * nmax * d;
            t.prompt(l, g, CLO_DTYPE_F32, static_cast<float*>(hk) + off, static_cast<float*>(hv) + off);
        }
    engine.bind_host_kv(hk, hv, (int64_t)L * H * nmax * d, (int64_t)H * nmax * d, (int64_t)nmax * d);
    std::vector<float> tq((size_t)L * HQ * d), aq(tq.size()), nk((size_t)L * H * d), nv(nk.size()), o(tq.size());
    t.step(0, tq.data(), aq.data(), nullptr, nullptr, CLO_DTYPE_F32);
    engine.prefill(tq.data());
    for (int s = 1; s <= steps; ++s) {
        t.step(s, tq.data(), aq.data(), nk.data(), nv.data(), CLO_DTYPE_F32);
        clo_step_io io{tq.data(), aq.data(), nk.data(), nv.data(), o.data(), 1};
        engine.decode_step(io);
    }
    const std::string js = engine.cache_state_json(0);
    FILE* f = std::fopen(out, "w");
    if (!f) return 21;
    std::fwrite(js.data(), 1, js.size(), f);
    std::fclose(f);
    const clo_metrics mt = engine.metrics();
    std::printf("shim decode ok: %llu hits, %llu misses\n", (unsigned long long)mt.hits, (unsigned long long)mt.misses);
    clo_host_free(hk);
    clo_host_free(hv);
    return 0;
}

int main(int argc, char** argv) {
    const bool expect_gpu = argc > 1 && std::string(argv[1]) == "gpu";
    if (std::fabs(compute_threshold(0.5, 0.8, 3.0) - (-0.95164126255001177)) > 1e-15) return 1;
    bool clamped = false;
    auto w = sink_recent_indices(100, 4, 64, &clamped);
    if (w.size() != 68 || w[4] != 36 || clamped) return 2;
    if (cache_bytes(1, 1000, 0, 0, 0, 128, 2) != 512000) return 3;
    try {
        compute_threshold(2.0, 0.8, 3.0);
        return 4;
    } catch (const ArgumentError&) {
    }
    EngineConfig cfg;
    cfg.shape = ModelShape{2, 4, 2, 128, 2};
    cfg.k = 8;
    HeadProfiles profiles(2, std::vector<HeadProfileEntry>(2));
    for (auto& layer : profiles)
        for (auto& e : layer) e.q_importance = {1.0, 1.0};
    PartitionPlan plan;
    plan.layers.resize(2);
    plan.layers[0].persistent_heads = {0, 1};
    try {
        DecodeEngine engine(cfg, profiles, plan, 64, 4);
        if (!expect_gpu) return 5;
    } catch (const CudaError&) {
        if (expect_gpu) return 6;
    }
    // traces: a missing file is an IoError (read_trace, trace_io.cpp:129-131)
    try {
        TraceSource t("/nonexistent/trace.bin");
        return 7;
    } catch (const IoError&) {
    }
    if (argc > 2) {  // a trace path: shape and step accessors
        TraceSource t(argv[2]);
        const ModelShape sh = t.shape();
        std::vector<float> tq((size_t)sh.num_layers * sh.num_q_heads * sh.head_dim);
        std::vector<float> aq(tq.size());
        t.step(0, tq.data(), aq.data(), nullptr, nullptr, CLO_DTYPE_F32);
        if (t.prompt_tokens() <= 0 || t.decode_steps() < 0) return 8;
        if (expect_gpu && argc > 3) return run_trace(t, argv[3]);
    }
    std::puts("shim ok");
    return 0;
}
