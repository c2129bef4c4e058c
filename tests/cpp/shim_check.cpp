// Compiles a runner-style caller against the kvsim-named C++ shim
// (include/clo/kvsim.hpp) and exercises the host-side pure functions; engine
// creation must fail loudly (CudaError) when no GPU is present.
#include <clo/kvsim.hpp>

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

using namespace clo::kvsim;

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
    }
    std::puts("shim ok");
    return 0;
}
