// profiler.cpp — head profiling on the GPU (profile_heads, profiler.cpp:19-125
// of the reference; §8f rank 4): per query head the expected adjacent-step
// query similarity s_hat and the importance alpha (blend weight of full
// attention against the sink/recent stream that best explains the exact
// top-k output), then per KV head kv_importance = max, s_hat = min, tau =
// compute_threshold, difficulty = compute_difficulty. Placement is left
// all-offloaded; clo_plan_partition assigns it.
//
// The probe workloads are traces (clo_trace: the reference's TraceSource).
// The heavy parts run as sm_100a kernels through the op-level entry points:
// exact top-k selection (bit-exact with topk_select_exact), and full /
// streaming / top-k attention in float64 over the float64 trace rows. The
// O(L*hq*steps*d) cosines for s_hat and the alpha fit (fit_importance,
// head_profile.cpp:32-46) are tiny double sums on the host.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "clo.h"
#include "host_common.hpp"

struct clo_trace;

namespace clo {
namespace {

// cosine_similarity (attention.cpp:155-168): sequential double sums, clamp.
double cosine_host(const double* a, const double* b, int n) {
    double ab = 0.0, aa = 0.0, bb = 0.0;
    for (int i = 0; i < n; ++i) {
        const double x = a[i], y = b[i];
        ab += x * y;
        aa += x * x;
        bb += y * y;
    }
    if (aa == 0.0 || bb == 0.0) return 0.0;
    const double v = ab / (std::sqrt(aa) * std::sqrt(bb));
    return std::clamp(v, -1.0, 1.0);
}

void check(clo_status st) {
    if (st != CLO_OK) fail(st, clo_last_error());
}

}  // namespace
}  // namespace clo

using namespace clo;

extern "C" {

void clo_profiler_config_defaults(clo_profiler_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof *c);
    c->blend_sequences = 1;  // profiler.hpp:12-27
    c->blend_steps = 8;
    c->topk = 1;
    c->sink_tokens = 4;
    c->recent_tokens = 64;
    c->eta = 0.8;
    c->p = 3.0;
    c->epsilon = 0.1;
}

clo_status clo_profile_heads(const clo_trace* const* sources, int n_sources, const clo_profiler_config* cfg,
                             const double* provided_importance, clo_head_profile* out) {
    return guarded([&] {
        if (!sources || n_sources <= 0) fail(CLO_ERR_ARGUMENT, "profiling needs at least one probe workload");
        if (!cfg || !out) fail(CLO_ERR_ARGUMENT, "null argument");
        clo_model_shape shape{};
        int n0 = 0, s0 = 0;
        check(clo_trace_info(sources[0], &shape, &n0, &s0, nullptr));
        const int L = shape.num_layers, HQ = shape.num_q_heads, H = shape.num_kv_heads, d = shape.head_dim;
        const int m = HQ / H;
        if (m > 16) fail(CLO_ERR_CONFIG, "GQA group size above 16 is not supported");  // clo_head_profile.q_importance
        std::vector<int> n_prompt(n_sources), n_steps(n_sources);
        for (int i = 0; i < n_sources; ++i) {
            clo_model_shape s{};
            check(clo_trace_info(sources[i], &s, &n_prompt[i], &n_steps[i], nullptr));
            if (s.num_layers != L || s.num_q_heads != HQ || s.num_kv_heads != H || s.head_dim != d)
                fail(CLO_ERR_ARGUMENT, "probe workloads disagree on the model shape");
            if (n_steps[i] < 1) fail(CLO_ERR_ARGUMENT, "probe workloads need at least two query steps");
        }
        // true queries of every source and step: [src][t][L][HQ][d], the trace's
        // doubles as TraceSource::true_query returns them
        std::vector<std::vector<double>> q(n_sources);
        for (int i = 0; i < n_sources; ++i) {
            q[i].resize((size_t)(n_steps[i] + 1) * L * HQ * d);
            for (int t = 0; t <= n_steps[i]; ++t)
                for (int l = 0; l < L; ++l)
                    check(clo_trace_hidden(sources[i], t, l, q[i].data() + ((size_t)t * L + l) * HQ * d));
        }
        auto qrow = [&](int i, int t, int l, int h) { return q[i].data() + (((size_t)t * L + l) * HQ + h) * d; };

        // s_hat (profile_similarity, head_profile.cpp:48-68): mean adjacent-step cosine
        std::vector<double> s_hat((size_t)L * HQ, 0.0);
        for (int l = 0; l < L; ++l) {
            std::vector<double> sum(HQ, 0.0);
            uint64_t pairs = 0;
            for (int i = 0; i < n_sources; ++i)
                for (int t = 0; t + 1 <= n_steps[i]; ++t) {
                    for (int h = 0; h < HQ; ++h) sum[h] += cosine_host(qrow(i, t, l, h), qrow(i, t + 1, l, h), d);
                    ++pairs;
                }
            for (int h = 0; h < HQ; ++h) s_hat[(size_t)l * HQ + h] = sum[h] / (double)pairs;
        }

        // importance (profiler.cpp:59-99)
        std::vector<double> imp((size_t)L * HQ, 0.0);
        if (provided_importance) {
            for (int l = 0; l < L; ++l)
                for (int g = 0; g < H; ++g)
                    for (int j = 0; j < m; ++j) {
                        const double v = provided_importance[((size_t)l * H + g) * m + j];
                        if (!(v >= 0.0 && v <= 1.0)) fail(CLO_ERR_CONFIG, "importance values must lie in [0, 1]");
                        imp[(size_t)l * HQ + g * m + j] = v;
                    }
        } else {
            int dev_count = 0;
            if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
                fail(CLO_ERR_CUDA, "no CUDA device: the profiler's attention runs on the GPU");
            const int n_blend = std::min(cfg->blend_sequences, n_sources);
            for (int i = 0; i < n_blend; ++i)
                if (cfg->topk > n_prompt[i]) fail(CLO_ERR_ARGUMENT, "blend-fit top-k exceeds the probe prompt length");
            // per (l, h): sum over samples of (target - stream)(full - stream) and (full - stream)^2
            std::vector<double> num((size_t)L * HQ, 0.0), den((size_t)L * HQ, 0.0);
            for (int i = 0; i < n_blend; ++i) {
                const int n = n_prompt[i];
                const int t_end = std::min(cfg->blend_steps - 1, n_steps[i]);
                const int S = t_end + 1;
                std::vector<double> hk((size_t)n * d), hv((size_t)n * d);
                DevBuf dk, dv, dq, dfull, dstream, dtarget, didx_all, didx_win, dsel;
                dk.alloc(sizeof(double) * n * d, false);
                dv.alloc(sizeof(double) * n * d, false);
                dq.alloc(sizeof(double) * (size_t)m * S * d, false);
                dfull.alloc(sizeof(double) * (size_t)m * S * d, false);
                dstream.alloc(sizeof(double) * (size_t)m * S * d, false);
                dtarget.alloc(sizeof(double) * d, false);
                dsel.alloc(sizeof(int32_t) * cfg->topk, false);
                std::vector<int32_t> all(n), win(n);
                for (int r = 0; r < n; ++r) all[r] = r;
                int nwin = 0, clamped = 0;
                check(clo_sink_recent_indices(n, cfg->sink_tokens, cfg->recent_tokens, win.data(), &nwin, &clamped));
                if (nwin == 0) fail(CLO_ERR_ARGUMENT, "empty sink/recent window");
                didx_all.alloc(sizeof(int32_t) * n, false);
                didx_win.alloc(sizeof(int32_t) * nwin, false);
                CLO_CUDA(cudaMemcpy(didx_all.p, all.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
                CLO_CUDA(cudaMemcpy(didx_win.p, win.data(), sizeof(int32_t) * nwin, cudaMemcpyHostToDevice));
                std::vector<double> qs((size_t)m * S * d), full((size_t)m * S * d), stream((size_t)m * S * d), target(d);
                for (int l = 0; l < L; ++l)
                    for (int g = 0; g < H; ++g) {
                        check(clo_trace_prompt(sources[i], l, g, CLO_DTYPE_F64, hk.data(), hv.data()));
                        CLO_CUDA(cudaMemcpy(dk.p, hk.data(), sizeof(double) * n * d, cudaMemcpyHostToDevice));
                        CLO_CUDA(cudaMemcpy(dv.p, hv.data(), sizeof(double) * n * d, cudaMemcpyHostToDevice));
                        // the group's queries of every blend step, [j][t][d] (widened exactly)
                        for (int j = 0; j < m; ++j)
                            for (int t = 0; t < S; ++t) {
                                const double* src = qrow(i, t, l, g * m + j);
                                for (int c = 0; c < d; ++c) qs[((size_t)j * S + t) * d + c] = src[c];
                            }
                        CLO_CUDA(cudaMemcpy(dq.p, qs.data(), sizeof(double) * qs.size(), cudaMemcpyHostToDevice));
                        // full and streaming attention for all m*S queries at once
                        check(clo_topk_attention(dq.as<double>(), m * S, dk.p, dv.p, CLO_DTYPE_F64, n, d,
                                                 didx_all.as<int32_t>(), n, dfull.as<double>(), nullptr));
                        check(clo_topk_attention(dq.as<double>(), m * S, dk.p, dv.p, CLO_DTYPE_F64, n, d,
                                                 didx_win.as<int32_t>(), nwin, dstream.as<double>(), nullptr));
                        CLO_CUDA(cudaMemcpy(full.data(), dfull.p, sizeof(double) * full.size(), cudaMemcpyDeviceToHost));
                        CLO_CUDA(cudaMemcpy(stream.data(), dstream.p, sizeof(double) * stream.size(),
                                            cudaMemcpyDeviceToHost));
                        for (int j = 0; j < m; ++j)
                            for (int t = 0; t < S; ++t) {
                                const double* qd = dq.as<double>() + ((size_t)j * S + t) * d;
                                // exact top-k (bit-exact with topk_select_exact), then its attention
                                check(clo_topk_select_exact(qd, dk.p, CLO_DTYPE_F64, n, d, cfg->topk,
                                                            dsel.as<int32_t>(), nullptr));
                                check(clo_topk_attention(qd, 1, dk.p, dv.p, CLO_DTYPE_F64, n, d, dsel.as<int32_t>(),
                                                         cfg->topk, dtarget.as<double>(), nullptr));
                                CLO_CUDA(cudaMemcpy(target.data(), dtarget.p, sizeof(double) * d, cudaMemcpyDeviceToHost));
                                const size_t o = ((size_t)j * S + t) * d;
                                const size_t lh = (size_t)l * HQ + g * m + j;
                                for (int c = 0; c < d; ++c) {  // fit_importance's sums, sample order
                                    const double dd = full[o + c] - stream[o + c];
                                    num[lh] += (target[c] - stream[o + c]) * dd;
                                    den[lh] += dd * dd;
                                }
                            }
                    }
            }
            for (size_t lh = 0; lh < imp.size(); ++lh)
                imp[lh] = den[lh] == 0.0 ? 0.0 : std::clamp(num[lh] / den[lh], 0.0, 1.0);
        }

        // per KV head (profiler.cpp:101-122)
        for (int l = 0; l < L; ++l)
            for (int g = 0; g < H; ++g) {
                clo_head_profile& e = out[(size_t)l * H + g];
                std::memset(&e, 0, sizeof e);
                double kv_imp = -1.0, kv_s = 2.0;
                for (int j = 0; j < m; ++j) {
                    e.q_importance[j] = imp[(size_t)l * HQ + g * m + j];
                    kv_imp = std::max(kv_imp, e.q_importance[j]);  // kv_importance_of_group
                    kv_s = std::min(kv_s, s_hat[(size_t)l * HQ + g * m + j]);  // kv_s_hat_of_group
                }
                e.kv_importance = kv_imp;
                e.s_hat = kv_s;
                check(clo_compute_threshold(kv_imp, cfg->eta, cfg->p, &e.tau));
                check(clo_compute_difficulty(e.tau, e.s_hat, cfg->epsilon, &e.difficulty));
                e.placement = CLO_PLACEMENT_OFFLOADED;
            }
    });
}

}  // extern "C"
