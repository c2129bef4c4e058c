// lookup.cuh — K2 `lookup_label`: the head-wise approximate cache decision
// (similarity_cache.cpp:29-72) fused with the label refresh, the miss work
// list, query widening and the query sign-hash, all on the device.
#pragma once

#include "common.cuh"
#include "engine_view.h"
#include "select.cuh"

namespace clo {

// cosine_similarity (attention.cpp:155-168) in sequential IEEE double.
// Returns the clamped value; *degenerate set on a zero norm.
__device__ __forceinline__ double cosine_seq(const double* a, const double* b, int n,
                                             bool* degenerate) {
    double ab = 0.0, aa = 0.0, bb = 0.0;
    for (int i = 0; i < n; ++i) {
        ab = dmac(ab, a[i], b[i]);
        aa = dmac(aa, a[i], a[i]);
        bb = dmac(bb, b[i], b[i]);
    }
    if (aa == 0.0 || bb == 0.0) {
        *degenerate = true;
        return 0.0;
    }
    *degenerate = false;
    double v = __ddiv_rn(ab, __dmul_rn(__dsqrt_rn(aa), __dsqrt_rn(bb)));
    return fmin(fmax(v, -1.0), 1.0);
}

// Same chains for a compile-time length, fully unrolled: the products are
// independent of the accumulators, so only the three DADD chains are serial.
template <int D>
__device__ __forceinline__ double cosine_seq_d(const double* a, const double* b, bool* degenerate) {
    double ab = 0.0, aa = 0.0, bb = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double x = a[i], y = b[i];
        ab = dmac(ab, x, y);
        aa = dmac(aa, x, x);
        bb = dmac(bb, y, y);
    }
    if (aa == 0.0 || bb == 0.0) {
        *degenerate = true;
        return 0.0;
    }
    *degenerate = false;
    double v = __ddiv_rn(ab, __dmul_rn(__dsqrt_rn(aa), __dsqrt_rn(bb)));
    return fmin(fmax(v, -1.0), 1.0);
}

__device__ __forceinline__ double cosine_any(const double* a, const double* b, int n, bool* degenerate) {
    if (n == 128) return cosine_seq_d<128>(a, b, degenerate);
    if (n == 64) return cosine_seq_d<64>(a, b, degenerate);
    return cosine_seq(a, b, n, degenerate);
}

// aggregate_similarity (similarity_cache.cpp:10-27); callers guarantee
// non-negative weights and positive sims.
__device__ __forceinline__ double aggregate_seq(const double* sims, const double* w, int m) {
    double wsum = 0.0;
    for (int i = 0; i < m; ++i) wsum = __dadd_rn(wsum, w[i]);
    double num = 0.0, den = 0.0;
    for (int i = 0; i < m; ++i) {
        const double wi = wsum > 0.0 ? w[i] : 1.0;
        num = __dadd_rn(num, wi);
        den = __dadd_rn(den, __ddiv_rn(wi, sims[i]));
    }
    return __ddiv_rn(num, den);
}

enum PrepareMode : int { kPrepPrefill = 0, kPrepDecode = 1 };
enum PrepareKind : int { kKindOffloaded = 0, kKindPersistent = 1, kKindAll = 2 };

struct PrepareArgs {
    EngineView v;
    SelScratch s;
    int layer;
    int mode;
    int kind;
    int count_gathered;  // decode steps count gathered bytes; prefill does not
};

void launch_prepare(const PrepareArgs& a, cudaStream_t stream);
void launch_lookup_op(int n_heads, int m, int d, double* labels, int32_t* valid,
                      const double* queries, const double* weights, const double* tau,
                      int32_t* hit, double* agg, double* sims, int32_t* reason,
                      cudaStream_t stream);
void launch_cosine_op(int n, int d, const double* a, const double* b, double* value,
                      int32_t* degenerate, cudaStream_t stream);
void launch_aggregate_op(int n, int m, const double* sims, const double* w, double* out,
                         int32_t* err, cudaStream_t stream);

}  // namespace clo
