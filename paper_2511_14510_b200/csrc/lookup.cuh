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

struct LookupShared {
    double sims[kMaxGroup];
    int degenerate, selected, item;
};

// The similarity-cache decision of (sequence b, KV head g) in a.layer, whole
// CTA (prepare_kernel's rank 0 and the fused per-layer selection kernel):
// q [m][d] holds the widened queries (the caller loaded and checked them),
// lab_s [m][d] the staged labels when the head is looked up. A selected head
// is appended to a.s's work list. Leaves (selected, item) in sh; ends with
// __syncthreads().
__device__ __forceinline__ void lookup_decide(const PrepareArgs& a, int b, int g, const double* q,
                                              const double* lab_s, LookupShared& sh) {
    const EngineView& v = a.v;
    const int l = a.layer, lg = l * v.H + g;
    const int seg = (b * v.L + l) * v.H + g;
    const bool pers = v.persistent[lg] != 0;
    const bool prefill = a.mode == kPrepPrefill;
    const int t = prefill ? 0 : *v.dev_step + 1;
    const int n_pool = prefill ? v.n_prompt : v.n_prompt + t - 1;
    const bool offl_sim = !pers && v.policy == 0;
    const bool lookup = !prefill && offl_sim && !v.always_hit;
    double* lab = v.labels + (((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m) * v.d;
    int* valid = v.label_valid + ((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m;
    if (threadIdx.x == 0) sh.degenerate = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        int selected = 0;
        if (prefill || pers) {
            selected = 1;
        } else if (v.policy == 3) {  // prefetch_only
            selected = 1;
            v.misses[seg] += 1;
            v.cache_last_update[seg] = t;
        } else if (v.always_hit) {  // engine.cpp:280-287
            v.history[(size_t)seg * v.max_steps + (t - 1)] = 1.0;
            v.hits[seg] += 1;
            v.last_lookup_hit[seg] = 1;
        }
        sh.selected = selected;
    }
    if (lookup) {
        // lookup (similarity_cache.cpp:29-72): one thread per group member,
        // sequential cosine chains over the staged labels
        if (threadIdx.x < v.m) {
            const int j = threadIdx.x;
            sh.sims[j] = 0.0;
            if (valid[j]) {
                bool deg;
                const double c = cosine_any(q + j * v.d, lab_s + j * v.d, v.d, &deg);
                sh.sims[j] = c;
                if (deg || c <= 0.0) atomicOr(&sh.degenerate, 2);
            } else {
                atomicOr(&sh.degenerate, 1);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const double tau = v.always_miss ? 2.0 : (v.has_tau_override ? v.tau_override : v.tau[lg]);
            double agg = 0.0;
            bool hit = false;
            if (sh.degenerate == 0) {  // all valid and all positive
                agg = aggregate_seq(sh.sims, v.qimp + (size_t)lg * v.m, v.m);
                hit = agg >= tau;
            }
            v.history[(size_t)seg * v.max_steps + (t - 1)] = agg;
            if (hit) {
                v.hits[seg] += 1;
                v.last_lookup_hit[seg] = 1;
            } else {
                v.last_lookup_hit[seg] = 0;
                v.misses[seg] += 1;
                v.cache_last_update[seg] = t;
                v.entry_last_update[seg] = t;
                sh.selected = 1;
            }
        }
        __syncthreads();
        if (sh.selected) {  // fused label refresh on miss
            for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) lab[i] = q[i];
            if (threadIdx.x < v.m) valid[threadIdx.x] = 1;
        }
    }
    if (prefill && offl_sim) {  // engine.cpp:192-200: labels := step-0 true queries
        for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) lab[i] = q[i];
        if (threadIdx.x < v.m) valid[threadIdx.x] = 1;
        if (threadIdx.x == 0) {
            v.entry_last_update[seg] = 0;
            v.cache_last_update[seg] = 0;
        }
    }
    __syncthreads();
    if (sh.selected && threadIdx.x == 0) {
        const int item = atomicAdd(&a.s.count[l], 1);
        sh.item = item;
        SelItem it;
        it.seg = seg;
        it.n = n_pool;
        const size_t row_bytes = (size_t)v.d * dtype_size(v.kv_dtype);
        if (pers)
            it.rows = (const char*)v.pk + ((size_t)b * v.NP + v.pidx[lg]) * v.nmax * row_bytes;
        else
            it.rows = v.kmirror ? (const char*)v.kmirror + ((size_t)b * v.NO + v.oidx[lg]) * v.nmax * row_bytes
                                : nullptr;
        it.codes = v.codes ? v.codes + (size_t)seg * v.code_stride : nullptr;
        // persistent heads select straight into their entry; offloaded heads
        // select into scratch and are reconciled with the old entry (delta gather)
        it.out_idx = pers ? v.entry_idx + (size_t)seg * v.k : a.s.sel + (size_t)item * v.k;
        it.out_score = nullptr;
        a.s.items[item] = it;
    }
    __syncthreads();
    if (sh.selected && v.retriever == 0) {  // the exact retriever scores the widened queries
        const int item = sh.item;
        for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) a.s.q64[(size_t)item * v.m * v.d + i] = q[i];
    }
}

// Widened queries of (b, g) in a.layer -> q [m][d] (non-finite -> error flag
// when `check`), and the labels -> lab_s when the head will be looked up.
// Whole CTA, one memory round trip; ends with __syncthreads().
__device__ __forceinline__ void lookup_stage(const PrepareArgs& a, int b, int g, bool check, double* q,
                                             double* lab_s) {
    const EngineView& v = a.v;
    const int l = a.layer, lg = l * v.H + g;
    const bool pers = v.persistent[lg] != 0;
    const bool prefill = a.mode == kPrepPrefill;
    const bool lookup = !prefill && !pers && v.policy == 0 && !v.always_hit;
    const float* qsrc = (prefill || pers) ? v.desc->true_q : v.desc->approx_q;
    const size_t qoff = (((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m) * v.d;
    const double* lab = v.labels + qoff;
    // One round trip: the finiteness flag is raised once after the loop (a
    // conditional atomic inside it kept the compiler from issuing the next
    // iteration's loads early: rank 0 spent 8-12 us here in the step graph,
    // profiles/r2/prepare_phase_probe_128ctas.txt, the other ranks 1.6 us).
    bool bad = false;
    for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) {
        const float x = __ldg(qsrc + qoff + i);
        bad |= !isfinite(x);
        q[i] = (double)x;
        if (check && lookup) lab_s[i] = lab[i];
    }
    if (check && bad) raise_err(v.err, kErrNonFiniteQuery);
    __syncthreads();
}

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
