// lookup.cu — K2: device-side similarity-cache decision + work-list build.
#include "lookup.cuh"

namespace clo {

namespace {

constexpr int kPrepThreads = 256;

// One CTA per (sequence, KV head) of one layer. Decides whether this head's
// top-k must be (re)selected this step, entirely on the device:
//   persistent heads   always, with the TRUE query (engine.cpp:269-274)
//   similarity policy  lookup(labels, approx queries, q_importance, tau)
//                      (engine.cpp:278-320): hit -> reuse the entry;
//                      miss -> labels := queries (fused, similarity_cache.cpp:63-70)
//   prefetch_only      always, with the approx query (engine.cpp:340-348)
//   prefill            every head, step-0 true query (engine.cpp:188-201)
// Selected heads are appended to the stream's work list with their widened
// queries and query sign bits.
__global__ void __launch_bounds__(kPrepThreads) prepare_kernel(PrepareArgs a) {
    const EngineView& v = a.v;
    const int b = blockIdx.x / v.H, g = blockIdx.x % v.H, l = a.layer;
    const int lg = l * v.H + g;
    const int seg = (b * v.L + l) * v.H + g;
    const bool pers = v.persistent[lg] != 0;
    if (a.kind == kKindOffloaded && pers) return;
    if (a.kind == kKindPersistent && !pers) return;

    extern __shared__ double dsm[];  // q [m][d], labels [m][d]
    double* q = dsm;
    double* lab_s = dsm + v.m * v.d;
    __shared__ double sims[kMaxGroup];
    __shared__ int s_degenerate, s_selected, s_item;

    const bool prefill = a.mode == kPrepPrefill;
    const int t = prefill ? 0 : *v.dev_step + 1;
    const int n_pool = prefill ? v.n_prompt : v.n_prompt + t - 1;
    const bool use_true = prefill || pers;
    const float* qsrc = use_true ? v.desc->true_q : v.desc->approx_q;
    const size_t qoff = (((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m) * v.d;
    for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) {
        const float x = qsrc[qoff + i];
        if (!isfinite(x)) raise_err(v.err, kErrNonFiniteQuery);
        q[i] = (double)x;
    }
    if (threadIdx.x == 0) s_selected = 0;
    __syncthreads();

    const bool offl_sim = !pers && v.policy == 0;
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
        s_selected = selected;
    }
    __syncthreads();

    if (!prefill && offl_sim && !v.always_hit) {
        // lookup (similarity_cache.cpp:29-72): one thread per group member.
        double* lab = v.labels + (((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m) * v.d;
        int* valid = v.label_valid + ((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m;
        if (threadIdx.x == 0) s_degenerate = 0;
        // stage the labels in shared memory: the sequential cosine chains then
        // read smem instead of paying an L2 round trip per element
        for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) lab_s[i] = lab[i];
        __syncthreads();
        if (threadIdx.x < v.m) {
            const int j = threadIdx.x;
            sims[j] = 0.0;
            if (valid[j]) {
                bool deg;
                const double c = cosine_any(q + j * v.d, lab_s + j * v.d, v.d, &deg);
                sims[j] = c;
                if (deg || c <= 0.0) atomicOr(&s_degenerate, 2);
            } else {
                atomicOr(&s_degenerate, 1);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const double tau = v.always_miss ? 2.0 : (v.has_tau_override ? v.tau_override : v.tau[lg]);
            double agg = 0.0;
            bool hit = false;
            if (s_degenerate == 0) {  // all valid and all positive
                agg = aggregate_seq(sims, v.qimp + (size_t)lg * v.m, v.m);
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
                s_selected = 1;
            }
        }
        __syncthreads();
        if (s_selected) {  // fused label refresh on miss
            for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) lab[i] = q[i];
            if (threadIdx.x < v.m) valid[threadIdx.x] = 1;
        }
    }
    if (prefill && offl_sim) {  // engine.cpp:192-200: labels := step-0 true queries
        double* lab = v.labels + (((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m) * v.d;
        int* valid = v.label_valid + ((size_t)b * v.L + l) * v.HQ + (size_t)g * v.m;
        for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) lab[i] = q[i];
        if (threadIdx.x < v.m) valid[threadIdx.x] = 1;
        if (threadIdx.x == 0) {
            v.entry_last_update[seg] = 0;
            v.cache_last_update[seg] = 0;
        }
    }
    if (!s_selected) return;

    if (threadIdx.x == 0) {
        const int item = atomicAdd(&a.s.count[l], 1);
        s_item = item;
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
    const int item = s_item;
    for (int i = threadIdx.x; i < v.m * v.d; i += blockDim.x) a.s.q64[(size_t)item * v.m * v.d + i] = q[i];
    if (v.retriever == 1)
        hash_queries_block(q, v.m, v.d, v.proj_t + (size_t)lg * v.d * v.bits, v.bits, v.words,
                           a.s.qbits + (size_t)item * v.m * v.words);
}

// Op-level lookup over independent groups (one warp-sized CTA each).
__global__ void lookup_op_kernel(int m, int d, double* labels, int32_t* valid,
                                 const double* queries, const double* weights, const double* tau,
                                 int32_t* hit_out, double* agg_out, double* sims_out,
                                 int32_t* reason_out) {
    const int h = blockIdx.x;
    __shared__ double sims[kMaxGroup];
    __shared__ int flags;
    double* lab = labels + (size_t)h * m * d;
    int32_t* val = valid + (size_t)h * m;
    const double* qs = queries + (size_t)h * m * d;
    if (threadIdx.x == 0) flags = 0;
    __syncthreads();
    if (threadIdx.x < m) {
        const int j = threadIdx.x;
        sims[j] = 0.0;
        if (val[j]) {
            bool deg;
            const double c = cosine_seq(qs + (size_t)j * d, lab + (size_t)j * d, d, &deg);
            sims[j] = c;
            if (deg || c <= 0.0) atomicOr(&flags, 2);
        } else {
            atomicOr(&flags, 1);
        }
    }
    __syncthreads();
    __shared__ int s_hit;
    if (threadIdx.x == 0) {
        int reason = 0, hit = 0;
        double agg = 0.0;
        if (flags & 1) {
            reason = 1;
        } else if (flags & 2) {
            reason = 2;
        } else {
            agg = aggregate_seq(sims, weights + (size_t)h * m, m);
            if (agg >= tau[h])
                hit = 1;
            else
                reason = 3;
        }
        hit_out[h] = hit;
        agg_out[h] = agg;
        reason_out[h] = reason;
        s_hit = hit;
    }
    __syncthreads();
    if (threadIdx.x < m) sims_out[(size_t)h * m + threadIdx.x] = sims[threadIdx.x];
    if (!s_hit) {
        for (int i = threadIdx.x; i < m * d; i += blockDim.x) lab[i] = qs[i];
        __syncthreads();
        if (threadIdx.x < m) val[threadIdx.x] = 1;
    }
}

__global__ void cosine_op_kernel(int n, int d, const double* a, const double* b, double* value,
                                 int32_t* degenerate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool deg;
    value[i] = cosine_seq(a + (size_t)i * d, b + (size_t)i * d, d, &deg);
    degenerate[i] = deg;
}

__global__ void aggregate_op_kernel(int n, int m, const double* sims, const double* w,
                                    double* out, int32_t* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int j = 0; j < m; ++j)
        if (w[(size_t)i * m + j] < 0.0) {
            atomicOr(err, 1);
            return;
        }
    for (int j = 0; j < m; ++j)
        if (sims[(size_t)i * m + j] <= 0.0) {
            atomicOr(err, 2);
            return;
        }
    out[i] = aggregate_seq(sims + (size_t)i * m, w + (size_t)i * m, m);
}

}  // namespace

void launch_prepare(const PrepareArgs& a, cudaStream_t stream) {
    const size_t sm = 2 * (size_t)a.v.m * a.v.d * sizeof(double);
    prepare_kernel<<<a.v.B * a.v.H, kPrepThreads, sm, stream>>>(a);
}

void launch_lookup_op(int n_heads, int m, int d, double* labels, int32_t* valid,
                      const double* queries, const double* weights, const double* tau,
                      int32_t* hit, double* agg, double* sims, int32_t* reason,
                      cudaStream_t stream) {
    lookup_op_kernel<<<n_heads, 32, 0, stream>>>(m, d, labels, valid, queries, weights, tau, hit,
                                                 agg, sims, reason);
}

void launch_cosine_op(int n, int d, const double* a, const double* b, double* value,
                      int32_t* degenerate, cudaStream_t stream) {
    cosine_op_kernel<<<(n + 127) / 128, 128, 0, stream>>>(n, d, a, b, value, degenerate);
}

void launch_aggregate_op(int n, int m, const double* sims, const double* w, double* out,
                         int32_t* err, cudaStream_t stream) {
    aggregate_op_kernel<<<(n + 127) / 128, 128, 0, stream>>>(n, m, sims, w, out, err);
}

}  // namespace clo
