// lookup.cu — K2: device-side similarity-cache decision + work-list build.
#include <cstdio>

#include "lookup.cuh"
#include "hash.cuh"

namespace clo {

namespace {

constexpr int kPrepThreads = 256;

// One CLUSTER of `words` CTAs per (sequence, KV head) of one layer (one CTA
// when the retriever is exact). Decides whether this head's top-k must be
// (re)selected this step, entirely on the device:
//   persistent heads   always, with the TRUE query (engine.cpp:269-274)
//   similarity policy  lookup(labels, approx queries, q_importance, tau)
//                      (engine.cpp:278-320): hit -> reuse the entry;
//                      miss -> labels := queries (fused, similarity_cache.cpp:63-70)
//   prefetch_only      always, with the approx query (engine.cpp:340-348)
//   prefill            every head, step-0 true query (engine.cpp:188-201)
// Rank 0 makes the decision and appends a selected head to the stream's work
// list with its widened queries; it publishes (selected, item) in its shared
// memory, and every rank r of a selected head then hashes code word r of the
// m queries against P's word slice staged by one bulk copy (hash.cuh): three
// dependent memory round trips per head instead of one per batch of P loads.
#ifdef CLO_PROBE
__device__ __forceinline__ unsigned __smid_probe() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
#endif

__global__ void __launch_bounds__(kPrepThreads) prepare_kernel(PrepareArgs a) {
    const EngineView& v = a.v;
    unsigned long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    CLO_PROBE_T(tp, 0)
    const int nr = a.v.retriever == 1 ? v.words : 1;  // cluster size
    const int rank = (int)(blockIdx.x % nr);
    const int bg = blockIdx.x / nr;
    const int b = bg / v.H, g = bg % v.H, l = a.layer;
    const int lg = l * v.H + g;
    const int seg = (b * v.L + l) * v.H + g;
    const bool pers = v.persistent[lg] != 0;
    if (a.kind == kKindOffloaded && pers) return;  // uniform over the cluster
    if (a.kind == kKindPersistent && !pers) return;

    extern __shared__ __align__(128) double dsm[];  // P slice [d][64] (hashing), q [m][d], labels [m][d]
    double* ps = dsm;
    double* q = dsm + (v.retriever == 1 ? (size_t)v.d * 64 : 0);
    double* lab_s = q + v.m * v.d;
    __shared__ LookupShared sh;
    __shared__ __align__(8) uint64_t bar;

    // code word `rank`'s P slice: its bulk copy is issued first and lands
    // while rank 0 stages and decides (the slice depends on (l, g, rank) only)
    const double* slice = v.proj_w + ((size_t)lg * v.words + rank) * v.d * 64;
    if (threadIdx.x == 0) {
        sh.selected = 0;
        if (nr > 1) {
            bulk::mbar_init(&bar);
            bulk::load_async(ps, slice, (uint32_t)v.d * 64 * 8, &bar);
        }
    }
    // queries (every rank hashes them) and, on rank 0, the labels: one round trip
    lookup_stage(a, b, g, rank == 0, q, lab_s);
    CLO_PROBE_T(tp, 1)

    if (rank == 0) lookup_decide(a, b, g, q, lab_s, sh);
    CLO_PROBE_T(tp, 2)
    if (v.retriever != 1) return;
    int selected = sh.selected, item = sh.item;
    if (nr > 1) {
        // rank 0's decision -> every rank (distributed shared memory)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (rank != 0) {
            uint32_t ra, rb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(bulk::smem_u32(&sh.selected)));
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rb) : "r"(bulk::smem_u32(&sh.item)));
            asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(selected) : "r"(ra) : "memory");
            asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(item) : "r"(rb) : "memory");
        }
        // rank 0 stays resident until every rank has read it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    CLO_PROBE_T(tp, 3)
    if (nr > 1) bulk::wait(&bar, 0);  // no CTA exits with its slice copy in flight
    if (!selected) return;
    // code word `rank` of the m query sign-hashes
    if (nr == 1) {
        for (int i = threadIdx.x; i < v.d * 64; i += blockDim.x) ps[i] = slice[i];
        __syncthreads();
    }
    CLO_PROBE_T(tp, 4)
    uint32_t* out32 = reinterpret_cast<uint32_t*>(a.s.qbits + (size_t)item * v.m * v.words);
    hash_word(ps, q, v.d, v.m, v.d, rank, v.bits, [&](int j) { return out32 + (size_t)j * v.words * 2; });
#ifdef CLO_PROBE
    CLO_PROBE_T(tp, 5)
    if (threadIdx.x == 0 && l == 6 && *v.dev_step + 1 == 12)
        printf("PREP %llu b%d g%d r%d sm%u: load %llu decide %llu sync %llu slice %llu hash %llu\n", tp[0], b, g, rank,
               __smid_probe(), tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4]);
#endif
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
    const int nr = a.v.retriever == 1 ? a.v.words : 1;
    const size_t sm = (a.v.retriever == 1 ? (size_t)a.v.d * 64 * sizeof(double) : 0) +
                      2 * (size_t)a.v.m * a.v.d * sizeof(double);
    cudaFuncSetAttribute(prepare_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);  // per device
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(a.v.B * a.v.H * nr));
    cfg.blockDim = dim3(kPrepThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)nr;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, prepare_kernel, a);
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
