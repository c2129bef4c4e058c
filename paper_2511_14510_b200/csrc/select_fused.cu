// select_fused.cu — the whole selection of one decode layer (offloaded heads,
// sign-hash retriever) in ONE kernel: lookup + query hash, scoring,
// threshold, compaction and the entry reconcile, one thread-block CLUSTER of
// CS CTAs per (sequence, KV head).
//
// Why: while the zero-copy gather keeps host reads queued in the memory
// system, every global synchronisation — a kernel boundary, a
// __threadfence() — waits behind that queue: measured on B200 beside a
// saturating gather, a graph edge between two empty kernels costs 9 us (32
// one-warp gather CTAs) to 40 us (128) instead of 0.4 us
// (tools/boundary_probe.cu, profiles/README.md round 2). The per-stage chain
// (prepare -> score -> threshold -> compact -> reconcile) paid that five times
// per layer and was the step's critical path (the transfer stream idled ~22%
// of the step waiting for fetch lists); a task-queue version synchronised
// through global counters paid it per task. Here a missed head is handled
// start to finish by its own cluster, whose ranks synchronise with the
// hardware cluster barrier and exchange through distributed shared memory:
//
//   rank 0     lookup_decide (lookup.cuh): the similarity decision, label
//              refresh and work-list entry; the decision reaches the other
//              ranks through DSMEM. Hits end here.
//   rank r     hashes code words r, r+CS, ... of the m approximate queries
//              against P's word slices staged by bulk copies (hash.cuh); the
//              words are exchanged through DSMEM
//   rank r     scores rows [r*n/CS, (r+1)*n/CS) (codes streamed by
//              cp.async.bulk through a 2-stage ring), writes the u16 keys and
//              its histogram of S
//   every rank sums the CS histograms (DSMEM) -> T = k-th largest S and the
//              number of S == T ties to keep; counts its rows > T and == T;
//              the counts give each rank its output offset and tie quota
//              (ties go by ascending index = rank order), and it writes its
//              part of the ascending selection
//   rank 0     reconciles the entry (reconcile.cuh): the layer's fetch list
//
// The result is the per-stage kernels' result bit for bit: the top-k of
// S(i) = max_j score_j(i) under (S desc, i asc), ascending
// (retrieval.cpp:33-46, :90-125; similarity_cache.cpp:180-201).
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdio>

#include "hash.cuh"
#include "lookup.cuh"
#include "reconcile.cuh"
#include "select_fused.cuh"

namespace clo {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPieceRows = 1024;
constexpr int kStages = 3;  // score ring depth (pieces of kPieceRows code rows in flight)
constexpr int kMaxBins = 8 * 64 + 1;  // nb = bits + 1 <= 513

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t remote(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(bulk::smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ int ld_remote_i32(const void* p, uint32_t rank) {
    int v;
    asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(remote(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_remote_u64(const void* p, uint32_t rank) {
    uint64_t v;
    asm volatile("ld.shared::cluster.b64 %0, [%1];" : "=l"(v) : "r"(remote(p, rank)) : "memory");
    return v;
}

// Ascending compaction of keys [start, end) (shared memory; row index =
// row_off + position): keeps S > T and the first `take` ties S == T (index
// order), writing at out[base...]. Warp w owns
// a contiguous 1/8 of the rows: pass 1 counts, an 8-warp prefix orders the
// warps, pass 2 emits with ballot ranks. Whole CTA; returns the rows written
// and sets *ties to the ties among them (block-uniform).
__device__ __forceinline__ int compact_rows(const uint16_t* keys, int start, int end, int row_off, uint16_t T, int base,
                                            int take, int32_t* out, int* s_gt, int* s_eq, int* ties) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int per = ((end - start + kWarps - 1) / kWarps + 31) / 32 * 32;
    const int w0 = min(end, start + warp * per), w1 = min(end, w0 + per);
    int gt = 0, eq = 0;
    for (int r = w0 + lane; r < w1; r += 32) {
        const uint16_t kv = keys[r];
        gt += kv > T;
        eq += kv == T;
    }
    gt = __reduce_add_sync(0xffffffffu, gt);
    eq = __reduce_add_sync(0xffffffffu, eq);
    if (lane == 0) {
        s_gt[warp] = gt;
        s_eq[warp] = eq;
    }
    __syncthreads();
    int eq_before = 0, pos = base, total = 0, tie_total = 0;
    for (int w = 0; w < kWarps; ++w) {
        const int tw = max(0, min(s_eq[w], take - tie_total));
        if (w < warp) {
            pos += s_gt[w] + tw;
            eq_before += s_eq[w];
        }
        total += s_gt[w] + tw;
        tie_total += tw;
    }
    for (int r0 = w0; r0 < w1; r0 += 32) {
        const int r = r0 + lane;
        const bool valid = r < w1;
        const uint16_t kv = valid ? keys[r] : (uint16_t)0;
        const bool is_eq = valid && kv == T;
        const unsigned eqm = __ballot_sync(0xffffffffu, is_eq);
        const bool sel = (valid && kv > T) || (is_eq && eq_before + __popc(eqm & lt) < take);
        const unsigned selm = __ballot_sync(0xffffffffu, sel);
        if (sel) out[pos + __popc(selm & lt)] = row_off + r;
        pos += __popc(selm);
        eq_before += __popc(eqm);
    }
    __syncthreads();  // s_gt / s_eq reusable
    *ties = tie_total;
    return total;
}

template <int W, int CS>
__global__ void __launch_bounds__(kThreads) layer_select_cluster_kernel(FusedSelectArgs f) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[kStages + 1];  // score ring, P slice
    __shared__ LookupShared lsh;
    __shared__ ReconcileSmem<kThreads> rsm;
    __shared__ uint64_t s_qw[kMaxGroup * W];  // the words this rank hashed [j][w]
    __shared__ uint64_t s_qb[kMaxGroup * W];  // every word of the m queries
    __shared__ uint32_t s_hist[kMaxBins];     // this rank's histogram of S
    __shared__ uint32_t s_tot[kMaxBins];      // the item's histogram
    __shared__ int s_cnt[2], s_T[2], s_gt[kWarps], s_eq[kWarps];
    const PrepareArgs& pa = f.prep;
    const EngineView& v = pa.v;
    const int l = pa.layer, m = v.m, nb = v.bits + 1;
    const uint32_t rank = cluster_rank();
    unsigned long long tp[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    CLO_PROBE_T(tp, 0)
    const int bg = blockIdx.x / CS;
    const int b = bg / v.H, g = bg % v.H, lg = l * v.H + g;
    if (v.persistent[lg]) return;  // uniform over the cluster
    const int seg = (b * v.L + l) * v.H + g;
    const int t = *v.dev_step + 1;
    const int n = v.n_prompt + t - 1;  // pre-append pool (engine.cpp:253-255)

    // shared memory: [keys of this rank's rows, u16][work area]; the work area
    // holds the P slice + queries + labels (lookup, hash), then the score ring
    // + per-warp histograms, then reconcile's lists
    const int per = ((n + CS - 1) / CS + kPieceRows - 1) / kPieceRows * kPieceRows;
    uint16_t* skeys = reinterpret_cast<uint16_t*>(smem);
    unsigned char* work = smem + f.keys_bytes;
    double* ps = reinterpret_cast<double*>(work);  // P slice [d][64]
    double* q = ps + (size_t)v.d * 64;             // [m][d]
    double* lab_s = q + (size_t)m * v.d;           // [m][d]
    if (threadIdx.x == 0) {
        lsh.selected = 0;
        for (int i = 0; i < kStages + 1; ++i) bulk::mbar_init(&bar[i]);
    }
    lookup_stage(pa, b, g, rank == 0, q, lab_s);
    if (rank == 0) lookup_decide(pa, b, g, q, lab_s, lsh);
    cluster_sync();
    const int selected = rank == 0 ? lsh.selected : ld_remote_i32(&lsh.selected, 0);
    const int item = rank == 0 ? lsh.item : ld_remote_i32(&lsh.item, 0);
    CLO_PROBE_T(tp, 1)
    cluster_sync();  // rank 0's decision has been read
    if (!selected) return;

    // ---- query sign bits: rank r hashes words r, r + CS, ...
    uint32_t slice_uses = 0;
    const double* pbase = v.proj_w + (size_t)lg * W * v.d * 64;
    for (int w = rank; w < W; w += CS) {
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk::load_async(ps, pbase + (size_t)w * v.d * 64, (uint32_t)v.d * 64 * 8, &bar[kStages]);
        }
        bulk::wait(&bar[kStages], slice_uses & 1);
        ++slice_uses;
        hash_word(ps, q, v.d, m, v.d, w, v.bits, [&](int j) { return reinterpret_cast<uint32_t*>(s_qw + j * W); });
        __syncthreads();
    }
    CLO_PROBE_T(tp, 2)
    cluster_sync();
    for (int x = threadIdx.x; x < m * W; x += blockDim.x) s_qb[x] = ld_remote_u64(&s_qw[x], (uint32_t)((x % W) % CS));
    for (int x = threadIdx.x; x < nb; x += blockDim.x) s_hist[x] = 0;

    // ---- score rows [r0, r1): S(i) = max_j (bits - popcount(q_j ^ code_i))
    const int r0 = min(n, (int)rank * per), r1 = min(n, r0 + per);
    const uint64_t* codes = v.codes + (size_t)seg * v.code_stride;
    {
        uint64_t* stage = reinterpret_cast<uint64_t*>(work);                                   // [kStages][kPieceRows * W]
        uint32_t* whist = reinterpret_cast<uint32_t*>(work + kStages * kPieceRows * W * 8);  // [kWarps][nb]
        for (int x = threadIdx.x; x < kWarps * nb; x += blockDim.x) whist[x] = 0;
        const int npieces = (r1 - r0 + kPieceRows - 1) / kPieceRows;
        auto issue = [&](int p) {  // thread 0
            const int row0 = r0 + p * kPieceRows;
            const int rows = min(kPieceRows, r1 - row0);
            const uint64_t* src = codes + (size_t)row0 * W;
            const uint32_t bytes = (reinterpret_cast<uintptr_t>(src) & 15) ? 0u : (uint32_t)rows * W * 8 / 16 * 16;
            if (bytes) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk::load_async(stage + (size_t)(p % kStages) * kPieceRows * W, src, bytes, &bar[p % kStages]);
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bulk::smem_u32(&bar[p % kStages])) : "memory");
            }
        };
        __syncthreads();  // whist cleared; every thread is done with the P slice
        if (threadIdx.x == 0)
            for (int p = 0; p < kStages && p < npieces; ++p) issue(p);
        uint32_t* myhist = whist + (threadIdx.x >> 5) * nb;
        for (int p = 0; p < npieces; ++p) {
            const int row0 = r0 + p * kPieceRows;
            const int rows = min(kPieceRows, r1 - row0);
            bulk::wait(&bar[p % kStages], (p / kStages) & 1);
            const uint64_t* st = stage + (size_t)(p % kStages) * kPieceRows * W;
            const bool staged = (reinterpret_cast<uintptr_t>(codes + (size_t)row0 * W) & 15) == 0;
            const int copied = staged ? rows * W * 8 / 16 * 16 / (W * 8) : 0;
#pragma unroll 4
            for (int r = threadIdx.x; r < rows; r += kThreads) {
                uint64_t c[W];
                if (r < copied) {
#pragma unroll
                    for (int w = 0; w < W; ++w) c[w] = st[(size_t)r * W + w];
                } else {
#pragma unroll
                    for (int w = 0; w < W; ++w) c[w] = __ldg(codes + (size_t)(row0 + r) * W + w);
                }
                int best = 0;
                for (int j = 0; j < m; ++j) {
                    int dist = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) dist += __popcll(c[w] ^ s_qb[j * W + w]);
                    best = max(best, v.bits - dist);
                }
                skeys[row0 - r0 + r] = static_cast<uint16_t>(best);
                atomicAdd(&myhist[best], 1u);
            }
            __syncthreads();  // ring slot p % kStages is free again
            if (threadIdx.x == 0 && p + kStages < npieces) issue(p + kStages);
        }
        for (int x = threadIdx.x; x < nb; x += blockDim.x) {
            uint32_t s = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s += whist[w * nb + x];
            s_hist[x] = s;
        }
    }
    CLO_PROBE_T(tp, 3)
    cluster_sync();

    // ---- threshold (every rank, from the CS histograms): T = k-th largest S,
    //      ties S == T to keep = k - #(S > T)
    for (int x = threadIdx.x; x < nb; x += blockDim.x) {
        uint32_t s = 0;
#pragma unroll
        for (int r = 0; r < CS; ++r) s += (uint32_t)ld_remote_i32(&s_hist[x], (uint32_t)r);
        s_tot[x] = s;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int running = 0, T = -1, gtT = 0;
        for (int top = nb - 1; top >= 0 && T < 0; top -= 32) {
            const int bi = top - lane;
            const int val = bi >= 0 ? (int)s_tot[bi] : 0;
            int incl = val;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, bi >= 0 && running + incl >= v.k);
            if (hit) {
                const int first = __ffs(hit) - 1;
                gtT = running + __shfl_sync(0xffffffffu, incl - val, first);
                T = top - first;
            }
            running += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            s_T[0] = T;
            s_T[1] = v.k - gtT;  // ties to keep
        }
    }
    __syncthreads();
    CLO_PROBE_T(tp, 4)
    const uint16_t T = (uint16_t)s_T[0];
    const int need_eq = s_T[1];
    {  // this rank's rows > T and == T
        int gt = 0, eq = 0;
        for (int r = threadIdx.x; r < r1 - r0; r += blockDim.x) {
            const uint16_t kv = skeys[r];
            gt += kv > T;
            eq += kv == T;
        }
        gt = __reduce_add_sync(0xffffffffu, gt);
        eq = __reduce_add_sync(0xffffffffu, eq);
        if ((threadIdx.x & 31) == 0) {
            s_gt[threadIdx.x >> 5] = gt;
            s_eq[threadIdx.x >> 5] = eq;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int G = 0, E = 0;
            for (int w = 0; w < kWarps; ++w) {
                G += s_gt[w];
                E += s_eq[w];
            }
            s_cnt[0] = G;
            s_cnt[1] = E;
        }
    }
    CLO_PROBE_T(tp, 5)
    cluster_sync();
    // output offset and tie quota of this rank (ties go by ascending index = rank order)
    int base = 0, quota = 0;
    {
        int eq_before = 0;
        for (int r = 0; r < CS; ++r) {
            const int gr = ld_remote_i32(&s_cnt[0], (uint32_t)r), er = ld_remote_i32(&s_cnt[1], (uint32_t)r);
            const int take = max(0, min(er, need_eq - eq_before));
            if (r < (int)rank) base += gr + take;
            if (r == (int)rank) quota = take;
            eq_before += er;
        }
    }
    __syncthreads();  // s_gt / s_eq were read above
    int32_t* out = f.prep.s.sel + (size_t)item * v.k;  // offloaded heads select into scratch (delta reconcile)
    for (int c0 = 0; c0 < r1 - r0; c0 += kScoreChunk) {
        int ties = 0;
        base += compact_rows(skeys, c0, min(r1 - r0, c0 + kScoreChunk), r0, T, base, quota, out, s_gt, s_eq, &ties);
        quota -= ties;
    }
    CLO_PROBE_T(tp, 6)
    cluster_sync();  // the whole selection is written; no rank's shared memory is read after this
    if (rank != 0) return;
    reconcile_item<kThreads>(f.rec, item, reinterpret_cast<int32_t*>(work), rsm);
#ifdef CLO_PROBE
    CLO_PROBE_T(tp, 7)
    if (threadIdx.x == 0 && l == 6 && t == 12)
        printf("SEL %llu b%d g%d: lookup %llu hash %llu score %llu thr %llu count %llu compact %llu reconcile %llu\n",
               tp[0], b, g, tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], tp[6] - tp[5],
               tp[7] - tp[6]);
#endif
}

}  // namespace

size_t fused_keys_bytes(int nmax, int cs) {
    const size_t per = ((size_t)(nmax + cs - 1) / cs + kPieceRows - 1) / kPieceRows * kPieceRows;
    return (per * 2 + 127) / 128 * 128;
}

size_t fused_select_smem(int words, int nb, int m, int d, int k, int nmax, int cs) {
    const size_t lookup = (size_t)d * 64 * 8 + 2 * (size_t)m * d * 8;
    const size_t score = (size_t)kStages * kPieceRows * words * 8 + (size_t)kWarps * nb * 4;
    const size_t rec = 4 * (size_t)k * 4;
    return fused_keys_bytes(nmax, cs) + std::max(std::max(lookup, score), rec);
}

bool fused_select_fits(int words, int nb, int m, int d, int k, int nmax) {
    return fused_select_smem(words, nb, m, d, k, nmax, fused_cluster_size()) <= 200 * 1024;
}

int fused_cluster_size() {
    static const int cs = [] {  // CLO_SELECT_CLUSTER: CTAs per missed head (4 or 8)
        const char* e = getenv("CLO_SELECT_CLUSTER");
        return e && atoi(e) == 4 ? 4 : 8;
    }();
    return cs;
}

void launch_fused_select(const FusedSelectArgs& f, cudaStream_t stream) {
    const EngineView& v = f.prep.v;
    const int cs = fused_cluster_size();
    const size_t sm = fused_select_smem(v.words, v.bits + 1, v.m, v.d, v.k, v.nmax, cs);
    FusedSelectArgs fa = f;
    fa.keys_bytes = (int)fused_keys_bytes(v.nmax, cs);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(v.B * v.H * cs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    switch (v.words * 16 + cs) {
#define CLO_WC(W, C)                                                                                        \
    case W * 16 + C:                                                                                        \
        cudaFuncSetAttribute(layer_select_cluster_kernel<W, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)sm);                                                                      \
        cudaLaunchKernelEx(&cfg, layer_select_cluster_kernel<W, C>, fa);                                     \
        break;
        CLO_WC(1, 4) CLO_WC(2, 4) CLO_WC(3, 4) CLO_WC(4, 4) CLO_WC(5, 4) CLO_WC(6, 4) CLO_WC(7, 4) CLO_WC(8, 4)
        CLO_WC(1, 8) CLO_WC(2, 8) CLO_WC(3, 8) CLO_WC(4, 8) CLO_WC(5, 8) CLO_WC(6, 8) CLO_WC(7, 8) CLO_WC(8, 8)
#undef CLO_WC
        default:
            break;
    }
}

}  // namespace clo
