// select_fused.cu — the whole selection of one decode layer (offloaded heads,
// sign-hash retriever) as ONE kernel: lookup + query hash, scoring,
// threshold, compaction and the entry reconcile.
//
// Why one kernel: while the zero-copy gather of the previous layer keeps the
// PCIe link busy, every kernel boundary on another stream waits for the
// memory system to drain the queued host reads — measured on B200 at 9 us
// (32 one-warp gather CTAs) to 40 us (128) per graph edge instead of 0.4 us
// (tools/boundary_probe.cu, profiles/README.md round 2). The per-stage chain
// (prepare -> score -> threshold -> compact -> reconcile) paid that five
// times per layer and became the step's critical path: the transfer stream
// sat idle ~22% of the step waiting for fetch lists. Here the stages are
// tasks of one persistent grid, claimed in order from a per-layer counter:
//
//   [0, B*H)               lookup of (sequence, KV head) p: the similarity
//                          decision (lookup_decide, lookup.cuh); on a miss the
//                          head becomes work item `item` and the CTA hashes
//                          the m approximate queries, one P^T word slice at a
//                          time from shared memory (hash.cuh)
//   then C*NC score tasks  (item, 4096-row chunk): S(i) and the chunk
//                          histogram; the CTA finishing an item's last chunk
//                          computes its threshold (threshold_item)
//   then C*NC compaction   (item, chunk) after the item's threshold; the CTA
//   tasks                  finishing an item's last chunk reconciles the entry
//                          (reconcile_item) and publishes its fetch list
//
// C (missed heads) is known once every lookup task is done; later tasks wait
// for that. A task only ever waits for tasks claimed before it, and a claimed
// task belongs to a running CTA, so the grid makes progress whatever the
// residency. Counters live in a per-layer control block (reset at step end).
// Results are identical to the per-stage kernels (same device functions).
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "hash.cuh"
#include "lookup.cuh"
#include "reconcile.cuh"
#include "select_dev.cuh"
#include "select_fused.cuh"

namespace clo {

namespace {

constexpr int kThreads = kScoreThreads;  // 256
constexpr int kWarps = kThreads / 32;
constexpr int kPieceRows = 1024;
constexpr int kPieces = kScoreChunk / kPieceRows;

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// thread 0 waits until *p >= target; the barrier then orders every thread's
// later reads after the producers' releases (fence + atomic)
__device__ __forceinline__ void wait_at_least(const int* p, int target) {
    if (threadIdx.x == 0) {
        int ns = 32;
        while (ld_acquire(p) < target) {
            __nanosleep(ns);
            ns = ns < 512 ? 2 * ns : ns;
        }
    }
    __syncthreads();
}

// thread 0: publish this CTA's writes, then count one more done; returns the
// previous value (broadcast through *s_old)
__device__ __forceinline__ int signal_done(int* counter, int* s_old) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) *s_old = atomicAdd(counter, 1);
    __syncthreads();
    return *s_old;
}

// S(i) of one 4096-row chunk (rows streamed by cp.async.bulk in 1024-row
// pieces through a 2-stage ring), keys as u16 and the chunk histogram.
// `uses` counts this CTA's completed uses of each ring barrier (phase bits).
template <int W>
__device__ void score_chunk(const SelArgs& a, int item, int chunk, uint64_t* stage, uint32_t* whist, uint64_t* qb,
                            uint64_t* bar, uint32_t (&uses)[2]) {
    const SelItem it = a.items[item];
    const int c0 = chunk * kScoreChunk;
    const int end = min(c0 + kScoreChunk, it.n);
    const int npieces = (end - c0 + kPieceRows - 1) / kPieceRows;
    const int warp = threadIdx.x >> 5;
    for (int x = threadIdx.x; x < kWarps * a.nb; x += blockDim.x) whist[x] = 0;
    for (int x = threadIdx.x; x < a.m * W; x += blockDim.x) {
        const int j = x / W, w = x % W;
        qb[x] = a.qbits[((size_t)item * a.m + j) * a.words + w];
    }
    __syncthreads();  // also: the previous task's reads of the ring are done
    auto issue = [&](int p) {  // thread 0
        const int row0 = c0 + p * kPieceRows;
        const int rows = min(kPieceRows, end - row0);
        const uint64_t* src = it.codes + (size_t)row0 * W;
        const uint32_t bytes = (reinterpret_cast<uintptr_t>(src) & 15) ? 0u : (uint32_t)rows * W * 8 / 16 * 16;
        uint64_t* b = &bar[p & 1];
        if (bytes) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk::load_async(stage + (size_t)(p & 1) * kPieceRows * W, src, bytes, b);
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bulk::smem_u32(b)) : "memory");
        }
    };
    if (threadIdx.x == 0) {
        issue(0);
        if (npieces > 1) issue(1);
    }
    uint16_t* keys = a.key16 + (size_t)item * a.nmax;
    uint32_t* myhist = whist + warp * a.nb;
    for (int p = 0; p < npieces; ++p) {
        const int row0 = c0 + p * kPieceRows;
        const int rows = min(kPieceRows, end - row0);
        bulk::wait(&bar[p & 1], uses[p & 1] & 1);
        const uint64_t* st = stage + (size_t)(p & 1) * kPieceRows * W;
        const bool staged = (reinterpret_cast<uintptr_t>(it.codes + (size_t)row0 * W) & 15) == 0;
        const int copied = staged ? rows * W * 8 / 16 * 16 / (W * 8) : 0;
#pragma unroll 4
        for (int r = threadIdx.x; r < rows; r += kThreads) {
            uint64_t c[W];
            if (r < copied) {
#pragma unroll
                for (int w = 0; w < W; ++w) c[w] = st[(size_t)r * W + w];
            } else {
#pragma unroll
                for (int w = 0; w < W; ++w) c[w] = __ldg(it.codes + (size_t)(row0 + r) * W + w);
            }
            int best = 0;
            for (int j = 0; j < a.m; ++j) {
                int dist = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) dist += __popcll(c[w] ^ qb[j * W + w]);
                best = max(best, a.bits - dist);
            }
            keys[row0 + r] = static_cast<uint16_t>(best);
            atomicAdd(&myhist[best], 1u);
        }
        ++uses[p & 1];
        __syncthreads();  // ring slot p & 1 is free again
        if (threadIdx.x == 0 && p + 2 < npieces) issue(p + 2);
    }
    uint32_t* out = a.chunk_hist + ((size_t)item * a.max_chunks + chunk) * a.nb;
    for (int b = threadIdx.x; b < a.nb; b += blockDim.x) {
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) sum += whist[w * a.nb + b];
        out[b] = sum;
    }
}

template <int W>
__global__ void __launch_bounds__(kThreads) layer_select_kernel(FusedSelectArgs f) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[3];  // score ring (2), P slice (1)
    __shared__ LookupShared lsh;
    __shared__ ReconcileSmem<kThreads> rsm;
    __shared__ int s_task, s_old, s_sts[2], s_gt[kWarps], s_eq[kWarps];
    const PrepareArgs& pa = f.prep;
    const SelArgs& sa = f.sel;
    const EngineView& v = pa.v;
    const int l = pa.layer;
    const int BH = v.B * v.H, NC = sa.max_chunks;
    int* ctl = f.ctl + (size_t)l * f.ctl_stride;
    int* claim = ctl;
    int* lookups_done = ctl + 1;
    int* score_done = ctl + 2;                   // [items_cap]
    int* thr_ready = score_done + f.items_cap;   // [items_cap]
    int* compact_done = thr_ready + f.items_cap; // [items_cap]
    uint32_t uses[2] = {0, 0};
    uint32_t slice_uses = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) bulk::mbar_init(&bar[i]);
    }
    __syncthreads();
    for (;;) {
        if (threadIdx.x == 0) s_task = atomicAdd(claim, 1);
        __syncthreads();
        const int t = s_task;
        if (t < BH) {
            // ---- lookup (+ query hash on a miss)
            const int b = t / v.H, g = t % v.H;
            double* ps = reinterpret_cast<double*>(smem);   // P slice [d][64]
            double* q = ps + (size_t)v.d * 64;              // [m][d]
            double* lab_s = q + (size_t)v.m * v.d;          // [m][d]
            if (v.persistent[l * v.H + g] == 0) {
                lookup_stage(pa, b, g, true, q, lab_s);
                lookup_decide(pa, b, g, q, lab_s, lsh);
                if (lsh.selected) {
                    const int item = lsh.item;
                    const double* base = v.proj_w + (size_t)(l * v.H + g) * v.words * v.d * 64;
                    uint32_t* out32 = reinterpret_cast<uint32_t*>(pa.s.qbits + (size_t)item * v.m * v.words);
                    for (int w = 0; w < v.words; ++w) {
                        if (threadIdx.x == 0) {
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            bulk::load_async(ps, base + (size_t)w * v.d * 64, (uint32_t)v.d * 64 * 8, &bar[2]);
                        }
                        bulk::wait(&bar[2], slice_uses & 1);
                        ++slice_uses;
                        hash_word(ps, q, v.d, v.m, v.d, w, v.bits,
                                  [&](int j) { return out32 + (size_t)j * v.words * 2; });
                        __syncthreads();  // the slice buffer is free
                    }
                }
            }
            signal_done(lookups_done, &s_old);
            continue;
        }
        wait_at_least(lookups_done, BH);
        const int C = *reinterpret_cast<const volatile int*>(sa.count);
        int u = t - BH;
        if (u < C * NC) {
            // ---- score one chunk; the item's last chunk computes its threshold
            const int item = u / NC, chunk = u % NC;
            const int nch = num_chunks(sa.items[item].n);
            if (chunk >= nch) continue;
            uint64_t* stage = reinterpret_cast<uint64_t*>(smem);
            uint32_t* whist = reinterpret_cast<uint32_t*>(smem + 2 * kPieceRows * W * 8);
            uint64_t* qb = reinterpret_cast<uint64_t*>(smem + 2 * kPieceRows * W * 8 +
                                                       ((size_t)kWarps * sa.nb * 4 + 7) / 8 * 8);
            score_chunk<W>(sa, item, chunk, stage, whist, qb, bar, uses);
            if (signal_done(score_done + item, &s_old) == nch - 1) {
                __threadfence();
                threshold_item(sa, item, reinterpret_cast<uint32_t*>(smem), s_sts);
                signal_done(thr_ready + item, &s_old);
            }
            continue;
        }
        u -= C * NC;
        if (u < C * NC) {
            // ---- compact one chunk; the item's last chunk reconciles the entry
            const int item = u / NC, chunk = u % NC;
            const int nch = num_chunks(sa.items[item].n);
            if (chunk >= nch) continue;
            wait_at_least(thr_ready + item, 1);
            compact_unit<uint16_t>(sa, item, chunk, s_gt, s_eq);
            if (signal_done(compact_done + item, &s_old) == nch - 1) {
                __threadfence();
                reconcile_item<kThreads>(f.rec, item, reinterpret_cast<int32_t*>(smem), rsm);
            }
            continue;
        }
        break;
    }
}

}  // namespace

size_t fused_select_smem(int words, int nb, int m, int d, int k, int max_chunks) {
    const size_t lookup = (size_t)d * 64 * 8 + 2 * (size_t)m * d * 8;
    const size_t score = 2 * (size_t)kPieceRows * words * 8 + ((size_t)kWarps * nb * 4 + 7) / 8 * 8 + (size_t)m * words * 8;
    const size_t thr = ((size_t)nb + 2 * (size_t)max_chunks) * 4;
    const size_t rec = 4 * (size_t)k * 4;
    return std::max(std::max(lookup, score), std::max(thr, rec));
}

void launch_fused_select(const FusedSelectArgs& f, int grid, cudaStream_t stream) {
    const SelArgs& a = f.sel;
    const size_t sm = fused_select_smem(a.words, a.nb, a.m, a.d, a.k, a.max_chunks);
    switch (a.words) {
#define CLO_W(W)                                                                                           \
    case W:                                                                                                \
        cudaFuncSetAttribute(layer_select_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        layer_select_kernel<W><<<grid, kThreads, sm, stream>>>(f);                                         \
        break;
        CLO_W(1) CLO_W(2) CLO_W(3) CLO_W(4) CLO_W(5) CLO_W(6) CLO_W(7) CLO_W(8)
#undef CLO_W
        default:
            break;
    }
}

}  // namespace clo
