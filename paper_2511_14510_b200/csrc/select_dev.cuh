// select_dev.cuh — CTA-wide device functions of the sign-hash selection
// (threshold of one item, compaction of one chunk), shared by the per-stage
// kernels in select.cu and the fused per-layer selection kernel.
#pragma once

#include "select.cuh"

namespace clo {

__device__ __forceinline__ int num_chunks(int n) { return (n + kScoreChunk - 1) / kScoreChunk; }

// Register-cached variant bound: chunks per warp x 32-bin blocks per lane.
// A chunk's bin counts are <= kScoreChunk < 2^16, so two blocks share a
// register (low / high half): 5 chunks x 5 registers per lane cover 512K-token
// items (129 chunks) with 1024 threads and 256-bit hashes (nb = 257 <= 320)
// without spilling under the 64-register cap; longer items take the loop.
constexpr int kThrCpw = 5, kThrBpl = 10;
static_assert(kScoreChunk < 65536, "u16 bin counts");

// T from the item's bin totals (tot, shared memory), by warp 0: walk bins from
// the top in blocks of 32 with suffix sums by warp scan. Writes sts.
__device__ __forceinline__ void threshold_walk(const SelArgs& a, const uint32_t* tot, int* sts) {
    const int lane = threadIdx.x & 31;
    int running = 0, T = -1, gtT = 0;
    for (int top = a.nb - 1; top >= 0 && T < 0; top -= 32) {
        const int b = top - lane;
        int v = b >= 0 ? (int)tot[b] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, b >= 0 && running + incl >= a.k);
        if (hit) {
            const int first = __ffs(hit) - 1;
            const int excl = __shfl_sync(0xffffffffu, incl - v, first);
            T = top - first;
            gtT = running + excl;
        }
        running += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
        sts[0] = T;
        sts[1] = gtT;
    }
}

// Per item: T = k-th largest S (ties resolved later by index), then each
// chunk's output offset and how many of its S == T ties it keeps.
// Whole CTA; smem = nb + 2*max_chunks words, sts = 2 ints. Ends with __syncthreads().
__device__ __forceinline__ void threshold_item(const SelArgs& a, int item, uint32_t* smem, int* sts) {
    uint32_t* tot = smem;                               // [nb]
    int* gt = reinterpret_cast<int*>(smem + a.nb);      // [max_chunks]
    int* eq = gt + a.max_chunks;                        // [max_chunks]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    {
        const SelItem it = a.items[item];
        const int nch = num_chunks(it.n);
        const uint32_t* hist = a.chunk_hist + (size_t)item * a.max_chunks * a.nb;
        const int nbb = (a.nb + 31) / 32;
        if (nch <= kThrCpw * nwarps && nbb <= kThrBpl) {
            // Warp w holds chunks w, w + nwarps, ... (up to 4) x all bins in
            // registers: every histogram load of the item is issued at once (one
            // L2 round trip instead of one per 32-bin block), and the per-chunk
            // counts above / at T come from the same registers.
            uint32_t hv[kThrCpw][kThrBpl / 2];
#pragma unroll
            for (int ci = 0; ci < kThrCpw; ++ci) {
                const int c = warp + ci * nwarps;
#pragma unroll
                for (int bp = 0; bp < kThrBpl / 2; ++bp) {
                    const int b0 = 2 * bp * 32 + lane, b1 = b0 + 32;
                    const uint32_t lo = c < nch && b0 < a.nb ? __ldcg(hist + (size_t)c * a.nb + b0) : 0u;
                    const uint32_t hi = c < nch && b1 < a.nb ? __ldcg(hist + (size_t)c * a.nb + b1) : 0u;
                    hv[ci][bp] = lo | (hi << 16);
                }
            }
            auto bin = [&](int ci, int bb) -> uint32_t { return (hv[ci][bb >> 1] >> ((bb & 1) * 16)) & 0xFFFFu; };
            for (int b = threadIdx.x; b < a.nb; b += blockDim.x) tot[b] = 0;
            __syncthreads();
#pragma unroll
            for (int bb = 0; bb < kThrBpl; ++bb) {
                uint32_t sum = 0;
#pragma unroll
                for (int ci = 0; ci < kThrCpw; ++ci) sum += bin(ci, bb);
                if (sum) atomicAdd(&tot[bb * 32 + lane], sum);
            }
            __syncthreads();
            if (warp == 0) threshold_walk(a, tot, sts);
            __syncthreads();
            const int T = sts[0];
#pragma unroll
            for (int ci = 0; ci < kThrCpw; ++ci) {
                const int c = warp + ci * nwarps;
                int g = 0, e = 0;
#pragma unroll
                for (int bb = 0; bb < kThrBpl; ++bb) {
                    const int b = bb * 32 + lane;
                    g += b > T ? (int)bin(ci, bb) : 0;
                    e += b == T ? (int)bin(ci, bb) : 0;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    g += __shfl_xor_sync(0xffffffffu, g, o);
                    e += __shfl_xor_sync(0xffffffffu, e, o);
                }
                if (lane == 0 && c < nch) {
                    gt[c] = g;
                    eq[c] = e;
                }
            }
        } else {
            if (nch <= 64) {  // one thread per bin walks the chunks
                for (int b = threadIdx.x; b < a.nb; b += blockDim.x) {
                    uint32_t s = 0;
#pragma unroll 8
                    for (int c = 0; c < nch; ++c) s += hist[(size_t)c * a.nb + b];
                    tot[b] = s;
                }
            } else {  // long items: warp w sums chunks w, w + nwarps, ... (coalesced bin rows)
                for (int b = threadIdx.x; b < a.nb; b += blockDim.x) tot[b] = 0;
                __syncthreads();
                for (int b0 = 0; b0 < a.nb; b0 += 32) {
                    const int b = b0 + lane;
                    if (b < a.nb) {
                        uint32_t s = 0;
#pragma unroll 4
                        for (int c = warp; c < nch; c += nwarps) s += hist[(size_t)c * a.nb + b];
                        if (s) atomicAdd(&tot[b], s);
                    }
                }
            }
            __syncthreads();
            if (warp == 0) threshold_walk(a, tot, sts);
            __syncthreads();
            const int T = sts[0];
            for (int c = warp; c < nch; c += nwarps) {
                const uint32_t* h = hist + (size_t)c * a.nb;
                int g = 0;
                for (int b = T + 1 + lane; b < a.nb; b += 32) g += h[b];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
                if (lane == 0) {
                    gt[c] = g;
                    eq[c] = h[T];
                }
            }
        }
        __syncthreads();
        const int need_eq = a.k - sts[1];
        if (warp == 0) {
            int base_run = 0, eq_run = 0;
            for (int c0 = 0; c0 < nch; c0 += 32) {
                const int c = c0 + lane;
                const int e = c < nch ? eq[c] : 0;
                int ie = e;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int t = __shfl_up_sync(0xffffffffu, ie, o);
                    if (lane >= o) ie += t;
                }
                const int eq_before = eq_run + ie - e;
                const int take = max(0, min(e, need_eq - eq_before));
                const int contrib = c < nch ? gt[c] + take : 0;
                int ic = contrib;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int t = __shfl_up_sync(0xffffffffu, ic, o);
                    if (lane >= o) ic += t;
                }
                if (c < nch) {
                    a.chunk_base[(size_t)item * a.max_chunks + c] = base_run + ic - contrib;
                    a.chunk_take[(size_t)item * a.max_chunks + c] = take;
                }
                base_run += __shfl_sync(0xffffffffu, ic, 31);
                eq_run += __shfl_sync(0xffffffffu, ie, 31);
            }
            if (lane == 0) {
                a.thresh[item] = (uint64_t)sts[0];
                a.need[item] = need_eq;
            }
        }
        __syncthreads();
    }
}

template <typename KeyT>
__device__ __forceinline__ double key_score(KeyT k);
template <>
__device__ __forceinline__ double key_score<uint16_t>(uint16_t k) { return (double)k; }
template <>
__device__ __forceinline__ double key_score<uint64_t>(uint64_t k) { return key_to_double(k); }

// Keeps S > T and the first chunk_take ties S == T (index order) of one chunk,
// writing indices ascending at chunk_base (select_topk's final ascending sort,
// retrieval.cpp:43, merge_group_topk's :197-199). Warp w owns 512 consecutive
// rows: pass 1 counts (coalesced key loads), a tiny 8-warp prefix in shared
// memory orders the warps, pass 2 re-reads the keys (L1) and emits with
// ballot/popc ranks — two barriers per chunk, no block-wide scans.
// One (item, chunk) unit, kScoreThreads threads; s_gt/s_eq = kScoreThreads/32
// ints each. Ends with __syncthreads() (when the chunk exists).
template <typename KeyT>
__device__ __forceinline__ void compact_body(const SelArgs& a, const SelItem& it, int item, int chunk, KeyT T, int take,
                                             int base, int* s_gt, int* s_eq) {
    constexpr int kW = kScoreThreads / 32;
    constexpr int kRowsPerWarp = kScoreChunk / kW;  // 512
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    {
        const int start = chunk * kScoreChunk;
        const int end = min(start + kScoreChunk, it.n);
        const KeyT* keys = (sizeof(KeyT) == 2 ? (const KeyT*)(a.key16 + (size_t)item * a.nmax)
                                              : (const KeyT*)(a.key64 + (size_t)item * a.nmax));
        const int w0 = start + warp * kRowsPerWarp, w1 = min(w0 + kRowsPerWarp, end);
        int gt = 0, eq = 0;
        for (int r = w0 + lane; r < w1; r += 32) {
            const KeyT kv = keys[r];
            gt += kv > T;
            eq += kv == T;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            gt += __shfl_xor_sync(0xffffffffu, gt, o);
            eq += __shfl_xor_sync(0xffffffffu, eq, o);
        }
        if (lane == 0) {
            s_gt[warp] = gt;
            s_eq[warp] = eq;
        }
        __syncthreads();
        int eq_before = 0, pos = base;
        for (int w = 0; w < warp; ++w) {
            pos += s_gt[w] + max(0, min(s_eq[w], take - eq_before));
            eq_before += s_eq[w];
        }
        for (int r0 = w0; r0 < w1; r0 += 32) {
            const int r = r0 + lane;
            const bool valid = r < w1;
            const KeyT kv = valid ? keys[r] : (KeyT)0;
            const bool is_eq = valid && kv == T;
            const unsigned eqm = __ballot_sync(0xffffffffu, is_eq);
            const bool sel = (valid && kv > T) || (is_eq && eq_before + __popc(eqm & lt) < take);
            const unsigned selm = __ballot_sync(0xffffffffu, sel);
            if (sel) {
                const int p = pos + __popc(selm & lt);
                it.out_idx[p] = r;
                if (it.out_score) it.out_score[p] = key_score<KeyT>(kv);
            }
            pos += __popc(selm);
            eq_before += __popc(eqm);
        }
        __syncthreads();
    }
}

template <typename KeyT>
__device__ __forceinline__ void compact_unit(const SelArgs& a, int item, int chunk, int* s_gt, int* s_eq) {
    const SelItem it = a.items[item];
    if (chunk * kScoreChunk >= it.n) return;
    compact_body<KeyT>(a, it, item, chunk, (KeyT)a.thresh[item], a.chunk_take[(size_t)item * a.max_chunks + chunk],
                       a.chunk_base[(size_t)item * a.max_chunks + chunk], s_gt, s_eq);
}

// Max bins of the fused quota (hash_bits <= 512).
constexpr int kMaxBins = 64 * kMaxHashWords + 1;

// threshold_item's result for ONE chunk, recomputed by that chunk's compaction
// CTA from the item's chunk histograms (sign-hash decode, items of <= 64
// chunks): one pass keeps, per bin, the item total, the sum over the chunks
// before this one and this chunk's own count. Then T = the k-th largest S,
// gt_before = sum over bins > T of the earlier chunks' counts, eq_before = the
// earlier chunks' ties; the greedy tie quotas of the earlier chunks sum to
// min(eq_before, need), so
//   base = gt_before + min(eq_before, need),
//   take = max(0, min(this chunk's ties, need - eq_before)),
// exactly the values threshold_item writes. Every CTA of an item derives the
// same T from the same counts: no cross-CTA handoff, and no separate
// threshold launch (one kernel boundary less in front of each gather: in the
// step graph a boundary waits for the host reads the running gather has
// queued, profiles/r2/README.md).
__device__ __forceinline__ void chunk_quota(const SelArgs& a, int item, int chunk, int nch, uint32_t* tot,
                                            uint32_t* pre, uint32_t* cur, int* sts, int* red, int& T, int& take,
                                            int& base) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint32_t* hist = a.chunk_hist + (size_t)item * a.max_chunks * a.nb;
    for (int b = threadIdx.x; b < a.nb; b += blockDim.x) {
        uint32_t s = 0, p = 0, x = 0;
#pragma unroll 8
        for (int c = 0; c < nch; ++c) {
            const uint32_t h = __ldcg(hist + (size_t)c * a.nb + b);
            if (c == chunk) {
                p = s;
                x = h;
            }
            s += h;
        }
        tot[b] = s;
        pre[b] = p;
        cur[b] = x;
    }
    __syncthreads();
    if (warp == 0) threshold_walk(a, tot, sts);
    __syncthreads();
    T = sts[0];
    const int need = a.k - sts[1];
    int g = 0;
    for (int b = threadIdx.x; b < a.nb; b += blockDim.x) g += b > T ? (int)pre[b] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
    if (lane == 0) red[warp] = g;
    __syncthreads();
    int gt_before = 0;
    for (int w = 0; w < nwarps; ++w) gt_before += red[w];
    const int eq_before = T >= 0 ? (int)pre[T] : 0, mine = T >= 0 ? (int)cur[T] : 0;
    base = gt_before + min(eq_before, need);
    take = max(0, min(mine, need - eq_before));
    __syncthreads();  // tot/pre/cur/red are reused by the next unit
}


}  // namespace clo
