// select.cu — K1 `score_select`: key scoring and bit-exact top-k selection.
// See select.cuh for the semantics and the reference functions restated.
#include <cub/block/block_scan.cuh>

#include <cstdlib>
#include <string>

#include "select.cuh"
#include "select_dev.cuh"
#include "reconcile.cuh"

namespace clo {

namespace {

constexpr int kWarps = kScoreThreads / 32;
constexpr int kRowsPerThread = kScoreChunk / kScoreThreads;  // 16


// ---------------------------------------------------------------- sign-hash

// S(i) = max_j (bits - popcount(q_j ^ code_i)) (hamming_affinity,
// retrieval.cpp:27-31) for every key of one 4096-row chunk, written as u16,
// plus the chunk's histogram of S (per-warp smem histograms, then summed).
template <int W>
__global__ void __launch_bounds__(kScoreThreads) score_signhash_kernel(SelArgs a) {
    extern __shared__ uint32_t smem[];
    uint32_t* whist = smem;                                   // [kWarps][nb]
    uint64_t* qb = reinterpret_cast<uint64_t*>(smem + kWarps * a.nb + (kWarps * a.nb & 1));
    const int units = *a.count * a.max_chunks;
    const int warp = threadIdx.x >> 5;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / a.max_chunks, chunk = u % a.max_chunks;
        const SelItem it = a.items[item];
        const int start = chunk * kScoreChunk;
        if (start >= it.n) continue;
        const int end = min(start + kScoreChunk, it.n);
        for (int i = threadIdx.x; i < kWarps * a.nb; i += blockDim.x) whist[i] = 0;
        for (int i = threadIdx.x; i < a.m * W; i += blockDim.x) {
            const int j = i / W, w = i % W;
            qb[i] = a.qbits[((size_t)item * a.m + j) * a.words + w];
        }
        __syncthreads();
        const uint64_t* codes = it.codes;
        uint16_t* keys = a.key16 + (size_t)item * a.nmax;
        uint32_t* myhist = whist + warp * a.nb;
#pragma unroll 4
        for (int r = start + threadIdx.x; r < end; r += kScoreThreads) {
            uint64_t c[W];
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(codes + (size_t)r * W);
            if constexpr (W % 2 == 0) {
#pragma unroll
                for (int w = 0; w < W / 2; ++w) {
                    ulonglong2 v = __ldg(src + w);
                    c[2 * w] = v.x;
                    c[2 * w + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int w = 0; w < W; ++w) c[w] = __ldg(codes + (size_t)r * W + w);
            }
            int best = 0;
            for (int j = 0; j < a.m; ++j) {
                int dist = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) dist += __popcll(c[w] ^ qb[j * W + w]);
                best = max(best, a.bits - dist);
            }
            keys[r] = static_cast<uint16_t>(best);
            atomicAdd(&myhist[best], 1u);
        }
        __syncthreads();
        uint32_t* out = a.chunk_hist + ((size_t)item * a.max_chunks + chunk) * a.nb;
        for (int b = threadIdx.x; b < a.nb; b += blockDim.x) {
            uint32_t s = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s += whist[w * a.nb + b];
            out[b] = s;
        }
        __syncthreads();
    }
}

// Same scoring with the codes streamed by the TMA engine: each 4096-row chunk
// is four 1024-row pieces, bulk-copied (cp.async.bulk, one instruction per
// piece from thread 0) into a 2-stage shared-memory ring while the CTA scores
// the previous piece, so every CTA keeps a whole piece (32 KiB at 256 bits) in
// flight instead of a few loads per thread. Rows of a partial last piece that
// fall past its last whole 16 bytes are read from global directly.
constexpr int kPieceRows = 1024;
constexpr int kPieces = kScoreChunk / kPieceRows;  // 4

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Row r's code words from the staged piece: 16-byte loads, the two halves of
// a row visited in rotated order ((r / (128 / row bytes)) mod chunks) so the
// eight threads of each shared-memory phase hit eight different 16-byte bank
// groups (plain row order collides 2-way at 32-byte rows).
template <int W>
__device__ __forceinline__ void load_code_row(const uint64_t* st, int r, uint64_t (&c)[W]) {
    if constexpr (W % 2 == 0 && W * 8 <= 128) {
        constexpr int kChunks = W / 2;
        constexpr int kPerGroup = 128 / (W * 8);
        const int rot = (r / kPerGroup) % kChunks;
        const ulonglong2* row = reinterpret_cast<const ulonglong2*>(st + (size_t)r * W);
        ulonglong2 v[kChunks];
#pragma unroll
        for (int i = 0; i < kChunks; ++i) v[i] = row[(i + rot) % kChunks];  // v[i] = chunk (i + rot)
#pragma unroll
        for (int ch = 0; ch < kChunks; ++ch) {  // register selects, no local-memory indexing
            ulonglong2 x = v[0];
#pragma unroll
            for (int i = 1; i < kChunks; ++i)
                if ((i + rot) % kChunks == ch) x = v[i];
            c[2 * ch] = x.x;
            c[2 * ch + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w) c[w] = st[(size_t)r * W + w];
    }
}

// S = max_j (bits - popcount(q_j ^ c)); M > 0: group size known at compile
// time (query words in registers), M == 0: runtime a.m, words from shared memory.
template <int W, int M>
__device__ __forceinline__ int score_row(const uint64_t (&c)[W], const uint64_t* qb, const uint64_t (&qr)[M > 0 ? M : 1][W],
                                         int m, int bits) {
    int best = 0;
    if constexpr (M > 0) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
            int dist = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) dist += __popcll(c[w] ^ qr[j][w]);
            best = max(best, bits - dist);
        }
    } else {
        for (int j = 0; j < m; ++j) {
            int dist = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) dist += __popcll(c[w] ^ qb[j * W + w]);
            best = max(best, bits - dist);
        }
    }
    return best;
}

template <int W, int M>
__global__ void __launch_bounds__(kScoreThreads) score_signhash_tma_kernel(SelArgs a, int agg) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* stage = reinterpret_cast<uint64_t*>(sm);                              // [2][kPieceRows*W]
    uint32_t* whist = reinterpret_cast<uint32_t*>(sm + 2 * kPieceRows * W * 8);     // [kWarps][nb]
    uint64_t* qb = reinterpret_cast<uint64_t*>(sm + 2 * kPieceRows * W * 8 +
                                               ((size_t)kWarps * a.nb * 4 + 7) / 8 * 8);  // [m][W]
    uint32_t* thr_sm = reinterpret_cast<uint32_t*>(qb + a.m * W);                        // threshold_item's
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int s_last, s_sts[2];
    const int units = *a.count * a.max_chunks;
    const int mine = units > (int)blockIdx.x ? (units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = mine * kPieces;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // rows [row0, row0 + rows) of piece i; rows = 0 for pieces past the item's end
    auto piece = [&](int i, int& item, int& chunk, int& row0, int& rows) {
        const int u = blockIdx.x + (i / kPieces) * gridDim.x;
        item = u / a.max_chunks;
        chunk = u % a.max_chunks;
        row0 = chunk * kScoreChunk + (i % kPieces) * kPieceRows;
        rows = max(0, min(kPieceRows, a.items[item].n - row0));
    };
    auto issue = [&](int i) {  // thread 0
        int item, chunk, row0, rows;
        piece(i, item, chunk, row0, rows);
        const uint64_t* src = a.items[item].codes + (size_t)row0 * W;
        // cp.async.bulk needs a 16-byte aligned source: a misaligned piece
        // (caller-provided codes at an odd word offset) is read by LSU loads
        const uint32_t bytes = (reinterpret_cast<uintptr_t>(src) & 15) ? 0u : (uint32_t)rows * W * 8 / 16 * 16;
        uint64_t* b = &bar[i & 1];
        if (bytes) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(stage + (size_t)(i & 1) * kPieceRows * W)),
                "l"(src), "r"(bytes), "r"(smem_addr(b))
                : "memory");
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
        }
    };
    if (threadIdx.x == 0 && total > 0) issue(0);
    for (int i = 0; i < total; ++i) {
        int item, chunk, row0, rows;
        piece(i, item, chunk, row0, rows);
        const int p = i % kPieces;
        if (p == 0) {  // a new chunk: its histogram and the item's query bits
            for (int x = threadIdx.x; x < kWarps * a.nb; x += blockDim.x) whist[x] = 0;
            for (int x = threadIdx.x; x < a.m * W; x += blockDim.x) {
                const int j = x / W, w = x % W;
                qb[x] = a.qbits[((size_t)item * a.m + j) * a.words + w];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0 && i + 1 < total) issue(i + 1);
        asm volatile(
            "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_addr(&bar[i & 1])),
            "r"((i >> 1) & 1)
            : "memory");
        const uint64_t* st = stage + (size_t)(i & 1) * kPieceRows * W;
        const uint64_t* codes = a.items[item].codes;
        const bool staged = (reinterpret_cast<uintptr_t>(codes + (size_t)row0 * W) & 15) == 0;
        const int copied = staged ? rows * W * 8 / 16 * 16 / (W * 8) : 0;  // whole rows in smem
        uint16_t* keys = a.key16 + (size_t)item * a.nmax;
        uint32_t* myhist = whist + warp * a.nb;
        uint64_t qr[M > 0 ? M : 1][W];
        if constexpr (M > 0) {
#pragma unroll
            for (int j = 0; j < M; ++j)
#pragma unroll
                for (int w = 0; w < W; ++w) qr[j][w] = qb[j * W + w];
        }
#pragma unroll 4
        for (int r = threadIdx.x; r < rows; r += kScoreThreads) {
            uint64_t c[W];
            if (r < copied) {
                load_code_row<W>(st, r, c);
            } else {
#pragma unroll
                for (int w = 0; w < W; ++w) c[w] = __ldg(codes + (size_t)(row0 + r) * W + w);
            }
            const int best = score_row<W, M>(c, qb, qr, a.m, a.bits);
            keys[row0 + r] = static_cast<uint16_t>(best);
            if (agg) {  // warp-aggregated: one shared atomic per distinct score
                const unsigned act = __activemask();
                const unsigned same = __match_any_sync(act, best);
                if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&myhist[best], (uint32_t)__popc(same));
            } else {
                atomicAdd(&myhist[best], 1u);
            }
        }
        __syncthreads();  // stage i & 1 is free; the chunk's histogram is complete after its last piece
        if (p == kPieces - 1) {
            uint32_t* out = a.chunk_hist + ((size_t)item * a.max_chunks + chunk) * a.nb;
            for (int b = threadIdx.x; b < a.nb; b += blockDim.x) {
                uint32_t sum = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) sum += whist[w * a.nb + b];
                out[b] = sum;
            }
            __syncthreads();
            // the CTA finishing the item's last chunk computes its threshold
            // (threshold_signhash_kernel's work, without another launch)
            const int nch = num_chunks(a.items[item].n);
            if (a.item_done && chunk < nch) {
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0) s_last = atomicAdd(&a.item_done[item], 1) == nch - 1;
                __syncthreads();
                if (s_last) {
                    __threadfence();
                    threshold_item(a, item, thr_sm, s_sts);
                    if (threadIdx.x == 0) a.item_done[item] = 0;  // ready for the next layer
                }
            }
        }
    }
}

// Per item: T = k-th largest S (ties resolved later by index), then each
// chunk's output offset and how many of its S == T ties it keeps.
__global__ void __launch_bounds__(1024) threshold_signhash_kernel(SelArgs a) {
    extern __shared__ uint32_t smem[];
    __shared__ int sts[2];
    const int count = *a.count;
    for (int item = blockIdx.x; item < count; item += gridDim.x) threshold_item(a, item, smem, sts);
}

// ---------------------------------------------------------------- compaction

template <typename KeyT>
__global__ void __launch_bounds__(kScoreThreads) compact_kernel(SelArgs a) {
    __shared__ int s_gt[kWarps], s_eq[kWarps];
    const int units = *a.count * a.max_chunks;
    for (int u = blockIdx.x; u < units; u += gridDim.x) compact_unit<KeyT>(a, u / a.max_chunks, u % a.max_chunks, s_gt, s_eq);
}

// Compaction with the threshold recomputed per CTA (chunk_quota): sign-hash
// items of <= quota_max_chunks() chunks, one launch instead of threshold +
// compaction (each CTA reads its item's nch x nb histogram words from L2).
int quota_max_chunks() {  // CLO_QUOTA_MAX_CHUNKS (experiment switch), default 64
    static const int v = [] {
        const char* e = getenv("CLO_QUOTA_MAX_CHUNKS");
        return e && atoi(e) > 0 ? atoi(e) : 64;
    }();
    return v;
}
__global__ void __launch_bounds__(kScoreThreads) compact_quota_kernel(SelArgs a) {
    __shared__ int s_gt[kWarps], s_eq[kWarps], s_sts[2], s_red[kWarps];
    __shared__ uint32_t s_tot[kMaxBins], s_pre[kMaxBins], s_cur[kMaxBins];
    const int units = *a.count * a.max_chunks;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / a.max_chunks, chunk = u % a.max_chunks;
        const SelItem it = a.items[item];
        if (chunk * kScoreChunk >= it.n) continue;
        int T, take, base;
        chunk_quota(a, item, chunk, num_chunks(it.n), s_tot, s_pre, s_cur, s_sts, s_red, T, take, base);
        compact_body<uint16_t>(a, it, item, chunk, (uint16_t)T, take, base, s_gt, s_eq);
    }
}

// Compaction of the offloaded heads whose CTA finishing an item's last chunk
// then reconciles that item's entry (reconcile_kernel's work, reconcile.cuh):
// the fetch list is ready when this kernel ends, one launch earlier.
__global__ void __launch_bounds__(kScoreThreads) compact_reconcile_kernel(SelArgs a, ReconcileArgs r) {
    __shared__ int s_gt[kWarps], s_eq[kWarps], s_last;
    __shared__ ReconcileSmem<kScoreThreads> rsm;
    extern __shared__ int32_t rs[];  // [4][k]
    int* done = a.item_done + a.max_items;
    const int units = *a.count * a.max_chunks;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / a.max_chunks, chunk = u % a.max_chunks;
        const int nch = num_chunks(a.items[item].n);
        if (chunk >= nch) continue;
        compact_unit<uint16_t>(a, item, chunk, s_gt, s_eq);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(&done[item], 1) == nch - 1;
        __syncthreads();
        if (s_last) {
            __threadfence();
            reconcile_item<kScoreThreads>(r, item, rs, rsm);
            if (threadIdx.x == 0) done[item] = 0;
        }
    }
}

// -------------------------------------------------------------------- exact

// S(i) = max_j sum_c q_j[c]*K[i][c] (retrieval.cpp:101-106, sequential IEEE
// double without FMA) -> orderable u64 key. Chunk 0 of each item also resets
// the radix state.
template <typename T>
__global__ void __launch_bounds__(kScoreThreads) score_exact_kernel(SelArgs a) {
    extern __shared__ double qs[];  // [m][d]
    const int units = *a.count * a.max_chunks;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / a.max_chunks, chunk = u % a.max_chunks;
        const SelItem it = a.items[item];
        const int start = chunk * kScoreChunk;
        if (start >= it.n) continue;
        const int end = min(start + kScoreChunk, it.n);
        if (chunk == 0) {
            for (int b = threadIdx.x; b < 256; b += blockDim.x) a.radix_hist[(size_t)item * 256 + b] = 0;
            if (threadIdx.x == 0) {
                a.need[item] = a.k;
                a.thresh[item] = 0;
            }
        }
        for (int i = threadIdx.x; i < a.m * a.d; i += blockDim.x)
            qs[i] = a.q64[(size_t)item * a.m * a.d + i];
        __syncthreads();
        const T* rows = static_cast<const T*>(it.rows);
        uint64_t* keys = a.key64 + (size_t)item * a.nmax;
        for (int r = start + threadIdx.x; r < end; r += blockDim.x) {
            const T* kr = rows + (size_t)r * a.d;
            double best = 0.0;
            for (int j = 0; j < a.m; ++j) {
                double s = 0.0;
                for (int c = 0; c < a.d; ++c) s = dmac(s, qs[j * a.d + c], to_f64<T>(kr[c]));
                if (j == 0 || s > best) best = s;
            }
            keys[r] = orderable_key(best);
        }
        __syncthreads();
    }
}

// One MSB-first 8-bit radix pass: histogram digit `shift` of the keys whose
// higher digits equal the prefix found so far.
__global__ void __launch_bounds__(kScoreThreads) radix_hist_kernel(SelArgs a, int shift) {
    __shared__ uint32_t h[256];
    const int units = *a.count * a.max_chunks;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / a.max_chunks, chunk = u % a.max_chunks;
        const SelItem it = a.items[item];
        const int start = chunk * kScoreChunk;
        if (start >= it.n) continue;
        const int end = min(start + kScoreChunk, it.n);
        for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
        __syncthreads();
        const uint64_t prefix = a.thresh[item];
        const uint64_t* keys = a.key64 + (size_t)item * a.nmax;
        for (int r = start + threadIdx.x; r < end; r += blockDim.x) {
            const uint64_t key = keys[r];
            if (shift == 56 || ((key ^ prefix) >> (shift + 8)) == 0)
                atomicAdd(&h[(key >> shift) & 255], 1u);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < 256; b += blockDim.x)
            if (h[b]) atomicAdd(&a.radix_hist[(size_t)item * 256 + b], h[b]);
        __syncthreads();
    }
}

// Picks the digit holding the need-th largest key, narrows the prefix and
// resets the histogram for the next pass.
__global__ void radix_pick_kernel(SelArgs a, int shift) {
    const int count = *a.count;
    const int lane = threadIdx.x;
    for (int item = blockIdx.x; item < count; item += gridDim.x) {
        uint32_t* h = a.radix_hist + (size_t)item * 256;
        const int need = a.need[item];
        int running = 0, D = -1, above = 0;
        for (int top = 255; top >= 0 && D < 0; top -= 32) {
            const int b = top - lane;
            const int v = (int)h[b];
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, running + incl >= need);
            if (hit) {
                const int first = __ffs(hit) - 1;
                above = running + __shfl_sync(0xffffffffu, incl - v, first);
                D = top - first;
            }
            running += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        for (int b = lane; b < 256; b += 32) h[b] = 0;
        if (lane == 0) {
            a.need[item] = need - above;
            a.thresh[item] |= (uint64_t)D << shift;
        }
    }
}

// Per chunk: count keys > T and == T (exact path; T complete after 8 passes).
__global__ void __launch_bounds__(kScoreThreads) count_chunks_kernel(SelArgs a) {
    using Scan = cub::BlockScan<int, kScoreThreads>;
    __shared__ int sg[kWarps], se[kWarps];
    const int units = *a.count * a.max_chunks;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / a.max_chunks, chunk = u % a.max_chunks;
        const SelItem it = a.items[item];
        const int start = chunk * kScoreChunk;
        if (start >= it.n) continue;
        const int end = min(start + kScoreChunk, it.n);
        const uint64_t T = a.thresh[item];
        const uint64_t* keys = a.key64 + (size_t)item * a.nmax;
        int g = 0, e = 0;
        for (int r = start + threadIdx.x; r < end; r += blockDim.x) {
            const uint64_t key = keys[r];
            g += key > T;
            e += key == T;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            g += __shfl_xor_sync(0xffffffffu, g, o);
            e += __shfl_xor_sync(0xffffffffu, e, o);
        }
        if ((threadIdx.x & 31) == 0) {
            sg[threadIdx.x >> 5] = g;
            se[threadIdx.x >> 5] = e;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int G = 0, E = 0;
            for (int w = 0; w < kWarps; ++w) {
                G += sg[w];
                E += se[w];
            }
            uint32_t* out = a.chunk_hist + ((size_t)item * a.max_chunks + chunk) * 2;
            out[0] = G;
            out[1] = E;
        }
        __syncthreads();
    }
}

// Per item: chunk offsets and tie quotas from the (gt, eq) counts.
__global__ void chunk_prefix_kernel(SelArgs a) {
    const int count = *a.count;
    const int lane = threadIdx.x;
    for (int item = blockIdx.x; item < count; item += gridDim.x) {
        const SelItem it = a.items[item];
        const int nch = num_chunks(it.n);
        const int need_eq = a.need[item];
        int base_run = 0, eq_run = 0;
        for (int c0 = 0; c0 < nch; c0 += 32) {
            const int c = c0 + lane;
            const uint32_t* h = a.chunk_hist + ((size_t)item * a.max_chunks + c) * 2;
            const int g = c < nch ? (int)h[0] : 0;
            const int e = c < nch ? (int)h[1] : 0;
            int ie = e;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, ie, o);
                if (lane >= o) ie += t;
            }
            const int take = max(0, min(e, need_eq - (eq_run + ie - e)));
            const int contrib = g + take;
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
    }
}

}  // namespace

// Group sizes with a compile-time kernel (query words in registers); others
// use the runtime-m kernel.
template <int W>
void launch_score_tma(const SelArgs& a, int grid, size_t sm, int agg, cudaStream_t stream) {
    switch (a.m) {
#define CLO_M(MM)                                                                                          \
    case MM:                                                                                               \
        cudaFuncSetAttribute(score_signhash_tma_kernel<W, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)sm);                                                                     \
        score_signhash_tma_kernel<W, MM><<<grid, kScoreThreads, sm, stream>>>(a, agg);                     \
        return;
        CLO_M(1) CLO_M(2) CLO_M(4) CLO_M(5) CLO_M(8)
#undef CLO_M
        default:
            cudaFuncSetAttribute(score_signhash_tma_kernel<W, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            score_signhash_tma_kernel<W, 0><<<grid, kScoreThreads, sm, stream>>>(a, agg);
    }
}

int launch_select_signhash(const SelArgs& a, cudaStream_t stream, const ReconcileArgs* rec) {
    const size_t sm_score = (size_t)kWarps * a.nb * 4 + 8 + (size_t)a.m * a.words * 8;
    static const bool tma = [] {  // CLO_SCORE=lsu: the register-load kernel
        const char* e = getenv("CLO_SCORE");
        return !(e && std::string(e) == "lsu");
    }();
    const size_t sm_tma = 2 * (size_t)kPieceRows * a.words * 8 + ((size_t)kWarps * a.nb * 4 + 7) / 8 * 8 +
                          (size_t)a.m * a.words * 8 + ((size_t)a.nb + 2 * (size_t)a.max_chunks) * 4;
    static const int grid_cap = [] {  // CLO_SCORE_GRID: experiment switch
        const char* e = getenv("CLO_SCORE_GRID");
        return e && atoi(e) > 0 ? atoi(e) : 8 * kNumSMs;  // measured: more CTAs than resident slots balance the chunks
    }();
    const int grid_tma = a.grid < grid_cap ? a.grid : grid_cap;
    static const int hist_agg = [] {  // CLO_SCORE_AGG=1: warp-aggregated histogram atomics
        const char* e = getenv("CLO_SCORE_AGG");
        return e && atoi(e) == 1 ? 1 : 0;
    }();
    switch (a.words) {
#define CLO_W(W)                                                                                            \
    case W:                                                                                                 \
        if (tma) {                                                                                          \
            launch_score_tma<W>(a, grid_tma, sm_tma, hist_agg, stream);                                     \
        } else {                                                                                            \
            score_signhash_kernel<W><<<a.grid, kScoreThreads, sm_score, stream>>>(a);                       \
        }                                                                                                   \
        break;
        CLO_W(1) CLO_W(2) CLO_W(3) CLO_W(4) CLO_W(5) CLO_W(6) CLO_W(7) CLO_W(8)
#undef CLO_W
        default:
            break;
    }
    const size_t sm_thr = (size_t)a.nb * 4 + (size_t)a.max_chunks * 8;
    // one CTA per item (the kernels grid-stride over *count <= max_items)
    const int items_grid = a.max_items > 0 ? (a.max_items < 1024 ? a.max_items : 1024) : (a.grid < 1024 ? a.grid : 1024);
    const bool tma_chained = tma && a.item_done;  // the score kernel's last chunk per item ran the threshold
    static const bool quota = [] {  // CLO_COMPACT_QUOTA=0: separate threshold launch
        const char* e = getenv("CLO_COMPACT_QUOTA");
        return !(e && e[0] == '0');
    }();
    if (quota && !tma_chained && !rec && a.max_chunks <= quota_max_chunks() && a.nb <= kMaxBins) {
        compact_quota_kernel<<<a.grid, kScoreThreads, 0, stream>>>(a);
        return 2;
    }
    if (!tma_chained) threshold_signhash_kernel<<<items_grid, 1024, sm_thr, stream>>>(a);
    if (rec && a.item_done) {
        const size_t sm_rec = 4 * sizeof(int32_t) * (size_t)a.k;
        cudaFuncSetAttribute(compact_reconcile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_rec);
        compact_reconcile_kernel<<<a.grid, kScoreThreads, sm_rec, stream>>>(a, *rec);
    } else {
        compact_kernel<uint16_t><<<a.grid, kScoreThreads, 0, stream>>>(a);
    }
    return tma_chained ? 2 : 3;
}

void launch_select_exact(const SelArgs& a, cudaStream_t stream) {
    const size_t sm_q = (size_t)a.m * a.d * 8;
    switch (a.dtype) {
        case kBF16:
            score_exact_kernel<__nv_bfloat16><<<a.grid, kScoreThreads, sm_q, stream>>>(a);
            break;
        case kF32:
            score_exact_kernel<float><<<a.grid, kScoreThreads, sm_q, stream>>>(a);
            break;
        default:
            score_exact_kernel<double><<<a.grid, kScoreThreads, sm_q, stream>>>(a);
            break;
    }
    // one CTA per item (the kernels grid-stride over *count <= max_items)
    const int items_grid = a.max_items > 0 ? (a.max_items < 1024 ? a.max_items : 1024) : (a.grid < 1024 ? a.grid : 1024);
    for (int shift = 56; shift >= 0; shift -= 8) {
        radix_hist_kernel<<<a.grid, kScoreThreads, 0, stream>>>(a, shift);
        radix_pick_kernel<<<items_grid, 32, 0, stream>>>(a, shift);
    }
    count_chunks_kernel<<<a.grid, kScoreThreads, 0, stream>>>(a);
    chunk_prefix_kernel<<<items_grid, 32, 0, stream>>>(a);
    compact_kernel<uint64_t><<<a.grid, kScoreThreads, 0, stream>>>(a);
}

namespace {
__global__ void __launch_bounds__(256) hash_queries_kernel(const double* q64, int m, int d,
                                                           const double* proj_t, int bits,
                                                           int words, uint64_t* qbits) {
    extern __shared__ double qs[];
    for (int i = threadIdx.x; i < m * d; i += blockDim.x) qs[i] = q64[i];
    __syncthreads();
    hash_queries_block(qs, m, d, proj_t, bits, words, qbits);
}
}  // namespace

void launch_hash_queries(const double* q64, int m, int d, const double* proj_t, int bits,
                         int words, uint64_t* qbits, cudaStream_t stream) {
    hash_queries_kernel<<<1, 256, (size_t)m * d * sizeof(double), stream>>>(q64, m, d, proj_t,
                                                                            bits, words, qbits);
}

}  // namespace clo
