// select.cuh — key scoring + top-k selection (K1 `score_select`).
//
// Semantics: DecodeEngine::group_topk (engine.cpp:211-223) = m calls of
// retrieve_scored (retrieval.cpp:90-125, select_topk :33-46) followed by
// merge_group_topk (similarity_cache.cpp:180-201). That equals ONE top-k over
// S(i) = max_j score_j(i) under (S desc, i asc), reported ascending
// (DESIGN.md §3 has the proof). The GPU computes it as:
//   score      S(i) per key -> u16 (sign-hash, S in [0, bits]) or orderable
//              u64 (exact, S a double), plus per-chunk histograms
//   threshold  sign-hash: T = the k-th largest S from the histograms;
//              exact: 8 MSB-first radix passes over the u64 keys
//   compact    keep S > T, plus the first `need` ties S == T in index order,
//              written ascending at per-chunk offsets (a two-level scan)
// Every result is an integer function of the bit-exact scores, so indices
// match the reference bit for bit.
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace clo {

struct SelItem {
    int seg;                // engine segment (or 0 for op-level calls)
    int n;                  // pool size: rows [0, n) are candidates
    const void* rows;       // exact: K rows [n][d] of dtype
    const uint64_t* codes;  // sign-hash: bits [n][words]
    int32_t* out_idx;       // [k] ascending selection
    double* out_score;      // [k] S(out_idx) or nullptr
};

struct SelArgs {
    const SelItem* items;
    const int* count;       // number of valid items
    int m, d, k, bits, words, nb, nmax, max_chunks, dtype;
    const double* q64;      // [item][m][d]
    const uint64_t* qbits;  // [item][m][words]
    uint16_t* key16;        // [item][nmax]
    uint64_t* key64;        // [item][nmax]
    uint32_t* chunk_hist;   // [item][max_chunks][nb]   (exact: [..][2] gt/eq)
    int* chunk_base;        // [item][max_chunks]
    int* chunk_take;        // [item][max_chunks]
    uint64_t* thresh;       // [item]
    int* need;              // [item]
    uint32_t* radix_hist;   // [item][256]
    int grid;               // CTAs for the grid-stride kernels
    int max_items;          // host-side upper bound of *count (sizes the per-item grids)
    int* item_done;         // [2][max_items] zeroed chunk counters, or null: the CTA finishing an item's
                            // last score chunk computes its threshold, the one finishing its last
                            // compaction chunk reconciles it (no separate threshold / reconcile launch)
};

// Host launchers (select.cu). All enqueue on `stream`; no host sync.
struct ReconcileArgs;
// rec: offloaded heads in a decode step — the compaction kernel also reconciles
// their entries (needs a.item_done); null: compaction only
// Returns the number of kernels launched.
int launch_select_signhash(const SelArgs& a, cudaStream_t stream, const ReconcileArgs* rec = nullptr);
void launch_select_exact(const SelArgs& a, cudaStream_t stream);
// Query sign bits for op-level calls (one CTA): q64 [m][d] -> qbits [m][words].
void launch_hash_queries(const double* q64, int m, int d, const double* proj_t, int bits,
                         int words, uint64_t* qbits, cudaStream_t stream);

// Sign bits of M queries (append_sign_row semantics, retrieval.cpp:14-25,
// as used for the query bits at :113-119): bit b = (sum_c P[b][c]*q[c]) >= 0
// summed sequentially in IEEE double. Called by a whole CTA (blockDim.x a
// multiple of 32). q64 [M][d] (smem), proj_t [d][bits] -> qbits [M][words].
// M is a template parameter so no FP64 work is issued for absent members.
// Sequential sign-hash dot products for a compile-time head dim: s_j +=
// P^T[c][b] * q_j[c] for c = 0..D-1 in source order (separately rounded
// multiply and add, bit-exact with the reference's scalar loop). Fully
// unrolled, no bounds predicates, 32 P^T loads in flight per batch; the
// products do not depend on the accumulators, so only the DADD chain is
// serial.
#ifndef CLO_HASH_BATCH
#define CLO_HASH_BATCH 32
#endif
template <int D, int M>
__device__ __forceinline__ void signhash_chain(const double* __restrict__ col, size_t stride, const double* q,
                                               int qstride, double (&s)[M]) {
    constexpr int kB = CLO_HASH_BATCH;  // P^T loads in flight per thread
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += kB) {
        double p[kB];
#pragma unroll
        for (int i = 0; i < kB; ++i) p[i] = __ldg(col + (size_t)(c0 + i) * stride);
#pragma unroll
        for (int i = 0; i < kB; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) s[j] = dmac(s[j], p[i], q[j * qstride + c0 + i]);
    }
}

template <int M, int D>
__device__ __forceinline__ void hash_queries_block_md(const double* q64, const double* proj_t, int bits, int words,
                                                      uint64_t* qbits_out) {
    uint32_t* out32 = reinterpret_cast<uint32_t*>(qbits_out);
    const int total = words * 64;
    for (int b0 = 0; b0 < total; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        double s[M];
#pragma unroll
        for (int j = 0; j < M; ++j) s[j] = 0.0;
        if (b < bits) signhash_chain<D, M>(proj_t + b, (size_t)bits, q64, D, s);
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const unsigned bal = __ballot_sync(0xffffffffu, b < bits && s[j] >= 0.0);
            if ((threadIdx.x & 31) == 0 && b < total) out32[j * words * 2 + (b >> 5)] = bal;
        }
    }
}

template <int M>
__device__ __forceinline__ void hash_queries_block_m(const double* q64, int d, const double* proj_t,
                                                     int bits, int words, uint64_t* qbits_out) {
    if (d == 128) return hash_queries_block_md<M, 128>(q64, proj_t, bits, words, qbits_out);
    if (d == 64) return hash_queries_block_md<M, 64>(q64, proj_t, bits, words, qbits_out);
    uint32_t* out32 = reinterpret_cast<uint32_t*>(qbits_out);
    const int total = words * 64;
    for (int b0 = 0; b0 < total; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        double s[M];
#pragma unroll
        for (int j = 0; j < M; ++j) s[j] = 0.0;
        if (b < bits) {
            // P^T loads batched 32 deep so the sequential DADD chains are not
            // serialised behind one L2 round trip per element
            for (int c0 = 0; c0 < d; c0 += 32) {
                double p[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) p[i] = c0 + i < d ? proj_t[(size_t)(c0 + i) * bits + b] : 0.0;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (c0 + i < d) {
#pragma unroll
                        for (int j = 0; j < M; ++j) s[j] = dmac(s[j], p[i], q64[j * d + c0 + i]);
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const unsigned bal = __ballot_sync(0xffffffffu, b < bits && s[j] >= 0.0);
            if ((threadIdx.x & 31) == 0 && b < total) out32[j * words * 2 + (b >> 5)] = bal;
        }
    }
}

__device__ __forceinline__ void hash_queries_block(const double* q64, int m, int d,
                                                   const double* proj_t, int bits, int words,
                                                   uint64_t* qbits_out) {
    switch (m) {
#define CLO_HQ(MM) \
    case MM: hash_queries_block_m<MM>(q64, d, proj_t, bits, words, qbits_out); return;
        CLO_HQ(1) CLO_HQ(2) CLO_HQ(3) CLO_HQ(4) CLO_HQ(5) CLO_HQ(6) CLO_HQ(7) CLO_HQ(8)
#undef CLO_HQ
        default:
            for (int j = 0; j < m; ++j)  // large groups: one member at a time
                hash_queries_block_m<1>(q64 + (size_t)j * d, d, proj_t, bits, words, qbits_out + (size_t)j * words);
    }
}

}  // namespace clo
