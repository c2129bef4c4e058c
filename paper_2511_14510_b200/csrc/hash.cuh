// hash.cuh — decode-time sign-hash of a few vectors against one projection
// word slice staged in shared memory.
//
// append_sign_row / the query bits (retrieval.cpp:14-25, :113-119): bit b of a
// vector x is (sum_c P[b][c] * x[c]) >= 0, summed in source order c = 0..d-1
// in IEEE double without FMA. The decode step hashes a handful of vectors per
// (layer, KV head) — the missed heads' approximate queries (lookup.cu) and
// every head's new key row (encode.cu) — so these kernels are latency-bound.
// Reading P^T from global memory costs one dependent round trip per batch of
// loads, and those round trips stretch several-fold while the zero-copy
// gather keeps the memory system full of PCIe reads (profiles/README.md,
// round 2). Here one CTA owns one 64-bit code word: a single bulk copy (TMA
// engine) brings the word's [d][64] slice of P^T (64 KiB at d = 128) into
// shared memory, and every chain then runs out of shared memory.
#pragma once

#include "common.cuh"

namespace clo {
namespace bulk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// One thread: arm `bar` for `bytes` and bulk-copy global -> shared (16-byte
// aligned, size a multiple of 16).
__device__ __forceinline__ void load_async(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

}  // namespace bulk

// Sequential chain of one bit against a staged slice ps [d][64].
template <int D>
__device__ __forceinline__ double slice_chain(const double* __restrict__ ps, int bit, const double* __restrict__ x) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) s = dmac(s, ps[c * 64 + bit], x[c]);
    return s;
}
__device__ __forceinline__ double slice_chain_any(const double* __restrict__ ps, int bit, const double* __restrict__ x,
                                                  int d) {
    if (d == 128) return slice_chain<128>(ps, bit, x);
    if (d == 64) return slice_chain<64>(ps, bit, x);
    double s = 0.0;
    for (int c = 0; c < d; ++c) s = dmac(s, ps[c * 64 + bit], x[c]);
    return s;
}

// Word w of the sign codes of M vectors xs [M][xstride] (shared memory) from
// the staged slice ps of that word. Whole CTA (blockDim.x a multiple of 32);
// M*64 chains are dealt to the threads, each warp covers 32 bits of one
// vector, so one ballot makes one 32-bit half-word. out(j) = vector j's code
// (words u64) as u32 pointer; bits >= `bits` are zero.
template <typename Out>
__device__ __forceinline__ void hash_word(const double* ps, const double* xs, int xstride, int M, int d, int w,
                                          int bits, Out out) {
    for (int ch = threadIdx.x; ch < M * 64; ch += blockDim.x) {
        const int j = ch >> 6, bit = ch & 63;
        const double s = slice_chain_any(ps, bit, xs + (size_t)j * xstride, d);
        const unsigned bal = __ballot_sync(0xffffffffu, w * 64 + bit < bits && s >= 0.0);
        if ((threadIdx.x & 31) == 0) out(j)[w * 2 + (bit >> 5)] = bal;
    }
}

}  // namespace clo
