// exchange.cuh — head-output all-gather of KV-head sharding (SURVEY.md §8e,
// north star item 5), fused into the attention epilogue.
//
// With the KV heads of a model split over `world` ranks (one GPU each,
// EngineConfig.kv_head_offset = rank * H_local), every rank computes the
// outputs of its own m*H_local query heads. The reference has no such
// exchange: its per-head loops (engine.cpp:377-409) write every head's output
// into one [h_q][d] row of collected_outputs (engine.cpp:403-405). Here the
// attention epilogue that produces a head's output stores it
//   * into the caller's out [B][L][hq_global][d] at this rank's head block, and
//   * straight into every peer's exchange slot (P2P stores over NVLink, or
//     plain stores when the peer engine shares the device),
// then raises each peer's per-layer arrival counter with a system-scope
// release. A finishing kernel at the end of the step graph acquires the
// counters and copies the peers' head blocks from the local slot into out.
// No host synchronisation and no separate collective launch: the transfer of
// layer l overlaps the attention of layers l+1...
//
// Slots are double-buffered by step parity. A rank can run at most one step
// ahead of a peer (its own finish waits for that peer's arrivals), so a peer
// never overwrites a slot its owner is still copying out.
#pragma once

#include "common.cuh"
#include "engine_view.h"

namespace clo {

// Bytes of the exchange buffer header (arrival counters [L] u32, padded).
__host__ __device__ inline size_t exchange_flag_bytes(int L) { return ((size_t)L * 4 + 255) / 256 * 256; }

// Offset (floats) of row (b, l, q_global) of slot `parity` in a peer buffer.
__device__ __forceinline__ size_t exchange_row(const EngineView& v, int parity, int b, int l, int q) {
    return (((size_t)parity * v.B + b) * v.L + l) * v.HQg + q;
}

// Epilogue store of output element e of local query head hq (= g*m + j).
__device__ __forceinline__ void emit_head_output(const EngineView& v, int t, int b, int l, int hq, int e,
                                                 float val) {
    const int q = v.q0 + hq;
    float* out = v.desc->out;
    if (out) out[(((size_t)b * v.L + l) * v.HQg + q) * v.d + e] = val;
    if (v.world > 1) {
        const size_t row = exchange_row(v, t & 1, b, l, q);
#pragma unroll 1
        for (int r = 0; r < v.world; ++r)
            if (r != v.rank) v.xslot[r][row * v.d + e] = val;
    }
}

// After every thread of the CTA stored its outputs of (b, l, g): publish them
// to the peers (one system-scope release increment per peer).
__device__ __forceinline__ void signal_head_output(const EngineView& v, int l) {
    if (v.world <= 1) return;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 1
        for (int r = 0; r < v.world; ++r)
            if (r != v.rank)
                asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(v.xflag[r] + l), "r"(1u) : "memory");
    }
}

// Same, when one warp stored all of the head's outputs.
__device__ __forceinline__ void signal_head_output_warp(const EngineView& v, int l) {
    if (v.world <= 1) return;
    __threadfence_system();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
#pragma unroll 1
        for (int r = 0; r < v.world; ++r)
            if (r != v.rank)
                asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(v.xflag[r] + l), "r"(1u) : "memory");
    }
}

// Step-end: wait for every peer's arrivals of this step, then copy their head
// blocks into out (one launch, on the compute stream before step_end).
void launch_exchange_finish(const EngineView& v, cudaStream_t stream);

}  // namespace clo
