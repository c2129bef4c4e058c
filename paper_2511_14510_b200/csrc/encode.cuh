// encode.cuh — sign-hash metadata on the GPU (K6 encode at prefill, K5 append).
#pragma once

#include "common.cuh"
#include "engine_view.h"

namespace clo {

// encode() sign bits (retrieval.cpp:60-78 / append_sign_row :14-25) of rows
// [0, n) of one key matrix: codes[r] bit b = (sum_c P[b][c]*K[r][c]) >= 0 in
// sequential IEEE double. rows may be UVA host memory. proj_t = P^T [d][bits].
// `segments` independent matrices: rows_base + s*rows_stride (elements),
// proj_t + s*proj_stride, codes + s*codes_stride; ptr arrays allow a
// per-segment layout.
struct EncodeSeg {
    const void* rows;       // [n][d] of dtype (device or UVA host)
    const double* proj_t;   // [d][bits]
    uint64_t* codes;        // [n][words]
};
void launch_encode(const EncodeSeg* segs_dev, int n_segs, int64_t n, int d, int bits, int dtype,
                   int* err, cudaStream_t stream);

// Phase 2 of decode_step (engine.cpp:360-370) for one layer: append the new
// token's K/V row of every head (host store via zero-copy store, persistent
// HBM store, exact-mode K mirror, sink/recent window ring slot,
// SinkRecentBuffer::advance similarity_cache.cpp:113-128) and its sign bits
// (update_metadata, retrieval.cpp:80-88).
void launch_append(const EngineView& v, int layer, cudaStream_t stream);

// Marks the step complete (device step counter) and clears the per-layer
// work-list counters for the next step.
void launch_step_end(const EngineView& v, int* count_a, int* count_b, cudaStream_t stream);

// Scans n*d values for non-finite entries (check_qkv, attention.cpp:11-23).
void launch_check_finite(const void* p, int dtype, int64_t count, int* err, int bit,
                         cudaStream_t stream);

// Window init at prefill: sink rows [0, min(sink,n)) and ring rows for the
// last min(n, recent) tokens (SinkRecentBuffer::reset_from, :103-111).
void launch_window_init(const EngineView& v, cudaStream_t stream);

}  // namespace clo
