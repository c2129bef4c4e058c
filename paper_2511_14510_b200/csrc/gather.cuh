// gather.cuh — K3 zero-copy gather launchers.
#pragma once

#include "common.cuh"
#include "engine_view.h"
#include "select.cuh"

namespace clo {

struct GatherEngineArgs {
    EngineView v;
    const SelItem* items;  // the prefetch stream's work list (missed offloaded heads)
    const int* count;      // [L]
    int layer;
    int count_bytes;
};

// Row size must be a multiple of 16 bytes (d*sizeof(dtype) % 16 == 0).
void launch_gather_engine(const GatherEngineArgs& a, int grid, cudaStream_t stream);
void launch_gather_op(const void* src, void* dst, const int32_t* idx, int row_bytes, int k,
                      int64_t n_rows, int* err, cudaStream_t stream);

}  // namespace clo
