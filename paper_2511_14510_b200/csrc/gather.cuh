// gather.cuh — K3 zero-copy gather + entry reconcile launchers.
#pragma once

#include "common.cuh"
#include "engine_view.h"
#include "select.cuh"

namespace clo {

struct ReconcileArgs {
    EngineView v;
    const SelItem* items;  // this layer's work list (missed offloaded heads)
    const int* count;      // [L]
    const int32_t* sel;    // [item][k] new ascending selections
    int32_t* fetch_tok;    // [L][items_cap][k] source: host token (>= 0) or -(victim slot + 1)
    int32_t* fetch_slot;   // destination entry slot
    int32_t* fetch_dem;    // victim slot the slot's leaving row moves to first, or -1
    int* fetch_count;      // [L][items_cap]
    int items_cap;         // B*H
    int layer;
    int fresh;             // prefill: no previous entry
};

struct GatherEngineArgs {
    EngineView v;
    const SelItem* items;
    const int* count;      // [L]
    const int32_t* fetch_tok;
    const int32_t* fetch_slot;
    const int32_t* fetch_dem;
    const int* fetch_count;
    int items_cap;
    int layer;
    int count_bytes;
};  // items: base of the per-layer work lists [L][items_cap] (gather_unit offsets by layer)

void launch_reconcile(const ReconcileArgs& a, cudaStream_t stream);
// Row size must be a multiple of 16 bytes (d*sizeof(dtype) % 16 == 0).
void launch_gather_engine(const GatherEngineArgs& a, int grid, cudaStream_t stream);
// GPU-centric transfer pipeline (one decode step): publish(l) after
// reconcile(l) on the selection stream; one persistent gather kernel per step
// on the transfer stream over `layers` (device array); wait_flag(l) on the
// compute stream before attention(l).
void launch_publish(const GatherEngineArgs& a, cudaStream_t stream);
void launch_gather_persistent(const GatherEngineArgs& a, const int* layers, int n_layers, int grid,
                              cudaStream_t stream);
void launch_wait_flag(const int* flag, const int* dev_step, cudaStream_t stream);
// ctas <= 0: default grid
void launch_gather_op(const void* src, void* dst, const int32_t* idx, int row_bytes, int k,
                      int64_t n_rows, int* err, int ctas, cudaStream_t stream);
void launch_gather_tma_op(const void* src, void* dst, const int32_t* idx, int row_bytes, int k,
                          int64_t n_rows, int* err, int ctas, cudaStream_t stream);
int reconcile_max_k();

}  // namespace clo
