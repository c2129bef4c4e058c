// attention.cuh — K4 `sparse_attn`: softmax attention of the m GQA query
// heads of one KV head over union(selection, sink/recent window)
// (topk_attention / attend_rows attention.cpp:33-55,91-105, union_indices
// engine.cpp:80-85, sink_recent_indices attention.cpp:107-128).
#pragma once

#include "common.cuh"
#include "engine_view.h"

namespace clo {

constexpr int kAttnThreads = 128;
constexpr int kAttnRows = 256;  // attend positions per CTA (split-K)

// Engine: one layer, grid (ceil((k + W)/kAttnRows), B*H). Reads the entry's
// HBM cache slots + the window ring (offloaded) or the full HBM KV
// (persistent); each KV row is read once for all m query heads. The last CTA
// of each head combines the split partials (no second launch).
void launch_attention_engine(const EngineView& v, int layer, cudaStream_t stream);
int attention_chunks(int k, int sink, int recent);
// TMA-staged production kernel (attention_tma.cu); false = unsupported shape
// (the caller falls back to launch_attention_engine's register kernel).
bool attention_tma_supported(int dtype, int d, int m, int k);
bool launch_attention_tma(const EngineView& v, int layer, cudaStream_t stream);
bool attention_supported(int dtype, int d, int m);
// Tensor-core production kernel (attention_mma.cu): bf16 rows, d 64/128,
// m <= 8; false = unsupported (or CLO_ATTN=tma|ffma), try the TMA kernel.
bool attention_mma_supported(int dtype, int d, int m, int k);
bool launch_attention_mma(const EngineView& v, int layer, cudaStream_t stream);
// floats of attn_part the tensor-core kernel's per-warp partials need
size_t attention_mma_partial_floats(int B, int H, int m, int d, int k, int sink, int recent);

// Op-level topk_attention for m queries over one matrix (validation separate).
void launch_attention_op(const double* q, int m, const void* keys, const void* values, int dtype,
                         int d, const int32_t* idx, int nidx, double* out, double* scratch,
                         cudaStream_t stream);
// Index validation: range and duplicates (bitmap [ceil(n/32)] u32, zeroed).
void launch_validate_indices(const int32_t* idx, int nidx, int64_t n, uint32_t* bitmap, int* err,
                             cudaStream_t stream);

}  // namespace clo
