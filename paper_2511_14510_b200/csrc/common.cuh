// common.cuh — shared device-side types and helpers for the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace clo {

constexpr int kNumSMs = 148;
constexpr int kMaxHashWords = 8;   // hash_bits <= 512
constexpr int kMaxGroup = 16;      // m = hq / hkv
constexpr int kMaxHeadDim = 256;
constexpr int kScoreChunk = 4096;  // rows per score/compact work unit
constexpr int kScoreThreads = 256;
constexpr int kMaxRanks = 8;      // KV-head shards of one model (one NVSwitch node)
constexpr int kSlotInEntry = 0x7fffffff;  // slot_age of a pool slot whose token is in the entry
constexpr int kSlotEmpty = -1;            // slot_age of a never-filled pool slot

enum DType : int { kBF16 = 0, kF32 = 1, kF64 = 2 };

__host__ __device__ inline int dtype_size(int dt) { return dt == kBF16 ? 2 : dt == kF32 ? 4 : 8; }

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
    return static_cast<double>(__bfloat162float(v));
}
template <>
__device__ __forceinline__ double to_f64<float>(float v) { return static_cast<double>(v); }
template <>
__device__ __forceinline__ double to_f64<double>(double v) { return v; }

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<double>(double v) { return static_cast<float>(v); }

// Sequential IEEE double accumulation without FMA contraction: the exact
// arithmetic of the reference's scalar SSE2 loops.
__device__ __forceinline__ double dmac(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
}

// Orderable 64-bit key of a finite double: larger key <=> larger value,
// -0.0 canonicalised to +0.0 so it ties with +0.0 like `!=`/`>` do
// (retrieval.cpp:36-39).
__device__ __forceinline__ uint64_t orderable_key(double v) {
    if (v == 0.0) v = 0.0;
    uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double key_to_double(uint64_t k) {
    uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    return __longlong_as_double(static_cast<long long>(u));
}

// Error flag bits written by kernels, read back by the host.
enum ErrBits : int {
    kErrNonFiniteQuery = 1,
    kErrNonFiniteKey = 2,
    kErrNonFiniteValue = 4,
    kErrIndexRange = 8,
    kErrDuplicate = 16,
    kErrContract = 32,
    kErrInternal = 64,
    kErrExchange = 128,  // head-output exchange: a peer stopped arriving
    kErrAlias = 256,     // layer-aliased host store: a step's new K/V rows differ across layers
};

// Phase timestamps for latency diagnosis (build with EXTRA=-DCLO_PROBE; never
// in the shipped library).
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#ifdef CLO_PROBE
#define CLO_PROBE_T(arr, i) \
    if (threadIdx.x == 0) (arr)[i] = globaltimer_ns();
#else
#define CLO_PROBE_T(arr, i)
#endif

__device__ __forceinline__ void raise_err(int* flag, int bits) {
    if (flag) atomicOr(flag, bits);
}

}  // namespace clo
