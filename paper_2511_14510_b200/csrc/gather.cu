// gather.cu — K3 `zero_copy_gather`: GPU threads read exactly the missed
// top-k K/V rows straight from pinned, UVA-mapped host memory over PCIe and
// write them into the HBM cache slots (update_entry's row copy,
// similarity_cache.cpp:74-87, gather_rows engine.cpp:98-102; the transfer the
// reference only models as bytes / pcie_peak_bw, pipeline_sim.cpp:12-22).
//
// Each thread keeps kUnroll K and kUnroll V 16-byte loads in flight before
// storing, so one CTA has 256 * 2 * kUnroll * 16 B = 32 KiB outstanding —
// enough CTAs resident across the 148 SMs to cover PCIe round-trip latency.
#include "gather.cuh"

namespace clo {

namespace {

constexpr int kGatherThreads = 256;
constexpr int kUnroll = 4;
constexpr int kVecsPerUnit = kGatherThreads * kUnroll;  // 16-byte vectors per work unit

__device__ __forceinline__ void copy_rows(const uint4* __restrict__ src_k, const uint4* __restrict__ src_v,
                                          uint4* __restrict__ dst_k, uint4* __restrict__ dst_v,
                                          const int32_t* __restrict__ idx, int vpr, int v0, int v1) {
    uint4 rk[kUnroll], rv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
        const int e = v0 + u * kGatherThreads + threadIdx.x;
        if (e < v1) {
            const int r = e / vpr, c = e - r * vpr;
            const size_t off = (size_t)idx[r] * vpr + c;
            rk[u] = src_k[off];
            rv[u] = src_v[off];
        }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
        const int e = v0 + u * kGatherThreads + threadIdx.x;
        if (e < v1) {
            dst_k[e] = rk[u];
            dst_v[e] = rv[u];
        }
    }
}

// Engine mode: work units = (missed offloaded head, block of rows).
__global__ void __launch_bounds__(kGatherThreads) gather_engine_kernel(GatherEngineArgs a) {
    const EngineView& v = a.v;
    const int row_bytes = v.d * dtype_size(v.kv_dtype);
    const int vpr = row_bytes / 16;
    const int total_vecs = v.k * vpr;
    const int units_per_item = (total_vecs + kVecsPerUnit - 1) / kVecsPerUnit;
    const int count = a.count[a.layer];
    const int units = count * units_per_item;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / units_per_item, part = u % units_per_item;
        const int seg = a.items[item].seg;
        const int g = seg % v.H, l = (seg / v.H) % v.L, b = seg / (v.H * v.L);
        const int o = b * v.NO + v.oidx[l * v.H + g];
        const size_t base = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
        const size_t esz = dtype_size(v.kv_dtype);
        const uint4* src_k = reinterpret_cast<const uint4*>((const char*)v.host_k + base * esz);
        const uint4* src_v = reinterpret_cast<const uint4*>((const char*)v.host_v + base * esz);
        uint4* dst_k = reinterpret_cast<uint4*>((char*)v.slot_k + (size_t)o * v.k * row_bytes);
        uint4* dst_v = reinterpret_cast<uint4*>((char*)v.slot_v + (size_t)o * v.k * row_bytes);
        const int v0 = part * kVecsPerUnit, v1 = min(total_vecs, v0 + kVecsPerUnit);
        copy_rows(src_k, src_v, dst_k, dst_v, v.entry_idx + (size_t)seg * v.k, vpr, v0, v1);
        if (a.count_bytes && threadIdx.x == 0)
            atomicAdd(v.gathered_bytes, (unsigned long long)(v1 - v0) * 16ull * 2ull);
    }
}

__global__ void __launch_bounds__(kGatherThreads) gather_op_kernel(const uint4* src, uint4* dst,
                                                                   const int32_t* idx, int vpr,
                                                                   int k, int64_t n_rows, int* err) {
    const int total = k * vpr;
    for (int v0 = blockIdx.x * kVecsPerUnit; v0 < total; v0 += gridDim.x * kVecsPerUnit) {
        uint4 r[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int e = v0 + u * kGatherThreads + threadIdx.x;
            if (e < total) {
                const int row = e / vpr, c = e - row * vpr;
                const int32_t ix = idx[row];
                if (ix < 0 || ix >= n_rows) {
                    atomicOr(err, kErrIndexRange);
                    r[u] = make_uint4(0, 0, 0, 0);
                } else {
                    r[u] = src[(size_t)ix * vpr + c];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int e = v0 + u * kGatherThreads + threadIdx.x;
            if (e < total) dst[e] = r[u];
        }
    }
}

}  // namespace

void launch_gather_engine(const GatherEngineArgs& a, int grid, cudaStream_t stream) {
    gather_engine_kernel<<<grid, kGatherThreads, 0, stream>>>(a);
}

void launch_gather_op(const void* src, void* dst, const int32_t* idx, int row_bytes, int k,
                      int64_t n_rows, int* err, cudaStream_t stream) {
    const int vpr = row_bytes / 16;
    const int units = (k * vpr + kVecsPerUnit - 1) / kVecsPerUnit;
    const int grid = units < kNumSMs * 8 ? (units > 0 ? units : 1) : kNumSMs * 8;
    gather_op_kernel<<<grid, kGatherThreads, 0, stream>>>(static_cast<const uint4*>(src),
                                                          static_cast<uint4*>(dst), idx, vpr, k,
                                                          n_rows, err);
}

}  // namespace clo
