// gather.cu — K3 `zero_copy_gather` and the entry reconcile (delta gather).
//
// update_entry (similarity_cache.cpp:74-87) replaces a missed head's whole
// entry with the rows of its new selection, copied from the host store
// (gather_rows engine.cpp:98-102); the reference only models that transfer
// as bytes / pcie_peak_bw (pipeline_sim.cpp:12-22). Here:
//   reconcile  (one CTA per missed head) merge-joins the old entry with the
//              new ascending selection: tokens present in both keep their
//              HBM slot; tokens that left free their slot; each new token
//              gets a freed slot and goes on the fetch list. The entry's
//              CONTENTS are exactly the reference's (same indices, same
//              rows); only the data movement shrinks to the rows that are
//              actually missing in HBM.
//   gather     GPU threads read exactly the fetch-list rows straight from
//              pinned, UVA-mapped host memory over PCIe (16-byte loads, 32 KiB
//              in flight per CTA) and store them into their slots.
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "gather.cuh"
#include "reconcile.cuh"

#ifndef CLO_REC_THREADS
#define CLO_REC_THREADS 1024
#endif

namespace clo {

namespace {

constexpr int kGatherThreads = 256;
constexpr int kUnroll = 4;
constexpr int kVecsPerUnit = kGatherThreads * kUnroll;  // 16-byte vectors per work unit
constexpr int kUnitUnroll = 8;                          // engine gather: loads in flight per thread
constexpr int kUnitVecs = kGatherThreads * kUnitUnroll;  // 32 KiB of one matrix per unit
constexpr int kRecThreads = CLO_REC_THREADS;


// One CTA per missed head (reconcile.cuh).
__global__ void __launch_bounds__(kRecThreads) reconcile_kernel(ReconcileArgs a) {
    __shared__ ReconcileSmem<kRecThreads> sm;
    extern __shared__ int32_t rs[];
    const int count = a.count[a.layer];
    for (int item = blockIdx.x; item < count; item += gridDim.x) reconcile_item<kRecThreads>(a, item, rs, sm);
}

// Work units = (missed head, matrix, block of move-list vectors). K and V are
// separate units (all of a head's K rows, then its V rows) so a CTA's
// outstanding reads stay within one host matrix region at a time.
// Interleaved host K|V (v.kv_fused): one unit covers whole 2*d-element token
// runs, split into the K and V slots on the way out.
// Per vector: load the source (host row over PCIe, or the victim slot of a
// promotion) and, when the move demotes, the slot's current vector; store the
// old vector to its victim slot and the new one into the entry slot.
__device__ __forceinline__ int gather_units_per_item(const EngineView& v) {
    const int vpr = v.d * dtype_size(v.kv_dtype) / 16;
    if (v.kv_fused) return (v.k * 2 * vpr + kUnitVecs - 1) / kUnitVecs;
    return 2 * ((v.k * vpr + kUnitVecs - 1) / kUnitVecs);
}

// One work unit of layer `layer` (all threads of the CTA).
__device__ __forceinline__ void gather_unit(const GatherEngineArgs& a, int layer, int u) {
    const EngineView& v = a.v;
    const int row_bytes = v.d * dtype_size(v.kv_dtype);
    const int vpr = row_bytes / 16;
    const int rvpr = (int)(v.row_stride * (int64_t)dtype_size(v.kv_dtype) / 16);  // host row pitch
    const bool fused = v.kv_fused;
    const int vpt = fused ? 2 * vpr : vpr;  // vectors per moved row (per matrix when split)
    const int upm = (v.k * vpt + kUnitVecs - 1) / kUnitVecs;
    const int upi = fused ? upm : 2 * upm;
    const int item = u / upi, rem = u % upi;
    const int mat = fused ? 0 : rem / upm, part = fused ? rem : rem % upm;  // mat 0 = K, 1 = V
    const size_t li = (size_t)layer * a.items_cap + item;
    const int v0 = part * kUnitVecs;
    const int v1 = min(a.fetch_count[li] * vpt, v0 + kUnitVecs);
    if (v0 >= v1) return;
    const int seg = a.items[li].seg;
    const int g = seg % v.H, l = (seg / v.H) % v.L, b = seg / (v.H * v.L);
    const size_t o = (size_t)b * v.NO + v.oidx[l * v.H + g];
    const size_t base = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
    const size_t esz = dtype_size(v.kv_dtype);
    const uint4* hsrc = reinterpret_cast<const uint4*>((const char*)(mat ? v.host_v : v.host_k) + base * esz);
    uint4* pk = reinterpret_cast<uint4*>((char*)v.slot_k + o * v.pool * row_bytes);
    uint4* pv = reinterpret_cast<uint4*>((char*)v.slot_v + o * v.pool * row_bytes);
    const int32_t* ftok = a.fetch_tok + li * v.k;
    const int32_t* fslot = a.fetch_slot + li * v.k;
    const int32_t* fdem = a.fetch_dem + li * v.k;
    uint4 r[kUnitUnroll], old[kUnitUnroll];
    uint4* dp[kUnitUnroll];
    uint4* vp[kUnitUnroll];
    int host = 0;
#pragma unroll
    for (int uu = 0; uu < kUnitUnroll; ++uu) {
        const int e = v0 + uu * kGatherThreads + threadIdx.x;
        vp[uu] = nullptr;
        if (e < v1) {
            const int row = e / vpt, c = e - row * vpt;
            // vector c of the moved row: K part (c < vpr) or V part (fused), or matrix `mat`
            const bool isv = fused ? c >= vpr : mat == 1;
            const int cc = fused && isv ? c - vpr : c;
            uint4* pool = isv ? pv : pk;
            const int slot = fslot[row], src = ftok[row], dem = fdem[row];
            dp[uu] = pool + (size_t)slot * vpr + cc;
            if (dem >= 0) {  // the slot's leaving row moves to the victim area first
                old[uu] = *dp[uu];
                vp[uu] = pool + (size_t)dem * vpr + cc;
            }
            if (src >= 0) {
                r[uu] = hsrc[(size_t)src * rvpr + c];  // PCIe: host row (K|V run when fused)
                ++host;
            } else {
                r[uu] = pool[(size_t)(-src - 1) * vpr + cc];  // promotion from the victim area
            }
        }
    }
#pragma unroll
    for (int uu = 0; uu < kUnitUnroll; ++uu) {
        const int e = v0 + uu * kGatherThreads + threadIdx.x;
        if (vp[uu]) *vp[uu] = old[uu];
        if (e < v1) *dp[uu] = r[uu];
    }
    if (a.count_bytes) {
        host = __reduce_add_sync(0xffffffffu, host);
        if ((threadIdx.x & 31) == 0 && host) atomicAdd(v.gathered_bytes, (unsigned long long)host * 16ull);
    }
}

// "Wide" LSU gather: few fat CTAs (T threads x U 16-byte loads in flight each)
// over a flat list of the layer's moved rows. With a shared-memory
// reservation that no other kernel's CTA fits beside, the gather owns a few
// SMs and the host reads queue only there: kernel boundaries elsewhere wait
// for the SM's own outstanding reads (profiles/r2: 2 us beside a gather on
// 16 SMs, 37 us beside one spread over 128). CLO_GATHER=wide (experiment).
template <int T, int U>
__global__ void __launch_bounds__(T) gather_wide_kernel(GatherEngineArgs a) {
    extern __shared__ int wpref[];  // [count + 1] first flat row of each item (then the reservation)
    const EngineView& v = a.v;
    const int row_bytes = v.d * dtype_size(v.kv_dtype);
    const int vpr = row_bytes / 16;
    const int rvpr = (int)(v.row_stride * (int64_t)dtype_size(v.kv_dtype) / 16);
    const bool fused = v.kv_fused;
    const int vpt = 2 * vpr;  // K then V vectors of a moved row
    const int count = a.count[a.layer];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        int run = 0;
        for (int i0 = 0; i0 < count; i0 += 32) {
            const int i = i0 + lane;
            const int fc = i < count ? a.fetch_count[(size_t)a.layer * a.items_cap + i] : 0;
            int incl = fc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (i < count) wpref[i] = run + incl - fc;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) wpref[count] = run;
    }
    __syncthreads();
    const long long total = (long long)wpref[count] * vpt;
    const size_t esz = dtype_size(v.kv_dtype);
    unsigned long long moved = 0;
    for (long long base = (long long)blockIdx.x * T * U; base < total; base += (long long)gridDim.x * T * U) {
        uint4 r[U], old[U];
        uint4* dp[U];
        uint4* vp[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const long long e = base + (long long)uu * T + threadIdx.x;
            dp[uu] = nullptr;
            vp[uu] = nullptr;
            if (e < total) {
                const int fr = (int)(e / vpt), c = (int)(e - (long long)fr * vpt);
                int lo = 0, hi = count;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (wpref[mid] <= fr)
                        lo = mid;
                    else
                        hi = mid;
                }
                const size_t li = (size_t)a.layer * a.items_cap + lo;
                const int j = fr - wpref[lo];
                const int seg = a.items[li].seg;
                const int g = seg % v.H, l = (seg / v.H) % v.L, b = seg / (v.H * v.L);
                const size_t o = (size_t)b * v.NO + v.oidx[l * v.H + g];
                const bool isv = c >= vpr;
                const int cc = isv ? c - vpr : c;
                uint4* pool = reinterpret_cast<uint4*>((char*)(isv ? v.slot_v : v.slot_k) + o * v.pool * row_bytes);
                const int slot = a.fetch_slot[li * v.k + j], src = a.fetch_tok[li * v.k + j];
                const int dem = a.fetch_dem[li * v.k + j];
                dp[uu] = pool + (size_t)slot * vpr + cc;
                if (dem >= 0) {
                    old[uu] = *dp[uu];
                    vp[uu] = pool + (size_t)dem * vpr + cc;
                }
                if (src >= 0) {
                    const size_t hb = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
                    const uint4* hs = reinterpret_cast<const uint4*>(
                        (const char*)(fused || !isv ? v.host_k : v.host_v) + hb * esz);
                    r[uu] = hs[(size_t)src * rvpr + (fused ? c : cc)];
                    ++moved;
                } else {
                    r[uu] = pool[(size_t)(-src - 1) * vpr + cc];
                }
            }
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            if (vp[uu]) *vp[uu] = old[uu];
            if (dp[uu]) *dp[uu] = r[uu];
        }
    }
    if (a.count_bytes) {
        moved = __reduce_add_sync(0xffffffffu, (unsigned)moved);
        if (lane == 0 && moved) atomicAdd(v.gathered_bytes, moved * 16ull);
    }
}

// Wide gather with the rows in flight held in SHARED memory (cp.async 16-byte
// copies, LDGSTS) instead of registers: T threads x U vectors per batch, two
// batches in flight per CTA (the next batch's host reads are issued before the
// current batch is stored), so a few CTAs keep megabytes of host reads in
// flight on their own SMs. CLO_GATHER=wide_smem (experiment).
template <int T, int U>
__global__ void __launch_bounds__(T) gather_wide_smem_kernel(GatherEngineArgs a) {
    extern __shared__ __align__(16) unsigned char wsm[];  // [2][U][T] uint4, then [count + 1] row prefix
    uint4* buf = reinterpret_cast<uint4*>(wsm);
    int* wpref = reinterpret_cast<int*>(wsm + 2 * (size_t)U * T * sizeof(uint4));
    const EngineView& v = a.v;
    const int row_bytes = v.d * dtype_size(v.kv_dtype);
    const int vpr = row_bytes / 16;
    const int rvpr = (int)(v.row_stride * (int64_t)dtype_size(v.kv_dtype) / 16);
    const bool fused = v.kv_fused;
    const int vpt = 2 * vpr;
    const int count = a.count[a.layer];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        int run = 0;
        for (int i0 = 0; i0 < count; i0 += 32) {
            const int i = i0 + lane;
            const int fc = i < count ? a.fetch_count[(size_t)a.layer * a.items_cap + i] : 0;
            int incl = fc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (i < count) wpref[i] = run + incl - fc;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) wpref[count] = run;
    }
    __syncthreads();
    const long long total = (long long)wpref[count] * vpt;
    const size_t esz = dtype_size(v.kv_dtype);
    // vector e of the flat list: its pool row base (K or V pool of its head)
    // and slot, plus the source (host row, or victim slot for a promotion)
    struct Vec {
        uint4* pool;
        int slot, dem, cc;
        const uint4* src;
    };
    auto locate = [&](long long e) {
        Vec x;
        const int fr = (int)(e / vpt), c = (int)(e - (long long)fr * vpt);
        int lo = 0, hi = count;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (wpref[mid] <= fr)
                lo = mid;
            else
                hi = mid;
        }
        const size_t li = (size_t)a.layer * a.items_cap + lo;
        const int j = fr - wpref[lo];
        const int seg = a.items[li].seg;
        const int g = seg % v.H, l = (seg / v.H) % v.L, b = seg / (v.H * v.L);
        const size_t o = (size_t)b * v.NO + v.oidx[l * v.H + g];
        const bool isv = c >= vpr;
        x.cc = isv ? c - vpr : c;
        x.pool = reinterpret_cast<uint4*>((char*)(isv ? v.slot_v : v.slot_k) + o * v.pool * row_bytes);
        x.slot = a.fetch_slot[li * v.k + j];
        x.dem = a.fetch_dem[li * v.k + j];
        const int src = a.fetch_tok[li * v.k + j];
        if (src >= 0) {
            const size_t hb = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
            x.src = reinterpret_cast<const uint4*>((const char*)(fused || !isv ? v.host_k : v.host_v) + hb * esz) +
                    (size_t)src * rvpr + (fused ? c : x.cc);
        } else {
            x.src = x.pool + (size_t)(-src - 1) * vpr + x.cc;
        }
        return x;
    };
    const long long step = (long long)gridDim.x * T * U;
    auto issue = [&](long long base, int half) {
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const long long e = base + (long long)uu * T + threadIdx.x;
            if (e < total) {
                const Vec x = locate(e);
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + ((size_t)half * U + uu) * T + threadIdx.x));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(x.src) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    unsigned long long moved = 0;
    long long base = (long long)blockIdx.x * T * U;
    if (base < total) issue(base, 0);
    for (int half = 0; base < total; base += step, half ^= 1) {
        if (base + step < total) {
            issue(base + step, half ^ 1);  // next batch's reads in flight during this batch's stores
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        // each thread stores the vectors it loaded (no barrier needed)
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const long long e = base + (long long)uu * T + threadIdx.x;
            if (e < total) {
                const Vec x = locate(e);
                uint4* dp = x.pool + (size_t)x.slot * vpr + x.cc;
                if (x.dem >= 0) x.pool[(size_t)x.dem * vpr + x.cc] = *dp;  // leaving row -> victim slot first
                *dp = buf[((size_t)half * U + uu) * T + threadIdx.x];
                moved += x.src < x.pool || x.src >= x.pool + (size_t)v.pool * vpr;  // host source
            }
        }
    }
    if (a.count_bytes) {
        moved = __reduce_add_sync(0xffffffffu, (unsigned)moved);
        if (lane == 0 && moved) atomicAdd(v.gathered_bytes, moved * 16ull);
    }
}

// One launch per layer (prefill, and the serialised profiling graph).
__global__ void __launch_bounds__(kGatherThreads) gather_engine_kernel(GatherEngineArgs a) {
    const int units = a.count[a.layer] * gather_units_per_item(a.v);
    for (int u = blockIdx.x; u < units; u += gridDim.x) gather_unit(a, a.layer, u);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Publishes layer l's fetch lists to the persistent transfer kernel (one
// thread, on the selection stream after reconcile): unit count, then the
// ready flag (release); a layer with nothing to fetch is marked done at once.
__global__ void publish_kernel(GatherEngineArgs a) {
    const EngineView& v = a.v;
    const int epoch = *v.dev_step + 1;
    const int units = a.count[a.layer] * gather_units_per_item(v);
    v.xfer_units[a.layer] = units;
    __threadfence();
    if (units == 0) st_release(&v.xfer_flag[a.layer], epoch);
    st_release(&v.xfer_ready[a.layer], epoch);
}

// Persistent transfer kernel: one launch per decode step on the high-priority
// transfer stream. Its CTAs walk the offloaded layers in order; for each they
// wait (device flag, no host involvement) until the layer's fetch lists are
// published, claim work units from a per-layer counter and stream them from
// pinned host memory into the HBM slots. The CTA finishing the layer's last
// unit raises its done flag. Back-to-back layers leave no launch gaps on the
// PCIe link.
__global__ void __launch_bounds__(kGatherThreads) gather_persistent_kernel(GatherEngineArgs a,
                                                                           const int* layers, int n_layers) {
    const EngineView& v = a.v;
    const int epoch = *v.dev_step + 1;
    __shared__ int s_u, s_units;
    for (int li = 0; li < n_layers; ++li) {
        const int l = layers[li];
        if (threadIdx.x == 0) {
            while (ld_acquire(&v.xfer_ready[l]) != epoch) __nanosleep(128);
            s_units = *((volatile int*)&v.xfer_units[l]);
        }
        __syncthreads();
        const int units = s_units;
        for (;;) {
            if (threadIdx.x == 0) s_u = atomicAdd(&v.xfer_claim[l], 1);
            __syncthreads();
            const int u = s_u;
            __syncthreads();
            if (u >= units) break;
            gather_unit(a, l, u);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(&v.xfer_done[l], 1) + 1 == units) st_release(&v.xfer_flag[l], epoch);
            }
        }
    }
}

// Compute-stream gate before attention(l): one thread waits for the layer's
// done flag, so the stream proceeds without any host synchronisation.
__global__ void wait_flag_kernel(const int* flag, const int* dev_step) {
    const int epoch = *dev_step + 1;
    while (ld_acquire(flag) != epoch) __nanosleep(128);
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

// ---------------------------------------------------------- TMA bulk gather
// Same copy, driven by the TMA unit instead of LSU loads: one 1D bulk copy
// (cp.async.bulk global->shared) per row straight out of pinned host memory
// into a shared-memory stage, completion on an mbarrier, then one bulk store
// of the 32-row stage to its contiguous destination. One warp per CTA keeps
// kTmaStages x 32 rows in flight without holding registers.
constexpr int kTmaStages = 4;
constexpr int kTmaRows = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32) gather_tma_kernel(const char* __restrict__ src, char* __restrict__ dst,
                                                        const int32_t* __restrict__ idx, int row_bytes, int k,
                                                        int64_t n_rows, int* err) {
    extern __shared__ __align__(128) char stage[];  // [kTmaStages][kTmaRows][row_bytes]
    __shared__ __align__(8) uint64_t bar[kTmaStages];
    const int lane = threadIdx.x;
    const int groups = (k + kTmaRows - 1) / kTmaRows;
    if (lane == 0) {
        for (int s = 0; s < kTmaStages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // this CTA's groups: blockIdx.x, blockIdx.x + gridDim.x, ...
    const int mine = groups > (int)blockIdx.x ? (groups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto load = [&](int i) {  // i-th group of this CTA into stage i % S
        const int g = blockIdx.x + i * gridDim.x;
        const int s = i % kTmaStages;
        const int rows = min(kTmaRows, k - g * kTmaRows);
        char* st = stage + (size_t)s * kTmaRows * row_bytes;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                         "r"(rows * row_bytes)
                         : "memory");
        }
        __syncwarp();
        if (lane < rows) {
            int32_t ix = idx[g * kTmaRows + lane];
            if (ix < 0 || ix >= n_rows) {
                atomicOr(err, kErrIndexRange);
                ix = 0;
            }
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(st + (size_t)lane * row_bytes)),
                "l"(src + (size_t)ix * row_bytes), "r"(row_bytes), "r"(smem_u32(&bar[s]))
                : "memory");
        }
    };
    for (int i = 0; i < min(kTmaStages, mine); ++i) load(i);
    for (int i = 0; i < mine; ++i) {
        const int g = blockIdx.x + i * gridDim.x;
        const int s = i % kTmaStages;
        const int rows = min(kTmaRows, k - g * kTmaRows);
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar[s])),
            "r"((i / kTmaStages) & 1)
            : "memory");
        if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                             dst + (size_t)g * kTmaRows * row_bytes),
                         "r"(smem_u32(stage + (size_t)s * kTmaRows * row_bytes)), "r"(rows * row_bytes)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // stage reusable
        }
        __syncwarp();
        if (i + kTmaStages < mine) load(i + kTmaStages);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Engine gather on the TMA engine (CLO_GATHER=tma): each warp streams groups
// of 32 fetch-list rows — lane r bulk-copies row r (one cp.async.bulk of a
// whole row) from pinned host memory into a shared-memory stage, completion on
// an mbarrier, then bulk-stores it to its HBM slot. kTmaStages groups per warp
// in flight. Groups are (missed head, matrix, 32-row block) of the layer.
constexpr int kTmaWarps = 4;  // max warps per CTA
constexpr int kTmaMaxStages = 8;

__global__ void __launch_bounds__(kTmaWarps * 32) gather_engine_tma_kernel(GatherEngineArgs a, int stages) {
    extern __shared__ __align__(128) char tstage[];  // [warp][stages][32][row_bytes]
    __shared__ __align__(8) uint64_t tbar[kTmaWarps][kTmaMaxStages];
    const EngineView& v = a.v;
    const int row_bytes = v.d * dtype_size(v.kv_dtype);
    const int vpr = row_bytes / 16;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool fused = v.kv_fused;                    // one [K|V] token run per lane and group
    const int nmat = fused ? 1 : 2;
    const int cbytes = fused ? 2 * row_bytes : row_bytes;  // bytes copied per row
    const int wpc = blockDim.x >> 5;
    const int gw = blockIdx.x * wpc + warp, nw = gridDim.x * wpc;
    char* st0 = tstage + (size_t)warp * stages * kTmaRows * cbytes;
    // The layer's NON-EMPTY 32-row groups as one flat list (a move list holds
    // fetch_count <= k rows): gpref[i] = first flat group of item i. Warps take
    // flat groups gw, gw + nw, ... so every warp gets the same number of real
    // groups (+-1) and none walks empty ones.
    int* gpref = reinterpret_cast<int*>(tstage + (size_t)wpc * stages * kTmaRows * cbytes *
                                                     (v.pool > v.k ? 2 : 1));
    const int count = a.count[a.layer];
    if (warp == 0) {
        int run = 0;
        for (int i0 = 0; i0 < count; i0 += 32) {
            const int i = i0 + lane;
            const int fc = i < count ? a.fetch_count[(size_t)a.layer * a.items_cap + i] : 0;
            const int gi = nmat * ((fc + kTmaRows - 1) / kTmaRows);
            int incl = gi;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (i < count) gpref[i] = run + incl - gi;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) gpref[count] = run;
        for (int s = 0; s < stages && lane == 0; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tbar[warp][s])));
    } else if (lane == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tbar[warp][s])));
    }
    if (lane == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int total = gpref[count];
    const int mine = total > gw ? (total - 1 - gw) / nw + 1 : 0;
    // Row of group i handled by this lane: destination entry slot in its
    // matrix (K, or K then V for fused runs), source = the host row (`host`
    // set) or the victim slot `prom` of a promotion; `dem` = the victim slot
    // the slot's leaving row moves to first (or -1).
    struct Row {
        int rows, mat, slot, prom, dem;
        size_t o;
        const char* host;
    };
    auto locate = [&](int i) {
        Row r{};
        const int gidx = gw + i * nw;
        int lo = 0, hi = count;  // the item whose flat range holds gidx: gpref[item] <= gidx < gpref[item + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (gpref[mid] <= gidx)
                lo = mid;
            else
                hi = mid;
        }
        const int item = lo;
        const size_t li = (size_t)a.layer * a.items_cap + item;
        const int nf = a.fetch_count[li];
        const int gi = (nf + kTmaRows - 1) / kTmaRows;  // groups per matrix of this item
        const int rem = gidx - gpref[item], grp = rem % gi;
        r.mat = rem / gi;
        r.rows = max(0, min(kTmaRows, nf - grp * kTmaRows));
        r.prom = -1;
        r.dem = -1;
        if (lane < r.rows) {
            const int seg = a.items[li].seg;
            const int g = seg % v.H, l = (seg / v.H) % v.L, b = seg / (v.H * v.L);
            r.o = (size_t)b * v.NO + v.oidx[l * v.H + g];
            const int j = grp * kTmaRows + lane;
            r.slot = a.fetch_slot[li * v.k + j];
            r.dem = a.fetch_dem[li * v.k + j];
            const int src = a.fetch_tok[li * v.k + j];
            if (src >= 0) {
                const size_t base = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
                r.host = (const char*)(r.mat ? v.host_v : v.host_k) + (base + (size_t)src * v.row_stride) * dtype_size(v.kv_dtype);
            } else {
                r.prom = -src - 1;
            }
        }
        return r;
    };
    auto row_ptr = [&](int m, size_t o, int slot) {  // pool row `slot` of matrix m
        return (char*)(m ? v.slot_v : v.slot_k) + (o * v.pool + slot) * (size_t)row_bytes;
    };
    // Leaving rows demoted by this move (reconcile's fetch_dem): the old row
    // of the entry slot is read into the demotion stage together with the new
    // row and stored to its victim slot before the new row lands.
    char* dst0 = tstage + ((size_t)wpc * stages * kTmaRows * cbytes) + (size_t)warp * stages * kTmaRows * cbytes;
    auto load = [&](int i) {
        const Row r = locate(i);
        const int s = i % stages;
        uint64_t* bar = &tbar[warp][s];
        const int ndem = __popc(__ballot_sync(0xffffffffu, r.dem >= 0));
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (r.rows)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                             "r"((r.rows + ndem) * cbytes)
                             : "memory");
            else
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
        }
        __syncwarp();
        if (r.dem >= 0) {  // the entry slot's current row(s), HBM
            const uint32_t dd = smem_u32(dst0 + ((size_t)s * kTmaRows + lane) * cbytes);
            for (int m = 0; m < (fused ? 2 : 1); ++m) {
                const int mm = fused ? m : r.mat;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        dd + m * row_bytes),
                    "l"(row_ptr(mm, r.o, r.slot)), "r"(row_bytes), "r"(smem_u32(bar))
                    : "memory");
            }
        }
        if (lane < r.rows) {
            const uint32_t dst = smem_u32(st0 + ((size_t)s * kTmaRows + lane) * cbytes);
            if (r.prom < 0) {  // over PCIe from pinned host memory
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                    "l"(r.host), "r"(cbytes), "r"(smem_u32(bar))
                    : "memory");
            } else {  // promotion: the victim slot's row(s) in HBM
                for (int m = 0; m < (fused ? 2 : 1); ++m) {  // fused: K then V row of the slot
                    const int mm = fused ? m : r.mat;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            dst + m * row_bytes),
                        "l"(row_ptr(mm, r.o, r.prom)), "r"(row_bytes), "r"(smem_u32(bar))
                        : "memory");
                }
            }
        }
    };
    for (int i = 0; i < min(stages, mine); ++i) load(i);
    unsigned long long moved = 0;
    for (int i = 0; i < mine; ++i) {
        const int s = i % stages;
        const Row r = locate(i);
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra W_%=;\n\t}" ::"r"(smem_u32(&tbar[warp][s])),
            "r"((i / stages) & 1)
            : "memory");
        if (r.dem >= 0) {  // demotion first: old row(s) -> victim slot
            const uint32_t da = smem_u32(dst0 + ((size_t)s * kTmaRows + lane) * cbytes);
            for (int m = 0; m < (fused ? 2 : 1); ++m)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 row_ptr(fused ? m : r.mat, r.o, r.dem)),
                             "r"(da + m * row_bytes), "r"(row_bytes)
                             : "memory");
        }
        if (lane < r.rows) {
            const uint32_t sa = smem_u32(st0 + ((size_t)s * kTmaRows + lane) * cbytes);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                             row_ptr(fused ? 0 : r.mat, r.o, r.slot)),
                         "r"(sa), "r"(row_bytes)
                         : "memory");
            if (fused)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 row_ptr(1, r.o, r.slot)),
                             "r"(sa + row_bytes), "r"(row_bytes)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // stage reusable
            if (r.prom < 0) moved += (unsigned long long)cbytes;
        }
        __syncwarp();
        if (i + stages < mine) load(i + stages);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) moved += __shfl_xor_sync(0xffffffffu, moved, o2);
    if (a.count_bytes && lane == 0 && moved) atomicAdd(v.gathered_bytes, moved);
}

}  // namespace

void launch_gather_tma_op(const void* src, void* dst, const int32_t* idx, int row_bytes, int k,
                          int64_t n_rows, int* err, int ctas, cudaStream_t stream) {
    const int groups = (k + kTmaRows - 1) / kTmaRows;
    const int grid = groups < ctas ? (groups > 0 ? groups : 1) : ctas;
    const size_t sm = (size_t)kTmaStages * kTmaRows * row_bytes;
    if (sm > 48 * 1024) cudaFuncSetAttribute(gather_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    gather_tma_kernel<<<grid, 32, sm, stream>>>(static_cast<const char*>(src), static_cast<char*>(dst), idx,
                                                 row_bytes, k, n_rows, err);
}

void launch_reconcile(const ReconcileArgs& a, cudaStream_t stream) {
    const size_t sm = sizeof(int32_t) * 4 * (size_t)a.v.k;  // nsel, need_pos, freed, dvict
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(reconcile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int grid = a.items_cap < 1024 ? a.items_cap : 1024;
    reconcile_kernel<<<grid, kRecThreads, sm, stream>>>(a);
}

// Copy variant by host-region size (measured, profiles/README.md): with
// per-head host regions up to 48 MiB (128K rows of 256 B) the TMA bulk copy
// (1 warp, 1 stage of 32 rows = 8 KiB shared memory, 112 CTAs) wins: its
// CTAs hold no registers for data in flight and co-reside with the attention
// and selection CTAs (configs[1]: +3.5%; 64K x 32 sequences: +24%). Over larger
// regions, where each row's host-address translation misses, the LSU copy
// (48 CTAs x 32 KiB of 16-byte loads in flight) keeps more requests
// outstanding and wins (512K: +8%, 1M: +20%).
// CLO_GATHER=lsu|tma forces a variant; CLO_GATHER_TMA_SHAPE="warps,stages".
void launch_gather_engine(const GatherEngineArgs& a, int ctas, cudaStream_t stream) {
    static const int mode = [] {  // 0 auto, 1 lsu, 2 tma, 3 wide
        const char* e = getenv("CLO_GATHER");
        if (!e || !*e) return 0;
        const std::string m(e);
        return m == "lsu" ? 1 : (m == "tma" ? 2 : (m == "wide" ? 3 : (m == "wide_smem" ? 4 : 0)));
    }();
    if (mode == 4) {  // wide, rows in flight in shared memory
        static const int shape = [] {  // CLO_GATHER_WIDE: 1: 512 x 8 (128 KiB/CTA), 2: 512 x 12 (192 KiB), 3: 1024 x 6 (192 KiB)
            const char* e = getenv("CLO_GATHER_WIDE");
            return e ? atoi(e) : 2;
        }();
        const int grid = ctas > 0 ? ctas : 16;
        const size_t pref = ((size_t)a.items_cap + 1) * sizeof(int);
#define CLO_WS(TT, UU)                                                                                        \
    {                                                                                                         \
        const size_t sm = 2 * (size_t)UU * TT * 16 + pref;                                                    \
        cudaFuncSetAttribute(gather_wide_smem_kernel<TT, UU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        gather_wide_smem_kernel<TT, UU><<<grid, TT, sm, stream>>>(a);                                          \
    }
        if (shape == 1) CLO_WS(512, 8) else if (shape == 3) CLO_WS(1024, 6) else CLO_WS(512, 12)
#undef CLO_WS
        return;
    }
    if (mode == 3) {
        static const int reserve = [] {  // CLO_GATHER_RESERVE: KiB of shared memory per wide CTA
            const char* e = getenv("CLO_GATHER_RESERVE");
            return e && atoi(e) >= 0 ? atoi(e) : 160;
        }();
        const size_t sm = std::max<size_t>(((size_t)a.items_cap + 1) * sizeof(int), (size_t)reserve * 1024);
        static const int shape = [] {  // CLO_GATHER_WIDE: threads x loads (1: 512x8, 2: 512x6, 3: 1024x4)
            const char* e = getenv("CLO_GATHER_WIDE");
            return e ? atoi(e) : 2;
        }();
        const int grid = ctas > 0 ? ctas : 16;
        if (shape == 1) {
            cudaFuncSetAttribute(gather_wide_kernel<512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            gather_wide_kernel<512, 8><<<grid, 512, sm, stream>>>(a);
        } else if (shape == 3) {
            cudaFuncSetAttribute(gather_wide_kernel<1024, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            gather_wide_kernel<1024, 4><<<grid, 1024, sm, stream>>>(a);
        } else {
            cudaFuncSetAttribute(gather_wide_kernel<512, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            gather_wide_kernel<512, 6><<<grid, 512, sm, stream>>>(a);
        }
        return;
    }
    static const int2 shape = [] {
        int2 r{1, 1};
        if (const char* e = getenv("CLO_GATHER_TMA_SHAPE")) {
            int w = 0, st = 0;
            if (sscanf(e, "%d,%d", &w, &st) == 2 && w >= 1 && w <= kTmaWarps && st >= 1 && st <= kTmaMaxStages)
                r = int2{w, st};
        }
        return r;
    }();
    const EngineView& v = a.v;
    const int row_bytes = v.d * dtype_size(v.kv_dtype);
    const int vpr = row_bytes / 16;
    const int cbytes = v.kv_fused ? 2 * row_bytes : row_bytes;
    const size_t sm = (size_t)shape.x * shape.y * kTmaRows * cbytes * (v.pool > v.k ? 2 : 1)  // + demotion stage
                      + ((size_t)a.items_cap + 1) * sizeof(int);                                 // + group prefix
    const bool small_region = (int64_t)v.nmax * row_bytes <= (int64_t)48 << 20;  // between the measured 32 / 64 MiB points
    const int use = mode == 0 ? (small_region && sm <= 200 * 1024 ? 2 : 1) : mode;
    if (use == 2 && sm <= 200 * 1024) {
        const int64_t groups = (int64_t)a.items_cap * (v.kv_fused ? 1 : 2) * ((v.k + kTmaRows - 1) / kTmaRows);
        const int64_t warps = ctas > 0 ? (int64_t)ctas * shape.x : 112;  // measured: 112 one-warp CTAs (104-120 beat 96 and 128)
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(warps, groups) / shape.x);
        cudaFuncSetAttribute(gather_engine_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        gather_engine_tma_kernel<<<grid, shape.x * 32, sm, stream>>>(a, shape.y);
        return;
    }
    // PCIe needs well over 100 KB in flight over large host regions (every
    // row's host translation misses). 48 CTAs x 32 KiB: on the final tree
    // (one box, same session) configs[2] 532 / 551 / 567 / 570 tokens/s with
    // 24 / 40 / 48 / 64 CTAs and configs[3] 781 / 789 / 811 with 24 / 40 / 48;
    // an earlier tree had favoured 24 at configs[3] (872 / 969 vs 864 / 900 on
    // two boxes), long contexts vary most between boxes (profiles/r2).
    const int64_t units = v.kv_fused ? (int64_t)a.items_cap * ((v.k * 2 * vpr + kUnitVecs - 1) / kUnitVecs)
                                     : (int64_t)a.items_cap * 2 * ((v.k * vpr + kUnitVecs - 1) / kUnitVecs);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctas > 0 ? ctas : 48, units));
    gather_engine_kernel<<<grid, kGatherThreads, 0, stream>>>(a);
}

void launch_publish(const GatherEngineArgs& a, cudaStream_t stream) { publish_kernel<<<1, 1, 0, stream>>>(a); }

void launch_gather_persistent(const GatherEngineArgs& a, const int* layers, int n_layers, int grid,
                              cudaStream_t stream) {
    gather_persistent_kernel<<<grid, kGatherThreads, 0, stream>>>(a, layers, n_layers);
}

void launch_wait_flag(const int* flag, const int* dev_step, cudaStream_t stream) {
    wait_flag_kernel<<<1, 1, 0, stream>>>(flag, dev_step);
}

void launch_gather_op(const void* src, void* dst, const int32_t* idx, int row_bytes, int k,
                      int64_t n_rows, int* err, int ctas, cudaStream_t stream) {
    const int vpr = row_bytes / 16;
    const int units = (k * vpr + kVecsPerUnit - 1) / kVecsPerUnit;
    const int cap = ctas > 0 ? ctas : kNumSMs * 8;
    const int grid = units < cap ? (units > 0 ? units : 1) : cap;
    gather_op_kernel<<<grid, kGatherThreads, 0, stream>>>(static_cast<const uint4*>(src),
                                                          static_cast<uint4*>(dst), idx, vpr, k,
                                                          n_rows, err);
}

int reconcile_max_k() { return 8192; }

}  // namespace clo
