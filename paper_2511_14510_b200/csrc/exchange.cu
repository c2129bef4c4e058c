// exchange.cu — step-end half of the fused head-output all-gather
// (exchange.cuh).
#include "exchange.cuh"

#include <algorithm>

namespace clo {

namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Waits until every layer's counter holds this step's arrivals from all peers
// (B * H_local * (world - 1) per step; counters are monotonic, compared
// wrap-safe). One warp: a spinning kernel must not hold SM slots that a peer
// sharing the device (tests, MPS) needs for its own attention.
__global__ void exchange_wait_kernel(EngineView v) {
    if (threadIdx.x != 0) return;
    const int t = *v.dev_step + 1;
    const unsigned target = (unsigned)t * (unsigned)(v.B * v.H * (v.world - 1));
    const unsigned* flags = v.xflag[v.rank];
    const uint64_t t0 = global_ns();
    for (int l = 0; l < v.L; ++l) {
        while ((int)(ld_acquire_sys(flags + l) - target) < 0) {
            if (global_ns() - t0 > v.xtimeout_ns) {
                raise_err(v.err, kErrExchange);
                return;
            }
            __nanosleep(100);
        }
    }
}

// Then the peers' head blocks (rows (b, l, q), q outside [q0, q0 + HQ)) of
// this step's slot -> out. Ordered after the wait by the stream; a timed-out
// wait leaves out's peer blocks as they were (the error flag reports it).
__global__ void __launch_bounds__(256) exchange_copy_kernel(EngineView v) {
    const int t = *v.dev_step + 1;
    const float* slot = v.xslot[v.rank];
    float* out = v.desc->out;
    const int vec = v.d / 4;  // d is a multiple of 8
    const int remote = v.HQg - v.HQ;
    const size_t total = (size_t)v.B * v.L * remote * vec;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % vec);
        size_t r = i / vec;
        int q = (int)(r % remote);
        r /= remote;
        const int l = (int)(r % v.L), b = (int)(r / v.L);
        if (q >= v.q0) q += v.HQ;
        const float4 x = __ldcv(reinterpret_cast<const float4*>(slot + exchange_row(v, t & 1, b, l, q) * v.d) + c);
        reinterpret_cast<float4*>(out + (((size_t)b * v.L + l) * v.HQg + q) * v.d)[c] = x;
    }
}

}  // namespace

void launch_exchange_finish(const EngineView& v, cudaStream_t stream) {
    const size_t vecs = (size_t)v.B * v.L * (v.HQg - v.HQ) * (v.d / 4);
    const int grid = (int)std::min<size_t>((vecs + 255) / 256, (size_t)kNumSMs);
    exchange_wait_kernel<<<1, 32, 0, stream>>>(v);
    exchange_copy_kernel<<<grid < 1 ? 1 : grid, 256, 0, stream>>>(v);
}

}  // namespace clo
