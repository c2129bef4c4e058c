// boundary_probe.cu — does a saturating zero-copy PCIe read stream slow down
// kernel boundaries on other streams? (round-2 diagnosis of the selection
// chain's in-graph slowdown)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/boundary_probe tools/boundary_probe.cu -lcuda
//   tools/boundary_probe [gather_ctas] [stages]
//
// Stream A: a long train of zero-copy gathers (one warp per CTA; each lane
// bulk-copies 512-byte rows from pinned host memory into shared memory, then
// into HBM — the engine's TMA gather). Stream B: a chain of N tiny kernels,
// or N kernels that each do one dependent global load, timed with events.
// Prints the chain's time per kernel alone and beside the gathers, plus the
// same for an LSU (register-load) gather.
#include <cuda_runtime.h>
#include <stdint.h>

#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));    \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// rows: random 512-byte rows of a host region; `iters` groups of 32 rows per warp
__global__ void tma_gather(const char* host, size_t host_rows, char* dev, int iters, int stages, unsigned seed) {
    extern __shared__ __align__(128) char st[];
    __shared__ __align__(8) uint64_t bar[8];
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned x = seed ^ (blockIdx.x * 9781u + lane * 6271u);
    auto load = [&](int i) {
        const int s = i % stages;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(32 * 512)
                         : "memory");
        __syncwarp();
        x = x * 1664525u + 1013904223u;
        const size_t row = x % host_rows;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                         sa(st + ((size_t)s * 32 + lane) * 512)),
                     "l"(host + row * 512), "r"(sa(&bar[s]))
                     : "memory");
    };
    for (int i = 0; i < stages && i < iters; ++i) load(i);
    for (int i = 0; i < iters; ++i) {
        const int s = i % stages;
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                sa(&bar[s])),
            "r"((i / stages) & 1)
            : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(
                         dev + (((size_t)blockIdx.x * 32 + lane) * 512)),
                     "r"(sa(st + ((size_t)s * 32 + lane) * 512))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        if (i + stages < iters) load(i + stages);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void lsu_gather(const uint4* host, size_t host_rows, uint4* dev, int iters, unsigned seed) {
    unsigned x = seed ^ (blockIdx.x * 9781u + threadIdx.x * 6271u);
    for (int i = 0; i < iters; ++i) {
        uint4 r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            r[u] = host[(x % host_rows) * 32 + (threadIdx.x & 31)];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) dev[((size_t)blockIdx.x * 8 + u) * blockDim.x + threadIdx.x] = r[u];
    }
}

__global__ void empty_kernel(int* p) {
    if (threadIdx.x == 1000000) *p = 1;
}
__global__ void load_kernel(int* p) {  // one dependent HBM round trip per kernel
    if (threadIdx.x == 0) p[1] = p[0] + 1;
}
// programmatic dependent launch: let the next kernel launch at once; `wait`
// = griddepcontrol.wait (full predecessor completion + flush) before the load
__global__ void pdl_kernel(int* p, int wait) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) p[1] = p[0] + 1;
}

int main(int argc, char** argv) {
    const int ctas = argc > 1 ? atoi(argv[1]) : 128;
    const int stages = argc > 2 ? atoi(argv[2]) : 1;
    const size_t host_bytes = (size_t)4 << 30;
    const size_t rows = host_bytes / 512;
    char* host;
    CK(cudaHostAlloc(&host, host_bytes, cudaHostAllocMapped));
    for (size_t i = 0; i < host_bytes; i += 4096) host[i] = 1;
    char* dev;
    CK(cudaMalloc(&dev, (size_t)1 << 30));
    int* flag;
    CK(cudaMalloc(&flag, 1 << 20));
    CK(cudaMemset(flag, 0, 1 << 20));
    cudaStream_t sa_, sb;
    CK(cudaStreamCreateWithFlags(&sa_, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, g0, g1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&g0));
    CK(cudaEventCreate(&g1));
    CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 512));
    const int N = 200;
    auto chain = [&](int which) {
        CK(cudaEventRecord(e0, sb));
        for (int i = 0; i < N; ++i) {
            if (which == 0)
                empty_kernel<<<1, 32, 0, sb>>>(flag);
            else if (which == 1)
                load_kernel<<<1, 32, 0, sb>>>(flag);
            else if (which == 2)
                load_kernel<<<148, 256, 0, sb>>>(flag);
            else {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(which == 5 ? 148 : 1);
                cfg.blockDim = dim3(which == 5 ? 256 : 32);
                cfg.stream = sb;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                CK(cudaLaunchKernelEx(&cfg, pdl_kernel, flag, which == 4 ? 1 : 0));
            }
        }
        CK(cudaEventRecord(e1, sb));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms * 1000.f / N;
    };
    const char* names[6] = {"empty<<<1,32>>>", "1-load<<<1,32>>>", "1-load<<<148,256>>>", "pdl-nowait<<<1,32>>>",
                            "pdl-wait<<<1,32>>>", "pdl-nowait<<<148,256>>>"};
    for (int w = 0; w < 6; ++w) chain(w);  // warm
    for (int w = 0; w < 6; ++w) printf("alone            %-22s %7.2f us/kernel\n", names[w], chain(w));
    // graph-captured chain (the engine's form)
    auto graph_chain = [&](int which) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(sb, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < N; ++i) {
            if (which == 0)
                empty_kernel<<<1, 32, 0, sb>>>(flag);
            else {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(1);
                cfg.blockDim = dim3(32);
                cfg.stream = sb;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                CK(cudaLaunchKernelEx(&cfg, pdl_kernel, flag, which == 2 ? 1 : 0));
            }
        }
        CK(cudaStreamEndCapture(sb, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphLaunch(ge, sb));
        CK(cudaStreamSynchronize(sb));
        CK(cudaEventRecord(e0, sb));
        CK(cudaGraphLaunch(ge, sb));
        CK(cudaEventRecord(e1, sb));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms * 1000.f / N;
    };
    const char* gnames[3] = {"graph empty", "graph pdl-nowait", "graph pdl-wait"};
    for (int w = 0; w < 3; ++w) printf("alone            %-22s %7.2f us/kernel\n", gnames[w], graph_chain(w));
    for (int w = 0; w < 3; ++w) {
        CK(cudaEventRecord(g0, sa_));
        tma_gather<<<ctas, 32, stages * 32 * 512, sa_>>>(host, rows, dev, 4000, stages, 999u + w);
        CK(cudaEventRecord(g1, sa_));
        usleep(2000);
        const float us = graph_chain(w);
        CK(cudaEventSynchronize(g1));
        printf("beside TMA gather %-22s %7.2f us/kernel\n", gnames[w], us);
    }
    for (int mode = 0; mode < 1; ++mode) {
        for (int w = 0; w < 6; ++w) {
            const int iters = 4000;
            CK(cudaEventRecord(g0, sa_));
            if (mode == 0)
                tma_gather<<<ctas, 32, stages * 32 * 512, sa_>>>(host, rows, dev, iters, stages, 12345u + w);
            else
                lsu_gather<<<ctas, 256, 0, sa_>>>((const uint4*)host, rows, (uint4*)dev, iters / 8, 777u + w);
            CK(cudaEventRecord(g1, sa_));
            // start the chain once the gather is in flight
            usleep(2000);
            const float us = chain(w);
            CK(cudaEventSynchronize(g1));
            float gms;
            CK(cudaEventElapsedTime(&gms, g0, g1));
            const double bytes = mode == 0 ? (double)ctas * iters * 32 * 512 : (double)ctas * (iters / 8) * 8 * 256 * 16;
            printf("beside %s gather %-22s %7.2f us/kernel   (gather %.1f GB/s, %.1f ms)\n", mode ? "LSU" : "TMA",
                   names[w], us, bytes / (gms * 1e6), gms);
        }
    }
    return 0;
}
