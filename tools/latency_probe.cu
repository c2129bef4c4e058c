// latency_probe.cu — memory latency seen by other kernels while a zero-copy
// gather streams host rows over PCIe, against the gather's depth.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/latency_probe tools/latency_probe.cu
//   tools/latency_probe
//
// For each gather shape (TMA bulk rows: one-warp CTAs x stages; LSU: 256-thread
// CTAs x 8 16-byte loads in flight per thread) it runs the gather on one
// stream and, beside it, (a) a one-thread pointer chase over an HBM buffer
// larger than L2 and over one that stays in L2 (ns per dependent load) and
// (b) a chain of empty graph-captured kernels (us per boundary). Prints the
// gather's GB/s next to them. Rows are 512 bytes (a bf16 d=128 K|V token),
// drawn from a pinned host buffer of PROBE_MIB MiB (default 4096: larger than
// L2, which caches host reads made by LSU loads).
#include <cuda_runtime.h>
#include <stdint.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_gather(const char* host, size_t rows, char* dev, int iters, int stages, unsigned seed,
                           volatile int* stop) {
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
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                         sa(st + ((size_t)s * 32 + lane) * 512)),
                     "l"(host + (size_t)(x % rows) * 512), "r"(sa(&bar[s]))
                     : "memory");
    };
    for (int i = 0; i < stages && i < iters; ++i) load(i);
    int i = 0;
    for (; i < iters; ++i) {
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
        if (*stop) break;
        if (i + stages < iters) load(i + stages);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    // drain the stages still in flight
    for (int j = i + 1; j < iters && j < i + stages; ++j)
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                sa(&bar[j % stages])),
            "r"((j / stages) & 1)
            : "memory");
}

// each warp copies whole 512-byte rows: lane l moves 16 bytes of a row; U rows in flight per warp
template <int U>
__global__ void lsu_gather(const uint4* host, size_t rows, uint4* dev, int iters, unsigned seed, volatile int* stop) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = seed ^ (blockIdx.x * 9781u + warp * 6271u);
    for (int i = 0; i < iters; ++i) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x = x * 1664525u + 1013904223u;
            r[u] = host[(size_t)(x % rows) * 32 + lane];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) dev[(((size_t)blockIdx.x * 8 + warp) * 8 + (u & 7)) * 32 + lane] = r[u];
        if (*stop) break;
    }
}

__global__ void chase(const uint32_t* next, int hops, unsigned long long* out) {
    uint32_t i = 0;
    const unsigned long long t0 = clock64();
    for (int h = 0; h < hops; ++h) i = __ldcg(next + i);
    const unsigned long long t1 = clock64();
    out[0] = t1 - t0;
    out[1] = i;
}

// cost of synchronisation primitives, ns per op (thread 0 of CTA 0 times 64 ops)
__device__ __forceinline__ void cl_sync(int relaxed) {
    if (relaxed)
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    else
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__global__ void sync_ops(int op, int* scratch, unsigned long long* out) {
    const unsigned long long t0 = clock64();
    for (int i = 0; i < 64; ++i) {
        switch (op) {
            case 0: __syncthreads(); break;
            case 1: __threadfence(); break;
            case 2: asm volatile("fence.acq_rel.cluster;" ::: "memory"); break;
            case 3: cl_sync(0); break;
            case 4: cl_sync(1); break;
            case 5: if (threadIdx.x == 0) atomicAdd(scratch + blockIdx.x, 1); __syncthreads(); break;
            case 6: scratch[blockIdx.x * 64 + threadIdx.x % 64] = i; __threadfence(); break;
            default: asm volatile("fence.acq_rel.gpu;" ::: "memory"); break;
        }
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

__global__ void empty_kernel(int* p) {
    if (threadIdx.x == 1000000) *p = 1;
}

int main() {
    const size_t host_bytes = (size_t)(getenv("PROBE_MIB") ? atoi(getenv("PROBE_MIB")) : 4096) << 20;
    const size_t rows = host_bytes / 512;
    char* host;
    CK(cudaHostAlloc(&host, host_bytes, cudaHostAllocMapped));
    for (size_t i = 0; i < host_bytes; i += 4096) host[i] = 1;
    char* dev;
    CK(cudaMalloc(&dev, (size_t)256 << 20));
    int* stop;
    CK(cudaMallocManaged(&stop, sizeof(int)));
    int* flag;
    CK(cudaMalloc(&flag, 64));
    int* flag_big;
    CK(cudaMalloc(&flag_big, 1 << 20));
    // pointer-chase rings: 512 MiB (HBM) and 4 MiB (L2), stride 4 KiB + random
    auto ring = [](size_t elems) {
        std::vector<uint32_t> v(elems);
        std::vector<uint32_t> perm(elems / 1024);
        for (size_t i = 0; i < perm.size(); ++i) perm[i] = (uint32_t)i;
        srand(7);
        for (size_t i = perm.size() - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
        for (size_t i = 0; i < perm.size(); ++i) v[(size_t)perm[i] * 1024] = perm[(i + 1) % perm.size()] * 1024;
        uint32_t* d;
        CK(cudaMalloc(&d, elems * 4));
        CK(cudaMemcpy(d, v.data(), elems * 4, cudaMemcpyHostToDevice));
        return d;
    };
    uint32_t* hbm_ring = ring((size_t)128 << 20);
    uint32_t* l2_ring = ring((size_t)1 << 20);
    unsigned long long* out;
    CK(cudaMalloc(&out, 16));
    cudaStream_t sg, sc;
    CK(cudaStreamCreateWithFlags(&sg, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 512));
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(sc, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < 100; ++i) empty_kernel<<<1, 32, 0, sc>>>(flag);
    CK(cudaStreamEndCapture(sc, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t e0, e1, g0, g1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&g0));
    CK(cudaEventCreate(&g1));
    auto measure = [&](const char* label) {
        unsigned long long h[2];
        chase<<<1, 1, 0, sc>>>(hbm_ring, 2000, out);
        CK(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, sc));
        CK(cudaStreamSynchronize(sc));
        const double hbm_ns = h[0] / 2000.0 / (clk_khz * 1e-6);
        chase<<<1, 1, 0, sc>>>(l2_ring, 2000, out);
        CK(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, sc));
        CK(cudaStreamSynchronize(sc));
        const double l2_ns = h[0] / 2000.0 / (clk_khz * 1e-6);
        CK(cudaEventRecord(e0, sc));
        CK(cudaGraphLaunch(ge, sc));
        CK(cudaEventRecord(e1, sc));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("%-22s hbm-miss load %7.0f ns  l2-hit load %7.0f ns  kernel boundary %6.2f us", label, hbm_ns, l2_ns,
               ms * 1000.f / 100);
        const char* names[8] = {"syncthreads", "threadfence", "fence.cluster", "clbar.rel", "clbar.relaxed",
                                "atomic+sync", "store+fence", "fence.acq_rel.gpu"};
        for (int op = 0; op < 8; ++op) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(8);
            cfg.blockDim = dim3(256);
            cfg.stream = sc;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 4;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, sync_ops, op, flag_big, out));
            CK(cudaMemcpyAsync(h, out, 8, cudaMemcpyDeviceToHost, sc));
            CK(cudaStreamSynchronize(sc));
            printf("  %s %.0f", names[op], h[0] / 64.0 / (clk_khz * 1e-6));
        }
    };
    measure("idle");
    printf("\n");
    struct Shape {
        int tma, ctas, stages;  // LSU: stages = rows in flight per warp (8 or 32)
    };
    std::vector<Shape> shapes = {{1, 16, 1}, {1, 32, 1}, {1, 48, 1}, {1, 64, 1}, {1, 128, 1}, {0, 16, 8}, {0, 48, 8}};
    for (const Shape& s : shapes) {
        *stop = 0;
        const int iters = 1 << 20;
        CK(cudaEventRecord(g0, sg));
        if (s.tma)
            tma_gather<<<s.ctas, 32, s.stages * 32 * 512, sg>>>(host, rows, dev, iters, s.stages, 12345u, stop);
        else
            (s.stages == 32 ? lsu_gather<32> : lsu_gather<8>)<<<s.ctas, 256, 0, sg>>>((const uint4*)host, rows, (uint4*)dev, iters, 777u, stop);
        CK(cudaEventRecord(g1, sg));
        usleep(20000);
        char label[64];
        snprintf(label, sizeof label, "%s %d x %d", s.tma ? "TMA" : "LSU", s.ctas, s.stages);
        measure(label);
        // gather rate over a fixed window
        *stop = 1;
        CK(cudaEventSynchronize(g1));
        float gms;
        CK(cudaEventElapsedTime(&gms, g0, g1));
        printf("   (ran %.1f ms)\n", gms);
    }
    // gather GB/s per shape, alone, fixed work
    for (const Shape& s : shapes) {
        *stop = 0;
        const int iters = s.tma ? 2000 : (s.stages == 32 ? 64 : 250);
        CK(cudaEventRecord(g0, sg));
        if (s.tma)
            tma_gather<<<s.ctas, 32, s.stages * 32 * 512, sg>>>(host, rows, dev, iters, s.stages, 999u, stop);
        else
            (s.stages == 32 ? lsu_gather<32> : lsu_gather<8>)<<<s.ctas, 256, 0, sg>>>((const uint4*)host, rows, (uint4*)dev, iters, 555u, stop);
        CK(cudaEventRecord(g1, sg));
        CK(cudaEventSynchronize(g1));
        float gms;
        CK(cudaEventElapsedTime(&gms, g0, g1));
        const double bytes = s.tma ? (double)s.ctas * iters * 32 * 512 : (double)s.ctas * iters * 8 * s.stages * 512;
        printf("%s %3d x %d alone: %.1f GB/s\n", s.tma ? "TMA" : "LSU", s.ctas, s.stages,
               bytes / (gms * 1e6));
    }
    return 0;
}
