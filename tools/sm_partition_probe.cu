// sm_partition_probe.cu — do kernel boundaries stall only on SMs that host
// queued zero-copy host reads?
//
// pdl_exit_probe showed that beside a 128-CTA TMA gather even a per-thread
// __threadfence() after a store, or a CTA exit, waits tens of microseconds:
// the wait looks per-SM (the SM drains its outstanding memory requests, which
// include the gather's queued host reads). If so, a gather whose CTAs each
// reserve a whole SM's shared memory (no other CTA can co-reside) keeps the
// rest of the GPU's boundaries fast.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/sm_partition_probe tools/sm_partition_probe.cu
//   tools/sm_partition_probe
//
// For each gather shape (CTAs x warps per CTA x stages per warp, shared-memory
// reservation): the gather's rate alone over a 4 GiB pinned region (random
// 512-byte rows), and the per-kernel time of a graph-captured chain of 200
// kernels (148 x 256 threads, one store + fence each) launched beside it.
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

// every warp: its own ring of `stages` 32-row stages; lane 0 arms, each lane copies one row
__global__ void tma_gather(const char* host, size_t host_rows, char* dev, int iters, int stages, unsigned seed) {
    extern __shared__ __align__(128) char st[];
    __shared__ __align__(8) uint64_t bar[32 * 8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    char* ring = st + (size_t)w * stages * 32 * 512;
    uint64_t* wb = bar + w * 8;
    if (lane == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&wb[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned x = seed ^ (blockIdx.x * 9781u + threadIdx.x * 6271u);
    auto load = [&](int i) {
        const int s = i % stages;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&wb[s])), "r"(32 * 512)
                         : "memory");
        __syncwarp();
        x = x * 1664525u + 1013904223u;
        const size_t row = x % host_rows;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                         sa(ring + ((size_t)s * 32 + lane) * 512)),
                     "l"(host + row * 512), "r"(sa(&wb[s]))
                     : "memory");
    };
    for (int i = 0; i < stages && i < iters; ++i) load(i);
    for (int i = 0; i < iters; ++i) {
        const int s = i % stages;
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                sa(&wb[s])),
            "r"((i / stages) & 1)
            : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(
                         dev + (((size_t)(blockIdx.x * 32 + w) * 32 + lane) * 512)),
                     "r"(sa(ring + ((size_t)s * 32 + lane) * 512))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        if (i + stages < iters) load(i + stages);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void chain_kernel(int* v, int i) {
    const int G = gridDim.x, b = blockIdx.x;
    if (threadIdx.x == 0) v[i * G + b] = (i ? v[(i - 1) * G + (b + 1) % G] : 0) + 1;
}

int main() {
    const size_t host_bytes = (size_t)4 << 30;
    const size_t rows = host_bytes / 512;
    char* host;
    CK(cudaHostAlloc(&host, host_bytes, cudaHostAllocMapped));
    for (size_t i = 0; i < host_bytes; i += 4096) host[i] = 1;
    char* dev;
    CK(cudaMalloc(&dev, (size_t)1 << 30));
    const int N = 200, G = 148;
    int* v;
    CK(cudaMalloc(&v, sizeof(int) * N * G));
    cudaStream_t sa_, sb;
    CK(cudaStreamCreateWithFlags(&sa_, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, g0, g1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&g0));
    CK(cudaEventCreate(&g1));
    CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(sb, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < N; ++i) chain_kernel<<<G, 256, 0, sb>>>(v, i);
    CK(cudaStreamEndCapture(sb, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    auto chain = [&]() {
        CK(cudaEventRecord(e0, sb));
        CK(cudaGraphLaunch(ge, sb));
        CK(cudaEventRecord(e1, sb));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms * 1000.f / N;
    };
    chain();
    printf("chain alone: %.2f us/kernel\n", chain());
    struct Shape {
        int ctas, warps, stages, reserve_kb;
    };
    const Shape shapes[] = {{128, 1, 1, 0},  {128, 1, 1, 225}, {32, 4, 1, 225}, {32, 4, 2, 225}, {40, 4, 1, 225},
                            {48, 3, 1, 225}, {24, 4, 2, 225},  {64, 2, 1, 225}, {32, 4, 1, 0},   {48, 4, 1, 225},
                            {40, 6, 1, 225}, {32, 8, 1, 225},  {56, 4, 1, 225}, {64, 4, 1, 225}};
    for (const Shape& s : shapes) {
        const size_t need = (size_t)s.warps * s.stages * 32 * 512;
        const size_t smem = need > (size_t)s.reserve_kb * 1024 ? need : (size_t)s.reserve_kb * 1024;
        // iterations per warp so that the gather moves ~16 GiB in total
        const int iters = (int)((16ull << 30) / ((size_t)s.ctas * s.warps * 32 * 512));
        // alone
        CK(cudaEventRecord(g0, sa_));
        tma_gather<<<s.ctas, s.warps * 32, smem, sa_>>>(host, rows, dev, iters / 4, s.stages, 7u);
        CK(cudaEventRecord(g1, sa_));
        CK(cudaEventSynchronize(g1));
        float gms;
        CK(cudaEventElapsedTime(&gms, g0, g1));
        const double alone = (double)s.ctas * s.warps * (iters / 4) * 32 * 512 / (gms * 1e6);
        // beside the chain
        CK(cudaEventRecord(g0, sa_));
        tma_gather<<<s.ctas, s.warps * 32, smem, sa_>>>(host, rows, dev, iters, s.stages, 11u);
        CK(cudaEventRecord(g1, sa_));
        usleep(3000);
        float tot = 0;
        const int R = 10;
        for (int r = 0; r < R; ++r) tot += chain();
        CK(cudaEventSynchronize(g1));
        CK(cudaEventElapsedTime(&gms, g0, g1));
        const double beside = (double)s.ctas * s.warps * iters * 32 * 512 / (gms * 1e6);
        printf("gather %3d CTAs x %d warps x %d stages, smem %3zu KiB: alone %5.1f GB/s | chain beside %6.2f us/kernel "
               "(gather %5.1f GB/s over %.0f ms)\n",
               s.ctas, s.warps, s.stages, smem >> 10, alone, tot / R, beside, gms);
    }
    printf("done\n");
    return 0;
}
