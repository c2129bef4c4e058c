// pdl_exit_probe.cu — can a kernel chain cross its boundaries without the
// grid-completion flush that waits behind queued zero-copy host reads?
// (round-2 follow-up of boundary_probe.cu: a plain graph edge costs ~37 us
// beside a 128-CTA gather, an early-trigger PDL edge ~1 us.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/pdl_exit_probe tools/pdl_exit_probe.cu
//   tools/pdl_exit_probe [gather_ctas]
//
// A graph-captured chain of N kernels (148 x 256 threads). Kernel i's CTA b
// writes v[i][b] = v[i-1][(b+1) % G] + 1, so a stale read anywhere shows as a
// final value below N. Edge variants:
//   full      plain stream order (grid completion + flush)
//   pdl-exit  programmatic edge, no explicit trigger (CTA exit), no wait
//   pdl-exitw programmatic edge, CTA-exit trigger, griddepcontrol.wait
//   pdl-cnt   programmatic edge, CTA-exit trigger, release counter per CTA
//             (fence + atomicAdd) and acquire spin in the consumer's prologue
//   conv-cnt  plain capture, edges converted to programmatic after capture
//             (cudaGraphAddDependencies_v2), counter protocol as pdl-cnt
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

__global__ void tma_gather(const char* host, size_t host_rows, char* dev, int iters, unsigned seed) {
    extern __shared__ __align__(128) char st[];
    __shared__ __align__(8) uint64_t bar[1];
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned x = seed ^ (blockIdx.x * 9781u + lane * 6271u);
    for (int i = 0; i < iters; ++i) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[0])), "r"(32 * 512)
                         : "memory");
        __syncwarp();
        x = x * 1664525u + 1013904223u;
        const size_t row = x % host_rows;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                         sa(st + (size_t)lane * 512)),
                     "l"(host + row * 512), "r"(sa(&bar[0]))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                sa(&bar[0])),
            "r"(i & 1)
            : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(
                         dev + (((size_t)blockIdx.x * 32 + lane) * 512)),
                     "r"(sa(st + (size_t)lane * 512))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// mode: 0 none, 1 griddepcontrol.wait, 2 counter acquire/release
__global__ void chain_kernel(int* v, int i, int mode, unsigned* cnt, unsigned epoch) {
    const int G = gridDim.x, b = blockIdx.x;
    if (mode == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (mode == 2 && i > 0) {
        if (threadIdx.x == 0) {
            unsigned c;
            const unsigned want = epoch * (unsigned)G;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(cnt + i - 1) : "memory");
            } while ((int)(c - want) < 0);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) v[i * G + b] = (i ? v[(i - 1) * G + (b + 1) % G] : 0) + 1;
    if (mode == 2) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(cnt + i, 1u);
        }
    }
}

int main(int argc, char** argv) {
    const int ctas = argc > 1 ? atoi(argv[1]) : 128;
    const size_t host_bytes = (size_t)4 << 30;
    const size_t rows = host_bytes / 512;
    char* host;
    CK(cudaHostAlloc(&host, host_bytes, cudaHostAllocMapped));
    for (size_t i = 0; i < host_bytes; i += 4096) host[i] = 1;
    char* dev;
    CK(cudaMalloc(&dev, (size_t)1 << 28));
    const int N = 200, G = 148;
    int* v;
    unsigned* cnt;
    CK(cudaMalloc(&v, sizeof(int) * N * G));
    CK(cudaMalloc(&cnt, sizeof(unsigned) * N));
    CK(cudaMemset(cnt, 0, sizeof(unsigned) * N));
    cudaStream_t sa_, sb;
    CK(cudaStreamCreateWithFlags(&sa_, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, g0, g1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&g0));
    CK(cudaEventCreate(&g1));
    CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 512));
    const char* names[5] = {"full", "pdl-exit", "pdl-exitw", "pdl-cnt", "conv-cnt"};
    cudaGraphExec_t ge[5];
    for (int w = 0; w < 5; ++w) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(sb, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < N; ++i) {
            const int mode = w == 2 ? 1 : (w >= 3 ? 2 : 0);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(256);
            cfg.stream = sb;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = (w >= 1 && w <= 3 && i > 0) ? 1 : 0;
            // epoch patched per replay through a device-side counter would be
            // the engine's form; here every replay gets its own graph exec
            // update, so pass epoch 1 and reset the counters between replays
            CK(cudaLaunchKernelEx(&cfg, chain_kernel, v, i, mode, cnt, 1u));
        }
        CK(cudaStreamEndCapture(sb, &g));
        if (w == 4) {  // convert every kernel->kernel edge to a programmatic one
            size_t ne = 0;
            CK(cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne));
            std::vector<cudaGraphNode_t> from(ne), to(ne);
            std::vector<cudaGraphEdgeData> ed(ne);
            CK(cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne));
            CK(cudaGraphRemoveDependencies_v2(g, from.data(), to.data(), ed.data(), ne));
            for (auto& e : ed) {
                e.from_port = cudaGraphKernelNodePortProgrammatic;
                e.type = cudaGraphDependencyTypeProgrammatic;
            }
            CK(cudaGraphAddDependencies_v2(g, from.data(), to.data(), ed.data(), ne));
        }
        CK(cudaGraphInstantiate(&ge[w], g, 0));
    }
    auto run = [&](int w) {
        CK(cudaMemsetAsync(v, 0, sizeof(int) * N * G, sb));
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * N, sb));
        CK(cudaEventRecord(e0, sb));
        CK(cudaGraphLaunch(ge[w], sb));
        CK(cudaEventRecord(e1, sb));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::vector<int> h(G);
        CK(cudaMemcpy(h.data(), v + (size_t)(N - 1) * G, sizeof(int) * G, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int b = 0; b < G; ++b) bad += h[b] != N;
        return std::make_pair(ms * 1000.f / N, bad);
    };
    for (int w = 0; w < 5; ++w) run(w);
    for (int w = 0; w < 5; ++w) {
        float best = 1e30f;
        int bad = 0;
        for (int r = 0; r < 5; ++r) {
            auto x = run(w);
            best = x.first < best ? x.first : best;
            bad += x.second;
        }
        printf("alone             %-10s %7.2f us/kernel  stale %d\n", names[w], best, bad);
    }
    for (int w = 0; w < 5; ++w) {
        float tot = 0;
        int bad = 0;
        const int R = 20;
        CK(cudaEventRecord(g0, sa_));
        tma_gather<<<ctas, 32, 32 * 512, sa_>>>(host, rows, dev, 20000, 999u + w);
        CK(cudaEventRecord(g1, sa_));
        usleep(3000);
        for (int r = 0; r < R; ++r) {
            auto x = run(w);
            tot += x.first;
            bad += x.second;
        }
        CK(cudaEventSynchronize(g1));
        float gms;
        CK(cudaEventElapsedTime(&gms, g0, g1));
        printf("beside TMA gather %-10s %7.2f us/kernel  stale %d  (gather %.1f GB/s over %.0f ms)\n", names[w],
               tot / R, bad, (double)ctas * 20000 * 32 * 512 / (gms * 1e6), gms);
    }
    printf("done\n");
    return 0;
}
