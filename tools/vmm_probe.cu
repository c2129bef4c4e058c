// vmm_probe.cu — experiment: does mapping the pinned host K/V store through
// the CUDA VMM API (cuMemCreate on a HOST_NUMA location, 2 MiB granularity)
// keep the zero-copy gather rate up over large stores, where cudaHostAlloc'd
// memory drops from ~48 GB/s (8 GB) to ~19 GB/s (34 GB)?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o vmm_probe vmm_probe.cu
// Run:   ./vmm_probe <store GiB> <heads> <rows per head>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

template <typename F>
F entry(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q));
    if (!fn) {
        std::printf("no entry point %s\n", name);
        std::exit(1);
    }
    return reinterpret_cast<F>(fn);
}

__global__ void gather(const uint4* __restrict__ src, uint4* __restrict__ dst, const int64_t* __restrict__ rows,
                       int nrows, int vpr) {
    const int64_t total = (int64_t)nrows * vpr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / vpr, c = i % vpr;
        dst[i] = src[rows[r] * vpr + c];
    }
}

int main(int argc, char** argv) {
    const double gib = argc > 1 ? atof(argv[1]) : 34.0;
    const int heads = argc > 2 ? atoi(argv[2]) : 64;
    const int per = argc > 3 ? atoi(argv[3]) : 2048;
    const size_t row = 256, vpr = row / 16;
    const size_t bytes = (size_t)(gib * (1ull << 30)) / (2ull << 20) * (2ull << 20);
    const int64_t nrows_store = bytes / row;
    const int64_t per_head = nrows_store / heads;
    CK(cudaSetDevice(0));
    CK(cudaFree(0));

    // random sorted rows per head
    std::mt19937_64 rng(7);
    std::vector<int64_t> rows;
    for (int h = 0; h < heads; ++h) {
        std::vector<int64_t> r(per);
        for (auto& x : r) x = h * per_head + (int64_t)(rng() % per_head);
        std::sort(r.begin(), r.end());
        rows.insert(rows.end(), r.begin(), r.end());
    }
    int64_t* drows;
    uint4* dst;
    CK(cudaMalloc(&drows, rows.size() * 8));
    CK(cudaMemcpy(drows, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dst, rows.size() * row));

    auto bench = [&](const char* what, const void* src) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a);
            gather<<<148 * 8, 256>>>((const uint4*)src, dst, drows, (int)rows.size(), (int)vpr);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = std::min(best, ms);
        }
        CK(cudaGetLastError());
        std::printf("%-34s store %.1f GiB, %d heads x %d rows: %.1f GB/s\n", what, bytes / double(1ull << 30), heads,
                    per, rows.size() * row / (best * 1e-3) / 1e9);
    };

    {  // baseline: cudaHostAlloc mapped
        void* p;
        CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
        CK(cudaMemset(p, 1, bytes));
        CK(cudaDeviceSynchronize());
        bench("cudaHostAlloc (mapped)", p);
        CK(cudaFreeHost(p));
    }
    {  // VMM: host-NUMA physical memory mapped into the GPU VA space
        auto pCreate = entry<CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                                          unsigned long long)>("cuMemCreate");
        auto pGran = entry<CUresult (*)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags)>(
            "cuMemGetAllocationGranularity");
        auto pReserve = entry<CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long)>(
            "cuMemAddressReserve");
        auto pMap = entry<CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long)>(
            "cuMemMap");
        auto pAccess = entry<CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t)>("cuMemSetAccess");
        for (int rec = 0; rec < 2; ++rec) {
            CUmemAllocationProp prop = {};
            prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
            prop.location.id = 0;
            size_t g = 0;
            CUresult r = pGran(&g, &prop, rec ? CU_MEM_ALLOC_GRANULARITY_RECOMMENDED : CU_MEM_ALLOC_GRANULARITY_MINIMUM);
            std::printf("host-NUMA granularity (%s): %zu (cu %d)\n", rec ? "recommended" : "minimum", g, (int)r);
            if (r != CUDA_SUCCESS) return 0;
            const size_t len = (bytes + g - 1) / g * g;
            CUmemGenericAllocationHandle h;
            r = pCreate(&h, len, &prop, 0);
            if (r != CUDA_SUCCESS) {
                std::printf("cuMemCreate host-NUMA failed: %d\n", (int)r);
                return 0;
            }
            CUdeviceptr va;
            r = pReserve(&va, len, 2ull << 20, 0, 0);
            if (r == CUDA_SUCCESS) r = pMap(va, len, 0, h, 0);
            CUmemAccessDesc ad[2] = {};
            ad[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            ad[0].location.id = 0;
            ad[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            if (r == CUDA_SUCCESS) r = pAccess(va, len, ad, 1);
            if (r != CUDA_SUCCESS) {
                std::printf("map/access failed: %d\n", (int)r);
                return 0;
            }
            CK(cudaMemset((void*)va, 1, bytes));
            CK(cudaDeviceSynchronize());
            bench(rec ? "VMM host-NUMA (recommended gran)" : "VMM host-NUMA (minimum gran)", (void*)va);
            // can the CPU touch it at the same address? (host access descriptor)
            ad[1].location.type = CU_MEM_LOCATION_TYPE_HOST;
            ad[1].location.id = 0;
            ad[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            r = pAccess(va, len, ad + 1, 1);
            std::printf("host access descriptor: %d\n", (int)r);
            if (r == CUDA_SUCCESS) {
                volatile unsigned char* c = (unsigned char*)va;
                std::printf("CPU reads byte: %d\n", (int)c[12345]);
            }
            // leak: process exits
        }
    }
    return 0;
}
