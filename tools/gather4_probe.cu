// gather4_probe.cu — does TMA tile::gather4 (sm_100a) fill the attention
// kernel's 128-byte-swizzled stage layout from 4 arbitrary rows per op?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/gather4_probe tools/gather4_probe.cu
// Prints "gather4 ok boxrows=R" for each tensor-map box height that works.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void probe(const CUtensorMap* tm, const int* rows, uint16_t* out, int tile_rows) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    const int bytes = tile_rows * 256;  // 128 bf16 per row
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        for (int hh = 0; hh < 2; ++hh)
            for (int q = 0; q < tile_rows / 4; ++q)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(s + hh * tile_rows * 128 + q * 512),
                    "l"(tm), "r"(hh * 64), "r"(rows[4 * q]), "r"(rows[4 * q + 1]), "r"(rows[4 * q + 2]),
                    "r"(rows[4 * q + 3]), "r"(b)
                    : "memory");
    }
    __syncthreads();
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(b)
        : "memory");
    // un-swizzle: row r, 16-byte chunk c at (c>>3)*(TM*128) + r*128 + (((c&7)^(r&7))<<4)
    for (int i = threadIdx.x; i < tile_rows * 16; i += blockDim.x) {
        const int r = i / 16, c = i % 16;
        const uint32_t off = (c >> 3) * (tile_rows * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
        const uint4 v = *reinterpret_cast<const uint4*>(sm + off);
        reinterpret_cast<uint4*>(out)[r * 16 + c] = v;
    }
}

int main() {
    const int N = 4096, D = 128, TM = 16;
    std::vector<uint16_t> h((size_t)N * D);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
    uint16_t* dsrc;
    cudaMalloc(&dsrc, h.size() * 2);
    cudaMemcpy(dsrc, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    int hrows[TM];
    for (int i = 0; i < TM; ++i) hrows[i] = (i * 977 + 13) % N;
    int* drows;
    cudaMalloc(&drows, sizeof hrows);
    cudaMemcpy(drows, hrows, sizeof hrows, cudaMemcpyHostToDevice);
    uint16_t* dout;
    cudaMalloc(&dout, TM * D * 2);
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<EncodeFn>(fn);
    int ok_any = 0;
    for (unsigned boxr : {1u, 4u}) {
        CUtensorMap tm;
        const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)N};
        const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
        const cuuint32_t box[2] = {64, boxr};
        const cuuint32_t es[2] = {1, 1};
        CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dsrc, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode boxrows=%u failed %d\n", boxr, (int)r);
            continue;
        }
        CUtensorMap* dtm;
        cudaMalloc(&dtm, sizeof tm);
        cudaMemcpy(dtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
        cudaMemset(dout, 0, TM * D * 2);
        probe<<<1, 128, TM * 256>>>(dtm, drows, dout, TM);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("boxrows=%u: %s\n", boxr, cudaGetErrorString(e));
            return 1;  // context is dead after a fault
        }
        std::vector<uint16_t> got(TM * D);
        cudaMemcpy(got.data(), dout, got.size() * 2, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < TM; ++r)
            for (int c = 0; c < D; ++c) bad += got[r * D + c] != h[(size_t)hrows[r] * D + c];
        printf("gather4 boxrows=%u: %s (%d mismatches)\n", boxr, bad ? "MISMATCH" : "ok", bad);
        ok_any |= !bad;
        cudaFree(dtm);
    }
    return ok_any ? 0 : 2;
}
