// attention_tma.cu — K4 sparse attention, TMA-staged variant (production path
// for bf16/f32 rows with d in {64, 128, 256}).
//
// Semantics: topk_attention / attend_rows (attention.cpp:33-55, 91-105) of the
// m GQA query heads of one KV head over union(selection, sink/recent window)
// (union_indices engine.cpp:80-85, sink_recent_indices attention.cpp:107-128),
// fp32 accumulation over the stored bf16/f32 rows.
//
// Structure (one CTA = 4 warps = up to 256 attend positions of one head):
//   * warp 0 streams 32-row K/V tiles into a 3-stage shared-memory ring with
//     cp.async.bulk (TMA 1D bulk copies, mbarrier complete_tx): one 8 KiB copy
//     per operand for a contiguous run of cache slots, one 256 B copy per row
//     for scattered rows (persistent heads, window rows);
//   * QK: 16 lanes per row (8 elements each), packed FFMA2, shuffle reduce;
//   * per-warp online softmax over the warp's 8 rows of each tile (exp2);
//   * PV: lanes own 4 consecutive head dims, packed FFMA2 over the warp's rows;
//   * the 4 warps and the split chunks are merged by the last CTA of the head.
// Each KV row is read from HBM exactly once for all m query heads.
#include <math_constants.h>

#include <cstdlib>

#include "attention.cuh"
#include "exchange.cuh"

namespace clo {

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kTileRows = 32;
constexpr int kStages = 3;
constexpr int kRowsPerWarp = kTileRows / kWarps;  // 8

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA 1D bulk copy global -> shared, completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float safe_exp2(float x) { return x == -CUDART_INF_F ? 0.f : exp2f(x); }
// weight of a partial with running max m under the merged max gm; an empty
// partial (m = -inf) weighs 0 even when gm is -inf too (no NaN)
__device__ __forceinline__ float wexp(float m, float gm) { return m == -CUDART_INF_F ? 0.f : exp2f(m - gm); }

// exp2 on the SFU without the denormal fix-up sequence (args <= 0 here; a
// result below 2^-126 flushing to 0 is irrelevant next to the row maximum)
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Transpose-reduce bookkeeping: the query a QK lane owns after the halving
// levels (bit `off` of sub selects the upper half at each level), and the
// lowest lane (in row group 0) owning query j.
template <int M, int LPR>
__device__ __forceinline__ int split_query(int sub) {
    int j = 0, width = M;
    for (int off = LPR / 2; width > 1; width >>= 1, off >>= 1)
        if (sub & off) j += width / 2;
    return j;
}
template <int M, int LPR>
__device__ __forceinline__ int split_lane(int j) {
    int lane = 0, width = M;
    for (int off = LPR / 2; width > 1; width >>= 1, off >>= 1)
        if (j >= width / 2) {
            lane |= off;
            j -= width / 2;
        }
    return lane;
}

template <typename T>
__device__ __forceinline__ void unpack8(const uint4& u, float2* f);  // 16 B -> float2 pairs
template <>
__device__ __forceinline__ void unpack8<__nv_bfloat16>(const uint4& u, float2* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = __bfloat1622float2(h[i]);
}
template <>
__device__ __forceinline__ void unpack8<float>(const uint4& u, float2* f) {
    f[0] = make_float2(__uint_as_float(u.x), __uint_as_float(u.y));
    f[1] = make_float2(__uint_as_float(u.z), __uint_as_float(u.w));
}

// PV operand: the lane's DPL consecutive dims of one row.
template <typename T, int DPL>
__device__ __forceinline__ void load_pv(const T* row, int lane, float2* f) {
    if constexpr (sizeof(T) == 2) {
        if constexpr (DPL == 4) {
            const uint2 u = *reinterpret_cast<const uint2*>(row + lane * 4);
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
            f[0] = __bfloat1622float2(h[0]);
            f[1] = __bfloat1622float2(h[1]);
        } else if constexpr (DPL == 2) {
            f[0] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(row + lane * 2));
        } else {  // 8
            const uint4 u = *reinterpret_cast<const uint4*>(row + lane * 8);
            unpack8<T>(u, f);
        }
    } else {
        if constexpr (DPL == 4) {
            const float4 u = *reinterpret_cast<const float4*>(row + lane * 4);
            f[0] = make_float2(u.x, u.y);
            f[1] = make_float2(u.z, u.w);
        } else if constexpr (DPL == 2) {
            f[0] = *reinterpret_cast<const float2*>(row + lane * 2);
        } else {
            const float4 u0 = *reinterpret_cast<const float4*>(row + lane * 8);
            const float4 u1 = *reinterpret_cast<const float4*>(row + lane * 8 + 4);
            f[0] = make_float2(u0.x, u0.y);
            f[1] = make_float2(u0.z, u0.w);
            f[2] = make_float2(u1.x, u1.y);
            f[3] = make_float2(u1.z, u1.w);
        }
    }
}

template <typename T, int D, int M, int LMAX>
__global__ void __launch_bounds__(kThreads, 4) attn_tma_kernel(EngineView v, int l) {
    constexpr int EPV = 16 / sizeof(T);          // elements per 16-byte vector
    constexpr int VPR = D / EPV;                 // vectors per row
    constexpr int LPR = VPR < LMAX ? VPR : LMAX; // QK lanes per row
    constexpr int VPL = VPR / LPR;               // QK vectors per lane
    constexpr int RPI = 32 / LPR;                // rows per QK warp-iteration
    constexpr int QIT = kRowsPerWarp / RPI;      // QK iterations per tile
    constexpr int E2 = VPL * EPV / 2;            // float2 per lane in QK
    constexpr int DPL = D / 32;                  // PV dims per lane
    constexpr int P2 = DPL / 2;                  // PV float2 per lane
    constexpr uint32_t kRowBytes = D * sizeof(T);
    static_assert(QIT >= 1 && DPL >= 2, "unsupported head_dim");
    // Transpose-reduce: when M is a power of two <= LPR, each QK lane ends up
    // owning ONE query's full dot (log2(LPR) shuffle levels for all M instead
    // of M*log2(LPR)); otherwise every lane reduces every query.
    constexpr bool kSplit = (M & (M - 1)) == 0 && M <= LPR;

    extern __shared__ __align__(128) unsigned char smem[];
    T* tiles = reinterpret_cast<T*>(smem);  // [kStages][2][kTileRows][D]
    __shared__ __align__(8) uint64_t full[kStages];
    __shared__ __align__(16) int32_t toks[kStages][kTileRows];  // tile tokens (dedup)
    __shared__ float pbuf[kWarps][kRowsPerWarp][M];
    __shared__ int s_last;

    const int c = blockIdx.x, nch = gridDim.x;
    const int bg = blockIdx.y;
    const int b = bg / v.H, g = bg % v.H;
    const int lg = l * v.H + g;
    const int seg = (b * v.L + l) * v.H + g;
    const bool pers = v.persistent[lg] != 0;
    const int t = *v.dev_step + 1;
    const int n_after = v.n_prompt + t;
    const int s1 = min(v.sink, n_after), r1 = min(v.recent, n_after);
    const int wstart = max(n_after - r1, s1);
    const int P = v.k + s1 + (n_after - wstart);
    const int p0 = c * kAttnRows, p1 = min(P, p0 + kAttnRows);
    const int ntiles = (p1 - p0 + kTileRows - 1) / kTileRows;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / LPR, sub = lane % LPR;

    const int32_t* idx = v.entry_idx + (size_t)seg * v.k;
    const size_t pslot = pers ? (size_t)b * v.NP + v.pidx[lg] : 0;
    const size_t oslot = pers ? 0 : (size_t)b * v.NO + v.oidx[lg];
    const int32_t* stok = pers ? nullptr : v.slot_tok + oslot * v.pool;
    const int wrows = v.sink + v.recent;
    const T* pk = static_cast<const T*>(v.pk) + pslot * v.nmax * D;
    const T* pv = static_cast<const T*>(v.pv) + pslot * v.nmax * D;
    const T* sk = static_cast<const T*>(v.slot_k) + oslot * v.pool * D;
    const T* sv = static_cast<const T*>(v.slot_v) + oslot * v.pool * D;
    const T* wk = static_cast<const T*>(v.win_k) + oslot * wrows * D;
    const T* wv = static_cast<const T*>(v.win_v) + oslot * wrows * D;

    // K/V rows of attend position pos
    auto rows_of = [&](int pos, const T*& kr, const T*& vr) {
        if (pos < v.k) {
            if (pers) {
                const int tok = idx[pos];
                kr = pk + (size_t)tok * D;
                vr = pv + (size_t)tok * D;
            } else {
                kr = sk + (size_t)pos * D;
                vr = sv + (size_t)pos * D;
            }
        } else {
            const int w = pos - v.k;
            const int tok = w < s1 ? w : wstart + (w - s1);
            if (pers) {
                kr = pk + (size_t)tok * D;
                vr = pv + (size_t)tok * D;
            } else {
                const int wr = tok < v.sink ? tok : v.sink + tok % v.recent;
                kr = wk + (size_t)wr * D;
                vr = wv + (size_t)wr * D;
            }
        }
    };
    // warp 0: stream tile `ti` into its stage (K rows, V rows and, for the
    // selected part, the tokens the window dedup needs)
    auto issue = [&](int ti) {
        const int s = ti % kStages;
        const int tp = p0 + ti * kTileRows;
        const int rows = min(kTileRows, p1 - tp);
        const int sel_rows = max(0, min(rows, v.k - tp));  // positions < k
        T* kdst = tiles + (size_t)(s * 2) * kTileRows * D;
        T* vdst = kdst + (size_t)kTileRows * D;
        // token copy: whole 16-byte groups (the buffers are padded)
        const uint32_t tok_bytes = sel_rows > 0 ? (uint32_t)((sel_rows + 3) & ~3) * 4u : 0u;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&full[s], 2u * rows * kRowBytes + tok_bytes);
            if (tok_bytes) bulk_g2s(toks[s], (pers ? idx : stok) + tp, tok_bytes, &full[s]);
        }
        __syncwarp();
        if (!pers && tp + rows <= v.k) {  // contiguous cache slots: two bulk copies
            if (lane == 0) {
                bulk_g2s(kdst, sk + (size_t)tp * D, rows * kRowBytes, &full[s]);
                bulk_g2s(vdst, sv + (size_t)tp * D, rows * kRowBytes, &full[s]);
            }
        } else if (lane < rows) {  // scattered rows: one bulk copy per row
            const T* kr;
            const T* vr;
            rows_of(tp + lane, kr, vr);
            bulk_g2s(kdst + (size_t)lane * D, kr, kRowBytes, &full[s]);
            bulk_g2s(vdst + (size_t)lane * D, vr, kRowBytes, &full[s]);
        }
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0)
        for (int ti = 0; ti < min(kStages - 1, ntiles); ++ti) issue(ti);

    // queries, pre-scaled by log2(e)/sqrt(d) so the softmax runs on exp2
    const float scale = 1.4426950408889634f * rsqrtf((float)D);
    float2 q[M][E2];
    {
        const float* qsrc = v.desc->true_q + (((size_t)b * v.L + l) * v.HQ + (size_t)g * M) * D;
        bool badq = false;
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
            for (int i = 0; i < VPL; ++i)
#pragma unroll
                for (int e = 0; e < EPV / 2; ++e) {
                    const float2 x = *reinterpret_cast<const float2*>(qsrc + (size_t)j * D + (sub + i * LPR) * EPV + 2 * e);
                    badq |= !isfinite(x.x) || !isfinite(x.y);
                    q[j][i * EPV / 2 + e] = make_float2(x.x * scale, x.y * scale);
                }
        if (badq) raise_err(v.err, kErrNonFiniteQuery);
    }

    // kSplit: mrun[0]/lrun[0] belong to query qj of this lane; else [j]
    constexpr int MR = kSplit ? 1 : M;
    const int qj = kSplit ? split_query<M, LPR>(sub) : 0;
    float mrun[MR], lrun[MR];
    float2 acc[M][P2];
#pragma unroll
    for (int j = 0; j < MR; ++j) {
        mrun[j] = -CUDART_INF_F;
        lrun[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
        for (int e = 0; e < P2; ++e) acc[j][e] = make_float2(0.f, 0.f);

    for (int ti = 0; ti < ntiles; ++ti) {
        if (warp == 0 && ti + kStages - 1 < ntiles) issue(ti + kStages - 1);
        const int s = ti % kStages;
        const int tp = p0 + ti * kTileRows;
        const int rows = min(kTileRows, p1 - tp);
        mbar_wait(&full[s], (ti / kStages) & 1);
        const T* kt = tiles + (size_t)(s * 2) * kTileRows * D;
        const T* vt = kt + (size_t)kTileRows * D;

        // ---- QK for this warp's rows ------------------------------------
        // kSplit: sc[it][0] is query qj(sub) of row it*RPI+grp; else sc[it][j].
        float sc[QIT][kSplit ? 1 : M];
#pragma unroll
        for (int it = 0; it < QIT; ++it) {
            const int r = warp * kRowsPerWarp + it * RPI + grp;
            float2 kf[E2];
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
                const uint4 u = *reinterpret_cast<const uint4*>(kt + (size_t)r * D + (sub + i * LPR) * EPV);
                unpack8<T>(u, kf + i * EPV / 2);
            }
            bool ok = r < rows;
            if (ok && (tp + r) < v.k) {  // dedup selected tokens against the window
                const int tok = toks[s][r];
                ok = !(tok < s1 || tok >= wstart);
            }
            float dj[M];
#pragma unroll
            for (int j = 0; j < M; ++j) {
                float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int e = 0; e < E2; ++e) a2 = __ffma2_rn(q[j][e], kf[e], a2);
                dj[j] = a2.x + a2.y;
            }
            if constexpr (kSplit) {
                int width = M, off = LPR / 2;
#pragma unroll
                for (; width > 1; width >>= 1, off >>= 1) {
                    const bool hi = sub & off;
#pragma unroll
                    for (int i = 0; i < width / 2; ++i) {
                        const float send = hi ? dj[i] : dj[i + width / 2];
                        const float keep = hi ? dj[i + width / 2] : dj[i];
                        dj[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                    }
                }
#pragma unroll
                for (; off >= 1; off >>= 1) dj[0] += __shfl_xor_sync(0xffffffffu, dj[0], off);
                sc[it][0] = ok ? dj[0] : -CUDART_INF_F;
            } else {
#pragma unroll
                for (int j = 0; j < M; ++j) {
#pragma unroll
                    for (int o = 1; o < LPR; o <<= 1) dj[j] += __shfl_xor_sync(0xffffffffu, dj[j], o);
                    sc[it][j] = ok ? dj[j] : -CUDART_INF_F;
                }
            }
        }
        // ---- online softmax over the warp's rows -------------------------
        float corr_all[M];
        if constexpr (kSplit) {
            float mt = sc[0][0];
#pragma unroll
            for (int it = 1; it < QIT; ++it) mt = fmaxf(mt, sc[it][0]);
#pragma unroll
            for (int o = LPR; o < 32; o <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, o));
            const float mnew = fmaxf(mrun[0], mt);
            const float corr = wexp(mrun[0], mnew);
            mrun[0] = mnew;
            float ps = 0.f;
#pragma unroll
            for (int it = 0; it < QIT; ++it) {
                const float p = sc[it][0] == -CUDART_INF_F ? 0.f : fast_exp2(sc[it][0] - mnew);
                sc[it][0] = p;
                ps += p;
            }
#pragma unroll
            for (int o = LPR; o < 32; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            lrun[0] = lrun[0] * corr + ps;
#pragma unroll
            for (int j = 0; j < M; ++j) corr_all[j] = __shfl_sync(0xffffffffu, corr, split_lane<M, LPR>(j));
            if ((sub & (LPR / M - 1)) == 0) {
#pragma unroll
                for (int it = 0; it < QIT; ++it) pbuf[warp][it * RPI + grp][qj] = sc[it][0];
            }
        } else {
#pragma unroll
            for (int j = 0; j < M; ++j) {
                float mt = sc[0][j];
#pragma unroll
                for (int it = 1; it < QIT; ++it) mt = fmaxf(mt, sc[it][j]);
#pragma unroll
                for (int o = LPR; o < 32; o <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, o));
                const float mnew = fmaxf(mrun[j], mt);
                corr_all[j] = wexp(mrun[j], mnew);
                mrun[j] = mnew;
                float ps = 0.f;
#pragma unroll
                for (int it = 0; it < QIT; ++it) {
                    const float p = sc[it][j] == -CUDART_INF_F ? 0.f : fast_exp2(sc[it][j] - mnew);
                    sc[it][j] = p;
                    ps += p;
                }
#pragma unroll
                for (int o = LPR; o < 32; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
                lrun[j] = lrun[j] * corr_all[j] + ps;
            }
            if (sub == 0) {
#pragma unroll
                for (int it = 0; it < QIT; ++it)
#pragma unroll
                    for (int j = 0; j < M; ++j) pbuf[warp][it * RPI + grp][j] = sc[it][j];
            }
        }
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const float2 c2 = make_float2(corr_all[j], corr_all[j]);
#pragma unroll
            for (int e = 0; e < P2; ++e) acc[j][e] = __fmul2_rn(acc[j][e], c2);
        }
        __syncwarp();
        // ---- PV over the warp's rows -------------------------------------
#pragma unroll
        for (int rr = 0; rr < kRowsPerWarp; ++rr) {
            const int r = warp * kRowsPerWarp + rr;
            if (r >= rows) break;  // rows past the tile end hold stale smem
            float2 vf[P2];
            load_pv<T, DPL>(vt + (size_t)r * D, lane, vf);
#pragma unroll
            for (int j = 0; j < M; ++j) {
                const float p = pbuf[warp][rr][j];
                const float2 p2 = make_float2(p, p);
#pragma unroll
                for (int e = 0; e < P2; ++e) acc[j][e] = __ffma2_rn(p2, vf[e], acc[j][e]);
            }
        }
        __syncthreads();  // stage s is free for the next issue
    }

    // ---- merge the 4 warps, then the split chunks of the head -------------
    float* red = reinterpret_cast<float*>(smem);  // [kWarps][M][D + 2] (tiles are done)
#pragma unroll
    for (int j = 0; j < M; ++j) {
#pragma unroll
        for (int e = 0; e < P2; ++e) {
            red[((size_t)warp * M + j) * (D + 2) + lane * DPL + 2 * e] = acc[j][e].x;
            red[((size_t)warp * M + j) * (D + 2) + lane * DPL + 2 * e + 1] = acc[j][e].y;
        }
        if constexpr (kSplit) {
            const float mj = __shfl_sync(0xffffffffu, mrun[0], split_lane<M, LPR>(j));
            const float lj = __shfl_sync(0xffffffffu, lrun[0], split_lane<M, LPR>(j));
            if (lane == 0) {
                red[((size_t)warp * M + j) * (D + 2) + D] = mj;
                red[((size_t)warp * M + j) * (D + 2) + D + 1] = lj;
            }
        } else if (lane == 0) {
            red[((size_t)warp * M + j) * (D + 2) + D] = mrun[j];
            red[((size_t)warp * M + j) * (D + 2) + D + 1] = lrun[j];
        }
    }
    __syncthreads();
    float* part = v.attn_part + ((size_t)bg * v.max_attn_chunks + c) * M * (D + 2);
    for (int i = threadIdx.x; i < M * D; i += blockDim.x) {
        const int j = i / D, e = i % D;
        float gm = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) gm = fmaxf(gm, red[((size_t)w * M + j) * (D + 2) + D]);
        float a = 0.f, s = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float cw = wexp(red[((size_t)w * M + j) * (D + 2) + D], gm);
            a += red[((size_t)w * M + j) * (D + 2) + e] * cw;
            s += red[((size_t)w * M + j) * (D + 2) + D + 1] * cw;
        }
        part[j * (D + 2) + e] = a;
        if (e == 0) {
            part[j * (D + 2) + D] = gm;
            part[j * (D + 2) + D + 1] = s;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&v.attn_count[bg], 1) == nch - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* pb = v.attn_part + (size_t)bg * v.max_attn_chunks * M * (D + 2);
    const size_t stride = (size_t)M * (D + 2);
    for (int i = threadIdx.x; i < M * D; i += blockDim.x) {
        const int j = i / D, e = i % D;
        float gm = -CUDART_INF_F;
        for (int cc = 0; cc < nch; ++cc) gm = fmaxf(gm, __ldcg(pb + cc * stride + j * (D + 2) + D));
        float a = 0.f, s = 0.f;
        for (int cc = 0; cc < nch; ++cc) {
            const float cw = wexp(__ldcg(pb + cc * stride + j * (D + 2) + D), gm);
            a += __ldcg(pb + cc * stride + j * (D + 2) + e) * cw;
            s += __ldcg(pb + cc * stride + j * (D + 2) + D + 1) * cw;
        }
        emit_head_output(v, t, b, l, g * M + j, e, a / s);
    }
    signal_head_output(v, l);
    if (threadIdx.x == 0) v.attn_count[bg] = 0;
}

template <typename T, int D, int M, int LMAX>
void launch_tma(const EngineView& v, int layer, dim3 grid, cudaStream_t stream) {
    const size_t tiles = (size_t)kStages * 2 * kTileRows * D * sizeof(T);
    const size_t red = (size_t)kWarps * M * (D + 2) * sizeof(float);
    const size_t sm = tiles > red ? tiles : red;
    cudaFuncSetAttribute(attn_tma_kernel<T, D, M, LMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attn_tma_kernel<T, D, M, LMAX><<<grid, kThreads, sm, stream>>>(v, layer);
}

// QK lanes per row: 8 (fewer shuffles, more q registers) or 16 (fewer
// registers); CLO_ATTN_LANES overrides the default for experiments.
int qk_lanes() {
    static int lanes = [] {
        const char* e = getenv("CLO_ATTN_LANES");
        return e && atoi(e) == 16 ? 16 : 8;
    }();
    return lanes;
}

template <typename T, int D>
bool launch_tma_m(const EngineView& v, int layer, dim3 grid, cudaStream_t stream) {
    const bool wide = qk_lanes() == 16;
    switch (v.m) {
#define CLO_TM(MM)                                                         \
    case MM:                                                               \
        if (wide)                                                          \
            launch_tma<T, D, MM, 16>(v, layer, grid, stream);              \
        else                                                               \
            launch_tma<T, D, MM, 8>(v, layer, grid, stream);               \
        return true;
        CLO_TM(1) CLO_TM(2) CLO_TM(3) CLO_TM(4) CLO_TM(5) CLO_TM(6) CLO_TM(7) CLO_TM(8)
#undef CLO_TM
        default:
            return false;
    }
}

}  // namespace

bool attention_tma_supported(int dtype, int d, int m, int k) {
    if (m < 1 || m > 8) return false;
    if (k % 4 != 0) return false;  // token bulk copies need 16-byte aligned rows of k ints
    if (dtype == kBF16) return d == 64 || d == 128 || d == 256;
    if (dtype == kF32) return d == 64 || d == 128;
    return false;
}

bool launch_attention_tma(const EngineView& v, int layer, cudaStream_t stream) {
    if (!attention_tma_supported(v.kv_dtype, v.d, v.m, v.k)) return false;
    dim3 grid(attention_chunks(v.k, v.sink, v.recent), v.B * v.H);
    if (v.kv_dtype == kBF16) {
        switch (v.d) {
            case 64: return launch_tma_m<__nv_bfloat16, 64>(v, layer, grid, stream);
            case 128: return launch_tma_m<__nv_bfloat16, 128>(v, layer, grid, stream);
            case 256: return launch_tma_m<__nv_bfloat16, 256>(v, layer, grid, stream);
        }
    } else {
        switch (v.d) {
            case 64: return launch_tma_m<float, 64>(v, layer, grid, stream);
            case 128: return launch_tma_m<float, 128>(v, layer, grid, stream);
        }
    }
    return false;
}

}  // namespace clo
