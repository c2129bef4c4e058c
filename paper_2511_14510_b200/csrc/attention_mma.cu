// attention_mma.cu — K4 sparse attention on the tensor cores (production path
// for bf16 rows with d in {64, 128}).
//
// Semantics: topk_attention / attend_rows (attention.cpp:33-55, 91-105) of the
// m GQA query heads of one KV head over union(selection, sink/recent window)
// (union_indices engine.cpp:80-85, sink_recent_indices attention.cpp:107-128).
//
// Why mma.sync and not tcgen05: the op is GEMV-shaped (m <= 8 query rows per
// KV row) and HBM-bound. The FFMA kernel (attention_tma.cu) spends ~83 issue
// slots per KV row and stalls on shuffle chains; here a warp-level
// m16n8k16 MMA does a 16-row x 8-key (or x 8-dim) tile in one instruction, so
// a KV row costs ~5 issue slots and the kernel is left waiting on HBM only.
// tcgen05's smallest tile (M = 64) would compute 8x more padding and route
// every partial through TMEM for no bandwidth gain.
//
// Exactness: K and V are bf16 (exact MMA operands). The fp32 query and the
// fp32 softmax weights are split hi + lo (two bf16 terms, residual < 2^-16
// relative), both terms go through the MMA in the SAME instruction — rows
// 0..7 of the A tile carry the hi parts of the m queries, rows 8..15 the lo
// parts — and the fp32 accumulators of a query's two rows are added. Result:
// fp32-class accuracy (~1e-5 relative) from bf16 tensor cores.
//
// Structure (persistent: 2 CTAs per SM, 4 independent warps each; see the
// work decomposition below):
//   * each warp streams its tiles into a private 3-stage shared-memory ring
//     with 16-byte cp.async (all lanes) into rows padded to 272 B, so
//     ldmatrix is bank-conflict free;
//   * QK: ldmatrix K (8 keys x 32 dims per x4) + m16n8k16, 2 key tiles x d/16;
//   * online softmax on the accumulators: a query's 4 lanes hold its 16 scores,
//     max over 2 shuffles, lazy rescaling (only when the max grows by > 2^8);
//   * PV: the probability accumulators ARE the A fragment of the next MMA
//     (split hi/lo on the fly), ldmatrix.trans V, m16n8k16 over d/8 dim tiles;
//   * per-warp partials merge in a small combine kernel (flash decoding).
// Each KV row is read from HBM exactly once for all m query heads.
#include <cooperative_groups.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "attention.cuh"
#include "exchange.cuh"

namespace clo {

namespace {

constexpr int kTileMin = 16;  // smallest tile (rows); tiles are TM = 16 or 32 rows
constexpr float kLazy = 8.0f; // rescale when the running max grows by more than 2^8

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D, fp32 accumulators
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
    return r;
}
// x = hi + lo with hi = bf16(x), lo = bf16(x - hi): packed pairs of both
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    hi = pack_bf16(x0, x1);
    const float h0 = __uint_as_float(hi << 16), h1 = __uint_as_float(hi & 0xFFFF0000u);
    lo = pack_bf16(x0 - h0, x1 - h1);
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float wexp(float m, float gm) { return m == -CUDART_INF_F ? 0.f : exp2f(m - gm); }

// Work decomposition (one layer): the attend positions of every head are cut
// into 16-row tiles; the B*H heads' tiles form one flat sequence of
// T = B*H*N tiles (N = tiles per head), split into G equal contiguous
// segments, one per CTA (G = 2 CTAs per SM, one wave). Warp w of CTA j streams
// tiles S_j + w, S_j + w + 4, ... across head boundaries without draining its
// ring; whenever its head changes it flushes a partial (m, l, O) for the head
// it leaves. Every warp's partial lives at slot ((j*4 + w)*R + r), r = the
// run's head minus the head of the segment's first tile. A second kernel
// merges each head's partials (flash-decoding combine) and emits the outputs.
constexpr int kMaxCtas = 2 * kNumSMs;

struct MmaPlan {
    int N;       // tiles per head
    long long T; // total tiles
    int G;       // CTAs
    int R;       // partial runs per warp
    int W;       // warps per CTA (each warp flushes its own partials)
    int single;  // G = c * B*H: CTA j serves piece j % c of head j / c (warps merge in shared memory)
    int c;       // CTAs per head when single
    int cluster; // single, c > 1: a head's c CTAs are one thread-block cluster and merge over DSMEM
    int seg[kMaxCtas + 1];  // segment starts S_j = j*T/G (T < 2^31)
};

__host__ __device__ __forceinline__ long long seg_start(const MmaPlan& pl, int j) { return pl.seg[j]; }

// Partial rows are D + 4 floats (O[D], m, l, pad): 16-byte aligned for float4.
//
// Flash-decoding merge of one head's partials by one warp. The warps whose
// tiles met head h are enumerated by the arithmetic that assigned them (CTAs
// whose segment meets [hN, (h+1)N), each of their W warps whose tile sequence
// S_j + w + W*i enters it); visiting them by (CTA, warp) visits their slots
// (= first tile in the head) in ascending order, so the merge is
// deterministic. Lane i owns contributor i: one round of (m, l) loads,
// shuffles for the maxima and denominators, then every lane sums its D/32
// output dims per query over the contributors.
template <int D, int M>
__device__ __noinline__ void combine_head(const EngineView& v, int l, int t, int h, const float* ph,
                                          const MmaPlan& pl, int lane) {
    const int hb = h / v.H, g = h - hb * v.H;
    const int h0 = h * pl.N, h1 = h0 + pl.N;
    int j0 = (int)((long long)h0 * pl.G / pl.T);
    while (j0 > 0 && pl.seg[j0] > h0) --j0;
    while (pl.seg[j0 + 1] <= h0) ++j0;
    int j1 = j0;  // last CTA meeting the head
    while (j1 + 1 < pl.G && pl.seg[j1 + 1] < h1) ++j1;
    const int ncand = (j1 - j0 + 1) * pl.W;
    // Lane c holds contributor c's slot, (m, l) and weights; the outputs are
    // accumulated with lane L owning float4 L % (D/4) of query rows
    // L / (D/4), L / (D/4) + QS, ...: each batch of contributors issues all
    // its partial loads before any use (one L2 round trip per batch).
    constexpr int V4 = D / 4;                 // float4 per partial row
    constexpr int QS = 32 / V4;               // query rows covered per pass
    constexpr int QP = (M + QS - 1) / QS;     // query rows per lane
    constexpr int BATCH = M <= 4 ? 4 : 2;     // contributors per load batch
    const int f4 = lane % V4, q0l = lane / V4;
    float gm[M], den[M];
    float4 acc[QP];
#pragma unroll
    for (int q = 0; q < M; ++q) {
        gm[q] = -CUDART_INF_F;
        den[q] = 0.f;
    }
#pragma unroll
    for (int qq = 0; qq < QP; ++qq) acc[qq] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = 0; c0 < ncand; c0 += 32) {
        const int c = c0 + lane;
        int slot = -1;
        if (c < ncand) {
            const int j = j0 + c / pl.W, w = c % pl.W;
            const int S0 = pl.seg[j], S1 = pl.seg[j + 1];
            const int lo = max(S0, h0), hi = min(S1, h1);
            int first = S0 + w;
            if (first < lo) first += (lo - first + pl.W - 1) / pl.W * pl.W;
            if (first < hi) slot = first - h0;
        }
        float m[M], lw[M];
#pragma unroll
        for (int q = 0; q < M; ++q) {
            m[q] = -CUDART_INF_F;
            lw[q] = 0.f;
            if (slot >= 0) {
                const float2 ml = __ldcg(reinterpret_cast<const float2*>(ph + ((size_t)slot * M + q) * (D + 4) + D));
                m[q] = ml.x;
                lw[q] = ml.y;
            }
        }
        float w[M];
#pragma unroll
        for (int q = 0; q < M; ++q) {  // rescale the running merge to the new maximum
            float cm = m[q];
#pragma unroll
            for (int o2 = 16; o2; o2 >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o2));
            const float ngm = fmaxf(gm[q], cm);
            const float corr = gm[q] == -CUDART_INF_F ? 0.f : exp2f(gm[q] - ngm);
            gm[q] = ngm;
            den[q] *= corr;
#pragma unroll
            for (int qq = 0; qq < QP; ++qq)
                if (q0l + qq * QS == q) {
                    acc[qq].x *= corr;
                    acc[qq].y *= corr;
                    acc[qq].z *= corr;
                    acc[qq].w *= corr;
                }
            w[q] = m[q] == -CUDART_INF_F ? 0.f : exp2f(m[q] - ngm);
            den[q] += w[q] * lw[q];
        }
        // compact the present contributors (slot order), then batch their loads
        const unsigned present = __ballot_sync(0xffffffffu, slot >= 0);
        const int np = __popc(present);
        const int rank = __popc(present & ((1u << lane) - 1));
        int src_of = 0;  // lane r: the lane holding the r-th present contributor
        for (int r = 0, mm = present; mm; ++r, mm &= mm - 1)
            if (lane == r) src_of = __ffs(mm) - 1;
        (void)rank;
        for (int r0 = 0; r0 < np; r0 += BATCH) {
            float4 x[BATCH][QP];
            float wb[BATCH][QP];
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int src = __shfl_sync(0xffffffffu, src_of, min(r0 + u, 31));
                const int sl = __shfl_sync(0xffffffffu, slot, src);
#pragma unroll
                for (int qq = 0; qq < QP; ++qq) {
                    const int q = q0l + qq * QS;
                    float wq = 0.f;
#pragma unroll
                    for (int z = 0; z < M; ++z) {
                        const float wz = __shfl_sync(0xffffffffu, w[z], src);
                        if (z == q) wq = wz;
                    }
                    const bool live = r0 + u < np && q < M;
                    wb[u][qq] = live ? wq : 0.f;
                    x[u][qq] = live ? __ldcg(reinterpret_cast<const float4*>(ph + ((size_t)sl * M + q) * (D + 4)) + f4)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
#pragma unroll
                for (int qq = 0; qq < QP; ++qq) {
                    acc[qq].x += wb[u][qq] * x[u][qq].x;
                    acc[qq].y += wb[u][qq] * x[u][qq].y;
                    acc[qq].z += wb[u][qq] * x[u][qq].z;
                    acc[qq].w += wb[u][qq] * x[u][qq].w;
                }
        }
    }
#pragma unroll
    for (int q = 0; q < M; ++q)
#pragma unroll
        for (int o2 = 16; o2; o2 >>= 1) den[q] += __shfl_xor_sync(0xffffffffu, den[q], o2);
#pragma unroll
    for (int qq = 0; qq < QP; ++qq) {
        const int q = q0l + qq * QS;
        if (q < M) {
            float dq = 0.f;
#pragma unroll
            for (int z = 0; z < M; ++z)
                if (z == q) dq = den[z];
            emit_head_output(v, t, hb, l, g * M + q, 4 * f4 + 0, acc[qq].x / dq);
            emit_head_output(v, t, hb, l, g * M + q, 4 * f4 + 1, acc[qq].y / dq);
            emit_head_output(v, t, hb, l, g * M + q, 4 * f4 + 2, acc[qq].z / dq);
            emit_head_output(v, t, hb, l, g * M + q, 4 * f4 + 3, acc[qq].w / dq);
        }
    }
    signal_head_output_warp(v, l);
}

template <int D, int M, int kWarpsM, int kStagesM, int kCtasPerSM, int kTileM, int kRegCap>
// kRegCap: see launch_mma_shape.
__global__ void __maxnreg__(kRegCap) attn_mma_stream_kernel(const __grid_constant__ EngineView v, int l, const __grid_constant__ MmaPlan pl,
                                                                       float* part) {
    using T = __nv_bfloat16;
    constexpr uint32_t kRowBytes = D * 2;
    constexpr uint32_t kMatBytes = kTileM * kRowBytes;    // one matrix tile, 128B-swizzled
    constexpr uint32_t kStageBytes = 2 * kMatBytes;       // K tile then V tile
    constexpr int KS = D / 16;                            // k-steps of QK
    constexpr int NT = D / 8;                             // dim tiles of PV
    constexpr int CPR = kRowBytes / 16;                   // 16-byte chunks per row
    constexpr int RPR = 32 / CPR;                         // rows per warp-wide copy round
    static_assert(M >= 1 && M <= 8, "m <= 8");

    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(16) int32_t toks[kWarpsM][kStagesM][kTileM];
    __shared__ __align__(8) uint64_t full[kWarpsM][kStagesM];
    // Stage layout = the TMA 128-byte swizzle: a matrix tile is D/64 column
    // halves of [kTileM rows][128 B]; 16-byte chunk cc of row r of a half sits
    // at r*128 + ((cc ^ (r & 7)) * 16). ldmatrix over 8 rows then hits 8
    // distinct bank groups, and contiguous slot tiles arrive as one 2D TMA box
    // per half.
    auto swz = [](int r, int c) -> uint32_t {  // row r, 16-byte chunk c of a matrix tile
        return (uint32_t)((c >> 3) * (kTileM * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
    };

    const int j = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int qg = lane >> 2, qc = lane & 3;  // MMA fragment row group / column pair
    const long long S0 = seg_start(pl, j), S1 = seg_start(pl, j + 1);
    const int mine = S1 - S0 > warp ? (int)((S1 - S0 - 1 - warp) / kWarpsM) + 1 : 0;
    const int head0 = (int)(S0 / pl.N);

    const int t = *v.dev_step + 1;
    const int n_after = v.n_prompt + t;
    const int s1 = min(v.sink, n_after), r1 = min(v.recent, n_after);
    const int wstart = max(n_after - r1, s1);
    const int P = v.k + s1 + (n_after - wstart);
    const int wrows = v.sink + v.recent;

    unsigned char* ring = smem + (size_t)warp * kStagesM * kStageBytes;

    // this warp's i-th tile -> stage i % S with 16-byte cp.async (LDGSTS):
    // each lane copies chunk `ch` of rows r0, r0 + RPR, ... of K and of V. One
    // commit group per tile (empty past the warp's last tile) keeps the
    // wait_group arithmetic uniform. (Per-row cp.async.bulk would serialise:
    // a bulk copy takes uniform operands, so 32 lanes' copies become a loop.)
    // issue cursor: head ih, tile iq of the next tile this warp copies (the
    // tile index advances by kWarpsM; no divisions in the loop)
    int ih = (int)((S0 + warp) / pl.N), iq = (int)((S0 + warp) % pl.N);
    int info_h = -1, b = 0, lg = 0, seg = 0;
    bool pers = false;
    size_t oslot = 0;
    auto issue = [&](int i) {
        if (i < mine) {
            if (ih != info_h) {  // per-head addressing, once per head
                info_h = ih;
                b = ih / v.H;
                const int g = ih - b * v.H;
                lg = l * v.H + g;
                seg = (b * v.L + l) * v.H + g;
                pers = v.persistent[lg] != 0;
                oslot = pers ? 0 : (size_t)b * v.NO + v.oidx[lg];
            }
            const int tp = iq * kTileM;
            iq += kWarpsM;
            while (iq >= pl.N) {
                iq -= pl.N;
                ++ih;
            }
            const int rows = min(kTileM, P - tp);
            const int sel_rows = max(0, min(rows, v.k - tp));
            const int s = i % kStagesM;
            const uint32_t st = smem_u32(ring + (size_t)s * kStageBytes);
            const int32_t* idx = v.entry_idx + (size_t)seg * v.k;
            if (lane < sel_rows)
                cp_async4(smem_u32(&toks[warp][s][lane]), (pers ? idx : v.slot_tok + oslot * v.pool) + tp + lane);
            const int ch = lane % CPR, r0 = lane / CPR;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our ldmatrix reads of the stage
            __syncwarp();
            if (!pers && tp + kTileM <= v.k && v.tmap_k) {
                // a run of contiguous cache slots: one 2D TMA box per matrix half
                if (lane == 0) {
                    uint64_t* bar = &full[warp][s];
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                                 "r"(kStageBytes)
                                 : "memory");
                    const int row0 = (int)(oslot * v.pool + tp);
#pragma unroll
                    for (int m2 = 0; m2 < 2; ++m2)
#pragma unroll
                        for (int hh = 0; hh < D / 64; ++hh)
                            asm volatile(
                                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                                " [%0], [%1, {%2, %3}], [%4];" ::"r"(st + m2 * kMatBytes + hh * kTileM * 128),
                                "l"(m2 ? v.tmap_v : v.tmap_k), "r"(hh * 64), "r"(row0), "r"(smem_u32(bar))
                                : "memory");
                }
            } else {
                const size_t pslot = pers ? (size_t)b * v.NP + v.pidx[lg] : 0;
                const T* pk = static_cast<const T*>(v.pk) + pslot * v.nmax * D;
                const T* pv = static_cast<const T*>(v.pv) + pslot * v.nmax * D;
                const T* sk = static_cast<const T*>(v.slot_k) + oslot * v.pool * D;
                const T* sv = static_cast<const T*>(v.slot_v) + oslot * v.pool * D;
                const T* wk = static_cast<const T*>(v.win_k) + oslot * wrows * D;
                const T* wv = static_cast<const T*>(v.win_v) + oslot * wrows * D;
#pragma unroll 1
                for (int rr = r0; rr < rows; rr += RPR) {
                    const int pos = tp + rr;
                    const T *kr, *vr;
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
                    cp_async16(st + swz(rr, ch), kr + ch * 8);
                    cp_async16(st + kMatBytes + swz(rr, ch), vr + ch * 8);
                }
                if (lane == 0)  // data readiness of LDGSTS stages: the commit group below
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[warp][s])) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    // zero this warp's ring once: rows past a partial tile's end then hold
    // finite stale values (weight 0), never uninitialised NaN patterns
    for (uint32_t i = lane; i < kStagesM * kStageBytes / 16; i += 32)
        reinterpret_cast<uint4*>(ring)[i] = make_uint4(0, 0, 0, 0);
    if (lane == 0)
        for (int s2 = 0; s2 < kStagesM; ++s2)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[warp][s2])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    for (int i = 0; i < kStagesM - 1; ++i) issue(i);

    // the queries of every head this CTA touches, staged once in shared memory
    // (a head switch then costs no global round trip)
    float* qs = reinterpret_cast<float*>(smem + (size_t)kWarpsM * kStagesM * kStageBytes);
    {
        const int nh = S1 > S0 ? (int)((S1 - 1) / pl.N) - head0 + 1 : 0;
        bool bad = false;
        for (int i = threadIdx.x; i < nh * M * D / 4; i += kWarpsM * 32) {
            const int hh = i / (M * D / 4), r = i - hh * (M * D / 4);
            const int h = head0 + hh, hb = h / v.H, g = h - hb * v.H;
            const float4 x = reinterpret_cast<const float4*>(
                v.desc->true_q + (((size_t)hb * v.L + l) * v.HQ + (size_t)g * M) * D)[r];
            bad |= !isfinite(x.x) || !isfinite(x.y) || !isfinite(x.z) || !isfinite(x.w);
            reinterpret_cast<float4*>(qs)[i] = x;
        }
        if (bad) raise_err(v.err, kErrNonFiniteQuery);
        __syncthreads();
    }
    const float qscale = 1.4426950408889634f * rsqrtf((float)D);  // log2(e)/sqrt(d): softmax on exp2
    uint32_t qa[KS][4];  // A rows qg = hi, qg+8 = lo of query qg
    auto load_q = [&](int h) {
        const float* qsrc = qs + (size_t)(h - head0) * M * D;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                float2 x = make_float2(0.f, 0.f);
                if (qg < M) x = *reinterpret_cast<const float2*>(qsrc + (size_t)qg * D + ks * 16 + hh * 8 + 2 * qc);
                split2(x.x * qscale, x.y * qscale, qa[ks][2 * hh], qa[ks][2 * hh + 1]);
            }
        }
    };

    float m_run = -CUDART_INF_F, l_run = 0.f;  // query qg (replicated over its 4 lanes)
    float o[NT][4];                            // rows qg (hi) / qg+8 (lo), dims 8nt + 2qc + {0,1}
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    int cur = -1;  // head of the open run

    // Partial of the run on head `cur` -> slot `run_first` (the run's first
    // tile within the head: unique per run, so the merge order below is
    // deterministic). The warp that brings
    // the head's tile count to N merges the head's partials in slot
    // order (flash-decoding combine) and emits the outputs: no second kernel.
    int run_tiles = 0, run_first = 0;
    int* tiles_done = v.attn_count;  // [B*H], self-resetting
    float* const part_base = part;
    auto flush = [&]() {
        float lsum = l_run + __shfl_xor_sync(0xffffffffu, l_run, 1);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
        float* ph = part_base + (size_t)cur * pl.N * M * (D + 4);
        if (qg < M) {
            float* pw = ph + ((size_t)run_first * M + qg) * (D + 4);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
                __stcg(reinterpret_cast<float2*>(pw + nt * 8 + 2 * qc),
                       make_float2(o[nt][0] + o[nt][2], o[nt][1] + o[nt][3]));
            if (qc == 0) __stcg(reinterpret_cast<float2*>(pw + D), make_float2(m_run, lsum));
        }
        m_run = -CUDART_INF_F;
        l_run = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
        __threadfence();
        __syncwarp();
        int last = 0;
        if (lane == 0) last = atomicAdd(&tiles_done[cur], run_tiles) + run_tiles == pl.N;
        if (!__shfl_sync(0xffffffffu, last, 0)) return;
        // ---- this warp completes head `cur`: merge its partials -----------
        __threadfence();
        if (lane == 0) tiles_done[cur] = 0;
        combine_head<D, M>(v, l, t, cur, ph, pl, lane);
    };

    int chd = (int)((S0 + warp) / pl.N), cq = (int)((S0 + warp) % pl.N);  // consume cursor
    for (int i = 0; i < mine; ++i) {
        issue(i + kStagesM - 1);
        const int h = chd, tp = cq * kTileM;
        cq += kWarpsM;
        while (cq >= pl.N) {
            cq -= pl.N;
            ++chd;
        }
        if (h != cur) {
            if (cur >= 0) flush();  // never in single mode: a CTA's tiles are one head
            load_q(h);
            cur = h;
            run_tiles = 0;
            run_first = tp / kTileM;
        }
        ++run_tiles;
        const int rows = min(kTileM, P - tp);
        const int s = i % kStagesM;
        asm volatile("cp.async.wait_group %0;" ::"n"(kStagesM - 1) : "memory");  // LDGSTS part of tile i
        asm volatile(
            "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(&full[warp][s])),
            "r"((i / kStagesM) & 1)
            : "memory");  // TMA part of tile i
        __syncwarp();
        const uint32_t kbase = smem_u32(ring + (size_t)s * kStageBytes);
        const uint32_t vbase = kbase + kMatBytes;

        // ---- S = Q K^T for TM keys: NK key tiles of 8, two independent
        // accumulator chains per key tile (even / odd k-steps) ---------------
        constexpr int NK = kTileM / 8;
        float sacc[NK][2][4];
#pragma unroll
        for (int nt = 0; nt < NK; ++nt) {
#pragma unroll
            for (int z = 0; z < 2; ++z) sacc[nt][z][0] = sacc[nt][z][1] = sacc[nt][z][2] = sacc[nt][z][3] = 0.f;
#pragma unroll
            for (int kp = 0; kp < KS / 2; ++kp) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kbase + swz(nt * 8 + (lane & 7), kp * 4 + (lane >> 3)), b0, b1, b2, b3);
                mma16816(sacc[nt][0], qa[2 * kp], b0, b1);
                mma16816(sacc[nt][1], qa[2 * kp + 1], b2, b3);
            }
        }
        // scores of keys 8nt + 2qc + e for query qg: hi row + lo row, both chains
        float sc[NK][2];
        float mt = -CUDART_INF_F;
#pragma unroll
        for (int nt = 0; nt < NK; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = nt * 8 + 2 * qc + e;
                bool ok = r < rows;
                if (ok && tp + r < v.k) {  // dedup selected tokens against the window
                    const int tok = toks[warp][s][r];
                    ok = !(tok < s1 || tok >= wstart);
                }
                const float x = (sacc[nt][0][e] + sacc[nt][0][2 + e]) + (sacc[nt][1][e] + sacc[nt][1][2 + e]);
                sc[nt][e] = ok ? x : -CUDART_INF_F;
                mt = fmaxf(mt, sc[nt][e]);
            }
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
        if (mt > m_run + kLazy) {  // lazy rescale (uniform over the query's 4 lanes)
            const float corr = m_run == -CUDART_INF_F ? 0.f : fast_exp2(m_run - mt);
            m_run = mt;
            l_run *= corr;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                o[nt][0] *= corr;
                o[nt][1] *= corr;
                o[nt][2] *= corr;
                o[nt][3] *= corr;
            }
        }
        // ---- O += P V per 16-key step: P = exp2(S - m) is the A fragment
        // (keys 2qc+{0,1} and 8+2qc+{0,1} of the step, rows qg = hi, qg+8 = lo);
        // ldmatrix.trans V (16 keys x 16 dims per x4) -------------------------
#pragma unroll
        for (int kt = 0; kt < kTileM / 16; ++kt) {
            uint32_t pa[4];
            float p[2][2];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float x = sc[2 * kt + nt][e];
                    p[nt][e] = x == -CUDART_INF_F ? 0.f : fast_exp2(x - m_run);
                    l_run += p[nt][e];
                }
            split2(p[0][0], p[0][1], pa[0], pa[1]);
            split2(p[1][0], p[1][1], pa[2], pa[3]);
#pragma unroll
            for (int nd = 0; nd < NT / 2; ++nd) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vbase + swz(kt * 16 + (lane >> 3 & 1) * 8 + (lane & 7), nd * 2 + (lane >> 4)), b0, b1, b2,
                          b3);
                mma16816(o[2 * nd], pa, b0, b1);
                mma16816(o[2 * nd + 1], pa, b2, b3);
            }
        }
        __syncwarp();  // stage s is free for the issue S-1 tiles on
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (!pl.single) {
        if (cur >= 0) flush();
        return;
    }
    // Head-aligned segments: the warps' (m, l, O) merge through shared memory
    // by the whole CTA (fixed warp order: deterministic). With c > 1 CTAs per
    // head, each CTA then writes one partial (m, l, unnormalised O) and the
    // last of the head's c CTAs merges them in piece order.
    __syncthreads();  // every warp is done with its ring
    float* red = reinterpret_cast<float*>(smem);  // [kWarpsM][M][D + 2]
    float* cpart = red + (size_t)kWarpsM * M * (D + 2);  // [M][D + 4] this CTA's partial (cluster merge)
    {
        float lsum = l_run + __shfl_xor_sync(0xffffffffu, l_run, 1);
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
        if (qg < M) {
            float* rw = red + ((size_t)warp * M + qg) * (D + 2);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                rw[nt * 8 + 2 * qc] = o[nt][0] + o[nt][2];
                rw[nt * 8 + 2 * qc + 1] = o[nt][1] + o[nt][3];
            }
            if (qc == 0) {
                rw[D] = m_run;
                rw[D + 1] = lsum;
            }
        }
    }
    __syncthreads();
    const int h = j / pl.c, piece = j - h * pl.c, hb = h / v.H, g = h - hb * v.H;
    float* ph = part + (size_t)h * pl.c * M * (D + 4);  // [c][M][D + 4] partials of head h
    for (int x = threadIdx.x; x < M * D; x += kWarpsM * 32) {
        const int q = x / D, e = x - q * D;
        float gm = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < kWarpsM; ++w) gm = fmaxf(gm, red[((size_t)w * M + q) * (D + 2) + D]);
        float a = 0.f, den = 0.f;
#pragma unroll
        for (int w = 0; w < kWarpsM; ++w) {
            const float cw = wexp(red[((size_t)w * M + q) * (D + 2) + D], gm);
            a += red[((size_t)w * M + q) * (D + 2) + e] * cw;
            den += red[((size_t)w * M + q) * (D + 2) + D + 1] * cw;
        }
        if (pl.c == 1) {
            emit_head_output(v, t, hb, l, g * M + q, e, a / den);
        } else if (pl.cluster) {  // this CTA's partial stays in its shared memory
            float* pp = cpart + (size_t)q * (D + 4);
            pp[e] = a;
            if (e == 0) {
                pp[D] = gm;
                pp[D + 1] = den;
            }
        } else {
            float* pp = ph + ((size_t)piece * M + q) * (D + 4);
            __stcg(pp + e, a);
            if (e == 0) {
                __stcg(pp + D, gm);
                __stcg(pp + D + 1, den);
            }
        }
    }
    if (pl.c > 1 && pl.cluster) {
        // The head's c CTAs form one cluster (rank = piece): rank 0 merges
        // the c partials in piece order over DSMEM (the same arithmetic and
        // order as the global-memory merge below), without a global fence —
        // a gpu-scope fence waits for every host read the concurrent gather
        // has queued (profiles/r2/pdl_exit_probe.txt), a cluster barrier does not.
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
        if (piece == 0) {
            for (int x = threadIdx.x; x < M * D; x += kWarpsM * 32) {
                const int q = x / D, e = x - q * D;
                float gm = -CUDART_INF_F;
                for (int cc = 0; cc < pl.c; ++cc) gm = fmaxf(gm, cl.map_shared_rank(cpart, cc)[(size_t)q * (D + 4) + D]);
                float a = 0.f, den = 0.f;
                for (int cc = 0; cc < pl.c; ++cc) {
                    const float* pp = cl.map_shared_rank(cpart, cc) + (size_t)q * (D + 4);
                    const float cw = wexp(pp[D], gm);
                    a += pp[e] * cw;
                    den += pp[D + 1] * cw;
                }
                emit_head_output(v, t, hb, l, g * M + q, e, a / den);
            }
        }
        cl.sync();  // the other CTAs' shared memory stays live until rank 0 has read it
    } else if (pl.c > 1) {
        __shared__ int s_last_cta;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last_cta = atomicAdd(&v.attn_count[h], 1) == pl.c - 1;
        __syncthreads();
        if (!s_last_cta) return;
        __threadfence();
        for (int x = threadIdx.x; x < M * D; x += kWarpsM * 32) {
            const int q = x / D, e = x - q * D;
            float gm = -CUDART_INF_F;
            for (int cc = 0; cc < pl.c; ++cc) gm = fmaxf(gm, __ldcg(ph + ((size_t)cc * M + q) * (D + 4) + D));
            float a = 0.f, den = 0.f;
            for (int cc = 0; cc < pl.c; ++cc) {
                const float* pp = ph + ((size_t)cc * M + q) * (D + 4);
                const float cw = wexp(__ldcg(pp + D), gm);
                a += __ldcg(pp + e) * cw;
                den += __ldcg(pp + D + 1) * cw;
            }
            emit_head_output(v, t, hb, l, g * M + q, e, a / den);
        }
        if (threadIdx.x == 0) v.attn_count[h] = 0;
    }
    signal_head_output(v, l);
}

bool attn_cluster_enabled() {  // CLO_ATTN_CLUSTER=0: c > 1 CTAs per head merge through global memory
    static const bool on = [] {
        const char* e = getenv("CLO_ATTN_CLUSTER");
        return !(e && e[0] == '0');
    }();
    return on;
}

MmaPlan make_plan(const EngineView& v, int W, int ctas_per_sm, int TM) {
    MmaPlan pl{};
    pl.W = W;
    const int Pmax = v.k + v.sink + v.recent;  // the attend count of a step is <= this and N is fixed
    pl.N = (Pmax + TM - 1) / TM;
    pl.T = (long long)v.B * v.H * pl.N;
    // One wave of CTAs. When the heads fit, G is a multiple of B*H so every
    // segment lies inside one head (c CTAs per head, no segment straddles a
    // head boundary); otherwise the flat split.
    const long long want = (long long)ctas_per_sm * kNumSMs;
    const long long BH = (long long)v.B * v.H;
    static const bool align = [] {
        const char* e = getenv("CLO_ATTN_ALIGN");
        return !(e && e[0] == '0');
    }();
    long long G = align && BH <= want ? BH * (want / BH) : want;
    const long long most = (pl.T + W - 1) / W;  // at least a tile per warp
    if (G > most) G = most;
    pl.G = (int)G;
    pl.single = G % BH == 0;
    pl.c = pl.single ? (int)(G / BH) : 0;
    for (int j = 0; j <= pl.G; ++j) pl.seg[j] = (int)((long long)j * pl.T / pl.G);
    const long long seg = (pl.T + pl.G - 1) / pl.G;
    pl.R = (int)((seg + pl.N - 1) / pl.N) + 1;
    return pl;
}

// Streaming shapes (warps per CTA x ring stages per warp x CTAs per SM): all
// fill ~210 KB of shared memory per SM with 16-row stages; deeper rings keep
// more bytes in flight per SM, more warps issue more in parallel.
struct MmaShape {
    int warps, stages, ctas, tile;
};
// Default: 8 warps x 3 stages, one CTA per SM (measured best, profiles/
// r1_attention_mma.md) while the heads fit one CTA each (B*H <= 148); with
// 148 < B*H <= 296 two 4-warp CTAs per SM keep one head per CTA (shared-
// memory merge, one wave) instead of the flat split.
MmaShape mma_shape(int heads) {
    static const int forced = [] {
        const char* e = getenv("CLO_ATTN_SHAPE");  // warps x stages x CTAs/SM x tile rows
        const std::string x = e ? e : "";
        if (x == "4x3x2x16") return 1;
        if (x == "4x3x1x32") return 2;
        if (x == "4x6x1x16") return 3;
        if (x == "8x3x1x16") return 4;
        return 0;
    }();
    switch (forced) {
        case 1: return MmaShape{4, 3, 2, 16};
        case 2: return MmaShape{4, 3, 1, 32};
        case 3: return MmaShape{4, 6, 1, 16};
        case 4: return MmaShape{8, 3, 1, 16};
        default: break;
    }
    if (heads > kNumSMs && heads <= 2 * kNumSMs) return MmaShape{4, 3, 2, 16};
    return MmaShape{8, 3, 1, 16};
}

template <int D, int M, int W, int S, int C, int TM, int RC>
void launch_mma_shape_rc(const EngineView& v, int layer, cudaStream_t stream) {
    const MmaPlan pl = make_plan(v, W, C, TM);
    const size_t ring = (size_t)W * S * 2 * TM * D * 2;
    const size_t sm = ring + (size_t)pl.R * M * D * sizeof(float);  // + staged queries
    // per device (a process may drive several GPUs); launches happen at graph
    // capture, so the host call is not on the replay path
    cudaFuncSetAttribute(attn_mma_stream_kernel<D, M, W, S, C, TM, RC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    EngineView vv = v;
    if (TM == 32) {  // the tensor maps whose boxes match the tile
        vv.tmap_k = v.tmap_k32;
        vv.tmap_v = v.tmap_v32;
    }
    auto kern = attn_mma_stream_kernel<D, M, W, S, C, TM, RC>;
    if (pl.single && pl.c > 1 && pl.c <= 16 && attn_cluster_enabled()) {
        // one cluster per head (DSMEM merge) when every cluster fits at once
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(pl.G);
        cfg.blockDim = dim3(W * 32);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = pl.c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (pl.c > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters * pl.c >= pl.G) {
            MmaPlan pc = pl;
            pc.cluster = 1;
            if (cudaLaunchKernelEx(&cfg, kern, vv, layer, pc, v.attn_part) == cudaSuccess) return;
        }
        cudaGetLastError();  // not co-schedulable here: the global-memory merge
    }
    kern<<<pl.G, W * 32, sm, stream>>>(vv, layer, pl, v.attn_part);
}

// Register cap: CLO_ATTN_REGCAP=184 lets an 8-warp CTA share its SM with a
// zero-copy gather CTA. Measured on B200 that slows the step by ~12%: the
// gather's PCIe reads need their warps issued promptly, and a co-resident
// attention CTA delays them (profiles/r1_attention_mma.md). Default: no cap.
template <int D, int M, int W, int S, int C, int TM>
void launch_mma_shape(const EngineView& v, int layer, cudaStream_t stream) {
    static const bool capped = [] {
        const char* e = getenv("CLO_ATTN_REGCAP");
        return e && atoi(e) > 0 && atoi(e) < 255;
    }();
    if (capped)
        launch_mma_shape_rc<D, M, W, S, C, TM, 184>(v, layer, stream);
    else
        launch_mma_shape_rc<D, M, W, S, C, TM, 255>(v, layer, stream);
}

template <int D, int M>
void launch_mma(const EngineView& v, int layer, cudaStream_t stream) {
    const MmaShape sh = mma_shape(v.B * v.H);
    if (sh.tile == 32) {
        launch_mma_shape<D, M, 4, 3, 1, 32>(v, layer, stream);
    } else if (sh.warps == 8) {
        launch_mma_shape<D, M, 8, 3, 1, 16>(v, layer, stream);
    } else if (sh.ctas == 2) {
        launch_mma_shape<D, M, 4, 3, 2, 16>(v, layer, stream);
    } else {
        launch_mma_shape<D, M, 4, 6, 1, 16>(v, layer, stream);
    }
}

template <int D>
bool launch_mma_m(const EngineView& v, int layer, cudaStream_t stream) {
    switch (v.m) {
#define CLO_MM(MM)                          \
    case MM:                                \
        launch_mma<D, MM>(v, layer, stream); \
        return true;
        CLO_MM(1) CLO_MM(2) CLO_MM(3) CLO_MM(4) CLO_MM(5) CLO_MM(6) CLO_MM(7) CLO_MM(8)
#undef CLO_MM
        default:
            return false;
    }
}

bool mma_disabled() {
    static const bool off = [] {
        const char* e = getenv("CLO_ATTN");
        return e && (std::string(e) == "tma" || std::string(e) == "ffma");
    }();
    return off;
}

}  // namespace

bool attention_mma_supported(int dtype, int d, int m, int k) {
    return dtype == kBF16 && (d == 64 || d == 128) && m >= 1 && m <= 8 && k % 4 == 0;
}

size_t attention_mma_partial_floats(int B, int H, int m, int d, int k, int sink, int recent) {
    EngineView v{};
    v.B = B;
    v.H = H;
    v.k = k;
    v.sink = sink;
    v.recent = recent;
    const int N = (k + sink + recent + kTileMin - 1) / kTileMin;
    const int slots = N > 2 * kNumSMs ? N : 2 * kNumSMs;  // per head: tile runs, or CTA pieces (c <= G)
    return (size_t)B * H * slots * m * (d + 4);  // partials, rows padded to 16 B
}

bool launch_attention_mma(const EngineView& v, int layer, cudaStream_t stream) {
    if (mma_disabled() || !attention_mma_supported(v.kv_dtype, v.d, v.m, v.k)) return false;
    return v.d == 64 ? launch_mma_m<64>(v, layer, stream) : launch_mma_m<128>(v, layer, stream);
}

}  // namespace clo
