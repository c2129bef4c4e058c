// attention.cu — K4 sparse attention (memory-bound, CUDA cores: decode is
// GEMV-shaped with m = 4-5 query rows per KV row, far below the tensor-core
// ridge point).
#include <math_constants.h>

#include "attention.cuh"
#include "exchange.cuh"

namespace clo {

namespace {

template <typename T>
struct Vec16;  // 16-byte vector of T
template <>
struct Vec16<__nv_bfloat16> {
    static constexpr int N = 8;
    __device__ __forceinline__ static void unpack(const uint4& u, float* f) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 x = __bfloat1622float2(h[i]);
            f[2 * i] = x.x;
            f[2 * i + 1] = x.y;
        }
    }
};
template <>
struct Vec16<float> {
    static constexpr int N = 4;
    __device__ __forceinline__ static void unpack(const uint4& u, float* f) {
        f[0] = __uint_as_float(u.x);
        f[1] = __uint_as_float(u.y);
        f[2] = __uint_as_float(u.z);
        f[3] = __uint_as_float(u.w);
    }
};

__device__ __forceinline__ float safe_exp2(float x) { return x == -CUDART_INF_F ? 0.f : exp2f(x); }
// weight of a partial with running max m under the merged max gm; an empty
// partial (m = -inf) weighs 0 even when gm is -inf too (no NaN)
__device__ __forceinline__ float wexp(float m, float gm) { return m == -CUDART_INF_F ? 0.f : exp2f(m - gm); }

template <typename T, int D, int M>
__global__ void __launch_bounds__(kAttnThreads) attn_engine_kernel(EngineView v, int l) {
    constexpr int EPL = Vec16<T>::N;
    constexpr int VPR = D / EPL;
    constexpr int LPR = VPR < 32 ? VPR : 32;
    constexpr int VPL = VPR / LPR;
    constexpr int RPW = 32 / LPR;
    constexpr int NW = kAttnThreads / 32;
    constexpr int E = VPL * EPL;  // elements per lane
    constexpr int U = 4;          // rows in flight per lane group

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
    const int W = s1 + (n_after - wstart);
    const int P = v.k + W;
    const int p0 = c * kAttnRows, p1 = min(P, p0 + kAttnRows);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / LPR, sub = lane % LPR;

    // queries, pre-scaled by log2(e)/sqrt(d) so softmax uses exp2
    const float scale = 1.4426950408889634f * rsqrtf((float)D);
    float q[M][E];
    const float* qsrc = v.desc->true_q + (((size_t)b * v.L + l) * v.HQ + (size_t)g * M) * D;
    bool badq = false;
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
        for (int i = 0; i < VPL; ++i)
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                const float x = qsrc[(size_t)j * D + (sub + i * LPR) * EPL + e];
                badq |= !isfinite(x);
                q[j][i * EPL + e] = x * scale;
            }
    if (badq) raise_err(v.err, kErrNonFiniteQuery);

    const int32_t* idx = v.entry_idx + (size_t)seg * v.k;
    const int32_t* stok = pers ? nullptr : v.slot_tok + (size_t)((size_t)b * v.NO + v.oidx[lg]) * v.pool;
    const int wrows = v.sink + v.recent;
    const size_t pslot = pers ? (size_t)b * v.NP + v.pidx[lg] : 0;
    const size_t oslot = pers ? 0 : (size_t)b * v.NO + v.oidx[lg];
    const T* pk = static_cast<const T*>(v.pk) + pslot * v.nmax * D;
    const T* pv = static_cast<const T*>(v.pv) + pslot * v.nmax * D;
    const T* sk = static_cast<const T*>(v.slot_k) + oslot * v.pool * D;
    const T* sv = static_cast<const T*>(v.slot_v) + oslot * v.pool * D;
    const T* wk = static_cast<const T*>(v.win_k) + oslot * wrows * D;
    const T* wv = static_cast<const T*>(v.win_v) + oslot * wrows * D;

    float mx[M], sm[M], acc[M][E];
#pragma unroll
    for (int j = 0; j < M; ++j) {
        mx[j] = -CUDART_INF_F;
        sm[j] = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) acc[j][e] = 0.f;
    }

    for (int base = p0 + warp * RPW * U; base < p1; base += NW * RPW * U) {
        uint4 kv[U][VPL], vv[U][VPL];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int pos = base + u * RPW + grp;
            ok[u] = pos < p1;
            const T* kr = nullptr;
            const T* vr = nullptr;
            int tok = 0;
            if (ok[u]) {
                if (pos < v.k) {
                    // persistent: the selection indexes the full HBM KV;
                    // offloaded: walk the cache slots (delta-gather layout)
                    tok = pers ? idx[pos] : stok[pos];
                    kr = pers ? pk + (size_t)tok * D : sk + (size_t)pos * D;
                    vr = pers ? pv + (size_t)tok * D : sv + (size_t)pos * D;
                } else {
                    const int w = pos - v.k;
                    tok = w < s1 ? w : wstart + (w - s1);
                    const int wr = tok < v.sink ? tok : v.sink + tok % v.recent;
                    kr = pers ? pk + (size_t)tok * D : wk + (size_t)wr * D;
                    vr = pers ? pv + (size_t)tok * D : wv + (size_t)wr * D;
                }
            }
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
                if (ok[u]) {
                    kv[u][i] = __ldg(reinterpret_cast<const uint4*>(kr) + sub + i * LPR);
                    vv[u][i] = __ldg(reinterpret_cast<const uint4*>(vr) + sub + i * LPR);
                } else {
                    kv[u][i] = make_uint4(0, 0, 0, 0);
                    vv[u][i] = make_uint4(0, 0, 0, 0);
                }
            }
            // dedup against the window (union_indices, engine.cpp:80-85); the
            // loads above do not wait on this test
            if (ok[u] && pos < v.k) ok[u] = !(tok < s1 || tok >= wstart);
        }
        float s[U][M];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float kf[E];
#pragma unroll
            for (int i = 0; i < VPL; ++i) Vec16<T>::unpack(kv[u][i], kf + i * EPL);
#pragma unroll
            for (int j = 0; j < M; ++j) {
                float d0 = 0.f;
#pragma unroll
                for (int e = 0; e < E; ++e) d0 = fmaf(q[j][e], kf[e], d0);
#pragma unroll
                for (int o = 1; o < LPR; o <<= 1) d0 += __shfl_xor_sync(0xffffffffu, d0, o);
                s[u][j] = ok[u] ? d0 : -CUDART_INF_F;
            }
        }
#pragma unroll
        for (int j = 0; j < M; ++j) {
            float nm = mx[j];
#pragma unroll
            for (int u = 0; u < U; ++u) nm = fmaxf(nm, s[u][j]);
            const float corr = safe_exp2(mx[j] - nm);
            mx[j] = nm;
            sm[j] *= corr;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[j][e] *= corr;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float vf[E];
#pragma unroll
            for (int i = 0; i < VPL; ++i) Vec16<T>::unpack(vv[u][i], vf + i * EPL);
#pragma unroll
            for (int j = 0; j < M; ++j) {
                const float p = (s[u][j] == -CUDART_INF_F) ? 0.f : exp2f(s[u][j] - mx[j]);
                sm[j] += p;
#pragma unroll
                for (int e = 0; e < E; ++e) acc[j][e] = fmaf(p, vf[e], acc[j][e]);
            }
        }
    }

    // merge the RPW row groups of the warp (lanes differing in the group bits)
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const float om = __shfl_xor_sync(0xffffffffu, mx[j], o);
            const float os = __shfl_xor_sync(0xffffffffu, sm[j], o);
            const float nm = fmaxf(mx[j], om);
            const float c1 = wexp(mx[j], nm), c2 = wexp(om, nm);
            sm[j] = sm[j] * c1 + os * c2;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const float oa = __shfl_xor_sync(0xffffffffu, acc[j][e], o);
                acc[j][e] = acc[j][e] * c1 + oa * c2;
            }
            mx[j] = nm;
        }
    }

    // merge warps through shared memory: [NW][M][D + 2]
    __shared__ float red[NW][M][D + 2];
    if (grp == 0) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
#pragma unroll
            for (int i = 0; i < VPL; ++i)
#pragma unroll
                for (int e = 0; e < EPL; ++e) red[warp][j][(sub + i * LPR) * EPL + e] = acc[j][i * EPL + e];
            if (sub == 0) {
                red[warp][j][D] = mx[j];
                red[warp][j][D + 1] = sm[j];
            }
        }
    }
    __syncthreads();
    float* part = v.attn_part + ((size_t)bg * v.max_attn_chunks + c) * M * (D + 2);
    for (int i = threadIdx.x; i < M * D; i += blockDim.x) {
        const int j = i / D, e = i % D;
        float gm = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < NW; ++w) gm = fmaxf(gm, red[w][j][D]);
        float a = 0.f, s = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float cw = wexp(red[w][j][D], gm);
            a += red[w][j][e] * cw;
            s += red[w][j][D + 1] * cw;
        }
        part[j * (D + 2) + e] = a;
        if (e == 0) {
            part[j * (D + 2) + D] = gm;
            part[j * (D + 2) + D + 1] = s;
        }
    }
    __threadfence();
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(&v.attn_count[bg], 1);
        s_last = prev == nch - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int i = threadIdx.x; i < M * D; i += blockDim.x) {
        const int j = i / D, e = i % D;
        const float* pb = v.attn_part + (size_t)bg * v.max_attn_chunks * M * (D + 2) + j * (D + 2);
        const size_t stride = (size_t)M * (D + 2);
        float gm = -CUDART_INF_F;
        for (int cc = 0; cc < nch; ++cc) gm = fmaxf(gm, __ldcg(pb + cc * stride + D));
        float a = 0.f, s = 0.f;
        for (int cc = 0; cc < nch; ++cc) {
            const float cw = wexp(__ldcg(pb + cc * stride + D), gm);
            a += __ldcg(pb + cc * stride + e) * cw;
            s += __ldcg(pb + cc * stride + D + 1) * cw;
        }
        emit_head_output(v, t, b, l, g * M + j, e, a / s);
    }
    signal_head_output(v, l);
    if (threadIdx.x == 0) v.attn_count[bg] = 0;
}

// ---------------------------------------------------------------- op-level

template <typename T, typename ACC>
__global__ void attn_op_kernel(const double* q, const T* keys, const T* values, int d,
                               const int32_t* idx, int nidx, double* out, double* scratch) {
    const int j = blockIdx.x;
    const double* qj = q + (size_t)j * d;
    ACC* sc = reinterpret_cast<ACC*>(scratch) + (size_t)j * nidx;
    __shared__ ACC red[256];
    const ACC inv_sqrt_d = (ACC)1 / sqrt((ACC)d);
    ACC mx = -(ACC)INFINITY;
    for (int i = threadIdx.x; i < nidx; i += blockDim.x) {
        const T* kr = keys + (size_t)idx[i] * d;
        ACC s = 0;
        for (int cc = 0; cc < d; ++cc) {
            if constexpr (sizeof(ACC) == 8)
                s = dmac(s, qj[cc], to_f64<T>(kr[cc]));
            else
                s = fmaf((float)qj[cc], to_f32<T>(kr[cc]), s);
        }
        s = s * inv_sqrt_d;
        sc[i] = s;
        mx = s > mx ? s : mx;
    }
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = red[threadIdx.x] > red[threadIdx.x + o] ? red[threadIdx.x] : red[threadIdx.x + o];
        __syncthreads();
    }
    mx = red[0];
    __syncthreads();
    ACC sum = 0;
    for (int i = threadIdx.x; i < nidx; i += blockDim.x) {
        const ACC e = exp(sc[i] - mx);
        sc[i] = e;
        sum += e;
    }
    red[threadIdx.x] = sum;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    const ACC denom = red[0];
    for (int cc = threadIdx.x; cc < d; cc += blockDim.x) {
        ACC a = 0;
        for (int i = 0; i < nidx; ++i) a += (sc[i] / denom) * (ACC)to_f64<T>(values[(size_t)idx[i] * d + cc]);
        out[(size_t)j * d + cc] = (double)a;
    }
}

__global__ void validate_idx_kernel(const int32_t* idx, int nidx, int64_t n, uint32_t* bitmap,
                                    int* err) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nidx; i += gridDim.x * blockDim.x) {
        const int32_t x = idx[i];
        if (x < 0 || x >= n) {
            atomicOr(err, kErrIndexRange);
            continue;
        }
        const uint32_t bit = 1u << (x & 31);
        const uint32_t old = atomicOr(&bitmap[x >> 5], bit);
        if (old & bit) atomicOr(err, kErrDuplicate);
    }
}

}  // namespace

int attention_chunks(int k, int sink, int recent) {
    return (k + sink + recent + kAttnRows - 1) / kAttnRows;
}

bool attention_supported(int dtype, int d, int m) {
    if (dtype != kBF16 && dtype != kF32) return false;
    if (!(d == 64 || d == 128 || d == 256 || d == 32 || d == 16 || d == 8)) return false;
    if (dtype == kF32 && d < 4) return false;
    return m >= 1 && m <= 8;
}

template <typename T, int D>
static void launch_attn_d(const EngineView& v, int layer, dim3 grid, cudaStream_t stream) {
    switch (v.m) {
#define CLO_M(MM) \
    case MM:      \
        attn_engine_kernel<T, D, MM><<<grid, kAttnThreads, 0, stream>>>(v, layer); break;
        CLO_M(1) CLO_M(2) CLO_M(3) CLO_M(4) CLO_M(5) CLO_M(6) CLO_M(7) CLO_M(8)
#undef CLO_M
        default:
            break;
    }
}

template <typename T>
static void launch_attn_t(const EngineView& v, int layer, dim3 grid, cudaStream_t stream) {
    switch (v.d) {
        case 8:
            if constexpr (sizeof(T) == 2) launch_attn_d<T, 8>(v, layer, grid, stream);
            break;
        case 16: launch_attn_d<T, 16>(v, layer, grid, stream); break;
        case 32: launch_attn_d<T, 32>(v, layer, grid, stream); break;
        case 64: launch_attn_d<T, 64>(v, layer, grid, stream); break;
        case 128: launch_attn_d<T, 128>(v, layer, grid, stream); break;
        case 256: launch_attn_d<T, 256>(v, layer, grid, stream); break;
        default: break;
    }
}

void launch_attention_engine(const EngineView& v, int layer, cudaStream_t stream) {
    dim3 grid(attention_chunks(v.k, v.sink, v.recent), v.B * v.H);
    if (v.kv_dtype == kBF16)
        launch_attn_t<__nv_bfloat16>(v, layer, grid, stream);
    else
        launch_attn_t<float>(v, layer, grid, stream);
}

void launch_attention_op(const double* q, int m, const void* keys, const void* values, int dtype,
                         int d, const int32_t* idx, int nidx, double* out, double* scratch,
                         cudaStream_t stream) {
    switch (dtype) {
        case kBF16:
            attn_op_kernel<__nv_bfloat16, float><<<m, 256, 0, stream>>>(
                q, static_cast<const __nv_bfloat16*>(keys), static_cast<const __nv_bfloat16*>(values), d,
                idx, nidx, out, scratch);
            break;
        case kF32:
            attn_op_kernel<float, float><<<m, 256, 0, stream>>>(
                q, static_cast<const float*>(keys), static_cast<const float*>(values), d, idx, nidx,
                out, scratch);
            break;
        default:
            attn_op_kernel<double, double><<<m, 256, 0, stream>>>(
                q, static_cast<const double*>(keys), static_cast<const double*>(values), d, idx,
                nidx, out, scratch);
            break;
    }
}

void launch_validate_indices(const int32_t* idx, int nidx, int64_t n, uint32_t* bitmap, int* err,
                             cudaStream_t stream) {
    if (nidx <= 0) return;
    const int grid = (nidx + 255) / 256 < 1024 ? (nidx + 255) / 256 : 1024;
    validate_idx_kernel<<<grid, 256, 0, stream>>>(idx, nidx, n, bitmap, err);
}

}  // namespace clo
