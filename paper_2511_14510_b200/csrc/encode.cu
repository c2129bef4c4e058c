// encode.cu — K6 (prefill sign-hash encode), K5 (per-step append), helpers.
#include "encode.cuh"
#include "hash.cuh"
#include "select.cuh"

namespace clo {

namespace {

constexpr int kEncRows = 32;
constexpr int kEncThreads = 256;

// One CTA = 32 rows of one segment x all bits. Rows are widened to double in
// shared memory; thread b walks c = 0..d-1 once, keeping 32 sequential row
// accumulators (P[b][c] read once per c, coalesced from P^T).
template <typename T>
__global__ void __launch_bounds__(kEncThreads) encode_kernel(const EncodeSeg* segs, int64_t n,
                                                             int d, int bits, int* err) {
    extern __shared__ double ks[];  // [kEncRows][d]
    const EncodeSeg sg = segs[blockIdx.y];
    const int words = (bits + 63) / 64;
    const int64_t r0 = (int64_t)blockIdx.x * kEncRows;
    const int nr = (int)(n - r0 < kEncRows ? n - r0 : kEncRows);
    const T* rows = static_cast<const T*>(sg.rows) + r0 * d;
    for (int i = threadIdx.x; i < nr * d; i += blockDim.x) {
        const double x = to_f64<T>(rows[i]);
        if (!isfinite(x)) raise_err(err, kErrNonFiniteKey);
        ks[i] = x;
    }
    __syncthreads();
    uint32_t* out32 = reinterpret_cast<uint32_t*>(sg.codes + r0 * words);
    for (int b0 = 0; b0 < words * 64; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        double s[kEncRows];
#pragma unroll
        for (int r = 0; r < kEncRows; ++r) s[r] = 0.0;
        if (b < bits) {
            for (int c = 0; c < d; ++c) {
                const double p = sg.proj_t[(size_t)c * bits + b];
#pragma unroll
                for (int r = 0; r < kEncRows; ++r) s[r] = dmac(s[r], p, ks[r * d + c]);
            }
        }
#pragma unroll
        for (int r = 0; r < kEncRows; ++r) {
            const unsigned bal = __ballot_sync(0xffffffffu, b < bits && s[r] >= 0.0);
            if ((threadIdx.x & 31) == 0 && r < nr && b < words * 64)
                out32[(size_t)r * words * 2 + (b >> 5)] = bal;
        }
    }
}

template <typename T>
__device__ __forceinline__ bool same_bits(T a, T b) {
    if constexpr (sizeof(T) == 2)
        return __bfloat16_as_ushort(a) == __bfloat16_as_ushort(b);
    else
        return __float_as_uint(a) == __float_as_uint(b);
}

template <typename T>
__device__ __forceinline__ void store_row(void* base, size_t row, int d, const T* src) {
    T* dst = static_cast<T*>(base) + row * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = src[i];
}

constexpr int kAppendTile = 16;  // new key rows hashed per pass of an append hash CTA

template <typename T>
__device__ __forceinline__ void append_hash(const EngineView& v, int l, int r) {
    const int g = r / v.words, w = r % v.words;
    const int lg = l * v.H + g;
    const int t = *v.dev_step + 1;
    const int row = v.n_prompt + t - 1;
    extern __shared__ __align__(128) double hsm[];  // P slice [d][64], rows [kAppendTile][d]
    double* ps = hsm;
    double* xs = hsm + (size_t)v.d * 64;
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        bulk::mbar_init(&bar);
        bulk::load_async(ps, v.proj_w + ((size_t)lg * v.words + w) * v.d * 64, (uint32_t)v.d * 64 * 8, &bar);
    }
    const T* nk = static_cast<const T*>(v.desc->new_k);
    for (int b0 = 0; b0 < v.B; b0 += kAppendTile) {
        const int nb = min(kAppendTile, v.B - b0);
        if (b0 > 0) __syncthreads();  // the previous tile's chains are done with xs
        for (int i = threadIdx.x; i < nb * v.d; i += blockDim.x) {
            const int bb = b0 + i / v.d, c = i % v.d;
            xs[i] = to_f64<T>(nk[(((size_t)bb * v.L + l) * v.H + g) * v.d + c]);
        }
        __syncthreads();
        if (b0 == 0) bulk::wait(&bar, 0);
        hash_word(ps, xs, v.d, nb, v.d, w, v.bits, [&](int j) {
            const size_t seg = ((size_t)(b0 + j) * v.L + l) * v.H + g;
            return reinterpret_cast<uint32_t*>(v.codes + seg * v.code_stride + (size_t)row * v.words);
        });
    }
}

// Phase 2 of one layer (engine.cpp:360-370). Two CTA roles in one grid:
//   blockIdx.x <  B*H   one (sequence, KV head): the new K/V row into the
//                       host store (or the persistent HBM store), the window
//                       ring and the K mirror
//   blockIdx.x >= B*H   one (KV head g, code word w): update_metadata's sign
//                       bits (append_sign_row, retrieval.cpp:14-25) of the new
//                       key of every sequence, word w only, against P's word
//                       slice staged in shared memory by one bulk copy
//                       (hash.cuh) -- P is read once per (g, w) instead of
//                       once per sequence in dependent batches.
template <typename T>
__global__ void __launch_bounds__(kEncThreads) append_kernel(EngineView v, int l) {
    if ((int)blockIdx.x >= v.B * v.H) {
        append_hash<T>(v, l, (int)blockIdx.x - v.B * v.H);
        return;
    }
    const int b = blockIdx.x / v.H, g = blockIdx.x % v.H;
    const int lg = l * v.H + g;
    const int seg = (b * v.L + l) * v.H + g;
    const bool pers = v.persistent[lg] != 0;
    const int t = *v.dev_step + 1;
    const int row = v.n_prompt + t - 1;  // n_pool: the new token's index
    __shared__ T kr[kMaxHeadDim], vr[kMaxHeadDim];
    const size_t off = (((size_t)b * v.L + l) * v.H + g) * v.d;
    const T* nk = static_cast<const T*>(v.desc->new_k) + off;
    const T* nv = static_cast<const T*>(v.desc->new_v) + off;
    for (int i = threadIdx.x; i < v.d; i += blockDim.x) {
        kr[i] = nk[i];
        vr[i] = nv[i];
        if (!isfinite(to_f64<T>(kr[i]))) raise_err(v.err, kErrNonFiniteKey);
        if (!isfinite(to_f64<T>(vr[i]))) raise_err(v.err, kErrNonFiniteValue);
    }
    __syncthreads();
    if (pers) {
        const size_t p = (size_t)b * v.NP + v.pidx[lg];
        store_row<T>(v.pk, p * v.nmax + row, v.d, kr);
        store_row<T>(v.pv, p * v.nmax + row, v.d, vr);
    } else {
        const size_t hb = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
        T* hk = static_cast<T*>(v.host_k_w) + hb + (size_t)row * v.row_stride;
        T* hv = static_cast<T*>(v.host_v_w) + hb + (size_t)row * v.row_stride;
        // layer_stride 0 aliases one host matrix across layers: sound only if
        // every layer appends the same row. Layer 0 (or the first offloaded
        // layer) writes it; later layers check their step input against layer
        // 0's (device memory) and raise kErrAlias instead of overwriting it.
        bool write = true;
        if (v.layer_stride == 0 && l > 0) {
            const size_t off0 = ((size_t)b * v.L * v.H + g) * v.d;  // layer 0, same (b, g)
            const T* nk0 = static_cast<const T*>(v.desc->new_k) + off0;
            const T* nv0 = static_cast<const T*>(v.desc->new_v) + off0;
            int diff = 0;
            for (int i = threadIdx.x; i < v.d; i += blockDim.x)
                diff |= !same_bits<T>(nk0[i], kr[i]) || !same_bits<T>(nv0[i], vr[i]);
            if (__syncthreads_or(diff)) {
                if (threadIdx.x == 0) raise_err(v.err, kErrAlias);
            }
            for (int l2 = 0; l2 < l && write; ++l2)  // the first offloaded layer of head g writes the row
                write = v.persistent[l2 * v.H + g] != 0;
        }
        if (write) {
            store_row<T>(hk, 0, v.d, kr);  // zero-copy store into the pinned host store
            store_row<T>(hv, 0, v.d, vr);
        }
        const size_t o = (size_t)b * v.NO + v.oidx[lg];
        const int wrows = v.sink + v.recent;
        if (row < v.sink) {
            store_row<T>(v.win_k, o * wrows + row, v.d, kr);
            store_row<T>(v.win_v, o * wrows + row, v.d, vr);
        }
        if (v.recent > 0) {
            store_row<T>(v.win_k, o * wrows + v.sink + row % v.recent, v.d, kr);
            store_row<T>(v.win_v, o * wrows + v.sink + row % v.recent, v.d, vr);
        }
        if (v.kmirror) store_row<T>(v.kmirror, o * v.nmax + row, v.d, kr);
    }
}

__global__ void step_end_kernel(int* dev_step, int* ca, int* cb, int L, int* claim, int* done) {
    if (threadIdx.x == 0) *dev_step += 1;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        ca[i] = 0;
        cb[i] = 0;
        if (claim) claim[i] = 0;
        if (done) done[i] = 0;
    }
}

template <typename T>
__global__ void check_finite_kernel(const T* p, int64_t count, int* err, int bit) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(to_f64<T>(p[i]));
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, bit);
}

template <typename T>
__global__ void window_init_kernel(EngineView v) {
    const int seg = blockIdx.x;
    const int g = seg % v.H, l = (seg / v.H) % v.L, b = seg / (v.H * v.L);
    const int lg = l * v.H + g;
    if (v.persistent[lg]) return;
    const size_t o = (size_t)b * v.NO + v.oidx[lg];
    const int n = v.n_prompt, wrows = v.sink + v.recent;
    const size_t hb = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
    const T* hk = static_cast<const T*>(v.host_k) + hb;
    const T* hv = static_cast<const T*>(v.host_v) + hb;
    T* wk = static_cast<T*>(v.win_k) + o * wrows * v.d;
    T* wv = static_cast<T*>(v.win_v) + o * wrows * v.d;
    const int ns = min(v.sink, n);
    for (int i = threadIdx.x; i < ns * v.d; i += blockDim.x) {
        const size_t src = (size_t)(i / v.d) * v.row_stride + i % v.d;
        wk[i] = hk[src];
        wv[i] = hv[src];
    }
    if (v.recent > 0) {
        const int t0 = max(0, n - v.recent);
        for (int i = threadIdx.x; i < (n - t0) * v.d; i += blockDim.x) {
            const int t = t0 + i / v.d, c = i % v.d;
            const size_t dst = (size_t)(v.sink + t % v.recent) * v.d + c;
            wk[dst] = hk[(size_t)t * v.row_stride + c];
            wv[dst] = hv[(size_t)t * v.row_stride + c];
        }
    }
}

}  // namespace

void launch_encode(const EncodeSeg* segs_dev, int n_segs, int64_t n, int d, int bits, int dtype,
                   int* err, cudaStream_t stream) {
    if (n <= 0 || n_segs <= 0) return;
    dim3 grid((unsigned)((n + kEncRows - 1) / kEncRows), (unsigned)n_segs);
    const size_t sm = (size_t)kEncRows * d * sizeof(double);  // 64 KiB at d = 256: opt in
    if (sm > 48 * 1024) {
        cudaFuncSetAttribute(encode_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(encode_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(encode_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    }
    switch (dtype) {
        case kBF16:
            encode_kernel<__nv_bfloat16><<<grid, kEncThreads, sm, stream>>>(segs_dev, n, d, bits, err);
            break;
        case kF32:
            encode_kernel<float><<<grid, kEncThreads, sm, stream>>>(segs_dev, n, d, bits, err);
            break;
        default:
            encode_kernel<double><<<grid, kEncThreads, sm, stream>>>(segs_dev, n, d, bits, err);
            break;
    }
}

void launch_append(const EngineView& v, int layer, cudaStream_t stream) {
    const int hash_ctas = v.retriever == 1 ? v.H * v.words : 0;
    const size_t sm = hash_ctas ? (size_t)v.d * (64 + kAppendTile) * sizeof(double) : 0;
    const unsigned grid = (unsigned)(v.B * v.H + hash_ctas);
    if (v.kv_dtype == kBF16) {
        cudaFuncSetAttribute(append_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        append_kernel<__nv_bfloat16><<<grid, kEncThreads, sm, stream>>>(v, layer);
    } else {
        cudaFuncSetAttribute(append_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        append_kernel<float><<<grid, kEncThreads, sm, stream>>>(v, layer);
    }
}

void launch_step_end(const EngineView& v, int* count_a, int* count_b, cudaStream_t stream) {
    step_end_kernel<<<1, 128, 0, stream>>>(v.dev_step, count_a, count_b, v.L, v.xfer_claim, v.xfer_done);
}

void launch_check_finite(const void* p, int dtype, int64_t count, int* err, int bit,
                         cudaStream_t stream) {
    if (count <= 0) return;
    int64_t blocks = (count + 255) / 256;
    const int grid = (int)(blocks < kNumSMs * 16 ? blocks : kNumSMs * 16);
    switch (dtype) {
        case kBF16:
            check_finite_kernel<<<grid, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(p), count, err, bit);
            break;
        case kF32:
            check_finite_kernel<<<grid, 256, 0, stream>>>(static_cast<const float*>(p), count, err, bit);
            break;
        default:
            check_finite_kernel<<<grid, 256, 0, stream>>>(static_cast<const double*>(p), count, err, bit);
            break;
    }
}

void launch_window_init(const EngineView& v, cudaStream_t stream) {
    if (v.kv_dtype == kBF16) {
        window_init_kernel<__nv_bfloat16><<<v.B * v.L * v.H, 256, 0, stream>>>(v);
    } else {
        window_init_kernel<float><<<v.B * v.L * v.H, 256, 0, stream>>>(v);
    }
}

}  // namespace clo
