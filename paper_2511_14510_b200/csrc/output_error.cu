// output_error.cu — EngineConfig::compute_oracle_error (engine.hpp:48) on the
// device: every decode step, every (sequence, layer, KV head) also takes the
// EXACT top-k with its true queries over the pre-append pool
// (group_topk(t, l, g, true, exact), engine.cpp:263-267), attends each query
// head over union(that selection, sink/recent window) in double
// (topk_attention / attend_rows, attention.cpp:33-55, engine.cpp:394-405) and
// accumulates relative_l2(step output, oracle output) (engine.cpp:87-96)
// into the sequence's output_err_sum / output_err_count
// (DecodeMetrics::mean_output_error, engine.cpp:67-69).
//
// A diagnostic, like in the reference: it reads every key of every head each
// step (offloaded heads over PCIe from the host store), so it is enabled only
// when asked for. One CTA per segment; results do not depend on the launch
// shape (exact integer selection; fp64 attention).
#include <cub/block/block_scan.cuh>

#include "output_error.cuh"

namespace clo {

namespace {

constexpr int kThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kThreads) output_error_kernel(EngineView v, int l, OutputErrorArgs a) {
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage scan;
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int s_need, s_run, s_nsel, s_nu;
    __shared__ double red[kThreads / 32];
    extern __shared__ double q[];  // [m][d]
    const int b = blockIdx.x / v.H, g = blockIdx.x % v.H, lg = l * v.H + g;
    const int seg = (b * v.L + l) * v.H + g;
    const int t = *v.dev_step + 1;
    const int n_pool = v.n_prompt + t - 1, n_after = n_pool + 1;
    const bool pers = v.persistent[lg] != 0;
    const int d = v.d, m = v.m;
    // K / V row r of this head: persistent HBM store or the host store (UVA)
    const T* kbase;
    const T* vbase;
    size_t rstride;
    if (pers) {
        const size_t p = ((size_t)b * v.NP + v.pidx[lg]) * v.nmax * d;
        kbase = static_cast<const T*>(v.pk) + p;
        vbase = static_cast<const T*>(v.pv) + p;
        rstride = d;
    } else {
        const size_t hb = (size_t)b * v.seq_stride + (size_t)l * v.layer_stride + (size_t)g * v.head_stride;
        kbase = static_cast<const T*>(v.host_k) + hb;
        vbase = static_cast<const T*>(v.host_v) + hb;
        rstride = v.row_stride;
    }
    const size_t qoff = (((size_t)b * v.L + l) * v.HQ + (size_t)g * m) * d;
    for (int i = threadIdx.x; i < m * d; i += blockDim.x) q[i] = (double)v.desc->true_q[qoff + i];
    __syncthreads();

    // exact scores S(i) = max_j q_j . k_i (sequential IEEE double, retrieval.cpp:101-106)
    uint64_t* keys = a.keys + (size_t)blockIdx.x * v.nmax;
    for (int i = threadIdx.x; i < n_pool; i += blockDim.x) {
        const T* kr = kbase + (size_t)i * rstride;
        double best = 0.0;
        for (int j = 0; j < m; ++j) {
            double s = 0.0;
            for (int c = 0; c < d; ++c) s = dmac(s, q[j * d + c], to_f64<T>(kr[c]));
            if (j == 0 || s > best) best = s;
        }
        keys[i] = orderable_key(best);
    }
    __syncthreads();

    // k-th largest key: 8 MSB-first radix passes (prefix, ties still needed)
    if (threadIdx.x == 0) {
        s_prefix = 0;
        s_need = v.k;
    }
    for (int shift = 56; shift >= 0; shift -= 8) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (int i = threadIdx.x; i < n_pool; i += blockDim.x) {
            const uint64_t key = keys[i];
            if (shift == 56 || ((key ^ prefix) >> (shift + 8)) == 0) atomicAdd(&hist[(key >> shift) & 255], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0, D = 0;
            for (int dgt = 255; dgt >= 0; --dgt) {
                if (run + (int)hist[dgt] >= s_need) {
                    D = dgt;
                    break;
                }
                run += (int)hist[dgt];
            }
            s_need -= run;
            s_prefix = prefix | ((uint64_t)D << shift);
        }
        __syncthreads();
    }
    const uint64_t T_ = s_prefix;
    const int need = s_need;  // ties == T taken in index order
    // ascending selection: key > T, or key == T among the first `need` ties
    int32_t* sel = a.sel + (size_t)blockIdx.x * (v.k + v.sink + v.recent);
    if (threadIdx.x == 0) {
        s_run = 0;
        s_nsel = 0;
    }
    __syncthreads();
    for (int i0 = 0; i0 < n_pool; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const uint64_t key = i < n_pool ? keys[i] : 0;
        const int tie = i < n_pool && key == T_;
        int tie_before, ties;
        Scan(scan).ExclusiveSum(tie, tie_before, ties);
        const int take = (i < n_pool) && (key > T_ || (tie && s_run + tie_before < need));
        __syncthreads();
        int pos, taken;
        Scan(scan).ExclusiveSum(take, pos, taken);
        if (take) sel[s_nsel + pos] = i;
        __syncthreads();
        if (threadIdx.x == 0) {
            s_run += ties;
            s_nsel += taken;
        }
        __syncthreads();
    }
    // union with the sink/recent window of n_after tokens (sink_recent_indices,
    // attention.cpp:107-125; union_indices, engine.cpp:80-86), ascending
    int32_t* uni = a.uni + (size_t)blockIdx.x * (v.k + v.sink + v.recent);
    if (threadIdx.x == 0) {
        const int sink = min(v.sink, n_after), recent = min(v.recent, n_after);
        const int r0 = max(n_after - recent, sink);
        int ia = 0, nu = 0;
        auto window_at = [&](int w) { return w < sink ? w : r0 + (w - sink); };
        const int nw = sink + max(0, n_after - r0);
        int iw = 0;
        const int ns = s_nsel;
        while (ia < ns || iw < nw) {
            const int x = ia < ns ? sel[ia] : 0x7fffffff;
            const int y = iw < nw ? window_at(iw) : 0x7fffffff;
            if (x < y) {
                uni[nu++] = x;
                ++ia;
            } else if (y < x) {
                uni[nu++] = y;
                ++iw;
            } else {
                uni[nu++] = x;
                ++ia;
                ++iw;
            }
        }
        s_nu = nu;
    }
    __syncthreads();
    const int nu = s_nu;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double* sc = a.scores + (size_t)blockIdx.x * (v.k + v.sink + v.recent);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto block_reduce = [&](double x, bool is_max) {
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, x, o);
            x = is_max ? fmax(x, y) : x + y;
        }
        if (lane == 0) red[warp] = x;
        __syncthreads();
        double r = red[0];
        for (int w = 1; w < kThreads / 32; ++w) r = is_max ? fmax(r, red[w]) : r + red[w];
        __syncthreads();
        return r;
    };
    for (int j = 0; j < m; ++j) {
        const double* qj = q + j * d;
        double mx = -INFINITY;
        for (int i = threadIdx.x; i < nu; i += blockDim.x) {
            const T* kr = kbase + (size_t)uni[i] * rstride;
            double s = 0.0;
            for (int c = 0; c < d; ++c) s += qj[c] * to_f64<T>(kr[c]);
            s *= inv_sqrt_d;
            sc[i] = s;
            mx = fmax(mx, s);
        }
        mx = block_reduce(mx, true);
        double den = 0.0;
        for (int i = threadIdx.x; i < nu; i += blockDim.x) {
            const double e = exp(sc[i] - mx);
            sc[i] = e;
            den += e;
        }
        den = block_reduce(den, false);
        // oracle output column c; the step's output for this query head
        const int h = v.q0 + g * m + j;
        const float* got = v.desc->out + (((size_t)b * v.L + l) * v.HQg + h) * d;
        double num = 0.0, dd = 0.0;
        for (int c = threadIdx.x; c < d; c += blockDim.x) {
            double o = 0.0;
            for (int i = 0; i < nu; ++i) o += (sc[i] / den) * to_f64<T>(vbase[(size_t)uni[i] * rstride + c]);
            const double diff = (double)got[c] - o;
            num += diff * diff;
            dd += o * o;
        }
        num = block_reduce(num, false);
        dd = block_reduce(dd, false);
        if (threadIdx.x == 0) a.err[((size_t)b * v.L + l) * v.HQ + g * m + j] += dd == 0.0 ? 0.0 : sqrt(num / dd);
        __syncthreads();  // sc reused by the next query head
    }
    (void)seg;
}

}  // namespace

void launch_output_error(const EngineView& v, int layer, const OutputErrorArgs& a, cudaStream_t stream) {
    const size_t sm = (size_t)v.m * v.d * sizeof(double);
    if (v.kv_dtype == kBF16)
        output_error_kernel<__nv_bfloat16><<<v.B * v.H, kThreads, sm, stream>>>(v, layer, a);
    else
        output_error_kernel<float><<<v.B * v.H, kThreads, sm, stream>>>(v, layer, a);
}

}  // namespace clo
