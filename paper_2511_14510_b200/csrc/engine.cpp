// engine.cpp — host side of the B200 DecodeEngine (engine.hpp:91-139,
// engine.cpp:106-557 of the reference). The host validates, allocates,
// uploads profiles/projections, and records ONE CUDA graph per decode step;
// every per-step decision (hit/miss, selection, transfer, append, attention)
// happens on the device.
#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <unistd.h>

#include <cuda.h>
#include <sstream>
#include <string>
#include <vector>

#include "attention.cuh"
#include "encode.cuh"
#include "exchange.cuh"
#include "gather.cuh"
#include "lookup.cuh"
#include "select.cuh"
#include "select_fused.cuh"
#include "output_error.cuh"

namespace clo {

namespace {

// Gather CTAs: enough outstanding PCIe reads to cover the host round trip
// without flooding the SMs the concurrent kernels need (CLO_GATHER_CTAS
// overrides for experiments).
int64_t gather_ctas() {  // CLO_GATHER_CTAS: override of the gather grid (0 = the variant's default)
    static const int64_t n = [] {
        const char* e = getenv("CLO_GATHER_CTAS");
        return e && atoi(e) > 0 ? (int64_t)atoi(e) : (int64_t)0;
    }();
    return n;
}

// Transfer synchronisation. "events" (default): one gather launch per layer
// on the transfer stream, ordered by graph edges (device-side dependencies,
// no host sync). "flags" (CLO_TRANSFER=flags): one persistent transfer kernel
// per step gated by device flags. The flag variant spins on flags set by
// later launches, so tools that serialise kernels (ncu, compute-sanitizer)
// would deadlock it; it is opt-in.
bool use_flag_transfer() {
    static const bool flags = [] {
        const char* e = getenv("CLO_TRANSFER");
        return e && std::string(e) == "flags";
    }();
    return flags;
}

// A peer whose arrivals are missing this long has stopped stepping (not a
// slow one); CLO_EXCHANGE_TIMEOUT_MS overrides the 20 s default.
unsigned long long exchange_timeout_ns() {
    static const unsigned long long ns = [] {
        const char* e = getenv("CLO_EXCHANGE_TIMEOUT_MS");
        const long long ms = e ? atoll(e) : 0;
        return (unsigned long long)(ms > 0 ? ms : 20000) * 1000000ull;
    }();
    return ns;
}

int grid_for(int64_t units) {
    const int64_t cap = (int64_t)kNumSMs * 8;
    if (units < 1) return 1;
    return (int)std::min<int64_t>(units, cap);
}

}  // namespace

Engine::Engine(const clo_engine_config& cfg, const double* tau, const double* q_importance,
               const int* persistent)
    : cfg_(cfg) {
    const clo_model_shape& s = cfg.shape;
    // ModelShape::validate (matrix.hpp:57-65)
    if (s.num_layers <= 0) fail(CLO_ERR_CONFIG, "num_layers must be positive");
    if (s.num_q_heads <= 0 || s.num_kv_heads <= 0) fail(CLO_ERR_CONFIG, "head counts must be positive");
    if (s.num_q_heads % s.num_kv_heads != 0)
        fail(CLO_ERR_CONFIG, "num_q_heads must be a multiple of num_kv_heads");
    if (s.head_dim <= 0) fail(CLO_ERR_CONFIG, "head_dim must be positive");
    if (s.bytes_per_element <= 0) fail(CLO_ERR_CONFIG, "bytes_per_element must be positive");
    // DecodeEngine ctor checks (engine.cpp:115-136)
    if (cfg.k < 1) fail(CLO_ERR_ARGUMENT, "k must be at least 1");
    if (cfg.k > cfg.n_prompt) fail(CLO_ERR_ARGUMENT, "k exceeds the prompt length; nothing to select from at step 0");
    if (cfg.sink_tokens < 0 || cfg.recent_tokens < 0) fail(CLO_ERR_ARGUMENT, "window sizes must be non-negative");
    if (cfg.policy == CLO_POLICY_LRU || cfg.policy == CLO_POLICY_LFU)
        fail(CLO_ERR_CONFIG, "block-cache policies (lru/lfu) are outside the CLO hot path");
    if (cfg.policy != CLO_POLICY_SIMILARITY && cfg.policy != CLO_POLICY_PREFETCH_ONLY)
        fail(CLO_ERR_CONFIG, "unknown policy");
    if (cfg.always_hit && cfg.always_miss) fail(CLO_ERR_CONFIG, "always_hit and always_miss are mutually exclusive");
    if (cfg.retriever != CLO_RETRIEVER_EXACT && cfg.retriever != CLO_RETRIEVER_SIGN_HASH)
        fail(CLO_ERR_CONFIG, "unknown retriever");
    if (cfg.retriever == CLO_RETRIEVER_SIGN_HASH && (cfg.hash_bits <= 0 || cfg.hash_bits % 8 != 0))
        fail(CLO_ERR_ARGUMENT, "hash_bits must be a positive multiple of 8");
    if (cfg.hash_bits > 64 * kMaxHashWords) fail(CLO_ERR_CONFIG, "hash_bits above 512 are not supported");
    if (cfg.batch < 1) fail(CLO_ERR_CONFIG, "batch must be positive");
    if (cfg.max_steps < 0) fail(CLO_ERR_CONFIG, "max_steps must be non-negative");
    if (cfg.kv_dtype != CLO_DTYPE_BF16 && cfg.kv_dtype != CLO_DTYPE_F32)
        fail(CLO_ERR_CONFIG, "kv_dtype must be BF16 or F32");
    const int m = s.num_q_heads / s.num_kv_heads;
    if (m > kMaxGroup) fail(CLO_ERR_CONFIG, "GQA group size above 16 is not supported");
    if (!attention_supported(cfg.kv_dtype, s.head_dim, m))
        fail(CLO_ERR_CONFIG, "head_dim must be one of 8/16/32/64/128/256 and the GQA group <= 8");
    if ((s.head_dim * (cfg.kv_dtype == CLO_DTYPE_BF16 ? 2 : 4)) % 16 != 0)
        fail(CLO_ERR_CONFIG, "K/V rows must be a multiple of 16 bytes");
    if (cfg.sink_tokens + cfg.recent_tokens > 4096) fail(CLO_ERR_CONFIG, "window too large");
    if (cfg.k > reconcile_max_k()) fail(CLO_ERR_CONFIG, "k above 8192 is not supported");
    // pool slots age by decode step in 16-bit radix keys (age + 1)
    if (cfg.max_steps > 65000) fail(CLO_ERR_CONFIG, "max_steps above 65000 is not supported");
    if (cfg.victim_rows > (1 << 20)) fail(CLO_ERR_CONFIG, "victim_rows above 2^20 is not supported");

    const int L = s.num_layers, H = s.num_kv_heads;
    tau_.assign(tau, tau + (size_t)L * H);
    qimp_.assign(q_importance, q_importance + (size_t)L * H * m);
    for (double w : qimp_)
        if (w < 0.0) fail(CLO_ERR_ARGUMENT, "importance weights must be non-negative");
    persistent_.resize((size_t)L * H);
    pidx_.assign((size_t)L * H, -1);
    oidx_.assign((size_t)L * H, -1);
    for (int i = 0; i < L * H; ++i) {
        persistent_[i] = persistent[i] ? 1 : 0;
        if (persistent_[i])
            pidx_[i] = np_++;
        else
            oidx_[i] = no_++;
    }
    layer_has_pers_.assign(L, 0);
    layer_has_off_.assign(L, 0);
    for (int l = 0; l < L; ++l)
        for (int g = 0; g < H; ++g) (persistent_[l * H + g] ? layer_has_pers_ : layer_has_off_)[l] = 1;

    sync_mode_ = cfg.sync_override >= 0 ? cfg.sync_override
                                        : (cfg.policy == CLO_POLICY_SIMILARITY ? CLO_SYNC_GPU_CENTRIC
                                                                               : CLO_SYNC_CPU_CENTRIC);

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        fail(CLO_ERR_CUDA, "no CUDA device: the CLO path has no CPU fallback");
    CLO_CUDA(cudaSetDevice(cfg.device));
    allocate();
}

Engine::~Engine() {
    cudaSetDevice(cfg_.device);
    for (int r = 0; r < kMaxRanks; ++r)
        if (xipc_[r]) cudaIpcCloseMemHandle(xbase_[r]);
    drop_graphs();
    for (auto& recs : prof_)
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    if (tl_base_) cudaEventDestroy(tl_base_);
    for (auto ev : ev_attn_) cudaEventDestroy(ev);
    for (auto ev : ev_pref_) cudaEventDestroy(ev);
    for (auto ev : ev_sel_) cudaEventDestroy(ev);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_join2_) cudaEventDestroy(ev_join2_);
    if (ev_join3_) cudaEventDestroy(ev_join3_);
    if (ev_step_) cudaEventDestroy(ev_step_);
    if (s_main_) cudaStreamDestroy(s_main_);
    if (s_pref_) cudaStreamDestroy(s_pref_);
    if (s_pref2_) cudaStreamDestroy(s_pref2_);
    if (s_xfer_) cudaStreamDestroy(s_xfer_);
    if (s_copy_) cudaStreamDestroy(s_copy_);
    for (int i = 0; i < 2; ++i) {
        if (ev_in_[i]) cudaEventDestroy(ev_in_[i]);
        if (ev_free_[i]) cudaEventDestroy(ev_free_[i]);
    }
    if (desc_host_) cudaFreeHost(desc_host_);
    for (auto ev : desc_ev_) cudaEventDestroy(ev);
}

void Engine::allocate() {
    const clo_model_shape& s = cfg_.shape;
    const int B = cfg_.batch, L = s.num_layers, H = s.num_kv_heads, HQ = s.num_q_heads;
    const int m = HQ / H, d = s.head_dim, k = cfg_.k;
    const size_t esz = cfg_.kv_dtype == CLO_DTYPE_BF16 ? 2 : 4;
    nmax_ = cfg_.n_prompt + cfg_.max_steps;
    max_chunks_ = (nmax_ + kScoreChunk - 1) / kScoreChunk;
    words_ = (cfg_.hash_bits + 63) / 64;
    code_stride_ = ((int64_t)nmax_ * words_ + 1) / 2 * 2;
    nb_ = cfg_.hash_bits + 1;
    const size_t segs = (size_t)B * L * H;
    const size_t wrows = (size_t)cfg_.sink_tokens + cfg_.recent_tokens;

    d_persistent_.alloc(sizeof(int) * L * H);
    d_pidx_.alloc(sizeof(int) * L * H);
    d_oidx_.alloc(sizeof(int) * L * H);
    CLO_CUDA(cudaMemcpy(d_persistent_.p, persistent_.data(), sizeof(int) * L * H, cudaMemcpyHostToDevice));
    CLO_CUDA(cudaMemcpy(d_pidx_.p, pidx_.data(), sizeof(int) * L * H, cudaMemcpyHostToDevice));
    CLO_CUDA(cudaMemcpy(d_oidx_.p, oidx_.data(), sizeof(int) * L * H, cudaMemcpyHostToDevice));
    d_tau_.alloc(sizeof(double) * L * H);
    d_qimp_.alloc(sizeof(double) * L * H * m);
    CLO_CUDA(cudaMemcpy(d_tau_.p, tau_.data(), sizeof(double) * L * H, cudaMemcpyHostToDevice));
    CLO_CUDA(cudaMemcpy(d_qimp_.p, qimp_.data(), sizeof(double) * L * H * m, cudaMemcpyHostToDevice));

    d_pk_.alloc((size_t)B * np_ * nmax_ * d * esz, false);
    d_pv_.alloc((size_t)B * np_ * nmax_ * d * esz, false);
    if (cfg_.retriever == CLO_RETRIEVER_EXACT) d_kmirror_.alloc((size_t)B * no_ * nmax_ * d * esz, false);
    // row pool per offloaded head: the entry's k rows + victim rows that left it
    // auto (victim_rows < 0): 8k rows per head (profiles/README.md: the PCIe
    // bytes saved grow with the area up to ~8k at 128K contexts), shrunk so
    // the victim areas take at most 40% of the HBM still free here
    int victim = cfg_.victim_rows;
    if (victim < 0) {
        victim = 8 * k;
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && B * no_ > 0) {
            const size_t per_row = 2 * (size_t)d * esz;  // K + V
            const size_t fit = (size_t)(0.4 * (double)free_b) / ((size_t)B * no_ * per_row);
            victim = (int)std::min<size_t>((size_t)victim, fit);
        }
    }
    pool_ = k + victim;
    d_slot_k_.alloc((size_t)B * no_ * pool_ * d * esz);
    d_slot_v_.alloc((size_t)B * no_ * pool_ * d * esz);
    d_win_k_.alloc((size_t)B * no_ * std::max<size_t>(wrows, 1) * d * esz);
    d_win_v_.alloc((size_t)B * no_ * std::max<size_t>(wrows, 1) * d * esz);
    d_entry_idx_.alloc(sizeof(int32_t) * segs * k + 64);  // +64: 16-byte rounded token bulk copies
    d_entry_slot_.alloc(sizeof(int32_t) * B * no_ * k);
    d_slot_tok_.alloc(sizeof(int32_t) * B * no_ * pool_ + 64);
    d_slot_age_.alloc(sizeof(int32_t) * B * no_ * pool_);
    d_vhead_.alloc(sizeof(int) * std::max(B * no_, 1));  // zeroed
    d_tok2slot_.alloc(sizeof(int32_t) * B * no_ * (size_t)nmax_);
    // empty pool: no token in any slot (-1), no slot for any token (-1), ages
    // kSlotEmpty (-1: oldest)
    static_assert(kSlotEmpty == -1, "pool ages are initialised by an 0xFF memset");
    CLO_CUDA(cudaMemset(d_slot_tok_.p, 0xFF, sizeof(int32_t) * B * no_ * pool_));
    CLO_CUDA(cudaMemset(d_slot_age_.p, 0xFF, sizeof(int32_t) * B * no_ * pool_));
    CLO_CUDA(cudaMemset(d_tok2slot_.p, 0xFF, sizeof(int32_t) * B * no_ * (size_t)nmax_));
    if (cfg_.retriever == CLO_RETRIEVER_SIGN_HASH) {
        d_codes_.alloc(sizeof(uint64_t) * segs * code_stride_ + 64, false);
        // projections P (retrieval.cpp:73-74), seed mix_seed(retriever_seed, l, g)
        // (engine.cpp:172-174); stored transposed [d][bits] for coalesced reads.
        std::vector<double> pt((size_t)L * H * d * cfg_.hash_bits);
        std::vector<double> p((size_t)cfg_.hash_bits * d);
        for (int l = 0; l < L; ++l)
            for (int g = 0; g < H; ++g) {
                const uint64_t seed = mix_seed3(cfg_.retriever_seed, (uint64_t)l,
                                                (uint64_t)(g + cfg_.kv_head_offset));
                sign_hash_projection(cfg_.hash_bits, d, seed, p.data());
                double* dst = pt.data() + ((size_t)l * H + g) * d * cfg_.hash_bits;
                for (int b = 0; b < cfg_.hash_bits; ++b)
                    for (int c = 0; c < d; ++c) dst[(size_t)c * cfg_.hash_bits + b] = p[(size_t)b * d + c];
            }
        d_proj_t_.alloc(sizeof(double) * pt.size(), false);
        CLO_CUDA(cudaMemcpy(d_proj_t_.p, pt.data(), sizeof(double) * pt.size(), cudaMemcpyHostToDevice));
        // the same P^T cut into 64-bit word slices [L*H][words][d][64] (zero past
        // `bits`): one contiguous bulk copy stages the slice a decode-time hash
        // CTA needs in shared memory (lookup.cu, encode.cu)
        std::vector<double> pw((size_t)L * H * words_ * d * 64, 0.0);
        for (size_t lg = 0; lg < (size_t)L * H; ++lg)
            for (int w = 0; w < words_; ++w)
                for (int c = 0; c < d; ++c)
                    for (int i = 0; i < 64 && w * 64 + i < cfg_.hash_bits; ++i)
                        pw[((lg * words_ + w) * d + c) * 64 + i] =
                            pt[(lg * d + c) * cfg_.hash_bits + w * 64 + i];
        d_proj_w_.alloc(sizeof(double) * pw.size(), false);
        CLO_CUDA(cudaMemcpy(d_proj_w_.p, pw.data(), sizeof(double) * pw.size(), cudaMemcpyHostToDevice));
    }
    if (cfg_.compute_oracle_error) {  // scratch of output_error.cu (keys, scores, lists, per-sequence sums)
        const size_t segs = (size_t)B * H, w = (size_t)cfg_.k + cfg_.sink_tokens + cfg_.recent_tokens;
        d_oerr_.alloc(sizeof(uint64_t) * segs * nmax_ + (sizeof(double) + 2 * sizeof(int32_t)) * segs * w +
                      sizeof(double) * B * L * HQ + 64);
    }
    d_labels_.alloc(sizeof(double) * B * L * HQ * d);
    d_label_valid_.alloc(sizeof(int) * B * L * HQ);
    d_hits_.alloc(sizeof(unsigned long long) * segs);
    d_misses_.alloc(sizeof(unsigned long long) * segs);
    d_cache_last_.alloc(sizeof(int) * segs);
    d_entry_last_.alloc(sizeof(int) * segs);
    d_last_hit_.alloc(sizeof(int) * segs);
    {
        std::vector<int> minus1(segs, -1);
        CLO_CUDA(cudaMemcpy(d_cache_last_.p, minus1.data(), sizeof(int) * segs, cudaMemcpyHostToDevice));
        CLO_CUDA(cudaMemcpy(d_entry_last_.p, minus1.data(), sizeof(int) * segs, cudaMemcpyHostToDevice));
    }
    d_history_.alloc(sizeof(double) * segs * std::max(cfg_.max_steps, 1));
    d_gathered_.alloc(sizeof(unsigned long long));
    d_step_.alloc(sizeof(int));
    d_desc_.alloc(sizeof(StepDesc));
    d_err_.alloc(sizeof(int));
    max_attn_chunks_ = attention_chunks(k, cfg_.sink_tokens, cfg_.recent_tokens);
    d_attn_part_.alloc(sizeof(float) * std::max<size_t>((size_t)B * H * max_attn_chunks_ * m * (d + 2),
                                                         attention_mma_partial_floats(B, H, m, d, k, cfg_.sink_tokens,
                                                                                      cfg_.recent_tokens)),
                       false);
    d_attn_count_.alloc(sizeof(int) * 2 * B * H);  // arrival + slot counters (self-resetting)
    d_xfer_.alloc(sizeof(int) * 5 * L);  // ready, units, claim, done, flag
    {
        std::vector<int> off;
        for (int l = 0; l < L; ++l)
            if (layer_has_off_[l]) off.push_back(l);
        n_off_layers_ = (int)off.size();
        d_off_layers_.alloc(sizeof(int) * std::max<size_t>(off.size(), 1));
        if (!off.empty())
            CLO_CUDA(cudaMemcpy(d_off_layers_.p, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
    }

    // TMA tensor maps over the cache slots for the tensor-core attention:
    // [B*NO*pool rows][d] bf16 (entry areas: rows o*pool + [0, k)), boxes of 64 columns x 16 or 32 rows, 128-byte
    // swizzle (the kernel's stage layout). cuTensorMapEncodeTiled comes from
    // the driver through the runtime's entry-point query (no -lcuda).
    static const bool no_tma_slots = [] {  // CLO_ATTN_NOTMA=1: slot tiles by LDGSTS (experiment switch)
        const char* e = getenv("CLO_ATTN_NOTMA");
        return e && atoi(e) == 1;
    }();
    if (cfg_.kv_dtype == CLO_DTYPE_BF16 && (d == 64 || d == 128) && no_ > 0 && !no_tma_slots) {
        using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess && fn) {
            auto encode = reinterpret_cast<EncodeFn>(fn);
            CUtensorMap maps[4];
            bool ok = true;
            const cuuint64_t rows = (cuuint64_t)B * no_ * pool_;
            for (int i = 0; i < 4; ++i) {
                const cuuint64_t dims[2] = {(cuuint64_t)d, rows};
                const cuuint64_t strides[1] = {(cuuint64_t)d * 2};
                const cuuint32_t box[2] = {64, i < 2 ? 16u : 32u};
                const cuuint32_t estr[2] = {1, 1};
                ok = ok && encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (i & 1) ? d_slot_v_.p : d_slot_k_.p,
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            }
            if (ok) {
                d_tmaps_.alloc(sizeof(maps));
                CLO_CUDA(cudaMemcpy(d_tmaps_.p, maps, sizeof(maps), cudaMemcpyHostToDevice));
            }
        }
        cudaGetLastError();
    }

    // staging for host-resident step inputs / outputs
    d_in_tq_.alloc(sizeof(float) * B * L * HQ * d, false);
    d_in_aq_.alloc(sizeof(float) * B * L * HQ * d, false);
    d_in_nk_.alloc(esz * B * L * H * d, false);
    d_in_nv_.alloc(esz * B * L * H * d, false);
    for (auto& b : d_in_) b.alloc(2 * sizeof(float) * B * L * HQ * d + 2 * esz * B * L * H * d, false);
    d_out_.alloc(sizeof(float) * B * L * HQ * d, false);

    {
        // CLO_SEL_STREAMS=2: even and odd layers' selections on two streams
        // (experiment, neutral on B200); default one selection stream
        const char* e = getenv("CLO_SEL_STREAMS");
        sel_streams_ = e && atoi(e) == 2 ? 2 : 1;
    }
    for (int i = 0; i < 3; ++i) {
        if (i == 2 && sel_streams_ < 2) break;
        SelScratch& sc = scratch_[i];
        auto& bufs = scratch_bufs_[i];
        const size_t items = (size_t)B * H;
        if (i < 2) {
            bufs[0].alloc(sizeof(int) * L);
            bufs[1].alloc(sizeof(SelItem) * items * L);  // per-layer work lists
        }
        bufs[2].alloc(sizeof(double) * items * m * d);
        bufs[3].alloc(sizeof(uint64_t) * items * m * words_);
        if (cfg_.retriever == CLO_RETRIEVER_SIGN_HASH)
            bufs[4].alloc(sizeof(uint16_t) * items * nmax_, false);
        else
            bufs[5].alloc(sizeof(uint64_t) * items * nmax_, false);
        bufs[6].alloc(sizeof(uint32_t) * items * max_chunks_ * std::max(nb_, 2), false);
        bufs[7].alloc(sizeof(int) * items * max_chunks_);
        bufs[8].alloc(sizeof(int) * items * max_chunks_);
        bufs[9].alloc(sizeof(uint64_t) * items);
        bufs[10].alloc(sizeof(int) * items);
        bufs[11].alloc(sizeof(uint32_t) * items * 256);
        bufs[17].alloc(sizeof(int) * 2 * items);  // chained-stage chunk counters (zero between launches)
        if (i >= 1) bufs[12].alloc(sizeof(int32_t) * items * k, false);  // offloaded: new selections
        if (i == 1) {  // per-layer work and fetch lists (shared by both selection streams)
            bufs[13].alloc(sizeof(int32_t) * L * items * k, false);
            bufs[14].alloc(sizeof(int32_t) * L * items * k, false);
            bufs[15].alloc(sizeof(int) * L * items);
            bufs[16].alloc(sizeof(int32_t) * L * items * k, false);
        }
        sc.count = i == 2 ? scratch_[1].count : bufs[0].as<int>();
        sc.items = i == 2 ? scratch_[1].items : bufs[1].as<SelItem>();
        sc.q64 = bufs[2].as<double>();
        sc.qbits = bufs[3].as<uint64_t>();
        sc.key16 = bufs[4].as<uint16_t>();
        sc.key64 = bufs[5].as<uint64_t>();
        sc.chunk_hist = bufs[6].as<uint32_t>();
        sc.chunk_base = bufs[7].as<int>();
        sc.chunk_take = bufs[8].as<int>();
        sc.thresh = bufs[9].as<uint64_t>();
        sc.need = bufs[10].as<int>();
        sc.radix_hist = bufs[11].as<uint32_t>();
        sc.sel = bufs[12].as<int32_t>();
        const auto& lists = scratch_bufs_[i == 2 ? 1 : i];
        sc.fetch_tok = lists[13].as<int32_t>();
        sc.fetch_slot = lists[14].as<int32_t>();
        sc.fetch_count = lists[15].as<int>();
        sc.fetch_dem = lists[16].as<int32_t>();
        sc.item_done = bufs[17].as<int>();
    }

    CLO_CUDA(cudaStreamCreateWithFlags(&s_main_, cudaStreamNonBlocking));
    {
        // The selection stream feeds the transfer stream: CLO_SEL_PRIO=high
        // schedules its CTAs ahead of attention's (experiment switch).
        const char* e = getenv("CLO_SEL_PRIO");
        int lo = 0, hi = 0;
        CLO_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const int p = e && std::string(e) == "high" ? hi : (e && std::string(e) == "mid" ? (lo + hi) / 2 : lo);
        CLO_CUDA(cudaStreamCreateWithPriority(&s_pref_, cudaStreamNonBlocking, p));
        if (sel_streams_ > 1) CLO_CUDA(cudaStreamCreateWithPriority(&s_pref2_, cudaStreamNonBlocking, p));
    }
    // The transfer stream gets the highest priority: when attention CTAs
    // retire, the next layer's gather CTAs are scheduled first so the PCIe
    // link does not idle behind compute.
    int prio_lo = 0, prio_hi = 0;
    CLO_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CLO_CUDA(cudaStreamCreateWithPriority(&s_xfer_, cudaStreamNonBlocking, prio_hi));
    CLO_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    CLO_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    CLO_CUDA(cudaEventCreateWithFlags(&ev_join2_, cudaEventDisableTiming));
    CLO_CUDA(cudaEventCreateWithFlags(&ev_join3_, cudaEventDisableTiming));
    ev_attn_.resize(L);
    ev_pref_.resize(L);
    ev_sel_.resize(L);
    for (int l = 0; l < L; ++l) {
        CLO_CUDA(cudaEventCreateWithFlags(&ev_attn_[l], cudaEventDisableTiming));
        CLO_CUDA(cudaEventCreateWithFlags(&ev_pref_[l], cudaEventDisableTiming));
        CLO_CUDA(cudaEventCreateWithFlags(&ev_sel_[l], cudaEventDisableTiming));
    }
    CLO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&desc_host_), sizeof(StepDesc) * kDescRing,
                           cudaHostAllocDefault));
    desc_ev_.resize(kDescRing);
    for (auto& ev : desc_ev_) CLO_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    desc_used_.assign(kDescRing, 0);
    CLO_CUDA(cudaDeviceSynchronize());
}

EngineView Engine::view() const {
    const clo_model_shape& s = cfg_.shape;
    EngineView v{};
    v.B = cfg_.batch;
    v.L = s.num_layers;
    v.H = s.num_kv_heads;
    v.HQ = s.num_q_heads;
    v.m = v.HQ / v.H;
    v.d = s.head_dim;
    v.k = cfg_.k;
    v.sink = cfg_.sink_tokens;
    v.recent = cfg_.recent_tokens;
    v.bits = cfg_.hash_bits;
    v.words = words_;
    v.nb = nb_;
    v.n_prompt = cfg_.n_prompt;
    v.nmax = nmax_;
    v.max_steps = std::max(cfg_.max_steps, 1);
    v.max_chunks = max_chunks_;
    v.retriever = cfg_.retriever;
    v.policy = cfg_.policy;
    v.always_miss = cfg_.always_miss;
    v.always_hit = cfg_.always_hit;
    v.has_tau_override = cfg_.has_tau_override;
    v.tau_override = cfg_.tau_override;
    v.kv_dtype = cfg_.kv_dtype;
    v.NP = np_;
    v.NO = no_;
    v.host_k = host_k_;
    v.host_v = host_v_;
    v.host_k_w = host_k_;
    v.host_v_w = host_v_;
    v.seq_stride = seq_stride_;
    v.layer_stride = layer_stride_;
    v.head_stride = head_stride_;
    v.row_stride = row_stride_ ? row_stride_ : cfg_.shape.head_dim;
    {
        const int64_t d = cfg_.shape.head_dim, esz = cfg_.kv_dtype == CLO_DTYPE_BF16 ? 2 : 4;
        v.kv_fused = host_k_ && v.row_stride == 2 * d &&
                     static_cast<const char*>(host_v_) == static_cast<const char*>(host_k_) + d * esz;
    }
    v.persistent = d_persistent_.as<int>();
    v.pidx = d_pidx_.as<int>();
    v.oidx = d_oidx_.as<int>();
    v.pk = d_pk_.p;
    v.pv = d_pv_.p;
    v.kmirror = d_kmirror_.p;
    v.slot_k = d_slot_k_.p;
    v.slot_v = d_slot_v_.p;
    v.win_k = d_win_k_.p;
    v.win_v = d_win_v_.p;
    v.entry_idx = d_entry_idx_.as<int32_t>();
    v.entry_slot = d_entry_slot_.as<int32_t>();
    v.slot_tok = d_slot_tok_.as<int32_t>();
    v.slot_age = d_slot_age_.as<int32_t>();
    v.tok2slot = d_tok2slot_.as<int32_t>();
    v.pool = pool_;
    v.vhead = d_vhead_.as<int>();
    v.codes = d_codes_.as<uint64_t>();
    v.code_stride = code_stride_;
    v.proj_t = d_proj_t_.as<double>();
    v.proj_w = d_proj_w_.as<double>();
    v.labels = d_labels_.as<double>();
    v.label_valid = d_label_valid_.as<int>();
    v.tau = d_tau_.as<double>();
    v.qimp = d_qimp_.as<double>();
    v.hits = d_hits_.as<unsigned long long>();
    v.misses = d_misses_.as<unsigned long long>();
    v.cache_last_update = d_cache_last_.as<int>();
    v.entry_last_update = d_entry_last_.as<int>();
    v.last_lookup_hit = d_last_hit_.as<int>();
    v.history = d_history_.as<double>();
    v.gathered_bytes = d_gathered_.as<unsigned long long>();
    v.dev_step = d_step_.as<int>();
    v.desc = d_desc_.as<StepDesc>();
    v.err = d_err_.as<int>();
    v.attn_part = d_attn_part_.as<float>();
    v.attn_count = d_attn_count_.as<int>();
    v.max_attn_chunks = max_attn_chunks_;
    {
        int* x = d_xfer_.as<int>();
        const int L = s.num_layers;
        v.xfer_ready = x;
        v.xfer_units = x + L;
        v.xfer_claim = x + 2 * L;
        v.xfer_done = x + 3 * L;
        v.xfer_flag = x + 4 * L;
    }
    v.world = world_;
    v.rank = rank_;
    v.xtimeout_ns = exchange_timeout_ns();
    if (d_tmaps_.p) {
        const char* tm = d_tmaps_.as<char>();
        v.tmap_k = tm;
        v.tmap_v = tm + sizeof(CUtensorMap);
        v.tmap_k32 = tm + 2 * sizeof(CUtensorMap);
        v.tmap_v32 = tm + 3 * sizeof(CUtensorMap);
    }
    v.HQg = world_ * s.num_q_heads;
    v.q0 = rank_ * s.num_q_heads;
    for (int r = 0; r < world_; ++r) {
        char* base = static_cast<char*>(xbase_[r]);
        v.xflag[r] = reinterpret_cast<unsigned*>(base);
        v.xslot[r] = reinterpret_cast<float*>(base + exchange_flag_bytes(s.num_layers));
    }
    return v;
}

SelArgs Engine::sel_args(int which, int layer) const {
    const clo_model_shape& s = cfg_.shape;
    const SelScratch& sc = which ? off_scratch(layer) : scratch_[0];
    SelArgs a{};
    a.items = sc.items + (size_t)layer * cfg_.batch * s.num_kv_heads;
    a.count = sc.count + layer;
    a.m = s.num_q_heads / s.num_kv_heads;
    a.d = s.head_dim;
    a.k = cfg_.k;
    a.bits = cfg_.hash_bits;
    a.words = words_;
    a.nb = nb_;
    a.nmax = nmax_;
    a.max_chunks = max_chunks_;
    a.dtype = cfg_.kv_dtype;
    a.q64 = sc.q64;
    a.qbits = sc.qbits;
    a.key16 = sc.key16;
    a.key64 = sc.key64;
    a.chunk_hist = sc.chunk_hist;
    a.chunk_base = sc.chunk_base;
    a.chunk_take = sc.chunk_take;
    a.thresh = sc.thresh;
    a.need = sc.need;
    a.radix_hist = sc.radix_hist;
    a.grid = grid_for((int64_t)cfg_.batch * s.num_kv_heads * max_chunks_);
    a.max_items = cfg_.batch * s.num_kv_heads;
    a.item_done = chained_select() >= 1 ? sc.item_done : nullptr;
    return a;
}

void Engine::prof_begin(cudaStream_t st) {
    if (capture_mode_ < 0) return;
    auto& recs = prof_[capture_mode_];
    size_t& used = prof_used_[capture_mode_];
    if (used == recs.size()) {
        ProfRec r{};
        CLO_CUDA(cudaEventCreate(&r.a));
        CLO_CUDA(cudaEventCreate(&r.b));
        recs.push_back(r);
    }
    CLO_CUDA(cudaEventRecordWithFlags(recs[used].a, st, cudaEventRecordExternal));
}

void Engine::prof_end(cudaStream_t st, const char* name, int layer) {
    if (capture_mode_ < 0) return;
    ProfRec& r = prof_[capture_mode_][prof_used_[capture_mode_]++];
    r.name = name;
    r.layer = layer;
    CLO_CUDA(cudaEventRecordWithFlags(r.b, st, cudaEventRecordExternal));
}

void Engine::drop_graphs() {  // views and pointers are baked into the graphs
    for (int m = 0; m < kGraphModes; ++m) {
        if (execs_[m]) cudaGraphExecDestroy(execs_[m]);
        if (graphs_[m]) cudaGraphDestroy(graphs_[m]);
        execs_[m] = nullptr;
        graphs_[m] = nullptr;
    }
}

OutputErrorArgs Engine::output_error_args() const {
    const size_t segs = (size_t)cfg_.batch * cfg_.shape.num_kv_heads;
    const size_t w = (size_t)cfg_.k + cfg_.sink_tokens + cfg_.recent_tokens;
    char* p = d_oerr_.as<char>();
    OutputErrorArgs a{};
    a.keys = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * segs * nmax_;
    a.scores = reinterpret_cast<double*>(p);
    p += sizeof(double) * segs * w;
    a.sel = reinterpret_cast<int32_t*>(p);
    p += sizeof(int32_t) * segs * w;
    a.uni = reinterpret_cast<int32_t*>(p);
    p += sizeof(int32_t) * segs * w;
    a.err = reinterpret_cast<double*>(p);
    return a;
}

double Engine::mean_output_error(int b) {  // DecodeMetrics::mean_output_error (engine.cpp:67-69)
    if (!cfg_.compute_oracle_error || steps_ == 0) return 0.0;
    const clo_model_shape& s = cfg_.shape;
    const size_t per = (size_t)s.num_layers * s.num_q_heads;
    std::vector<double> e(per);
    synchronize();
    CLO_CUDA(cudaMemcpy(e.data(), output_error_args().err + (size_t)b * per, sizeof(double) * per,
                        cudaMemcpyDeviceToHost));
    double sum = 0.0;
    for (double x : e) sum += x;  // fixed order: layer, query head
    return sum / (double)(per * steps_);
}

int Engine::chained_select() const {
    // CLO_CHAIN_SELECT=thr: the CTA finishing an item's last score chunk computes
    // its threshold (no threshold launch); =all: also the CTA finishing its last
    // compaction chunk reconciles it (no reconcile launch); 0: neither
    static const int mode = [] {
        const char* e = getenv("CLO_CHAIN_SELECT");
        if (!e) return 0;
        const std::string m(e);
        return m == "all" || m == "1" ? 2 : (m == "thr" ? 1 : 0);
    }();
    if (cfg_.retriever != CLO_RETRIEVER_SIGN_HASH) return 0;
    return mode == 2 && (size_t)cfg_.k * 16 > 200 * 1024 ? 1 : mode;
}

ReconcileArgs Engine::reconcile_args(int layer, int fresh) const {
    const SelScratch& sc = off_scratch(layer);
    const size_t items = (size_t)cfg_.batch * cfg_.shape.num_kv_heads;
    ReconcileArgs ra{};
    ra.v = view();
    ra.items = sc.items + (size_t)layer * items;
    ra.count = sc.count;
    ra.sel = sc.sel;
    ra.fetch_tok = sc.fetch_tok;
    ra.fetch_slot = sc.fetch_slot;
    ra.fetch_dem = sc.fetch_dem;
    ra.fetch_count = sc.fetch_count;
    ra.items_cap = (int)items;
    ra.layer = layer;
    ra.fresh = fresh;
    return ra;
}

void Engine::enqueue_select(int which, int layer, cudaStream_t st, bool with_reconcile) {
    SelArgs a = sel_args(which, layer);
    prof_begin(st);
    if (cfg_.retriever == CLO_RETRIEVER_SIGN_HASH) {
        // decode, offloaded heads, chained stages: the compaction kernel also
        // reconciles each item's entry (one launch instead of two)
        const ReconcileArgs ra = reconcile_args(layer, 0);
        launches_ += launch_select_signhash(a, st, with_reconcile && chained_select() == 2 ? &ra : nullptr);
    } else {
        launch_select_exact(a, st);
        launches_ += 21;
    }
    prof_end(st, which ? "select_offloaded" : "select_persistent", layer);
}

void Engine::enqueue_prepare(int which, int layer, int mode, int kind, cudaStream_t st) {
    PrepareArgs pa{};
    pa.v = view();
    pa.s = which ? off_scratch(layer) : scratch_[0];
    pa.s.items += (size_t)layer * cfg_.batch * cfg_.shape.num_kv_heads;
    pa.layer = layer;
    pa.mode = mode;
    pa.kind = kind;
    prof_begin(st);
    launch_prepare(pa, st);
    prof_end(st, which ? "lookup_offloaded" : "lookup_persistent", layer);
    launches_ += 1;
}

void Engine::enqueue_reconcile(int layer, int fresh, cudaStream_t st) {
    const ReconcileArgs ra = reconcile_args(layer, fresh);
    prof_begin(st);
    launch_reconcile(ra, st);  // demotions travel with the gather's moves
    prof_end(st, "reconcile", layer);
    launches_ += 1;
}

bool Engine::fused_select() const {
    static const bool off = [] {  // CLO_FUSED_SELECT=1: one cluster kernel per layer (experiment; slower on B200)
        const char* e = getenv("CLO_FUSED_SELECT");
        return !(e && e[0] == '1');
    }();
    return !off && cfg_.retriever == CLO_RETRIEVER_SIGN_HASH &&
           fused_select_fits(words_, nb_, cfg_.shape.num_q_heads / cfg_.shape.num_kv_heads, cfg_.shape.head_dim, cfg_.k,
                             nmax_);
}

void Engine::enqueue_fused_select(int layer, cudaStream_t st) {
    const size_t items = (size_t)cfg_.batch * cfg_.shape.num_kv_heads;
    FusedSelectArgs f{};
    f.prep.v = view();
    f.prep.s = off_scratch(layer);
    f.prep.s.items += (size_t)layer * items;
    f.prep.layer = layer;
    f.prep.mode = kPrepDecode;
    f.prep.kind = kKindOffloaded;
    f.sel = sel_args(1, layer);
    const SelScratch& sc = off_scratch(layer);
    f.rec.v = f.prep.v;
    f.rec.items = sc.items + (size_t)layer * items;
    f.rec.count = sc.count;
    f.rec.sel = sc.sel;
    f.rec.fetch_tok = sc.fetch_tok;
    f.rec.fetch_slot = sc.fetch_slot;
    f.rec.fetch_dem = sc.fetch_dem;
    f.rec.fetch_count = sc.fetch_count;
    f.rec.items_cap = (int)items;
    f.rec.layer = layer;
    f.rec.fresh = 0;
    prof_begin(st);
    launch_fused_select(f, st);
    prof_end(st, "select_offloaded", layer);
    launches_ += 1;
}

GatherEngineArgs Engine::gather_args(int layer, int count_bytes) const {
    const SelScratch& sc = scratch_[1];
    GatherEngineArgs ga{};
    ga.v = view();
    ga.items = sc.items;  // base of the per-layer work lists
    ga.count = sc.count;
    ga.fetch_tok = sc.fetch_tok;
    ga.fetch_slot = sc.fetch_slot;
    ga.fetch_dem = sc.fetch_dem;
    ga.fetch_count = sc.fetch_count;
    ga.items_cap = cfg_.batch * cfg_.shape.num_kv_heads;
    ga.layer = layer;
    ga.count_bytes = count_bytes;
    return ga;
}

void Engine::enqueue_gather(int layer, int count_bytes, cudaStream_t st) {
    const GatherEngineArgs ga = gather_args(layer, count_bytes);
    prof_begin(st);
    launch_gather_engine(ga, (int)gather_ctas(), st);  // picks the copy variant and its grid (gather.cu)
    prof_end(st, "gather_zero_copy", layer);
    launches_ += 1;
}

void Engine::bind_host_kv(void* k, void* v, int64_t seq_stride, int64_t layer_stride,
                          int64_t head_stride, int64_t row_stride) {
    if (!k || !v) fail(CLO_ERR_ARGUMENT, "host K/V pointers must be non-null");
    for (void* p : {k, v}) {
        cudaPointerAttributes at{};
        CLO_CUDA(cudaPointerGetAttributes(&at, p));
        if (at.type != cudaMemoryTypeHost)
            fail(CLO_ERR_ARGUMENT,
                 "host K/V must be pinned, UVA-mapped memory (clo_host_alloc or cudaHostRegister)");
    }
    if (prefilled_) fail(CLO_ERR_CONTRACT, "bind the host K/V store before prefill, not after");
    if (seq_stride < 0 || layer_stride < 0 || head_stride < 0) fail(CLO_ERR_ARGUMENT, "negative stride");
    const int d = cfg_.shape.head_dim;
    const int esz = cfg_.kv_dtype == CLO_DTYPE_BF16 ? 2 : 4;
    for (int64_t st : {seq_stride, layer_stride, head_stride})
        if (st * esz % 16 != 0) fail(CLO_ERR_ARGUMENT, "seq/layer/head strides must be multiples of 16 bytes");
    if (row_stride == 0) row_stride = d;
    if (row_stride < d) fail(CLO_ERR_ARGUMENT, "row_stride must be at least head_dim");
    if (row_stride * esz % 16 != 0) fail(CLO_ERR_ARGUMENT, "row_stride must be a multiple of 16 bytes");
    for (const void* p : {(const void*)k, (const void*)v})
        if (reinterpret_cast<uintptr_t>(p) % 16 != 0) fail(CLO_ERR_ARGUMENT, "host K/V must be 16-byte aligned");
    row_stride_ = row_stride;
    host_k_ = k;
    host_v_ = v;
    seq_stride_ = seq_stride;
    layer_stride_ = layer_stride;
    head_stride_ = head_stride;
    drop_graphs();  // pointers are baked into the graphs
}

namespace {
// Exchange handle: what a peer needs to map this engine's exchange buffer.
// Engines in the same process (same pid) share the pointer directly; other
// processes open the CUDA IPC handle (peer access over NVLink when the
// devices differ, a plain mapping when they share one).
struct ExchangeHandle {
    uint32_t magic;
    int32_t pid, device, rank, world, B, L, HQg, d;
    uint64_t base, bytes;
    cudaIpcMemHandle_t ipc;
};
constexpr uint32_t kExchangeMagic = 0xC10E8C01u;
static_assert(sizeof(ExchangeHandle) <= CLO_EXCHANGE_HANDLE_BYTES, "exchange handle too large");
}  // namespace

void Engine::peer_handle(int rank, int world, void* out) {
    const clo_model_shape& s = cfg_.shape;
    if (world < 1 || world > kMaxRanks) fail(CLO_ERR_CONFIG, "world must be in [1, 8]");
    if (rank < 0 || rank >= world) fail(CLO_ERR_ARGUMENT, "rank out of range");
    if (cfg_.kv_head_offset != rank * s.num_kv_heads)
        fail(CLO_ERR_CONFIG, "KV-head shards must be contiguous blocks: kv_head_offset != rank * num_kv_heads");
    if (steps_ > 0) fail(CLO_ERR_CONTRACT, "attach the exchange before the first decode step");
    CLO_CUDA(cudaSetDevice(cfg_.device));
    const int HQg = world * s.num_q_heads;
    const size_t bytes = exchange_flag_bytes(s.num_layers) +
                         sizeof(float) * 2 * (size_t)cfg_.batch * s.num_layers * HQg * s.head_dim;
    d_xbuf_.alloc(bytes);  // zeroed: counters start at 0
    d_out_.alloc(sizeof(float) * (size_t)cfg_.batch * s.num_layers * HQg * s.head_dim, false);
    world_ = 1;  // until attach_peers succeeds
    rank_ = rank;
    ExchangeHandle h{};
    h.magic = kExchangeMagic;
    h.pid = (int32_t)getpid();
    h.device = cfg_.device;
    h.rank = rank;
    h.world = world;
    h.B = cfg_.batch;
    h.L = s.num_layers;
    h.HQg = HQg;
    h.d = s.head_dim;
    h.base = (uint64_t)(uintptr_t)d_xbuf_.p;
    h.bytes = bytes;
    CLO_CUDA(cudaIpcGetMemHandle(&h.ipc, d_xbuf_.p));
    std::memset(out, 0, CLO_EXCHANGE_HANDLE_BYTES);
    std::memcpy(out, &h, sizeof h);
}

void Engine::attach_peers(const void* handles) {
    if (!d_xbuf_.p) fail(CLO_ERR_CONTRACT, "export this engine's exchange handle first");
    if (steps_ > 0) fail(CLO_ERR_CONTRACT, "attach the exchange before the first decode step");
    CLO_CUDA(cudaSetDevice(cfg_.device));
    ExchangeHandle self{};
    std::memcpy(&self, static_cast<const char*>(handles) + (size_t)rank_ * CLO_EXCHANGE_HANDLE_BYTES, sizeof self);
    if (self.magic != kExchangeMagic || self.base != (uint64_t)(uintptr_t)d_xbuf_.p)
        fail(CLO_ERR_ARGUMENT, "handles[rank] is not this engine's exchange handle");
    const int world = self.world;
    for (int r = 0; r < kMaxRanks; ++r)
        if (xipc_[r]) {
            cudaIpcCloseMemHandle(xbase_[r]);
            xipc_[r] = false;
        }
    xbase_.fill(nullptr);
    for (int r = 0; r < world; ++r) {
        ExchangeHandle h{};
        std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * CLO_EXCHANGE_HANDLE_BYTES, sizeof h);
        if (h.magic != kExchangeMagic) fail(CLO_ERR_ARGUMENT, "malformed exchange handle");
        if (h.rank != r || h.world != world || h.B != self.B || h.L != self.L || h.HQg != self.HQg || h.d != self.d)
            fail(CLO_ERR_CONFIG, "exchange handles disagree on rank order, world or output shape");
        if (r == rank_) {
            xbase_[r] = d_xbuf_.p;
        } else if (h.pid == self.pid) {  // same process: the pointer is valid here
            if (h.device != cfg_.device) {
                int ok = 0;
                CLO_CUDA(cudaDeviceCanAccessPeer(&ok, cfg_.device, h.device));
                if (!ok) fail(CLO_ERR_CUDA, "no peer access between the shards' devices");
                const cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CLO_CUDA(e);
                cudaGetLastError();
            }
            xbase_[r] = (void*)(uintptr_t)h.base;
        } else {
            void* p = nullptr;
            CLO_CUDA(cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
            xbase_[r] = p;
            xipc_[r] = true;
        }
    }
    world_ = world;
    drop_graphs();
}

void Engine::set_desc(const StepDesc& d, cudaStream_t st) {
    const int slot = desc_next_;
    desc_next_ = (desc_next_ + 1) % kDescRing;
    if (desc_used_[slot]) CLO_CUDA(cudaEventSynchronize(desc_ev_[slot]));
    desc_host_[slot] = d;
    CLO_CUDA(cudaMemcpyAsync(d_desc_.p, desc_host_ + slot, sizeof(StepDesc), cudaMemcpyHostToDevice, st));
    CLO_CUDA(cudaEventRecord(desc_ev_[slot], st));
    desc_used_[slot] = 1;
}

void Engine::prefill(const float* true_q0, int on_host, cudaStream_t user) {
    if (prefilled_) fail(CLO_ERR_CONTRACT, "prefill ran twice");
    if (!host_k_) fail(CLO_ERR_CONTRACT, "bind the host K/V store before prefill");
    if (!true_q0) fail(CLO_ERR_ARGUMENT, "true_q0 must be non-null");
    CLO_CUDA(cudaSetDevice(cfg_.device));
    const clo_model_shape& s = cfg_.shape;
    const int B = cfg_.batch, L = s.num_layers, H = s.num_kv_heads, HQ = s.num_q_heads, d = s.head_dim;
    const size_t esz = cfg_.kv_dtype == CLO_DTYPE_BF16 ? 2 : 4;
    const int n = cfg_.n_prompt;
    cudaStream_t st = s_main_;
    CLO_CUDA(cudaStreamSynchronize(user));

    // step-0 queries
    const size_t qbytes = sizeof(float) * B * L * HQ * d;
    const float* tq = true_q0;
    if (on_host) {
        CLO_CUDA(cudaMemcpyAsync(d_in_tq_.p, true_q0, qbytes, cudaMemcpyHostToDevice, st));
        tq = d_in_tq_.as<float>();
    }
    StepDesc desc{tq, tq, nullptr, nullptr, nullptr};
    set_desc(desc, st);
    CLO_CUDA(cudaMemsetAsync(d_err_.p, 0, sizeof(int), st));

    // Load prompt rows: stage each distinct host matrix once in HBM, encode its
    // sign bits for every layer that aliases it, fill persistent KV / K mirror.
    DevBuf stage_k, stage_v;
    stage_k.alloc((size_t)n * d * esz, false);
    stage_v.alloc((size_t)n * d * esz, false);
    std::vector<EncodeSeg> segs;
    DevBuf d_segs;
    d_segs.alloc(sizeof(EncodeSeg) * L);
    const char* hk = static_cast<const char*>(host_k_);
    const char* hv = static_cast<const char*>(host_v_);
    for (int b = 0; b < B; ++b)
        for (int g = 0; g < H; ++g) {
            int l0 = 0;
            while (l0 < L) {
                const int l1 = layer_stride_ == 0 ? L : l0 + 1;  // layers sharing this host buffer
                const size_t hoff = ((size_t)b * seq_stride_ + (size_t)l0 * layer_stride_ + (size_t)g * head_stride_) * esz;
                const size_t pitch = (size_t)(row_stride_ ? row_stride_ : d) * esz;
                CLO_CUDA(cudaMemcpy2DAsync(stage_k.p, (size_t)d * esz, hk + hoff, pitch, (size_t)d * esz, n,
                                           cudaMemcpyHostToDevice, st));
                CLO_CUDA(cudaMemcpy2DAsync(stage_v.p, (size_t)d * esz, hv + hoff, pitch, (size_t)d * esz, n,
                                           cudaMemcpyHostToDevice, st));
                launch_check_finite(stage_k.p, cfg_.kv_dtype, (int64_t)n * d, d_err_.as<int>(), kErrNonFiniteKey, st);
                launch_check_finite(stage_v.p, cfg_.kv_dtype, (int64_t)n * d, d_err_.as<int>(), kErrNonFiniteValue, st);
                launches_ += 2;
                segs.clear();
                for (int l = l0; l < l1; ++l) {
                    const int lg = l * H + g;
                    const size_t seg = ((size_t)b * L + l) * H + g;
                    if (cfg_.retriever == CLO_RETRIEVER_SIGN_HASH)
                        segs.push_back({stage_k.p, d_proj_t_.as<double>() + (size_t)lg * d * cfg_.hash_bits,
                                        d_codes_.as<uint64_t>() + seg * code_stride_});
                    if (persistent_[lg]) {
                        const size_t p = (size_t)b * np_ + pidx_[lg];
                        CLO_CUDA(cudaMemcpyAsync(d_pk_.as<char>() + p * nmax_ * d * esz, stage_k.p,
                                                 (size_t)n * d * esz, cudaMemcpyDeviceToDevice, st));
                        CLO_CUDA(cudaMemcpyAsync(d_pv_.as<char>() + p * nmax_ * d * esz, stage_v.p,
                                                 (size_t)n * d * esz, cudaMemcpyDeviceToDevice, st));
                    } else if (d_kmirror_.p) {
                        const size_t o = (size_t)b * no_ + oidx_[lg];
                        CLO_CUDA(cudaMemcpyAsync(d_kmirror_.as<char>() + o * nmax_ * d * esz, stage_k.p,
                                                 (size_t)n * d * esz, cudaMemcpyDeviceToDevice, st));
                    }
                }
                if (!segs.empty()) {
                    CLO_CUDA(cudaMemcpyAsync(d_segs.p, segs.data(), sizeof(EncodeSeg) * segs.size(),
                                             cudaMemcpyHostToDevice, st));
                    launch_encode(d_segs.as<EncodeSeg>(), (int)segs.size(), n, d, cfg_.hash_bits,
                                  cfg_.kv_dtype, d_err_.as<int>(), st);
                    launches_ += 1;
                }
                // the staging buffers and segs are reused: serialise
                CLO_CUDA(cudaStreamSynchronize(st));
                l0 = l1;
            }
        }
    launch_window_init(view(), st);
    launches_ += 1;

    // Step-0 selection with true queries (engine.cpp:188-201).
    for (int l = 0; l < L; ++l) {
        if (layer_has_off_[l]) {
            enqueue_prepare(1, l, kPrepPrefill, kKindOffloaded, st);
            enqueue_select(1, l, st);
            enqueue_reconcile(l, 1, st);
            enqueue_gather(l, 0, st);
        }
        if (layer_has_pers_[l]) {
            enqueue_prepare(0, l, kPrepPrefill, kKindPersistent, st);
            enqueue_select(0, l, st);
        }
    }
    for (int i = 0; i < 2; ++i) CLO_CUDA(cudaMemsetAsync(scratch_[i].count, 0, sizeof(int) * L, st));
    CLO_CUDA(cudaMemsetAsync(d_step_.p, 0, sizeof(int), st));
    CLO_CUDA(cudaStreamSynchronize(st));
    CLO_CUDA(cudaGetLastError());
    check_device_error();
    prefilled_ = true;
}

void Engine::capture_graph(int mode) {
    const clo_model_shape& s = cfg_.shape;
    const int L = s.num_layers;
    const uint64_t before = launches_;
    const bool profiled = mode == kGraphSerial;
    const bool flags = mode == kGraphProd && use_flag_transfer();
    capture_mode_ = mode == kGraphProd ? -1 : mode;
    prof_used_[mode] = 0;
    cudaGraph_t* graph_out = &graphs_[mode];
    cudaGraphExec_t* exec_out = &execs_[mode];
    // Three streams: selection (lookup + score/select of offloaded heads),
    // transfer (zero-copy gathers, back to back on the PCIe link) and compute
    // (persistent-head selection, append, attention). Work lists are per
    // layer, so the selection stream can run ahead of the transfer stream.
    // The instrumented (profiled) graph serialises everything on one stream so
    // each kernel's event-bracketed time is its own, not time spent queued
    // behind the other streams (the share of the step, like an ncu launch list).
    // CLO_SEL_STREAMS=2 (experiment): even layers' selections on one stream,
    // odd layers' on another, each with its own stage intermediates
    // (off_scratch), so the chain in front of gather(l) no longer queues
    // behind layer l-1's chain. On B200 it halves the link's wait for fetch
    // lists but the overlapping selection kernels slow the gathers and
    // attention by as much (1595 vs 1595 tokens/s, profiles/r2/experiments.jsonl).
    const bool dual = !profiled && !flags && sel_streams_ > 1;
    cudaStream_t s_pref_a = profiled ? s_main_ : s_pref_;
    cudaStream_t s_pref_b = dual ? s_pref2_ : s_pref_a;
    cudaStream_t s_xfer = profiled ? s_main_ : s_xfer_;
    CLO_CUDA(cudaStreamBeginCapture(s_main_, cudaStreamCaptureModeThreadLocal));
    if (mode == kGraphTimeline) {
        if (!tl_base_) CLO_CUDA(cudaEventCreate(&tl_base_));
        CLO_CUDA(cudaEventRecordWithFlags(tl_base_, s_main_, cudaEventRecordExternal));
    }
    CLO_CUDA(cudaEventRecord(ev_fork_, s_main_));
    if (!profiled) {
        CLO_CUDA(cudaStreamWaitEvent(s_pref_a, ev_fork_, 0));
        if (dual) CLO_CUDA(cudaStreamWaitEvent(s_pref_b, ev_fork_, 0));
        CLO_CUDA(cudaStreamWaitEvent(s_xfer, ev_fork_, 0));
        // one persistent transfer kernel per step streams every offloaded
        // layer's fetch list as soon as the selection stream publishes it
        if (n_off_layers_ > 0 && flags) {
            launch_gather_persistent(gather_args(0, 1), d_off_layers_.as<int>(), n_off_layers_,
                                     gather_ctas() > 0 ? (int)gather_ctas() : 48, s_xfer);
            launches_ += 1;
        }
    }
    for (int l = 0; l < L; ++l) {
        cudaStream_t s_pref = (l & 1) ? s_pref_b : s_pref_a;
        if (layer_has_off_[l]) {
            // The lookup/selection/transfer of layer l uses approximate queries,
            // available once layer l-1 starts, i.e. after attention(l-2):
            // it overlaps the compute of layer l-1 (speculative prefetch,
            // engine.cpp:246-251).
            if (l >= 2) CLO_CUDA(cudaStreamWaitEvent(s_pref, ev_attn_[l - 2], 0));
            if (fused_select()) {
                enqueue_fused_select(l, s_pref);  // lookup .. reconcile in one kernel (select_fused.cu)
            } else {
                enqueue_prepare(1, l, kPrepDecode, kKindOffloaded, s_pref);
                enqueue_select(1, l, s_pref, true);
                if (chained_select() < 2) enqueue_reconcile(l, 0, s_pref);
            }
            if (!flags) {
                // one gather launch per layer, ordered by graph edges
                CLO_CUDA(cudaEventRecord(ev_sel_[l], s_pref));
                CLO_CUDA(cudaStreamWaitEvent(s_xfer, ev_sel_[l], 0));
                enqueue_gather(l, 1, s_xfer);
                CLO_CUDA(cudaEventRecord(ev_pref_[l], s_xfer));
            } else {
                launch_publish(gather_args(l, 1), s_pref);  // device flag for the transfer kernel
                launches_ += 1;
            }
        }
        if (layer_has_pers_[l]) {
            enqueue_prepare(0, l, kPrepDecode, kKindPersistent, s_main_);
            enqueue_select(0, l, s_main_);
        }
        prof_begin(s_main_);
        launch_append(view(), l, s_main_);
        prof_end(s_main_, "append", l);
        if (layer_has_off_[l]) {  // layer l's rows must be in HBM before its attention
            if (flags) {
                launch_wait_flag(d_xfer_.as<int>() + 4 * cfg_.shape.num_layers + l, d_step_.as<int>(), s_main_);
                launches_ += 1;
            } else {
                CLO_CUDA(cudaStreamWaitEvent(s_main_, ev_pref_[l], 0));
            }
        }
        prof_begin(s_main_);
        if (!launch_attention_mma(view(), l, s_main_) && !launch_attention_tma(view(), l, s_main_))
            launch_attention_engine(view(), l, s_main_);
        prof_end(s_main_, "attention", l);
        launches_ += 2;
        CLO_CUDA(cudaEventRecord(ev_attn_[l], s_main_));
    }
    if (!profiled) {
        CLO_CUDA(cudaEventRecord(ev_join_, s_pref_a));
        CLO_CUDA(cudaStreamWaitEvent(s_main_, ev_join_, 0));
        if (dual) {
            CLO_CUDA(cudaEventRecord(ev_join3_, s_pref_b));
            CLO_CUDA(cudaStreamWaitEvent(s_main_, ev_join3_, 0));
        }
        CLO_CUDA(cudaEventRecord(ev_join2_, s_xfer));
        CLO_CUDA(cudaStreamWaitEvent(s_main_, ev_join2_, 0));
    }
    if (world_ > 1) {  // peers' head outputs of this step -> out (exchange.cuh)
        prof_begin(s_main_);
        launch_exchange_finish(view(), s_main_);
        prof_end(s_main_, "exchange_finish", -1);
        launches_ += 2;
    }
    if (cfg_.compute_oracle_error) {  // engine.cpp:257-267, 394-405: exact-top-k output error
        const OutputErrorArgs oa = output_error_args();
        for (int l = 0; l < L; ++l) launch_output_error(view(), l, oa, s_main_);
        launches_ += L;
    }
    launch_step_end(view(), scratch_[0].count, scratch_[1].count, s_main_);
    launches_ += 1;
    CLO_CUDA(cudaStreamEndCapture(s_main_, graph_out));
    capture_mode_ = -1;
    CLO_CUDA(cudaGraphInstantiate(exec_out, *graph_out, 0));
    launches_ = before;  // captured launches are counted per replay
    size_t nn = 0;
    CLO_CUDA(cudaGraphGetNodes(*graph_out, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CLO_CUDA(cudaGraphGetNodes(*graph_out, nodes.data(), &nn));
    int kn = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        CLO_CUDA(cudaGraphNodeGetType(nd, &t));
        kn += t == cudaGraphNodeTypeKernel;
    }
    if (mode == kGraphProd) kernels_per_step_ = kn;  // the production graph's kernel count
}

StepDesc Engine::make_desc(const clo_step_io& io, cudaStream_t user) {
    const clo_model_shape& s = cfg_.shape;
    const int B = cfg_.batch, L = s.num_layers, H = s.num_kv_heads, HQ = s.num_q_heads, d = s.head_dim;
    const size_t esz = cfg_.kv_dtype == CLO_DTYPE_BF16 ? 2 : 4;
    StepDesc desc{};
    if (io.on_host) {
        // Inputs go through a double-buffered staging slot on the copy stream:
        // this step's H2D overlaps the previous step's graph (only the graph
        // that read this slot two steps ago must have finished), and the
        // step's graph waits for its own copies.
        const size_t qb = sizeof(float) * B * L * HQ * d, kb = esz * B * L * H * d;
        if (!s_copy_) {  // created on first host-buffer step: device-I/O engines keep 3 streams
            CLO_CUDA(cudaStreamCreateWithFlags(&s_copy_, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                CLO_CUDA(cudaEventCreateWithFlags(&ev_in_[i], cudaEventDisableTiming));
                CLO_CUDA(cudaEventCreateWithFlags(&ev_free_[i], cudaEventDisableTiming));
            }
        }
        const int slot = in_slot_;
        in_slot_ ^= 1;
        if (in_used_[slot]) CLO_CUDA(cudaStreamWaitEvent(s_copy_, ev_free_[slot], 0));
        char* base = d_in_[slot].as<char>();
        CLO_CUDA(cudaMemcpyAsync(base, io.true_q, qb, cudaMemcpyHostToDevice, s_copy_));
        CLO_CUDA(cudaMemcpyAsync(base + qb, io.approx_q, qb, cudaMemcpyHostToDevice, s_copy_));
        CLO_CUDA(cudaMemcpyAsync(base + 2 * qb, io.new_k, kb, cudaMemcpyHostToDevice, s_copy_));
        CLO_CUDA(cudaMemcpyAsync(base + 2 * qb + kb, io.new_v, kb, cudaMemcpyHostToDevice, s_copy_));
        CLO_CUDA(cudaEventRecord(ev_in_[slot], s_copy_));
        CLO_CUDA(cudaStreamWaitEvent(user, ev_in_[slot], 0));
        pending_free_ = slot;
        desc.true_q = reinterpret_cast<const float*>(base);
        desc.approx_q = reinterpret_cast<const float*>(base + qb);
        desc.new_k = base + 2 * qb;
        desc.new_v = base + 2 * qb + kb;
        desc.out = d_out_.as<float>();
    } else {
        desc.true_q = io.true_q;
        desc.approx_q = io.approx_q;
        desc.new_k = io.new_k;
        desc.new_v = io.new_v;
        desc.out = io.out ? io.out : d_out_.as<float>();
    }
    return desc;
}

void Engine::launch_step(int mode, const clo_step_io& io, cudaStream_t user) {
    if (!prefilled_) fail(CLO_ERR_CONTRACT, "decode_step before prefill");
    if (steps_ >= cfg_.max_steps) fail(CLO_ERR_CONTRACT, "decode_step past the end of the workload");
    if (!io.true_q || !io.approx_q || !io.new_k || !io.new_v)
        fail(CLO_ERR_ARGUMENT, "step inputs must be non-null");
    CLO_CUDA(cudaSetDevice(cfg_.device));
    const clo_model_shape& s = cfg_.shape;
    // Steps may be issued on different streams: each one reads the single
    // device descriptor and mutates shared engine state, so step t+1 waits
    // for step t's graph wherever it was launched.
    if (!ev_step_) CLO_CUDA(cudaEventCreateWithFlags(&ev_step_, cudaEventDisableTiming));
    if (step_stream_set_ && step_stream_ != user) CLO_CUDA(cudaStreamWaitEvent(user, ev_step_, 0));
    set_desc(make_desc(io, user), user);
    if (!execs_[mode]) capture_graph(mode);
    CLO_CUDA(cudaGraphLaunch(execs_[mode], user));
    CLO_CUDA(cudaEventRecord(ev_step_, user));
    step_stream_ = user;
    step_stream_set_ = true;
    launches_ += kernels_per_step_;
    if (pending_free_ >= 0) {  // the staging slot is reusable once this graph is done
        CLO_CUDA(cudaEventRecord(ev_free_[pending_free_], user));
        in_used_[pending_free_] = true;
        pending_free_ = -1;
    }
    if (io.on_host && io.out)
        CLO_CUDA(cudaMemcpyAsync(io.out, d_out_.p,
                                 sizeof(float) * cfg_.batch * s.num_layers * world_ * s.num_q_heads * s.head_dim,
                                 cudaMemcpyDeviceToHost, user));
    CLO_CUDA(cudaGetLastError());
    ++steps_;
}

std::vector<clo_kernel_time> Engine::profile_step(const clo_step_io& io, cudaStream_t user) {
    if (!execs_[kGraphProd] && prefilled_) capture_graph(kGraphProd);  // kernels_per_step_
    launch_step(kGraphSerial, io, user);
    CLO_CUDA(cudaStreamSynchronize(user));
    check_device_error();
    std::vector<clo_kernel_time> out;
    const auto& recs = prof_[kGraphSerial];
    for (size_t i = 0; i < prof_used_[kGraphSerial]; ++i) {
        clo_kernel_time kt{};
        std::snprintf(kt.name, sizeof kt.name, "%s", recs[i].name);
        kt.layer = recs[i].layer;
        CLO_CUDA(cudaEventElapsedTime(&kt.ms, recs[i].a, recs[i].b));
        out.push_back(kt);
    }
    return out;
}

// Measured LayerTiming (pipeline_sim.hpp:61-72) of one step, from the
// timeline graph's event timestamps (production streams, so overlap is real):
//   compute   = append + attention           (the compute stream's own work)
//   transfer  = the layer's zero-copy gather (raw, before overlap)
//   exposed   = how long attention(l) waited for its gather after the compute
//               stream was ready (append(l) done), capped at transfer
//   hidden    = transfer - exposed          (overlapped with earlier layers)
//   mgmt      = lookup (+ fused label refresh) + reconcile (entry bookkeeping)
//   retrieval = scoring + top-k selection
//   sync      = 0: GPU-centric, no host round trip inside the step
//   total     = compute + exposed + mgmt + sync + retrieval (schedule_layer's
//               formula, pipeline_sim.cpp:39); wall = the measured layer-to-
//               layer time on the compute stream (selection and transfer
//               overlap it, so wall < total when the pipeline works).
void Engine::timeline_step(const clo_step_io& io, cudaStream_t user) {
    if (!execs_[kGraphProd] && prefilled_) capture_graph(kGraphProd);
    launch_step(kGraphTimeline, io, user);
    CLO_CUDA(cudaStreamSynchronize(user));
    check_device_error();
    const int L = cfg_.shape.num_layers;
    if (timeline_.empty()) {
        timeline_.assign(L, clo_layer_timing{});
        for (int l = 0; l < L; ++l) timeline_[l].layer = l;
    }
    struct Span {
        double a = -1, b = -1;
    };
    auto at = [&](cudaEvent_t ev) {
        float ms = 0.f;
        CLO_CUDA(cudaEventElapsedTime(&ms, tl_base_, ev));
        return (double)ms * 1e-3;
    };
    std::vector<std::array<double, 4>> dur(L);                    // compute, transfer, mgmt, retrieval
    std::vector<Span> append(L), attn(L), gather(L);
    for (auto& d : dur) d.fill(0.0);
    const auto& recs = prof_[kGraphTimeline];
    spans_.clear();
    for (size_t i = 0; i < prof_used_[kGraphTimeline]; ++i) {
        const ProfRec& r = recs[i];
        const double a = at(r.a), b = at(r.b), d = b - a;
        clo_kernel_span sp{};
        std::snprintf(sp.name, sizeof sp.name, "%s", r.name);
        sp.layer = r.layer;
        sp.start_ms = (float)(a * 1e3);
        sp.end_ms = (float)(b * 1e3);
        spans_.push_back(sp);
        if (r.layer < 0 || r.layer >= L) continue;
        const std::string n = r.name;
        if (n == "append") {
            dur[r.layer][0] += d;
            append[r.layer] = {a, b};
        } else if (n == "attention") {
            dur[r.layer][0] += d;
            attn[r.layer] = {a, b};
        } else if (n == "gather_zero_copy") {
            dur[r.layer][1] += d;
            gather[r.layer] = {a, b};
        } else if (n.rfind("lookup", 0) == 0 || n == "reconcile") {
            dur[r.layer][2] += d;
        } else if (n.rfind("select", 0) == 0) {
            dur[r.layer][3] += d;
        }
    }
    for (int l = 0; l < L; ++l) {
        clo_layer_timing& t = timeline_[l];
        const double transfer = dur[l][1];
        double exposed = 0.0;
        if (gather[l].b >= 0 && append[l].b >= 0 && attn[l].a >= 0)
            exposed = std::min(transfer, std::max(0.0, attn[l].a - append[l].b));
        t.compute_s += dur[l][0];
        t.transfer_s += transfer;
        t.exposed_s += exposed;
        t.hidden_s += transfer - exposed;
        t.mgmt_s += dur[l][2];
        t.retrieval_s += dur[l][3];
        t.total_s += dur[l][0] + exposed + dur[l][2] + dur[l][3];
        const double prev = l > 0 ? attn[l - 1].b : 0.0;
        t.wall_s += attn[l].b >= 0 ? attn[l].b - prev : 0.0;
    }
    ++timeline_steps_;
}

std::string Engine::timeline_json() const {
    // breakdown_to_json's schema (pipeline_sim.cpp:115-135): "transfer_s" there
    // is the EXPOSED transfer; raw transfer and the wall clock are extra keys.
    char buf[64];
    auto num = [&](double v) {
        std::snprintf(buf, sizeof buf, "%.12g", v);
        return std::string(buf);
    };
    auto row = [&](const clo_layer_timing& t) {
        return "\"compute_s\": " + num(t.compute_s) + ", \"transfer_s\": " + num(t.exposed_s) +
               ", \"hidden_s\": " + num(t.hidden_s) + ", \"mgmt_s\": " + num(t.mgmt_s) +
               ", \"sync_s\": " + num(t.sync_s) + ", \"retrieval_s\": " + num(t.retrieval_s) +
               ", \"total_s\": " + num(t.total_s) + ", \"transfer_raw_s\": " + num(t.transfer_s) +
               ", \"wall_s\": " + num(t.wall_s);
    };
    clo_layer_timing tot{};
    std::string out = "{\n  \"steps\": " + std::to_string(timeline_steps_) + ",\n  \"layers\": [";
    for (size_t l = 0; l < timeline_.size(); ++l) {
        const clo_layer_timing& t = timeline_[l];
        out += (l ? ",\n    {" : "\n    {") + std::string("\"layer\": ") + std::to_string(t.layer) + ", " + row(t) + "}";
        tot.compute_s += t.compute_s;
        tot.transfer_s += t.transfer_s;
        tot.hidden_s += t.hidden_s;
        tot.exposed_s += t.exposed_s;
        tot.mgmt_s += t.mgmt_s;
        tot.sync_s += t.sync_s;
        tot.retrieval_s += t.retrieval_s;
        tot.total_s += t.total_s;
        tot.wall_s += t.wall_s;
    }
    out += "\n  ],\n  \"total\": {" + row(tot) + "}\n}\n";
    return out;
}

void Engine::decode_step(const clo_step_io& io, cudaStream_t user) { launch_step(kGraphProd, io, user); }

void Engine::synchronize() {
    CLO_CUDA(cudaSetDevice(cfg_.device));
    CLO_CUDA(cudaDeviceSynchronize());
    check_device_error();
}

void Engine::check_device_error() {
    int err = 0;
    CLO_CUDA(cudaMemcpy(&err, d_err_.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (!err) return;
    CLO_CUDA(cudaMemset(d_err_.p, 0, sizeof(int)));
    if (err & kErrNonFiniteQuery) fail(CLO_ERR_NUMERIC, "non-finite query entry");
    if (err & kErrNonFiniteKey) fail(CLO_ERR_NUMERIC, "non-finite key entry");
    if (err & kErrNonFiniteValue) fail(CLO_ERR_NUMERIC, "non-finite value entry");
    if (err & kErrContract) fail(CLO_ERR_CONTRACT, "device-side contract violation");
    if (err & kErrAlias)
        fail(CLO_ERR_CONTRACT,
             "layer_stride 0 aliases one host K/V store across layers, but a step's new K/V rows differ "
             "between layers");
    if (err & kErrExchange)
        fail(CLO_ERR_CUDA, "head-output exchange timed out: a peer rank stopped stepping");
    fail(CLO_ERR_INTERNAL, "device-side error flag " + std::to_string(err));
}

uint64_t Engine::entry_bytes() const {
    return 2ull * (uint64_t)cfg_.k * cfg_.shape.head_dim * cfg_.shape.bytes_per_element;
}

int Engine::held_tokens() const {  // SinkRecentBuffer::held_tokens (similarity_cache.cpp:113-118)
    const int n = cfg_.n_prompt + steps_;
    const int sink = std::min(n, cfg_.sink_tokens);
    return sink + std::min(n - sink, cfg_.recent_tokens);
}

template <typename T>
static std::vector<T> fetch(const DevBuf& b, size_t count, size_t offset = 0) {
    std::vector<T> out(count);
    if (count) CLO_CUDA(cudaMemcpy(out.data(), b.as<T>() + offset, sizeof(T) * count, cudaMemcpyDeviceToHost));
    return out;
}

clo_metrics Engine::metrics() {
    synchronize();
    const clo_model_shape& s = cfg_.shape;
    const size_t segs = (size_t)cfg_.batch * s.num_layers * s.num_kv_heads;
    auto hits = fetch<unsigned long long>(d_hits_, segs);
    auto misses = fetch<unsigned long long>(d_misses_, segs);
    auto gathered = fetch<unsigned long long>(d_gathered_, 1);
    clo_metrics m{};
    m.steps = steps_;
    for (size_t i = 0; i < segs; ++i) {
        m.hits += hits[i];
        m.misses += misses[i];
    }
    m.lookups = m.hits + m.misses;
    m.hit_ratio = m.lookups ? (double)m.hits / (double)m.lookups : 0.0;
    m.transferred_bytes = m.misses * entry_bytes();
    m.persistent_bytes = (uint64_t)cfg_.batch * np_ * steps_ * entry_bytes();
    m.gathered_bytes_device = gathered[0];
    const uint64_t rows = (uint64_t)cfg_.n_prompt + steps_;
    const uint64_t row_bytes = 2ull * s.head_dim * s.bytes_per_element;
    m.host_bytes = (uint64_t)no_ * rows * row_bytes;
    m.device_persistent_bytes = (uint64_t)np_ * rows * row_bytes;
    m.cache_bytes_current =
        steps_ == 0 ? 0
                    : clo_cache_bytes(no_, cfg_.k, no_ ? held_tokens() : 0, s.num_layers, s.num_q_heads,
                                      s.head_dim, s.bytes_per_element);
    m.sync_mode = sync_mode_;
    m.mean_output_error = 0.0;
    for (int b = 0; b < cfg_.batch; ++b) m.mean_output_error += mean_output_error(b) / cfg_.batch;
    return m;
}

clo_head_state Engine::head_state(int b, int l, int g, int32_t* entry_indices, double* history) {
    const clo_model_shape& s = cfg_.shape;
    if (b < 0 || b >= cfg_.batch || l < 0 || l >= s.num_layers || g < 0 || g >= s.num_kv_heads)
        fail(CLO_ERR_INDEX, "head out of range");
    synchronize();
    const size_t seg = ((size_t)b * s.num_layers + l) * s.num_kv_heads + g;
    const int lg = l * s.num_kv_heads + g;
    const int m = s.num_q_heads / s.num_kv_heads;
    clo_head_state st{};
    st.placement = persistent_[lg] ? CLO_PLACEMENT_PERSISTENT : CLO_PLACEMENT_OFFLOADED;
    st.hits = fetch<unsigned long long>(d_hits_, 1, seg)[0];
    st.misses = fetch<unsigned long long>(d_misses_, 1, seg)[0];
    st.transferred_bytes = persistent_[lg] ? 0 : st.misses * entry_bytes();
    st.persistent_bytes = persistent_[lg] ? steps_ * entry_bytes() : 0;
    st.last_update_step = fetch<int>(d_cache_last_, 1, seg)[0];
    st.entry_last_update_step = fetch<int>(d_entry_last_, 1, seg)[0];
    auto valid = fetch<int>(d_label_valid_, m, ((size_t)b * s.num_layers + l) * s.num_q_heads + (size_t)g * m);
    st.labels_valid = 0;
    for (int v : valid) st.labels_valid += v != 0;
    st.window_held_tokens = persistent_[lg] ? 0 : held_tokens();
    const bool has_history = !persistent_[lg] && cfg_.policy == CLO_POLICY_SIMILARITY;
    st.n_history = has_history ? steps_ : 0;
    if (entry_indices) {
        auto idx = fetch<int32_t>(d_entry_idx_, cfg_.k, seg * cfg_.k);
        std::copy(idx.begin(), idx.end(), entry_indices);
    }
    if (history && st.n_history) {
        auto h = fetch<double>(d_history_, st.n_history, seg * std::max(cfg_.max_steps, 1));
        std::copy(h.begin(), h.end(), history);
    }
    return st;
}

void Engine::entry_rows(int b, int l, int g, void* k_rows, void* v_rows) {
    const clo_model_shape& s = cfg_.shape;
    if (b < 0 || b >= cfg_.batch || l < 0 || l >= s.num_layers || g < 0 || g >= s.num_kv_heads)
        fail(CLO_ERR_INDEX, "head out of range");
    const int lg = l * s.num_kv_heads + g;
    if (persistent_[lg]) fail(CLO_ERR_ARGUMENT, "persistent heads have no cache entry");
    synchronize();
    const size_t esz = cfg_.kv_dtype == CLO_DTYPE_BF16 ? 2 : 4;
    const size_t bytes = (size_t)cfg_.k * s.head_dim * esz;
    const size_t o = (size_t)b * no_ + oidx_[lg];
    // CacheEntry::k_rows/v_rows are in entry (ascending index) order; the
    // head's row pool holds them at arbitrary slots, entry_slot maps them back.
    auto slot_of = fetch<int32_t>(d_entry_slot_, cfg_.k, o * cfg_.k);
    const size_t rb = (size_t)s.head_dim * esz;
    const size_t pool_bytes = (size_t)pool_ * rb;
    std::vector<char> tmp(pool_bytes);
    (void)bytes;
    for (int which = 0; which < 2; ++which) {
        void* dst = which ? v_rows : k_rows;
        if (!dst) continue;
        const DevBuf& src = which ? d_slot_v_ : d_slot_k_;
        CLO_CUDA(cudaMemcpy(tmp.data(), src.as<char>() + o * pool_bytes, pool_bytes, cudaMemcpyDeviceToHost));
        for (int i = 0; i < cfg_.k; ++i)
            std::memcpy(static_cast<char*>(dst) + (size_t)i * rb, tmp.data() + (size_t)slot_of[i] * rb, rb);
    }
}

static void json_num(std::ostringstream& os, double v) {
    char buf[64];
    if (v == std::floor(v) && std::fabs(v) < 1e15) {
        std::snprintf(buf, sizeof buf, "%.1f", v);
    } else {
        std::snprintf(buf, sizeof buf, "%.17g", v);
    }
    os << buf;
}

std::string Engine::cache_state_json(int b) {
    // engine.cpp:464-530, same keys and nesting.
    const clo_model_shape& s = cfg_.shape;
    if (b < 0 || b >= cfg_.batch) fail(CLO_ERR_INDEX, "sequence out of range");
    clo_metrics tot{};
    {
        synchronize();
        const size_t L = s.num_layers, H = s.num_kv_heads;
        auto hits = fetch<unsigned long long>(d_hits_, L * H, (size_t)b * L * H);
        auto misses = fetch<unsigned long long>(d_misses_, L * H, (size_t)b * L * H);
        for (size_t i = 0; i < L * H; ++i) {
            tot.hits += hits[i];
            tot.misses += misses[i];
        }
    }
    clo_metrics all = metrics();
    const uint64_t lookups = tot.hits + tot.misses;
    std::ostringstream os;
    os << "{\n  \"policy\": \"" << (cfg_.policy == CLO_POLICY_SIMILARITY ? "similarity" : "prefetch_only")
       << "\",\n  \"sync_mode\": \"" << (sync_mode_ == CLO_SYNC_GPU_CENTRIC ? "gpu_centric" : "cpu_centric")
       << "\",\n  \"k\": " << cfg_.k << ",\n  \"sink_tokens\": " << cfg_.sink_tokens
       << ",\n  \"recent_tokens\": " << cfg_.recent_tokens << ",\n  \"steps_run\": " << steps_
       << ",\n  \"totals\": {\n    \"hits\": " << tot.hits << ",\n    \"misses\": " << tot.misses
       << ",\n    \"hit_ratio\": ";
    json_num(os, lookups ? (double)tot.hits / (double)lookups : 0.0);
    os << ",\n    \"transferred_bytes\": " << tot.misses * entry_bytes()
       << ",\n    \"persistent_served_bytes\": " << (uint64_t)np_ * steps_ * entry_bytes()
       << ",\n    \"cache_bytes\": " << all.cache_bytes_current << ",\n    \"host_bytes\": " << all.host_bytes
       << ",\n    \"device_persistent_bytes\": " << all.device_persistent_bytes << ",\n    \"mean_output_error\": ";
    json_num(os, mean_output_error(b));  // this sequence's DecodeMetrics::mean_output_error
    os << "\n  },\n  \"layers\": [";
    std::vector<int32_t> idx(cfg_.k);
    std::vector<double> hist(std::max(cfg_.max_steps, 1));
    for (int l = 0; l < s.num_layers; ++l) {
        os << (l ? "," : "") << "\n    {\n      \"layer\": " << l << ",\n      \"heads\": [";
        for (int g = 0; g < s.num_kv_heads; ++g) {
            clo_head_state st = head_state(b, l, g, idx.data(), hist.data());
            const bool off = st.placement == CLO_PLACEMENT_OFFLOADED;
            os << (g ? "," : "") << "\n        {\n          \"kv_head\": " << g << ",\n          \"placement\": \""
               << (off ? "offloaded" : "persistent") << "\",\n          \"hits\": " << st.hits
               << ",\n          \"misses\": " << st.misses << ",\n          \"transferred_bytes\": "
               << st.transferred_bytes << ",\n          \"persistent_served_bytes\": " << st.persistent_bytes;
            if (off) {
                os << ",\n          \"window_held_tokens\": " << st.window_held_tokens;
                if (cfg_.policy == CLO_POLICY_SIMILARITY) {
                    os << ",\n          \"entry_indices\": [";
                    for (int i = 0; i < cfg_.k; ++i) os << (i ? ", " : "") << idx[i];
                    os << "],\n          \"entry_last_update_step\": " << st.entry_last_update_step
                       << ",\n          \"labels_valid\": " << st.labels_valid
                       << ",\n          \"aggregated_history\": [";
                    for (int i = 0; i < st.n_history; ++i) {
                        if (i) os << ", ";
                        json_num(os, hist[i]);
                    }
                    os << "]";
                }
            }
            os << "\n        }";
        }
        os << "\n      ]\n    }";
    }
    os << "\n  ]\n}";
    return os.str();
}

}  // namespace clo
