// abi.cpp — the C-ABI (include/clo.h): engine entry points, op-level entry
// points and the host-side pure functions of the path.
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cerrno>
#include <cstdio>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include <numbers>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "attention.cuh"
#include "encode.cuh"
#include "engine.hpp"
#include "gather.cuh"
#include "host_common.hpp"
#include "lookup.cuh"
#include "select.cuh"

namespace clo {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

// rng.hpp:11-22 (splitmix64 seed derivation).
static uint64_t mix1(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t mix_seed3(uint64_t base, uint64_t a, uint64_t b) {
    const uint64_t ba = mix1(base ^ mix1(a));
    return mix1(ba ^ mix1(b + 0x6a09e667f3bcc909ULL));
}

// encode()'s projection (retrieval.cpp:73-74, fill_normal rng.hpp:24-27):
// the host's libstdc++ mt19937_64 + normal_distribution<double>, the same
// implementation-defined generator the reference links against.
void sign_hash_projection(int hash_bits, int d, uint64_t seed, double* out) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> dist(0.0, 1.0);
    const size_t n = (size_t)hash_bits * d;
    for (size_t i = 0; i < n; ++i) out[i] = dist(gen);
}

namespace {

struct Stream {
    cudaStream_t s;
    explicit Stream(void* p) : s(static_cast<cudaStream_t>(p)) {}
};

void require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        fail(CLO_ERR_CUDA, "no CUDA device: the CLO path has no CPU fallback");
}

// Device error word for synchronous op-level validation.
struct OpErr {
    DevBuf buf;
    OpErr() { buf.alloc(sizeof(int)); }
    int read(cudaStream_t s) {
        int v = 0;
        CLO_CUDA(cudaMemcpyAsync(&v, buf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CLO_CUDA(cudaStreamSynchronize(s));
        return v;
    }
    int* ptr() { return buf.as<int>(); }
};

int dsize(int dtype) {
    if (dtype == CLO_DTYPE_BF16) return 2;
    if (dtype == CLO_DTYPE_F32) return 4;
    if (dtype == CLO_DTYPE_F64) return 8;
    fail(CLO_ERR_ARGUMENT, "unknown dtype");
}

DevBuf* upload_projection_t(int bits, int d, uint64_t seed, DevBuf* buf) {
    std::vector<double> p((size_t)bits * d), pt((size_t)bits * d);
    sign_hash_projection(bits, d, seed, p.data());
    for (int b = 0; b < bits; ++b)
        for (int c = 0; c < d; ++c) pt[(size_t)c * bits + b] = p[(size_t)b * d + c];
    buf->alloc(sizeof(double) * pt.size(), false);
    CLO_CUDA(cudaMemcpy(buf->p, pt.data(), sizeof(double) * pt.size(), cudaMemcpyHostToDevice));
    return buf;
}

}  // namespace

}  // namespace clo

using namespace clo;

extern "C" {

void clo_engine_config_defaults(clo_engine_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->shape.head_dim = 128;
    c->shape.bytes_per_element = 2;
    c->sink_tokens = 4;
    c->recent_tokens = 64;
    c->retriever = CLO_RETRIEVER_EXACT;
    c->hash_bits = 256;
    c->retriever_seed = 1;
    c->policy = CLO_POLICY_SIMILARITY;
    c->sync_override = -1;
    c->batch = 1;
    c->kv_dtype = CLO_DTYPE_BF16;
    c->victim_rows = -1;
}

const char* clo_last_error(void) { return g_last_error.c_str(); }

const char* clo_build_info(void) {
    return "clo-b200 abi=1 arch=sm_100a kernels=prepare,score_signhash,threshold_signhash,"
           "compact,score_exact,radix,gather_zero_copy,append,attention_split_k,encode";
}

clo_status clo_engine_create(const clo_engine_config* cfg, const double* tau,
                             const double* q_importance, const int* persistent, clo_engine** out) {
    return guarded([&] {
        if (!cfg || !tau || !q_importance || !persistent || !out)
            fail(CLO_ERR_ARGUMENT, "null argument");
        *out = reinterpret_cast<clo_engine*>(new Engine(*cfg, tau, q_importance, persistent));
    });
}

void clo_engine_destroy(clo_engine* e) { delete reinterpret_cast<Engine*>(e); }

#define ENG reinterpret_cast<Engine*>(e)

clo_status clo_engine_bind_host_kv(clo_engine* e, void* k, void* v, int64_t seq_stride,
                                   int64_t layer_stride, int64_t head_stride) {
    return guarded([&] { ENG->bind_host_kv(k, v, seq_stride, layer_stride, head_stride, 0); });
}

clo_status clo_engine_bind_host_kv_ex(clo_engine* e, void* k, void* v, int64_t seq_stride, int64_t layer_stride,
                                      int64_t head_stride, int64_t row_stride) {
    return guarded([&] { ENG->bind_host_kv(k, v, seq_stride, layer_stride, head_stride, row_stride); });
}

clo_status clo_prefill(clo_engine* e, const float* true_q0, int on_host, void* stream) {
    return guarded([&] { ENG->prefill(true_q0, on_host, static_cast<cudaStream_t>(stream)); });
}

clo_status clo_decode_step(clo_engine* e, const clo_step_io* io, void* stream) {
    return guarded([&] {
        if (!io) fail(CLO_ERR_ARGUMENT, "null step io");
        ENG->decode_step(*io, static_cast<cudaStream_t>(stream));
    });
}

clo_status clo_engine_synchronize(clo_engine* e) {
    return guarded([&] { ENG->synchronize(); });
}

clo_status clo_get_metrics(clo_engine* e, clo_metrics* out) {
    return guarded([&] { *out = ENG->metrics(); });
}

clo_status clo_get_head_state(clo_engine* e, int seq, int layer, int kv_head, clo_head_state* st,
                              int32_t* entry_indices, double* aggregated_history) {
    return guarded([&] { *st = ENG->head_state(seq, layer, kv_head, entry_indices, aggregated_history); });
}

clo_status clo_get_entry_rows(clo_engine* e, int seq, int layer, int kv_head, void* k_rows,
                              void* v_rows) {
    return guarded([&] { ENG->entry_rows(seq, layer, kv_head, k_rows, v_rows); });
}

clo_status clo_cache_state_json(clo_engine* e, int seq, char* buf, size_t cap, size_t* needed) {
    return guarded([&] {
        std::string s = ENG->cache_state_json(seq);
        if (needed) *needed = s.size() + 1;
        if (buf && cap) {
            const size_t n = std::min(cap - 1, s.size());
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
        }
    });
}

clo_status clo_engine_profile_step(clo_engine* e, const clo_step_io* io, void* stream,
                                   clo_kernel_time* out, int cap, int* count) {
    return guarded([&] {
        if (!io) fail(CLO_ERR_ARGUMENT, "null step io");
        auto recs = ENG->profile_step(*io, static_cast<cudaStream_t>(stream));
        const int n = (int)std::min<size_t>(recs.size(), cap > 0 ? (size_t)cap : 0);
        for (int i = 0; i < n; ++i) out[i] = recs[i];
        if (count) *count = (int)recs.size();
    });
}

clo_status clo_engine_timeline_step(clo_engine* e, const clo_step_io* io, void* stream) {
    return guarded([&] {
        if (!e || !io) fail(CLO_ERR_ARGUMENT, "null argument");
        reinterpret_cast<Engine*>(e)->timeline_step(*io, static_cast<cudaStream_t>(stream));
    });
}

clo_status clo_get_timeline(clo_engine* e, clo_layer_timing* per_layer, int cap, clo_layer_timing* totals,
                            uint64_t* steps) {
    return guarded([&] {
        if (!e) fail(CLO_ERR_ARGUMENT, "null engine");
        const Engine* en = reinterpret_cast<Engine*>(e);
        const auto& tl = en->timeline();
        const int L = en->config().shape.num_layers;
        if (per_layer && cap < L) fail(CLO_ERR_ARGUMENT, "per_layer needs num_layers entries");
        clo_layer_timing tot{};
        tot.layer = -1;
        for (int l = 0; l < L; ++l) {
            clo_layer_timing t{};
            t.layer = l;
            if (!tl.empty()) t = tl[l];
            if (per_layer) per_layer[l] = t;
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
        if (totals) *totals = tot;
        if (steps) *steps = en->timeline_steps();
    });
}

clo_status clo_timeline_spans(clo_engine* e, clo_kernel_span* out, int cap, int* count) {
    return guarded([&] {
        if (!e) fail(CLO_ERR_ARGUMENT, "null engine");
        const auto& sp = reinterpret_cast<Engine*>(e)->last_spans();
        if (count) *count = (int)sp.size();
        for (int i = 0; out && i < cap && i < (int)sp.size(); ++i) out[i] = sp[i];
    });
}

clo_status clo_timeline_json(clo_engine* e, char* buf, size_t cap, size_t* needed) {
    return guarded([&] {
        if (!e) fail(CLO_ERR_ARGUMENT, "null engine");
        const std::string js = reinterpret_cast<Engine*>(e)->timeline_json();
        if (needed) *needed = js.size() + 1;
        if (buf && cap) {
            const size_t n = std::min(js.size(), cap - 1);
            std::memcpy(buf, js.data(), n);
            buf[n] = 0;
        }
    });
}

uint64_t clo_engine_kernel_launches(const clo_engine* e) {
    return reinterpret_cast<const Engine*>(e)->launches();
}

int clo_engine_kernels_per_step(const clo_engine* e) {
    return reinterpret_cast<const Engine*>(e)->kernels_per_step();
}

clo_status clo_engine_exchange_handle(clo_engine* e, int rank, int world, void* handle_out) {
    return guarded([&] {
        if (!e || !handle_out) fail(CLO_ERR_ARGUMENT, "null argument");
        reinterpret_cast<Engine*>(e)->peer_handle(rank, world, handle_out);
    });
}

clo_status clo_engine_attach_peers(clo_engine* e, const void* handles) {
    return guarded([&] {
        if (!e || !handles) fail(CLO_ERR_ARGUMENT, "null argument");
        reinterpret_cast<Engine*>(e)->attach_peers(handles);
    });
}

// ----------------------------------------------------------------- host memory

namespace {
// Hugepage-backed pinned allocations (mmap + MADV_HUGEPAGE + cudaHostRegister):
// random 256-byte row reads spread over hundreds of MiB per head otherwise pay
// GPU TLB misses on 4 KiB sysmem mappings.
std::mutex g_huge_mu;
std::unordered_map<void*, size_t> g_huge;
}  // namespace

clo_status clo_host_alloc_numa(size_t bytes, int flags, int numa_node, void** out) {
    return guarded([&] {
        require_device();
        if (!(flags & CLO_HOST_HUGEPAGES) && numa_node < 0) {
            CLO_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
            return;
        }
        const size_t page = (flags & CLO_HOST_HUGEPAGES) ? size_t(2) << 20 : size_t(4) << 10;
        const size_t len = (bytes + page - 1) / page * page;
        void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) fail(CLO_ERR_IO, "mmap of the host K/V store failed");
        if (flags & CLO_HOST_HUGEPAGES) madvise(p, len, MADV_HUGEPAGE);
        if (numa_node >= 0) {
            // mbind(MPOL_BIND) through the raw syscall (no libnuma in the image):
            // the pages are allocated on `numa_node` when first touched below
            constexpr int kMaxNodes = 1024;
            if (numa_node >= kMaxNodes) {
                munmap(p, len);
                fail(CLO_ERR_ARGUMENT, "numa_node out of range");
            }
            unsigned long mask[kMaxNodes / (8 * sizeof(unsigned long))] = {};
            mask[numa_node / (8 * sizeof(unsigned long))] |= 1ul << (numa_node % (8 * sizeof(unsigned long)));
            constexpr int kMpolBind = 2;
            if (syscall(SYS_mbind, p, len, kMpolBind, mask, (unsigned long)kMaxNodes, 0u) != 0) {
                munmap(p, len);
                fail(CLO_ERR_IO, "mbind of the host K/V store to NUMA node " + std::to_string(numa_node) +
                                     " failed: " + std::strerror(errno));
            }
        }
        // fault the pages in (under the NUMA policy) before pinning, from
        // several threads: a store of tens of GB takes seconds on one core
        {
            const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
            const size_t per = (len / nt + page - 1) / page * page;
            std::vector<std::thread> th;
            for (unsigned i = 0; i < nt; ++i) {
                const size_t a = i * per, b = std::min(len, a + per);
                if (a < b) th.emplace_back([=] { std::memset(static_cast<char*>(p) + a, 0, b - a); });
            }
            for (auto& t : th) t.join();
        }
        cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
        if (e != cudaSuccess) {
            munmap(p, len);
            cuda_check(e, "cudaHostRegister(hugepage store)");
        }
        std::lock_guard<std::mutex> lk(g_huge_mu);
        g_huge[p] = len;
        *out = p;
    });
}

clo_status clo_host_alloc_ex(size_t bytes, int flags, void** out) {
    return clo_host_alloc_numa(bytes, flags, -1, out);
}

clo_status clo_host_alloc(size_t bytes, void** out) { return clo_host_alloc_ex(bytes, 0, out); }

clo_status clo_device_numa_node(int device, int* node) {
    return guarded([&] {
        if (!node) fail(CLO_ERR_ARGUMENT, "node must be non-null");
        require_device();
        char bus[32] = {};
        CLO_CUDA(cudaDeviceGetPCIBusId(bus, sizeof bus, device));
        for (char* c = bus; *c; ++c) *c = (char)std::tolower((unsigned char)*c);
        *node = -1;
        const std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
        if (FILE* f = std::fopen(path.c_str(), "r")) {
            int v = -1;
            if (std::fscanf(f, "%d", &v) == 1) *node = v;
            std::fclose(f);
        }
    });
}

clo_status clo_host_free(void* p) {
    return guarded([&] {
        size_t len = 0;
        {
            std::lock_guard<std::mutex> lk(g_huge_mu);
            auto it = g_huge.find(p);
            if (it != g_huge.end()) {
                len = it->second;
                g_huge.erase(it);
            }
        }
        if (len) {
            CLO_CUDA(cudaHostUnregister(p));
            munmap(p, len);
        } else {
            CLO_CUDA(cudaFreeHost(p));
        }
    });
}
clo_status clo_host_register(void* p, size_t bytes) {
    return guarded([&] {
        require_device();
        CLO_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    });
}
clo_status clo_host_unregister(void* p) {
    return guarded([&] { CLO_CUDA(cudaHostUnregister(p)); });
}

// ------------------------------------------------------------------- op-level

clo_status clo_sign_hash_projection(int hash_bits, int d, uint64_t seed, double* out_host) {
    return guarded([&] {
        if (hash_bits <= 0 || hash_bits % 8 != 0) fail(CLO_ERR_ARGUMENT, "hash_bits must be a positive multiple of 8");
        if (d <= 0) fail(CLO_ERR_SHAPE, "width must be positive");
        sign_hash_projection(hash_bits, d, seed, out_host);
    });
}

clo_status clo_encode_sign_hash(const void* keys_dev, int dtype, int64_t n, int d, int hash_bits,
                                uint64_t seed, uint64_t* codes_dev, void* stream) {
    return guarded([&] {
        require_device();
        if (hash_bits <= 0 || hash_bits % 8 != 0) fail(CLO_ERR_ARGUMENT, "hash_bits must be a positive multiple of 8");
        if (hash_bits > 512) fail(CLO_ERR_CONFIG, "hash_bits above 512 are not supported");
        if (d <= 0 || d > kMaxHeadDim) fail(CLO_ERR_SHAPE, "unsupported key width");
        dsize(dtype);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf pt, segs;
        upload_projection_t(hash_bits, d, seed, &pt);
        EncodeSeg sg{keys_dev, pt.as<double>(), codes_dev};
        segs.alloc(sizeof(EncodeSeg), false);
        CLO_CUDA(cudaMemcpy(segs.p, &sg, sizeof sg, cudaMemcpyHostToDevice));
        OpErr err;
        launch_encode(segs.as<EncodeSeg>(), 1, n, d, hash_bits, dtype, err.ptr(), s);
        CLO_CUDA(cudaGetLastError());
        if (err.read(s) & kErrNonFiniteKey) fail(CLO_ERR_NUMERIC, "non-finite key entry");
    });
}

clo_status clo_group_topk(const double* queries_dev, int m, int d, int retriever,
                          const void* keys_dev, int dtype, const uint64_t* codes_dev,
                          int hash_bits, uint64_t seed, int64_t n, int k, int32_t* out_idx_dev,
                          double* out_score_dev, void* stream) {
    return guarded([&] {
        require_device();
        if (k <= 0) fail(CLO_ERR_ARGUMENT, "k must be positive");
        if (k > n) fail(CLO_ERR_ARGUMENT, "k exceeds the number of encoded keys");
        if (m <= 0 || m > kMaxGroup) fail(CLO_ERR_ARGUMENT, "group size must be in [1, 16]");
        if (d <= 0 || d > kMaxHeadDim) fail(CLO_ERR_SHAPE, "unsupported query width");
        if (n > (int64_t)1 << 30) fail(CLO_ERR_ARGUMENT, "too many keys");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int words = (hash_bits + 63) / 64;
        const int max_chunks = (int)((n + kScoreChunk - 1) / kScoreChunk);
        DevBuf items, count, qbits, keys, hist, base, take, thresh, need, radix, pt;
        SelItem it{0, (int)n, keys_dev, codes_dev, out_idx_dev, out_score_dev};
        items.alloc(sizeof(SelItem), false);
        CLO_CUDA(cudaMemcpy(items.p, &it, sizeof it, cudaMemcpyHostToDevice));
        count.alloc(sizeof(int), false);
        const int one = 1;
        CLO_CUDA(cudaMemcpy(count.p, &one, sizeof one, cudaMemcpyHostToDevice));
        SelArgs a{};
        a.items = items.as<SelItem>();
        a.count = count.as<int>();
        a.m = m;
        a.d = d;
        a.k = k;
        a.nmax = (int)n;
        a.max_chunks = max_chunks;
        a.dtype = dtype;
        a.q64 = queries_dev;
        a.grid = std::min(max_chunks, kNumSMs * 8);
        a.max_items = 1;
        base.alloc(sizeof(int) * max_chunks, false);
        take.alloc(sizeof(int) * max_chunks, false);
        thresh.alloc(sizeof(uint64_t));
        need.alloc(sizeof(int));
        a.chunk_base = base.as<int>();
        a.chunk_take = take.as<int>();
        a.thresh = thresh.as<uint64_t>();
        a.need = need.as<int>();
        if (retriever == CLO_RETRIEVER_SIGN_HASH) {
            if (hash_bits <= 0 || hash_bits % 8 != 0) fail(CLO_ERR_ARGUMENT, "hash_bits must be a positive multiple of 8");
            if (hash_bits > 512) fail(CLO_ERR_CONFIG, "hash_bits above 512 are not supported");
            if (!codes_dev) fail(CLO_ERR_ARGUMENT, "sign-hash retrieval needs codes");
            upload_projection_t(hash_bits, d, seed, &pt);
            qbits.alloc(sizeof(uint64_t) * m * words);
            launch_hash_queries(queries_dev, m, d, pt.as<double>(), hash_bits, words, qbits.as<uint64_t>(), s);
            keys.alloc(sizeof(uint16_t) * n, false);
            a.bits = hash_bits;
            a.words = words;
            a.nb = hash_bits + 1;
            a.qbits = qbits.as<uint64_t>();
            a.key16 = keys.as<uint16_t>();
            hist.alloc(sizeof(uint32_t) * max_chunks * a.nb, false);
            a.chunk_hist = hist.as<uint32_t>();
            launch_select_signhash(a, s);
        } else if (retriever == CLO_RETRIEVER_EXACT) {
            if (!keys_dev) fail(CLO_ERR_ARGUMENT, "exact retrieval needs keys");
            dsize(dtype);
            keys.alloc(sizeof(uint64_t) * n, false);
            a.key64 = keys.as<uint64_t>();
            hist.alloc(sizeof(uint32_t) * max_chunks * 2, false);
            a.chunk_hist = hist.as<uint32_t>();
            radix.alloc(sizeof(uint32_t) * 256);
            a.radix_hist = radix.as<uint32_t>();
            launch_select_exact(a, s);
        } else {
            fail(CLO_ERR_ARGUMENT, "unknown retriever");
        }
        CLO_CUDA(cudaGetLastError());
        CLO_CUDA(cudaStreamSynchronize(s));
    });
}

clo_status clo_topk_select_exact(const double* q_dev, const void* keys_dev, int dtype, int64_t n,
                                 int d, int k, int32_t* out_idx_dev, void* stream) {
    // attention.cpp:71-89 — the exact retriever with one query.
    return clo_group_topk(q_dev, 1, d, CLO_RETRIEVER_EXACT, keys_dev, dtype, nullptr, 0, 0, n, k,
                          out_idx_dev, nullptr, stream);
}

clo_status clo_merge_group_topk(const int* sizes_host, int m, const int32_t* idx_dev,
                                const double* score_dev, int k, int32_t* out_idx_dev,
                                void* stream) {
    // similarity_cache.cpp:180-201 over arbitrary proposals: union keyed by
    // index with the best score, then the same exact top-k machinery over a
    // dense (score, index) table.
    return guarded([&] {
        require_device();
        if (k <= 0) fail(CLO_ERR_ARGUMENT, "k must be positive");
        if (m <= 0) fail(CLO_ERR_ARGUMENT, "no proposals to merge");
        int total = 0;
        for (int j = 0; j < m; ++j) total += sizes_host[j];
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        std::vector<int32_t> idx(total);
        std::vector<double> sc(total);
        if (total) {
            CLO_CUDA(cudaMemcpyAsync(idx.data(), idx_dev, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, s));
            CLO_CUDA(cudaMemcpyAsync(sc.data(), score_dev, sizeof(double) * total, cudaMemcpyDeviceToHost, s));
            CLO_CUDA(cudaStreamSynchronize(s));
        }
        // Union with first-inserted-then-raised best score (std::map semantics).
        std::vector<std::pair<int32_t, double>> u;
        {
            std::vector<int> order(total);
            for (int i = 0; i < total; ++i) order[i] = i;
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return idx[a] < idx[b]; });
            for (int i : order) {
                if (!u.empty() && u.back().first == idx[i]) {
                    if (sc[i] > u.back().second) u.back().second = sc[i];
                } else {
                    u.push_back({idx[i], sc[i]});
                }
            }
        }
        if ((int)u.size() < k) fail(CLO_ERR_ARGUMENT, "merged union smaller than k");
        // Rank on the device: a dense key table where row r is union member r;
        // the exact selector orders by (score desc, row asc) = (score desc, index asc)
        // because u is index-sorted. Row numbers map back to indices.
        const int n = (int)u.size();
        std::vector<double> keys(n);
        for (int i = 0; i < n; ++i) keys[i] = u[i].second;
        DevBuf dkeys, dq, dout;
        dkeys.alloc(sizeof(double) * n, false);
        dq.alloc(sizeof(double), false);
        dout.alloc(sizeof(int32_t) * k, false);
        const double one = 1.0;
        CLO_CUDA(cudaMemcpy(dkeys.p, keys.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
        CLO_CUDA(cudaMemcpy(dq.p, &one, sizeof one, cudaMemcpyHostToDevice));
        clo_status st = clo_group_topk(dq.as<double>(), 1, 1, CLO_RETRIEVER_EXACT, dkeys.p, CLO_DTYPE_F64,
                                       nullptr, 0, 0, n, k, dout.as<int32_t>(), nullptr, stream);
        if (st != CLO_OK) fail(st, g_last_error);
        std::vector<int32_t> rows(k);
        CLO_CUDA(cudaMemcpy(rows.data(), dout.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
        for (int i = 0; i < k; ++i) rows[i] = u[rows[i]].first;  // rows ascending => indices ascending
        CLO_CUDA(cudaMemcpy(out_idx_dev, rows.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice));
    });
}

clo_status clo_lookup(int n_heads, int m, int d, double* labels_dev, int32_t* label_valid_dev,
                      const double* queries_dev, const double* weights_dev, const double* tau_dev,
                      int32_t* hit_dev, double* agg_dev, double* sims_dev, int32_t* reason_dev,
                      void* stream) {
    return guarded([&] {
        require_device();
        if (m <= 0) fail(CLO_ERR_ARGUMENT, "empty lookup group");
        if (m > kMaxGroup) fail(CLO_ERR_ARGUMENT, "group size above 16");
        if (n_heads <= 0) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // weights must be non-negative (aggregate_similarity :14-15), checked up front
        std::vector<double> w((size_t)n_heads * m);
        CLO_CUDA(cudaMemcpyAsync(w.data(), weights_dev, sizeof(double) * w.size(), cudaMemcpyDeviceToHost, s));
        CLO_CUDA(cudaStreamSynchronize(s));
        for (double x : w)
            if (x < 0.0) fail(CLO_ERR_ARGUMENT, "importance weights must be non-negative");
        launch_lookup_op(n_heads, m, d, labels_dev, label_valid_dev, queries_dev, weights_dev, tau_dev,
                         hit_dev, agg_dev, sims_dev, reason_dev, s);
        CLO_CUDA(cudaGetLastError());
        CLO_CUDA(cudaStreamSynchronize(s));
    });
}

clo_status clo_cosine_similarity(int n_pairs, int d, const double* a_dev, const double* b_dev,
                                 double* value_dev, int32_t* degenerate_dev, void* stream) {
    return guarded([&] {
        require_device();
        if (d <= 0) fail(CLO_ERR_ARGUMENT, "cosine of empty vectors");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (n_pairs > 0) launch_cosine_op(n_pairs, d, a_dev, b_dev, value_dev, degenerate_dev, s);
        CLO_CUDA(cudaGetLastError());
        CLO_CUDA(cudaStreamSynchronize(s));
    });
}

clo_status clo_aggregate_similarity(int n_groups, int m, const double* sims_dev,
                                    const double* weights_dev, double* out_dev, void* stream) {
    return guarded([&] {
        require_device();
        if (m <= 0) fail(CLO_ERR_SHAPE, "similarity and weight counts must match and be non-empty");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        OpErr err;
        if (n_groups > 0) launch_aggregate_op(n_groups, m, sims_dev, weights_dev, out_dev, err.ptr(), s);
        CLO_CUDA(cudaGetLastError());
        const int e = err.read(s);
        if (e & 1) fail(CLO_ERR_ARGUMENT, "importance weights must be non-negative");
        if (e & 2) fail(CLO_ERR_ARGUMENT, "aggregation requires strictly positive similarities");
    });
}

clo_status clo_gather_rows(const void* src, int dtype, int d, int64_t n_rows,
                           const int32_t* idx_dev, int k, void* dst_dev, void* stream) {
    return guarded([&] {
        require_device();
        const int row_bytes = d * dsize(dtype);
        if (row_bytes % 16 != 0) fail(CLO_ERR_SHAPE, "rows must be a multiple of 16 bytes");
        if (k < 0) fail(CLO_ERR_ARGUMENT, "negative row count");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        OpErr err;
        if (k > 0) launch_gather_op(src, dst_dev, idx_dev, row_bytes, k, n_rows, err.ptr(), 0, s);
        CLO_CUDA(cudaGetLastError());
        if (err.read(s) & kErrIndexRange) fail(CLO_ERR_INDEX, "matrix row out of range");
    });
}

clo_status clo_gather_rows_ex(const void* src, int dtype, int d, int64_t n_rows,
                              const int32_t* idx_dev, int k, void* dst_dev, int engine, int ctas,
                              int* err_dev, void* stream) {
    return guarded([&] {
        const int row_bytes = d * dsize(dtype);
        if (row_bytes % 16 != 0) fail(CLO_ERR_SHAPE, "rows must be a multiple of 16 bytes");
        if (!err_dev) fail(CLO_ERR_ARGUMENT, "err_dev must be a device int");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (k <= 0) return;
        if (engine == 1)
            launch_gather_tma_op(src, dst_dev, idx_dev, row_bytes, k, n_rows, err_dev, ctas > 0 ? ctas : 64, s);
        else
            launch_gather_op(src, dst_dev, idx_dev, row_bytes, k, n_rows, err_dev, ctas, s);
        CLO_CUDA(cudaGetLastError());
    });
}

clo_status clo_gather_rows_cpu_staged(const void* src_host, int dtype, int d, int64_t n_rows,
                                      const int32_t* idx_host, int k, void* staging_host,
                                      void* dst_dev, int threads, void* stream) {
    return guarded([&] {
        require_device();
        const size_t row_bytes = (size_t)d * dsize(dtype);
        for (int i = 0; i < k; ++i)
            if (idx_host[i] < 0 || idx_host[i] >= n_rows) fail(CLO_ERR_INDEX, "matrix row out of range");
        threads = std::max(1, threads);
        std::vector<std::thread> pool;
        const char* src = static_cast<const char*>(src_host);
        char* stg = static_cast<char*>(staging_host);
        for (int w = 0; w < threads; ++w)
            pool.emplace_back([&, w] {
                for (int i = w; i < k; i += threads)
                    std::memcpy(stg + (size_t)i * row_bytes, src + (size_t)idx_host[i] * row_bytes, row_bytes);
            });
        for (auto& t : pool) t.join();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        CLO_CUDA(cudaMemcpyAsync(dst_dev, staging_host, (size_t)k * row_bytes, cudaMemcpyHostToDevice, s));
    });
}

clo_status clo_topk_attention(const double* q_dev, int m, const void* keys_dev,
                              const void* values_dev, int dtype, int64_t n, int d,
                              const int32_t* idx_dev, int nidx, double* out_dev, void* stream) {
    return guarded([&] {
        require_device();
        if (n == 0) fail(CLO_ERR_ARGUMENT, "attention over an empty sequence");
        if (d <= 0) fail(CLO_ERR_SHAPE, "query width does not match key width");
        if (m <= 0) fail(CLO_ERR_ARGUMENT, "no queries");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        OpErr err;
        // check_qkv (attention.cpp:11-23): the full finiteness scan, in order q, K, V.
        launch_check_finite(q_dev, CLO_DTYPE_F64, (int64_t)m * d, err.ptr(), kErrNonFiniteQuery, s);
        launch_check_finite(keys_dev, dtype, n * d, err.ptr(), kErrNonFiniteKey, s);
        launch_check_finite(values_dev, dtype, n * d, err.ptr(), kErrNonFiniteValue, s);
        int e = err.read(s);
        if (e & kErrNonFiniteQuery) fail(CLO_ERR_NUMERIC, "non-finite query entry");
        if (e & kErrNonFiniteKey) fail(CLO_ERR_NUMERIC, "non-finite key entry");
        if (e & kErrNonFiniteValue) fail(CLO_ERR_NUMERIC, "non-finite value entry");
        if (nidx <= 0) fail(CLO_ERR_ARGUMENT, "empty attention index set");
        DevBuf bitmap;
        bitmap.alloc(sizeof(uint32_t) * ((n + 31) / 32));
        launch_validate_indices(idx_dev, nidx, n, bitmap.as<uint32_t>(), err.ptr(), s);
        e = err.read(s);
        if (e & kErrIndexRange) fail(CLO_ERR_INDEX, "attention index out of range");
        if (e & kErrDuplicate) fail(CLO_ERR_ARGUMENT, "duplicate attention index");
        DevBuf scratch;
        scratch.alloc(sizeof(double) * (size_t)m * nidx, false);
        launch_attention_op(q_dev, m, keys_dev, values_dev, dtype, d, idx_dev, nidx, out_dev,
                            scratch.as<double>(), s);
        CLO_CUDA(cudaGetLastError());
        CLO_CUDA(cudaStreamSynchronize(s));
    });
}

// ------------------------------------------------------------ host functions

clo_status clo_sink_recent_indices(int n, int sink_count, int recent_count, int32_t* out,
                                   int* count, int* clamped) {
    return guarded([&] {  // attention.cpp:107-128
        if (n <= 0) fail(CLO_ERR_ARGUMENT, "sequence must be non-empty");
        if (sink_count < 0 || recent_count < 0) fail(CLO_ERR_ARGUMENT, "window sizes must be non-negative");
        bool cut = false;
        int sink = sink_count, recent = recent_count;
        if (sink > n) {
            sink = n;
            cut = true;
        }
        if (recent > n) {
            recent = n;
            cut = true;
        }
        int c = 0;
        for (int i = 0; i < sink; ++i) out[c++] = i;
        for (int i = std::max(n - recent, sink); i < n; ++i) out[c++] = i;
        *count = c;
        if (clamped) *clamped = cut;
    });
}

clo_status clo_compute_threshold(double s, double eta, double p, double* tau) {
    return guarded([&] {  // head_profile.cpp:17-25
        if (!(s >= 0.0 && s <= 1.0)) fail(CLO_ERR_ARGUMENT, "importance must lie in [0, 1]");
        if (!(eta > -1.0 && eta <= 1.0)) fail(CLO_ERR_ARGUMENT, "eta must lie in (-1, 1]");
        if (!(p >= 1.0)) fail(CLO_ERR_ARGUMENT, "p must be at least 1");
        const double theta_star = std::acos(eta);
        const double lambda = std::pow(s, p);
        const double theta = lambda * theta_star + (1.0 - lambda) * std::numbers::pi;
        *tau = std::cos(theta);
    });
}

clo_status clo_compute_difficulty(double tau, double s_hat, double epsilon, double* out) {
    return guarded([&] {  // head_profile.cpp:27-30
        if (!(epsilon > 0.0)) fail(CLO_ERR_ARGUMENT, "epsilon must be positive");
        *out = tau - (s_hat - epsilon);
    });
}

clo_status clo_plan_partition(const double* difficulty, int L, int H, double t_comp_s,
                              double pcie_bw, double mem_head_bytes,
                              uint64_t persist_bytes_per_head, uint64_t hbm_budget_bytes,
                              int* persistent_out, int* n_p_out, int* n_dropped_out) {
    return guarded([&] {  // head_profile.cpp:80-154
        if (L <= 0) fail(CLO_ERR_ARGUMENT, "plan_partition: empty head-profile list");
        if (!(t_comp_s > 0.0) || !(pcie_bw > 0.0) || !(mem_head_bytes > 0.0))
            fail(CLO_ERR_ARGUMENT, "plan_partition: every cost term must be > 0");
        const int n_p = (int)std::floor(t_comp_s * pcie_bw / mem_head_bytes);
        std::fill(persistent_out, persistent_out + (size_t)L * H, 0);
        for (int l = 0; l < L; ++l) {
            if (l == 0) {
                for (int h = 0; h < H; ++h) persistent_out[h] = 1;
                continue;
            }
            std::vector<int> pos;
            for (int h = 0; h < H; ++h)
                if (difficulty[(size_t)l * H + h] > 0.0) pos.push_back(h);
            const int n_persist = std::max((int)pos.size() - n_p, 0);
            std::sort(pos.begin(), pos.end(), [&](int a, int b) {
                const double da = difficulty[(size_t)l * H + a], db = difficulty[(size_t)l * H + b];
                if (da != db) return da > db;
                return a < b;
            });
            pos.resize(n_persist);
            for (int h : pos) persistent_out[(size_t)l * H + h] = 1;
        }
        const uint64_t layer0 = (uint64_t)H * persist_bytes_per_head;
        if (hbm_budget_bytes > 0 && layer0 > hbm_budget_bytes)
            fail(CLO_ERR_CONFIG, "plan_partition: the layer-0 heads alone exceed the HBM budget");
        int dropped = 0;
        if (hbm_budget_bytes > 0) {
            for (;;) {
                uint64_t total = 0;
                for (size_t i = 0; i < (size_t)L * H; ++i)
                    if (persistent_out[i]) total += persist_bytes_per_head;
                if (total <= hbm_budget_bytes) break;
                int dl = -1, dh = -1;
                for (int l = 1; l < L; ++l)
                    for (int h = 0; h < H; ++h) {
                        if (!persistent_out[(size_t)l * H + h]) continue;
                        if (dl < 0 || difficulty[(size_t)l * H + h] < difficulty[(size_t)dl * H + dh]) {
                            dl = l;
                            dh = h;
                        }
                    }
                if (dl < 0) fail(CLO_ERR_CONFIG, "plan_partition: no plan fits the HBM budget, even without optional persistent heads");
                persistent_out[(size_t)dl * H + dh] = 0;
                ++dropped;
            }
        }
        *n_p_out = n_p;
        if (n_dropped_out) *n_dropped_out = dropped;
    });
}

uint64_t clo_cache_bytes(int offloaded_heads, int entry_k, int held_window_tokens, int num_layers,
                         int num_q_heads, int head_dim, int bytes_per_element) {
    // similarity_cache.cpp:167-178
    const uint64_t per_entry = 2ull * entry_k * head_dim * bytes_per_element;
    const uint64_t per_window = 2ull * held_window_tokens * head_dim * bytes_per_element;
    const uint64_t labels = (uint64_t)num_layers * num_q_heads * head_dim * bytes_per_element;
    return (uint64_t)offloaded_heads * (per_entry + per_window) + labels;
}

}  // extern "C"
