/*
 * clo.h — C-ABI of the B200-native CLO offloaded-KV decode path
 * (paper_2511_14510_b200/libclo.so).
 *
 * The reference (kvsim, /root/reference/proj) exposes a C++ API only; there is
 * no C ABI, plugin registry or FFI. This header is the
 * drop-in boundary for that API: POD structs mirroring the reference config
 * structs, an opaque engine handle replacing kvsim::DecodeEngine, op-level
 * entry points replacing the free functions of attention.hpp / retrieval.hpp /
 * similarity_cache.hpp / head_profile.hpp, and status codes 1:1 with the
 * exception taxonomy of errors.hpp:10-41. include/clo/kvsim.hpp re-exposes the
 * same class and method names in C++ over this header.
 *
 * Citations: /root/reference/proj/<file>:<line>.
 *
 * Conventions
 *  - Plain pointers and sizes; no torch types. "dev" pointers are CUDA device
 *    (or UVA-mapped pinned host) addresses, "host" pointers are CPU memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Engine calls are asynchronous on the stream unless documented otherwise;
 *    nothing inside clo_decode_step synchronises the host (GPU-centric sync,
 *    pipeline_sim.hpp:12).
 *  - There is no CPU fallback: every compute entry point launches sm_100a
 *    kernels and fails with CLO_ERR_CUDA when no device is usable.
 */
#ifndef CLO_H
#define CLO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CLO_ABI_VERSION 1

/* errors.hpp:10-41 — one code per exception type, plus CUDA/internal. */
typedef enum clo_status {
    CLO_OK = 0,
    CLO_ERR_SHAPE = 1,     /* ShapeError */
    CLO_ERR_ARGUMENT = 2,  /* ArgumentError */
    CLO_ERR_NUMERIC = 3,   /* NumericError */
    CLO_ERR_INDEX = 4,     /* IndexError */
    CLO_ERR_CONTRACT = 5,  /* ContractError */
    CLO_ERR_CONFIG = 6,    /* ConfigError */
    CLO_ERR_IO = 7,        /* IoError */
    CLO_ERR_CUDA = 8,      /* CUDA runtime failure / no device */
    CLO_ERR_INTERNAL = 9
} clo_status;

typedef enum clo_retriever { /* retrieval.hpp:11 RetrieverVariant */
    CLO_RETRIEVER_EXACT = 0,
    CLO_RETRIEVER_SIGN_HASH = 1
} clo_retriever;

typedef enum clo_policy { /* engine.hpp:19 Policy (LRU/LFU are out of scope) */
    CLO_POLICY_SIMILARITY = 0,
    CLO_POLICY_LRU = 1,
    CLO_POLICY_LFU = 2,
    CLO_POLICY_PREFETCH_ONLY = 3
} clo_policy;

typedef enum clo_sync_mode { /* pipeline_sim.hpp:12 SyncMode */
    CLO_SYNC_CPU_CENTRIC = 0,
    CLO_SYNC_GPU_CENTRIC = 1
} clo_sync_mode;

typedef enum clo_dtype { /* storage type of K/V rows */
    CLO_DTYPE_BF16 = 0,
    CLO_DTYPE_F32 = 1,
    CLO_DTYPE_F64 = 2 /* op-level entry points only */
} clo_dtype;

typedef enum clo_placement { /* head_profile.hpp:11 Placement */
    CLO_PLACEMENT_OFFLOADED = 0,
    CLO_PLACEMENT_PERSISTENT = 1
} clo_placement;

/* matrix.hpp:46-66 ModelShape */
typedef struct clo_model_shape {
    int num_layers;
    int num_q_heads;
    int num_kv_heads;
    int head_dim;
    int bytes_per_element; /* modeled element width for byte accounting */
} clo_model_shape;

/* engine.hpp:30-49 EngineConfig (+ B200 fields at the end). */
typedef struct clo_engine_config {
    clo_model_shape shape;
    int k;             /* entry size in tokens */
    int sink_tokens;   /* default 4 */
    int recent_tokens; /* default 64 */
    int retriever;     /* clo_retriever */
    int hash_bits;     /* default 256; multiple of 8, <= 512 */
    uint64_t retriever_seed;
    int policy; /* clo_policy: SIMILARITY or PREFETCH_ONLY */
    int always_miss;
    int always_hit;
    int has_tau_override;
    double tau_override;
    int sync_override; /* -1: policy default (engine.cpp:140-142) */
    int collect_outputs;
    int compute_oracle_error; /* EngineConfig::compute_oracle_error (engine.hpp:48): each step also takes the
                                 exact top-k with the true queries and accumulates the relative L2 error of
                                 the outputs against attention over it (a diagnostic: it reads every key) */
    /* --- B200 fields ----------------------------------------------------- */
    int batch;        /* sequences served by this engine (the runner's tasks) */
    int n_prompt;     /* StepSource::prompt_tokens() */
    int max_steps;    /* StepSource::decode_steps() */
    int kv_dtype;     /* clo_dtype of K/V rows (BF16 or F32) */
    int kv_head_offset; /* first global KV head of this shard (seeds, profiles) */
    int device;       /* CUDA ordinal */
    int victim_rows;  /* HBM rows per offloaded head kept beyond the entry: rows
                       * that left the entry stay resident (least recently left
                       * evicted first), so a token that returns to a later
                       * selection is not fetched over PCIe again. Entry
                       * contents are unchanged; only data movement shrinks.
                       * < 0: auto (8*k, capped at 40% of the free HBM); 0: none. */
} clo_engine_config;

/* Fills the reference defaults (engine.hpp:30-49): sink 4, recent 64,
 * sign-hash off (exact), hash_bits 256, seed 1, similarity policy,
 * sync_override -1, batch 1, kv_dtype BF16, victim_rows -1 (auto). */
void clo_engine_config_defaults(clo_engine_config* cfg);

typedef struct clo_engine clo_engine;

/* DecodeEngine(cfg, profiles, plan, source) — engine.hpp:93-94, engine.cpp:106-157.
 *   tau          [L * hkv]      HeadProfileEntry.tau (head_profile.hpp:16-23)
 *   q_importance [L * hkv * m]  HeadProfileEntry.q_importance
 *   persistent   [L * hkv]      1 where PartitionPlan.layers[l].persistent_heads
 *                               names head g (head_profile.hpp:85-97)
 * Allocates all HBM state (cache slots, codes, persistent KV, labels,
 * windows, scratch). */
clo_status clo_engine_create(const clo_engine_config* cfg, const double* tau,
                             const double* q_importance, const int* persistent,
                             clo_engine** out);
void clo_engine_destroy(clo_engine* e);

/* Host K/V store of the offloaded heads (HeadStore::k/v, engine.hpp:76-85):
 * caller-owned pinned, UVA-mapped memory (clo_host_alloc or
 * cudaHostRegister'ed), row-major rows of head_dim elements of kv_dtype.
 * Row r of (seq b, layer l, kv head g) lives at
 *   base + b*seq_stride + l*layer_stride + g*head_stride + r*head_dim
 * (strides in elements; seq/layer/head strides must be multiples of 16
 * bytes). layer_stride 0 aliases one buffer across layers: every layer then
 * reads the same prompt rows, and each decode step must append the SAME new
 * K/V row to every layer of a (seq, kv head) — the engine checks that on the
 * device and reports CLO_ERR_CONTRACT at the next synchronising call when a
 * step's rows differ between layers. Bind before clo_prefill (rebinding
 * afterwards is a CLO_ERR_CONTRACT).
 * Rows [0, n_prompt) must hold the prompt before clo_prefill; decode steps
 * append row n_prompt + t - 1 at step t. */
clo_status clo_engine_bind_host_kv(clo_engine* e, void* k_host, void* v_host,
                                   int64_t seq_stride, int64_t layer_stride,
                                   int64_t head_stride);

/* Same, with an explicit row stride (elements, >= head_dim; row r at
 * ... + r*row_stride). row_stride = 2*head_dim with v_host = k_host +
 * head_dim is the interleaved layout: one token's K and V rows are one
 * contiguous 2*head_dim run, so a fetched token costs one host page
 * translation instead of two (profiles/README.md: long contexts). */
clo_status clo_engine_bind_host_kv_ex(clo_engine* e, void* k_host, void* v_host,
                                      int64_t seq_stride, int64_t layer_stride,
                                      int64_t head_stride, int64_t row_stride);

/* prefill() — engine.cpp:163-209. true_q0 [B][L][hq][d] f32: step-0 true
 * queries. Encodes retrieval metadata on the GPU, loads persistent heads into
 * HBM, fills sink/recent windows, selects the step-0 top-k and gathers the
 * initial entries. `on_host` says where true_q0 lives. Synchronous. */
clo_status clo_prefill(clo_engine* e, const float* true_q0, int on_host, void* stream);

/* Per-step inputs (StepSource, synthetic_model.hpp:16-28) and outputs. */
typedef struct clo_step_io {
    const float* true_q;   /* [B][L][hq][d] */
    const float* approx_q; /* [B][L][hq][d] */
    const void* new_k;     /* [B][L][hkv][d] kv_dtype */
    const void* new_v;     /* [B][L][hkv][d] kv_dtype */
    float* out;            /* [B][L][hq][d] attention outputs (NULL: not kept) */
    int on_host;           /* 1: host buffers, copied in/out inside the call */
} clo_step_io;

/* decode_step() — engine.cpp:225-415. Asynchronous on `stream`: one CUDA-graph
 * launch (two internal streams: selection/transfer of layer l overlaps the
 * attention of layer l-1), no host synchronisation. With on_host=1 the input
 * H2D and output D2H copies are enqueued on the same stream (pinned host
 * buffers give full overlap). Errors detected on the device (non-finite
 * inputs, ContractError guards) are reported by the next synchronising call. */
clo_status clo_decode_step(clo_engine* e, const clo_step_io* io, void* stream);
/* Steps may be issued on different streams; each step is ordered after the
 * previous one (an event recorded after every step's graph). */

/* Blocks until every queued step finished; returns a deferred device error. */
clo_status clo_engine_synchronize(clo_engine* e);

/* DecodeMetrics (engine.hpp:59-73), summed over the batch. Synchronous. */
typedef struct clo_metrics {
    uint64_t steps;
    uint64_t hits;
    uint64_t misses;
    uint64_t lookups;
    double hit_ratio;
    uint64_t transferred_bytes;      /* modeled: misses * 2*k*d*bytes_per_element */
    uint64_t persistent_bytes;       /* persistent heads: steps * entry_bytes */
    uint64_t gathered_bytes_device;  /* measured: bytes the gather kernels read over PCIe */
    uint64_t cache_bytes_current;    /* modeled_cache_bytes() per sequence */
    uint64_t host_bytes;             /* host_bytes() per sequence */
    uint64_t device_persistent_bytes;/* device_persistent_bytes() per sequence */
    int sync_mode;                   /* clo_sync_mode */
    double mean_output_error;        /* DecodeMetrics::mean_output_error over all sequences (0 unless
                                        compute_oracle_error) */
} clo_metrics;
clo_status clo_get_metrics(clo_engine* e, clo_metrics* out);

/* Per-head state (HeadMetrics + CacheEntry + labels + window) of sequence b.
 * entry_indices [k] and aggregated_history [steps] may be NULL. Synchronous. */
typedef struct clo_head_state {
    uint64_t hits, misses, transferred_bytes, persistent_bytes;
    int last_update_step;       /* HeadCacheStats.last_update_step */
    int entry_last_update_step; /* CacheEntry.last_update_step */
    int labels_valid;
    int window_held_tokens;
    int placement;              /* clo_placement */
    int n_history;
} clo_head_state;
clo_status clo_get_head_state(clo_engine* e, int seq, int layer, int kv_head,
                              clo_head_state* st, int32_t* entry_indices,
                              double* aggregated_history);

/* The HBM cache-slot rows of an offloaded head's entry (CacheEntry::k_rows /
 * v_rows), copied to host buffers of k*d kv_dtype elements. Synchronous. */
clo_status clo_get_entry_rows(clo_engine* e, int seq, int layer, int kv_head, void* k_rows,
                              void* v_rows);

/* cache_state_json() — engine.cpp:464-530, same keys, for sequence `seq`.
 * Writes at most cap bytes (NUL-terminated); *needed gets the full size. */
clo_status clo_cache_state_json(clo_engine* e, int seq, char* buf, size_t cap, size_t* needed);

/* One decode step (same semantics as clo_decode_step) through an instrumented
 * copy of the step graph with event-record nodes around every kernel; fills
 * one record per kernel launch with its device time. Synchronous. Used by the
 * benchmark to measure per-kernel rooflines inside the graph. */
typedef struct clo_kernel_time {
    char name[32];
    int layer;
    float ms;
} clo_kernel_time;
clo_status clo_engine_profile_step(clo_engine* e, const clo_step_io* io, void* stream,
                                   clo_kernel_time* out, int cap, int* count);

/* Measured per-layer breakdown in the reference's LayerTiming categories
 * (pipeline_sim.hpp:61-72; DecodeEngine::timeline() engine.hpp:105). The
 * reference MODELS these times (schedule_layer, pipeline_sim.cpp:24-43);
 * here they are CUDA-event timestamps of a decode step run through a copy of
 * the step graph with the production stream layout:
 *   compute   = append + attention of the layer
 *   transfer  = the layer's zero-copy gather (raw, before overlap)
 *   exposed   = time attention(l) waited for that gather after the compute
 *               stream was ready; hidden = transfer - exposed
 *   mgmt      = lookup (fused label refresh) + entry reconcile
 *   retrieval = scoring + top-k selection
 *   sync      = 0 (GPU-centric: no host round trip in the step)
 *   total     = compute + exposed + mgmt + sync + retrieval (the reference's
 *               formula, which serialises management and retrieval)
 *   wall      = measured layer-to-layer time on the compute stream. */
typedef struct clo_layer_timing {
    int layer;
    double compute_s, transfer_s, hidden_s, exposed_s, mgmt_s, sync_s, retrieval_s, total_s;
    double wall_s;
} clo_layer_timing;
/* One decode step (clo_decode_step semantics) that also accumulates the
 * timeline. Synchronous. */
clo_status clo_engine_timeline_step(clo_engine* e, const clo_step_io* io, void* stream);
/* PipelineTimeline: per_layer [cap >= L] summed over timeline steps, totals
 * summed over layers (either may be NULL). */
clo_status clo_get_timeline(clo_engine* e, clo_layer_timing* per_layer, int cap, clo_layer_timing* totals,
                            uint64_t* steps);
/* Kernel spans of the most recent timeline step (start/end ms since the
 * step's graph began; production stream layout, so spans overlap). */
typedef struct clo_kernel_span {
    char name[32];
    int layer;
    float start_ms, end_ms;
} clo_kernel_span;
clo_status clo_timeline_spans(clo_engine* e, clo_kernel_span* out, int cap, int* count);
/* breakdown_to_json (pipeline_sim.cpp:115-135): {"steps", "layers": [...],
 * "total"}, where "transfer_s" is the exposed transfer as in the reference,
 * plus "transfer_raw_s" and "wall_s". */
clo_status clo_timeline_json(clo_engine* e, char* buf, size_t cap, size_t* needed);

/* Number of sm_100a kernels the engine enqueued since creation. */
uint64_t clo_engine_kernel_launches(const clo_engine* e);
/* Kernels per decode step (graph nodes that are kernels). */
int clo_engine_kernels_per_step(const clo_engine* e);

/* Multi-GPU (KV-head sharding): the head-output all-gather,
 * fused into the attention epilogue over peer memory (no NCCL launch).
 * The reference has no distributed path; this replaces the one exchange the
 * sharded step needs: every layer's per-head outputs (engine.cpp:403-405,
 * collected_outputs [t][l] -> h_q x d) reaching every rank.
 *
 * Rank r's engine serves KV heads [r*H, (r+1)*H) of a model with world*H KV
 * heads (cfg.kv_head_offset = r*H; shape.num_*_heads are the LOCAL counts).
 * Protocol (one process or thread per rank, any host transport for the
 * handle bytes, e.g. torch.distributed.all_gather_object):
 *   1. clo_engine_exchange_handle(e, rank, world, h)   -> CLO_EXCHANGE_HANDLE_BYTES
 *   2. exchange the handles; handles[r] = rank r's bytes, concatenated
 *   3. clo_engine_attach_peers(e, handles), then a host barrier
 * From then on io->out of every step is [B][L][world*hq][d]: the attention
 * kernels store each head's output into out and into every peer's exchange
 * slot (P2P stores over NVLink, CUDA IPC mappings across processes), raise a
 * per-layer arrival counter with a system-scope release, and the last kernel
 * of the step graph acquires the counters and copies the peers' blocks.
 * Ranks must step in lockstep; a peer that stops stepping surfaces as
 * CLO_ERR_CUDA ("exchange timed out") at the next synchronising call.
 * Must be called before the first decode step. */
#define CLO_EXCHANGE_HANDLE_BYTES 256
clo_status clo_engine_exchange_handle(clo_engine* e, int rank, int world, void* handle_out);
clo_status clo_engine_attach_peers(clo_engine* e, const void* handles);

const char* clo_last_error(void);

/* ------------------------------------------------------------------------ */
/* Pinned host memory (UVA-mapped, portable): the host KV store.            */
clo_status clo_host_alloc(size_t bytes, void** out);
/* flags: CLO_HOST_HUGEPAGES backs the store with transparent huge pages
 * (mmap + MADV_HUGEPAGE, then cudaHostRegister), so GPU threads reading random
 * rows across a large store do not miss in the TLB on every 4 KiB page.
 * Freed with clo_host_free. */
#define CLO_HOST_HUGEPAGES 1
clo_status clo_host_alloc_ex(size_t bytes, int flags, void** out);
/* Same, with every page bound (mbind MPOL_BIND, first touch under the policy,
 * then cudaHostRegister) to host NUMA node `numa_node`: the node of the PCIe
 * root the GPU that gathers from this store hangs off, so its zero-copy reads
 * never cross the socket interconnect. numa_node < 0 means
 * no binding (= clo_host_alloc_ex). Freed with clo_host_free. */
clo_status clo_host_alloc_numa(size_t bytes, int flags, int numa_node, void** out);
/* NUMA node of CUDA device `device`'s PCIe root (sysfs numa_node of its PCI
 * bus id); -1 when the host does not report one (single-node hosts). */
clo_status clo_device_numa_node(int device, int* node);
clo_status clo_host_free(void* p);
clo_status clo_host_register(void* p, size_t bytes);
clo_status clo_host_unregister(void* p);

/* ------------------------------------------------------------------------ */
/* Op-level entry points (device pointers; synchronous: they validate the   */
/* way the reference throws and return the status).                          */

/* Projection P [hash_bits][d] of encode() (retrieval.cpp:73-74): libstdc++
 * mt19937_64(seed) + normal_distribution<double>. Host function. */
clo_status clo_sign_hash_projection(int hash_bits, int d, uint64_t seed, double* out_host);

/* encode(keys, kSignHash) bits (retrieval.cpp:60-78, append_sign_row :14-25):
 * codes [n][ceil(hash_bits/64)] u64, bit b of row j = (sum_c P[b][c]*K[j][c]) >= 0
 * in sequential IEEE double. keys: n rows of d elements of `dtype`. */
clo_status clo_encode_sign_hash(const void* keys_dev, int dtype, int64_t n, int d, int hash_bits,
                                uint64_t seed, uint64_t* codes_dev, void* stream);

/* Group top-k (engine.cpp:211-223 = retrieve_scored retrieval.cpp:90-125 for
 * each of m queries + merge_group_topk similarity_cache.cpp:180-201), fused as
 * one top-k over S(i) = max_j score_j(i) (proof: DESIGN.md §3). m = 1 is
 * retrieve_scored. queries [m][d] f64. Exact: keys_dev (dtype). Sign-hash:
 * codes_dev from clo_encode_sign_hash with the same seed. out_idx [k]
 * ascending; out_score [k] = S(out_idx) (nullable). */
clo_status clo_group_topk(const double* queries_dev, int m, int d, int retriever,
                          const void* keys_dev, int dtype, const uint64_t* codes_dev,
                          int hash_bits, uint64_t seed, int64_t n, int k, int32_t* out_idx_dev,
                          double* out_score_dev, void* stream);

/* topk_select_exact (attention.cpp:71-89). */
clo_status clo_topk_select_exact(const double* q_dev, const void* keys_dev, int dtype, int64_t n,
                                 int d, int k, int32_t* out_idx_dev, void* stream);

/* merge_group_topk (similarity_cache.cpp:180-201) over explicit proposals:
 * sizes [m] host; idx/score concatenated on device. */
clo_status clo_merge_group_topk(const int* sizes_host, int m, const int32_t* idx_dev,
                                const double* score_dev, int k, int32_t* out_idx_dev,
                                void* stream);

/* lookup (similarity_cache.cpp:29-72) for n_heads independent groups:
 * labels [H][m][d] f64 (refreshed on miss), label_valid [H][m], queries
 * [H][m][d] f64, weights [H][m], tau [H]. Outputs hit/reason [H], agg [H],
 * sims [H][m]. reason: 0 none, 1 invalid label, 2 non-positive, 3 below tau. */
clo_status clo_lookup(int n_heads, int m, int d, double* labels_dev, int32_t* label_valid_dev,
                      const double* queries_dev, const double* weights_dev, const double* tau_dev,
                      int32_t* hit_dev, double* agg_dev, double* sims_dev, int32_t* reason_dev,
                      void* stream);

/* cosine_similarity (attention.cpp:155-168) for n pairs of d-vectors. */
clo_status clo_cosine_similarity(int n_pairs, int d, const double* a_dev, const double* b_dev,
                                 double* value_dev, int32_t* degenerate_dev, void* stream);

/* aggregate_similarity (similarity_cache.cpp:10-27), n groups of m. */
clo_status clo_aggregate_similarity(int n_groups, int m, const double* sims_dev,
                                    const double* weights_dev, double* out_dev, void* stream);

/* Zero-copy gather (gather_rows engine.cpp:98-102 + update_entry's row copy):
 * dst[i] = src[idx[i]] for i < k, rows of d elements. src may be pinned UVA
 * host memory (read over PCIe by GPU threads) or device memory. */
clo_status clo_gather_rows(const void* src, int dtype, int d, int64_t n_rows,
                           const int32_t* idx_dev, int k, void* dst_dev, void* stream);

/* Gather-copy baseline (TransferEngine::kGatherCopy, pipeline_sim.cpp:12-22):
 * `threads` CPU threads gather rows into a pinned staging buffer, then one
 * cudaMemcpyAsync H2D. idx_host [k]. */
/* Asynchronous variant for benchmarking the transfer engines: engine 0 = LSU
 * zero-copy gather (16-byte loads), 1 = TMA bulk-copy gather (one
 * cp.async.bulk per row from pinned host memory). `ctas` caps the grid
 * (<= 0: default). Index errors are OR'ed into *err_dev; no synchronisation. */
clo_status clo_gather_rows_ex(const void* src, int dtype, int d, int64_t n_rows,
                              const int32_t* idx_dev, int k, void* dst_dev, int engine, int ctas,
                              int* err_dev, void* stream);

clo_status clo_gather_rows_cpu_staged(const void* src_host, int dtype, int d, int64_t n_rows,
                                      const int32_t* idx_host, int k, void* staging_host,
                                      void* dst_dev, int threads, void* stream);

/* topk_attention (attention.cpp:91-105, attend_rows :33-55) for m queries over
 * one K/V matrix: validation (finite q/K/V, index range, duplicates) then
 * softmax(q.K_idx/sqrt(d)).V_idx; accumulation f32 for bf16/f32 storage, f64
 * for f64. q [m][d] f64, out [m][d] f64. */
clo_status clo_topk_attention(const double* q_dev, int m, const void* keys_dev,
                              const void* values_dev, int dtype, int64_t n, int d,
                              const int32_t* idx_dev, int nidx, double* out_dev, void* stream);

/* Host-side pieces of the path (pure functions). */
clo_status clo_sink_recent_indices(int n, int sink, int recent, int32_t* out, int* count,
                                   int* clamped);                     /* attention.cpp:107-128 */
clo_status clo_compute_threshold(double s, double eta, double p, double* tau); /* head_profile.cpp:17-25 */
clo_status clo_compute_difficulty(double tau, double s_hat, double epsilon, double* out);
clo_status clo_plan_partition(const double* difficulty, int L, int H, double t_comp_s,
                              double pcie_bw, double mem_head_bytes,
                              uint64_t persist_bytes_per_head, uint64_t hbm_budget_bytes,
                              int* persistent_out, int* n_p_out, int* n_dropped_out);
uint64_t clo_cache_bytes(int offloaded_heads, int entry_k, int held_window_tokens, int num_layers,
                         int num_q_heads, int head_dim, int bytes_per_element);

/* ------------------------------------------------------------------------ */
/* Workload traces: the reference's wire format (trace_io.hpp:12-64,         */
/* trace_io.cpp:83-266). Host functions; a trace is one sequence.            */
typedef struct clo_trace clo_trace;
/* read_trace (trace_io.cpp:129-183): validates magic, version, widths and
 * trailing bytes the same way (CLO_ERR_IO / CLO_ERR_CONFIG). */
clo_status clo_trace_open(const char* path, clo_trace** out);
void clo_trace_close(clo_trace* t);
clo_status clo_trace_info(const clo_trace* t, clo_model_shape* shape, int* n_prompt, int* n_steps,
                          int* element_width);
/* TraceSource::prompt_k/v (trace_io.cpp:230-236): n_prompt x d rows of
 * (layer, kv_head) converted to `dtype` (bf16 RNE, f32 or f64). */
clo_status clo_trace_prompt(const clo_trace* t, int layer, int kv_head, int dtype, void* k_out,
                            void* v_out);
/* TraceSource::true_query / approx_query / new_k_row / new_v_row
 * (trace_io.cpp:238-266) of step t, in the engine's clo_step_io layout:
 * true_q/approx_q [L][hq][d] f32 (approx = the layer l-1 hidden block, layer 0
 * its own), new_k/new_v [L][hkv][d] of `dtype` (t >= 1). Any output may be NULL. */
clo_status clo_trace_step(const clo_trace* t, int step, float* true_q, float* approx_q, void* new_k,
                          void* new_v, int dtype);
/* The raw hidden block [hq][d] (float64) of (step, layer): TraceSource::true_query's
 * values before any narrowing. */
clo_status clo_trace_hidden(const clo_trace* t, int step, int layer, double* out);
/* write_trace (trace_io.cpp:83-127) from arrays: prompt_k/v [L][hkv][n_prompt][d],
 * true_q [n_steps+1][L][hq][d] (the hidden blocks), new_k/v [n_steps][L][hkv][d];
 * element_width 4 or 8; also writes the <path>.json sidecar. */
clo_status clo_trace_write(const char* path, const clo_model_shape* shape, int n_prompt, int n_steps,
                           int element_width, const double* prompt_k, const double* prompt_v,
                           const double* true_q, const double* new_k, const double* new_v);

/* ------------------------------------------------------------------------ */
/* Head profiling (profile_heads, profiler.cpp:19-125; head_profile.hpp:16-75) */
typedef struct clo_profiler_config { /* ProfilerInputs, profiler.hpp:12-27 */
    int blend_sequences; /* default 1: the blend fit uses the first N sources */
    int blend_steps;     /* default 8 */
    int topk;            /* target selection size for the blend fit, default 1 */
    int sink_tokens;     /* default 4 */
    int recent_tokens;   /* default 64 */
    double eta, p, epsilon; /* defaults 0.8, 3.0, 0.1 */
} clo_profiler_config;
void clo_profiler_config_defaults(clo_profiler_config* cfg);
/* HeadProfileEntry (head_profile.hpp:16-23); q_importance has m valid entries. */
typedef struct clo_head_profile {
    double q_importance[16];
    double kv_importance, s_hat, tau, difficulty;
    int placement; /* clo_placement: always OFFLOADED here (plan_partition assigns) */
} clo_head_profile;
/* profile_heads over probe traces: s_hat = mean adjacent-step cosine of the
 * true queries; importance alpha per query head = clamp(sum (topk - stream)
 * (full - stream) / sum (full - stream)^2, 0, 1) over the first blend_steps
 * steps of the first blend_sequences sources, where full / streaming / top-k
 * attention (exact top-k of cfg->topk keys) run on the GPU in float64 over
 * the prompt rows; then kv_importance = max, s_hat = min over the group, tau,
 * difficulty. provided_importance [L][hkv][m] (nullable) replaces the fit.
 * out [L*hkv]. Synchronous. */
clo_status clo_profile_heads(const clo_trace* const* sources, int n_sources, const clo_profiler_config* cfg,
                             const double* provided_importance, clo_head_profile* out);

/* Build/diagnostic info: "sm_100a", ABI version, compiled kernels. */
const char* clo_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* CLO_H */
