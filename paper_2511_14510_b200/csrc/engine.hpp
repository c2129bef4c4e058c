// engine.hpp — host-side B200 DecodeEngine (mirrors kvsim::DecodeEngine,
// engine.hpp:91-139 of the reference).
#pragma once

#include <array>
#include <string>
#include <vector>

#include "clo.h"
#include "common.cuh"
#include "engine_view.h"
#include "host_common.hpp"
#include "gather.cuh"
#include "select.cuh"

namespace clo {

class Engine {
  public:
    Engine(const clo_engine_config& cfg, const double* tau, const double* q_importance,
           const int* persistent);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void bind_host_kv(void* k, void* v, int64_t seq_stride, int64_t layer_stride, int64_t head_stride,
                      int64_t row_stride);  // row_stride 0 = head_dim
    void prefill(const float* true_q0, int on_host, cudaStream_t user);
    void decode_step(const clo_step_io& io, cudaStream_t user);
    void synchronize();
    clo_metrics metrics();
    clo_head_state head_state(int b, int l, int g, int32_t* entry_indices, double* history);
    void entry_rows(int b, int l, int g, void* k_rows, void* v_rows);
    std::string cache_state_json(int b);

    // One decode step through an instrumented copy of the step graph: external
    // event-record nodes around every kernel, so per-launch device time is
    // measured inside the graph (bench roofline). Synchronous.
    std::vector<clo_kernel_time> profile_step(const clo_step_io& io, cudaStream_t user);
    // One decode step through the timeline graph (production stream layout +
    // event records): accumulates the measured per-layer breakdown in the
    // reference's LayerTiming categories (pipeline_sim.hpp:61-86). Synchronous.
    void timeline_step(const clo_step_io& io, cudaStream_t user);
    const std::vector<clo_layer_timing>& timeline() const { return timeline_; }
    uint64_t timeline_steps() const { return timeline_steps_; }
    std::string timeline_json() const;
    // Kernel spans of the last timeline step: start/end ms since the step began.
    const std::vector<clo_kernel_span>& last_spans() const { return spans_; }

    // KV-head sharding: fused head-output all-gather over peer memory
    // (exchange.cuh). peer_handle() describes this engine's exchange buffer;
    // attach_peers() maps every rank's buffer (P2P / CUDA IPC).
    void peer_handle(int rank, int world, void* out);
    void attach_peers(const void* handles);

    uint64_t launches() const { return launches_; }
    int kernels_per_step() const { return kernels_per_step_; }
    const clo_engine_config& config() const { return cfg_; }

  private:
    static constexpr int kDescRing = 256;

    void allocate();
    EngineView view() const;
    SelArgs sel_args(int which, int layer) const;
    void enqueue_prepare(int which, int layer, int mode, int kind, cudaStream_t st);
    void enqueue_select(int which, int layer, cudaStream_t st, bool with_reconcile = false);
    int chained_select() const;
    struct OutputErrorArgs output_error_args() const;
    double mean_output_error(int b);
    ReconcileArgs reconcile_args(int layer, int fresh) const;
    void enqueue_reconcile(int layer, int fresh, cudaStream_t st);
    void enqueue_gather(int layer, int count_bytes, cudaStream_t st);
    void enqueue_fused_select(int layer, cudaStream_t st);
    bool fused_select() const;
    GatherEngineArgs gather_args(int layer, int count_bytes) const;
    enum GraphMode { kGraphProd = 0, kGraphSerial = 1, kGraphTimeline = 2, kGraphModes = 3 };
    void capture_graph(int mode);
    void drop_graphs();
    void launch_step(int mode, const clo_step_io& io, cudaStream_t user);
    void prof_begin(cudaStream_t st);
    void prof_end(cudaStream_t st, const char* name, int layer);
    StepDesc make_desc(const clo_step_io& io, cudaStream_t user);
    void set_desc(const StepDesc& d, cudaStream_t st);
    void check_device_error();
    uint64_t entry_bytes() const;
    int held_tokens() const;

    clo_engine_config cfg_;
    std::vector<double> tau_, qimp_;
    std::vector<int> persistent_, pidx_, oidx_, layer_has_pers_, layer_has_off_;
    int np_ = 0, no_ = 0;
    int sync_mode_ = CLO_SYNC_GPU_CENTRIC;
    int nmax_ = 0, max_chunks_ = 0, words_ = 0, nb_ = 0, max_attn_chunks_ = 0;
    int64_t code_stride_ = 0;
    int pool_ = 0;  // HBM row-pool slots per offloaded head (k + victim rows)
    cudaEvent_t ev_step_ = nullptr;     // recorded after each step's graph (cross-stream step order)
    cudaStream_t step_stream_ = nullptr;  // stream of the previous step
    bool step_stream_set_ = false;  // u64 words per segment's codes, even (16-byte aligned segments)

    void* host_k_ = nullptr;
    void* host_v_ = nullptr;
    int64_t seq_stride_ = 0, layer_stride_ = 0, head_stride_ = 0, row_stride_ = 0;

    DevBuf d_persistent_, d_pidx_, d_oidx_, d_tau_, d_qimp_;
    DevBuf d_pk_, d_pv_, d_kmirror_, d_slot_k_, d_slot_v_, d_win_k_, d_win_v_;
    DevBuf d_entry_idx_, d_entry_slot_, d_slot_tok_, d_slot_age_, d_tok2slot_, d_vhead_, d_codes_, d_proj_t_, d_proj_w_, d_labels_, d_label_valid_;
    DevBuf d_hits_, d_misses_, d_cache_last_, d_entry_last_, d_last_hit_, d_history_, d_gathered_;
    DevBuf d_step_, d_desc_, d_err_, d_attn_part_, d_attn_count_, d_xfer_, d_off_layers_;
    int n_off_layers_ = 0;
    DevBuf d_in_tq_, d_in_aq_, d_in_nk_, d_in_nv_, d_out_;
    DevBuf d_tmaps_;  // 4 CUtensorMaps over the cache slots (attention TMA boxes)
    DevBuf d_oerr_;   // compute_oracle_error scratch (output_error.cuh)
    // host-input staging, double-buffered: step t+1's H2D copies run on a copy
    // stream while step t's graph still executes
    std::array<DevBuf, 2> d_in_;
    int in_slot_ = 0;
    cudaStream_t s_copy_ = nullptr;
    std::array<cudaEvent_t, 2> ev_in_{}, ev_free_{};
    std::array<bool, 2> in_used_{};
    int pending_free_ = -1;  // slot whose consumer graph is being launched
    // 0: compute stream (persistent heads); 1, 2: the two selection streams
    // (offloaded heads of even / odd layers). 2 owns only the per-stage
    // intermediates; its per-layer work and fetch lists alias 1's.
    std::array<SelScratch, 3> scratch_{};
    std::array<std::array<DevBuf, 18>, 3> scratch_bufs_;
    int sel_streams_ = 1;  // CLO_SEL_STREAMS: selection streams (layers by parity)
    const SelScratch& off_scratch(int layer) const { return scratch_[sel_streams_ > 1 && (layer & 1) ? 2 : 1]; }

    cudaStream_t s_main_ = nullptr, s_pref_ = nullptr, s_pref2_ = nullptr, s_xfer_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_join2_ = nullptr, ev_join3_ = nullptr;
    std::vector<cudaEvent_t> ev_attn_, ev_pref_, ev_sel_;
    std::array<cudaGraph_t, kGraphModes> graphs_{};
    std::array<cudaGraphExec_t, kGraphModes> execs_{};
    int capture_mode_ = -1;  // instrumented mode being captured (event records), -1 none
    struct ProfRec {
        cudaEvent_t a, b;
        const char* name;
        int layer;
    };
    std::array<std::vector<ProfRec>, kGraphModes> prof_;
    std::array<size_t, kGraphModes> prof_used_{};
    cudaEvent_t tl_base_ = nullptr;           // timeline graph origin
    std::vector<clo_layer_timing> timeline_;  // [L], summed over timeline steps
    uint64_t timeline_steps_ = 0;
    std::vector<clo_kernel_span> spans_;
    StepDesc* desc_host_ = nullptr;
    std::vector<cudaEvent_t> desc_ev_;
    std::vector<int> desc_used_;
    int desc_next_ = 0;

    // head-output exchange
    int world_ = 1, rank_ = 0;
    DevBuf d_xbuf_;                        // [flags][2][B][L][HQg][d]
    std::array<void*, kMaxRanks> xbase_{};  // every rank's exchange buffer, mapped here
    std::array<bool, kMaxRanks> xipc_{};    // opened through cudaIpcOpenMemHandle

    bool prefilled_ = false;
    int steps_ = 0;
    uint64_t launches_ = 0;
    int kernels_per_step_ = 0;
};

}  // namespace clo
