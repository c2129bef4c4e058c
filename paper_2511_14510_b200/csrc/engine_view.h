// engine_view.h — POD view of the engine's device state, passed by value to
// every engine kernel. Layouts (all row-major; s = (b*L + l)*H + g is the
// segment = one (sequence, layer, KV head) unit of the reference's per-head
// loops, engine.cpp:260-409):
//
//   host_k/host_v   pinned UVA host KV of every head (HeadStore::k/v):
//                   base + b*seq_stride + l*layer_stride + g*head_stride + row*d
//   pk/pv           [B*NP][nmax][d]   persistent heads' full KV in HBM
//   kmirror         [B*NO][nmax][d]   exact retriever only: HBM copy of the
//                                     offloaded heads' K (parity mode)
//   slot_k/slot_v   [B*NO][pool][d]   HBM row pool of each offloaded head: the
//                                     k rows of CacheEntry::k_rows/v_rows plus up
//                                     to `victim` rows that left the entry lately
//                                     (pool = k + victim)
//   win_k/win_v     [B*NO][sink+recent][d]  SinkRecentBuffer (sink rows, then ring)
//   entry_idx       [B*L*H][k] int32  offloaded: CacheEntry::indices;
//                                     persistent: this step's selection
//   entry_slot      [B*NO][k]         offloaded: pool slot of the i-th entry token
//   slot_tok/slot_age [B*NO][pool]    token held by each slot (-1 empty) / step it
//                                     left the entry (kSlotInEntry while in it, -2
//                                     empty): least recently left is evicted first
//   tok2slot        [B*NO][nmax]      pool slot holding each token, -1 if none
//   codes           [B*L*H][code_stride] u64 sign-hash bits (RetrievalMetadata::bits):
//                   row j of segment s at codes + s*code_stride + j*words;
//                   code_stride = nmax*words rounded up to an even word count so
//                   every segment starts 16-byte aligned (TMA bulk copies)
//   proj_t          [L*H][d][bits] f64  projection transposed (P^T)
//   proj_w          [L*H][words][d][64] f64  the same, one contiguous slice per 64-bit code word
//   labels          [B*L*hq][d] f64, label_valid [B*L*hq]   (QueryLabel)
//   tau [L*H], qimp [L*H][m]                       (HeadProfileEntry)
//   seg counters    hits/misses [B*L*H] u64, last_update/entry_last_update,
//                   last_lookup_hit, history [B*L*H][max_steps] f64
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace clo {

struct SelItem;

struct StepDesc {
    const float* true_q;   // [B][L][hq][d]
    const float* approx_q; // [B][L][hq][d]
    const void* new_k;     // [B][L][H][d]
    const void* new_v;
    float* out;            // [B][L][hq][d]
};

// Per-stream selection scratch (one for the prefetch stream, one for the
// compute stream).
struct SelScratch {
    int* count;            // [L] items appended by prepare for layer l
    SelItem* items;        // [B*H] work items (select.cuh)
    double* q64;           // [B*H][m][d] widened queries of each item
    uint64_t* qbits;       // [B*H][m][words]
    uint16_t* key16;       // [B*H][nmax] sign-hash scores S(i)
    uint64_t* key64;       // [B*H][nmax] exact: orderable keys of S(i)
    uint32_t* chunk_hist;  // [B*H][max_chunks][nb]
    int* chunk_base;       // [B*H][max_chunks]
    int* chunk_take;       // [B*H][max_chunks]
    uint64_t* thresh;      // [B*H] threshold key T
    int* need;             // [B*H] ties to take / remaining k during radix passes
    uint32_t* radix_hist;  // [B*H][256] exact radix pass histogram
    int32_t* sel;          // [B*H][k] offloaded items: the new selection (ascending)
    int32_t* fetch_tok;    // [L][B*H][k] move list: source (host token, or -(victim slot + 1))
    int32_t* fetch_slot;   // [L][B*H][k]   destination entry slot
    int32_t* fetch_dem;    // [L][B*H][k]   victim slot the leaving row moves to first, or -1
    int* fetch_count;      // [L][B*H]
    int* item_done;        // [2][B*H] chunk counters of the chained score/threshold and compact/reconcile
};

struct EngineView {
    // shape
    int B, L, H, HQ, m, d, k, sink, recent, bits, words, nb;
    int n_prompt, nmax, max_steps, max_chunks;
    int retriever, policy, always_miss, always_hit, has_tau_override;
    double tau_override;
    int kv_dtype;
    int NP, NO;            // persistent / offloaded (l,g) pairs
    // host KV
    const void* host_k;
    const void* host_v;
    void* host_k_w;        // same pointers, writable (append)
    void* host_v_w;
    int64_t seq_stride, layer_stride, head_stride;
    int64_t row_stride;  // host elements between consecutive rows of one head (head_dim, or 2*head_dim interleaved)
    int kv_fused;        // interleaved host K|V (host_v = host_k + d, row_stride = 2d): gather a token's K|V run at once
    // placement
    const int* persistent; // [L*H]
    const int* pidx;       // [L*H] index among persistent (l,g) or -1
    const int* oidx;       // [L*H] index among offloaded (l,g) or -1
    // HBM stores
    void* pk;
    void* pv;
    void* kmirror;
    void* slot_k;
    void* slot_v;
    void* win_k;
    void* win_v;
    int32_t* entry_idx;
    int32_t* entry_slot;   // [B*NO][k] slot holding the i-th (ascending) entry token
    int32_t* slot_tok;     // [B*NO][pool] token held by each slot (-1: empty)
    int32_t* slot_age;     // [B*NO][pool] step the slot's token left the entry
    int32_t* tok2slot;     // [B*NO][nmax] slot of each resident token (-1: not in HBM)
    int pool;              // slots per offloaded head (k + victim rows)
    int* vhead;            // [B*NO] FIFO cursor over each head's victim area (offset in [0, victim))
    uint64_t* codes;
    int64_t code_stride;   // u64 words per segment (even)
    const double* proj_t;
    const double* proj_w;  // [L*H][words][d][64] f64: P^T in 64-bit word slices (zero past bits)
    double* labels;
    int* label_valid;
    const double* tau;
    const double* qimp;
    // metrics
    unsigned long long* hits;
    unsigned long long* misses;
    int* cache_last_update;
    int* entry_last_update;
    int* last_lookup_hit;
    double* history;
    unsigned long long* gathered_bytes;
    // step state
    int* dev_step;         // completed decode steps
    const StepDesc* desc;
    int* err;
    // attention partials
    float* attn_part;      // [B*H][max_attn_chunks][m][d + 2]
    int* attn_count;       // [B*H] arrival counters (self-resetting)
    int max_attn_chunks;
    // persistent transfer kernel (GPU-centric sync): per-layer device flags,
    // epoch = the decode step they refer to
    int* xfer_ready;       // [L] epoch when layer l's fetch lists are published
    int* xfer_units;       // [L] work units of layer l
    int* xfer_claim;       // [L] next unit to claim (reset at step end)
    int* xfer_done;        // [L] units finished (reset at step end)
    int* xfer_flag;        // [L] epoch when every unit of layer l landed in HBM
    // head-output exchange (KV-head sharding, exchange.cuh). world == 1: none;
    // out is then [B][L][HQ][d] (HQg == HQ, q0 == 0).
    int world, rank;
    int HQg;               // query heads of the whole model (out's head extent)
    int q0;                // first global query head of this shard
    float* xslot[kMaxRanks];     // rank r's exchange slots [2][B][L][HQg][d]
    unsigned* xflag[kMaxRanks];  // rank r's per-layer arrival counters [L]
    unsigned long long xtimeout_ns;  // a peer silent this long is reported lost
    // TMA tensor maps (CUtensorMap, 64-byte aligned, device memory) over the
    // row pools [B*NO*pool][d] bf16 (row o*pool + slot): 128-byte swizzled
    // boxes of 64 columns x the attention tile rows, read over the entry area
    // (slots [0, k)); null when not built (f32 rows, other d)
    const void* tmap_k;    // 16-row boxes
    const void* tmap_v;
    const void* tmap_k32;  // 32-row boxes
    const void* tmap_v32;
};

}  // namespace clo
