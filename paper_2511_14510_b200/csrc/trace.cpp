// trace.cpp — the reference's workload trace wire format (trace_io.hpp:12-64,
// trace_io.cpp:83-266): reader, writer and the TraceSource accessors, as
// host-side C-ABI functions (include/clo.h, clo_trace_*). A trace recorded by
// the reference (record_trace + write_trace) replays on the GPU engine with
// the same queries and rows; with element_width 4 and f32 KV storage every
// value the engine consumes is bit-identical to what the reference consumes.
//
// Layout (little-endian): "KVSIMTRC", u32 version 1, u32 layers, num_q_heads,
// num_kv_heads, head_dim, n_prompt, n_steps, element_width (4|8); then per
// layer, per KV head: prompt K (n_prompt x d), prompt V; then per step
// t = 0..n_steps: per layer the hidden block (hq x d = concatenated true
// queries), and for t >= 1 per layer the new K rows (hkv x d) then V rows.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include <cuda_bf16.h>

#include "clo.h"
#include "host_common.hpp"

struct clo_trace {
    clo_model_shape shape{};
    int n_prompt = 0, n_steps = 0, element_width = 8;
    // all payload widened to double, in file order
    std::vector<double> prompt;  // [L][hkv][2][n_prompt][d]   (K then V)
    std::vector<double> hidden;  // [n_steps+1][L][hq*d]
    std::vector<double> step;    // [n_steps][L][2][hkv][d]    (K then V)
};

namespace clo {
namespace {

constexpr char kMagic[8] = {'K', 'V', 'S', 'I', 'M', 'T', 'R', 'C'};
constexpr uint32_t kVersion = 1;

void validate_shape(const clo_model_shape& s, int n_prompt, int n_steps, int width) {
    // ModelShape::validate (matrix.hpp:57-65) + TraceData::validate (trace_io.cpp:55-81)
    if (s.num_layers <= 0 || s.num_q_heads <= 0 || s.num_kv_heads <= 0 || s.head_dim <= 0)
        fail(CLO_ERR_CONFIG, "trace shape must be positive");
    if (s.num_q_heads % s.num_kv_heads != 0) fail(CLO_ERR_CONFIG, "num_q_heads must be a multiple of num_kv_heads");
    if (n_prompt <= 0) fail(CLO_ERR_CONFIG, "trace must hold a non-empty prompt");
    if (n_steps < 0) fail(CLO_ERR_CONFIG, "trace step count must be non-negative");
    if (width != 4 && width != 8) fail(CLO_ERR_CONFIG, "trace element_width must be 4 or 8");
}

void read_block(std::ifstream& in, double* dst, size_t count, int width) {
    if (width == 8) {
        in.read(reinterpret_cast<char*>(dst), (std::streamsize)(count * sizeof(double)));
    } else {
        std::vector<float> tmp(count);
        in.read(reinterpret_cast<char*>(tmp.data()), (std::streamsize)(count * sizeof(float)));
        for (size_t i = 0; i < count; ++i) dst[i] = tmp[i];
    }
    if (!in) fail(CLO_ERR_IO, "trace file truncated");
}

void write_block(std::ofstream& out, const double* src, size_t count, int width) {
    if (width == 8) {
        out.write(reinterpret_cast<const char*>(src), (std::streamsize)(count * sizeof(double)));
    } else {
        std::vector<float> tmp(src, src + count);
        out.write(reinterpret_cast<const char*>(tmp.data()), (std::streamsize)(count * sizeof(float)));
    }
}

// double -> storage element (bf16 round-to-nearest-even, or f32)
void store(const double* src, size_t count, int dtype, void* dst) {
    if (dtype == CLO_DTYPE_F32) {
        float* o = static_cast<float*>(dst);
        for (size_t i = 0; i < count; ++i) o[i] = (float)src[i];
    } else if (dtype == CLO_DTYPE_BF16) {
        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(dst);
        for (size_t i = 0; i < count; ++i) o[i] = __float2bfloat16_rn((float)src[i]);
    } else if (dtype == CLO_DTYPE_F64) {
        std::memcpy(dst, src, count * sizeof(double));
    } else {
        fail(CLO_ERR_ARGUMENT, "unknown dtype");
    }
}

size_t hq_d(const clo_trace& t) { return (size_t)t.shape.num_q_heads * t.shape.head_dim; }

}  // namespace
}  // namespace clo

using namespace clo;

extern "C" {

clo_status clo_trace_open(const char* path, clo_trace** out) {
    return guarded([&] {
        if (!path || !out) fail(CLO_ERR_ARGUMENT, "null argument");
        *out = nullptr;
        std::ifstream in(path, std::ios::binary);
        if (!in) fail(CLO_ERR_IO, std::string("cannot open trace file: ") + path);
        char magic[8];
        in.read(magic, sizeof magic);
        if (!in || std::memcmp(magic, kMagic, sizeof kMagic) != 0) fail(CLO_ERR_IO, std::string("not a trace file: ") + path);
        uint32_t hdr[8];
        in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
        if (!in) fail(CLO_ERR_IO, "trace file truncated");
        if (hdr[0] != kVersion) fail(CLO_ERR_IO, "unsupported trace version");
        auto* t = new clo_trace();
        try {
            t->shape = {(int)hdr[1], (int)hdr[2], (int)hdr[3], (int)hdr[4], 2};
            t->n_prompt = (int)hdr[5];
            t->n_steps = (int)hdr[6];
            t->element_width = (int)hdr[7];
            if (t->element_width != 4 && t->element_width != 8) fail(CLO_ERR_IO, "trace element_width must be 4 or 8");
            validate_shape(t->shape, t->n_prompt, t->n_steps, t->element_width);
            const size_t L = t->shape.num_layers, H = t->shape.num_kv_heads, d = t->shape.head_dim;
            const size_t n = t->n_prompt, S = t->n_steps;
            t->prompt.resize(L * H * 2 * n * d);
            t->hidden.resize((S + 1) * L * hq_d(*t));
            t->step.resize(S * L * 2 * H * d);
            for (size_t i = 0; i < L * H * 2; ++i) read_block(in, t->prompt.data() + i * n * d, n * d, t->element_width);
            for (size_t s = 0; s <= S; ++s) {
                read_block(in, t->hidden.data() + s * L * hq_d(*t), L * hq_d(*t), t->element_width);
                if (s >= 1) read_block(in, t->step.data() + (s - 1) * L * 2 * H * d, L * 2 * H * d, t->element_width);
            }
            in.peek();
            if (!in.eof()) fail(CLO_ERR_IO, "trailing bytes after trace payload");
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
    });
}

void clo_trace_close(clo_trace* t) { delete t; }

clo_status clo_trace_info(const clo_trace* t, clo_model_shape* shape, int* n_prompt, int* n_steps,
                          int* element_width) {
    return guarded([&] {
        if (!t) fail(CLO_ERR_ARGUMENT, "null trace");
        if (shape) *shape = t->shape;
        if (n_prompt) *n_prompt = t->n_prompt;
        if (n_steps) *n_steps = t->n_steps;
        if (element_width) *element_width = t->element_width;
    });
}

clo_status clo_trace_prompt(const clo_trace* t, int layer, int kv_head, int dtype, void* k_out, void* v_out) {
    return guarded([&] {
        if (!t) fail(CLO_ERR_ARGUMENT, "null trace");
        if (layer < 0 || layer >= t->shape.num_layers || kv_head < 0 || kv_head >= t->shape.num_kv_heads)
            fail(CLO_ERR_INDEX, "prompt head out of range");  // .at() in TraceSource::prompt_k
        const size_t nd = (size_t)t->n_prompt * t->shape.head_dim;
        const double* base = t->prompt.data() + ((size_t)layer * t->shape.num_kv_heads + kv_head) * 2 * nd;
        if (k_out) store(base, nd, dtype, k_out);
        if (v_out) store(base + nd, nd, dtype, v_out);
    });
}

clo_status clo_trace_step(const clo_trace* t, int step, float* true_q, float* approx_q, void* new_k, void* new_v,
                          int dtype) {
    return guarded([&] {
        if (!t) fail(CLO_ERR_ARGUMENT, "null trace");
        if (step < 0 || step > t->n_steps) fail(CLO_ERR_INDEX, "trace step out of range");
        const int L = t->shape.num_layers, H = t->shape.num_kv_heads, d = t->shape.head_dim;
        const size_t blk = hq_d(*t);
        const double* hid = t->hidden.data() + (size_t)step * L * blk;
        for (int l = 0; l < L; ++l) {
            // true_query: the layer's own block; approx_query: the layer l-1
            // block (layer 0 falls back to its own), trace_io.cpp:238-252
            const double* own = hid + (size_t)l * blk;
            const double* prev = hid + (size_t)(l > 0 ? l - 1 : 0) * blk;
            for (size_t i = 0; i < blk; ++i) {
                if (true_q) true_q[(size_t)l * blk + i] = (float)own[i];
                if (approx_q) approx_q[(size_t)l * blk + i] = (float)prev[i];
            }
        }
        if (new_k || new_v) {
            if (step < 1) fail(CLO_ERR_ARGUMENT, "new KV rows exist only for decode steps");
            const size_t hd = (size_t)H * d;
            const double* st = t->step.data() + (size_t)(step - 1) * L * 2 * hd;
            const size_t esz = dtype == CLO_DTYPE_BF16 ? 2 : dtype == CLO_DTYPE_F32 ? 4 : 8;
            for (int l = 0; l < L; ++l) {
                if (new_k) store(st + (size_t)l * 2 * hd, hd, dtype, static_cast<char*>(new_k) + (size_t)l * hd * esz);
                if (new_v) store(st + (size_t)l * 2 * hd + hd, hd, dtype, static_cast<char*>(new_v) + (size_t)l * hd * esz);
            }
        }
    });
}

clo_status clo_trace_hidden(const clo_trace* t, int step, int layer, double* out) {
    return guarded([&] {
        if (!t || !out) fail(CLO_ERR_ARGUMENT, "null argument");
        if (step < 0 || step > t->n_steps) fail(CLO_ERR_INDEX, "trace step out of range");
        if (layer < 0 || layer >= t->shape.num_layers) fail(CLO_ERR_INDEX, "trace layer out of range");
        const size_t blk = hq_d(*t);
        std::memcpy(out, t->hidden.data() + ((size_t)step * t->shape.num_layers + layer) * blk, blk * sizeof(double));
    });
}

clo_status clo_trace_write(const char* path, const clo_model_shape* shape, int n_prompt, int n_steps,
                           int element_width, const double* prompt_k, const double* prompt_v, const double* true_q,
                           const double* new_k, const double* new_v) {
    return guarded([&] {
        if (!path || !shape || !prompt_k || !prompt_v || !true_q) fail(CLO_ERR_ARGUMENT, "null argument");
        validate_shape(*shape, n_prompt, n_steps, element_width);
        if (n_steps > 0 && (!new_k || !new_v)) fail(CLO_ERR_ARGUMENT, "decode steps need new K/V rows");
        const size_t L = shape->num_layers, H = shape->num_kv_heads, HQ = shape->num_q_heads, d = shape->head_dim;
        const size_t n = n_prompt;
        std::ofstream out(path, std::ios::binary);
        if (!out) fail(CLO_ERR_IO, std::string("cannot open trace file for writing: ") + path);
        out.write(kMagic, sizeof kMagic);
        const uint32_t hdr[8] = {kVersion, (uint32_t)L, (uint32_t)HQ, (uint32_t)H, (uint32_t)d,
                                 (uint32_t)n_prompt, (uint32_t)n_steps, (uint32_t)element_width};
        out.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
        for (size_t l = 0; l < L; ++l)
            for (size_t g = 0; g < H; ++g) {
                write_block(out, prompt_k + (l * H + g) * n * d, n * d, element_width);
                write_block(out, prompt_v + (l * H + g) * n * d, n * d, element_width);
            }
        for (size_t s = 0; s <= (size_t)n_steps; ++s) {
            write_block(out, true_q + s * L * HQ * d, L * HQ * d, element_width);
            if (s >= 1)
                for (size_t l = 0; l < L; ++l) {
                    write_block(out, new_k + ((s - 1) * L + l) * H * d, H * d, element_width);
                    write_block(out, new_v + ((s - 1) * L + l) * H * d, H * d, element_width);
                }
        }
        if (!out) fail(CLO_ERR_IO, std::string("failed writing trace file: ") + path);
        out.close();
        // JSON sidecar mirroring the header (trace_io.cpp:111-126)
        std::ofstream side(std::string(path) + ".json", std::ios::binary);
        if (!side) fail(CLO_ERR_IO, std::string("cannot open trace sidecar for writing: ") + path + ".json");
        side << "{\n  \"format\": \"kvsim-trace\",\n  \"version\": " << kVersion << ",\n  \"layers\": " << L
             << ",\n  \"num_q_heads\": " << HQ << ",\n  \"num_kv_heads\": " << H << ",\n  \"head_dim\": " << d
             << ",\n  \"n_prompt\": " << n_prompt << ",\n  \"n_steps\": " << n_steps
             << ",\n  \"element_width\": " << element_width
             << ",\n  \"hidden_block\": \"concatenated per-head query vectors per layer and step\"\n}\n";
    });
}

}  // extern "C"
