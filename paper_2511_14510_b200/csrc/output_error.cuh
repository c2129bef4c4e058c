// output_error.cuh — EngineConfig::compute_oracle_error on the device (output_error.cu).
#pragma once

#include "common.cuh"
#include "engine_view.h"

namespace clo {

struct OutputErrorArgs {
    uint64_t* keys;                   // [B*H][nmax] exact-score keys of one layer
    int32_t* sel;                     // [B*H][k + sink + recent] exact top-k (ascending)
    int32_t* uni;                     // [B*H][k + sink + recent] union with the window
    double* scores;                   // [B*H][k + sink + recent] attention weights
    double* err;                      // [B][L][HQ] relative L2 errors summed over the steps (one writer
                                      // per element and step: deterministic); output_err_count is
                                      // steps * L * HQ per sequence
};

// After the step's attention of layer `layer` (and its append).
void launch_output_error(const EngineView& v, int layer, const OutputErrorArgs& a, cudaStream_t stream);

}  // namespace clo
