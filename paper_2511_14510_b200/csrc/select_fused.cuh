// select_fused.cuh — one kernel for a decode layer's whole selection chain
// (offloaded heads, sign-hash retriever): see select_fused.cu.
#pragma once

#include "gather.cuh"
#include "lookup.cuh"
#include "select.cuh"

namespace clo {

struct FusedSelectArgs {
    PrepareArgs prep;   // decode lookup of the layer's offloaded heads (s.items offset to the layer)
    SelArgs sel;        // the same layer's work list and selection scratch
    ReconcileArgs rec;  // its entry reconcile / fetch lists
    int* ctl;           // [L][ctl_stride] task counters, zeroed at step end
    int ctl_stride;     // 2 + 3 * items_cap
    int items_cap;      // B*H
};

inline int fused_ctl_stride(int items_cap) { return 2 + 3 * items_cap; }
size_t fused_select_smem(int words, int nb, int m, int d, int k, int max_chunks);
void launch_fused_select(const FusedSelectArgs& f, int grid, cudaStream_t stream);

}  // namespace clo
