// select_fused.cuh — one kernel for a decode layer's whole selection chain
// (offloaded heads, sign-hash retriever), one cluster per (sequence, KV head):
// see select_fused.cu.
#pragma once

#include "gather.cuh"
#include "lookup.cuh"
#include "select.cuh"

namespace clo {

struct FusedSelectArgs {
    PrepareArgs prep;   // decode lookup of the layer's offloaded heads (s.items offset to the layer)
    SelArgs sel;        // the layer's selection scratch (u16 keys)
    ReconcileArgs rec;  // its entry reconcile / fetch lists
    int keys_bytes;     // shared memory for one rank's u16 keys (set by the launcher)
};

size_t fused_select_smem(int words, int nb, int m, int d, int k, int nmax, int cs);
// the fused kernel holds a rank's keys in shared memory: contexts up to ~512K rows
bool fused_select_fits(int words, int nb, int m, int d, int k, int nmax);
int fused_cluster_size();
void launch_fused_select(const FusedSelectArgs& f, cudaStream_t stream);

}  // namespace clo
