// reconcile.cuh — update_entry's bookkeeping for one missed head (delta
// gather), as a CTA-wide device function: called by reconcile_kernel (one
// CTA per item) and by the fused per-layer selection kernel (the CTA that
// finishes an item's last compaction chunk).
#pragma once

#include <cub/block/block_scan.cuh>

#include "gather.cuh"

namespace clo {

__device__ __forceinline__ int lower_bound(const int32_t* a, int n, int32_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Reconcile of one missed head's entry with its new selection (one CTA per
// head). A head's HBM rows are a pool: the ENTRY AREA, slots [0, k), holds
// the entry's rows (CacheEntry::k_rows/v_rows, in slot order; entry_slot maps
// entry position -> slot) and is what attention streams; the VICTIM AREA,
// slots [k, pool), keeps rows that left the entry lately.
//   1. new tokens already in the entry area keep their slot;
//   2. the other new tokens take the entry slots the leaving tokens free
//      (both in ascending order). Each arrives from the victim area if it is
//      resident there (a promotion, an HBM copy), else over PCIe;
//   3. each leaving token's row is demoted into the victim area, a FIFO ring
//      per head: the slots after the head's cursor (demoted longest ago, or
//      emptied by promotions) are overwritten first; this step's promotion
//      sources are skipped.
// Demotions, promotions and host fetches are all the gather kernels' move
// list: a move first copies its slot's leaving row to the victim slot, then
// stores the incoming row (HBM or PCIe) into the slot. The entry's contents are exactly
// the reference's (update_entry, similarity_cache.cpp:74-87); only which rows
// cross PCIe changes.
//
// Move list of item i (fetch_*[layer][i][j], j < fetch_count): fetch_slot =
// destination entry slot; fetch_tok = source token (host row) when >= 0, or
// -(victim slot + 1) for a promotion; fetch_dem = the victim slot the slot's
// leaving row is demoted to (by the same move, before the slot is overwritten), or -1.
template <int T>
struct ReconcileSmem {
    typename cub::BlockScan<int, T>::TempStorage scan;
    int nprom;
};

// One item, whole CTA of T threads (T == blockDim.x); rs = 4*k ints of
// shared memory. Ends with __syncthreads().
template <int T>
__device__ __forceinline__ void reconcile_item(const ReconcileArgs& a, int item, int32_t* rs, ReconcileSmem<T>& sm) {
    using Scan = cub::BlockScan<int, T>;
    const EngineView& v = a.v;
    const int k = v.k, P = v.pool, V = P - k;
    int32_t* nsel = rs;            // [k] new selection (ascending)
    int32_t* need_pos = rs + k;    // [k] entry positions of the incoming tokens
    int32_t* freed = rs + 2 * k;   // [k] freed entry slots (ascending); first a kept flag per slot
    int32_t* dvict = rs + 3 * k;   // [k] demotion targets (ascending victim slots)
    const int t = a.fresh ? 0 : *v.dev_step + 1;
    const int per = (k + T - 1) / T;
    const int r0 = threadIdx.x * per, r1 = min(k, r0 + per);
    {
        const int seg = a.items[item].seg;
        const int g = seg % v.H, l = (seg / v.H) % v.L, b = seg / (v.H * v.L);
        const size_t o = (size_t)b * v.NO + v.oidx[l * v.H + g];
        int32_t* e_idx = v.entry_idx + (size_t)seg * k;
        int32_t* e_slot = v.entry_slot + o * k;
        int32_t* s_tok = v.slot_tok + o * P;
        int32_t* s_age = v.slot_age + o * P;
        int32_t* t2s = v.tok2slot + o * v.nmax;
        const int32_t* sel = a.sel + (size_t)item * k;
        for (int i = threadIdx.x; i < k; i += blockDim.x) {
            nsel[i] = sel[i];
            freed[i] = 0;  // kept flags of the entry slots
        }
        if (threadIdx.x == 0) sm.nprom = 0;
        __syncthreads();
        // 1) classify the new tokens
        int nin = 0, nprom = 0;
        for (int i = r0; i < r1; ++i) {
            const int s = t2s[nsel[i]];
            if (s >= 0 && s < k) {
                freed[s] = 1;
                e_slot[i] = s;
            } else {
                ++nin;
                if (s >= k) {
                    s_age[s] = kSlotInEntry;  // promotion source: not a demotion target
                    ++nprom;
                }
            }
        }
        if (nprom) atomicAdd(&sm.nprom, nprom);
        int nbase, total;
        Scan(sm.scan).ExclusiveSum(nin, nbase, total);
        for (int i = r0; i < r1; ++i) {
            const int s = t2s[nsel[i]];
            if (s < 0 || s >= k) need_pos[nbase++] = i;
        }
        __syncthreads();
        // 2) freed entry slots, ascending (exactly `total` of them)
        int nf = 0;
        for (int e = r0; e < r1; ++e) nf += !freed[e];
        int fbase;
        Scan(sm.scan).ExclusiveSum(nf, fbase);
        constexpr int kPer = (8192 + T - 1) / T;  // k <= reconcile_max_k()
        int fl[kPer];  // this thread's freed slots (per <= kPer)
        int nfl = 0;
        for (int e = r0; e < r1; ++e)
            if (!freed[e]) fl[nfl++] = e;
        __syncthreads();  // every kept flag read before the list overwrites them
        for (int i = 0; i < nfl; ++i) freed[fbase + i] = fl[i];
        // 3) demotion targets: the victim area is a FIFO ring walked by a
        //    per-head cursor, so the slots after the cursor hold the rows
        //    demoted longest ago (or emptied by promotions). Take the next
        //    ndem slots in ring order, skipping this step's promotion
        //    sources; the window is at most total + nprom slots: O(moves).
        int ndem = 0;
        if (!a.fresh && total > 0 && V > 0) {
            const int vh = v.vhead[o];
            const int W = min(V, total + sm.nprom);
            const int wper = (W + T - 1) / T;
            const int q0 = threadIdx.x * wper, q1 = min(W, q0 + wper);
            int nc = 0;
            for (int q = q0; q < q1; ++q) nc += s_age[k + (vh + q) % V] != kSlotInEntry;
            int cbase, ncand;
            Scan(sm.scan).ExclusiveSum(nc, cbase, ncand);
            ndem = min(total, ncand);
            for (int q = q0; q < q1 && cbase < ndem; ++q) {
                const int p = k + (vh + q) % V;
                if (s_age[p] == kSlotInEntry) continue;
                dvict[cbase] = p;
                if (++cbase == ndem) v.vhead[o] = (vh + q + 1) % V;  // past the last slot taken
            }
        }
        __syncthreads();
        // 4) pair incoming j -> freed slot j (-> its leaving row demoted to dvict[j]);
        //    update the maps to the state after the gather's moves
        int32_t* ftok = a.fetch_tok + ((size_t)a.layer * a.items_cap + item) * k;
        int32_t* fslot = a.fetch_slot + ((size_t)a.layer * a.items_cap + item) * k;
        int32_t* fdem = a.fetch_dem + ((size_t)a.layer * a.items_cap + item) * k;
        for (int j = threadIdx.x; j < total; j += blockDim.x) {
            const int e = freed[j], pos = need_pos[j], tok = nsel[pos];
            const int x = s_tok[e];  // the leaving token (-1 before the first fill)
            const int s = t2s[tok];  // >= k: resident in the victim area
            int dem = -1;
            if (j < ndem && x >= 0) {
                dem = dvict[j];
                const int y = s_tok[dem];
                if (y >= 0) t2s[y] = -1;  // evicted (y is in neither selection)
                t2s[x] = dem;
                s_tok[dem] = x;
                s_age[dem] = t;
            } else if (x >= 0) {
                t2s[x] = -1;
            }
            if (s >= k) {  // promotion: the victim slot empties
                s_tok[s] = -1;
                s_age[s] = kSlotEmpty;
            }
            t2s[tok] = e;
            s_tok[e] = tok;
            e_slot[pos] = e;
            ftok[j] = s >= k ? -(s + 1) : tok;
            fslot[j] = e;
            fdem[j] = dem;
        }
        for (int i = threadIdx.x; i < k; i += blockDim.x) e_idx[i] = nsel[i];
        if (threadIdx.x == 0) a.fetch_count[(size_t)a.layer * a.items_cap + item] = total;
        __syncthreads();
    }
}


}  // namespace clo
