// dm_state.h -- the device data manager handle (dm.cu) and the asynchronous
// plan entry points the device batcher (batcher.cu) drives.
#pragma once
#include <vector>

#include "bh_state.h"
#include "common.cuh"

using namespace gc;

struct gc_dm {
    gc_ctx *ctx = nullptr;
    int64_t capacity = 0, slot_bytes = 0;
    int mode = 2;  // 0 redundant, 1 reuse, 2 reuse_sorted (MemoryMode, memory.py:30-33)
    int nslots = 0;
    int64_t free_slots = 0;
    int64_t universe = 0;
    DBuf<int> slot_of, pins, firstpos, buf_of_slot;
    DBuf<double> last_use;
    // plan scratch / outputs
    DBuf<int> ids, sorted_ids, bounds, member_of, distinct, missing, missing_sorted, cand, cand_s, cand_v,
        free_list, addr, runflag, members_tx, iota_slots, nsel;
    DBuf<unsigned char> flag;
    DBuf<unsigned long long> tkeys, tkeys_s;
    DBuf<float4> pool;  // staged payloads, slot_bytes per slot
    // the last plan's transfer list on the device (REDUNDANT: position p -> slot p)
    const int *last_transfer = nullptr;
    int last_nt = 0;
    bool last_redundant = false;
    DBuf<int> members;  // combined request: member buckets
    DBuf<signed char> kinds;  // per plan position: 0 node record, 1 bucket particles
    // last plan (host copies)
    std::vector<int64_t> h_transfer, h_addr, h_tx, h_bounds, h_evicted;
    int64_t total_bytes = 0, indirection_bytes = 0;
    bool indirect = true;
    // asynchronous plans (the device batcher): device counts [distinct, missing,
    // free slots, error flags], per-position kinds in plan order
    DBuf<int> dcnt;
    DBuf<signed char> kinds_s;
    bool free_stale = false;  // free_slots changed on the device (async plans)
    // SortedIndexArray of the observed indices (hr/memory.py:125-179, 252-256):
    // the sorted distinct set on the device, membership flags, counters
    DBuf<int> obs_set, obs_in, obs_ids, obs_first, obs_m, obs_T, obs_tree, obs_new;
    DBuf<unsigned char> obs_flag;
    DBuf<unsigned long long> obs_cmp;
    int64_t obs_n = 0, obs_inserts = 0;
};

namespace gc {
// Asynchronous (no host synchronisation) plan of one combined request whose
// positions are already on the device: ids[P] (int32 buffer ids), kinds[P]
// (0 node, 1 bucket particles), member bounds[M + 1] and member_of[P].  Same
// decisions as gc_dm_build_plan; returns false (nothing enqueued) when the
// plan could need an eviction (ids above the slot count) -- the caller then
// takes the synchronous path.  row[0] += transferred buffers, row[1] +=
// transactions (device).
bool dm_plan_async(gc_dm *dm, const int *ids, const signed char *kinds, int P, const int *bounds,
                   const int *member_of, int M, int64_t max_id, double now, long long *row);
// stage the last async plan's missing buffers and run the member force kernel
// (members[M] = DFS buckets) into the tree's force array
void dm_members_async(gc_dm *dm, gc_bh *bh, const int *members, int M, const int *bounds, int P, double g, double eps);
// error flags accumulated by async plans (reset on read)
int dm_async_errors(gc_dm *dm);
void dm_refresh_free(gc_dm *dm);
void dm_grow_universe(gc_dm *dm, int64_t maxid);
void dm_reserve(gc_dm *dm, int64_t P, int64_t M);
}  // namespace gc
