// bh_state.h -- the Barnes-Hut handle shared by bh.cu (walk, forces, C ABI)
// and bh_build.cu (device tree build).
#pragma once
#include "bh_kernels.cuh"
#include "bh_tree.h"
#include "common.cuh"

#include <algorithm>
#include <cmath>

using namespace gc;

struct BuildWs {  // device-build scratch, kept across builds (no per-step cudaMalloc/cudaFree)
    DBuf<int> nsel2, cpos, ccnt, cbase, bsum, lvlf, big;
    DBuf<double> pos, mass, scratch;
    DBuf<unsigned long long> k1, k2, k1p, k1s, k2s;
    DBuf<int> idx, perm1, perm;
    DBuf<int> lstart, lcount, cstart, ccount, leaf_key, leaf_id, nleaf;
    DBuf<double4> lcenter, ccenter;
    DBuf<int> lk_s;
    DBuf<int> pidx;
    DBuf<double4> com;
    DBuf<double> cmax, cmax_out;
    DBuf<int> nfg_of, fg_base, bad;
    DBuf<signed char> dl, el;  // bottom-up build: adjacent / bucket-window key prefixes
    DBuf<int> range, wcnt, wscan, parent, arrive;
    DBuf<unsigned> words;
    DBuf<double4> spos;  // particles in tree order, float64 (x, y, z, m)
};

struct gc_bh {
    gc_ctx *ctx = nullptr;
    HostTree tree;  // host mirror (valid when host_tree_valid)
    bool have_tree = false;
    bool host_tree_valid = false;
    bool force_fused = true;
    int overlap = 0;  // 1: the force kernel a PDL dependent of the walk (measured neutral); 2: one walk + force kernel (gc_bh_set_overlap)
    cudaStream_t force_stream = nullptr;
    cudaEvent_t ov_pre = nullptr, ov_done = nullptr;
    DBuf<int> d_fq, d_fq_tail;
    bool grec_valid = false;  // d_grec matches the current union lists
    bool staging_sized = false;  // the staging buffer holds the current lists' runs  // reorganise into shared memory inside the force kernel (gc_bh_set_force_mode)
    // tree metadata (always valid once particles are set)
    int64_t n = 0, n_nodes = 0, n_buckets = 0, bucket_size = 8;
    int dim = 3;
    double box = 1.0;
    // device tree topology (device build; downloaded on demand)
    DBuf<double4> d_ncenter;  // per node: center.xyz, half
    DBuf<double> d_nmass;
    DBuf<int> d_first_child, d_nchild, d_pstart, d_pcount, d_buckets;
    std::vector<WalkGroup> h_wg;  // host copy, valid when h_wg_valid
    int n_wg = 0;
    bool h_wg_valid = false;
    int n_fg = 0;  // force groups (device array d_fg)
    // device tree
    DBuf<float4> d_recs;  // walk records: float32 com + packed links
    DBuf<double4> d_com64;  // float64 com (exact opening test)
    DBuf<double4> d_bgeo;  // per bucket (DFS index): center.xyz, half
    DBuf<float4> d_bgeo32;  // float32 copy (w < 0: not exact in float32)
    DBuf<float4> d_parts;  // DFS-sorted particles (x, y, z, m) fp32
    DBuf<int> d_porder;  // original id of each sorted particle
    DBuf<int> d_part_bucket;  // DFS bucket index of each sorted particle
    DBuf<float4> d_rec_hi, d_rec_lo;  // force records: com hi (fp32) + mass, com lo
    DBuf<int2> d_prange;  // per node: (first sorted particle, count) for buckets
    DBuf<int2> d_brange;  // per bucket (DFS index): (first sorted particle, count)
    DBuf<int> d_bucket_ids;  // identity member list for the member kernel
    DBuf<WalkGroup> d_wg;
    DBuf<ForceGroup> d_fg;
    float walk_dd2 = 0.f, walk_dd3 = 0.f;
    DBuf<float2> d_tt;
    // union lists (device walk)
    int rg0 = 0, rg1 = -1;  // walk-group range this handle evaluates (multi-GPU shard)
    bool have_union = false;
    bool params_valid = false;  // walk thresholds for (tree, theta) uploaded
    double cap_theta = -1.0;
    bool stats_valid = false;  // d_bstat describes the current tree + theta
    // chunked union-list pool (bh_kernels.cuh: UnionPool)
    DBuf<int> d_cnext, d_gfirst, d_gcount, d_grec, d_top;
    // staging runs of source records per force group (expand_kernel -> force_group_kernel)
    DBuf<int64_t> d_rbase;
    DBuf<float4> d_srec;
    DBuf<unsigned> d_smask;
    DBuf<int> d_fg_order, d_next;
    // scheduling hints (make_orders): heaviest-first walk groups, longest-run-first
    // force groups of the last completed walk; used while the sizes match
    DBuf<int> d_wcost;  // cycles / 16 of each walk group in the last walk (LPT key)
    DBuf<long long> d_wg_total;  // their sum (split threshold)
    DBuf<int> d_wg_order, d_wnext, d_fg_lpt, d_okey, d_okey2, d_oidx;
    int order_ng = -1, order_nf = -1, order_rg0 = -1;
    bool orders_fresh = false;
    int64_t staging_cap = 0;
    DBuf<int4> d_ent;
    int pool_chunks = 0;
    DBuf<int64_t> d_bstat;
    int64_t n_union = 0;
    float cgrid = 0.f;  // float32 ulp bound of every tree coordinate (force-group origins)
    double cmax = 0.0;  // coordinate bound of the tree (set_tree_bounds)
    // periodic walk (gc_bh_set_periodic): images {-nrep..nrep}^3 of the box of side per_L
    int per_nrep = 0;
    double per_L = 0.0;
    float cgrid_per = 0.f;
    // per-bucket CSR (host-supplied lists)
    bool have_member_lists = false;
    DBuf<int64_t> d_nptr, d_pptr;
    DBuf<int> d_naddr, d_paddr;
    // outputs
    DBuf<double> d_out, d_pot;
    // Ewald kernel class: root moments, staging of the reduction, tables, outputs
    DBuf<double> d_ew_mom, d_ew_part, d_ewf, d_ewp;
    DBuf<double4> d_ew_real, d_ew_k;
    bool ew_mom_valid = false;
    std::vector<int64_t> h_item_count;
    int64_t n_list_entries = 0;
    DBuf<int64_t> d_bptr;
    // per-bucket lists resident on the device after gc_bh_get_lists (ids
    // requested): d_list_val2 = 2 id + kind in bucket order, d_bptr / h_list_ptr
    bool dev_lists_valid = false;
    std::vector<int64_t> h_list_ptr;
    DBuf<int> d_pre, d_list_key, d_list_key2, d_list_val, d_list_val2;
    DBuf<int> d_flag;
    WalkParams wp{};
    bool stats_dirty = false;  // d_bstat newer than the host copies
    // walk begin/end, forces begin/end, reorganisation end (= force kernel begin)
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    BuildWs ws;
    int sort_levels = 10;  // key levels the device build sorts first (grows to 16 when a run exceeds a bucket)
    // distributed BH (bh_dist.py): cubes the device build must split whatever
    // their local count (they straddle ranks; globally they split), as
    // (level, left-aligned key prefix) sorted; walk-group cut points (DFS
    // bucket indices no walk group may straddle) of an assembled tree
    DBuf<ulonglong2> d_forced_key;
    DBuf<int> d_forced_lvl;
    int n_forced = 0;
    std::vector<int64_t> wg_cuts;
    int64_t h2d = 0, d2h = 0;  // bytes moved host<->device since the last reset
    cudaStream_t side = nullptr;  // device build: mass upload overlapping the sort
    cudaEvent_t side_done = nullptr, main_ready = nullptr;
    // scheduling hints (make_orders) run on their own stream, overlapping the
    // force download; the next build / walk / force launch waits for them
    cudaStream_t order_stream = nullptr;
    cudaEvent_t order_ready = nullptr, order_done = nullptr;
    bool order_pending = false;
    DBuf<unsigned char> order_scratch;
    ~gc_bh()
    {
        for (auto &e : ev)
            if (e) cudaEventDestroy(e);
        if (side_done) cudaEventDestroy(side_done);
        if (main_ready) cudaEventDestroy(main_ready);
        if (side) cudaStreamDestroy(side);
        if (order_stream) {
            cudaStreamSynchronize(order_stream);
            cudaStreamDestroy(order_stream);
        }
        if (order_ready) cudaEventDestroy(order_ready);
        if (force_stream) {
            cudaStreamSynchronize(force_stream);
            cudaStreamDestroy(force_stream);
        }
        if (ov_pre) cudaEventDestroy(ov_pre);
        if (ov_done) cudaEventDestroy(ov_done);
        if (order_done) cudaEventDestroy(order_done);
    }
};

namespace gc {
// Coordinate bounds of a tree (cmax >= |every com / particle coordinate|):
// the walk's float32 error band and the force groups' origin grid.
inline void set_tree_bounds(gc_bh *bh, double cmax)
{
    cmax = std::max(cmax, 1e-30);
    bh->cmax = cmax;
    // |v32 - v64| <= delta for every opening-test component (walk_group_kernel):
    // com rounding + two float32 subtractions, each <= 2^-24 * |operand|
    const double delta = 1.25 * 6.0 * std::ldexp(1.0, -24) * cmax;
    bh->walk_dd2 = (float)(2.0 * delta * (1.0 + 1e-6));
    bh->walk_dd3 = (float)(3.0 * delta * delta * (1.0 + 1e-6));
    int e = 0;
    std::frexp(cmax, &e);  // cmax < 2^e, so ulp32(x) <= 2^(e-24) for every |x| <= cmax
    bh->cgrid = (float)std::ldexp(1.0, e - 24);
}
// the main stream waits for the last asynchronous make_orders
inline void wait_orders(gc_bh *bh)
{
    if (bh->order_pending) {
        GC_CUDA(cudaStreamWaitEvent(bh->ctx->stream, bh->order_done, 0));
        bh->order_pending = false;
    }
}
// octant keys of the device build (bb_keys) for host positions (gc_bh_keys)
void device_keys(gc_ctx *ctx, int64_t n, int dim, const double *pos, double box, uint64_t *k1, uint64_t *k2);
void device_build_tree(gc_bh *bh, const double *pos, const double *mass, int64_t n, int dim, double box,
                       int64_t bucket_size);
void ensure_host_tree(gc_bh *bh);
}  // namespace gc
