// bh.cu -- host side of the Barnes-Hut bucket force path + its C ABI.
// Device code and design notes: bh_kernels.cuh.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "bh_state.h"

#ifndef WALK_LPT
#define WALK_LPT 1  // walk groups heaviest first (0: depth-first order)
#endif
#ifndef WALK_COST_LPT
#define WALK_COST_LPT 1  // heaviest = most cycles in the last walk (0: most union entries)
#endif

using namespace gc;


namespace {

void upload_tree(gc_bh *bh)
{
    cudaStream_t s = bh->ctx->stream;
    const HostTree &t = bh->tree;
    const int64_t nn = t.n_nodes(), nb = (int64_t)t.buckets.size();
    GC_REQUIRE(t.n < (1ll << PSTART_BITS) && nn < (1ll << NODE_BITS), GC_E_VALUE,
               "tree too large for the packed node ids / bucket words");
    std::vector<float4> recs(nn), hi(nn), lo(nn);
    std::vector<double4> c64(nn);
    std::vector<int2> pr(nn);
    std::vector<int> level(nn, 0);
    for (int64_t i = 0; i < nn; ++i)
        for (int c = 0; c < t.n_child[i]; ++c) level[t.first_child[i] + c] = level[i] + 1;
    double cmax = 0.0;
    for (int64_t i = 0; i < nn; ++i) {
        GC_REQUIRE(level[i] < MAX_LEVELS, GC_E_VALUE, "tree deeper than 63 levels");
        GC_REQUIRE(2.0 * t.half[i] == std::ldexp(t.box, -level[i]), GC_E_VALUE, "node size not dyadic in box");
        float h3[3], l3[3];
        for (int k = 0; k < 3; ++k) {
            h3[k] = (float)t.com[3 * i + k];
            l3[k] = (float)(t.com[3 * i + k] - (double)h3[k]);
            cmax = std::max(cmax, std::fabs(t.com[3 * i + k]));
            cmax = std::max(cmax, std::fabs(t.center[3 * i + k]) + t.half[i]);
        }
        int word;
        if (t.first_child[i] < 0) {
            GC_REQUIRE(t.pcount[i] <= 32, GC_E_VALUE,
                       "bucket with more than 32 particles (coincident points) on the group path");
            word = wr_bucket_word((int)t.pstart[i], (int)t.pcount[i]);
        } else {
            word = (int)(t.first_child[i] << 3) | (t.n_child[i] - 1);
        }
        float wf;
        std::memcpy(&wf, &word, 4);
        recs[i] = make_float4(h3[0], h3[1], h3[2], wf);
        c64[i] = make_double4(t.com[3 * i], t.com[3 * i + 1], t.com[3 * i + 2], 0.0);
        hi[i] = make_float4(h3[0], h3[1], h3[2], (float)t.node_mass[i]);
        lo[i] = make_float4(l3[0], l3[1], l3[2], 0.f);
        pr[i] = make_int2((int)t.pstart[i], (int)t.pcount[i]);
    }
    set_tree_bounds(bh, cmax);

    std::vector<double4> bg(nb);
    std::vector<float4> bg32(nb);
    std::vector<int2> br(nb);
    std::vector<int> bids(nb);
    std::vector<int> pb(t.n);
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t id = t.buckets[b];
        bg[b] = make_double4(t.center[3 * id], t.center[3 * id + 1], t.center[3 * id + 2], t.half[id]);
        const float f0 = (float)bg[b].x, f1 = (float)bg[b].y, f2 = (float)bg[b].z, fh = (float)bg[b].w;
        const bool ex = f0 == bg[b].x && f1 == bg[b].y && f2 == bg[b].z && fh == bg[b].w;
        bg32[b] = make_float4(f0, f1, f2, ex ? fh : -1.f);
        br[b] = make_int2((int)t.pstart[id], (int)t.pcount[id]);
        bids[b] = (int)b;
        for (int64_t k = 0; k < t.pcount[id]; ++k) pb[t.pstart[id] + k] = (int)b;
    }
    // walk groups: WG_BUCKETS consecutive buckets; force groups: <= 32 targets
    // of consecutive buckets inside one walk group
    // (an assembled distributed tree may cut them at given buckets: its own
    // buckets then form whole walk groups, gc_bh_set_tree)
    bh->h_wg.clear();
    std::vector<ForceGroup> h_fg;
    size_t cut = 0;
    for (int64_t b0 = 0; b0 < nb;) {
        while (cut < bh->wg_cuts.size() && bh->wg_cuts[cut] <= b0) ++cut;
        const int64_t lim = cut < bh->wg_cuts.size() ? bh->wg_cuts[cut] : nb;
        WalkGroup wg;
        wg.bfirst = (int)b0;
        wg.nbucket = (int)std::min<int64_t>(WG_BUCKETS, lim - b0);
        b0 += wg.nbucket;
        wg.fg_first = (int)h_fg.size();
        const int wi = (int)bh->h_wg.size();
        const int64_t gb0 = wg.bfirst, gb1 = gb0 + wg.nbucket;
        for (int64_t b = gb0; b < gb1;) {
            ForceGroup fg;
            fg.pstart = (int)t.pstart[t.buckets[b]];
            fg.wg = wi;
            fg.boff = (int)(b - gb0);
            int tg = 0;
            while (b < gb1 && tg + t.pcount[t.buckets[b]] <= 32) {
                tg += (int)t.pcount[t.buckets[b]];
                ++b;
            }
            GC_REQUIRE(tg > 0, GC_E_VALUE, "bucket with more than 32 particles (coincident points) on the group path");
            fg.ntarget = tg;
            fg.nb = (int)(b - gb0) - fg.boff;
            h_fg.push_back(fg);
        }
        wg.nfg = (int)h_fg.size() - wg.fg_first;
        GC_REQUIRE(wg.nfg <= 32, GC_E_VALUE, "walk group with more than 32 force groups");
        bh->h_wg.push_back(wg);
    }
    bh->d_recs.upload(recs.data(), nn, s);
    bh->d_com64.upload(c64.data(), nn, s);
    bh->d_rec_hi.upload(hi.data(), nn, s);
    bh->d_rec_lo.upload(lo.data(), nn, s);
    bh->d_prange.upload(pr.data(), nn, s);
    bh->d_bgeo.upload(bg.data(), nb, s);
    bh->d_bgeo32.upload(bg32.data(), nb, s);
    bh->d_brange.upload(br.data(), nb, s);
    bh->d_bucket_ids.upload(bids.data(), nb, s);
    bh->d_part_bucket.upload(pb.data(), t.n, s);
    bh->d_wg.upload(bh->h_wg.data(), bh->h_wg.size(), s);
    bh->n_wg = (int)bh->h_wg.size();
    bh->h_wg_valid = true;
    bh->d_fg.upload(h_fg.data(), h_fg.size(), s);
    bh->n_fg = (int)h_fg.size();
    bh->h2d += nn * (int64_t)(3 * sizeof(float4) + sizeof(double4) + sizeof(int2)) +
               nb * (int64_t)(sizeof(double4) + sizeof(float4) + sizeof(int2) + sizeof(int)) +
               t.n * (int64_t)sizeof(int) + (int64_t)bh->h_wg.size() * (int64_t)sizeof(WalkGroup) +
               (int64_t)h_fg.size() * (int64_t)sizeof(ForceGroup);
    GC_CUDA(cudaStreamSynchronize(s));
}

void upload_particles(gc_bh *bh, const double *pos, const double *mass)
{
    const HostTree &t = bh->tree;
    std::vector<float4> parts(t.n);
    std::vector<int> ord(t.n);
    for (int64_t i = 0; i < t.n; ++i) {
        const int64_t p = t.order[i];
        float c[3] = {0.f, 0.f, 0.f};
        for (int k = 0; k < t.dim; ++k) c[k] = (float)pos[p * t.dim + k];
        parts[i] = make_float4(c[0], c[1], c[2], (float)mass[p]);
        ord[i] = (int)p;
    }
    bh->d_parts.upload(parts.data(), t.n, bh->ctx->stream);
    bh->d_porder.upload(ord.data(), t.n, bh->ctx->stream);
    bh->h2d += t.n * (int64_t)(sizeof(float4) + sizeof(int));
    GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
}

template <class T>
void exclusive_scan(gc_ctx *ctx, const T *in, T *out, int64_t n)
{
    size_t bytes = 0;
    GC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
    ctx->scratch.resize(bytes);
    GC_CUDA(cub::DeviceScan::ExclusiveSum(ctx->scratch.p, bytes, in, out, n, ctx->stream));
}

// host copy of the walk groups (device builds fetch it only for sub-ranges)
void ensure_h_wg(gc_bh *bh)
{
    if (bh->h_wg_valid) return;
    bh->h_wg.resize(bh->n_wg);
    bh->d_wg.download(bh->h_wg.data(), bh->n_wg, bh->ctx->stream);
    GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
    bh->h_wg_valid = true;
}

// first force group of walk group g (g == n_wg: one past the last)
int wg_fg_first(gc_bh *bh, int g)
{
    if (g <= 0) return 0;
    if (g >= bh->n_wg) return bh->n_fg;
    ensure_h_wg(bh);
    return bh->h_wg[g].fg_first;
}

UnionPool pool_view(gc_bh *bh)
{
    UnionPool U;
    U.ent = bh->d_ent.p;
    U.cnext = bh->d_cnext.p;
    U.gfirst = bh->d_gfirst.p;
    U.gcount = bh->d_gcount.p;
    U.grec = bh->d_grec.p;
    U.top = bh->d_top.p;
    U.nchunks = bh->pool_chunks;
    return U;
}

void size_staging(gc_bh *bh, int64_t records)
{
    records = (records + TILE - 1) / TILE * TILE;
    bh->d_srec.resize(records + TILE);  // + one tile: the last cp.async stage may read past a run
    bh->d_smask.resize(records + TILE);
    bh->staging_cap = records;
}

__global__ void bb_iota_kernel(int n, int *p)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// d_grec for the current union lists (all force groups)
void ensure_grec(gc_bh *bh)
{
    if (bh->grec_valid || !bh->have_union) return;
    const int nf = bh->n_fg;
    bh->d_grec.resize(std::max(nf, 1));
    if (nf > 0) {
        grec_kernel<<<grid_for(nf, WARPS_PER_BLOCK), 32 * WARPS_PER_BLOCK, 0, bh->ctx->stream>>>(nf, pool_view(bh));
        check_launch("grec_kernel");
    }
    bh->grec_valid = true;
}

struct RoundRun {  // records of a force group's staging run (multiple of PFLUSH); 0 past the end
    const int *grec;
    int n;
    __host__ __device__ int64_t operator()(int i) const
    {
        return i < n ? (int64_t)((grec[i] + PFLUSH - 1) & ~(PFLUSH - 1)) : 0;
    }
};

void size_pool(gc_bh *bh, int64_t chunks)
{
    GC_REQUIRE(chunks * CHUNK < (1ll << 31), GC_E_VALUE, "union-list pool exceeds 2^31 entries");
    bh->d_ent.resize((chunks + 1) * CHUNK);  // + the overflow sink chunk
    bh->d_cnext.resize(chunks + 1);
    bh->pool_chunks = (int)chunks;
}

// Opening-test thresholds for (tree, theta).
void walk_params(gc_bh *bh, double theta)
{
    if (bh->params_valid && bh->cap_theta == theta) return;
    GC_REQUIRE(bh->per_nrep == 0 || (bh->dim == 3 && bh->per_L == bh->box), GC_E_VALUE,
               "the periodic walk needs a 3-D tree whose box is the periodic box");
    const double th2 = theta * theta;
    const double root = bh->box;
    // Per-level float32 thresholds on the float32 s ~ d^2 (walk_group_kernel).
    // Exact rule: accept iff d^2 > T = size^2 / theta^2 (nbody.py:178), decided
    // with a 2^-22 relative margin (ta, tr) for the float64 rounding.  The
    // float32 s differs from the exact sum by at most
    //   E(s) = dd2 * sum(v) + dd3 + 4.8e-7 s <= dd2 * sqrt(3.000001 s) + dd3 + 4.8e-7 s,
    // so s > A certainly accepts when A - E(A) >= ta and s < R certainly rejects
    // when R + E(R) <= tr (both sides monotone in s there); A and R solve the
    // quadratics in sqrt(s), widened by 1e-6 and rounded outwards.
    double dd2 = bh->walk_dd2, dd3 = bh->walk_dd3;
    if (bh->per_nrep > 0) {
        // periodic images: coordinates up to cmax + nrep L, one more float32
        // rounding (com + shift) in every component
        const double cp = bh->cmax + bh->per_nrep * bh->per_L;
        const double delta = 1.25 * 8.0 * std::ldexp(1.0, -24) * cp;
        dd2 = (float)(2.0 * delta * (1.0 + 1e-6));
        dd3 = (float)(3.0 * delta * delta * (1.0 + 1e-6));
        int e = 0;
        std::frexp(cp, &e);
        bh->cgrid_per = (float)std::ldexp(1.0, e - 24);
        GC_REQUIRE(std::fmod(bh->per_L, (double)bh->cgrid_per) == 0.0, GC_E_VALUE,
                   "periodic box side must be a multiple of the float32 coordinate grid");
    }
    const double c = 4.8e-7, k = dd2 * std::sqrt(3.000001);
    std::vector<float2> tt(MAX_LEVELS);
    for (int l = 0; l < MAX_LEVELS; ++l) {
        const double size = std::ldexp(root, -l);
        const double T = theta > 0.0 ? size * size / th2 : HUGE_VAL;
        const double ta = T * (1.0 + std::ldexp(1.0, -22)), tr = T * (1.0 - std::ldexp(1.0, -22));
        float A = HUGE_VALF, R = -HUGE_VALF;
        if (std::isfinite(ta)) {
            const double u = (k + std::sqrt(k * k + 4.0 * (1.0 - c) * (dd3 + ta))) / (2.0 * (1.0 - c));
            const double a = u * u * (1.0 + 1e-6);
            if (a < 3e38) A = std::nextafter((float)a, HUGE_VALF);
        }
        if (tr > dd3) {
            if (std::isfinite(tr)) {
                const double u = (-k + std::sqrt(k * k + 4.0 * (1.0 + c) * (tr - dd3))) / (2.0 * (1.0 + c));
                R = std::nextafter((float)(u * u * (1.0 - 1e-6)), 0.f);
            } else {
                R = HUGE_VALF;  // theta = 0: nothing is ever accepted, every node is certainly rejected
            }
        }
        tt[l].x = A;
        tt[l].y = R;
    }
    bh->d_tt.upload(tt.data(), MAX_LEVELS, bh->ctx->stream);
    bh->wp.theta = theta;
    bh->wp.theta2 = th2;
    bh->wp.root_size = root;
    bh->wp.dd2 = (float)dd2;
    bh->wp.dd3 = (float)dd3;
    bh->wp.nrep = bh->per_nrep;
    bh->wp.per_L = bh->per_L;
    bh->wp.tt = bh->d_tt.p;
    bh->params_valid = true;
    bh->cap_theta = theta;
    bh->stats_valid = false;
    bh->orders_fresh = false;
    bh->have_union = false;
    bh->dev_lists_valid = false;
}

// One walk launch over the handle's walk-group range (asynchronous).
void launch_walk(gc_bh *bh, bool write, bool stats, int *fq = nullptr, int *fq_tail = nullptr, int fq_base = 0,
                 bool setup_only = false)
{
    wait_orders(bh);
    cudaStream_t s = bh->ctx->stream;
    const int nf = bh->n_fg;
    const int g0 = bh->rg0, g1 = bh->rg1 < 0 ? bh->n_wg : bh->rg1;
    const int ng = g1 - g0;
    const WalkGroup *wg = bh->d_wg.p + g0;
    const unsigned grid = grid_for(std::max(ng, 1), WALK_WPB);
    bh->d_flag.resize(1);
    bh->d_flag.zero(s);
    if (stats) {
        bh->d_bstat.resize(2 * bh->n_buckets);
        bh->d_bstat.zero(s);
    }
    if (write) {
        // first guess ~128 entries per bucket (and image); an overflow grows it to the walk's demand
        const int64_t nimg = bh->per_nrep > 0 ? (int64_t)(2 * bh->per_nrep + 1) * (2 * bh->per_nrep + 1) * (2 * bh->per_nrep + 1) : 1;
        const int64_t guess = (2 * bh->n_buckets + 2 * (int64_t)nf) * (nimg > 1 ? 4 : 1) + 64;
        if (bh->pool_chunks < guess) size_pool(bh, guess);
        bh->d_gfirst.resize(nf);
        bh->d_gcount.resize(nf);
        bh->d_gcount.zero(s);
        bh->d_grec.resize(nf);
        bh->d_grec.zero(s);
        bh->d_top.resize(1);
        bh->d_top.zero(s);
    }
    if (ng <= 0) return;
    if (WALK_COST_LPT) bh->d_wcost.resize(std::max<int64_t>(bh->n_wg, 1));
    const UnionPool U = pool_view(bh);
    // the staged mode needs every force group's record count (its run length);
    // the fused force kernel does not, and the walk skips counting
    const bool nrec = !bh->force_fused;
    auto k = write ? (stats ? (nrec ? walk_group_kernel<true, true, true> : walk_group_kernel<true, true, false>)
                            : (nrec ? walk_group_kernel<true, false, true> : walk_group_kernel<true, false, false>))
                   : walk_group_kernel<false, true>;
    if (bh->per_nrep > 0) {  // periodic walk: the image loop instances (fused force path only)
        GC_REQUIRE(bh->force_fused, GC_E_STATE, "the periodic walk feeds the fused force path only");
        k = write ? (stats ? walk_group_kernel<true, true, false, true> : walk_group_kernel<true, false, false, true>)
                  : walk_group_kernel<false, true, false, true>;
    }
    int per_sm = 0;
    GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * WALK_WPB, 0));
    const unsigned pgrid = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)per_sm * bh->ctx->prop.multiProcessorCount, grid));
    bh->d_wnext.resize(1);
    bh->d_wnext.zero(s);
    const bool ordered = WALK_LPT && bh->order_ng == ng && bh->order_rg0 == g0;
    if (WALK_COST_LPT) GC_CUDA(cudaMemsetAsync(bh->d_wcost.p + g0, 0, sizeof(int) * ng, s));
    if (setup_only) return;  // the caller launches a kernel with the walk inside (walk_force_kernel)
    // with hints: 2 ng work items (heavy groups split in two, -1 padding)
    k<<<pgrid, 32 * WALK_WPB, 0, s>>>(ordered ? 2 * ng : ng, wg, bh->d_fg.p, bh->d_recs.p, bh->d_com64.p,
                                             bh->d_bgeo.p, bh->d_bgeo32.p, bh->wp, U, bh->d_bstat.p, bh->d_flag.p,
                                             ordered ? bh->d_wg_order.p : nullptr, bh->d_wnext.p,
                                             WALK_COST_LPT ? bh->d_wcost.p + g0 : nullptr, fq, fq_tail, fq_base);
    check_launch("walk_group_kernel");
}

#ifndef WALK_SPLIT
#define WALK_SPLIT 0  // > 0: split walk groups costing more than this x the mean into two work items (measured slower: each half re-walks most of the tree)
#endif
__global__ void bh_wg_cost_kernel(int ng, const WalkGroup *__restrict__ wg, const int *__restrict__ gcount,
                                  const int *__restrict__ wcost, int *__restrict__ cost)
{
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ng) return;
    int e = 0;
    if (wcost) {
        e = wcost[g];  // measured cycles of the last walk (/16)
    } else {
        for (int f = wg[g].fg_first; f < wg[g].fg_first + wg[g].nfg; ++f) e += gcount[f];
    }
    cost[g] = e;
}

__global__ void bh_sum_kernel(int n, const int *__restrict__ v, long long *__restrict__ out)
{
    typedef cub::BlockReduce<long long, 1024> Red;
    __shared__ typename Red::TempStorage ts;
    long long t = 0;
    for (int i = threadIdx.x; i < n; i += 1024) t += v[i];
    t = Red(ts).Sum(t);
    if (threadIdx.x == 0) *out = t;
}

// work items of the next walk: a group, or its two halves (by force groups)
// when it costs more than WALK_SPLIT x the mean; keys for the LPT sort
__global__ void bh_wg_items_kernel(int ng, const WalkGroup *__restrict__ wg, const int *__restrict__ cost,
                                   const long long *__restrict__ total, int *__restrict__ key, int *__restrict__ code)
{
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ng) return;
    const int c = cost[g];
    const bool split = WALK_SPLIT > 0 && wg[g].nfg >= 2 && (double)c * ng > WALK_SPLIT * (double)*total;
    key[2 * g] = split ? c / 2 : c;
    code[2 * g] = 4 * g + (split ? 1 : 0);
    key[2 * g + 1] = split ? c / 2 : -1;
    code[2 * g + 1] = split ? 4 * g + 2 : -1;
}

__global__ void bh_fg_key_kernel(int nf, const int *__restrict__ grec, int *__restrict__ key, int *__restrict__ idx)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    key[f] = grec[f];
    idx[f] = f;
}

// Scheduling hints for the persistent walk and force kernels, computed on the
// device (asynchronously) from a completed walk: walk groups heaviest first
// (union entries ~ nodes visited), force groups longest staging run first.
// Exact for later walks of the same tree; after a new tree of the same shape
// (a time step) they are a stale but close hint -- order never changes results.
void make_orders(gc_bh *bh)
{
    if (!bh->order_stream) {
        GC_CUDA(cudaStreamCreateWithFlags(&bh->order_stream, cudaStreamNonBlocking));
        GC_CUDA(cudaEventCreateWithFlags(&bh->order_ready, cudaEventDisableTiming));
        GC_CUDA(cudaEventCreateWithFlags(&bh->order_done, cudaEventDisableTiming));
    }
    wait_orders(bh);
    GC_CUDA(cudaEventRecord(bh->order_ready, bh->ctx->stream));  // the walk / force launch just enqueued
    cudaStream_t s = bh->order_stream;
    GC_CUDA(cudaStreamWaitEvent(s, bh->order_ready, 0));
    const int g0 = bh->rg0, g1 = bh->rg1 < 0 ? bh->n_wg : bh->rg1;
    const int ng = g1 - g0, nf = bh->n_fg;
    if (ng <= 0) return;
    const int f0 = wg_fg_first(bh, g0);
    const int f1 = wg_fg_first(bh, g1);
    const int nfr = f1 - f0;
    auto &k0 = bh->d_okey, &k1 = bh->d_okey2, &i0 = bh->d_oidx;
    const int m = std::max(2 * ng, nfr);
    k0.resize(m); k1.resize(m); i0.resize(m);
    bh->d_wg_order.resize(2 * ng);
    bh->d_fg_lpt.resize(nfr);
    bh->d_wg_total.resize(1);
    bh_wg_cost_kernel<<<grid_for(ng, 256), 256, 0, s>>>(ng, bh->d_wg.p + g0, bh->d_gcount.p,
                                                         WALK_COST_LPT ? bh->d_wcost.p + g0 : nullptr, k1.p);
    bh_sum_kernel<<<1, 1024, 0, s>>>(ng, k1.p, bh->d_wg_total.p);
    size_t bytes = 0;
    bh_wg_items_kernel<<<grid_for(ng, 256), 256, 0, s>>>(ng, bh->d_wg.p + g0, k1.p, bh->d_wg_total.p, k0.p, i0.p);
    bytes = 0;
    GC_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, k0.p, k1.p, i0.p, bh->d_wg_order.p, 2 * ng, 0, 32,
                                                      s));
    bh->order_scratch.resize(bytes);
    GC_CUDA(cub::DeviceRadixSort::SortPairsDescending(bh->order_scratch.p, bytes, k0.p, k1.p, i0.p, bh->d_wg_order.p,
                                                      2 * ng, 0, 32, s));
    // force groups longest first by union entries (a proxy of the run length: the walk does not count records)
    bh_fg_key_kernel<<<grid_for(nfr, 256), 256, 0, s>>>(nfr, bh->d_gcount.p + f0, k0.p, i0.p);
    bytes = 0;
    GC_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, k0.p, k1.p, i0.p, bh->d_fg_lpt.p, nfr, 0, 32, s));
    bh->order_scratch.resize(bytes);
    GC_CUDA(cub::DeviceRadixSort::SortPairsDescending(bh->order_scratch.p, bytes, k0.p, k1.p, i0.p, bh->d_fg_lpt.p, nfr,
                                                      0, 32, s));
    check_launch("make_orders");
    GC_CUDA(cudaEventRecord(bh->order_done, s));
    bh->order_pending = true;
    bh->order_ng = ng;
    bh->order_nf = nfr;
    bh->order_rg0 = g0;
    bh->orders_fresh = true;
}

// Synchronise and surface walk failures.  A pool overflow grows the pool to
// the size the walk asked for and returns true (the caller re-walks).
bool walk_overflowed(gc_bh *bh)
{
    cudaStream_t s = bh->ctx->stream;
    int flag = 0, top = 0;
    bh->d_flag.download(&flag, 1, s);
    if (bh->d_top.p) bh->d_top.download(&top, 1, s);
    GC_CUDA(cudaStreamSynchronize(s));
    GC_REQUIRE(!(flag & 1), GC_E_VALUE, "tree deeper than the walk stack (box too large for half_size >= 1e-9)");
    if (flag & 2) {
        size_pool(bh, (int64_t)top + top / 8 + 64);
        return true;
    }
    if (flag & 4) {  // staging run overflow (expand_kernel): size it to the walk's demand
        int64_t need = 0;
        bh->d_rbase.download(&need, 1, s, bh->d_rbase.n - 1);
        GC_CUDA(cudaStreamSynchronize(s));
        size_staging(bh, need + need / 16);
        return true;
    }
    return false;
}

// Device lists for theta: the walk writes the union pool (and the per-bucket
// stats when requested).  Steady state (same tree and theta, stats known) is
// fully asynchronous; a fresh walk with stats synchronises and retries on a
// pool overflow.
void run_walk(gc_bh *bh, double theta, bool want_stats)
{
    GC_REQUIRE(theta >= 0.0, GC_E_VALUE, "theta must be >= 0");
    GC_REQUIRE(bh->have_tree, GC_E_STATE, "no particles set");
    walk_params(bh, theta);
    const bool stats = want_stats && !bh->stats_valid;
    GC_CUDA(cudaEventRecord(bh->ev[0], bh->ctx->stream));
    launch_walk(bh, true, stats);
    GC_CUDA(cudaEventRecord(bh->ev[1], bh->ctx->stream));
    bh->have_union = true;
    bh->dev_lists_valid = false;
    bh->have_member_lists = false;
    bh->grec_valid = !bh->force_fused;  // the staged mode's walk counted the records
    if (stats) bh->staging_sized = false;  // a new tree / theta (else the lists repeat)
    if (stats) {
        while (walk_overflowed(bh)) launch_walk(bh, true, true);
        bh->stats_valid = true;
        bh->stats_dirty = true;
        // exact staging size of this tree / theta (staged mode; the asynchronous steady state never overflows)
        if (bh->force_fused) return;
        std::vector<int> rec(bh->n_fg);
        bh->d_grec.download(rec.data(), bh->n_fg, bh->ctx->stream);
        GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
        int64_t need = 0;
        for (int r : rec) need += (r + PFLUSH - 1) & ~(PFLUSH - 1);
        if (need > bh->staging_cap) size_staging(bh, need + need / 16);
        bh->staging_sized = true;
    }
}

// Host copies of the per-bucket stats (item counts, entry totals); runs a
// stats-only walk when the current tree/theta has none.
void sync_walk_stats(gc_bh *bh)
{
    cudaStream_t s = bh->ctx->stream;
    if (!bh->stats_valid) {
        GC_REQUIRE(bh->params_valid, GC_E_STATE, "no walk has run (call gc_bh_walk)");
        launch_walk(bh, false, true);
        GC_REQUIRE(!walk_overflowed(bh), GC_E_STATE, "walk overflow in a stats-only walk");
        bh->stats_valid = true;
        bh->stats_dirty = true;
    }
    if (!bh->stats_dirty) return;
    const int64_t nb = bh->n_buckets;
    std::vector<int64_t> st(2 * nb);
    bh->d_bstat.download(st.data(), 2 * nb, s);
    GC_CUDA(cudaStreamSynchronize(s));
    bh->h_item_count.resize(nb);
    int64_t ent = 0;
    for (int64_t b = 0; b < nb; ++b) {
        ent += st[2 * b];
        bh->h_item_count[b] = st[2 * b + 1];
    }
    bh->n_list_entries = ent;
    bh->stats_dirty = false;
}

// Make sure the union pool holds complete lists of the last walk.
void ensure_union_complete(gc_bh *bh)
{
    GC_REQUIRE(bh->have_union, GC_E_STATE, "no device walk has run");
    while (walk_overflowed(bh)) launch_walk(bh, true, false);
}

// The default force kernel: the reorganisation into shared memory fused in
// (PER: the periodic walk's image-tagged entries).
using FusedFn = void (*)(int, const ForceGroup *, const UnionPool, const Staging, const float4 *, const float4 *,
                         const float4 *, const int *, const int *, const WalkGroup *, float, float, double, int,
                         double *, double *, int, double);
template <bool OVL>
FusedFn fused_kernel(bool eps0, bool pot, bool per = false)
{
    if (per) return eps0 ? force_fused_kernel<true, false, OVL, true> : force_fused_kernel<false, false, OVL, true>;
    return eps0 ? (pot ? force_fused_kernel<true, true, OVL> : force_fused_kernel<true, false, OVL>)
                : (pot ? force_fused_kernel<false, true, OVL> : force_fused_kernel<false, false, OVL>);
}

void launch_forces(gc_bh *bh, double g, double eps, bool pot = false)
{
    wait_orders(bh);
    gc_ctx *ctx = bh->ctx;
    cudaStream_t s = ctx->stream;
    bh->d_out.resize(bh->n * bh->dim);
    if (pot) bh->d_pot.resize(bh->n);
    const float eps2 = (float)(eps * eps);
    const bool eps0 = bh_use_cube(eps2);
    GC_CUDA(cudaEventRecord(bh->ev[2], s));
    if (bh->have_union) {
        const int g0 = bh->rg0, g1 = bh->rg1 < 0 ? bh->n_wg : bh->rg1;
        const int f0 = wg_fg_first(bh, g0);
        const int f1 = wg_fg_first(bh, g1);
        const int nfg = f1 - f0;
        const unsigned grid = grid_for(std::max(nfg, 1), WARPS_PER_BLOCK);
        UnionPool U = pool_view(bh);
        U.gfirst += f0;
        U.gcount += f0;
        U.grec += f0;
        if (bh->force_fused) {  // reorganisation into shared memory inside the force kernel
            bh->d_next.resize(1);
            bh->d_next.zero(s);
            const bool lpt = bh->order_nf == nfg && bh->order_rg0 == g0;
            if (!lpt) {
                bh->d_fg_order.resize(nfg);
                if (nfg > 0) bb_iota_kernel<<<grid_for(nfg, 256), 256, 0, s>>>(nfg, bh->d_fg_order.p);
            }
            Staging S{};
            S.order = lpt ? bh->d_fg_lpt.p : bh->d_fg_order.p;
            S.next = bh->d_next.p;
            GC_CUDA(cudaEventRecord(bh->ev[4], s));
            const bool per = bh->per_nrep > 0;
            GC_REQUIRE(!(per && pot), GC_E_STATE, "potentials are not evaluated by the periodic walk");
            auto k = fused_kernel<false>(eps0, pot, per);
            if (nfg > 0) {
                int per_sm = 0;
                GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * WARPS_PER_BLOCK, 0));
                const unsigned pgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(
                    (int64_t)per_sm * ctx->prop.multiProcessorCount, grid_for(nfg, WARPS_PER_BLOCK)));
                k<<<pgrid, 32 * WARPS_PER_BLOCK, 0, s>>>(nfg, bh->d_fg.p + f0, U, S, bh->d_parts.p, bh->d_rec_hi.p,
                                                         bh->d_rec_lo.p, bh->d_part_bucket.p, bh->d_porder.p,
                                                         bh->d_wg.p, per ? bh->cgrid_per : bh->cgrid, eps2, g, bh->dim,
                                                         bh->d_out.p, bh->d_pot.p, bh->per_nrep, bh->per_L);
                check_launch("force_fused_kernel");
            }
            if (!bh->orders_fresh) make_orders(bh);
            GC_CUDA(cudaEventRecord(bh->ev[3], s));
            return;
        }
        GC_REQUIRE(bh->per_nrep == 0, GC_E_STATE, "the periodic walk feeds the fused force path only");
        // staging runs: exclusive scan of the rounded record counts
        ensure_grec(bh);
        bh->d_rbase.resize(nfg + 1);
        {
            auto it = cub::TransformInputIterator<int64_t, RoundRun, cub::CountingInputIterator<int>>(
                cub::CountingInputIterator<int>(0), RoundRun{U.grec, nfg});
            size_t bytes = 0;
            GC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, bh->d_rbase.p, nfg + 1, s));
            ctx->scratch.resize(bytes);
            GC_CUDA(cub::DeviceScan::ExclusiveSum(ctx->scratch.p, bytes, it, bh->d_rbase.p, nfg + 1, s));
        }
        // the staging must hold every run: sized exactly by a staged stats walk,
        // else (lists from a fused-mode walk) from the scan's total, once per walk
        if (!bh->staging_sized) {
            int64_t need = 0;
            bh->d_rbase.download(&need, 1, s, nfg);
            GC_CUDA(cudaStreamSynchronize(s));
            if (need > bh->staging_cap) size_staging(bh, need + need / 16 + 1024);
            bh->staging_sized = true;
        }
        // the persistent force kernel hands out force groups longest run first
        // when a previous walk of this tree/range fixed that order, else in
        // depth-first order (sorting every step costs more than its tail saves)
        bh->d_next.resize(1);
        bh->d_next.zero(s);
        const bool lpt = bh->order_nf == nfg && bh->order_rg0 == g0;
        if (!lpt) {
            bh->d_fg_order.resize(nfg);
            if (nfg > 0) bb_iota_kernel<<<grid_for(nfg, 256), 256, 0, s>>>(nfg, bh->d_fg_order.p);
        }
        Staging S;
        S.rec = bh->d_srec.p;
        S.mask = bh->d_smask.p;
        S.rbase = bh->d_rbase.p;
        S.order = lpt ? bh->d_fg_lpt.p : bh->d_fg_order.p;
        S.next = bh->d_next.p;
        S.cap = bh->staging_cap;
        if (nfg > 0) {
            expand_kernel<<<grid, 32 * WARPS_PER_BLOCK, 0, s>>>(nfg, bh->d_fg.p + f0, U, bh->d_parts.p, bh->d_rec_hi.p,
                                                                bh->d_rec_lo.p, bh->cgrid, S, bh->d_flag.p);
            check_launch("expand_kernel");
        }
        GC_CUDA(cudaEventRecord(bh->ev[4], s));
        auto k = eps0 ? (pot ? force_group_kernel<true, true> : force_group_kernel<true, false>)
                      : (pot ? force_group_kernel<false, true> : force_group_kernel<false, false>);
        if (nfg > 0) {
            int per_sm = 0;
            GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * WARPS_PER_BLOCK, 0));
            const unsigned pgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(
                (int64_t)per_sm * ctx->prop.multiProcessorCount, grid_for(nfg, WARPS_PER_BLOCK)));
            k<<<pgrid, 32 * WARPS_PER_BLOCK, 0, s>>>(nfg, bh->d_fg.p + f0, U.grec, S, bh->d_parts.p,
                                                     bh->d_part_bucket.p, bh->d_porder.p, bh->d_wg.p, bh->cgrid, eps2,
                                                     g, bh->dim, bh->d_out.p, bh->d_pot.p);
            check_launch("force_group_kernel");
        }
        if (!bh->orders_fresh) make_orders(bh);  // hints for the next walk / force launch
    } else if (bh->have_member_lists) {
        GC_REQUIRE(!pot, GC_E_STATE, "potentials need device lists (gc_bh_walk)");
        const int nb = (int)bh->n_buckets;
        const unsigned grid = grid_for(nb, WARPS_PER_BLOCK);
        auto k = eps0 ? force_member_kernel<true> : force_member_kernel<false>;
        GC_CUDA(cudaEventRecord(bh->ev[4], s));
        k<<<grid, 32 * WARPS_PER_BLOCK, 0, s>>>(nb, bh->d_bucket_ids.p, bh->d_brange.p, bh->d_nptr.p,
                                                bh->d_naddr.p, bh->d_pptr.p, bh->d_paddr.p, bh->d_parts.p,
                                                bh->d_porder.p, bh->d_rec_hi.p, bh->d_rec_lo.p, bh->d_prange.p,
                                                bh->d_parts.p, eps2, g, bh->dim, bh->d_out.p);
        check_launch("force_member_kernel");
    } else {
        throw Error{GC_E_STATE, "no interaction lists (call gc_bh_walk or gc_bh_set_lists)"};
    }
    GC_CUDA(cudaEventRecord(bh->ev[3], s));
}

}  // namespace

// Walk and forces of one step overlapped (fused mode): the walk publishes
// each finished walk group's force groups to a device queue and the force
// kernel, launched concurrently on a second stream, consumes them in that
// order -- its blocks take the SM slots the walk's tail frees.
// warps per block of walk_force_kernel that start on force groups
// (GC_WF_FORCE_FIRST, 0 .. WARPS_PER_BLOCK - 1)
static int wf_force_first()
{
    static const int v = [] {
        const char *e = getenv("GC_WF_FORCE_FIRST");
        const int x = e ? atoi(e) : 0;
        return std::max(0, std::min(WARPS_PER_BLOCK - 1, x));
    }();
    return v;
}

void run_overlapped(gc_bh *bh, double theta, double g, double eps)
{
    GC_REQUIRE(theta >= 0.0, GC_E_VALUE, "theta must be >= 0");
    GC_REQUIRE(bh->have_tree, GC_E_STATE, "no particles set");
    walk_params(bh, theta);
    wait_orders(bh);
    gc_ctx *ctx = bh->ctx;
    cudaStream_t s = ctx->stream;
    if (!bh->force_stream) {
        GC_CUDA(cudaStreamCreateWithFlags(&bh->force_stream, cudaStreamNonBlocking));
        GC_CUDA(cudaEventCreateWithFlags(&bh->ov_pre, cudaEventDisableTiming));
        GC_CUDA(cudaEventCreateWithFlags(&bh->ov_done, cudaEventDisableTiming));
    }
    const int g0 = bh->rg0, g1 = bh->rg1 < 0 ? bh->n_wg : bh->rg1;
    const int f0 = wg_fg_first(bh, g0), f1 = wg_fg_first(bh, g1), nfg = f1 - f0;
    bh->d_fq.resize(std::max(nfg, 1));
    GC_CUDA(cudaMemsetAsync(bh->d_fq.p, 0xff, sizeof(int) * std::max(nfg, 1), s));
    bh->d_fq_tail.resize(1);
    bh->d_fq_tail.zero(s);
    bh->d_out.resize(bh->n * bh->dim);
    bh->d_next.resize(1);
    bh->d_next.zero(s);
    GC_CUDA(cudaEventRecord(bh->ev[0], s));
    if (bh->overlap == 2 && nfg > 0 && f0 == 0) {  // one persistent kernel: walk items, then force groups (whole range)
        const int g0w = bh->rg0, ng = (bh->rg1 < 0 ? bh->n_wg : bh->rg1) - g0w;
        launch_walk(bh, true, false, nullptr, nullptr, 0, /*setup_only=*/true);
        const float eps2 = (float)(eps * eps);
        auto k = bh_use_cube(eps2) ? walk_force_kernel<true> : walk_force_kernel<false>;
        int per_sm = 0;
        GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * WARPS_PER_BLOCK, 0));
        const unsigned pgrid = (unsigned)std::max(1, per_sm * ctx->prop.multiProcessorCount);
        const bool ordered = WALK_LPT && bh->order_ng == ng && bh->order_rg0 == g0w;
        UnionPool U = pool_view(bh);
        Staging S{};
        S.next = bh->d_next.p;
        S.fq = bh->d_fq.p;
        k<<<pgrid, 32 * WARPS_PER_BLOCK, 0, s>>>(
            ordered ? 2 * ng : ng, bh->d_wg.p + g0w, bh->d_fg.p, bh->d_recs.p, bh->d_com64.p, bh->d_bgeo.p,
            bh->d_bgeo32.p, bh->wp, U, bh->d_bstat.p, bh->d_flag.p, ordered ? bh->d_wg_order.p : nullptr,
            bh->d_wnext.p, WALK_COST_LPT ? bh->d_wcost.p + g0w : nullptr, bh->d_fq.p, bh->d_fq_tail.p, f0, nfg, S,
            bh->d_parts.p, bh->d_rec_hi.p, bh->d_rec_lo.p, bh->d_part_bucket.p, bh->d_porder.p, bh->cgrid, eps2, g,
            bh->dim, bh->d_out.p, wf_force_first());
        check_launch("walk_force_kernel");
        bh->have_union = true;
        bh->dev_lists_valid = false;
        bh->have_member_lists = false;
        GC_CUDA(cudaEventRecord(bh->ev[1], s));
        GC_CUDA(cudaEventRecord(bh->ev[2], s));
        GC_CUDA(cudaEventRecord(bh->ev[4], s));
        GC_CUDA(cudaEventRecord(bh->ev[3], s));
        if (!bh->orders_fresh) make_orders(bh);
        return;
    }
    launch_walk(bh, true, false, bh->d_fq.p, bh->d_fq_tail.p, f0);
    bh->have_union = true;
    bh->dev_lists_valid = false;
    bh->have_member_lists = false;
    bh->grec_valid = false;
    // the force kernel: programmatic dependent launch on the same stream -- it
    // may start once every walk block has a warp out of work (the walk's
    // tail); readiness per force group comes from the queue, not grid order
    cudaStream_t fs = s;  // nothing may sit between the two launches
    if (nfg > 0) {
        UnionPool U = pool_view(bh);
        U.gfirst += f0;
        U.gcount += f0;
        U.grec += f0;
        Staging S{};
        S.next = bh->d_next.p;
        S.fq = bh->d_fq.p;
        const float eps2 = (float)(eps * eps);
        auto k = fused_kernel<true>(bh_use_cube(eps2), false);
        int per_sm = 0;
        GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * WARPS_PER_BLOCK, 0));
        const unsigned pgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(
            (int64_t)per_sm * ctx->prop.multiProcessorCount, grid_for(nfg, WARPS_PER_BLOCK)));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(pgrid);
        cfg.blockDim = dim3(32 * WARPS_PER_BLOCK);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = fs;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const ForceGroup *fgp = bh->d_fg.p + f0;
        GC_CUDA(cudaLaunchKernelEx(&cfg, k, nfg, fgp, U, S, (const float4 *)bh->d_parts.p,
                                   (const float4 *)bh->d_rec_hi.p, (const float4 *)bh->d_rec_lo.p,
                                   (const int *)bh->d_part_bucket.p, (const int *)bh->d_porder.p,
                                   (const WalkGroup *)bh->d_wg.p, bh->cgrid, eps2, g, bh->dim, bh->d_out.p,
                                   bh->d_pot.p, 0, 0.0));
        check_launch("force_fused_kernel (overlap)");
    }
    // timings in this mode: walk = the whole overlapped step, force = 0
    GC_CUDA(cudaEventRecord(bh->ev[1], fs));
    GC_CUDA(cudaEventRecord(bh->ev[2], fs));
    GC_CUDA(cudaEventRecord(bh->ev[4], fs));
    GC_CUDA(cudaEventRecord(bh->ev[3], fs));
    if (!bh->orders_fresh) make_orders(bh);  // the next walk's order
}

extern "C" {

gc_status gc_bh_create(gc_ctx *ctx, gc_bh **out)
{
    return guard([&] {
        GC_REQUIRE(ctx && out, GC_E_VALUE, "null argument");
        gc_bh *bh = new gc_bh();
        bh->ctx = ctx;
        for (auto &e : bh->ev) GC_CUDA(cudaEventCreate(&e));
        *out = bh;
    });
}

gc_status gc_bh_destroy(gc_bh *bh)
{
    return guard([&] { delete bh; });
}

gc_status gc_bh_set_particles(gc_bh *bh, int64_t n, int32_t dim, const double *pos, const double *mass, double box,
                              int64_t bucket_size)
{
    return guard([&] {
        GC_REQUIRE(bh && pos && mass, GC_E_VALUE, "null argument");
        GC_REQUIRE(n >= 1, GC_E_VALUE, "need at least one particle");
        GC_REQUIRE(bucket_size >= 1, GC_E_VALUE, "bucket_size must be >= 1");
        GC_REQUIRE(bucket_size <= 32, GC_E_VALUE, "bucket_size must be <= 32 on the B200 path");
        GC_REQUIRE(dim >= 1 && dim <= 3, GC_E_VALUE, "dim must be 1..3");
        wait_orders(bh);  // make_orders may still read the previous tree's groups
        device_build_tree(bh, pos, mass, n, dim, box, bucket_size);
        bh->have_tree = true;
        bh->have_union = bh->have_member_lists = false;
        bh->dev_lists_valid = false;
        bh->ew_mom_valid = false;
        bh->params_valid = false;
        bh->stats_valid = false;
        bh->stats_dirty = false;
        bh->orders_fresh = false;
        bh->rg0 = 0;
        bh->rg1 = -1;
    });
}

// walk instrumentation (builds with -DWALK_PROF=1 only; zeros otherwise):
// node visits, sum of active buckets, visits with an empty half, decisions emitted
gc_status gc_debug_walk_prof(int64_t out[6], int32_t reset)
{
    return guard([&] {
        GC_REQUIRE(out, GC_E_VALUE, "null argument");
#if WALK_PROF
        unsigned long long v[8];
        GC_CUDA(cudaMemcpyFromSymbol(v, g_walk_prof, sizeof(v)));
        for (int k = 0; k < 4; ++k) out[k] = (int64_t)v[k];
        out[4] = (int64_t)(v[5] - v[4]);  // first warp out of groups, ns after the first start
        out[5] = (int64_t)(v[6] - v[4]);  // last warp done
        if (reset) {
            const unsigned long long z[8] = {0, 0, 0, 0, ~0ull, ~0ull, 0, 0};
            GC_CUDA(cudaMemcpyToSymbol(g_walk_prof, z, sizeof(z)));
        }
#else
        (void)reset;
        for (int k = 0; k < 6; ++k) out[k] = 0;
#endif
    });
}

// --- distributed BH (bh_dist.py) -------------------------------------------

gc_status gc_bh_set_forced_splits(gc_bh *bh, int64_t n, const int32_t *level, const uint64_t *prefix)
{
    return guard([&] {
        GC_REQUIRE(bh && (n == 0 || (level && prefix)), GC_E_VALUE, "null argument");
        std::vector<std::pair<int, std::pair<uint64_t, uint64_t>>> v((size_t)n);
        for (int64_t i = 0; i < n; ++i) {
            GC_REQUIRE(level[i] >= 0 && level[i] <= 42, GC_E_VALUE, "forced level out of range");
            v[i] = {level[i], {prefix[2 * i] & 0x7fffffffffffffffull, prefix[2 * i + 1] & 0x7fffffffffffffffull}};
        }
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        std::vector<int> lv(v.size());
        std::vector<ulonglong2> kv(v.size());
        for (size_t i = 0; i < v.size(); ++i) {
            lv[i] = v[i].first;
            kv[i] = make_ulonglong2(v[i].second.first, v[i].second.second);
        }
        bh->n_forced = (int)v.size();
        if (v.empty()) {  // cleared: the build takes the bottom-up path again
            bh->d_forced_lvl.resize(1);
            bh->d_forced_key.resize(1);
            return;
        }
        bh->d_forced_lvl.upload(lv.data(), lv.size(), bh->ctx->stream);
        bh->d_forced_key.upload(kv.data(), kv.size(), bh->ctx->stream);
        GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
    });
}

gc_status gc_bh_keys(gc_ctx *ctx, int64_t n, int32_t dim, const double *pos, double box, uint64_t *k1, uint64_t *k2)
{
    return guard([&] {
        GC_REQUIRE(ctx && pos && k1 && k2, GC_E_VALUE, "null argument");
        GC_REQUIRE(dim >= 1 && dim <= 3 && n >= 0, GC_E_VALUE, "bad shape");
        device_keys(ctx, n, dim, pos, box, k1, k2);
    });
}

gc_status gc_bh_set_tree(gc_bh *bh, int64_t n_nodes, int32_t dim, double box, int64_t bucket_size,
                         const double *center, const double *half, const double *mass, const double *com,
                         const int64_t *first_child, const int32_t *n_child, const int64_t *pstart,
                         const int64_t *pcount, int64_t n_buckets, const int64_t *buckets, int64_t n_parts,
                         const int64_t *order, const double *pos, const double *pmass, int64_t n_cuts,
                         const int64_t *cuts)
{
    return guard([&] {
        GC_REQUIRE(bh && center && half && mass && com && first_child && n_child && pstart && pcount && buckets &&
                       order && pos && pmass,
                   GC_E_VALUE, "null argument");
        GC_REQUIRE(n_nodes >= 1 && n_buckets >= 1 && n_parts >= 1 && dim >= 1 && dim <= 3, GC_E_VALUE, "bad sizes");
        // validate the layout (the upload indexes by these values)
        std::vector<char> seen((size_t)n_parts, 0);
        for (int64_t b = 0; b < n_buckets; ++b) {
            const int64_t id = buckets[b];
            GC_REQUIRE(id >= 0 && id < n_nodes && first_child[id] < 0, GC_E_VALUE, "bucket list entry is not a leaf");
            GC_REQUIRE(pstart[id] >= 0 && pcount[id] >= 1 && pstart[id] + pcount[id] <= n_parts, GC_E_VALUE,
                       "bucket particle range out of bounds");
            for (int64_t k = 0; k < pcount[id]; ++k) {
                const int64_t p = order[pstart[id] + k];
                GC_REQUIRE(p >= 0 && p < n_parts && !seen[p], GC_E_VALUE, "order is not a permutation of the particles");
                seen[p] = 1;
            }
        }
        for (int64_t i = 0; i < n_nodes; ++i)
            GC_REQUIRE(first_child[i] < 0 || (n_child[i] >= 1 && first_child[i] > i && first_child[i] + n_child[i] <= n_nodes),
                       GC_E_VALUE, "bad child range");
        wait_orders(bh);
        HostTree &t = bh->tree;
        t.n = n_parts;
        t.dim = dim;
        t.box = box;
        t.bucket_size = bucket_size;
        t.center.assign(3 * (size_t)n_nodes, 0.0);
        t.com.assign(3 * (size_t)n_nodes, 0.0);
        for (int64_t i = 0; i < n_nodes; ++i)
            for (int k = 0; k < dim; ++k) {
                t.center[3 * i + k] = center[i * dim + k];
                t.com[3 * i + k] = com[i * dim + k];
            }
        t.half.assign(half, half + n_nodes);
        t.node_mass.assign(mass, mass + n_nodes);
        t.first_child.assign(first_child, first_child + n_nodes);
        t.n_child.assign(n_child, n_child + n_nodes);
        t.pstart.assign(pstart, pstart + n_nodes);
        t.pcount.assign(pcount, pcount + n_nodes);
        t.buckets.assign(buckets, buckets + n_buckets);
        t.order.assign(order, order + n_parts);
        bh->wg_cuts.assign(cuts, cuts + n_cuts);
        std::sort(bh->wg_cuts.begin(), bh->wg_cuts.end());
        bh->host_tree_valid = true;
        bh->n = n_parts;
        bh->dim = dim;
        bh->box = box;
        bh->bucket_size = bucket_size;
        bh->n_nodes = n_nodes;
        bh->n_buckets = n_buckets;
        upload_tree(bh);
        upload_particles(bh, pos, pmass);
        bh->ws.pos.upload(pos, (size_t)n_parts * dim, bh->ctx->stream);
        bh->ws.mass.upload(pmass, (size_t)n_parts, bh->ctx->stream);
        bh->wg_cuts.clear();
        bh->have_tree = true;
        bh->have_union = bh->have_member_lists = false;
        bh->dev_lists_valid = false;
        bh->ew_mom_valid = false;
        bh->params_valid = false;
        bh->stats_valid = false;
        bh->stats_dirty = false;
        bh->orders_fresh = false;
        bh->rg0 = 0;
        bh->rg1 = -1;
    });
}

gc_status gc_bh_set_overlap(gc_bh *bh, int32_t on)
{
    return guard([&] {
        GC_REQUIRE(bh, GC_E_VALUE, "null argument");
        GC_REQUIRE(on >= 0 && on <= 2, GC_E_VALUE, "overlap mode 0, 1 or 2");
        bh->overlap = on;
    });
}

// One step's walk + forces, asynchronous (gc_bh_walk + gc_bh_forces_async;
// overlapped when gc_bh_set_overlap(1) and the force path is fused).
gc_status gc_bh_walk_forces_async(gc_bh *bh, double theta, double g, double eps)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        // the overlapped walk has no overflow re-walk: only for a (tree, theta)
        // whose pool was sized by a completed stats walk
        if (bh->overlap && bh->force_fused && bh->per_nrep == 0 && bh->stats_valid && bh->params_valid &&
            bh->cap_theta == theta) {
            run_overlapped(bh, theta, g, eps);
        } else {
            run_walk(bh, theta, true);
            launch_forces(bh, g, eps);
        }
    });
}

gc_status gc_bh_set_force_mode(gc_bh *bh, int32_t fused)
{
    return guard([&] {
        GC_REQUIRE(bh, GC_E_VALUE, "null argument");
        bh->force_fused = fused != 0;
    });
}

gc_status gc_bh_set_periodic(gc_bh *bh, int32_t nrep, double L)
{
    return guard([&] {
        GC_REQUIRE(bh, GC_E_VALUE, "null argument");
        GC_REQUIRE(nrep == 0 || nrep == 1, GC_E_VALUE, "nrep must be 0 or 1 (27 images: the image index fits the entry tag)");
        GC_REQUIRE(nrep == 0 || (L > 0.0 && (!bh->have_tree || (bh->dim == 3 && L == bh->box))), GC_E_VALUE,
                   "the periodic box is the tree's 3-D box (L = box)");
        if (bh->per_nrep != nrep || bh->per_L != L) {
            bh->per_nrep = nrep;
            bh->per_L = nrep ? L : 0.0;
            bh->params_valid = false;  // thresholds and coordinate bounds change
            bh->stats_valid = false;
            bh->have_union = false;
            bh->dev_lists_valid = false;
            bh->orders_fresh = false;
        }
    });
}

gc_status gc_bh_sizes(gc_bh *bh, int64_t out[5])
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        out[0] = bh->n_nodes;
        out[1] = bh->n_buckets;
        out[2] = out[3] = out[4] = 0;
        if (bh->params_valid) {
            sync_walk_stats(bh);
            out[2] = bh->n_list_entries;
        }
        if (bh->have_union) {
            ensure_union_complete(bh);
            const size_t nf = bh->d_gcount.n;
            std::vector<int> cnt(nf), rec(nf);
            ensure_grec(bh);
            bh->d_gcount.download(cnt.data(), nf, bh->ctx->stream);
            bh->d_grec.download(rec.data(), nf, bh->ctx->stream);
            GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
            for (size_t f = 0; f < nf; ++f) {
                out[3] += cnt[f];
                out[4] += rec[f];
            }
        }
    });
}

gc_status gc_bh_get_tree(gc_bh *bh, double *center, double *half, double *mass, double *com, int64_t *first_child,
                         int32_t *n_child, int64_t *pcount, int64_t *buckets, int64_t *pidx)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        ensure_host_tree(bh);
        const HostTree &t = bh->tree;
        const int64_t nn = t.n_nodes();
        const int d = t.dim;
        for (int64_t i = 0; i < nn; ++i) {
            for (int k = 0; k < d; ++k) {
                if (center) center[i * d + k] = t.center[3 * i + k];
                if (com) com[i * d + k] = t.com[3 * i + k];
            }
            if (half) half[i] = t.half[i];
            if (mass) mass[i] = t.node_mass[i];
            if (first_child) first_child[i] = t.first_child[i];
            if (n_child) n_child[i] = t.n_child[i];
            if (pcount) pcount[i] = t.pcount[i];
        }
        if (buckets) std::memcpy(buckets, t.buckets.data(), sizeof(int64_t) * t.buckets.size());
        if (pidx) std::memcpy(pidx, t.order.data(), sizeof(int64_t) * t.n);
    });
}

gc_status gc_bh_walk(gc_bh *bh, double theta)
{
    return guard([&] {
        GC_REQUIRE(bh, GC_E_VALUE, "null argument");
        run_walk(bh, theta, true);
    });
}

gc_status gc_bh_get_lists(gc_bh *bh, int64_t *ptr, int64_t *ids, int8_t *kind, int64_t *item_count)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_union, GC_E_STATE, "no device walk has run");
        // with a walk-group range (gc_bh_set_range) the buckets outside it get empty lists
        ensure_union_complete(bh);
        sync_walk_stats(bh);
        cudaStream_t s = bh->ctx->stream;
        const int64_t nb = bh->n_buckets;
        std::vector<int64_t> st(2 * nb);
        bh->d_bstat.download(st.data(), 2 * nb, s);
        GC_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> bptr(nb + 1, 0);
        for (int64_t b = 0; b < nb; ++b) bptr[b + 1] = bptr[b] + st[2 * b];
        const int64_t tot = bptr[nb];
        if (ptr) std::memcpy(ptr, bptr.data(), sizeof(int64_t) * (nb + 1));
        if (item_count)
            for (int64_t b = 0; b < nb; ++b) item_count[b] = st[2 * b + 1];
        if (ids || kind) {
            GC_REQUIRE(bh->per_nrep == 0, GC_E_STATE,
                       "periodic lists carry image shifts: only per-bucket counts (ptr, item_count) are available");
            GC_REQUIRE(tot < (1ll << 31), GC_E_VALUE, "more than 2^31 list entries");
            const int f0 = wg_fg_first(bh, bh->rg0), nf = wg_fg_first(bh, bh->rg1 < 0 ? bh->n_wg : bh->rg1) - f0;
            UnionPool U = pool_view(bh);
            U.gfirst += f0;
            U.gcount += f0;
            // preorder (depth-first, children in octant order) index of every node
            ensure_host_tree(bh);
            const HostTree &t = bh->tree;
            const int64_t nn = t.n_nodes();
            std::vector<int> pre(nn), todo{0};
            int counter = 0;
            while (!todo.empty()) {
                const int v = todo.back();
                todo.pop_back();
                pre[v] = counter++;
                for (int c = t.n_child[v] - 1; c >= 0; --c) todo.push_back((int)(t.first_child[v] + c));
            }
            bh->d_pre.upload(pre.data(), nn, s);
            bh->d_bptr.upload(bptr.data(), nb + 1, s);
            auto &k0 = bh->d_list_key, &k1 = bh->d_list_key2, &v0 = bh->d_list_val, &v1 = bh->d_list_val2;
            k0.resize(tot); k1.resize(tot); v0.resize(tot); v1.resize(tot);
            union_to_lists_kernel<<<grid_for(nf, WARPS_PER_BLOCK), 32 * WARPS_PER_BLOCK, 0, s>>>(
                nf, bh->d_fg.p + f0, bh->d_wg.p, U, bh->d_bptr.p, bh->d_pre.p, k0.p, v0.p);
            check_launch("union_to_lists_kernel");
            size_t bytes = 0;
            GC_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, k0.p, k1.p, v0.p, v1.p, (int)tot, (int)nb,
                                                        bh->d_bptr.p, bh->d_bptr.p + 1, s));
            bh->ctx->scratch.resize(bytes);
            GC_CUDA(cub::DeviceSegmentedSort::SortPairs(bh->ctx->scratch.p, bytes, k0.p, k1.p, v0.p, v1.p, (int)tot,
                                                        (int)nb, bh->d_bptr.p, bh->d_bptr.p + 1, s));
            std::vector<int> tmp(tot);
            v1.download(tmp.data(), tot, s);
            GC_CUDA(cudaStreamSynchronize(s));
            for (int64_t i = 0; i < tot; ++i) {
                if (ids) ids[i] = tmp[i] >> 1;
                if (kind) kind[i] = (int8_t)(tmp[i] & 1);
            }
            // the per-bucket lists stay on the device (d_list_val2: 2 id + kind,
            // d_bptr offsets): the device batcher submits them without a copy
            bh->h_list_ptr = bptr;
            bh->dev_lists_valid = true;
        }
    });
}

gc_status gc_bh_set_lists(gc_bh *bh, int64_t n_buckets, const int64_t *ptr, const int64_t *ids, const int8_t *kind)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        GC_REQUIRE(n_buckets == bh->n_buckets, GC_E_VALUE, "list count != bucket count");
        ensure_host_tree(bh);
        cudaStream_t s = bh->ctx->stream;
        const HostTree &t = bh->tree;
        std::vector<int64_t> np(n_buckets + 1, 0), pp(n_buckets + 1, 0);
        std::vector<int> na, pa;
        na.reserve(ptr[n_buckets]);
        bh->h_item_count.assign(n_buckets, 0);
        for (int64_t b = 0; b < n_buckets; ++b) {
            int64_t items = 0;
            for (int64_t e = ptr[b]; e < ptr[b + 1]; ++e) {
                const int64_t id = ids[e];
                GC_REQUIRE(id >= 0 && id < t.n_nodes(), GC_E_VALUE, "list entry is not a node id");
                if (kind[e] == 0) {
                    na.push_back((int)id);
                    items += 1;
                } else {
                    GC_REQUIRE(t.first_child[id] < 0, GC_E_VALUE, "particle entry is not a bucket");
                    pa.push_back((int)id);
                    items += t.pcount[id];
                }
            }
            np[b + 1] = (int64_t)na.size();
            pp[b + 1] = (int64_t)pa.size();
            bh->h_item_count[b] = items;
        }
        bh->d_nptr.upload(np.data(), n_buckets + 1, s);
        bh->d_pptr.upload(pp.data(), n_buckets + 1, s);
        bh->d_naddr.upload(na.data(), na.size(), s);
        bh->d_paddr.upload(pa.data(), pa.size(), s);
        GC_CUDA(cudaStreamSynchronize(s));
        bh->n_list_entries = ptr[n_buckets];
        bh->have_member_lists = true;
        bh->have_union = false;
    });
}

gc_status gc_bh_forces_async(gc_bh *bh, double g, double eps)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        launch_forces(bh, g, eps);
    });
}

gc_status gc_bh_forces(gc_bh *bh, double g, double eps, double *out)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree && out, GC_E_STATE, "no particles set");
        launch_forces(bh, g, eps);
        // a walk that overflowed the union pool is re-run (pool grown) before its forces count
        while (bh->have_union && walk_overflowed(bh)) {
            launch_walk(bh, true, false);
            launch_forces(bh, g, eps);
        }
        bh->d_out.download(out, bh->n * bh->dim, bh->ctx->stream);
        bh->d2h += bh->n * bh->dim * (int64_t)sizeof(double);
        GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
    });
}

gc_status gc_bh_forces_potential(gc_bh *bh, double g, double eps, double *out, double *pot)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree && out && pot, GC_E_STATE, "no particles set");
        GC_REQUIRE(bh->have_union, GC_E_STATE, "potentials need device lists (gc_bh_walk)");
        ensure_union_complete(bh);
        launch_forces(bh, g, eps, true);
        bh->d_out.download(out, bh->n * bh->dim, bh->ctx->stream);
        bh->d_pot.download(pot, bh->n, bh->ctx->stream);
        GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
    });
}

gc_status gc_bh_interactions(gc_bh *bh, int64_t *out)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        sync_walk_stats(bh);
        ensure_host_tree(bh);
        int64_t tot = 0;
        const HostTree &t = bh->tree;
        for (size_t b = 0; b < bh->h_item_count.size(); ++b) tot += t.pcount[t.buckets[b]] * bh->h_item_count[b];
        *out = tot;
    });
}

// Pairs the force kernel evaluates for the current union lists: out[0] = sum
// over force groups of padded records x 32 lanes (issued), out[1] = padded
// records x targets (lanes with a target); useful interactions are
// gc_bh_interactions (mask efficiency = useful / out[1]).
gc_status gc_bh_pair_stats(gc_bh *bh, int64_t out[2])
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_union && out, GC_E_STATE, "no device walk has run");
        cudaStream_t s = bh->ctx->stream;
        const int nf = bh->n_fg;
        std::vector<int> rec(nf);
        std::vector<ForceGroup> fg(nf);
        ensure_grec(bh);
        bh->d_grec.download(rec.data(), nf, s);
        bh->d_fg.download(fg.data(), nf, s);
        GC_CUDA(cudaStreamSynchronize(s));
        int64_t issued = 0, lanes = 0;
        for (int f = 0; f < nf; ++f) {
            const int64_t padded = (rec[f] + PFLUSH - 1) & ~(PFLUSH - 1);
            issued += 32 * padded;
            lanes += (int64_t)fg[f].ntarget * padded;
        }
        out[0] = issued;
        out[1] = lanes;
    });
}

gc_status gc_bh_set_range(gc_bh *bh, int64_t wg_begin, int64_t wg_end)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        const int64_t ng = (int64_t)bh->n_wg;
        GC_REQUIRE(wg_begin >= 0 && wg_begin <= wg_end && wg_end <= ng, GC_E_VALUE, "bad walk-group range");
        bh->rg0 = (int)wg_begin;
        bh->rg1 = (int)wg_end;
        bh->have_union = false;
        bh->stats_valid = false;  // stats cover the walked range
        bh->orders_fresh = false;
    });
}

gc_status gc_bh_groups(gc_bh *bh, int64_t *n_walk_groups, int64_t *wg_first_bucket)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        *n_walk_groups = (int64_t)bh->n_wg;
        if (wg_first_bucket) {
            ensure_h_wg(bh);
            for (size_t g = 0; g < bh->h_wg.size(); ++g) wg_first_bucket[g] = bh->h_wg[g].bfirst;
            wg_first_bucket[bh->h_wg.size()] = bh->n_buckets;
        }
    });
}

gc_status gc_bh_bucket_work(gc_bh *bh, int64_t *work)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no particles set");
        sync_walk_stats(bh);
        ensure_host_tree(bh);
        const HostTree &t = bh->tree;
        for (size_t b = 0; b < t.buckets.size(); ++b)
            work[b] = b < bh->h_item_count.size() ? t.pcount[t.buckets[b]] * bh->h_item_count[b] : 0;
    });
}

gc_status gc_bh_timings(gc_bh *bh, double out[3])
{
    return guard([&] {
        GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
        // asynchronous walk + forces: an overflowed pool is grown, the step must be repeated
        GC_REQUIRE(!(bh->have_union && walk_overflowed(bh)), GC_E_STATE,
                   "union-list pool overflow (pool grown; re-run gc_bh_walk)");
        float a = 0.f, b = 0.f, c = 0.f;
        out[0] = out[1] = out[2] = 0.0;
        if (cudaEventElapsedTime(&a, bh->ev[0], bh->ev[1]) == cudaSuccess) out[0] = a;
        if (cudaEventElapsedTime(&b, bh->ev[4], bh->ev[3]) == cudaSuccess) out[1] = b;
        if (cudaEventElapsedTime(&c, bh->ev[2], bh->ev[4]) == cudaSuccess) out[2] = c;
        cudaGetLastError();
    });
}

gc_status gc_bh_io_bytes(gc_bh *bh, int64_t out[2], int32_t reset)
{
    return guard([&] {
        out[0] = bh->h2d;
        out[1] = bh->d2h;
        if (reset) bh->h2d = bh->d2h = 0;
    });
}

gc_status gc_bh_step(gc_bh *bh, int64_t n, int32_t dim, const double *pos, const double *mass, double box,
                     int64_t bucket_size, double theta, double g, double eps, double *out)
{
    if (bh) bh->h2d = bh->d2h = 0;
    gc_status st = gc_bh_set_particles(bh, n, dim, pos, mass, box, bucket_size);
    if (st) return st;
    if (bh->overlap && bh->force_fused && bh->per_nrep == 0) {
        st = guard([&] {
            run_overlapped(bh, theta, g, eps);
            // a walk that overflowed the union pool is re-run (pool grown) before its forces count
            while (walk_overflowed(bh)) {
                launch_walk(bh, true, false);
                launch_forces(bh, g, eps);
            }
            bh->d_out.download(out, bh->n * bh->dim, bh->ctx->stream);
            bh->d2h += bh->n * bh->dim * (int64_t)sizeof(double);
            GC_CUDA(cudaStreamSynchronize(bh->ctx->stream));
        });
        return st;
    }
    st = guard([&] { run_walk(bh, theta, false); });  // no per-bucket stats on the step path
    if (st) return st;
    return gc_bh_forces(bh, g, eps, out);
}

}  // extern "C"

namespace gc {
// KernelSpec of the real kernels (replaces hr/devicesim.py:83-108 presets).
// out: threads_per_block, registers_per_thread, shared_mem_per_block,
// members_per_block (work requests one block serves), occupancy blocks/SM.
void bh_kernel_spec(const char *cls, int64_t out[5])
{
    const void *fn;
    if (!strcmp(cls, "walk")) fn = (const void *)walk_group_kernel<true, true>;
    else if (!strcmp(cls, "force_member")) fn = (const void *)force_member_kernel<false>;
    else if (!strcmp(cls, "force")) fn = (const void *)force_group_kernel<false, false>;
    else throw Error{GC_E_VALUE, std::string("unknown kernel class ") + cls};
    cudaFuncAttributes a;
    GC_CUDA(cudaFuncGetAttributes(&a, fn));
    int blocks = 0;
    const int wpb = !strcmp(cls, "walk") ? WALK_WPB : WARPS_PER_BLOCK;
    GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, 32 * wpb, 0));
    out[0] = 32 * wpb;
    out[1] = a.numRegs;
    out[2] = (int64_t)a.sharedSizeBytes;
    out[3] = wpb;
    out[4] = blocks;
}
}  // namespace gc
