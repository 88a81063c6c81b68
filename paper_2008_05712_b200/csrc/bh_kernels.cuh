// bh_kernels.cuh -- device code of the Barnes-Hut bucket force path (sm_100a).
//
// Replaces the per-bucket Python loop of eval_forces (hr/workloads/nbody.py:216-250)
// and its numba kernel forces_from_points (hr/kernels.py:70-98), plus the
// opening-angle walk build_interaction_lists (nbody.py:160-199).
//
//  * WALK GROUPS: 32 consecutive buckets (depth-first order), one warp, lane j =
//    bucket j.  The walk is warp-cooperative: every lane evaluates the
//    reference's opening test for its own bucket, the warp descends a node iff
//    some still-active lane opens it.  Each visited node is emitted once per
//    walk group as a UNION entry (node id, accept mask, particle mask); bucket
//    j's interaction list is exactly the entries with bit j set, in emission
//    (= the reference's DFS) order.  Opening tests run in float32 with a
//    rigorous error bound; lanes inside the uncertainty band redo the
//    reference's float64 test bit-exactly (fma-chain norm, IEEE divide).
//  * FORCE GROUPS: <= 32 target particles from consecutive buckets of one walk
//    group, one warp, lane = target.  The walk group's union entries are
//    expanded warp-cooperatively (warp scan) into a shared-memory queue of
//    source records and every record is broadcast to all lanes; lanes whose
//    bucket does not list the entry use mass 0.  FP32 FMA + one MUFU.RSQ on
//    r^6 per interaction; node centres of mass carry a float32 hi/lo split;
//    partial sums are flushed into float64 every FLUSH records.
//  * MEMBER kernel: the per-work-request form (one warp per bucket, lanes
//    split its list) for lists handed in by the host runtime or staged by the
//    data manager.
#pragma once
#include <stdint.h>

namespace gc {

constexpr int WARPS_PER_BLOCK = 8;
constexpr int STACK_CAP = 384;  // pending sibling groups: <= 8 per level; depth <= log2(box/1e-9) (nbody.py:94)
constexpr int MAX_LEVELS = 64;
constexpr int QWIN = 128;  // window of expanded source records per warp
constexpr int FLUSH = 8;  // fp32 partial sums are flushed to fp64 every FLUSH records (the mask loads assume 8)
constexpr int NODE_BITS = 26;  // stack entries pack node | level << NODE_BITS

#ifndef GC_BPL
#define GC_BPL 2
#endif
#ifndef WALK_HALF_SKIP
#define WALK_HALF_SKIP 0
#endif
#ifndef WALK_EMIT_SKIP
#define WALK_EMIT_SKIP 0
#endif
#ifndef WALK_RELU_ADD
#define WALK_RELU_ADD 1
#endif
#ifndef WALK_PROF
#define WALK_PROF 0
#endif
#if WALK_PROF
// [node visits, sum popc(act), visits with one half of act empty, sum popc(acc | part)]
__device__ unsigned long long g_walk_prof[8];  // + [4] first warp start, [5] first warp exit, [6] last warp exit
#endif
constexpr int BPL = GC_BPL;  // buckets per lane in the walk
constexpr int WG_BUCKETS = 32 * BPL;  // buckets per walk group (lane l holds buckets l, l + 32, ...)

struct WalkGroup {
    int bfirst;  // first bucket (depth-first index)
    int nbucket;  // <= WG_BUCKETS
    int fg_first;  // its force groups: [fg_first, fg_first + nfg)
    int nfg;  // <= 32
};

struct ForceGroup {
    int pstart;  // first target in the DFS-sorted particle array
    int ntarget;  // <= 32
    int wg;  // walk group that emits its list
    int boff;  // its buckets: walk-group buckets [boff, boff + nb); list masks use bit j = bucket boff + j
    int nb;  // <= 32
};

struct WalkParams {
    double theta, theta2, root_size;
    float dd2, dd3;  // 2*delta and 3*delta^2: float32 coordinate error bound
    const float2 *tt;  // per level: s > x certainly accepts, s < y certainly rejects (error band folded in)
    int nrep;  // periodic walk (PER instances): images {-nrep..nrep}^3 of the box ...
    double per_L;  // ... of side per_L
};

// periodic images: index i = ((ix + nrep) s + iy + nrep) s + iz + nrep, s = 2 nrep + 1;
// a union entry of image i carries node | i << IMG_SHIFT (node ids < 2^26)
constexpr int IMG_SHIFT = 26;
__host__ __device__ __forceinline__ void image_shift(int img, int nrep, double L, double sh[3])
{
    const int side = 2 * nrep + 1;
    sh[0] = (img / (side * side) - nrep) * L;
    sh[1] = ((img / side) % side - nrep) * L;
    sh[2] = (img % side - nrep) * L;
}

// Walk record per node: float32 centre of mass and a packed word
//   internal: (first_child << 3) | (n_child - 1)                   (>= 8)
//   bucket:   INT_MIN | (pstart << 5) | (pcount - 1), pcount <= 32  (< 0)
constexpr int PSTART_BITS = 26;  // sorted-particle index range of the packed bucket word
__host__ __device__ __forceinline__ int wr_bucket_word(int pstart, int pcount)
{
    return (int)(0x80000000u | ((unsigned)pstart << 5) | (unsigned)(pcount - 1));
}
__device__ __forceinline__ bool wr_bucket(int w) { return w < 0; }
__device__ __forceinline__ int wr_first(int w) { return w >> 3; }
__device__ __forceinline__ int wr_nchild(int w) { return (w & 7) + 1; }
__device__ __forceinline__ int wr_pcount(int w) { return (w & 31) + 1; }
__device__ __forceinline__ int wr_pstart(int w) { return (w >> 5) & ((1 << PSTART_BITS) - 1); }

// ---------------------------------------------------------------------------
// exact float64 opening test (nbody.py:155-157, 178)
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool mac_accept64(const double4 c, const double size, const double4 bg, double theta,
                                             double theta2)
{
    // delta = |com - center| - half ; max(delta, 0)
    const double v0 = fmax(__dsub_rn(fabs(__dsub_rn(c.x, bg.x)), bg.w), 0.0);
    const double v1 = fmax(__dsub_rn(fabs(__dsub_rn(c.y, bg.y)), bg.w), 0.0);
    const double v2 = fmax(__dsub_rn(fabs(__dsub_rn(c.z, bg.z)), bg.w), 0.0);
    // np.linalg.norm -> OpenBLAS ddot: fma chain
    const double s = __fma_rn(v2, v2, __fma_rn(v1, v1, __dmul_rn(v0, v0)));
    if (!(s > 0.0)) return false;  // d > 0.0 fails
    if (s > 1e-280) {  // decided with a 1e-12 relative margin without sqrt/div
        const double q = __dmul_rn(size, size);
        const double r = __dmul_rn(theta2, s);
        if (q < r * (1.0 - 1e-12)) return true;
        if (q > r * (1.0 + 1e-12)) return false;
    }
    return __ddiv_rn(size, __dsqrt_rn(s)) < theta;
}

// ---------------------------------------------------------------------------
// Union lists live in a chunked pool: every force group owns a chain of
// CHUNK-entry chunks allocated on the fly (one atomicAdd per CHUNK entries),
// so a walk over a new tree needs no counting pass.  Entry i of force group f
// is in chunk chain position i / CHUNK, slot i % CHUNK.
// ---------------------------------------------------------------------------
constexpr int CHUNK = 128;  // multiple of 32: a warp's 32-entry read never straddles chunks

// Union entry: (node id, accept mask, particle mask, node's walk word) -- the
// masks are over the walk group's buckets (already restricted to the force
// group); the word gives an opened bucket's particle range without a lookup.
struct UnionPool {
    int4 *ent;
    int *cnext;  // next chunk of the chain
    int *gfirst;  // first chunk per force group
    int *gcount;  // entries per force group
    int *grec;  // source records per force group (node records + opened-bucket particles)
    int *top;  // chunks handed out (may exceed nchunks: overflow, size to retry with)
    int nchunks;  // chunk nchunks is a sink for writes after an overflow
};

// ---------------------------------------------------------------------------
// group walk.  WRITE: emit union entries into the pool; STATS: per-bucket
// [entries, items] (item_count, nbody.py:187-189).
//
// The warp pops a SIBLING GROUP (the children of one opened node, contiguous
// level-order ids) and tests every child against its 32 buckets in one pass,
// pushing the sibling groups of the children some bucket opens.  Each bucket
// sees exactly the reference's decisions (nbody.py:176-186: a node is tested
// for a bucket iff the bucket opened its parent), so its entries are the
// reference's interaction list; only the emission order differs from the
// reference's depth-first order, which union_to_lists restores (sort by
// preorder index) for the per-bucket API.  One pass per sibling group
// amortises the stack traffic over ~7 children.
// ---------------------------------------------------------------------------
#ifndef WALK_MINB
#define WALK_MINB 3
#endif
#ifndef GC_WALK_WPB
#define GC_WALK_WPB 8
#endif
constexpr int WALK_WPB = GC_WALK_WPB;  // warps per walk block (occupancy granularity)
#ifndef WALK_UNROLL
#define WALK_UNROLL 2
#endif
constexpr int kWalkUnroll = WALK_UNROLL;  // sibling-loop unroll
#define WALK_ARGS_DECL                                                                                         \
    int ngroups, const WalkGroup *__restrict__ groups, const ForceGroup *__restrict__ fgroups,                  \
        const float4 *__restrict__ recs, const double4 *__restrict__ com64, const double4 *__restrict__ bgeo,   \
        const float4 *__restrict__ bgeo32, const WalkParams P, UnionPool U, int64_t *__restrict__ bstat,        \
        int *__restrict__ flag, const int *__restrict__ order, int *__restrict__ next, int *__restrict__ wcost,  \
        int *__restrict__ fq, int *__restrict__ fq_tail, int fq_base
#define WALK_ARGS ngroups, groups, fgroups, recs, com64, bgeo, bgeo32, P, U, bstat, flag, order, next, wcost, fq, fq_tail, fq_base
// per-warp walk stack: pending sibling groups (first | (nc - 1) << NODE_BITS,
// active buckets 0-31), active buckets 32-63, level
struct WalkSmem {
    int2 stack[STACK_CAP];
    unsigned act_hi[STACK_CAP];
    unsigned char lvl[STACK_CAP];
};
// level thresholds into shared memory (block-wide, before any warp walks)
__device__ __forceinline__ void load_thresholds(const WalkParams &P, float2 *tt_s)
{
    for (int i = threadIdx.x; i < MAX_LEVELS; i += blockDim.x)
        tt_s[i] = WALK_RELU_ADD ? make_float2(4.f * P.tt[i].x, 4.f * P.tt[i].y) : P.tt[i];
    __syncthreads();
}
template <bool WRITE, bool STATS, bool NREC, bool PER>
__device__ __forceinline__ void walk_group_body(WALK_ARGS_DECL, WalkSmem &ws, float2 *tt_s)
{
    using u64 = unsigned long long;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent warps: walk groups handed out dynamically, in `order` (heaviest
    // first, from the previous walk of this tree) when known
#if WALK_PROF
    {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        if (lane == 0) atomicMin(&g_walk_prof[4], t0);
    }
#endif
    for (;;) {
    int gi = 0;
    if (lane == 0) gi = atomicAdd(next, 1);
    gi = __shfl_sync(0xffffffffu, gi, 0);
    if (gi >= ngroups) {
        // no work left for this warp: a programmatically dependent force
        // kernel (overlap mode) may start taking SM slots
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#if WALK_PROF
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (lane == 0) {
            atomicMin(&g_walk_prof[5], t1);
            atomicMax(&g_walk_prof[6], t1);
        }
#endif
        break;
    }
    // work item: a walk group, or one half of a heavy group's force groups
    // (order entries g * 4 + part, part 0 = all, 1 / 2 = first / second half;
    // negative = no item)
    const int code = order ? order[gi] : 4 * gi;
    if (code < 0) continue;
    const int g = code >> 2, part = code & 3;
    const long long tg0 = clock64();
    const WalkGroup gd = groups[g];
    const int fhalf = (gd.nfg + 1) >> 1;
    const int fa = part == 2 ? fhalf : 0, fb = part == 1 ? fhalf : gd.nfg;  // force groups [fa, fb)
    // lane holds buckets lane and lane + 32 of the group
    float4 bf[BPL];
    u64 inexact = 0ull;  // geometry not float32-exact: always take the float64 test
#pragma unroll
    for (int k = 0; k < BPL; ++k) {
        const int j = lane + 32 * k;
        bf[k] = j < gd.nbucket ? bgeo32[gd.bfirst + j] : make_float4(0.f, 0.f, 0.f, -1.f);
        inexact |= (u64)__ballot_sync(0xffffffffu, bf[k].w < 0.f) << (32 * k);
#if WALK_RELU_ADD
        // NaN propagates through u + |u|: sv = NaN fails both tests -> float64 path
        if (bf[k].w < 0.f) bf[k].x = __int_as_float(0x7fc00000);
#endif
        bf[k].w = fabsf(bf[k].w);
    }
    u64 full = gd.nbucket >= 64 ? ~0ull : ((1ull << gd.nbucket) - 1ull);
    int blo = 0, bhi = gd.nbucket;  // buckets of this item
    if (part) {
        const ForceGroup f0 = fgroups[gd.fg_first + fa], f1 = fgroups[gd.fg_first + fb - 1];
        blo = f0.boff;
        bhi = f1.boff + f1.nb;
        full &= (bhi >= 64 ? ~0ull : ((1ull << bhi) - 1ull)) & ~((1ull << blo) - 1ull);
    }
    const u64 exact = ~inexact;
    int2 *stack = ws.stack;
    unsigned *sact = ws.act_hi;
    unsigned char *slvl = ws.lvl;
    int sp = 0;
    // lane f < nfg emits the list of force group fg_first + f (masks shifted to
    // its own buckets); its current chunk always has room for slot w % CHUNK
    const bool emits = lane < fb - fa;
    const int my_fg = gd.fg_first + fa + (emits ? lane : 0);
    int boff = 0;
    u64 fgm = 0ull;
    if (emits) {
        const ForceGroup fg = fgroups[my_fg];
        boff = fg.boff;
        fgm = ((1ull << fg.nb) - 1ull) << boff;
    }
    int w = 0, chunk = 0, nrec = 0;
    int4 *wp = U.ent;  // next entry slot of this lane's force group
    if (WRITE && emits) {
        chunk = atomicAdd(U.top, 1);
        if (chunk >= U.nchunks) {  // overflow: park in the sink chunk, the host re-walks
            atomicOr(flag, 2);
            chunk = U.nchunks;
        }
        U.gfirst[my_fg] = chunk;
        wp = U.ent + (int64_t)chunk * CHUNK;
    }
    int my_entries[BPL] = {}, my_items[BPL] = {};
#if WALK_PROF
    unsigned long long pv = 0, pa = 0, ph = 0, pe = 0;
#endif
    // periodic walk (PER): the same walk once per image of the box, node
    // centres of mass shifted by the image vector; one chain per force group
    const int nimg = PER ? (2 * P.nrep + 1) * (2 * P.nrep + 1) * (2 * P.nrep + 1) : 1;
    for (int img = 0; img < nimg; ++img) {
    if (sp < 0) break;  // stack overflow in an earlier image (flagged)
    sp = 0;
    float sx = 0.f, sy = 0.f, sz = 0.f;
    double4 sh64 = make_double4(0.0, 0.0, 0.0, 0.0);
    if (PER) {
        double sh[3];
        image_shift(img, P.nrep, P.per_L, sh);
        sx = (float)sh[0];
        sy = (float)sh[1];
        sz = (float)sh[2];
        sh64 = make_double4(sh[0], sh[1], sh[2], 0.0);
    }
    const int img_tag = PER ? img << IMG_SHIFT : 0;
    // the root is a sibling group of one, tested by every bucket
    int first = 0, nc = 1, lvl = 0;
    u64 act = full;
    while (true) {
        const float2 th = tt_s[lvl];
        const int last = first + nc - 1;
        float4 nd = recs[first];
#pragma unroll kWalkUnroll
        for (int node = first; node <= last; ++node) {
            const float4 nd_next = recs[min(node + 1, last)];  // prefetch the next sibling
            const int wd = __float_as_int(nd.w);
            const bool is_bucket = wr_bucket(wd);
            // float32 opening test with error bound: certain accept / certain reject
            u64 acc = 0ull, rej = 0ull;
#pragma unroll
            for (int k = 0; k < BPL; ++k) {
#if WALK_HALF_SKIP
                if (BPL > 1 && (unsigned)(act >> (32 * k)) == 0u) continue;  // warp-uniform: no active bucket here
#endif
#if WALK_RELU_ADD
                // 2 max(u, 0) = u + |u| exactly: an FADD (FMA pipe) instead of an
                // FMNMX (ALU pipe, the walk's bottleneck); sv = 4 s exactly, and
                // the level thresholds are stored x4 (tt_s)
                const float u0 = fabsf((PER ? nd.x + sx : nd.x) - bf[k].x) - bf[k].w;
                const float u1 = fabsf((PER ? nd.y + sy : nd.y) - bf[k].y) - bf[k].w;
                const float u2 = fabsf((PER ? nd.z + sz : nd.z) - bf[k].z) - bf[k].w;
                const float v0 = u0 + fabsf(u0), v1 = u1 + fabsf(u1), v2 = u2 + fabsf(u2);
#else
                const float v0 = fmaxf(fabsf(nd.x - bf[k].x) - bf[k].w, 0.f);
                const float v1 = fmaxf(fabsf(nd.y - bf[k].y) - bf[k].w, 0.f);
                const float v2 = fmaxf(fabsf(nd.z - bf[k].z) - bf[k].w, 0.f);
#endif
                const float sv = fmaf(v2, v2, fmaf(v1, v1, v0 * v0));
                acc |= (u64)__ballot_sync(0xffffffffu, sv > th.x) << (32 * k);
                rej |= (u64)__ballot_sync(0xffffffffu, sv < th.y) << (32 * k);
            }
#if WALK_RELU_ADD
            acc &= act;  // inexact buckets: NaN, in neither mask
#else
            acc &= act & exact;
            rej &= exact;
#endif
            const u64 unsure = ~rej & ~acc & act;
            if (unsure) {  // rare: the reference's float64 test (warp-uniform branch)
#pragma unroll
                for (int k = 0; k < BPL; ++k) {
                    bool a = false;
                    if ((unsure >> (lane + 32 * k)) & 1ull) {
                        double4 c64 = com64[node];
                        if (PER) {  // float64 com + s (the periodic restatement, orc_periodic_forces)
                            c64.x += sh64.x;
                            c64.y += sh64.y;
                            c64.z += sh64.z;
                        }
                        a = mac_accept64(c64, ldexp(P.root_size, -lvl), bgeo[gd.bfirst + lane + 32 * k],
                                         P.theta, P.theta2);
                    }
                    acc |= (u64)__ballot_sync(0xffffffffu, a) << (32 * k);
                }
            }
            const u64 part = is_bucket ? (act & ~acc) : 0ull;
#if WALK_PROF
            pv += 1;
            pa += __popcll(act);
            ph += ((unsigned)act == 0u || (unsigned)(act >> 32) == 0u) ? 1 : 0;
            pe += __popcll(acc | part);
#endif
#if WALK_EMIT_SKIP
            if (WRITE && (acc | part)) {  // warp-uniform: nodes every active bucket opens emit nothing
#else
            if (WRITE) {
#endif
                const unsigned ma = (unsigned)((acc & fgm) >> boff), mp = (unsigned)((part & fgm) >> boff);
                const bool hit = (ma | mp) != 0u;
                if (emits) *wp = make_int4(node | img_tag, (int)ma, (int)mp, wd);
                w += hit ? 1 : 0;
                wp += hit ? 1 : 0;
                if (NREC) nrec += (ma ? 1 : 0) + (mp ? wr_pcount(wd) : 0);
                if (hit && (w & (CHUNK - 1)) == 0) {  // chunk full: link the next one
                    int cn = atomicAdd(U.top, 1);
                    if (cn >= U.nchunks) {
                        atomicOr(flag, 2);
                        cn = U.nchunks;
                    }
                    U.cnext[chunk] = cn;
                    chunk = cn;
                    wp = U.ent + (int64_t)cn * CHUNK;
                }
            }
            if (STATS) {
#pragma unroll
                for (int k = 0; k < BPL; ++k) {
                    const bool a = (acc >> (lane + 32 * k)) & 1ull, p = (part >> (lane + 32 * k)) & 1ull;
                    my_entries[k] += (a || p) ? 1 : 0;
                    my_items[k] += a ? 1 : (p ? wr_pcount(wd) : 0);  // item_count (nbody.py:187-189)
                }
            }
            const u64 open = is_bucket ? 0ull : (act & ~acc);
            if (open) {  // the children wait as one sibling group (nbody.py:184-186)
                if (sp >= STACK_CAP) {
                    if (lane == 0) atomicOr(flag, 1);
                    sp = -1;
                    break;
                }
                // every lane stores the same (warp-uniform) entry: no divergent branch
                stack[sp] = make_int2(wr_first(wd) | ((wd & 7) << NODE_BITS), (int)(unsigned)open);
                sact[sp] = (unsigned)(open >> 32);
                slvl[sp] = (unsigned char)(lvl + 1);
                ++sp;
            }
            nd = nd_next;
        }
        if (sp <= 0) break;
        --sp;
        __syncwarp();
        const int2 top = stack[sp];
        first = top.x & ((1 << NODE_BITS) - 1);
        nc = (top.x >> NODE_BITS) + 1;
        act = (u64)(unsigned)top.y | ((u64)sact[sp] << 32);
        lvl = slvl[sp];
        __syncwarp();
    }
    }  // images
#if WALK_PROF
    if (lane == 0) {
        atomicAdd(&g_walk_prof[0], pv);
        atomicAdd(&g_walk_prof[1], pa);
        atomicAdd(&g_walk_prof[2], ph);
        atomicAdd(&g_walk_prof[3], pe);
    }
#endif
    if (wcost && lane == 0) atomicAdd(wcost + g, (int)min((clock64() - tg0) >> 4, (long long)(INT_MAX / 4)));  // next LPT key
    if (WRITE && emits) {
        U.gcount[my_fg] = w;
        if (NREC) U.grec[my_fg] = nrec;
    }
    if (WRITE && fq) {  // overlap mode: the item's force groups are ready for the force kernel
        __syncwarp();
        __threadfence();
        int base = 0;
        if (lane == 0) base = atomicAdd(fq_tail, fb - fa);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (emits) atomicExch(fq + base + lane, my_fg - fq_base);
    }
    if (STATS) {
#pragma unroll
        for (int k = 0; k < BPL; ++k) {
            const int j = lane + 32 * k;
            if (j >= blo && j < bhi) {
                bstat[2 * (int64_t)(gd.bfirst + j)] = my_entries[k];
                bstat[2 * (int64_t)(gd.bfirst + j) + 1] = my_items[k];
            }
        }
    }
    }  // persistent loop
}

template <bool WRITE, bool STATS, bool NREC = false, bool PER = false>
__global__ void __launch_bounds__(32 * WALK_WPB, WALK_MINB)
walk_group_kernel(int ngroups, const WalkGroup *__restrict__ groups, const ForceGroup *__restrict__ fgroups,
                  const float4 *__restrict__ recs, const double4 *__restrict__ com64,
                  const double4 *__restrict__ bgeo, const float4 *__restrict__ bgeo32, const WalkParams P,
                  UnionPool U, int64_t *__restrict__ bstat, int *__restrict__ flag, const int *__restrict__ order,
                  int *__restrict__ next, int *__restrict__ wcost, int *__restrict__ fq = nullptr,
                  int *__restrict__ fq_tail = nullptr, int fq_base = 0)
{
    __shared__ WalkSmem ws_s[WALK_WPB];
    __shared__ float2 tt_s[MAX_LEVELS];
    load_thresholds(P, tt_s);
    walk_group_body<WRITE, STATS, NREC, PER>(WALK_ARGS, ws_s[threadIdx.x >> 5], tt_s);
}

// Per-bucket walk_order / kind CSR from the union lists (parity + drop-in API):
// each bucket's entries in emission order as (preorder key, id * 2 + kind);
// a segmented sort by key then restores the reference's depth-first order.
static __global__ void __launch_bounds__(32 * WARPS_PER_BLOCK)
union_to_lists_kernel(int nfg, const ForceGroup *__restrict__ fgroups, const WalkGroup *__restrict__ wgroups,
                      const UnionPool U, const int64_t *__restrict__ bptr, const int *__restrict__ preorder,
                      int *__restrict__ key, int *__restrict__ val)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (f >= nfg) return;
    const ForceGroup fg = fgroups[f];
    const unsigned bit = 1u << lane;
    const bool mine = lane < fg.nb;  // lane = the force group's bucket boff + lane
    int64_t cur = mine ? bptr[wgroups[fg.wg].bfirst + fg.boff + lane] : 0;
    const int n = U.gcount[f];
    int chunk = n > 0 ? U.gfirst[f] : 0;
    for (int e = 0; e < n; ++e) {
        if (e > 0 && (e & (CHUNK - 1)) == 0) chunk = U.cnext[chunk];
        const int4 en = U.ent[(int64_t)chunk * CHUNK + (e & (CHUNK - 1))];
        if (mine && ((unsigned)(en.y | en.z) & bit)) {
            key[cur] = preorder[en.x];
            val[cur] = 2 * en.x + (((unsigned)en.y & bit) ? 0 : 1);
            ++cur;
        }
    }
}

// Source records per force group (node records + opened-bucket particles)
// from its union list, one warp per force group: the staged mode's run
// lengths and the pair statistics (the walk itself does not count them).
static __global__ void __launch_bounds__(32 * WARPS_PER_BLOCK) grec_kernel(int nfg, const UnionPool U)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (f >= nfg) return;
    const int n = U.gcount[f];
    int chunk = n > 0 ? U.gfirst[f] : 0, r = 0;
    for (int e0 = 0; e0 < n; e0 += CHUNK) {
        if (e0 > 0) chunk = U.cnext[chunk];
        for (int e = e0 + lane; e < min(n, e0 + CHUNK); e += 32) {
            const int4 en = U.ent[(int64_t)chunk * CHUNK + (e & (CHUNK - 1))];
            r += (en.y ? 1 : 0) + (en.z ? wr_pcount(en.w) : 0);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0) U.grec[f] = r;
}

// ---------------------------------------------------------------------------
// force kernels
// ---------------------------------------------------------------------------
// single MUFU.RSQ of r^6 when eps^6 is a normal float (r^6 >= eps^6); otherwise
// (eps = 0 or tiny, bh_use_cube) the EPS0 instances cube rsqrt(r^2), taking 0
// for r^2 <= kCubeFloor (coincident sources: dx = 0, and 1/r^3 would overflow)
constexpr float kCubeFloor = 1e-25f;
__host__ __device__ inline bool bh_use_cube(float eps2)
{
    return (double)eps2 * (double)eps2 * (double)eps2 < 1.1754943508222875e-38;  // FLT_MIN
}
__device__ __forceinline__ float rsqrt_approx(float x)
{
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// One source record against one target in absolute coordinates.
template <bool EPS0, bool POT>
__device__ __forceinline__ void interact(const float4 h, const float3 l, const float m_eff, const float3 xi,
                                         const float eps2, float3 &a, float &pot)
{
    const float dx = (h.x - xi.x) + l.x, dy = (h.y - xi.y) + l.y, dz = (h.z - xi.z) + l.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, eps2)));
    float inv3;
    if (EPS0) {  // no softening floor: r^6 may leave the float range, cube 1/r instead
        const float ir = rsqrt_approx(r2);
        inv3 = r2 > kCubeFloor ? ir * ir * ir : 0.f;  // coincident source (kernels.py:83-84)
    } else {
        inv3 = rsqrt_approx(r2 * r2 * r2);
    }
    const float w = m_eff * inv3;
    a.x = fmaf(dx, w, a.x);
    a.y = fmaf(dy, w, a.y);
    a.z = fmaf(dz, w, a.z);
    if (POT) pot = fmaf((dx != 0.f || dy != 0.f || dz != 0.f) ? w : 0.f, r2, pot);  // m / sqrt(r^2 + eps^2); coincident skipped (kernels.py:78-84)
}

// One group-relative source record (x, y, z, m) against one target.
template <bool EPS0, bool POT>
__device__ __forceinline__ void interact_rel(const float4 q, const float m_eff, const float3 xi, const float eps2,
                                             float3 &a, float &pot)
{
    const float dx = q.x - xi.x, dy = q.y - xi.y, dz = q.z - xi.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, eps2)));
    float inv3;
    if (EPS0) {  // no softening floor: r^6 may leave the float range, cube 1/r instead
        const float ir = rsqrt_approx(r2);
        inv3 = r2 > kCubeFloor ? ir * ir * ir : 0.f;  // coincident source (kernels.py:83-84)
    } else {
        inv3 = rsqrt_approx(r2 * r2 * r2);
    }
    const float w = m_eff * inv3;
    a.x = fmaf(dx, w, a.x);
    a.y = fmaf(dy, w, a.y);
    a.z = fmaf(dz, w, a.z);
    if (POT) pot = fmaf((dx != 0.f || dy != 0.f || dz != 0.f) ? w : 0.f, r2, pot);  // m / sqrt(r^2 + eps^2); coincident skipped (kernels.py:78-84)
}

__device__ __forceinline__ float warp_min(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Reference point of a force group, per dimension, from its targets' range
// [lo, hi]: a multiple of cgrid (>= the float32 ulp of every coordinate of the
// tree) between 0 and the targets, so target - c and nearby particle - c are
// exact in float32 (both multiples of ulp(p), |p - c| <= |p|).
__device__ __forceinline__ float group_origin(float lo, float hi, float cgrid, float inv_cgrid)
{
    if (lo >= 0.f) return floorf(lo * inv_cgrid) * cgrid;
    if (hi <= 0.f) return -floorf(-hi * inv_cgrid) * cgrid;
    return 0.f;
}

// ---------------------------------------------------------------------------
// Reorganisation + force kernels.
//
// EXPAND (the BH form of the paper's data reorganisation):
// one warp per force group gathers every source record its union list names
// -- the node's centre of mass (hi + lo) and mass, or an opened bucket's
// particles -- from their scattered homes into ONE contiguous staging run of
// float4 (x, y, z, m) records in the group's float32 frame (node COM hi + lo
// folded in once per record instead of once per pair), plus a bucket mask
// per record.  Runs start at multiples of PFLUSH records and are padded with
// massless records.
//
// FORCE: one warp per force group, lane = target, streams its run through
// shared memory (cp.async double buffer, TILE records per stage), transposes
// each stage into PAIRS, A (x0 x1 y0 y1) / B (z0 z1 m0 m1), and evaluates two
// records per step with FADD2/FFMA2/FMUL2 (sm_100 f32x2): half the issue
// slots of scalar FP32 for the same arithmetic.
// ---------------------------------------------------------------------------
constexpr int PFLUSH = 16;  // records per fp64 flush (8 per packed half); run granularity
#ifndef FORCE_TILE
#define FORCE_TILE 64
#endif
constexpr int TILE = FORCE_TILE;  // records per cp.async stage (multiple of 64: 2 records + 2 masks per lane)

struct Staging {
    float4 *rec;  // per record: x, y, z (group frame), m
    unsigned *mask;  // per record: buckets (bits of the walk group) that use it
    const int64_t *rbase;  // first record of each force group's run (multiple of PFLUSH)
    const int *order;  // force groups in processing order
    int *next;  // dynamic work counter of the force kernel
    int *fq;  // overlap mode: force groups in walk-completion order (-1: not yet published)
    int64_t cap;  // records
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// The force group's frame: origin from its targets (see group_origin).
struct GroupFrame {
    float cx, cy, cz;
};
__device__ __forceinline__ GroupFrame group_frame(float4 xp, float cgrid)
{
    const float inv_cgrid = 1.0f / cgrid;  // power of two: exact
    GroupFrame f;
    f.cx = group_origin(warp_min(xp.x), warp_max(xp.x), cgrid, inv_cgrid);
    f.cy = group_origin(warp_min(xp.y), warp_max(xp.y), cgrid, inv_cgrid);
    f.cz = group_origin(warp_min(xp.z), warp_max(xp.z), cgrid, inv_cgrid);
    return f;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

#ifndef EXPAND_MINB
#define EXPAND_MINB 4
#endif
static __global__ void __launch_bounds__(32 * WARPS_PER_BLOCK, EXPAND_MINB)
expand_kernel(int nfg, const ForceGroup *__restrict__ fgroups, const UnionPool U, const float4 *__restrict__ parts,
              const float4 *__restrict__ rec_hi, const float4 *__restrict__ rec_lo, float cgrid, const Staging S,
              int *__restrict__ flag)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (gi >= nfg) return;
    const int64_t rb = S.rbase[gi];
    const int nrec = U.grec[gi];
    const int padded = (nrec + PFLUSH - 1) & ~(PFLUSH - 1);
    if (rb + padded > S.cap) {  // staging too small: the host resizes and re-runs
        if (lane == 0) atomicOr(flag, 4);
        return;
    }
    const ForceGroup fg = fgroups[gi];
    const float4 xp = parts[fg.pstart + min(lane, fg.ntarget - 1)];
    const GroupFrame F = group_frame(xp, cgrid);
    float4 *rec = S.rec + rb;
    unsigned *msk = S.mask + rb;
    // union chunks stream through shared memory, one chunk ahead (cp.async)
    __shared__ __align__(16) int4 ebuf[WARPS_PER_BLOCK][2][CHUNK];
    const int n = U.gcount[gi];
    const int nchunk = (n + CHUNK - 1) / CHUNK;
    int chunk = n > 0 ? U.gfirst[gi] : 0;
    auto fetch = [&](int c, int buf) {
#pragma unroll
        for (int k = 0; k < CHUNK / 32; ++k) cp_async16(&ebuf[warp][buf][lane + 32 * k], U.ent + (int64_t)c * CHUNK + lane + 32 * k);
        cp_async_commit();
    };
    if (nchunk > 0) fetch(chunk, 0);
    int out = 0;  // records written so far
    // one union entry -> its node record and/or its opened bucket's particles
    auto emit = [&](const int4 en, const float4 h, const float4 l) {
        const unsigned mx = (unsigned)en.y, my = (unsigned)en.z;
        const int hasnode = mx ? 1 : 0;
        const int pc = my ? wr_pcount(en.w) : 0;
        const int cnt = hasnode + pc;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int r = out + incl - cnt;  // this entry's first record
        if (mx) {
            rec[r] = make_float4((h.x - F.cx) + l.x, (h.y - F.cy) + l.y, (h.z - F.cz) + l.z, h.w);
            msk[r] = mx;
        }
        // opened buckets: particle k of every entry in round k (loads grouped by 4)
        const int maxpc = (int)__reduce_max_sync(0xffffffffu, (unsigned)pc);
        const float4 *src = parts + wr_pstart(en.w);
        float4 *dst = rec + r + hasnode;
        for (int k0 = 0; k0 < maxpc; k0 += 4) {
            float4 q[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k0 + k < pc) q[k] = src[k0 + k];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k0 + k < pc) {
                    dst[k0 + k] = make_float4(q[k].x - F.cx, q[k].y - F.cy, q[k].z - F.cz, q[k].w);
                    msk[r + hasnode + k0 + k] = my;
                }
        }
        out += total;
    };
    for (int e0 = 0; e0 < n; e0 += 32) {
        const int ci = e0 / CHUNK;
        if ((e0 & (CHUNK - 1)) == 0) {
            __syncwarp();  // the previous chunk's buffer is refilled below
            if (ci + 1 < nchunk) {
                chunk = U.cnext[chunk];
                fetch(chunk, (ci + 1) & 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
        }
        const int e = e0 + lane;
        const int4 en = e < n ? ebuf[warp][ci & 1][e & (CHUNK - 1)] : make_int4(0, 0, 0, 0);
        float4 h = make_float4(0.f, 0.f, 0.f, 0.f), l = h;
        if (en.y) {
            h = rec_hi[en.x];
            l = rec_lo[en.x];
        }
        emit(en, h, l);
    }
    if (out + lane < padded) {
        rec[out + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        msk[out + lane] = 0u;
    }
}

#ifndef FORCE_SCALAR
#define FORCE_SCALAR 0  // 1: scalar FP32 inner loop (A/B reference for the packed f32x2 loop)
#endif
#ifndef FORCE_MINB
#define FORCE_MINB 4  // blocks per SM the force kernel is register-budgeted for
#endif
template <bool EPS0, bool POT>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK, FORCE_MINB)
force_group_kernel(int nfg, const ForceGroup *__restrict__ fgroups, const int *__restrict__ grec, const Staging S,
                   const float4 *__restrict__ parts, const int *__restrict__ part_bucket,
                   const int *__restrict__ porder, const WalkGroup *__restrict__ wgroups, float cgrid, float eps2,
                   double g, int dim, double *__restrict__ out, double *__restrict__ pot_out)
{
    __shared__ __align__(16) float4 t_rec[WARPS_PER_BLOCK][2][TILE];  // cp.async stages (AoS)
    __shared__ __align__(16) unsigned t_m[WARPS_PER_BLOCK][2][TILE];
    __shared__ __align__(16) float4 t_a[WARPS_PER_BLOCK][TILE / 2];  // pairs: x0 x1 y0 y1
    __shared__ __align__(16) float4 t_b[WARPS_PER_BLOCK][TILE / 2];  // pairs: z0 z1 m0 m1
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4 *qa = t_a[warp];
    float4 *qb = t_b[warp];
    const float2 e2 = f2(eps2, eps2);
    // persistent warps: force groups handed out dynamically
    for (int slot = lane == 0 ? atomicAdd(S.next, 1) : 0;;) {
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot >= nfg) break;
        const int gi = S.order[slot];
        const ForceGroup fg = fgroups[gi];
        const int64_t rb = S.rbase[gi];
        const int padded = (grec[gi] + PFLUSH - 1) & ~(PFLUSH - 1);
        // a run beyond the staging capacity was not written (expand flagged it; the host re-runs)
        const int ntile = rb + padded > S.cap ? 0 : (padded + TILE - 1) / TILE;
        // stage tile t of the run into buffer t & 1 (2 records + 2 masks per lane)
        auto issue = [&](int t) {
            const int64_t r0 = rb + (int64_t)t * TILE;
            const int buf = t & 1;
#pragma unroll
            for (int k = 0; k < TILE / 32; ++k)
                cp_async16(&t_rec[warp][buf][lane + 32 * k], S.rec + r0 + lane + 32 * k);
#pragma unroll
            for (int k = 0; k < TILE / 4; k += 32)
                if (k + lane < TILE / 4) cp_async16(&t_m[warp][buf][4 * (k + lane)], S.mask + r0 + 4 * (k + lane));
            cp_async_commit();
        };
        if (ntile > 0) issue(0);
        const bool tgt = lane < fg.ntarget;
        const int p = fg.pstart + (tgt ? lane : 0);
        const float4 xp = parts[p];
        const unsigned mybit = tgt ? (1u << (part_bucket[p] - wgroups[fg.wg].bfirst - fg.boff)) : 0u;
        const GroupFrame F = group_frame(xp, cgrid);
        // target in group coordinates (exact), negated and duplicated for the packed subtract
        const float2 nx = f2(F.cx - xp.x, F.cx - xp.x), ny = f2(F.cy - xp.y, F.cy - xp.y),
                     nz = f2(F.cz - xp.z, F.cz - xp.z);
        double ax = 0.0, ay = 0.0, az = 0.0, ap = 0.0;
        for (int t = 0; t < ntile; ++t) {
            if (t + 1 < ntile) {
                issue(t + 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            const int buf = t & 1;
            if (!FORCE_SCALAR) {  // transpose the stage into pairs
#pragma unroll
                for (int k = 0; k < TILE / 64; ++k) {
                    const int pi = lane + 32 * k;
                    const float4 r0 = t_rec[warp][buf][2 * pi], r1 = t_rec[warp][buf][2 * pi + 1];
                    qa[pi] = make_float4(r0.x, r1.x, r0.y, r1.y);
                    qb[pi] = make_float4(r0.z, r1.z, r0.w, r1.w);
                }
            }
            __syncwarp();
#if FORCE_SCALAR
            const unsigned *qm = t_m[warp][buf];
            const int nin = min(TILE, padded - t * TILE);
            const float4 *qr = t_rec[warp][buf];
            const float3 xr = make_float3(-nx.x, -ny.x, -nz.x);
            for (int j0 = 0; j0 < nin; j0 += PFLUSH) {
                float3 a = make_float3(0.f, 0.f, 0.f);
                float pt = 0.f;
#pragma unroll
                for (int kk = 0; kk < PFLUSH; kk += 4) {
                    const uint4 k4 = *reinterpret_cast<const uint4 *>(qm + j0 + kk);
                    const unsigned ks[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const float4 q = qr[j0 + kk + h];
                        const float me = (ks[h] & mybit) ? q.w : 0.f;
                        interact_rel<EPS0, POT>(q, me, xr, eps2, a, pt);
                    }
                }
                ax += (double)a.x;
                ay += (double)a.y;
                az += (double)a.z;
                if (POT) ap += (double)pt;
            }
#else
            const unsigned *qm = t_m[warp][buf];
            const int nin = min(TILE, padded - t * TILE);
            for (int j0 = 0; j0 < nin; j0 += PFLUSH) {
                float2 sx = f2(0.f, 0.f), sy = f2(0.f, 0.f), sz = f2(0.f, 0.f), sp = f2(0.f, 0.f);
#pragma unroll
                for (int kk = 0; kk < PFLUSH; kk += 4) {
                    const uint4 k4 = *reinterpret_cast<const uint4 *>(qm + j0 + kk);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int pi = (j0 + kk) / 2 + h;
                        const float4 A = qa[pi];
                        const float4 B = qb[pi];
                        const unsigned k0 = h ? k4.z : k4.x, k1 = h ? k4.w : k4.y;
                        const float2 dx = __fadd2_rn(f2(A.x, A.y), nx);
                        const float2 dy = __fadd2_rn(f2(A.z, A.w), ny);
                        const float2 dz = __fadd2_rn(f2(B.x, B.y), nz);
                        float2 r2 = __ffma2_rn(dz, dz, e2);
                        r2 = __ffma2_rn(dy, dy, r2);
                        r2 = __ffma2_rn(dx, dx, r2);
                        float i0, i1;
                        if (EPS0) {  // no softening floor: cube 1/r (r^6 may leave the float range)
                            const float j0 = rsqrt_approx(r2.x), j1 = rsqrt_approx(r2.y);
                            i0 = r2.x > kCubeFloor ? j0 * j0 * j0 : 0.f;  // coincident source (kernels.py:83-84)
                            i1 = r2.y > kCubeFloor ? j1 * j1 * j1 : 0.f;
                        } else {
                            const float2 r6 = __fmul2_rn(__fmul2_rn(r2, r2), r2);
                            i0 = rsqrt_approx(r6.x);
                            i1 = rsqrt_approx(r6.y);
                        }
                        const float2 me = f2((k0 & mybit) ? B.z : 0.f, (k1 & mybit) ? B.w : 0.f);
                        const float2 w = __fmul2_rn(me, f2(i0, i1));
                        sx = __ffma2_rn(dx, w, sx);
                        sy = __ffma2_rn(dy, w, sy);
                        sz = __ffma2_rn(dz, w, sz);
                        if (POT) {  // m / sqrt(r^2 + eps^2); coincident skipped
                            // coincident sources skipped exactly as kernels.py:78-84 (all dx == 0)
                            const float2 wp = f2((dx.x != 0.f || dy.x != 0.f || dz.x != 0.f) ? w.x : 0.f,
                                                 (dx.y != 0.f || dy.y != 0.f || dz.y != 0.f) ? w.y : 0.f);
                            sp = __ffma2_rn(wp, r2, sp);
                        }
                    }
                }
                // fold the packed halves in float32 (8 + 8 terms), accumulate in float64
                ax += (double)(sx.x + sx.y);
                ay += (double)(sy.x + sy.y);
                az += (double)(sz.x + sz.y);
                if (POT) ap += (double)(sp.x + sp.y);
            }
#endif
            __syncwarp();  // stage t & 1 and the pair buffer are rewritten next
        }
        if (tgt) {
            const int orig = porder[p];
            const double gm = g * (double)xp.w;
            out[(int64_t)orig * dim + 0] = gm * ax;
            if (dim > 1) out[(int64_t)orig * dim + 1] = gm * ay;
            if (dim > 2) out[(int64_t)orig * dim + 2] = gm * az;
            if (POT) pot_out[orig] = -gm * ap;  // -G m_i sum_j m_j / sqrt(r^2 + eps^2)
        }
        if (lane == 0) slot = atomicAdd(S.next, 1);
    }
}

// ---------------------------------------------------------------------------
// FUSED reorganisation + force (the default step): the same record sequence
// EXPAND would write into the group's HBM staging run is produced straight
// into a per-warp shared-memory ring, already in the PAIR layout the packed
// force loop reads, and consumed PFLUSH records at a time.  Record order,
// PFLUSH grouping and end padding equal the staged path's, so forces are
// bit-identical to expand_kernel + force_group_kernel; the 1.4 GB staging
// round trip through HBM disappears (sources are gathered from the
// L2-resident tree records and particles).
// ---------------------------------------------------------------------------
#ifndef FUSED_PREFETCH
#define FUSED_PREFETCH 1
#endif
#ifndef FUSED_RING
#define FUSED_RING 128
#endif
constexpr int RING = FUSED_RING;
__device__ __forceinline__ int ld_acquire_gpu(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <bool CG>
__device__ __forceinline__ int ld_list(const int *p)
{
    return CG ? __ldcg(p) : *p;
}
constexpr int RING_LOW = RING / 2;  // produce while fewer records wait (RING >= RING_LOW + 33: one entry always fits)
#define FORCE_ARGS_DECL                                                                                        \
    int nfg, const ForceGroup *__restrict__ fgroups, const UnionPool U, const Staging S,                        \
        const float4 *__restrict__ parts, const float4 *__restrict__ rec_hi, const float4 *__restrict__ rec_lo,  \
        const int *__restrict__ part_bucket, const int *__restrict__ porder, const WalkGroup *__restrict__ wgroups, \
        float cgrid, float eps2, double g, int dim, double *__restrict__ out, double *__restrict__ pot_out,     \
        int per_nrep, double per_L
#define FORCE_ARGS nfg, fgroups, U, S, parts, rec_hi, rec_lo, part_bucket, porder, wgroups, cgrid, eps2, g, dim, out, pot_out, per_nrep, per_L
// per-warp ring of the fused force kernel: record pairs (x0 x1 y0 y1 | z0 z1 m0 m1) + masks
struct RingSmem {
    float4 a[RING / 2];
    float4 b[RING / 2];
    unsigned m[RING];
};
template <bool EPS0, bool POT, bool OVL, bool PER>
__device__ __forceinline__ void force_fused_body(FORCE_ARGS_DECL, RingSmem &rs)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *ra = reinterpret_cast<float *>(rs.a);
    float *rb = reinterpret_cast<float *>(rs.b);
    unsigned *rm = rs.m;
    const float2 e2 = f2(eps2, eps2);
    // record pos -> ring: pair (pos % RING) / 2, half pos & 1
    auto put = [&](int pos, float x, float y, float z, float m, unsigned msk) {
        const int q = pos & (RING - 1), o = (q >> 1) * 4 + (q & 1);
        ra[o] = x;
        ra[o + 2] = y;
        rb[o] = z;
        rb[o + 2] = m;
        rm[q] = msk;
    };
    for (int slot = lane == 0 ? atomicAdd(S.next, 1) : 0;;) {
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot >= nfg) break;
        int gi;
        if (OVL) {  // overlap mode: wait until the walk published this slot (acquire)
            if (lane == 0)
                while ((gi = ld_acquire_gpu(S.fq + slot)) < 0) __nanosleep(64);
            gi = __shfl_sync(0xffffffffu, gi, 0);
        } else {
            gi = S.order[slot];
        }
        const ForceGroup fg = fgroups[gi];
        const bool tgt = lane < fg.ntarget;
        const int p = fg.pstart + (tgt ? lane : 0);
        const float4 xp = parts[p];
        const unsigned mybit = tgt ? (1u << (part_bucket[p] - wgroups[fg.wg].bfirst - fg.boff)) : 0u;
        const GroupFrame F = group_frame(xp, cgrid);
        const float2 nx = f2(F.cx - xp.x, F.cx - xp.x), ny = f2(F.cy - xp.y, F.cy - xp.y),
                     nz = f2(F.cz - xp.z, F.cz - xp.z);
        double ax = 0.0, ay = 0.0, az = 0.0, ap = 0.0;
        // union lists: in overlap mode the walk wrote them during this launch,
        // and neighbouring force groups share lines an SM may have cached in
        // L1 before this group was published -- read them L2-coherent (.cg)
        const int n = ld_list<OVL>(U.gcount + gi);
        int chunk_cur = n > 0 ? ld_list<OVL>(U.gfirst + gi) : 0, cur_ci = 0;
        int chunk_nxt = (n > CHUNK) ? ld_list<OVL>(U.cnext + chunk_cur) : 0;
        int ebase = 0, wr = 0, rd = 0;
        auto load_entry = [&](int e) {
            int4 en = make_int4(0, 0, 0, 0);
            if (e < n) {
                const int c = (e / CHUNK == cur_ci) ? chunk_cur : chunk_nxt;
                en = OVL ? __ldcg(U.ent + (int64_t)c * CHUNK + (e & (CHUNK - 1))) : U.ent[(int64_t)c * CHUNK + (e & (CHUNK - 1))];
            }
            return en;
        };
#if FUSED_PREFETCH
        int pf_base = -1;
        int4 en_pf = make_int4(0, 0, 0, 0);
#if FUSED_PREFETCH > 1
        float4 h_pf = make_float4(0.f, 0.f, 0.f, 0.f), l_pf = h_pf;
#endif
#endif
        for (;;) {
            // produce: whole entries, in order, while the ring holds < RING_LOW records
            while (ebase < n && wr - rd < RING_LOW) {
                const int e = ebase + lane;
#if FUSED_PREFETCH
                const int4 en = pf_base == ebase ? en_pf : load_entry(e);
#else
                const int4 en = load_entry(e);
#endif
                const unsigned mx = (unsigned)en.y, my = (unsigned)en.z;
                const int hasnode = mx ? 1 : 0;
                const int pc = my ? wr_pcount(en.w) : 0;
                const int cnt = hasnode + pc;
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                const bool take = e < n && incl <= RING - (wr - rd);
                const unsigned tm = __ballot_sync(0xffffffffu, take);
                const int ntake = __popc(tm);  // incl is nondecreasing: the taken lanes are a prefix
                const int total = ntake ? __shfl_sync(0xffffffffu, incl, ntake - 1) : 0;
                if (take) {
                    const int r = wr + incl - cnt;
                    // the frame origin of this entry's sources: F, or (periodic) F minus
                    // the image shift -- exact: F and the shift are multiples of cgrid
                    float ox = F.cx, oy = F.cy, oz = F.cz;
                    int nid = en.x;
                    if (PER) {
                        double sh[3];
                        image_shift(en.x >> IMG_SHIFT, per_nrep, per_L, sh);
                        ox = F.cx - (float)sh[0];
                        oy = F.cy - (float)sh[1];
                        oz = F.cz - (float)sh[2];
                        nid = en.x & ((1 << IMG_SHIFT) - 1);
                    }
                    if (mx) {
#if FUSED_PREFETCH > 1
                        const bool pre = !PER && pf_base == ebase;
                        const float4 h = pre ? h_pf : rec_hi[nid], l = pre ? l_pf : rec_lo[nid];
#else
                        const float4 h = rec_hi[nid], l = rec_lo[nid];
#endif
                        put(r, (h.x - ox) + l.x, (h.y - oy) + l.y, (h.z - oz) + l.z, h.w, mx);
                    }
                    const float4 *src = parts + wr_pstart(en.w);
                    for (int k = 0; k < pc; ++k) {
                        const float4 q = src[k];
                        put(r + hasnode + k, q.x - ox, q.y - oy, q.z - oz, q.w, my);
                    }
                }
                wr += total;
                ebase += ntake;
                if (ebase / CHUNK != cur_ci && ebase < n) {  // moved into the next chunk of the chain
                    chunk_cur = chunk_nxt;
                    cur_ci = ebase / CHUNK;
                    chunk_nxt = ((cur_ci + 1) * CHUNK < n) ? ld_list<OVL>(U.cnext + chunk_cur) : 0;
                }
            }
#if FUSED_PREFETCH
            if (ebase < n) {  // the next batch's entries load while this one is consumed
                en_pf = load_entry(ebase + lane);
                pf_base = ebase;
#if FUSED_PREFETCH > 1
                if (en_pf.y) {
                    h_pf = rec_hi[en_pf.x & ((1 << IMG_SHIFT) - 1)];
                    l_pf = rec_lo[en_pf.x & ((1 << IMG_SHIFT) - 1)];
                }
#endif
            }
#endif
            if (ebase >= n && wr - rd < PFLUSH && wr > rd) {  // end of the run: pad the last group
                const int padded = (wr + PFLUSH - 1) & ~(PFLUSH - 1);
                if (wr + lane < padded) put(wr + lane, 0.f, 0.f, 0.f, 0.f, 0u);
                wr = padded;
            }
            if (wr - rd < PFLUSH) break;  // ebase == n and the ring is empty
            __syncwarp();
            // consume every complete PFLUSH group
            for (; wr - rd >= PFLUSH; rd += PFLUSH) {
                const int q0 = rd & (RING - 1);
                const float4 *qa = rs.a + q0 / 2;
                const float4 *qb = rs.b + q0 / 2;
                const unsigned *qm = rm + q0;
                float2 sx = f2(0.f, 0.f), sy = f2(0.f, 0.f), sz = f2(0.f, 0.f), sp = f2(0.f, 0.f);
#pragma unroll
                for (int kk = 0; kk < PFLUSH; kk += 4) {
                    const uint4 k4 = *reinterpret_cast<const uint4 *>(qm + kk);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float4 A = qa[kk / 2 + h];
                        const float4 B = qb[kk / 2 + h];
                        const unsigned k0 = h ? k4.z : k4.x, k1 = h ? k4.w : k4.y;
                        const float2 dx = __fadd2_rn(f2(A.x, A.y), nx);
                        const float2 dy = __fadd2_rn(f2(A.z, A.w), ny);
                        const float2 dz = __fadd2_rn(f2(B.x, B.y), nz);
                        float2 r2 = __ffma2_rn(dz, dz, e2);
                        r2 = __ffma2_rn(dy, dy, r2);
                        r2 = __ffma2_rn(dx, dx, r2);
                        float i0, i1;
                        if (EPS0) {  // no softening floor: cube 1/r (r^6 may leave the float range)
                            const float j0 = rsqrt_approx(r2.x), j1 = rsqrt_approx(r2.y);
                            i0 = r2.x > kCubeFloor ? j0 * j0 * j0 : 0.f;  // coincident source (kernels.py:83-84)
                            i1 = r2.y > kCubeFloor ? j1 * j1 * j1 : 0.f;
                        } else {
                            const float2 r6 = __fmul2_rn(__fmul2_rn(r2, r2), r2);
                            i0 = rsqrt_approx(r6.x);
                            i1 = rsqrt_approx(r6.y);
                        }
                        const float2 me = f2((k0 & mybit) ? B.z : 0.f, (k1 & mybit) ? B.w : 0.f);
                        const float2 w = __fmul2_rn(me, f2(i0, i1));
                        sx = __ffma2_rn(dx, w, sx);
                        sy = __ffma2_rn(dy, w, sy);
                        sz = __ffma2_rn(dz, w, sz);
                        if (POT) {
                            // coincident sources skipped exactly as kernels.py:78-84 (all dx == 0)
                            const float2 wp = f2((dx.x != 0.f || dy.x != 0.f || dz.x != 0.f) ? w.x : 0.f,
                                                 (dx.y != 0.f || dy.y != 0.f || dz.y != 0.f) ? w.y : 0.f);
                            sp = __ffma2_rn(wp, r2, sp);
                        }
                    }
                }
                ax += (double)(sx.x + sx.y);
                ay += (double)(sy.x + sy.y);
                az += (double)(sz.x + sz.y);
                if (POT) ap += (double)(sp.x + sp.y);
            }
            __syncwarp();  // consumed slots are rewritten by the next production
        }
        if (tgt) {
            const int orig = porder[p];
            const double gm = g * (double)xp.w;
            out[(int64_t)orig * dim + 0] = gm * ax;
            if (dim > 1) out[(int64_t)orig * dim + 1] = gm * ay;
            if (dim > 2) out[(int64_t)orig * dim + 2] = gm * az;
            if (POT) pot_out[orig] = -gm * ap;
        }
        __syncwarp();
        if (lane == 0) slot = atomicAdd(S.next, 1);
    }
}

template <bool EPS0, bool POT, bool OVL = false, bool PER = false>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK, FORCE_MINB)
force_fused_kernel(int nfg, const ForceGroup *__restrict__ fgroups, const UnionPool U, const Staging S,
                   const float4 *__restrict__ parts, const float4 *__restrict__ rec_hi,
                   const float4 *__restrict__ rec_lo, const int *__restrict__ part_bucket,
                   const int *__restrict__ porder, const WalkGroup *__restrict__ wgroups, float cgrid, float eps2,
                   double g, int dim, double *__restrict__ out, double *__restrict__ pot_out, int per_nrep = 0,
                   double per_L = 0.0)
{
    __shared__ __align__(16) RingSmem rs_s[WARPS_PER_BLOCK];
    force_fused_body<EPS0, POT, OVL, PER>(FORCE_ARGS, rs_s[threadIdx.x >> 5]);
}

// WALK + FORCE in one persistent kernel (gc_bh_set_overlap(2)): every warp
// first takes walk items (publishing each walk group's force groups to the
// readiness queue), then, with the walk's items exhausted, force groups in
// publication order -- the ALU-bound walk and the FP-bound force loop share
// the SMs instead of running back to back.  No deadlock: a force warp only
// waits for force groups of walk items that resident warps of this same
// grid have claimed.
#ifndef WF_MINB
#define WF_MINB 3
#endif
template <bool EPS0>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK, WF_MINB)
walk_force_kernel(WALK_ARGS_DECL, int nfg, const Staging S, const float4 *__restrict__ parts,
                  const float4 *__restrict__ rec_hi, const float4 *__restrict__ rec_lo,
                  const int *__restrict__ part_bucket, const int *__restrict__ porder, float cgrid, float eps2,
                  double g, int dim, double *__restrict__ out, int force_first)
{
    // a warp is in its walk phase or in its force phase: one private region
    // per warp holds either view
    union __align__(16) WarpSmem {
        WalkSmem w;
        RingSmem r;
    };
    __shared__ WarpSmem u_s[WARPS_PER_BLOCK];
    __shared__ float2 tt_s[MAX_LEVELS];
    WarpSmem &u = u_s[threadIdx.x >> 5];
    load_thresholds(P, tt_s);
    // warps (threadIdx.x >> 5) < force_first consume force groups from the
    // readiness queue from the start (co-resident with the walking warps on
    // every SM), then help with any walk items left; the others walk first
    const bool ff = (int)(threadIdx.x >> 5) < force_first;
    if (!ff) walk_group_body<true, false, false, false>(WALK_ARGS, u.w, tt_s);
    __syncwarp();
    force_fused_body<EPS0, false, true, false>(nfg, fgroups, U, S, parts, rec_hi, rec_lo, part_bucket, porder, groups,
                                               cgrid, eps2, g, dim, out, nullptr, 0, 0.0, u.r);
}

template <bool EPS0>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK)
force_member_kernel(int nmember, const int *__restrict__ member_bucket, const int2 *__restrict__ brange,
                    const int64_t *__restrict__ nptr, const int *__restrict__ naddr,
                    const int64_t *__restrict__ pptr, const int *__restrict__ paddr,
                    const float4 *__restrict__ parts, const int *__restrict__ porder,
                    const float4 *__restrict__ rec_hi, const float4 *__restrict__ rec_lo,
                    const int2 *__restrict__ prange, const float4 *__restrict__ src_parts, float eps2,
                    double g, int dim, double *__restrict__ out)
{
    constexpr int MAXT = 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mi = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (mi >= nmember) return;
    const int2 br = brange[member_bucket[mi]];
    for (int t0 = 0; t0 < br.y; t0 += MAXT) {
        const int nt = min(MAXT, br.y - t0);
        float3 xt[MAXT];
        double ad[MAXT][3];
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
            const float4 q = t < nt ? parts[br.x + t0 + t] : make_float4(0, 0, 0, 0);
            xt[t] = make_float3(q.x, q.y, q.z);
            ad[t][0] = ad[t][1] = ad[t][2] = 0.0;
        }
        float pt = 0.f;
        for (int64_t k0 = nptr[mi]; k0 < nptr[mi + 1]; k0 += 32 * FLUSH) {
            float3 a[MAXT];
#pragma unroll
            for (int t = 0; t < MAXT; ++t) a[t] = make_float3(0.f, 0.f, 0.f);
            for (int64_t k = k0 + lane; k < min(k0 + 32 * FLUSH, nptr[mi + 1]); k += 32) {
                const int id = naddr[k];
                const float4 h = rec_hi[id];
                const float4 l = rec_lo[id];
#pragma unroll
                for (int t = 0; t < MAXT; ++t)
                    if (t < nt) interact<EPS0, false>(h, make_float3(l.x, l.y, l.z), h.w, xt[t], eps2, a[t], pt);
            }
#pragma unroll
            for (int t = 0; t < MAXT; ++t) {
                ad[t][0] += a[t].x;
                ad[t][1] += a[t].y;
                ad[t][2] += a[t].z;
            }
        }
        for (int64_t k = pptr[mi] + lane; k < pptr[mi + 1]; k += 32) {
            const int2 pr = prange[paddr[k]];
            float3 a[MAXT];
#pragma unroll
            for (int t = 0; t < MAXT; ++t) a[t] = make_float3(0.f, 0.f, 0.f);
            for (int q = 0; q < pr.y; ++q) {
                const float4 s = src_parts[pr.x + q];
#pragma unroll
                for (int t = 0; t < MAXT; ++t)
                    if (t < nt) interact<EPS0, false>(s, make_float3(0.f, 0.f, 0.f), s.w, xt[t], eps2, a[t], pt);
            }
#pragma unroll
            for (int t = 0; t < MAXT; ++t) {
                ad[t][0] += a[t].x;
                ad[t][1] += a[t].y;
                ad[t][2] += a[t].z;
            }
        }
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
            if (t < nt) {
                double dx = ad[t][0], dy = ad[t][1], dz = ad[t][2];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    dx += __shfl_xor_sync(0xffffffffu, dx, o);
                    dy += __shfl_xor_sync(0xffffffffu, dy, o);
                    dz += __shfl_xor_sync(0xffffffffu, dz, o);
                }
                if (lane == 0) {
                    const int orig = porder[br.x + t0 + t];
                    const double gm = g * (double)parts[br.x + t0 + t].w;
                    out[(int64_t)orig * dim] = gm * dx;
                    if (dim > 1) out[(int64_t)orig * dim + 1] = gm * dy;
                    if (dim > 2) out[(int64_t)orig * dim + 2] = gm * dz;
                }
            }
        }
    }
}

}  // namespace gc
