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
constexpr int STACK_CAP = 384;  // >= 1 + 7*depth; depth <= log2(box/1e-9) (nbody.py:94)
constexpr int MAX_LEVELS = 64;
constexpr int QWIN = 128;  // window of expanded source records per warp
constexpr int FLUSH = 8;  // fp32 partial sums are flushed to fp64 every FLUSH records (the mask loads assume 8)
constexpr int NODE_BITS = 26;  // stack entries pack node | level << NODE_BITS

struct WalkGroup {
    int bfirst;  // first bucket (depth-first index)
    int nbucket;  // <= 32
    int fg_first;  // its force groups: [fg_first, fg_first + nfg)
    int nfg;
};

struct ForceGroup {
    int pstart;  // first target in the DFS-sorted particle array
    int ntarget;  // <= 32
    int wg;  // walk group that emits its list
    unsigned bmask;  // its buckets, as bits of the walk group (bit j = bucket bfirst + j)
};

struct WalkParams {
    double theta, theta2, root_size;
    float dd2, dd3;  // 2*delta and 3*delta^2: float32 coordinate error bound
    const float2 *tt;  // per level: (certain-accept, certain-reject) thresholds on d^2
};

// Walk record per node: float32 centre of mass and a packed word
//   internal: (first_child << 3) | (n_child - 1)     (>= 8)
//   bucket:   -pcount                                (<= -1)
__device__ __forceinline__ bool wr_bucket(int w) { return w < 0; }
__device__ __forceinline__ int wr_first(int w) { return w >> 3; }
__device__ __forceinline__ int wr_nchild(int w) { return (w & 7) + 1; }

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
constexpr int CHUNK = 64;  // multiple of 32: a warp's 32-entry read never straddles chunks

struct UnionPool {
    int *uid;  // node id per entry
    uint2 *umask;  // (accept mask, particle mask) over the walk group's buckets
    int *cnext;  // next chunk of the chain
    int *gfirst;  // first chunk per force group
    int *gcount;  // entries per force group
    int *top;  // chunks handed out (may exceed nchunks: overflow, size to retry with)
    int nchunks;
};

// ---------------------------------------------------------------------------
// group walk.  WRITE: emit union entries into the pool; STATS: per-bucket
// [entries, items] (item_count, nbody.py:187-189).
// ---------------------------------------------------------------------------
template <bool WRITE, bool STATS>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK, 4)
walk_group_kernel(int ngroups, const WalkGroup *__restrict__ groups, const unsigned *__restrict__ fg_mask,
                  const float4 *__restrict__ recs, const double4 *__restrict__ com64,
                  const double4 *__restrict__ bgeo, const float4 *__restrict__ bgeo32, const WalkParams P,
                  UnionPool U, int64_t *__restrict__ bstat, int *__restrict__ flag)
{
    __shared__ int2 stack_s[WARPS_PER_BLOCK][STACK_CAP];
    __shared__ float2 tt_s[MAX_LEVELS];
    for (int i = threadIdx.x; i < MAX_LEVELS; i += blockDim.x) tt_s[i] = P.tt[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (g >= ngroups) return;
    const WalkGroup gd = groups[g];
    const bool has = lane < gd.nbucket;
    const float4 bf = has ? bgeo32[gd.bfirst + lane] : make_float4(0.f, 0.f, 0.f, -1.f);
    const bool exact32 = bf.w >= 0.f;  // bucket geometry representable in float32
    const unsigned full = gd.nbucket == 32 ? 0xffffffffu : ((1u << gd.nbucket) - 1u);
    const unsigned bit = 1u << lane;
    int2 *stack = stack_s[warp];
    int sp = 0;
    // lane f < nfg emits the list of force group fg_first + f
    const bool emits = lane < gd.nfg;
    const int my_fg = gd.fg_first + (emits ? lane : 0);
    const unsigned fgm = emits ? fg_mask[my_fg] : 0u;
    int w = 0, chunk = 0;
    int my_entries = 0, my_items = 0;
    int node = 0, lvl = 0;
    unsigned act = full;
    float4 nd = recs[0];
    while (true) {
        const int wd = __float_as_int(nd.w);
        const bool is_bucket = wr_bucket(wd);
        const int fc = wr_first(wd);
        // speculative loads of both possible successors
        const int2 top = sp > 0 ? stack[sp - 1] : make_int2(0, 0);
        const float4 n_open = recs[is_bucket ? 0 : fc];
        const float4 n_pop = recs[top.x & ((1 << NODE_BITS) - 1)];
        // float32 opening test with error bound: certain accept / reject
        const float v0 = fmaxf(fabsf(nd.x - bf.x) - bf.w, 0.f);
        const float v1 = fmaxf(fabsf(nd.y - bf.y) - bf.w, 0.f);
        const float v2 = fmaxf(fabsf(nd.z - bf.z) - bf.w, 0.f);
        const float s = fmaf(v2, v2, fmaf(v1, v1, v0 * v0));
        const float err = fmaf(P.dd2, v0 + v1 + v2, fmaf(s, 4.8e-7f, P.dd3));
        const float2 th = tt_s[lvl];
        const bool mine = act & bit;
        bool acc = mine && exact32 && (s - err > th.x);
        const bool unsure = mine && !acc && !(exact32 && (s + err < th.y));
        if (__any_sync(0xffffffffu, unsure)) {
            if (unsure)
                acc = mac_accept64(com64[node], ldexp(P.root_size, -lvl), bgeo[gd.bfirst + lane], P.theta, P.theta2);
        }
        const unsigned acc_m = __ballot_sync(0xffffffffu, acc);
        const unsigned part_m = is_bucket ? (act & ~acc_m) : 0u;
        const unsigned hit = (acc_m | part_m) & fgm;
        if (WRITE && hit) {
            const int slot = w & (CHUNK - 1);
            if (slot == 0) {
                const int c = atomicAdd(U.top, 1);
                if (w == 0) U.gfirst[my_fg] = c;
                else if (chunk < U.nchunks) U.cnext[chunk] = c;
                chunk = c;
            }
            if (chunk < U.nchunks) {
                const int at = chunk * CHUNK + slot;
                U.uid[at] = node;
                U.umask[at] = make_uint2(acc_m & fgm, part_m & fgm);
            } else if (slot == 0) {
                atomicOr(flag, 2);
            }
        }
        w += hit ? 1 : 0;
        if (STATS) {
            const bool a = acc_m & bit, p = part_m & bit;
            my_entries += (a || p) ? 1 : 0;
            my_items += a ? 1 : (p ? -wd : 0);  // item_count (nbody.py:187-189)
        }
        const unsigned open = is_bucket ? 0u : (act & ~acc_m);
        if (open) {
            // children 1..nc-1 wait on the stack (reversed, nbody.py:186); child 0 is next
            const int nc = wr_nchild(wd);
            if (sp + nc - 1 > STACK_CAP) {
                if (lane == 0) atomicOr(flag, 1);
                break;
            }
            if (lane < nc - 1) stack[sp + lane] = make_int2((fc + (nc - 1 - lane)) | ((lvl + 1) << NODE_BITS), (int)open);
            sp += nc - 1;
            __syncwarp();
            node = fc;
            ++lvl;
            act = open;
            nd = n_open;
        } else {
            if (sp == 0) break;
            --sp;
            __syncwarp();
            node = top.x & ((1 << NODE_BITS) - 1);
            lvl = top.x >> NODE_BITS;
            act = (unsigned)top.y;
            nd = n_pop;
        }
    }
    if (WRITE && emits) U.gcount[my_fg] = w;
    if (STATS && has) {
        bstat[2 * (int64_t)(gd.bfirst + lane)] = my_entries;
        bstat[2 * (int64_t)(gd.bfirst + lane) + 1] = my_items;
    }
}

// Per-bucket walk_order / kind CSR from the union lists (parity + drop-in API).
static __global__ void __launch_bounds__(32 * WARPS_PER_BLOCK)
union_to_lists_kernel(int nfg, const ForceGroup *__restrict__ fgroups, const WalkGroup *__restrict__ wgroups,
                      const UnionPool U, const int64_t *__restrict__ bptr, int *__restrict__ ids,
                      int8_t *__restrict__ kind)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (f >= nfg) return;
    const ForceGroup fg = fgroups[f];
    const unsigned bit = 1u << lane;
    const bool mine = fg.bmask & bit;
    int64_t cur = mine ? bptr[wgroups[fg.wg].bfirst + lane] : 0;
    const int n = U.gcount[f];
    int chunk = n > 0 ? U.gfirst[f] : 0;
    for (int e = 0; e < n; ++e) {
        if (e > 0 && (e & (CHUNK - 1)) == 0) chunk = U.cnext[chunk];
        const int at = chunk * CHUNK + (e & (CHUNK - 1));
        const uint2 m = U.umask[at];
        if (mine && ((m.x | m.y) & bit)) {
            ids[cur] = U.uid[at];
            kind[cur] = (m.x & bit) ? 0 : 1;
            ++cur;
        }
    }
}

// ---------------------------------------------------------------------------
// force kernels
// ---------------------------------------------------------------------------
// single MUFU.RSQ (r^6 >= eps^6 is a normal float whenever eps > 0)
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
    const float r6 = r2 * r2 * r2;
    float inv3 = rsqrt_approx(r6);
    if (EPS0) inv3 = r2 > 0.f ? inv3 : 0.f;  // coincident source (kernels.py:83-84)
    const float w = m_eff * inv3;
    a.x = fmaf(dx, w, a.x);
    a.y = fmaf(dy, w, a.y);
    a.z = fmaf(dz, w, a.z);
    if (POT) pot = fmaf(r2 != eps2 ? w : 0.f, r2, pot);  // m / sqrt(r^2 + eps^2); coincident skipped
}

// One group-relative source record (x, y, z, m) against one target.
template <bool EPS0, bool POT>
__device__ __forceinline__ void interact_rel(const float4 q, const float m_eff, const float3 xi, const float eps2,
                                             float3 &a, float &pot)
{
    const float dx = q.x - xi.x, dy = q.y - xi.y, dz = q.z - xi.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, eps2)));
    const float r6 = r2 * r2 * r2;
    float inv3 = rsqrt_approx(r6);
    if (EPS0) inv3 = r2 > 0.f ? inv3 : 0.f;  // coincident source (kernels.py:83-84)
    const float w = m_eff * inv3;
    a.x = fmaf(dx, w, a.x);
    a.y = fmaf(dy, w, a.y);
    a.z = fmaf(dz, w, a.z);
    if (POT) pot = fmaf(r2 != eps2 ? w : 0.f, r2, pot);  // m / sqrt(r^2 + eps^2); coincident skipped
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

// Force-group kernel.  One warp per force group, lane = target.  Entries are
// read 32 at a time; their records (one node record and/or the opened
// bucket's particles) are expanded warp-cooperatively into a shared-memory
// window in group-relative float32 coordinates (node COM hi + lo folded in
// once per record, not once per pair), then broadcast to all lanes.
template <bool EPS0, bool POT>
__global__ void __launch_bounds__(32 * WARPS_PER_BLOCK, 4)
force_group_kernel(int nfg, const ForceGroup *__restrict__ fgroups, const UnionPool U,
                   const float4 *__restrict__ parts, const int *__restrict__ part_bucket,
                   const int *__restrict__ porder, const WalkGroup *__restrict__ wgroups,
                   const float4 *__restrict__ rec_hi, const float4 *__restrict__ rec_lo,
                   const int2 *__restrict__ prange, float cgrid, float eps2, double g, int dim,
                   double *__restrict__ out, double *__restrict__ pot_out)
{
    __shared__ __align__(16) float4 q_rec[WARPS_PER_BLOCK][QWIN];
    __shared__ __align__(16) unsigned q_msk[WARPS_PER_BLOCK][QWIN];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (gi >= nfg) return;
    const ForceGroup fg = fgroups[gi];
    const int wfirst = wgroups[fg.wg].bfirst;
    const bool tgt = lane < fg.ntarget;
    const int p = fg.pstart + (tgt ? lane : 0);
    const float4 xp = parts[p];
    const unsigned mybit = tgt ? (1u << (part_bucket[p] - wfirst)) : 0u;
    const float inv_cgrid = 1.0f / cgrid;  // power of two: exact
    const float cx = group_origin(warp_min(xp.x), warp_max(xp.x), cgrid, inv_cgrid);
    const float cy = group_origin(warp_min(xp.y), warp_max(xp.y), cgrid, inv_cgrid);
    const float cz = group_origin(warp_min(xp.z), warp_max(xp.z), cgrid, inv_cgrid);
    const float3 xi = make_float3(xp.x - cx, xp.y - cy, xp.z - cz);  // exact
    float4 *qr = q_rec[warp];
    unsigned *qm = q_msk[warp];
    double ax = 0.0, ay = 0.0, az = 0.0, ap = 0.0;
    const int n = U.gcount[gi];
    int chunk = n > 0 ? U.gfirst[gi] : 0;
    for (int e0 = 0; e0 < n; e0 += 32) {
        if (e0 > 0 && (e0 & (CHUNK - 1)) == 0) chunk = U.cnext[chunk];
        const int e = e0 + lane;
        int node = 0;
        uint2 m = make_uint2(0u, 0u);
        int2 pr = make_int2(0, 0);
        if (e < n) {
            const int at = chunk * CHUNK + (e & (CHUNK - 1));
            node = U.uid[at];
            m = U.umask[at];
        }
        if (m.y) pr = prange[node];
        const int hasnode = m.x ? 1 : 0;
        const int nrec = hasnode + (m.y ? pr.y : 0);
        // warp inclusive scan of record counts
        int incl = nrec;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int first = incl - nrec;
        const int psrc = pr.x - hasnode;  // particle record r >= hasnode is parts[psrc + r]
        for (int w0 = 0; w0 < total; w0 += QWIN) {
            const int nin = min(QWIN, total - w0);
            const int padded = (nin + FLUSH - 1) & ~(FLUSH - 1);
            // cooperative expansion: slot s of the window belongs to the lane
            // whose [first, incl) holds w0 + s (binary search over the scan)
            for (int s0 = 0; s0 < padded; s0 += 32) {
                const int s = s0 + lane;
                const int gs = w0 + s;
                int own = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    const int v = __shfl_sync(0xffffffffu, incl, own + step - 1);
                    if (v <= gs) own += step;
                }
                own = min(own, 31);
                const int o_first = __shfl_sync(0xffffffffu, first, own);
                const int o_node = __shfl_sync(0xffffffffu, node, own);
                const unsigned o_mx = __shfl_sync(0xffffffffu, m.x, own);
                const unsigned o_my = __shfl_sync(0xffffffffu, m.y, own);
                const int o_psrc = __shfl_sync(0xffffffffu, psrc, own);
                if (s < nin) {
                    const int r = gs - o_first;
                    float4 q;
                    unsigned mk;
                    if (o_mx && r == 0) {
                        const float4 h = rec_hi[o_node];
                        const float4 l = rec_lo[o_node];
                        q = make_float4((h.x - cx) + l.x, (h.y - cy) + l.y, (h.z - cz) + l.z, h.w);
                        mk = o_mx;
                    } else {
                        const float4 h = parts[o_psrc + r];
                        q = make_float4(h.x - cx, h.y - cy, h.z - cz, h.w);
                        mk = o_my;
                    }
                    qr[s] = q;
                    qm[s] = mk;
                } else if (s < padded) {  // massless padding up to a FLUSH multiple
                    qr[s] = make_float4(0.f, 0.f, 0.f, 0.f);
                    qm[s] = 0u;
                }
            }
            __syncwarp();
            for (int j0 = 0; j0 < padded; j0 += FLUSH) {
                float3 a = make_float3(0.f, 0.f, 0.f);
                float pt = 0.f;
                const uint4 k0 = *reinterpret_cast<const uint4 *>(qm + j0);
                const uint4 k1 = *reinterpret_cast<const uint4 *>(qm + j0 + 4);
                const unsigned ks[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
                for (int jj = 0; jj < FLUSH; ++jj) {
                    const float4 q = qr[j0 + jj];
                    const float me = (ks[jj] & mybit) ? q.w : 0.f;
                    interact_rel<EPS0, POT>(q, me, xi, eps2, a, pt);
                }
                ax += (double)a.x;
                ay += (double)a.y;
                az += (double)a.z;
                if (POT) ap += (double)pt;
            }
            __syncwarp();
        }
    }
    if (tgt) {
        const int orig = porder[p];
        const double gm = g * (double)xp.w;
        out[(int64_t)orig * dim + 0] = gm * ax;
        if (dim > 1) out[(int64_t)orig * dim + 1] = gm * ay;
        if (dim > 2) out[(int64_t)orig * dim + 2] = gm * az;
        if (POT) pot_out[orig] = -gm * ap;  // -G m_i sum_j m_j / sqrt(r^2 + eps^2)
    }
}

// Member kernel: one warp per work request (bucket), lanes split its list.
// naddr/paddr are node ids (direct) or data-manager slots (staged pool);
// node terms come from rec_hi/rec_lo[addr], particle terms from
// src_parts[prange[addr].x + k].
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
