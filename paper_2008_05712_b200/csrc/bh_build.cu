// bh_build.cu -- bucket-tree build on the GPU, bit-identical to the reference
// build_bucket_tree + _fill_mass + _collect_buckets (hr/workloads/nbody.py:78-143).
//
//  1. Octant keys.  Every particle descends the reference's cells in float64:
//     digit q_L = sum_k (x_k >= c_k) << k, child centre c + (+-1)*half/2
//     (nbody.py:97-108), for every level at which a node may still split
//     (half >= 1e-9, nbody.py:94).  3 bits per level, two 64-bit words.  For a
//     power-of-two box every centre is an exact dyadic fraction of the box, so
//     the digits are the bits of x / box in fixed point (bb_keys_dyadic).
//  2. One stable radix sort by (key, original id): every node of the
//     reference is a contiguous range of this order, its children are the
//     sub-ranges of equal next digit in ascending digit (= octant) order.
//  3. Nodes bottom-up from the sorted keys (bb_lcp / bb_node_levels /
//     bb_emit_nodes): a particle starts the nodes of levels (d_i, c_i] where
//     d_i is its common prefix with its predecessor; one scan over per-level
//     run-start bitmaps gives the reference's breadth-first ids and the
//     depth-first bucket order.  (The level-synchronous cooperative expansion
//     remains for distributed builds with forced cubes.)
//  4. Each bucket's particles re-sorted by original id (the reference keeps
//     ascending particle_idx), particles gathered once in tree order.
//  5. Masses/centres of mass with the reference's float64 rounding sequence:
//     bucket mass = numpy pairwise sum, COM = sequential column sum / mass;
//     internal nodes add children in order -- one bottom-up pass, the last
//     child to finish computes its parent (bb_bucket_pass).
//  6. Force/walk records, bucket geometry and walk/force groups in HBM.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "bh_state.h"

namespace gc {

constexpr int BB_TPB = 256;
constexpr int MAX_KEY_LEVELS = 42;  // 2 x 21 levels x 3 bits

__device__ __forceinline__ int key_digit(unsigned long long k1, unsigned long long k2, int L)
{
    return L < 21 ? (int)((k1 >> (3 * (20 - L))) & 7ull) : (int)((k2 >> (3 * (41 - L))) & 7ull);
}

__global__ void bb_keys(int n, int dim, const double *__restrict__ pos, double box, int nlev,
                        unsigned long long *__restrict__ k1, unsigned long long *__restrict__ k2, int *__restrict__ idx)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double c[3], x[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        c[k] = box * 0.5;  // x * 0.5 == x / 2 exactly (nbody.py:83-108 halvings)
        x[k] = k < dim ? pos[(int64_t)i * dim + k] : 0.0;
    }
    double h = box * 0.5;
    unsigned long long a = 0, b = 0;
    for (int L = 0; L < nlev; ++L) {
        int q = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) q |= (k < dim && x[k] >= c[k] ? 1 : 0) << k;
        if (L < 21) a |= (unsigned long long)q << (3 * (20 - L));
        else b |= (unsigned long long)q << (3 * (41 - L));
        const double ch = h * 0.5;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (k < dim) c[k] = __dadd_rn(c[k], ((q >> k) & 1) ? ch : -ch);
        h = ch;
    }
    k1[i] = a;
    k2[i] = b;
    idx[i] = i;
}

// power-of-two box: every centre of the descent is an exact dyadic multiple of
// the box (no rounding in c +- half/2), so x >= c at level L is bit L of the
// fixed-point t = x / box (exact scaling) -- integer digits, same keys
__device__ __forceinline__ unsigned long long spread3(unsigned long long x)  // bit j -> bit 3j (21 bits)
{
    x &= 0x1fffffull;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}


__global__ void bb_keys_dyadic(int n, int dim, const double *__restrict__ pos, double inv_box, int nlev,
                               unsigned long long *__restrict__ k1, unsigned long long *__restrict__ k2,
                               int *__restrict__ idx)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double scale = ldexp(1.0, nlev);
    const unsigned long long top = (1ull << nlev) - 1ull;
    unsigned long long a = 0, b = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (k >= dim) break;
        const double t = pos[(int64_t)i * dim + k] * inv_box;
        // m: the nlev digits of this coordinate, level 0 in bit nlev - 1
        const unsigned long long m = t >= 1.0 ? top : (t >= 0.0 ? (unsigned long long)(t * scale) : 0ull);  // NaN: 0
        // levels 0..20 -> k1 (level L at bit 3 (20 - L) + k), levels 21..41 -> k2
        const unsigned long long hi = nlev >= 21 ? m >> (nlev - 21) : m << (21 - nlev);
        const unsigned long long lo = nlev > 21 ? m << (42 - nlev) : 0ull;
        a |= spread3(hi) << k;
        b |= spread3(lo) << k;
    }
    k1[i] = a;
    k2[i] = b;
    idx[i] = i;
}

// a run of more than `bucket` equal sorted keys (above bit `shift`): some node
// at the deepest sorted level still splits
__global__ void bb_long_runs(int n, int bucket, const unsigned long long *__restrict__ ks, int shift,
                             int *__restrict__ flag)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i + bucket >= n) return;
    if ((ks[i] >> shift) == (ks[i + bucket] >> shift)) *flag = 1;
}

__global__ void bb_fill(int n, int *p, int v)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}


__global__ void bb_gather_u64(int n, const int *__restrict__ perm, const unsigned long long *__restrict__ src,
                              unsigned long long *__restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}


// children of the splitting nodes of level L, per node: within a node's
// position range the level-L digit is sorted, so child q starts at the lower
// bound of q (8 binary searches per node instead of per-position passes)
__device__ __forceinline__ int digit_lower_bound(int lo, int hi, int q, int L, const unsigned long long *__restrict__ k1,
                                                 const unsigned long long *__restrict__ k2)
{
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_digit(k1[mid], k2[mid], L) < q) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}



// ---------------------------------------------------------------------------
// All levels of the expansion in ONE cooperative launch (grid-wide syncs
// replace a host round trip per level).  Per level: store the level's nodes
// (buckets = non-splitting), count each splitting node's children by digit
// lower bounds, grid-wide exclusive scan of the counts, emit the children as
// the next level (level-order ids = position order, children in octant order).
// ---------------------------------------------------------------------------
// warp-cooperative lower bound (32 probes per round: log32 instead of log2
// dependent loads; the top levels' nodes span most of the particles)
__device__ __forceinline__ int warp_digit_lower_bound(int lo, int hi, int q, int L,
                                                      const unsigned long long *__restrict__ k1,
                                                      const unsigned long long *__restrict__ k2)
{
    const int lane = threadIdx.x & 31;
    while (hi - lo > 32) {
        const int step = (hi - lo + 31) / 32;
        const int pos = lo + lane * step;
        const bool lt = pos < hi && key_digit(k1[pos], k2[pos], L) < q;
        const int k = __popc(__ballot_sync(0xffffffffu, lt));  // samples 0..k-1 lie below q
        if (k == 0) return lo;
        const int nlo = lo + (k - 1) * step + 1;
        hi = min(hi, lo + k * step);
        lo = nlo;
    }
    const int pos = lo + lane;
    const bool lt = pos < hi && key_digit(k1[pos], k2[pos], L) < q;
    return lo + __popc(__ballot_sync(0xffffffffu, lt));
}

constexpr int BIG_NODE = 512;  // nodes wider than this are cut by a whole warp

struct LevelArgs {
    int n, dim, nlev, cap_nodes;
    long long bucket;
    double box;
    const unsigned long long *k1, *k2;
    int *start[2], *count[2];
    double4 *center[2];
    int *cpos, *cnt, *cbase, *bsum;
    double4 *ncenter;
    int *pstart, *pcount, *first_child, *nchild;
    int *leaf_key, *leaf_id, *nleaf;
    int *lvl_first, *nlevels, *overflow;
    int *big, *nbig;  // this level's wide splitting nodes (warp-cooperative cuts)
    // cubes split regardless of their count (distributed build: they straddle
    // ranks), sorted by (level, prefix); prefix = key bits of levels < L
    const int *forced_lvl;
    const ulonglong2 *forced_key;
    int n_forced;
};

__device__ __forceinline__ ulonglong2 key_prefix(unsigned long long k1, unsigned long long k2, int L)
{
    // digits of levels 0 .. L - 1 (level l at bits 3 (20 - l) of k1, 3 (41 - l) of k2)
    const unsigned long long m1 = L >= 21 ? ~0ull : (L == 0 ? 0ull : ~0ull << (3 * (21 - L)));
    const unsigned long long m2 = L <= 21 ? 0ull : (L >= 42 ? ~0ull : ~0ull << (3 * (42 - L)));
    return make_ulonglong2(k1 & m1 & 0x7fffffffffffffffull, k2 & m2 & 0x7fffffffffffffffull);
}

// does the node of level L starting at sorted position st split?  (nbody.py:94,
// plus the forced cubes of a distributed build)
__device__ __forceinline__ bool node_splits(const LevelArgs &A, int ct, double half, int L, int st)
{
    if (!(half >= 1e-9)) return false;
    if (ct > A.bucket) return true;
    if (A.n_forced == 0 || ct == 0) return false;
    const ulonglong2 k = key_prefix(A.k1[st], A.k2[st], L);
    int lo = 0, hi = A.n_forced;  // first entry >= (L, k)
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int ml = A.forced_lvl[mid];
        const ulonglong2 mk = A.forced_key[mid];
        const bool less = ml < L || (ml == L && (mk.x < k.x || (mk.x == k.x && mk.y < k.y)));
        if (less) lo = mid + 1;
        else hi = mid;
    }
    return lo < A.n_forced && A.forced_lvl[lo] == L && A.forced_key[lo].x == k.x && A.forced_key[lo].y == k.y;
}

__device__ __forceinline__ int block_sum(int v, int *red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    int t = 0;
    for (int w = 0; w < nw; ++w) t += red[w];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(BB_TPB) bb_levels_coop(LevelArgs A)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int red[BB_TPB / 32];
    __shared__ int wsum[BB_TPB / 32];
    const int T = (int)grid.size(), tid = (int)grid.thread_rank();
    const int nb = (int)gridDim.x, b = (int)blockIdx.x;
    const int nq = 1 << A.dim;
    int m = 1, id0 = 0, cur = 0, L = 0;
    double half = A.box * 0.5;
    for (;; ++L) {
        if (tid == 0) A.lvl_first[L] = id0;
        // 1: store this level, count the children of splitting nodes
        for (int p = tid; p < m; p += T) {
            const int st = A.start[cur][p], ct = A.count[cur][p];
            const bool sp = node_splits(A, ct, half, L, st);  // nbody.py:94 (+ forced cubes)
            const int id = id0 + p;
            A.ncenter[id] = A.center[cur][p];
            A.pstart[id] = st;
            A.pcount[id] = sp ? 0 : ct;
            if (!sp) {
                const int k = atomicAdd(A.nleaf, 1);
                A.leaf_key[k] = st;
                A.leaf_id[k] = id;
            }
            int nonempty = 0;
            if (sp && L < A.nlev && ct > BIG_NODE) {
                A.big[atomicAdd(A.nbig, 1)] = p;  // cut below by a warp
            } else if (sp && L < A.nlev) {
                const int e = st + ct;
                int lo = st;
                for (int q = 0; q < nq; ++q) {
                    const int next = q + 1 < nq ? digit_lower_bound(lo, e, q + 1, L, A.k1, A.k2) : e;
                    A.cpos[9 * p + q] = lo;
                    nonempty += next > lo ? 1 : 0;
                    lo = next;
                }
                A.cpos[9 * p + nq] = e;
            }
            A.cnt[p] = nonempty;
        }
        if (L >= A.nlev) break;  // no node of this level can split (half < 1e-9)
        grid.sync();
        // 1b: wide nodes, one warp each (deep levels have none: no extra barrier)
        const int nbig = *(volatile int *)A.nbig;
        if (nbig > 0) {
            const int gw = tid >> 5, nw = T >> 5, lane = tid & 31;
            for (int k = gw; k < nbig; k += nw) {
                const int p = A.big[k];
                const int st = A.start[cur][p], e = st + A.count[cur][p];
                int lo = st, nonempty = 0;
                for (int q = 0; q < nq; ++q) {
                    const int next = q + 1 < nq ? warp_digit_lower_bound(lo, e, q + 1, L, A.k1, A.k2) : e;
                    if (lane == 0) A.cpos[9 * p + q] = lo;
                    nonempty += next > lo ? 1 : 0;
                    lo = next;
                }
                if (lane == 0) {
                    A.cpos[9 * p + nq] = e;
                    A.cnt[p] = nonempty;
                }
            }
            grid.sync();
            if (tid == 0) *A.nbig = 0;  // read by every thread above; reset for the next level
        }
        // 2: grid-wide exclusive scan of cnt[0, m) in per-block chunks
        const int chunk = (m + nb - 1) / nb;
        const int c0 = min(m, b * chunk), c1 = min(m, c0 + chunk);
        int local = 0;
        for (int p = c0 + (int)threadIdx.x; p < c1; p += blockDim.x) local += A.cnt[p];
        const int bs = block_sum(local, red);
        if (threadIdx.x == 0) A.bsum[b] = bs;
        grid.sync();
        int off = 0, mc = 0;
        for (int k = (int)threadIdx.x; k < nb; k += blockDim.x) {
            const int v = A.bsum[k];
            mc += v;
            off += k < b ? v : 0;
        }
        off = block_sum(off, red);
        mc = block_sum(mc, red);
        for (int t0 = c0; t0 < c1; t0 += blockDim.x) {  // block-wide scan of the chunk, tile by tile
            const int p = t0 + (int)threadIdx.x;
            const int v = p < c1 ? A.cnt[p] : 0;
            int incl = v;
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            int wo = 0, tile = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                wo += w < warp ? wsum[w] : 0;
                tile += wsum[w];
            }
            if (p < c1) A.cbase[p] = off + wo + incl - v;
            off += tile;
            __syncthreads();
        }
        if (mc == 0) break;
        if (id0 + m + mc > A.cap_nodes) {
            if (tid == 0) *A.overflow = 1;
            break;
        }
        __syncthreads();
        // 3: the children become level L + 1 (same chunk as the scan: cbase is this block's)
        const int nxt = cur ^ 1;
        for (int p = c0 + (int)threadIdx.x; p < c1; p += blockDim.x) {
            const int ct = A.count[cur][p];
            if (!node_splits(A, ct, half, L, A.start[cur][p])) continue;
            const double4 pc = A.center[cur][p];
            const double ch = pc.w * 0.5;  // == pc.w / 2 exactly
            int c = A.cbase[p];
            const int cfirst = c;
            for (int q = 0; q < nq; ++q) {
                const int a = A.cpos[9 * p + q], e = A.cpos[9 * p + q + 1];
                if (e <= a) continue;
                A.start[nxt][c] = a;
                A.count[nxt][c] = e - a;
                double4 cc;
                cc.x = A.dim > 0 ? __dadd_rn(pc.x, (q & 1) ? ch : -ch) : pc.x;
                cc.y = A.dim > 1 ? __dadd_rn(pc.y, (q & 2) ? ch : -ch) : pc.y;
                cc.z = A.dim > 2 ? __dadd_rn(pc.z, (q & 4) ? ch : -ch) : pc.z;
                cc.w = ch;
                A.center[nxt][c] = cc;
                ++c;
            }
            A.first_child[id0 + p] = id0 + m + cfirst;
            A.nchild[id0 + p] = c - cfirst;
        }
        grid.sync();
        id0 += m;
        m = mc;
        cur = nxt;
        half *= 0.5;
    }
    if (tid == 0) {
        A.lvl_first[L + 1] = id0 + m;
        *A.nlevels = L + 1;
    }
}





// ---------------------------------------------------------------------------
// Bottom-up enumeration of the same tree (no forced cubes): no level loop, no
// grid-wide barrier.  With d_i = common prefix (levels) of sorted keys i-1, i
// and e_i = common prefix of keys i, i+bucket:
//   * particle i starts a level-L run iff L > d_i;
//   * a run is longer than `bucket` (its node splits, below level nlev) iff it
//     holds a window [j, j + bucket] with e_j >= its level -- so the level-d_i
//     run around i splits iff max(e_j, j in [i - bucket, i]) >= d_i, and the
//     run starting at i at level L >= d_i + 1 splits iff e_i >= L;
//   * a splitting run's ancestors are longer still: they split too.
// Hence particle i starts the nodes of levels a_i = d_i + 1 .. c_i =
// max(a_i, min(e_i + 1, nlev)) when its parent run splits (none otherwise),
// and the node of level c_i is a bucket.  Level-order ids (the reference's
// breadth-first numbering, nbody.py:110-123) are ONE exclusive scan over
// per-level bitmaps of run starts, level-major; an extra row numbers the
// buckets in start order (= depth-first order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int key_lcp(unsigned long long a1, unsigned long long a2, unsigned long long b1,
                                       unsigned long long b2, int cap)
{
    const unsigned long long x1 = a1 ^ b1, x2 = a2 ^ b2;
    const int l = x1 ? (__clzll(x1) - 1) / 3 : (x2 ? 21 + (__clzll(x2) - 1) / 3 : 42);  // bit 63 unused
    return min(l, cap);
}

__global__ void bb_lcp(int n, int bucket, int cap, const unsigned long long *__restrict__ k1,
                       const unsigned long long *__restrict__ k2, signed char *__restrict__ d,
                       signed char *__restrict__ e)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long a1 = k1[i], a2 = k2[i];
    d[i] = (signed char)(i == 0 ? -1 : key_lcp(k1[i - 1], k2[i - 1], a1, a2, cap));
    e[i] = (signed char)(i + bucket < n ? key_lcp(a1, a2, k1[i + bucket], k2[i + bucket], cap) : -1);
}

// node levels [a_i, c_i] per particle (range = a | c << 8, -1: none), the
// per-level run-start bitmaps (rows 0 .. NL - 1) and the bucket row NL, with
// their popcounts for the scan
__global__ void bb_node_levels(int n, int bucket, int nlev, int NL, int W, const signed char *__restrict__ d,
                               const signed char *__restrict__ e, int *__restrict__ range,
                               unsigned *__restrict__ words, int *__restrict__ wcnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31, w = i >> 5;
    int a = -1, c = -1;
    if (i < n) {
        if (i == 0) {
            a = 0;
            c = max(0, min((int)e[0] + 1, nlev));
        } else {
            const int di = d[i];
            if (di < nlev) {
                int mx = -1;
                for (int j = max(0, i - bucket); j <= i; ++j) mx = max(mx, (int)e[j]);
                if (mx >= di) {
                    a = di + 1;
                    c = max(a, min((int)e[i] + 1, nlev));
                }
            }
        }
        range[i] = a < 0 ? -1 : (a | c << 8);
    }
    if (w >= W) return;  // whole warps only
    for (int L = 0; L <= NL; ++L) {
        const bool on = a >= 0 && (L == NL || (a <= L && L <= c));
        const unsigned b = __ballot_sync(0xffffffffu, on);
        if (lane == 0) {
            words[(size_t)L * W + w] = b;
            wcnt[(size_t)L * W + w] = __popc(b);
        }
    }
}

__global__ void bb_level_firsts(int NL, int W, const int *__restrict__ S, int *__restrict__ out)
{
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L <= NL + 1) out[L] = S[(size_t)L * W];  // out[NL] = nodes, out[NL + 1] = nodes + buckets
}

__global__ void bb_emit_nodes(int n, int dim, int NL, int W, double box, const unsigned long long *__restrict__ k1,
                              const unsigned long long *__restrict__ k2, const int *__restrict__ range,
                              const unsigned *__restrict__ words, const int *__restrict__ S,
                              const signed char *__restrict__ d, double4 *__restrict__ ncenter,
                              int *__restrict__ pstart, int *__restrict__ pcount, int *__restrict__ first_child,
                              int *__restrict__ nchild, int *__restrict__ parent, int *__restrict__ buckets,
                              int *__restrict__ bstart)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = range[i];
    if (r < 0) return;
    const int a = r & 255, c = r >> 8, w = i >> 5, bit = i & 31;
    const unsigned lt = (1u << bit) - 1u;
    const unsigned long long a1 = k1[i], a2 = k2[i];
    // centres along the key's path with the coop build's float64 sequence
    double4 cc = make_double4(box / 2.0, dim > 1 ? box / 2.0 : 0.0, dim > 2 ? box / 2.0 : 0.0, box / 2.0);
    for (int L = 0; L <= c; ++L) {
        if (L >= a) {
            const size_t o = (size_t)L * W + w;
            const int id = S[o] + __popc(words[o] & lt);
            ncenter[id] = cc;
            pstart[id] = i;
            if (L < c) {
                pcount[id] = 0;
                first_child[id] = S[o + W] + __popc(words[o + W] & lt);
            } else {  // bucket: its run ends where the keys part above level c
                int end = i + 1;
                while (end < n && d[end] >= c) ++end;
                pcount[id] = end - i;
                first_child[id] = -1;
                nchild[id] = 0;
                const size_t ob = (size_t)NL * W + w;
                const int bi = S[ob] + __popc(words[ob] & lt) - S[(size_t)NL * W];
                buckets[bi] = id;
                bstart[bi] = i;
            }
            if (L > 0) {  // the level L - 1 run holding i (this id's parent)
                const size_t oq = (size_t)(L - 1) * W + w;
                const unsigned wq = words[oq];
                parent[id] = S[oq] + __popc(wq & lt) + (int)((wq >> bit) & 1u) - 1;
            } else {
                parent[id] = -1;
            }
        }
        const int q = key_digit(a1, a2, L);
        const double ch = cc.w * 0.5;
        if (dim > 0) cc.x = __dadd_rn(cc.x, (q & 1) ? ch : -ch);
        if (dim > 1) cc.y = __dadd_rn(cc.y, (q & 2) ? ch : -ch);
        if (dim > 2) cc.z = __dadd_rn(cc.z, (q & 4) ? ch : -ch);
        cc.w = ch;
    }
}

// children of a node are consecutive ids with the same parent
__global__ void bb_nchild(int nn, const int *__restrict__ parent, const int *__restrict__ first_child,
                          int *__restrict__ nchild)
{
    const int id = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (id >= nn) return;
    const int p = parent[id];
    if (id == nn - 1 || parent[id + 1] != p) nchild[p] = id + 1 - first_child[p];
}

// numpy pairwise summation (np.sum of a 1-D float64 array)
__device__ double np_pairwise(const double *a, int n)
{
    if (n < 8) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = __dadd_rn(s, a[i]);
        return s;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int i = 8;
        const int lim = n - (n % 8);
        for (; i < lim; i += 8)
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                             __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) s = __dadd_rn(s, a[i]);
        return s;
    }
    int h = n / 2;
    h -= h % 8;
    return __dadd_rn(np_pairwise(a, h), np_pairwise(a + h, n - h));
}

// particle ids of a bucket in ascending order (nbody.py:110 keeps
// particle_idx ascending): a bitonic network in registers (ids are distinct)
template <int N>
__device__ __forceinline__ void bitonic_sort_regs(int (&v)[N])
{
#pragma unroll
    for (int k = 2; k <= N; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const int a = v[i], b = v[l];
                    const bool up = (i & k) == 0;
                    v[i] = up ? min(a, b) : max(a, b);
                    v[l] = up ? max(a, b) : min(a, b);
                }
            }
}

template <int N>
__device__ __forceinline__ void bucket_sort_net(int s, int c, const int *__restrict__ perm, int *__restrict__ pidx)
{
    int v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = i < c ? perm[s + i] : INT_MAX;
    bitonic_sort_regs<N>(v);
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (i < c) pidx[s + i] = v[i];
}

// climb from a finished node: the last child of a node to arrive sums that
// node's children in order (nbody.py:129-135)
__device__ __forceinline__ void mass_climb(int p, int dim, const int *__restrict__ parent,
                                           const int *__restrict__ first_child, const int *__restrict__ nchild,
                                           int *__restrict__ arrive, double *nmass, double4 *com)
{
    while (p >= 0) {
        const int fc = first_child[p], nc = nchild[p], pp = parent[p];  // issued before the arrival
        int old;  // release: this thread's node results are visible before its arrival
        asm volatile("atom.release.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(arrive + p) : "memory");
        if (old != nc - 1) return;
        // the last arrival: every sibling released before arriving; read them from
        // L2 (.cg, no stale L1 lines), all loads issued before the in-order sums
        double cm[8];
        double2 cxy[8], czw[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k < nc) {
                cm[k] = __ldcg(nmass + fc + k);
                cxy[k] = __ldcg(reinterpret_cast<const double2 *>(com + fc + k));
                czw[k] = __ldcg(reinterpret_cast<const double2 *>(com + fc + k) + 1);
            }
        }
        double ms = 0.0, c3[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k < nc) {
                ms = __dadd_rn(ms, cm[k]);
                c3[0] = __dadd_rn(c3[0], __dmul_rn(cxy[k].x, cm[k]));
                if (dim > 1) c3[1] = __dadd_rn(c3[1], __dmul_rn(cxy[k].y, cm[k]));
                if (dim > 2) c3[2] = __dadd_rn(c3[2], __dmul_rn(czw[k].x, cm[k]));
            }
        }
        nmass[p] = ms;
        com[p] = make_double4(__ddiv_rn(c3[0], ms), dim > 1 ? __ddiv_rn(c3[1], ms) : 0.0,
                              dim > 2 ? __ddiv_rn(c3[2], ms) : 0.0, 0.0);
        p = pp;
    }
}

// Every bucket in one pass (thread = bucket): its particle ids in ascending
// original id (nbody.py:110), the particles gathered into tree order (float32
// records, original ids, bucket of each particle), the bucket's mass (numpy
// pairwise order) and COM (sequential) from registers, its geometry, then the
// climb to the root.  Buckets of more than 8 particles take the general path
// through global scratch (sorted ids in pidx, float64 particles in spos).
__global__ void bb_bucket_pass(int nb, int dim, const int *__restrict__ buckets, const int *__restrict__ pstart,
                               const int *__restrict__ pcount, const int *__restrict__ perm,
                               const double *__restrict__ pos, const double *__restrict__ mass,
                               const double4 *__restrict__ ncenter, const int *__restrict__ parent,
                               const int *__restrict__ first_child, const int *__restrict__ nchild,
                               int *__restrict__ arrive, double *nmass, double4 *com, float4 *__restrict__ parts,
                               int *__restrict__ porder, int *__restrict__ part_bucket, double4 *__restrict__ bgeo,
                               float4 *__restrict__ bgeo32, int2 *__restrict__ brange, int *__restrict__ bids,
                               int *__restrict__ pidx, double4 *__restrict__ spos, double *__restrict__ scratch)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int id = buckets[b];
    const int s = pstart[id], c = pcount[id];
    double m;
    double4 cm;
    if (c <= 8) {
        int v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = i < c ? perm[s + i] : INT_MAX;
        bitonic_sort_regs<8>(v);
        double4 q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (i < c) {
                const int p = v[i];
                q[i] = make_double4(pos[(int64_t)p * dim], dim > 1 ? pos[(int64_t)p * dim + 1] : 0.0,
                                    dim > 2 ? pos[(int64_t)p * dim + 2] : 0.0, mass[p]);
            } else {
                q[i] = make_double4(0.0, 0.0, 0.0, 0.0);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (i < c) {
                parts[s + i] = make_float4((float)q[i].x, (float)q[i].y, (float)q[i].z, (float)q[i].w);
                porder[s + i] = v[i];
                part_bucket[s + i] = b;
            }
        }
        // numpy pairwise: sequential below 8, the fixed 8-leaf tree at 8
        if (c == 8) {
            m = __dadd_rn(__dadd_rn(__dadd_rn(q[0].w, q[1].w), __dadd_rn(q[2].w, q[3].w)),
                          __dadd_rn(__dadd_rn(q[4].w, q[5].w), __dadd_rn(q[6].w, q[7].w)));
        } else {
            m = 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < c) m = __dadd_rn(m, q[i].w);
        }
        double ax = __dmul_rn(q[0].x, q[0].w), ay = __dmul_rn(q[0].y, q[0].w), az = __dmul_rn(q[0].z, q[0].w);
#pragma unroll
        for (int i = 1; i < 8; ++i) {
            if (i < c) {
                ax = __dadd_rn(ax, __dmul_rn(q[i].x, q[i].w));
                ay = __dadd_rn(ay, __dmul_rn(q[i].y, q[i].w));
                az = __dadd_rn(az, __dmul_rn(q[i].z, q[i].w));
            }
        }
        cm = make_double4(__ddiv_rn(ax, m), dim > 1 ? __ddiv_rn(ay, m) : 0.0, dim > 2 ? __ddiv_rn(az, m) : 0.0, 0.0);
    } else {
        if (c <= 32) {
            bucket_sort_net<32>(s, c, perm, pidx);
        } else {
            for (int i = 0; i < c; ++i) {
                const int v = perm[s + i];
                int j = i - 1;
                while (j >= 0 && pidx[s + j] > v) {
                    pidx[s + j + 1] = pidx[s + j];
                    --j;
                }
                pidx[s + j + 1] = v;
            }
        }
        for (int i = 0; i < c; ++i) {
            const int p = pidx[s + i];
            const double4 q = make_double4(pos[(int64_t)p * dim], dim > 1 ? pos[(int64_t)p * dim + 1] : 0.0,
                                           dim > 2 ? pos[(int64_t)p * dim + 2] : 0.0, mass[p]);
            spos[s + i] = q;
            scratch[s + i] = q.w;
            parts[s + i] = make_float4((float)q.x, (float)q.y, (float)q.z, (float)q.w);
            porder[s + i] = p;
            part_bucket[s + i] = b;
        }
        m = np_pairwise(scratch + s, c);
        double a3[3] = {0.0, 0.0, 0.0};
        for (int k = 0; k < dim; ++k) {
            const double *ps = reinterpret_cast<const double *>(spos + s) + k;
            double acc = __dmul_rn(ps[0], scratch[s]);
            for (int i = 1; i < c; ++i) acc = __dadd_rn(acc, __dmul_rn(ps[4 * i], scratch[s + i]));
            a3[k] = __ddiv_rn(acc, m);
        }
        cm = make_double4(a3[0], a3[1], a3[2], 0.0);
    }
    nmass[id] = m;
    com[id] = cm;
    // bucket geometry (walk tests: float32 copy when exact, else flagged)
    const double4 g = ncenter[id];
    bgeo[b] = g;
    const float f0 = (float)g.x, f1 = (float)g.y, f2 = (float)g.z, fh = (float)g.w;
    const bool ex = f0 == g.x && f1 == g.y && f2 == g.z && fh == g.w;
    bgeo32[b] = make_float4(f0, f1, f2, ex ? fh : -1.f);
    brange[b] = make_int2(s, c);
    bids[b] = b;
    mass_climb(parent[id], dim, parent, first_child, nchild, arrive, nmass, com);
}

// parent of every node from the children ranges (cooperative-build path)
__global__ void bb_parents(int nn, const int *__restrict__ first_child, const int *__restrict__ nchild,
                           int *__restrict__ parent)
{
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= nn) return;
    if (id == 0) parent[0] = -1;
    const int fc = first_child[id];
    if (fc < 0) return;
    for (int ch = fc; ch < fc + nchild[id]; ++ch) parent[ch] = id;
}

// walk/force records of every node (same encoding as the host upload path)
__global__ void bb_records(int nn, const double4 *__restrict__ com, const double *__restrict__ nmass,
                           const int *__restrict__ first_child, const int *__restrict__ nchild,
                           const int *__restrict__ pstart, const int *__restrict__ pcount,
                           const double4 *__restrict__ ncenter, float4 *__restrict__ recs, double4 *__restrict__ com64,
                           float4 *__restrict__ rec_hi, float4 *__restrict__ rec_lo, int2 *__restrict__ prange,
                           double *__restrict__ cmax)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const double4 c = com[i];
    const float hx = (float)c.x, hy = (float)c.y, hz = (float)c.z;
    const int fc = first_child[i];
    // buckets of > 32 particles are rejected by bb_groups before any walk
    const int word = fc < 0 ? wr_bucket_word(pstart[i], min(pcount[i], 32)) : ((fc << 3) | (nchild[i] - 1));
    recs[i] = make_float4(hx, hy, hz, __int_as_float(word));
    com64[i] = c;
    rec_hi[i] = make_float4(hx, hy, hz, (float)nmass[i]);
    rec_lo[i] = make_float4((float)(c.x - (double)hx), (float)(c.y - (double)hy), (float)(c.z - (double)hz), 0.f);
    prange[i] = make_int2(pstart[i], pcount[i]);
    const double4 g = ncenter[i];
    double mx = fmax(fmax(fabs(c.x), fabs(c.y)), fabs(c.z));
    mx = fmax(mx, fmax(fmax(fabs(g.x), fabs(g.y)), fabs(g.z)) + g.w);
    cmax[i] = mx;
}



// walk groups of 32 buckets; force groups greedily packed (<= 32 targets)
// inside each walk group, as the host path: pass 0 counts, pass 1 writes
// Walk / force groups, one warp per walk group: lanes load the group's bucket
// ranges, the greedy force-group cuts (<= 32 targets of consecutive buckets)
// are made from registers via shuffles (PASS 0 counts, PASS 1 writes).
#ifndef FG_MAXB
#define FG_MAXB 32  // buckets per force group (<= 32 targets in any case)
#endif
#ifndef FG_MINT
#define FG_MINT 0  // > 0: also cut a force group of >= FG_MINT targets where the next bucket does not touch the last
#endif
template <int PASS>
__global__ void bb_groups(int nwg, int nb, const int2 *__restrict__ brange, int *__restrict__ nfg_of,
                          const int *__restrict__ fg_base, WalkGroup *__restrict__ wg, ForceGroup *__restrict__ fg,
                          int *__restrict__ bad, const double4 *__restrict__ bgeo)
{
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= nwg) return;
    const int b0 = w * WG_BUCKETS, b1 = min(nb, b0 + WG_BUCKETS);
    int2 r[BPL];
#pragma unroll
    for (int k = 0; k < BPL; ++k) r[k] = b0 + lane + 32 * k < b1 ? brange[b0 + lane + 32 * k] : make_int2(0, 0);
    int k = 0, start = 0, tg = 0, ps = 0;
    bool ok = true;
#if FG_MINT
    float4 gq[BPL];
#pragma unroll
    for (int q = 0; q < BPL; ++q) {
        const int bj = b0 + lane + 32 * q;
        const double4 g = bj < b1 ? bgeo[bj] : make_double4(0, 0, 0, 0);
        gq[q] = make_float4((float)g.x, (float)g.y, (float)g.z, (float)g.w);
    }
    float4 prev = make_float4(0.f, 0.f, 0.f, 0.f);
#endif
    for (int j = 0; j <= b1 - b0; ++j) {
        int cnt = 0, pst = 0;
        bool jump = false;
        if (j < b1 - b0) {
            const int2 v = j < 32 ? make_int2(__shfl_sync(0xffffffffu, r[0].x, j), __shfl_sync(0xffffffffu, r[0].y, j))
                                  : make_int2(__shfl_sync(0xffffffffu, r[1].x, j - 32),
                                              __shfl_sync(0xffffffffu, r[1].y, j - 32));
            cnt = v.y;
            pst = v.x;
#if FG_MINT
            const int q = j < 32 ? 0 : 1, src = j & 31;
            const float4 cur = make_float4(__shfl_sync(0xffffffffu, gq[q].x, src), __shfl_sync(0xffffffffu, gq[q].y, src),
                                           __shfl_sync(0xffffffffu, gq[q].z, src), __shfl_sync(0xffffffffu, gq[q].w, src));
            const float d = fmaxf(fmaxf(fabsf(cur.x - prev.x), fabsf(cur.y - prev.y)), fabsf(cur.z - prev.z));
            jump = j > 0 && d > 1.001f * (cur.w + prev.w);  // the cells do not touch
            prev = cur;
#endif
        }
        // close the current group before bucket j if it would exceed 32 targets (or at the end)
        if (j == b1 - b0 || (j > start && (tg + cnt > 32 || j - start >= FG_MAXB || (FG_MINT && jump && tg >= FG_MINT)))) {
            if (tg == 0) ok = false;
            if (PASS == 1 && lane == 0) {
                ForceGroup g;
                g.pstart = ps;
                g.ntarget = tg;
                g.wg = w;
                g.boff = start;
                g.nb = j - start;
                fg[fg_base[w] + k] = g;
            }
            ++k;
            start = j;
            tg = 0;
        }
        if (j < b1 - b0) {
            if (tg == 0) ps = pst;
            tg += cnt;
            if (cnt > 32) ok = false;
        }
    }
    if (lane == 0) {
        if (!ok) atomicOr(bad, 1);
        if (k > 32) atomicOr(bad, 2);
        if (PASS == 0) nfg_of[w] = k;
        else wg[w] = WalkGroup{b0, b1 - b0, fg_base[w], k};
    }
}

template <class F>
void cubc(gc_ctx *ctx, F &&f)
{
    size_t bytes = 0;
    GC_CUDA(f(nullptr, bytes));
    ctx->scratch.resize(bytes);
    GC_CUDA(f(ctx->scratch.p, bytes));
}

void device_keys(gc_ctx *ctx, int64_t n64, int dim, const double *pos_h, double box, uint64_t *k1_h, uint64_t *k2_h)
{
    cudaStream_t s = ctx->stream;
    const int n = (int)n64;
    int nlev = 0;
    for (double h = box / 2.0; h >= 1e-9 && nlev <= MAX_KEY_LEVELS; h /= 2.0) ++nlev;
    GC_REQUIRE(nlev <= MAX_KEY_LEVELS, GC_E_VALUE, "box too large for the device build keys");
    if (n == 0) return;
    DBuf<double> pos;
    DBuf<unsigned long long> k1, k2;
    DBuf<int> idx;
    pos.upload(pos_h, (size_t)n * dim, s);
    k1.resize(n);
    k2.resize(n);
    idx.resize(n);
    bb_keys<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, dim, pos.p, box, nlev, k1.p, k2.p, idx.p);
    check_launch("bb_keys");
    GC_CUDA(cudaMemcpyAsync(k1_h, k1.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
    GC_CUDA(cudaMemcpyAsync(k2_h, k2.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
    GC_CUDA(cudaStreamSynchronize(s));
}

// GC_BUILD_PROF=1: live per-phase device times of the build (CUDA events)
struct BuildProf {
    bool on = false;
    cudaStream_t s = nullptr;
    std::vector<std::pair<const char *, cudaEvent_t>> ev;
    std::vector<std::chrono::steady_clock::time_point> ht;
    BuildProf(cudaStream_t st) : s(st)
    {
        static const bool env = getenv("GC_BUILD_PROF") != nullptr;
        on = env;
        mark("start");
    }
    void mark(const char *name)
    {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.emplace_back(name, e);
        ht.push_back(std::chrono::steady_clock::now());
    }
    ~BuildProf()
    {
        if (!on) return;
        cudaEventSynchronize(ev.back().second);
        fprintf(stderr, "device_build_tree:");
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
            fprintf(stderr, " %s %.3f", ev[i].first, ms);
        }
        float tot = 0.f;
        cudaEventElapsedTime(&tot, ev.front().second, ev.back().second);
        fprintf(stderr, " | total %.3f ms\n  host:", tot);
        for (size_t i = 1; i < ht.size(); ++i)
            fprintf(stderr, " %s %.3f", ev[i].first, std::chrono::duration<double, std::milli>(ht[i] - ht[i - 1]).count());
        fprintf(stderr, "\n");
        for (auto &p : ev) cudaEventDestroy(p.second);
    }
};

void device_build_tree(gc_bh *bh, const double *pos_h, const double *mass_h, int64_t n64, int dim, double box,
                       int64_t bucket)
{
    BuildProf prof(bh->ctx->stream);
    gc_ctx *ctx = bh->ctx;
    cudaStream_t s = ctx->stream;
    GC_REQUIRE(n64 < (1 << PSTART_BITS), GC_E_VALUE, "too many particles for one tree (packed bucket words)");
    const int n = (int)n64;
    // levels at which a node may still split (half >= 1e-9, nbody.py:94)
    int nlev = 0;
    for (double h = box / 2.0; h >= 1e-9 && nlev <= MAX_KEY_LEVELS; h /= 2.0) ++nlev;
    GC_REQUIRE(nlev <= MAX_KEY_LEVELS, GC_E_VALUE, "box too large for the device build keys");

    auto &pos = bh->ws.pos;
    auto &mass = bh->ws.mass;
    auto &scratch = bh->ws.scratch;
    pos.upload(pos_h, (size_t)n * dim, s);
    prof.mark("h2d");
    // masses are first needed by the bucket masses: copy them on a side stream
    // while the keys, the sort and the level expansion run
    if (!bh->side) {
        GC_CUDA(cudaStreamCreateWithFlags(&bh->side, cudaStreamNonBlocking));
        GC_CUDA(cudaEventCreateWithFlags(&bh->side_done, cudaEventDisableTiming));
        GC_CUDA(cudaEventCreateWithFlags(&bh->main_ready, cudaEventDisableTiming));
    }
    mass.resize(n);
    GC_CUDA(cudaEventRecord(bh->main_ready, s));  // earlier work on `mass` (previous build) is done
    GC_CUDA(cudaStreamWaitEvent(bh->side, bh->main_ready, 0));
    GC_CUDA(cudaMemcpyAsync(mass.p, mass_h, sizeof(double) * n, cudaMemcpyHostToDevice, bh->side));
    GC_CUDA(cudaEventRecord(bh->side_done, bh->side));
    bh->h2d += (int64_t)n * (dim + 1) * (int64_t)sizeof(double);
    auto &k1 = bh->ws.k1;
    auto &k2 = bh->ws.k2;
    auto &k1p = bh->ws.k1p;
    auto &k1s = bh->ws.k1s;
    auto &k2s = bh->ws.k2s;
    auto &idx = bh->ws.idx;
    auto &scratch_i = bh->ws.nsel2;
    auto &perm1 = bh->ws.perm1;
    auto &perm = bh->ws.perm;
    k1.resize(n); k2.resize(n); k1p.resize(n); k1s.resize(n); k2s.resize(n);
    idx.resize(n); perm1.resize(n); perm.resize(n);
    // stable sort by (k1, k2), ties by original id.  Digits of a level no
    // node splits at do not change the tree, so first sort by the top Ls
    // levels only; if some run of equal top keys is longer than a bucket (a
    // node of that level would split), redo it with SORT_LEVELS_MAX levels,
    // then with all levels (LSD on k2, then k1).  Ls starts at 10 (30 bits,
    // four 8-bit radix passes: enough for clustered 1M) and sticks per handle
    // at the depth the last build needed (Plummer: 16).  (Measured: splitting
    // the 48-bit sort into 32-bit + 16-bit key passes is not faster at 1M.)
    constexpr int SORT_LEVELS_MAX = 16;  // 48 bits: six passes
    int bexp = 0;
    if (std::frexp(box, &bexp) == 0.5)
        bb_keys_dyadic<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, dim, pos.p, 1.0 / box, nlev, k1.p, k2.p, idx.p);
    else
        bb_keys<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, dim, pos.p, box, nlev, k1.p, k2.p, idx.p);
    check_launch("bb_keys");
    prof.mark("keys");
    scratch_i.resize(1);
    int deep = bh->n_forced > 0 ? 1 : 0;  // forced cubes may split below the top levels
    int Ls = std::min(bh->sort_levels, SORT_LEVELS_MAX);
    // a run of equal top keys longer than a bucket: checked on the device, read
    // back at the level-count sync below (a deeper sort redoes the levels there)
    bool check_deep = false;
    auto sort_top = [&](int levels) {
        const int top_bits = 3 * std::min(nlev, levels);
        cubc(ctx, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, k1.p, k1s.p, idx.p, perm.p, n, 63 - top_bits, 63, s);
        });
        // k1s holds the full keys in the sorted order; k2 follows the permutation
        bb_gather_u64<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, perm.p, k2.p, k2s.p);
        check_deep = nlev > levels;
        scratch_i.zero(s);
        if (check_deep)
            bb_long_runs<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, (int)bucket, k1s.p, 63 - top_bits, scratch_i.p);
    };
    auto sort_deep = [&] {
        cubc(ctx, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, k2.p, k2s.p, idx.p, perm1.p, n, 0, 64, s);
        });
        bb_gather_u64<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, perm1.p, k1.p, k1p.p);
        cubc(ctx, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, k1p.p, k1s.p, perm1.p, perm.p, n, 0, 64, s);
        });
        bb_gather_u64<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, perm.p, k2.p, k2s.p);
        check_deep = false;
        scratch_i.zero(s);
    };
    if (deep) sort_deep();
    else sort_top(Ls);
    prof.mark("radix");
    check_launch("bb sort");
    prof.mark("sort");

    int nn = 0, nb = 0;
    auto &lk_s = bh->ws.lk_s;
    if (bh->n_forced == 0) {
      for (;;) {  // once, or twice when the top-level sort was not deep enough
        // bottom-up enumeration (bb_lcp / bb_node_levels / one scan / bb_emit_nodes)
        const int Ds = deep ? nlev : std::min(nlev, Ls);  // sorted key depth
        const int NL = Ds + 1;  // node levels 0 .. Ds
        const int W = (n + 31) / 32;
        auto &dl = bh->ws.dl, &el = bh->ws.el;
        auto &range = bh->ws.range, &wcnt = bh->ws.wcnt, &wscan = bh->ws.wscan, &par = bh->ws.parent;
        auto &words = bh->ws.words;
        dl.resize(n);
        el.resize(n);
        range.resize(n);
        const size_t nw = (size_t)(NL + 1) * W;
        words.resize(nw);
        wcnt.resize(nw + 1);
        wscan.resize(nw + 1);
        GC_CUDA(cudaMemsetAsync(wcnt.p + nw, 0, sizeof(int), s));
        bb_lcp<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, (int)bucket, Ds, k1s.p, k2s.p, dl.p, el.p);
        bb_node_levels<<<grid_for(32 * W, BB_TPB), BB_TPB, 0, s>>>(n, (int)bucket, nlev, NL, W, dl.p, el.p, range.p,
                                                                    words.p, wcnt.p);
        cubc(ctx, [&](void *t, size_t &b) { return cub::DeviceScan::ExclusiveSum(t, b, wcnt.p, wscan.p, nw + 1, s); });
        auto &lvlf = bh->ws.lvlf;
        lvlf.resize(NL + 3);
        bb_level_firsts<<<1, 64, 0, s>>>(NL, W, wscan.p, lvlf.p);
        GC_CUDA(cudaMemcpyAsync(lvlf.p + NL + 2, scratch_i.p, sizeof(int), cudaMemcpyDeviceToDevice, s));
        check_launch("bb node levels");
        prof.mark("levels");
        std::vector<int> lf(NL + 3);
        lvlf.download(lf.data(), NL + 3, s);
        GC_CUDA(cudaStreamSynchronize(s));
        if (check_deep && lf[NL + 2]) {  // a run longer than a bucket below the sorted levels
            if (Ls < SORT_LEVELS_MAX && nlev > Ls) {
                Ls = SORT_LEVELS_MAX;
                bh->sort_levels = Ls;  // sticks for the next builds of this handle
                sort_top(Ls);
            } else {
                deep = 1;
                sort_deep();
            }
            continue;
        }
        nn = lf[NL];
        nb = lf[NL + 1] - nn;
        const size_t cap = std::max<size_t>((size_t)3 * n + 1024, (size_t)nn);
        bh->d_ncenter.resize(cap);
        bh->d_pstart.resize(cap);
        bh->d_pcount.resize(cap);
        bh->d_first_child.resize(cap);
        bh->d_nchild.resize(cap);
        par.resize(cap);
        bh->d_buckets.resize(nb);
        lk_s.resize(nb);
        bb_emit_nodes<<<grid_for(n, BB_TPB), BB_TPB, 0, s>>>(n, dim, NL, W, box, k1s.p, k2s.p, range.p, words.p,
                                                             wscan.p, dl.p, bh->d_ncenter.p, bh->d_pstart.p,
                                                             bh->d_pcount.p, bh->d_first_child.p, bh->d_nchild.p,
                                                             par.p, bh->d_buckets.p, lk_s.p);
        if (nn > 1)
            bb_nchild<<<grid_for(nn - 1, BB_TPB), BB_TPB, 0, s>>>(nn, par.p, bh->d_first_child.p, bh->d_nchild.p);
        check_launch("bb emit nodes");
        break;
      }
        prof.mark("emit");
    } else {
        // forced cubes (distributed build): the level-synchronous cooperative expansion
        // level-synchronous expansion
        auto &lstart = bh->ws.lstart;
        auto &lcount = bh->ws.lcount;
        auto &cstart = bh->ws.cstart;
        auto &ccount = bh->ws.ccount;
        auto &leaf_key = bh->ws.leaf_key;
        auto &leaf_id = bh->ws.leaf_id;
        auto &nleaf = bh->ws.nleaf;
        auto &lcenter = bh->ws.lcenter;
        auto &ccenter = bh->ws.ccenter;
        const int cap_nodes = 3 * n + 1024;
        bh->d_ncenter.resize(cap_nodes);
        bh->d_pstart.resize(cap_nodes);
        bh->d_pcount.resize(cap_nodes);
        bh->d_first_child.resize(cap_nodes);
        bh->d_nchild.resize(cap_nodes);
        bb_fill<<<grid_for(cap_nodes, BB_TPB), BB_TPB, 0, s>>>(cap_nodes, bh->d_first_child.p, -1);
        bh->d_nchild.zero(s);
        leaf_key.resize(n + 1);
        leaf_id.resize(n + 1);
        nleaf.resize(1);
        nleaf.zero(s);
        auto &cpos = bh->ws.cpos;
        auto &cnt = bh->ws.ccnt;
        auto &cbase = bh->ws.cbase;
        // level arrays (ping-pong, <= n nodes per level), the root as level 0
        lstart.resize(n);
        lcount.resize(n);
        lcenter.resize(n);
        cstart.resize(n);
        ccount.resize(n);
        ccenter.resize(n);
        cpos.resize((size_t)9 * n + 9);
        cnt.resize(n + 1);
        cbase.resize(n + 1);
        {
            int z = 0;
            GC_CUDA(cudaMemcpyAsync(lstart.p, &z, sizeof(int), cudaMemcpyHostToDevice, s));
            GC_CUDA(cudaMemcpyAsync(lcount.p, &n, sizeof(int), cudaMemcpyHostToDevice, s));
            const double4 root = make_double4(box / 2.0, dim > 1 ? box / 2.0 : 0.0, dim > 2 ? box / 2.0 : 0.0, box / 2.0);
            GC_CUDA(cudaMemcpyAsync(lcenter.p, &root, sizeof(double4), cudaMemcpyHostToDevice, s));
        }
        // co-resident grid of the cooperative level kernel (this context's device)
        int per_sm = 0;
        GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bb_levels_coop, BB_TPB, 0));
        const int coop_blocks = std::max(1, std::min(per_sm, 1)) * ctx->prop.multiProcessorCount;
        auto &bsum = bh->ws.bsum;
        auto &lvlf = bh->ws.lvlf;
        bsum.resize(coop_blocks);
        lvlf.resize(MAX_KEY_LEVELS + 4);
        LevelArgs A;
        A.n = n;
        A.dim = dim;
        A.nlev = nlev;
        A.cap_nodes = cap_nodes;
        A.bucket = bucket;
        A.box = box;
        A.k1 = k1s.p;
        A.k2 = k2s.p;
        A.start[0] = lstart.p;
        A.start[1] = cstart.p;
        A.count[0] = lcount.p;
        A.count[1] = ccount.p;
        A.center[0] = lcenter.p;
        A.center[1] = ccenter.p;
        A.cpos = cpos.p;
        A.cnt = cnt.p;
        A.cbase = cbase.p;
        A.bsum = bsum.p;
        A.ncenter = bh->d_ncenter.p;
        A.pstart = bh->d_pstart.p;
        A.pcount = bh->d_pcount.p;
        A.first_child = bh->d_first_child.p;
        A.nchild = bh->d_nchild.p;
        A.leaf_key = leaf_key.p;
        A.leaf_id = leaf_id.p;
        A.nleaf = nleaf.p;
        auto &big = bh->ws.big;
        big.resize(n + 1);
        A.big = big.p;
        A.nbig = big.p + n;
        GC_CUDA(cudaMemsetAsync(big.p + n, 0, sizeof(int), s));
        A.forced_lvl = bh->d_forced_lvl.p;
        A.forced_key = bh->d_forced_key.p;
        A.n_forced = bh->n_forced;
        A.lvl_first = lvlf.p;
        A.nlevels = lvlf.p + MAX_KEY_LEVELS + 2;
        A.overflow = lvlf.p + MAX_KEY_LEVELS + 3;
        GC_CUDA(cudaMemsetAsync(lvlf.p, 0, sizeof(int) * (MAX_KEY_LEVELS + 4), s));
        void *kargs[] = {&A};
        GC_CUDA(cudaLaunchCooperativeKernel((void *)bb_levels_coop, coop_blocks, BB_TPB, kargs, 0, s));
        check_launch("bb_levels_coop");
        std::vector<int> lf(MAX_KEY_LEVELS + 4);
        lvlf.download(lf.data(), MAX_KEY_LEVELS + 4, s);
        GC_CUDA(cudaStreamSynchronize(s));
        GC_REQUIRE(!lf[MAX_KEY_LEVELS + 3], GC_E_VALUE, "node capacity exceeded");
        const int nlevels = lf[MAX_KEY_LEVELS + 2];
        nn = lf[nlevels];  // level firsts lf[0 .. nlevels]: the last is the node count
        GC_CUDA(cudaMemcpyAsync(&nb, nleaf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        GC_CUDA(cudaStreamSynchronize(s));

        // buckets in depth-first order = by start position
        bh->d_buckets.resize(nb);
        lk_s.resize(nb);
        cubc(ctx, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, leaf_key.p, lk_s.p, leaf_id.p, bh->d_buckets.p, nb, 0, 32, s);
        });
    }
    // every bucket in one pass: particle order, tree-ordered particles, bucket
    // mass / COM and geometry, the climb to the root
    GC_CUDA(cudaStreamWaitEvent(s, bh->side_done, 0));
    bh->d_nmass.resize(nn);
    auto &com = bh->ws.com;
    com.resize(nn);
    scratch.resize(n);
    auto &par = bh->ws.parent;
    if (bh->n_forced != 0) {  // the cooperative build writes no parents
        par.resize(std::max<size_t>(nn, 1));
        bb_parents<<<grid_for(nn, BB_TPB), BB_TPB, 0, s>>>(nn, bh->d_first_child.p, bh->d_nchild.p, par.p);
    }
    auto &pidx = bh->ws.pidx;
    auto &spos = bh->ws.spos;
    pidx.resize(n);
    spos.resize(n);
    bh->d_parts.resize(n);
    bh->d_porder.resize(n);
    bh->d_part_bucket.resize(n);
    bh->d_bgeo.resize(nb);
    bh->d_bgeo32.resize(nb);
    bh->d_brange.resize(nb);
    bh->d_bucket_ids.resize(nb);
    auto &arrive = bh->ws.arrive;
    arrive.resize(std::max(nn, 1));
    GC_CUDA(cudaMemsetAsync(arrive.p, 0, sizeof(int) * nn, s));
    bb_bucket_pass<<<grid_for(nb, 128), 128, 0, s>>>(
        nb, dim, bh->d_buckets.p, bh->d_pstart.p, bh->d_pcount.p, perm.p, pos.p, mass.p, bh->d_ncenter.p, par.p,
        bh->d_first_child.p, bh->d_nchild.p, arrive.p, bh->d_nmass.p, com.p, bh->d_parts.p, bh->d_porder.p,
        bh->d_part_bucket.p, bh->d_bgeo.p, bh->d_bgeo32.p, bh->d_brange.p, bh->d_bucket_ids.p, pidx.p, spos.p,
        scratch.p);
    check_launch("bb bucket pass");
    prof.mark("buckets+mass");

    // records
    auto &cmax = bh->ws.cmax;
    auto &cmax_out = bh->ws.cmax_out;
    cmax.resize(nn);
    cmax_out.resize(1);
    bh->d_recs.resize(nn);
    bh->d_com64.resize(nn);
    bh->d_rec_hi.resize(nn);
    bh->d_rec_lo.resize(nn);
    bh->d_prange.resize(nn);
    bb_records<<<grid_for(nn, BB_TPB), BB_TPB, 0, s>>>(nn, com.p, bh->d_nmass.p, bh->d_first_child.p, bh->d_nchild.p,
                                                       bh->d_pstart.p, bh->d_pcount.p, bh->d_ncenter.p, bh->d_recs.p,
                                                       bh->d_com64.p, bh->d_rec_hi.p, bh->d_rec_lo.p, bh->d_prange.p,
                                                       cmax.p);
    cubc(ctx, [&](void *t, size_t &b) { return cub::DeviceReduce::Max(t, b, cmax.p, cmax_out.p, nn, s); });
    check_launch("bb records");
    prof.mark("records");
    // groups
    const int nwg = (nb + WG_BUCKETS - 1) / WG_BUCKETS;
    auto &nfg_of = bh->ws.nfg_of;
    auto &fg_base = bh->ws.fg_base;
    auto &bad = bh->ws.bad;
    nfg_of.resize(nwg + 1);
    fg_base.resize(nwg + 1);
    bad.resize(1);
    bad.zero(s);
    bb_groups<0><<<grid_for(nwg, BB_TPB / 32), BB_TPB, 0, s>>>(nwg, nb, bh->d_brange.p, nfg_of.p, nullptr, nullptr,
                                                          nullptr, bad.p, bh->d_bgeo.p);
    GC_CUDA(cudaMemsetAsync(nfg_of.p + nwg, 0, sizeof(int), s));
    cubc(ctx, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, nfg_of.p, fg_base.p, nwg + 1, s);
    });
    // every force group holds >= 1 bucket: nb bounds the group count, so the
    // second pass needs no host round trip; counts and checks come back at the end
    bh->d_wg.resize(nwg);
    bh->d_fg.resize(std::max(nb, 1));
    bb_groups<1><<<grid_for(nwg, BB_TPB / 32), BB_TPB, 0, s>>>(nwg, nb, bh->d_brange.p, nullptr, fg_base.p, bh->d_wg.p,
                                                          bh->d_fg.p, bad.p, bh->d_bgeo.p);
    check_launch("bb groups");
    prof.mark("groups");
    int nfg = 0, badh = 0;
    GC_CUDA(cudaMemcpyAsync(&nfg, fg_base.p + nwg, sizeof(int), cudaMemcpyDeviceToHost, s));
    GC_CUDA(cudaMemcpyAsync(&badh, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    double cm = 0.0;
    GC_CUDA(cudaMemcpyAsync(&cm, cmax_out.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    GC_CUDA(cudaStreamSynchronize(s));
    GC_REQUIRE(!(badh & 1), GC_E_VALUE, "bucket with more than 32 particles (coincident points) on the group path");
    GC_REQUIRE(!(badh & 2), GC_E_VALUE, "walk group with more than 32 force groups");
    bh->d_fg.n = nfg;
    bh->n_wg = nwg;
    bh->h_wg_valid = false;  // fetched on demand (sub-range launches, gc_bh_groups)
    bh->n_fg = nfg;
    set_tree_bounds(bh, cm);
    GC_CUDA(cudaEventSynchronize(bh->side_done));  // long done: the caller may reuse its mass buffer
    bh->n = n;
    bh->dim = dim;
    bh->box = box;
    bh->bucket_size = bucket;
    bh->n_nodes = nn;
    bh->n_buckets = nb;
    bh->host_tree_valid = false;
}

// host mirror of a device-built tree (parity checks, list validation)
void ensure_host_tree(gc_bh *bh)
{
    if (bh->host_tree_valid) return;
    cudaStream_t s = bh->ctx->stream;
    HostTree &t = bh->tree;
    const int64_t nn = bh->n_nodes, nb = bh->n_buckets;
    std::vector<double4> c(nn), cm(nn);
    std::vector<double> m(nn);
    std::vector<int> fc(nn), nc(nn), ps(nn), pc(nn), bk(nb), po(bh->n);
    bh->d_ncenter.download(c.data(), nn, s);
    bh->d_com64.download(cm.data(), nn, s);
    bh->d_nmass.download(m.data(), nn, s);
    bh->d_first_child.download(fc.data(), nn, s);
    bh->d_nchild.download(nc.data(), nn, s);
    bh->d_pstart.download(ps.data(), nn, s);
    bh->d_pcount.download(pc.data(), nn, s);
    bh->d_buckets.download(bk.data(), nb, s);
    bh->d_porder.download(po.data(), bh->n, s);
    GC_CUDA(cudaStreamSynchronize(s));
    t.n = bh->n;
    t.dim = bh->dim;
    t.box = bh->box;
    t.bucket_size = bh->bucket_size;
    t.center.resize(3 * nn);
    t.com.resize(3 * nn);
    t.half.resize(nn);
    t.node_mass.assign(m.begin(), m.end());
    t.first_child.resize(nn);
    t.n_child.resize(nn);
    t.pstart.resize(nn);
    t.pcount.resize(nn);
    for (int64_t i = 0; i < nn; ++i) {
        t.center[3 * i] = c[i].x;
        t.center[3 * i + 1] = c[i].y;
        t.center[3 * i + 2] = c[i].z;
        t.half[i] = c[i].w;
        t.com[3 * i] = cm[i].x;
        t.com[3 * i + 1] = cm[i].y;
        t.com[3 * i + 2] = cm[i].z;
        t.first_child[i] = fc[i];
        t.n_child[i] = fc[i] < 0 ? 0 : nc[i];
        t.pstart[i] = ps[i];
        t.pcount[i] = pc[i];
    }
    t.buckets.assign(bk.begin(), bk.end());
    t.order.assign(po.begin(), po.end());
    bh->host_tree_valid = true;
}

}  // namespace gc
