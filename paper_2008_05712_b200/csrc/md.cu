// md.cu -- cell-pair molecular dynamics on sm_100a: the reference's 2-D
// soft-repulsion patch MD (hr/workloads/md.py) and the 3-D cutoff
// Lennard-Jones workload of the north star (no reference implementation;
// restated in oracle/gcharm_oracle.c).
//
// Work decomposition.  The reference enumerates, per patch, the self pair and
// the half-shell neighbours (md.py:21, 55-73, 138-162) and scatters Newton's
// third law.  Here one thread owns one atom and visits the FULL shell (9
// cells in 2-D, 27 in 3-D), so no atomics or scatter are needed.  Every pair
// is evaluated in the reference's canonical orientation -- the atom of the
// half-shell owner first, its partner shifted by the periodic image
// (md.py:139-160) -- so the float64 separation and r^2 bits, and therefore
// every cutoff decision, equal the reference's; the partner side takes the
// negated force.  Self-cell pairs use ascending original index (i < j,
// md_self_forces kernels.py:142-143).
//
// Per step (md_run, captured into one CUDA graph): cell assignment + counting
// sort (atomics, then a per-cell sort by original id so the result is
// deterministic), the force kernel, and the integrator of md_step
// (md.py:166-190).
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "md_common.cuh"

namespace gc {

constexpr int MD_TPB = 128;
#ifndef MD_LJ_FAST
#define MD_LJ_FAST 1
#endif
#ifndef MD_LJ_COLUMN
#define MD_LJ_COLUMN 1
#endif

enum { LAW_SOFT = 0, LAW_LJ = 1 };

struct MDParams {
    int dim;
    int nx, ny, nz;  // cells per dimension (reference: rows, cols, 1)
    double cell;  // cell (patch) side
    double bx, by, bz;  // box
    int periodic;
    double cutoff, c2;
    double stiffness;  // soft law
    double eps, sig2;  // LJ law
    // x slab of a global periodic grid (multi-GPU spatial decomposition):
    // local cell x = 1 is global cell gx0; local x = 0 and nx - 1 are ghost
    // planes; x image shifts follow the GLOBAL grid (gnx cells, box gbx).  A
    // whole domain is slab = 0, gx0 = 1, gnx = nx, gbx = bx.
    int slab, gx0, gnx;
    double gbx;
};

// x image shift of a neighbour cell at local x index qx (global wrap)
__device__ __forceinline__ double md_xshift(int qx, const MDParams &P)
{
    const int gx = P.gx0 - 1 + qx;
    return gx < 0 ? -P.gbx : (gx >= P.gnx ? P.gbx : 0.0);
}

__device__ __forceinline__ bool md_forward(int dx, int dy, int dz)
{
    // half shell (md.py:21 in 2-D; its 3-D analogue in the oracle)
    return dx > 0 || (dx == 0 && dy > 0) || (dx == 0 && dy == 0 && dz > 0);
}

// md_step integrator (md.py:171-189): v += F dt (unit mass); x += v dt; then
// periodic wrap (np.remainder) or reflecting walls + clip to hi - 1e-12
__device__ __forceinline__ void md_advance(double x[3], double v[3], const double f[3], const MDParams &P, double dt)
{
    const double hi[3] = {P.slab ? P.gbx : P.bx, P.by, P.bz};  // slabs wrap x in the global box
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (k >= P.dim) break;
        v[k] = __dadd_rn(v[k], __dmul_rn(f[k], dt));
        x[k] = __dadd_rn(x[k], __dmul_rn(v[k], dt));
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (k >= P.dim) break;
        if (P.periodic) {
            // np.remainder (npy_divmod) fast path for one box of travel: fmod is
            // exact there, and negative values take the rounded x + box
            const double b = hi[k];
            if (x[k] >= 0.0 && x[k] < b) x[k] = x[k] == 0.0 ? 0.0 : x[k];
            else if (x[k] >= b && x[k] < 2.0 * b) x[k] = __dsub_rn(x[k], b);
            else if (x[k] < 0.0 && x[k] > -b) x[k] = __dadd_rn(x[k], b);
            else x[k] = np_remainder(x[k], b);
        } else {
            if (x[k] < 0.0) {
                x[k] = -x[k];
                v[k] = -v[k];
            }
            if (x[k] > hi[k]) {
                x[k] = __dsub_rn(__dmul_rn(2.0, hi[k]), x[k]);
                v[k] = -v[k];
            }
            x[k] = fmin(fmax(x[k], 0.0), __dsub_rn(hi[k], 1e-12));
        }
    }
}

// cell of a position: numpy floor_divide for the 2-D patches (md.py:187-189),
// floor(x / cell) for the 3-D cells; clamped to the grid
__device__ __forceinline__ int md_cell_index(const double x[3], const MDParams &P, int use_npy)
{
    int c3[3];
    const int dims[3] = {P.slab ? P.gnx : P.nx, P.ny, P.nz};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (k >= P.dim) {
            c3[k] = 0;
            continue;
        }
        const double f = use_npy ? np_floordiv(x[k], P.cell) : floor(__ddiv_rn(x[k], P.cell));
        long long ck = (long long)f;
        if (ck > dims[k] - 1) ck = dims[k] - 1;
        if (ck < 0) ck = 0;
        c3[k] = (int)ck;
    }
    if (P.slab) {  // global x cell -> local slab index (ghost planes wrap around the periodic box)
        int lx = c3[0] - (P.gx0 - 1);
        if (lx < 0) lx += P.gnx;
        if (lx >= P.nx) lx -= P.gnx;
        c3[0] = min(max(lx, 0), P.nx - 1);
    }
    return (c3[0] * P.ny + c3[1]) * P.nz + c3[2];
}

template <int LAW, int DIM>
__global__ void __launch_bounds__(MD_TPB)
md_force_kernel(int n, const double4 *__restrict__ spos, const int *__restrict__ sidx,
                const int *__restrict__ cell_start, const int *__restrict__ scell, const MDParams P,
                double4 *__restrict__ out)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double4 a = spos[k];
    const long long ia = __double_as_longlong(a.w);  // global id (self-cell orientation)
    const int c = scell[k];
    const int cz = c % P.nz, cy = (c / P.nz) % P.ny, cx = c / (P.nz * P.ny);
    double fx = 0.0, fy = 0.0, fz = 0.0, en = 0.0;
    constexpr int RZ = DIM == 3 ? 1 : 0;
    for (int ox = -1; ox <= 1; ++ox)
        for (int oy = -1; oy <= 1; ++oy)
            for (int oz = -RZ; oz <= RZ; ++oz) {
                int qx = cx + ox, qy = cy + oy, qz = cz + oz;
                double sx = md_xshift(qx, P), sy = 0.0, sz = 0.0;  // image shift of the neighbour cell
                if (qx < 0 || qx >= P.nx) {
                    if (!P.periodic || P.slab) continue;
                    qx = qx < 0 ? qx + P.nx : qx - P.nx;
                }
                if (qy < 0 || qy >= P.ny) {
                    if (!P.periodic) continue;
                    sy = qy < 0 ? -P.by : P.by;
                    qy = qy < 0 ? qy + P.ny : qy - P.ny;
                }
                if (qz < 0 || qz >= P.nz) {
                    if (!P.periodic) continue;
                    sz = qz < 0 ? -P.bz : P.bz;
                    qz = qz < 0 ? qz + P.nz : qz - P.nz;
                }
                const int q = (qx * P.ny + qy) * P.nz + qz;
                const bool self = ox == 0 && oy == 0 && oz == 0;
                const bool fwd_cell = md_forward(ox, oy, oz);
                for (int j = cell_start[q]; j < cell_start[q + 1]; ++j) {
                    if (j == k) continue;
                    const double4 b = spos[j];
                    bool fwd = fwd_cell;
                    if (self) fwd = ia < __double_as_longlong(b.w);
                    // canonical orientation: owner atom minus (partner + shift)
                    double d0, d1, d2 = 0.0;
                    if (fwd) {
                        d0 = __dsub_rn(a.x, __dadd_rn(b.x, sx));
                        d1 = __dsub_rn(a.y, __dadd_rn(b.y, sy));
                        if (DIM == 3) d2 = __dsub_rn(a.z, __dadd_rn(b.z, sz));
                    } else {
                        d0 = __dsub_rn(b.x, __dadd_rn(a.x, -sx));
                        d1 = __dsub_rn(b.y, __dadd_rn(a.y, -sy));
                        if (DIM == 3) d2 = __dsub_rn(b.z, __dadd_rn(a.z, -sz));
                    }
                    double r2 = __dmul_rn(d0, d0);
                    r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
                    if (DIM == 3) r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
                    if (r2 >= P.c2 || r2 < 1e-12) continue;
                    double mag;
                    if (LAW == LAW_SOFT) {
                        const double r = __dsqrt_rn(r2);
                        mag = __ddiv_rn(__dmul_rn(P.stiffness, __dsub_rn(P.cutoff, r)), r);
                    } else {
                        const double s2 = __ddiv_rn(P.sig2, r2);
                        const double s6 = __dmul_rn(__dmul_rn(s2, s2), s2);
                        const double s12 = __dmul_rn(s6, s6);
                        mag = __ddiv_rn(__dmul_rn(__dmul_rn(24.0, P.eps), __dsub_rn(__dmul_rn(2.0, s12), s6)), r2);
                        en = __dadd_rn(en, __dmul_rn(0.5, __dmul_rn(__dmul_rn(4.0, P.eps), __dsub_rn(s12, s6))));
                    }
                    const double g0 = __dmul_rn(d0, mag), g1 = __dmul_rn(d1, mag);
                    const double g2 = DIM == 3 ? __dmul_rn(d2, mag) : 0.0;
                    if (fwd) {
                        fx += g0;
                        fy += g1;
                        fz += g2;
                    } else {
                        fx -= g0;
                        fy -= g1;
                        fz -= g2;
                    }
                }
            }
    out[sidx[k]] = make_double4(fx, fy, fz, en);
}

// ---------------------------------------------------------------------------
// Block-per-cell force kernel (the throughput path).
//   phase 0: the 27 (9) neighbour cells' atoms are staged in shared memory as
//            float32 positions relative to the home cell corner;
//   phase A: each warp takes every other home atom; lanes scan 32 staged
//            neighbours at a time with a float32 r^2 test widened by a
//            rigorous error band and append survivors to the atom's list;
//   phase B: 1, 2 or 4 threads per home atom walk its list and evaluate each
//            survivor exactly as the reference does (float64, canonical
//            orientation) -- the exact test decides the cutoff.
// Lists are written in a fixed order, so results are deterministic.
// ---------------------------------------------------------------------------
constexpr int MDC_THREADS = 128;
constexpr int MDC_NB = 640;  // staged neighbours per home cell
constexpr int MDC_HOME = 16;  // home atoms per pass (lane = home atom, 16 per half warp)
constexpr int MDC_PARTS = 8;  // neighbour slots split into 8 strided parts (2 per warp)
constexpr int MDC_LIST = 24;  // survivors per (home atom, part) (overflow -> full scan)

__device__ __forceinline__ void md_offset_of(int code, int &ox, int &oy, int &oz)
{
    ox = code / 9 - 1;
    oy = (code / 3) % 3 - 1;
    oz = code % 3 - 1;
}

// per neighbour-cell offset: image shift (xyz) and half-shell direction (w: 1
// forward, 0 backward, 2 self cell)
template <int LAW, int DIM>
__device__ __forceinline__ void md_pair_exact(const double4 a, const long long ia, const double4 b, const double4 sh,
                                              const MDParams &P, double &fx, double &fy, double &fz, double &en)
{
    const double sx = sh.x, sy = sh.y, sz = sh.z;
    const bool fwd = sh.w == 2.0 ? ia < __double_as_longlong(b.w) : sh.w == 1.0;
    double d0, d1, d2 = 0.0;
    if (fwd) {
        d0 = __dsub_rn(a.x, __dadd_rn(b.x, sx));
        d1 = __dsub_rn(a.y, __dadd_rn(b.y, sy));
        if (DIM == 3) d2 = __dsub_rn(a.z, __dadd_rn(b.z, sz));
    } else {
        d0 = __dsub_rn(b.x, __dadd_rn(a.x, -sx));
        d1 = __dsub_rn(b.y, __dadd_rn(a.y, -sy));
        if (DIM == 3) d2 = __dsub_rn(b.z, __dadd_rn(a.z, -sz));
    }
    double r2 = __dmul_rn(d0, d0);
    r2 = __dadd_rn(r2, __dmul_rn(d1, d1));
    if (DIM == 3) r2 = __dadd_rn(r2, __dmul_rn(d2, d2));
    // the cutoff decision above is the reference's, bit for bit; the force
    // law below uses a correctly rounded reciprocal instead of two IEEE
    // divisions (~1 ulp from the reference's values)
    if (r2 >= P.c2 || r2 < 1e-12) return;
    double mag;
    if (LAW == LAW_SOFT) {
        const double r = __dsqrt_rn(r2);
        mag = __dmul_rn(P.stiffness, __dsub_rn(__dmul_rn(P.cutoff, __drcp_rn(r)), 1.0));
    } else {
        const double inv = __drcp_rn(r2);
        const double s2 = P.sig2 * inv;
        const double s6 = s2 * s2 * s2;
        const double s12 = s6 * s6;
        mag = 24.0 * P.eps * (2.0 * s12 - s6) * inv;
        en += 2.0 * P.eps * (s12 - s6);
    }
    if (fwd) {
        fx = fma(d0, mag, fx);
        fy = fma(d1, mag, fy);
        if (DIM == 3) fz = fma(d2, mag, fz);
    } else {
        fx = fma(-d0, mag, fx);
        fy = fma(-d1, mag, fy);
        if (DIM == 3) fz = fma(-d2, mag, fz);
    }
}

// Pair whose cutoff decision is already certain (float32 r^2 well inside the
// cutoff): the same float64 force law in one orientation (home atom minus
// shifted partner), reciprocal by float seed + two Newton steps.
template <int LAW, int DIM>
__device__ __forceinline__ void md_pair_inside(const double4 a, const double4 b, const double4 sh, const MDParams &P,
                                               double &fx, double &fy, double &fz, double &en)
{
    const double d0 = a.x - (b.x + sh.x), d1 = a.y - (b.y + sh.y), d2 = DIM == 3 ? a.z - (b.z + sh.z) : 0.0;
    const double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
    double inv = (double)__frcp_rn((float)r2);
    inv = fma(inv, fma(-r2, inv, 1.0), inv);
    inv = fma(inv, fma(-r2, inv, 1.0), inv);
    double mag;
    if (LAW == LAW_SOFT) {
        const double rinv = rsqrt(r2);
        mag = P.stiffness * (P.cutoff * rinv - 1.0);
    } else {
        const double s2 = P.sig2 * inv;
        const double s6 = s2 * s2 * s2;
        const double s12 = s6 * s6;
        mag = 24.0 * P.eps * (2.0 * s12 - s6) * inv;
        en += 2.0 * P.eps * (s12 - s6);
    }
    fx = fma(d0, mag, fx);
    fy = fma(d1, mag, fy);
    if (DIM == 3) fz = fma(d2, mag, fz);
}

// Optional fused integrator epilogue (md_step, md.py:171-189): the home atom's
// velocity and position are advanced as soon as its force is known (other
// blocks read the cell-sorted copy, not pos), its new cell is assigned and
// counted for the next step's cell sort.
struct MDInteg {
    double4 *pos, *vel;
    int *cell_of, *count;
    double dt;
    int use_npy;
};

template <int DIM>
__device__ __forceinline__ void md_integrate_one(long long ia, double3 f3, const MDParams &P, const MDInteg &I)
{
    const double4 p = I.pos[ia], q = I.vel[ia];
    double x[3] = {p.x, p.y, p.z}, v[3] = {q.x, q.y, q.z};
    const double f[3] = {f3.x, f3.y, f3.z};
    md_advance(x, v, f, P, I.dt);
    I.pos[ia] = make_double4(x[0], x[1], x[2], 0.0);
    I.vel[ia] = make_double4(v[0], v[1], v[2], 0.0);
    const int c = md_cell_index(x, P, I.use_npy);
    I.cell_of[ia] = c;
    atomicAdd(&I.count[c], 1);
}

template <int LAW, int DIM, bool INTEG>
__global__ void __launch_bounds__(MDC_THREADS, 8)
md_cell_kernel(const double4 *__restrict__ spos, const int *__restrict__ sidx, const int *__restrict__ cell_start,
               const MDParams P, float band, float inner, double4 *__restrict__ out, const MDInteg I)
{
    __shared__ float4 nb[MDC_NB];  // rel xyz (float32 filter), packed (sorted index << 5 | offset code)
    __shared__ int qstart[27];
    __shared__ unsigned short lists[MDC_HOME][MDC_PARTS][MDC_LIST];
    __shared__ int lover[MDC_HOME];
    __shared__ int pre[28];
    __shared__ int qs[27];
    __shared__ double4 shtab[27];
    const int c = blockIdx.x + (P.slab ? P.ny * P.nz : 0);  // slabs: owned cells only (skip ghost plane 0)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cz = c % P.nz, cy = (c / P.nz) % P.ny, cx = c / (P.nz * P.ny);
    const double orx = cx * P.cell, ory = cy * P.cell, orz = cz * P.cell;
    constexpr int NOFF = 27;
    // neighbour cells and their populations (offset code = (ox+1)*9 + (oy+1)*3 + (oz+1))
    if (tid < NOFF) {
        int ox, oy, oz;
        md_offset_of(tid, ox, oy, oz);
        int qx = cx + ox, qy = cy + oy, qz = cz + oz;
        bool ok = DIM == 3 || oz == 0;
        if (qx < 0 || qx >= P.nx) { ok = ok && P.periodic && !P.slab; qx = (qx + P.nx) % P.nx; }
        if (qy < 0 || qy >= P.ny) { ok = ok && P.periodic; qy = (qy + P.ny) % P.ny; }
        if (qz < 0 || qz >= P.nz) { ok = ok && P.periodic; qz = (qz + P.nz) % P.nz; }
        const int q = (qx * P.ny + qy) * P.nz + qz;
        qs[tid] = ok ? q : -1;
        qstart[tid] = ok ? cell_start[q] : 0;
        const int rx = cx + ox, ry = cy + oy, rz = cz + oz;
        shtab[tid] = make_double4(md_xshift(rx, P), ry < 0 ? -P.by : (ry >= P.ny ? P.by : 0.0),
                                  rz < 0 ? -P.bz : (rz >= P.nz ? P.bz : 0.0),
                                  tid == 13 ? 2.0 : (md_forward(ox, oy, oz) ? 1.0 : 0.0));
        pre[tid + 1] = ok ? cell_start[q + 1] - cell_start[q] : 0;
    }
    __syncthreads();
    if (warp == 0) {  // inclusive warp scan of the populations
        int v = lane < NOFF ? pre[lane + 1] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane < NOFF) pre[lane + 1] = v;
        if (lane == 0) pre[0] = 0;
    }
    __syncthreads();
    const int nnb = pre[NOFF];
    const int h0 = cell_start[c], nh = cell_start[c + 1] - h0;
    const int self0 = pre[13];  // home atoms' slot range among the staged neighbours
    if (nnb > MDC_NB) {
        // staging overflow (pathological density): exact scan straight from global
        for (int i = tid; i < nh; i += MDC_THREADS) {
            const double4 a = spos[h0 + i];
            const long long ia = __double_as_longlong(a.w);
            const int li = sidx[h0 + i];
            double fx = 0.0, fy = 0.0, fz = 0.0, en = 0.0;
            for (int k = 0; k < NOFF; ++k) {
                if (qs[k] < 0) continue;
                for (int j = cell_start[qs[k]]; j < cell_start[qs[k] + 1]; ++j)
                    if (j != h0 + i) md_pair_exact<LAW, DIM>(a, ia, spos[j], shtab[k], P, fx, fy, fz, en);
            }
            out[li] = make_double4(fx, fy, fz, en);
            if (INTEG) md_integrate_one<DIM>(li, make_double3(fx, fy, fz), P, I);
        }
        return;
    }
    // phase 0: stage all neighbours at once (independent loads)
    for (int s = tid; s < nnb; s += MDC_THREADS) {
        int lo = 0, hi = NOFF;  // pre[lo] <= s < pre[lo + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= s) lo = mid;
            else hi = mid;
        }
        const int j = qstart[lo] + (s - pre[lo]);
        const double4 b = spos[j];
        const double4 sh = shtab[lo];
        nb[s] = make_float4((float)((b.x + sh.x) - orx), (float)((b.y + sh.y) - ory), (float)((b.z + sh.z) - orz),
                            __int_as_float((j << 5) | lo));
    }
    // phase A lanes: home atom ia = lane % 16, part = 2 * warp + lane / 16;
    // phase B threads: home atom tid / 8, part tid % 8 (its own list)
    const int pa_i = lane & 15, pa_part = 2 * warp + (lane >> 4);
    const int pb_i = tid / MDC_PARTS, pb_part = tid % MDC_PARTS;
    for (int hb = 0; hb < nh; hb += MDC_HOME) {
        const int nhc = min(MDC_HOME, nh - hb);
        if (tid < MDC_HOME) lover[tid] = 0;
        __syncthreads();
        // phase A: float32 candidate filter, each lane appends to its own list
        if (pa_i < nhc) {
            const int si = self0 + hb + pa_i;
            const float4 xi = nb[si];
            int cnt = 0;
            unsigned short *lst = lists[pa_i][pa_part];
            for (int sl = pa_part; sl < nnb; sl += MDC_PARTS) {
                const float4 xj = nb[sl];
                const float dx = xj.x - xi.x, dy = xj.y - xi.y, dz = xj.z - xi.z;
                const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                if (r2 < band && sl != si) {  // bit 15: inside the error band, take the exact test
                    if (cnt < MDC_LIST) lst[cnt] = (unsigned short)(sl | (r2 < inner && r2 > 1e-6f ? 0 : 0x8000));
                    ++cnt;
                }
            }
            if (cnt > MDC_LIST) atomicOr(&lover[pa_i], 1);
            if (cnt < MDC_LIST) lst[cnt] = 0xffff;  // terminator
        }
        __syncthreads();
        // phase B: exact float64 on survivors
        double fx = 0.0, fy = 0.0, fz = 0.0, en = 0.0;
        long long ia = -1;
        int li = -1;
        if (pb_i < nhc) {
            const int hj = __float_as_int(nb[self0 + hb + pb_i].w) >> 5;
            const double4 a = spos[hj];
            ia = __double_as_longlong(a.w);
            li = sidx[hj];
            if (!lover[pb_i]) {
                const unsigned short *lst = lists[pb_i][pb_part];
                for (int e = 0; e < MDC_LIST; ++e) {
                    const int sl = lst[e];
                    if (sl == 0xffff) break;
                    const int pk = __float_as_int(nb[sl & 0x7fff].w);
                    if (sl & 0x8000) md_pair_exact<LAW, DIM>(a, ia, spos[pk >> 5], shtab[pk & 31], P, fx, fy, fz, en);
                    else md_pair_inside<LAW, DIM>(a, spos[pk >> 5], shtab[pk & 31], P, fx, fy, fz, en);
                }
            } else {  // list overflow: exact scan of this part's slots
                const int si = self0 + hb + pb_i;
                for (int sl = pb_part; sl < nnb; sl += MDC_PARTS) {
                    if (sl == si) continue;
                    const int pk = __float_as_int(nb[sl].w);
                    md_pair_exact<LAW, DIM>(a, ia, spos[pk >> 5], shtab[pk & 31], P, fx, fy, fz, en);
                }
            }
        }
        for (int o = 1; o < MDC_PARTS; o <<= 1) {
            fx += __shfl_xor_sync(0xffffffffu, fx, o);
            fy += __shfl_xor_sync(0xffffffffu, fy, o);
            fz += __shfl_xor_sync(0xffffffffu, fz, o);
            en += __shfl_xor_sync(0xffffffffu, en, o);
        }
        if (pb_i < nhc && pb_part == 0) {
            out[li] = make_double4(fx, fy, fz, en);
            if (INTEG) md_integrate_one<DIM>(li, make_double3(fx, fy, fz), P, I);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// 3-D Lennard-Jones cell kernel (the configs[1] / configs[4] throughput path).
// One block per home cell, as md_cell_kernel, rebuilt for instruction count:
//   staging: half a warp per neighbour cell copies its atoms (coalesced) into
//            shared memory twice -- float64 raw positions + global id for the
//            pair math (nbd) and float32 image-shifted offsets from the home
//            corner in PAIR layout (x0 x1 y0 y1 | z0 z1) for the filter;
//   filter:  thread = (home atom, part); HOME = 8/16/32 home atoms (next power
//            of two of the cell's population) x PARTS = 128 / HOME parts; two
//            candidates per step with FADD2/FFMA2; a survivor of the widened
//            float32 test sets one bit of a per-thread mask (32 steps per
//            chunk), no list traffic;
//   pairs:   the same thread walks the set bits and evaluates each survivor in
//            float64 from shared memory in its own orientation; pairs whose
//            float64 r^2 lies within 1e-12 of the cutoff (or below 1e-6) take
//            md_pair_exact -- the reference's canonical orientation, cutoff
//            decision bit for bit.  Parts are summed by shuffles in fixed
//            order, so results are deterministic (slab runs bit-identical).
// ---------------------------------------------------------------------------
constexpr int MDL_THREADS = 128;
constexpr int MDL_NB = 512;  // staged neighbour slots (27 cells)
constexpr int MDL_PADP = 16;  // far-away pad pairs after the last staged pair (>= max parts)
__global__ void __launch_bounds__(MDL_THREADS, 7)
md_lj3_kernel(const double4 *__restrict__ spos, const int *__restrict__ sidx, const int *__restrict__ cell_start,
              const MDParams P, float band, double4 *__restrict__ out)
{
    __shared__ double4 nbd[MDL_NB];  // raw float64 position, w = global id bits
    __shared__ float4 nba[MDL_NB / 2 + MDL_PADP];  // pairs: x0 x1 y0 y1 (shifted, relative to the home corner)
    __shared__ float2 nbz[MDL_NB / 2 + MDL_PADP];  // pairs: z0 z1
    __shared__ unsigned char nbc[MDL_NB];  // neighbour-cell offset code
    __shared__ int pre[28], qs[27], qst[27];
    __shared__ double4 shtab[27];
    const int c = blockIdx.x + (P.slab ? P.ny * P.nz : 0);  // slabs: owned cells only
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cz = c % P.nz, cy = (c / P.nz) % P.ny, cx = c / (P.nz * P.ny);
    const double orx = cx * P.cell, ory = cy * P.cell, orz = cz * P.cell;
    if (tid < 27) {
        int ox, oy, oz;
        md_offset_of(tid, ox, oy, oz);
        int qx = cx + ox, qy = cy + oy, qz = cz + oz;
        bool ok = true;
        if (qx < 0 || qx >= P.nx) { ok = P.periodic && !P.slab; qx = (qx + P.nx) % P.nx; }
        if (qy < 0 || qy >= P.ny) { ok = ok && P.periodic; qy = (qy + P.ny) % P.ny; }
        if (qz < 0 || qz >= P.nz) { ok = ok && P.periodic; qz = (qz + P.nz) % P.nz; }
        const int q = (qx * P.ny + qy) * P.nz + qz;
        qs[tid] = ok ? q : -1;
        qst[tid] = ok ? cell_start[q] : 0;
        pre[tid + 1] = ok ? cell_start[q + 1] - cell_start[q] : 0;
        const int rx = cx + ox, ry = cy + oy, rz = cz + oz;
        shtab[tid] = make_double4(md_xshift(rx, P), ry < 0 ? -P.by : (ry >= P.ny ? P.by : 0.0),
                                  rz < 0 ? -P.bz : (rz >= P.nz ? P.bz : 0.0),
                                  tid == 13 ? 2.0 : (md_forward(ox, oy, oz) ? 1.0 : 0.0));
    }
    __syncthreads();
    if (warp == 0) {  // inclusive scan of the populations
        int v = lane < 27 ? pre[lane + 1] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane < 27) pre[lane + 1] = v;
        if (lane == 0) pre[0] = 0;
    }
    __syncthreads();
    const int nnb = pre[27];
    const int h0 = cell_start[c], nh = cell_start[c + 1] - h0;
    const int self0 = pre[13];
    if (nnb > MDL_NB) {  // staging overflow (pathological density): exact scan from global memory
        for (int i = tid; i < nh; i += MDL_THREADS) {
            const double4 a = spos[h0 + i];
            const long long ia = __double_as_longlong(a.w);
            double fx = 0.0, fy = 0.0, fz = 0.0, en = 0.0;
            for (int k = 0; k < 27; ++k) {
                if (qs[k] < 0) continue;
                for (int j = cell_start[qs[k]]; j < cell_start[qs[k] + 1]; ++j)
                    if (j != h0 + i) md_pair_exact<LAW_LJ, 3>(a, ia, spos[j], shtab[k], P, fx, fy, fz, en);
            }
            out[sidx[h0 + i]] = make_double4(fx, fy, fz, en);
        }
        return;
    }
    // staging: half-warp h of warp w copies neighbour cells 2 w + h, 2 w + h + 8, ...
    float *fa = reinterpret_cast<float *>(nba);
    float *fzp = reinterpret_cast<float *>(nbz);
    const int hl = lane & 15;
    for (int k = 2 * warp + (lane >> 4); k < 27; k += 2 * (MDL_THREADS / 32)) {
        const int n = pre[k + 1] - pre[k], s0 = pre[k];
        const double4 sh = shtab[k];
        const double ox = orx - sh.x, oy = ory - sh.y, oz = orz - sh.z;  // filter offsets only
        for (int j = hl; j < n; j += 16) {
            const double4 b = spos[qst[k] + j];
            const int s = s0 + j;
            nbd[s] = b;
            nbc[s] = (unsigned char)k;
            const int o = (s >> 1) * 4 + (s & 1);
            fa[o] = (float)(b.x - ox);
            fa[o + 2] = (float)(b.y - oy);
            fzp[(s >> 1) * 2 + (s & 1)] = (float)(b.z - oz);
        }
    }
    // far-away pads: the odd last slot and MDL_PADP whole pairs (filter reads past npair)
    for (int s = nnb + tid; s < 2 * ((nnb + 1) / 2 + MDL_PADP); s += MDL_THREADS) {
        const int o = (s >> 1) * 4 + (s & 1);
        fa[o] = 1e30f;
        fa[o + 2] = 1e30f;
        fzp[(s >> 1) * 2 + (s & 1)] = 1e30f;
    }
    __syncthreads();
    const int npair = (nnb + 1) >> 1;
    const double lo = P.c2 * (1.0 - 1e-12), hi = P.c2 * (1.0 + 1e-12);
    const double e24 = 24.0 * P.eps, e2 = 2.0 * P.eps;
    for (int hb = 0; hb < nh; hb += 32) {
        const int nhc = min(32, nh - hb);
        const int lg = nhc <= 8 ? 3 : (nhc <= 16 ? 4 : 5);  // HOME = 2^lg home atoms x PARTS parts
        const int parts = MDL_THREADS >> lg;
        const int hi_ = tid >> (7 - lg), part = tid & (parts - 1);
        const bool act = hi_ < nhc;
        const int si = self0 + hb + (act ? hi_ : 0);
        const float xi = fa[(si >> 1) * 4 + (si & 1)], yi = fa[(si >> 1) * 4 + (si & 1) + 2],
                    zi = fzp[(si >> 1) * 2 + (si & 1)];
        const float2 nx2 = make_float2(-xi, -xi), ny2 = make_float2(-yi, -yi), nz2 = make_float2(-zi, -zi);
        const double4 a = nbd[si];
        const long long ia = __double_as_longlong(a.w);
        double fx = 0.0, fy = 0.0, fzz = 0.0, en = 0.0;
        const int nstep = (npair + parts - 1) / parts;  // block-uniform
        for (int c0 = 0; c0 < nstep; c0 += 32) {
            // filter 32 steps: bit k of w0 / w1 = slot 2 pr / 2 pr + 1 of step c0 + k survives
            unsigned w0 = 0u, w1 = 0u;
            const int ks = min(32, nstep - c0);
            int pr = part + parts * c0;
#pragma unroll 4
            for (int k = 0; k < ks; ++k, pr += parts) {
                const float4 A = nba[pr];
                const float2 Z = nbz[pr];
                const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx2);
                const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny2);
                const float2 dz = __fadd2_rn(Z, nz2);
                float2 r2 = __fmul2_rn(dz, dz);
                r2 = __ffma2_rn(dy, dy, r2);
                r2 = __ffma2_rn(dx, dx, r2);
                w0 |= (r2.x < band ? 1u : 0u) << k;
                w1 |= (r2.y < band ? 1u : 0u) << k;
            }
            if (!act) w0 = w1 = 0u;
            // survivors in float64 from shared memory
            while (w0 | w1) {
                int sl;
                if (w0) {
                    const int k = __ffs(w0) - 1;
                    w0 &= w0 - 1u;
                    sl = 2 * (part + parts * (c0 + k));
                } else {
                    const int k = __ffs(w1) - 1;
                    w1 &= w1 - 1u;
                    sl = 2 * (part + parts * (c0 + k)) + 1;
                }
                const double4 b = nbd[sl];
                const double4 sh = shtab[nbc[sl]];
                const double d0 = a.x - (b.x + sh.x), d1 = a.y - (b.y + sh.y), d2 = a.z - (b.z + sh.z);
                const double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
                if ((r2 > lo && r2 < hi) || r2 < 1e-6) {  // at the cutoff / coincident: the reference's own test
                    md_pair_exact<LAW_LJ, 3>(a, ia, b, sh, P, fx, fy, fzz, en);
                } else if (r2 < P.c2) {
                    double inv = (double)__frcp_rn((float)r2);
                    inv = fma(inv, fma(-r2, inv, 1.0), inv);
                    inv = fma(inv, fma(-r2, inv, 1.0), inv);
                    const double s2 = P.sig2 * inv;
                    const double s6 = s2 * s2 * s2;
                    const double s12 = s6 * s6;
                    const double mag = e24 * (2.0 * s12 - s6) * inv;
                    en = fma(e2, s12 - s6, en);
                    fx = fma(d0, mag, fx);
                    fy = fma(d1, mag, fy);
                    fzz = fma(d2, mag, fzz);
                }
            }
        }
        for (int o = 1; o < parts; o <<= 1) {
            fx += __shfl_xor_sync(0xffffffffu, fx, o);
            fy += __shfl_xor_sync(0xffffffffu, fy, o);
            fzz += __shfl_xor_sync(0xffffffffu, fzz, o);
            en += __shfl_xor_sync(0xffffffffu, en, o);
        }
        if (act && part == 0) out[sidx[h0 + hb + hi_]] = make_double4(fx, fy, fzz, en);
    }
}

// ---------------------------------------------------------------------------
// 3-D Lennard-Jones COLUMN kernel (the default throughput path for grids of
// at least 3 cells per dimension).  One block per column of KZ home cells
// along z: the 3 x 3 x (KZ + 2) neighbour region is staged once for all
// KZ x ~13.5 home atoms (half the staging of one block per cell); every
// region cell starts at an even slot (a far-away pad fills odd cells), so a
// home atom's 27 neighbour cells are 9 pair-aligned slot runs.
//   thread = (home atom, part): PARTS = 256 / next power of two of the home
//            count; part p takes a contiguous share of every run's slot pairs;
//   filter:  float32 r^2 against the widened cutoff band, two candidates per
//            step (FADD2 / FFMA2); survivors are appended straight to the
//            thread's shared-memory list (no bit masks);
//   pairs:   one pass over the list in float64 from the image-shifted staged
//            positions: pairs well inside the cutoff take the force law in the
//            home atom's orientation (reciprocal from a float seed + one Newton
//            step); pairs at the cutoff (or coincident) take the reference's
//            canonical orientation and cutoff test (md_pair_exact, bit for
//            bit); parts are summed by shuffles in fixed order (deterministic:
//            slab runs are bit-identical to the whole domain).
// ---------------------------------------------------------------------------
#ifndef MDK_KZ_SET
#define MDK_KZ_SET 4
#endif
#ifndef MDK_NB_SET
#define MDK_NB_SET 1024
#endif
#ifndef MDK_LIST_SET
#define MDK_LIST_SET 48
#endif
#ifndef MDK_MINB
#define MDK_MINB 3
#endif

constexpr int MDK_KZ = MDK_KZ_SET;  // home cells per column block
constexpr int MDK_THREADS = 256;
constexpr int MDK_NR = 9 * (MDK_KZ + 2);  // region cells
constexpr int MDK_NB = MDK_NB_SET;  // staged region slots incl. pads (overflow -> exact scan from global memory)
constexpr int MDK_LIST = MDK_LIST_SET;  // survivors per thread (overflow -> the thread rescans its candidates exactly)
constexpr int MDK_HOMES = 256;  // home atoms per pass
constexpr int MDK_SMEM = MDK_NB * 32 + MDK_LIST * MDK_THREADS * 2 + (MDK_NB / 2) * 24 + MDK_NB + MDK_HOMES * 2;

__global__ void __launch_bounds__(MDK_THREADS, MDK_MINB)
md_lj3c_kernel(const double4 *__restrict__ spos, const int *__restrict__ sidx, const int *__restrict__ cell_start,
               const MDParams P, float band, int ncol_z, double4 *__restrict__ out, const int *__restrict__ cols)
{
    // dynamic shared memory (MDK_SMEM bytes)
    extern __shared__ __align__(16) unsigned char mdk_smem[];
    double4 *nbs = reinterpret_cast<double4 *>(mdk_smem);  // [NB] image-shifted float64 position, w = global id bits
    unsigned short *lst = reinterpret_cast<unsigned short *>(nbs + MDK_NB);  // [LIST][THREADS] survivor slots
    float4 *nba = reinterpret_cast<float4 *>(lst + MDK_LIST * MDK_THREADS);  // [NB/2] pairs x0 x1 y0 y1 (region frame)
    float2 *nbz = reinterpret_cast<float2 *>(nba + MDK_NB / 2);  // [NB/2] pairs z0 z1
    unsigned char *nbc = reinterpret_cast<unsigned char *>(nbz + MDK_NB / 2);  // [NB] region cell of the slot
    unsigned short *hslot = reinterpret_cast<unsigned short *>(nbc + MDK_NB);  // [HOMES] home atoms' slots
    __shared__ int pre[MDK_NR + 1], qst[MDK_NR], pop[MDK_NR];
    __shared__ double4 shtab[MDK_NR];  // image shift of the region cell
    __shared__ int pfx[MDK_THREADS];  // inclusive prefix of the list lengths over a home's parts
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // column: home cells (cx, cy, cz0 .. cz0 + kz - 1); a batched launch
    // (combined work requests of columns) names its columns
    const int col = cols ? cols[blockIdx.x] : (int)blockIdx.x;
    const int czb = col % ncol_z, cxy = col / ncol_z;
    const int cy = cxy % P.ny, cx = cxy / P.ny + (P.slab ? 1 : 0);  // slabs: owned x planes only
    const int cz0 = czb * MDK_KZ, kz = min(MDK_KZ, P.nz - cz0);
    constexpr int RZ = MDK_KZ + 2;
    if (tid < MDK_NR) {
        const int dxy = tid / RZ, dz = tid - dxy * RZ;
        const int ox = dxy / 3 - 1, oy = dxy - 3 * (dxy / 3) - 1;
        int qx = cx + ox, qy = cy + oy, qz = cz0 - 1 + dz;
        bool ok = dz <= kz + 1;
        double sy = 0.0, sz = 0.0;
        if (qx < 0 || qx >= P.nx) {
            ok = ok && P.periodic && !P.slab;
            qx = qx < 0 ? qx + P.nx : qx - P.nx;
        }
        if (qy < 0) { ok = ok && P.periodic; qy += P.ny; sy = -P.by; }
        else if (qy >= P.ny) { ok = ok && P.periodic; qy -= P.ny; sy = P.by; }
        if (qz < 0) { ok = ok && P.periodic; qz += P.nz; sz = -P.bz; }
        else if (qz >= P.nz) { ok = ok && P.periodic; qz -= P.nz; sz = P.bz; }
        const int q = (qx * P.ny + qy) * P.nz + qz;
        const int a0 = ok ? cell_start[q] : 0;
        const int n = ok ? cell_start[q + 1] - a0 : 0;
        qst[tid] = a0;
        pop[tid] = n;
        pre[tid + 1] = (n + 1) & ~1;  // even slot count per cell (pair-aligned runs)
        shtab[tid] = make_double4(md_xshift(cx + ox, P), sy, sz, 0.0);
    }
    __syncthreads();
    if (warp == 0) {  // inclusive scan of the padded populations, 32 cells per round with a carry
        int carry = 0;
        for (int c0 = 0; c0 < MDK_NR; c0 += 32) {
            int v = c0 + lane < MDK_NR ? pre[c0 + lane + 1] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            v += carry;
            if (c0 + lane < MDK_NR) pre[c0 + lane + 1] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) pre[0] = 0;
    }
    __syncthreads();
    const int nnb = pre[MDK_NR];
    const int hr0 = 4 * RZ + 1;  // home cells are region cells (1, 1, 1 .. kz)
    int nh = 0;
    for (int r = hr0; r < hr0 + kz; ++r) nh += pop[r];
    const double orx = (cx - 1) * P.cell, ory = (cy - 1) * P.cell, orz = (cz0 - 1) * P.cell;
    if (nnb > MDK_NB || nh > MDK_HOMES) {  // staging overflow (pathological density): exact scan from global memory
        for (int r = hr0; r < hr0 + kz; ++r) {
            const int hz = r - 4 * RZ;
            for (int i = tid; i < pop[r]; i += MDK_THREADS) {
                const int j0 = qst[r] + i;
                const double4 a = spos[j0];
                const long long ia = __double_as_longlong(a.w);
                double fx = 0.0, fy = 0.0, fz = 0.0, en = 0.0;
                for (int rr = 0; rr < MDK_NR; ++rr) {
                    const int dxy = rr / RZ, dz = rr - dxy * RZ;
                    if (dz < hz - 1 || dz > hz + 1) continue;
                    const int ox = dxy / 3 - 1, oy = dxy - 3 * (dxy / 3) - 1, oz = dz - hz;
                    const double4 sh = shtab[rr];
                    const double4 shf =
                        make_double4(sh.x, sh.y, sh.z, (ox | oy | oz) == 0 ? 2.0 : (md_forward(ox, oy, oz) ? 1.0 : 0.0));
                    for (int k = 0; k < pop[rr]; ++k) {
                        const int j = qst[rr] + k;
                        if (j != j0) md_pair_exact<LAW_LJ, 3>(a, ia, spos[j], shf, P, fx, fy, fz, en);
                    }
                }
                out[sidx[j0]] = make_double4(fx, fy, fz, en);
            }
        }
        return;
    }
    // staging: half-warp h copies region cells h, h + 16, ... (coalesced within a cell)
    float *fa = reinterpret_cast<float *>(nba);
    float *fzp = reinterpret_cast<float *>(nbz);
    for (int r = tid >> 4; r < MDK_NR; r += MDK_THREADS / 16) {
        const int n = pop[r], s0 = pre[r], np = pre[r + 1] - s0;
        const double4 sh = shtab[r];
        for (int j = tid & 15; j < np; j += 16) {
            const int s = s0 + j;
            const int o = (s >> 1) * 4 + (s & 1);
            if (j < n) {
                const double4 b = spos[qst[r] + j];
                const double4 bs = make_double4(b.x + sh.x, b.y + sh.y, b.z + sh.z, b.w);
                nbs[s] = bs;
                fa[o] = (float)(bs.x - orx);
                fa[o + 2] = (float)(bs.y - ory);
                fzp[(s >> 1) * 2 + (s & 1)] = (float)(bs.z - orz);
                if (r >= hr0 && r < hr0 + kz) {  // home atom: its slot, in slot order
                    int hb = 0;
                    for (int rr = hr0; rr < r; ++rr) hb += pop[rr];
                    hslot[hb + j] = (unsigned short)s;
                }
            } else {  // pad slot: far away
                fa[o] = 1e30f;
                fa[o + 2] = 1e30f;
                fzp[(s >> 1) * 2 + (s & 1)] = 1e30f;
            }
            nbc[s] = (unsigned char)r;
        }
    }
    __syncthreads();
    const double lo = P.c2 * (1.0 - 1e-12), hi = P.c2 * (1.0 + 1e-12);
    const double e24 = 24.0 * P.eps, e2 = 2.0 * P.eps;
    // PARTS = 256 / (next power of two >= nh), at most 16
    int lgh = 4;
    while ((1 << lgh) < nh) ++lgh;
    const int lgp = 8 - lgh;
    const int parts = 1 << lgp;
    const int hi_ = tid >> lgp, part = tid & (parts - 1);
    const bool act = hi_ < nh;
    const int si = hslot[act ? hi_ : 0];
    const int hr = nbc[si];
    const int hz = hr - 4 * RZ;  // region z index of the home cell (1 .. kz)
    const float xi = fa[(si >> 1) * 4 + (si & 1)], yi = fa[(si >> 1) * 4 + (si & 1) + 2],
                zi = fzp[(si >> 1) * 2 + (si & 1)];
    const float2 nx2 = make_float2(-xi, -xi), ny2 = make_float2(-yi, -yi), nz2 = make_float2(-zi, -zi);
    const double4 a = nbs[si];
    // filter: the 9 runs (dx, dy) x region z [hz - 1, hz + 1], each part a
    // contiguous share of the pairs; a survivor is stored at the list end and
    // the end advances (predicated, no branch) -- a run whose share could
    // overflow the list takes the guarded loop
    unsigned short *lp = lst + tid;
    int cnt = 0;
    if (act) {
        // (a per-atom cell pre-test -- skip z cells of a run farther than the
        // band, ~25 % fewer candidates -- measured 9 % SLOWER: homes of a warp
        // then run different trip counts)
        for (int dxy = 0; dxy < 9; ++dxy) {
            const int p0 = pre[dxy * RZ + hz - 1] >> 1, p1 = pre[dxy * RZ + hz + 2] >> 1;
            const int len = p1 - p0;
            const int c0 = p0 + (len * part >> lgp), c1 = p0 + (len * (part + 1) >> lgp);
            if (cnt + 2 * (c1 - c0) <= MDK_LIST) {
                int wo = cnt * MDK_THREADS + tid;  // element offset of the list end
                const float4 *pa = nba + c0;
                const float2 *pz = nbz + c0;
                int s2 = 2 * c0;
#pragma unroll 4
                for (int k = 0; k < c1 - c0; ++k) {
                    const float4 A = pa[k];
                    const float2 Z = pz[k];
                    const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx2);
                    const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny2);
                    const float2 dz = __fadd2_rn(Z, nz2);
                    float2 r2 = __fmul2_rn(dz, dz);
                    r2 = __ffma2_rn(dy, dy, r2);
                    r2 = __ffma2_rn(dx, dx, r2);
                    if (r2.x < band) {
                        lst[wo] = (unsigned short)s2;
                        wo += MDK_THREADS;
                    }
                    if (r2.y < band) {
                        lst[wo] = (unsigned short)(s2 + 1);
                        wo += MDK_THREADS;
                    }
                    s2 += 2;
                }
                cnt = (wo - tid) / MDK_THREADS;
            } else {
                for (int pr = c0; pr < c1; ++pr) {
                    const float4 A = nba[pr];
                    const float2 Z = nbz[pr];
                    const float2 dx = __fadd2_rn(make_float2(A.x, A.y), nx2);
                    const float2 dy = __fadd2_rn(make_float2(A.z, A.w), ny2);
                    const float2 dz = __fadd2_rn(Z, nz2);
                    float2 r2 = __fmul2_rn(dz, dz);
                    r2 = __ffma2_rn(dy, dy, r2);
                    r2 = __ffma2_rn(dx, dx, r2);
                    if (r2.x < band) {
                        if (cnt < MDK_LIST) lp[cnt * MDK_THREADS] = (unsigned short)(2 * pr);
                        ++cnt;
                    }
                    if (r2.y < band) {
                        if (cnt < MDK_LIST) lp[cnt * MDK_THREADS] = (unsigned short)(2 * pr + 1);
                        ++cnt;
                    }
                }
            }
        }
    }
    // the home's survivors are re-dealt evenly over its parts (lists differ in
    // length; the float64 loop runs the longest list of the warp): combined
    // entry e = part + parts * i lives in the list of the part q whose prefix
    // range contains e
    const bool over = __any_sync(0xffffffffu, cnt > MDK_LIST);
    const int mine = min(cnt, MDK_LIST);
    int incl = mine;  // inclusive prefix over the parts of this home (lanes part 0 .. parts - 1)
    for (int o = 1; o < parts; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (part >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, (lane & ~(parts - 1)) + parts - 1);
    const int gbase = tid - part;  // list column of part 0 of this home
    pfx[tid] = incl;
    __syncwarp();
    double fx = 0.0, fy = 0.0, fzz = 0.0, en = 0.0;
    // the reference's own test (canonical orientation, md_pair_exact) for a
    // pair at the cutoff or coincident -- rare; deferred out of the main loop
    auto pair_exact = [&](int sl) {
        if (sl == si) return;
        const int r = nbc[sl];
        const int dxy = r / RZ, dz = r - dxy * RZ;
        const int ox = dxy / 3 - 1, oy = dxy - 3 * (dxy / 3) - 1, oz = dz - hz;
        const double4 sh = shtab[r];
        const double4 shf =
            make_double4(sh.x, sh.y, sh.z, (ox | oy | oz) == 0 ? 2.0 : (md_forward(ox, oy, oz) ? 1.0 : 0.0));
        const double4 b = spos[qst[r] + (sl - pre[r])];  // the unshifted position
        const double4 ah = spos[qst[hr] + (si - pre[hr])];
        md_pair_exact<LAW_LJ, 3>(ah, __double_as_longlong(ah.w), b, shf, P, fx, fy, fzz, en);
    };
    if (!over) {
        unsigned long long defer = 0ull;  // list entries (bit = combined index / parts) for pair_exact
        int ne = 0;
        int q = 0, base = 0;  // the part holding combined entry e, and its prefix start (nondecreasing in e)
        for (int e = part; e < total; e += parts, ++ne) {
            while (q < parts - 1 && e >= pfx[gbase + q]) base = pfx[gbase + q++];
            const int sl = lst[(e - base) * MDK_THREADS + gbase + q];
            const double4 bs = nbs[sl];
            const double d0 = a.x - bs.x, d1 = a.y - bs.y, d2 = a.z - bs.z;
            const double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
            const bool exact = (r2 > lo && r2 < hi) || r2 < 1e-6;
            if (exact) defer |= 1ull << ne;
            // certain pairs: the force law in the home atom's orientation,
            // reciprocal from a float seed + one Newton step (2^-46 relative)
            double inv = (double)__frcp_rn((float)r2);
            inv = fma(inv, fma(-r2, inv, 1.0), inv);
            const double s2 = P.sig2 * inv;
            const double s6 = s2 * s2 * s2;
            const double s12 = s6 * s6;
            const bool in = !exact && r2 < P.c2;
            const double mag = in ? e24 * fma(2.0, s12, -s6) * inv : 0.0;
            const double ep = fma(e2, s12 - s6, en);  // (inf - inf for the home atom itself: not taken)
            en = in ? ep : en;
            fx = fma(d0, mag, fx);
            fy = fma(d1, mag, fy);
            fzz = fma(d2, mag, fzz);
        }
        for (ne = 0; defer; defer >>= 1, ++ne) {
            if (!(defer & 1ull)) continue;
            const int e = part + ne * parts;
            int q = 0, base = 0;
            for (int k = 0; k < parts - 1; ++k) {
                const int ik = pfx[gbase + k];
                if (e >= ik) {
                    q = k + 1;
                    base = ik;
                }
            }
            pair_exact(lst[(e - base) * MDK_THREADS + gbase + q]);
        }
    } else if (act) {  // a list overflowed in this warp: exact rescan of every thread's own share
        const double4 ah = spos[qst[hr] + (si - pre[hr])];
        const long long ia = __double_as_longlong(ah.w);
        for (int dxy = 0; dxy < 9; ++dxy) {
            const int p0 = pre[dxy * RZ + hz - 1] >> 1, p1 = pre[dxy * RZ + hz + 2] >> 1;
            const int len = p1 - p0;
            const int c0 = p0 + (len * part >> lgp), c1 = p0 + (len * (part + 1) >> lgp);
            for (int sl = 2 * c0; sl < 2 * c1; ++sl) {
                const int r = nbc[sl], k = sl - pre[r];
                if (k >= pop[r] || sl == si) continue;  // pad slot / the home atom itself
                const int dxy2 = r / RZ, dz = r - dxy2 * RZ;
                const int ox = dxy2 / 3 - 1, oy = dxy2 - 3 * (dxy2 / 3) - 1, oz = dz - hz;
                const double4 sh = shtab[r];
                const double4 shf =
                    make_double4(sh.x, sh.y, sh.z, (ox | oy | oz) == 0 ? 2.0 : (md_forward(ox, oy, oz) ? 1.0 : 0.0));
                md_pair_exact<LAW_LJ, 3>(ah, ia, spos[qst[r] + k], shf, P, fx, fy, fzz, en);
            }
        }
    }
    for (int o = 1; o < parts; o <<= 1) {
        fx += __shfl_xor_sync(0xffffffffu, fx, o);
        fy += __shfl_xor_sync(0xffffffffu, fy, o);
        fzz += __shfl_xor_sync(0xffffffffu, fzz, o);
        en += __shfl_xor_sync(0xffffffffu, en, o);
    }
    if (act && part == 0) out[sidx[qst[hr] + (si - pre[hr])]] = make_double4(fx, fy, fzz, en);
}

// cell of every atom (unfused path)
__global__ void md_assign_kernel(int n, const double4 *__restrict__ pos, const MDParams P, int use_npy,
                                 int *__restrict__ cell_of, int *__restrict__ count)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 p = pos[i];
    const double x[3] = {p.x, p.y, p.z};
    const int c = md_cell_index(x, P, use_npy);
    cell_of[i] = c;
    atomicAdd(&count[c], 1);
}

__global__ void md_count_kernel(int n, const int *__restrict__ cell_of, int *__restrict__ count)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(&count[cell_of[i]], 1);
}

__global__ void md_scatter_kernel(int n, const int *__restrict__ cell_start, const int *__restrict__ cell_of,
                                  int *__restrict__ count, int *__restrict__ perm)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = cell_of[i];
    perm[cell_start[c] + atomicSub(&count[c], 1) - 1] = i;  // counts end at zero
}

// Rank sort of a cell's atoms by global id (deterministic order for any
// atomic scatter order, the same order on every slab) fused with the gather:
// spos = (x, y, z, global id bits), sidx = local index.  Whole warp per cell.
__device__ __forceinline__ void md_sortgather_cell(int c, int lane, const int *__restrict__ cell_start,
                                                   int *__restrict__ perm, const double4 *__restrict__ pos,
                                                   const long long *__restrict__ gid, double4 *__restrict__ spos,
                                                   int *__restrict__ sidx, int *__restrict__ scell)
{
    const int s = cell_start[c], n = cell_start[c + 1] - s;
    if (n > 32) {  // rare: serial insertion sort by global id, then gather
        if (lane == 0)
            for (int i = s + 1; i < s + n; ++i) {
                const int v = perm[i];
                const long long gv = gid[v];
                int j = i - 1;
                while (j >= s && gid[perm[j]] > gv) {
                    perm[j + 1] = perm[j];
                    --j;
                }
                perm[j + 1] = v;
            }
        __syncwarp();
        for (int k = lane; k < n; k += 32) {
            const int i = perm[s + k];
            double4 p = pos[i];
            p.w = __longlong_as_double(gid[i]);
            spos[s + k] = p;
            sidx[s + k] = i;
            scell[s + k] = c;
        }
        __syncwarp();
        return;
    }
    const int v = lane < n ? perm[s + lane] : -1;
    const long long g = lane < n ? gid[v] : LLONG_MAX;
    const int g32 = lane < n ? (int)g : INT_MAX;  // global ids < 2^31 (gc_md_set_slab / set_system)
    int rank = 0;
    for (int k = 0; k < n; ++k) rank += __shfl_sync(0xffffffffu, g32, k) < g32;
    __syncwarp();
    if (lane < n) {
        perm[s + rank] = v;
        double4 p = pos[v];
        p.w = __longlong_as_double(g);
        spos[s + rank] = p;
        sidx[s + rank] = v;
        scell[s + rank] = c;
    }
    __syncwarp();
}

// two cells per warp: half-warp rank sorts when both hold <= 16 atoms (the
// common case at ~13.5 atoms per cell), else the whole warp per cell
__global__ void md_sortgather_kernel(int ncell, const int *__restrict__ cell_start, int *__restrict__ perm,
                                     const double4 *__restrict__ pos, const long long *__restrict__ gid,
                                     double4 *__restrict__ spos, int *__restrict__ sidx, int *__restrict__ scell)
{
    const int c0 = 2 * (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    const int lane = threadIdx.x & 31;
    if (c0 >= ncell) return;
    const bool two = c0 + 1 < ncell;
    const int s0 = cell_start[c0], n0 = cell_start[c0 + 1] - s0;
    const int s1 = two ? cell_start[c0 + 1] : 0, n1 = two ? cell_start[c0 + 2] - s1 : 0;
    if (n0 > 16 || n1 > 16) {
        md_sortgather_cell(c0, lane, cell_start, perm, pos, gid, spos, sidx, scell);
        if (two) md_sortgather_cell(c0 + 1, lane, cell_start, perm, pos, gid, spos, sidx, scell);
        return;
    }
    const int h = lane >> 4, l = lane & 15;
    const int c = c0 + h, s = h ? s1 : s0, n = h ? n1 : n0;
    const bool on = l < n;
    const int v = on ? perm[s + l] : -1;
    const long long g = on ? gid[v] : LLONG_MAX;
    const int g32 = on ? (int)g : INT_MAX;
    const int nm = max(n0, n1);
    int rank = 0;
    for (int k = 0; k < nm; ++k) rank += __shfl_sync(0xffffffffu, g32, k, 16) < g32;  // own half's lane k
    __syncwarp();
    if (on) {
        perm[s + rank] = v;
        double4 p = pos[v];
        p.w = __longlong_as_double(g);
        spos[s + rank] = p;
        sidx[s + rank] = v;
        scell[s + rank] = c;
    }
}

// md_step integrator (md.py:171-189) fused with the cell assignment of the
// new positions and the per-cell counts of the next cell sort (one thread per
// owned atom, coalesced)
__global__ void md_integrate_assign_kernel(int n, double4 *__restrict__ pos, double4 *__restrict__ vel,
                                           const double4 *__restrict__ force, const MDParams P, double dt,
                                           int use_npy, int *__restrict__ cell_of, int *__restrict__ count)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 p = pos[i], q = vel[i], f4 = force[i];
    double x[3] = {p.x, p.y, p.z}, v[3] = {q.x, q.y, q.z};
    const double f[3] = {f4.x, f4.y, f4.z};
    md_advance(x, v, f, P, dt);
    pos[i] = make_double4(x[0], x[1], x[2], 0.0);
    vel[i] = make_double4(v[0], v[1], v[2], 0.0);
    const int c = md_cell_index(x, P, use_npy);
    cell_of[i] = c;
    atomicAdd(&count[c], 1);
}

// md_step integrator (md.py:171-189), one atom per thread (unfused path)
__global__ void md_integrate_kernel(int n, double4 *__restrict__ pos, double4 *__restrict__ vel,
                                    const double4 *__restrict__ force, const MDParams P, double dt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x[3] = {pos[i].x, pos[i].y, pos[i].z};
    double v[3] = {vel[i].x, vel[i].y, vel[i].z};
    const double f[3] = {force[i].x, force[i].y, force[i].z};
    md_advance(x, v, f, P, dt);
    pos[i] = make_double4(x[0], x[1], x[2], 0.0);
    vel[i] = make_double4(v[0], v[1], v[2], 0.0);
}

// ghost atoms [base, base + n) of x plane `plane`: y / z cells from the
// position, x plane from the side they arrived on (a one-slab ring would
// otherwise map its own boundary atoms back onto owned planes)
__global__ void md_ghost_assign_kernel(int n, int base, int plane, const double4 *__restrict__ pos, const MDParams P,
                                       int *__restrict__ cell_of, int *__restrict__ count)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double4 p = pos[base + k];
    const double x[3] = {p.x, p.y, p.z};
    const int c = md_cell_index(x, P, 0);
    const int cyz = c % (P.ny * P.nz);
    const int cg = plane * (P.ny * P.nz) + cyz;
    cell_of[base + k] = cg;
    atomicAdd(&count[cg], 1);
}

// --- slab decomposition helpers (multi-GPU MD, md_dist.py) -------------------
// owned atoms of local x plane `plane` -> packed records: ghosts (x, y, z, gid
// bits); migrants (x, y, z, gid bits) + (vx, vy, vz, 0).  Order is irrelevant:
// every cell is re-sorted by global id.
__global__ void md_pack_kernel(int n_owned, const int *__restrict__ cell_of, int plane_cells, int plane,
                               const double4 *__restrict__ pos, const double4 *__restrict__ vel,
                               const long long *__restrict__ gid, int with_vel, double4 *__restrict__ out,
                               long long cap, int *__restrict__ cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_owned || cell_of[i] / plane_cells != plane) return;
    const int k = atomicAdd(cnt, 1);
    if (k >= cap) return;
    const double4 p = pos[i];
    if (with_vel) {
        out[2 * k] = make_double4(p.x, p.y, p.z, __longlong_as_double(gid[i]));
        out[2 * k + 1] = vel[i];
    } else {
        out[k] = make_double4(p.x, p.y, p.z, __longlong_as_double(gid[i]));
    }
}

// records -> atoms [base, base + n): positions and ids (+ velocities)
__global__ void md_unpack_kernel(int n, const double4 *__restrict__ rec, int with_vel, int base,
                                 double4 *__restrict__ pos, double4 *__restrict__ vel, long long *__restrict__ gid)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double4 r = with_vel ? rec[2 * k] : rec[k];
    pos[base + k] = make_double4(r.x, r.y, r.z, 0.0);
    gid[base + k] = __double_as_longlong(r.w);
    if (with_vel) vel[base + k] = rec[2 * k + 1];
}

// keep owned atoms still inside the slab (local x planes 1 .. nx - 2)
__global__ void md_keep_kernel(int n_owned, const int *__restrict__ cell_of, int plane_cells, int nx,
                               const double4 *__restrict__ pos, const double4 *__restrict__ vel,
                               const long long *__restrict__ gid, double4 *__restrict__ tpos,
                               double4 *__restrict__ tvel, long long *__restrict__ tgid, int *__restrict__ cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_owned) return;
    const int lx = cell_of[i] / plane_cells;
    if (lx < 1 || lx > nx - 2) return;
    const int k = atomicAdd(cnt, 1);
    tpos[k] = pos[i];
    tvel[k] = vel[i];
    tgid[k] = gid[i];
}

// --- device-count slab path (no host round trip per step) -----------------
// dn = [owned atoms, all atoms (owned + ghosts), overflow flags, scratch]; the
// kernels run over the capacity and read their counts from dn.
__global__ void mdv_pack_kernel(const int *__restrict__ dn, const int *__restrict__ cell_of, int plane_cells, int plane,
                                const double4 *__restrict__ pos, const double4 *__restrict__ vel,
                                const long long *__restrict__ gid, int with_vel, double4 *__restrict__ out, int cap,
                                int *__restrict__ cnt, int *__restrict__ flags)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= dn[0] || cell_of[i] / plane_cells != plane) return;
    const int k = atomicAdd(cnt, 1);
    if (k >= cap) {
        atomicOr(flags, 1);  // message capacity exceeded
        return;
    }
    const double4 p = pos[i];
    if (with_vel) {
        out[2 * k] = make_double4(p.x, p.y, p.z, __longlong_as_double(gid[i]));
        out[2 * k + 1] = vel[i];
    } else {
        out[k] = make_double4(p.x, p.y, p.z, __longlong_as_double(gid[i]));
    }
}

// received records -> atoms [base, base + n), base = dn[bslot] (+ *add), n = min(*cnt, cap)
__global__ void mdv_unpack_kernel(const int *__restrict__ cnt, int cap, const double4 *__restrict__ rec, int with_vel,
                                  const int *__restrict__ dn, int bslot, const int *__restrict__ add, int atom_cap,
                                  double4 *__restrict__ pos, double4 *__restrict__ vel, long long *__restrict__ gid,
                                  int *__restrict__ flags)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = min(*cnt, cap);
    if (k >= n) return;
    const int i = dn[bslot] + (add ? *add : 0) + k;
    if (i >= atom_cap) {
        atomicOr(flags, 2);  // atom capacity exceeded
        return;
    }
    const double4 r = with_vel ? rec[2 * k] : rec[k];
    pos[i] = make_double4(r.x, r.y, r.z, 0.0);
    gid[i] = __double_as_longlong(r.w);
    if (with_vel) vel[i] = rec[2 * k + 1];
}

// dn[1] = dn[0] + left + right (ghosts appended); or, after a migration,
// dn[0] = dn[1] = kept + left + right
__global__ void mdv_counts_kernel(int *__restrict__ dn, const int *__restrict__ nl, const int *__restrict__ nr, int cap,
                                  int migrate, int atom_cap)
{
    const int l = min(*nl, cap), r = min(*nr, cap);
    int n = (migrate ? dn[3] : dn[0]) + l + r;
    if (n > atom_cap) {
        dn[2] |= 2;
        n = atom_cap;
    }
    if (migrate) dn[0] = n;
    dn[1] = n;
}

__global__ void mdv_assign_kernel(const int *__restrict__ dn, int lo_slot, int hi_slot, const int *__restrict__ nl,
                                  int cap, const double4 *__restrict__ pos, const MDParams P, int use_npy,
                                  int *__restrict__ cell_of, int *__restrict__ count)
{
    // atoms [dn[lo_slot], dn[hi_slot]): owned cells from the position; ghosts
    // (lo_slot = 0, hi_slot = 1) get the x plane of the side they arrived on
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lo = lo_slot < 0 ? 0 : dn[lo_slot], hi = dn[hi_slot];
    if (i < lo || i >= hi) return;
    const double4 p = pos[i];
    const double x[3] = {p.x, p.y, p.z};
    int c = md_cell_index(x, P, use_npy);
    if (lo_slot >= 0) {  // ghost: x plane from the arrival side
        const int plane = (i - lo) < min(*nl, cap) ? 0 : P.nx - 1;
        c = plane * (P.ny * P.nz) + c % (P.ny * P.nz);
    }
    cell_of[i] = c;
    atomicAdd(&count[c], 1);
}

__global__ void mdv_scatter_kernel(const int *__restrict__ dn, const int *__restrict__ cell_start,
                                   const int *__restrict__ cell_of, int *__restrict__ count, int *__restrict__ perm)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= dn[1]) return;
    const int c = cell_of[i];
    perm[cell_start[c] + atomicSub(&count[c], 1) - 1] = i;
}

__global__ void mdv_integrate_assign_kernel(const int *__restrict__ dn, double4 *__restrict__ pos,
                                            double4 *__restrict__ vel, const double4 *__restrict__ force,
                                            const MDParams P, double dt, int use_npy, int *__restrict__ cell_of,
                                            int *__restrict__ count)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= dn[0]) return;
    const double4 p = pos[i], q = vel[i], f4 = force[i];
    double x[3] = {p.x, p.y, p.z}, v[3] = {q.x, q.y, q.z};
    const double f[3] = {f4.x, f4.y, f4.z};
    md_advance(x, v, f, P, dt);
    pos[i] = make_double4(x[0], x[1], x[2], 0.0);
    vel[i] = make_double4(v[0], v[1], v[2], 0.0);
    const int c = md_cell_index(x, P, use_npy);
    cell_of[i] = c;
    atomicAdd(&count[c], 1);
}

// owned atoms still inside the slab -> tmp (dn[3] counts them)
__global__ void mdv_keep_kernel(int *__restrict__ dn, const int *__restrict__ cell_of, int plane_cells, int nx,
                                const double4 *__restrict__ pos, const double4 *__restrict__ vel,
                                const long long *__restrict__ gid, double4 *__restrict__ tpos,
                                double4 *__restrict__ tvel, long long *__restrict__ tgid)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= dn[0]) return;
    const int lx = cell_of[i] / plane_cells;
    if (lx < 1 || lx > nx - 2) return;
    const int k = atomicAdd(&dn[3], 1);
    tpos[k] = pos[i];
    tvel[k] = vel[i];
    tgid[k] = gid[i];
}

__global__ void mdv_copy_kept_kernel(const int *__restrict__ dn, const double4 *__restrict__ tpos,
                                     const double4 *__restrict__ tvel, const long long *__restrict__ tgid,
                                     double4 *__restrict__ pos, double4 *__restrict__ vel, long long *__restrict__ gid)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= dn[3]) return;
    pos[i] = tpos[i];
    vel[i] = tvel[i];
    gid[i] = tgid[i];
}

}  // namespace gc

using namespace gc;

struct gc_md {
    gc_ctx *ctx = nullptr;
    MDParams P{};
    int law = LAW_SOFT;
    int n = 0, ncell = 0;
    int use_npy = 0;  // reference 2-D patches use numpy floor_divide
    bool cell_path = true;  // block-per-cell kernel (false: thread-per-atom kernel)
    bool lj_fast = MD_LJ_FAST != 0;  // 3-D LJ: md_lj3_kernel (else md_cell_kernel)
    bool lj_column = MD_LJ_COLUMN != 0;  // 3-D LJ: column blocks (md_lj3c_kernel) where the grid allows
    DBuf<double4> pos, vel, spos, force;  // pos/vel/gid/cell_of: owned atoms [0, n_owned), then ghosts
    DBuf<int> cell_of, scell, sidx, count, cell_start, perm;
    DBuf<long long> gid;  // global atom id (cell order, self-pair orientation)
    int n_owned = 0;
    // device-count slab path: counts live in dn (mdv_* kernels), capacity in atoms
    DBuf<int> dn;
    int atom_cap = 0;
    bool dev_counts = false;
    // slab scratch (pack / migrate)
    DBuf<int> flag, sel, nsel;
    DBuf<double4> tmp4;
    DBuf<long long> tmp8;
    cudaGraphExec_t graph = nullptr;
    int graph_steps = 0;
    double graph_dt = 0.0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~gc_md()
    {
        if (graph) cudaGraphExecDestroy(graph);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

namespace {

// Cell sort from the per-cell counts: exclusive scan -> cell_start, scatter
// (count is consumed back to zero, ready for the next step's counting),
// per-cell rank sort by original id fused with the gather into spos.
void md_sort_counted(gc_md *md)
{
    cudaStream_t s = md->ctx->stream;
    const int n = md->n, nc = md->ncell;
    size_t bytes = 0;
    GC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, md->count.p, md->cell_start.p, nc + 1, s));
    md->ctx->scratch.resize(bytes);
    GC_CUDA(cub::DeviceScan::ExclusiveSum(md->ctx->scratch.p, bytes, md->count.p, md->cell_start.p, nc + 1, s));
    md_scatter_kernel<<<grid_for(n, MD_TPB), MD_TPB, 0, s>>>(n, md->cell_start.p, md->cell_of.p, md->count.p,
                                                             md->perm.p);
    md_sortgather_kernel<<<grid_for((nc + 1) / 2, MD_TPB / 32), MD_TPB, 0, s>>>(nc, md->cell_start.p, md->perm.p, md->pos.p,
                                                                      md->gid.p, md->spos.p, md->sidx.p, md->scell.p);
    check_launch("md sort");
}

void md_sort(gc_md *md, bool assign)
{
    cudaStream_t s = md->ctx->stream;
    const int n = md->n, nc = md->ncell;
    GC_CUDA(cudaMemsetAsync(md->count.p, 0, sizeof(int) * (nc + 1), s));
    if (assign)
        md_assign_kernel<<<grid_for(n, MD_TPB), MD_TPB, 0, s>>>(n, md->pos.p, md->P, md->use_npy, md->cell_of.p,
                                                                md->count.p);
    else
        md_count_kernel<<<grid_for(n, MD_TPB), MD_TPB, 0, s>>>(n, md->cell_of.p, md->count.p);
    md_sort_counted(md);
}

template <int LAW, int DIM>
void md_cell_launch(gc_md *md, bool integ, double dt)
{
    // float32 filter: r^2 < band keeps a candidate, r^2 < inner decides it is
    // inside the cutoff; the margin >> the float32 error of relative
    // coordinates within two cells (see md_cell_kernel)
    const double ext = 3.0 * md->P.cell;
    const double margin = 1e-5 * ext * ext + 1e-6;
    const float band = (float)(md->P.c2 + margin);
    const float inner = (float)(md->P.c2 - margin);
    MDInteg I{md->pos.p, md->vel.p, md->cell_of.p, md->count.p, dt, md->use_npy};
    cudaStream_t s = md->ctx->stream;
    const int blocks = md->P.slab ? (md->P.nx - 2) * md->P.ny * md->P.nz : md->ncell;  // home = owned cells
    if (blocks <= 0) return;
    if (LAW == LAW_LJ && DIM == 3 && !integ && md->lj_fast) {
        if (md->lj_column && md->P.nx >= 3 && md->P.ny >= 3 && md->P.nz >= 3) {
            // column blocks: the float32 coordinates span (KZ + 2) cells -> widen the band accordingly
            const double extc = (MDK_KZ + 2) * md->P.cell;
            const float bandc = (float)(md->P.c2 + 1e-5 * extc * extc + 1e-6);
            const int ncz = (md->P.nz + MDK_KZ - 1) / MDK_KZ;
            const int cols = (md->P.slab ? md->P.nx - 2 : md->P.nx) * md->P.ny * ncz;
            // per device (cheap): a process may drive several GPUs
            GC_CUDA(cudaFuncSetAttribute(md_lj3c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MDK_SMEM));
            md_lj3c_kernel<<<cols, MDK_THREADS, MDK_SMEM, s>>>(md->spos.p, md->sidx.p, md->cell_start.p, md->P, bandc, ncz,
                                                        md->force.p, nullptr);
            check_launch("md_lj3c_kernel");
            return;
        }
        md_lj3_kernel<<<blocks, MDL_THREADS, 0, s>>>(md->spos.p, md->sidx.p, md->cell_start.p, md->P, band,
                                                     md->force.p);
        check_launch("md_lj3_kernel");
        return;
    }
    if (integ)
        md_cell_kernel<LAW, DIM, true><<<blocks, MDC_THREADS, 0, s>>>(md->spos.p, md->sidx.p, md->cell_start.p, md->P,
                                                                       band, inner, md->force.p, I);
    else
        md_cell_kernel<LAW, DIM, false><<<blocks, MDC_THREADS, 0, s>>>(md->spos.p, md->sidx.p, md->cell_start.p, md->P,
                                                                        band, inner, md->force.p, I);
    check_launch("md_cell_kernel");
}

// forces of the current (sorted) state; with integ, the fused step epilogue
void md_cell_forces(gc_md *md, bool integ, double dt)
{
    if (md->law == LAW_LJ) {
        if (md->P.dim == 3) md_cell_launch<LAW_LJ, 3>(md, integ, dt);
        else md_cell_launch<LAW_LJ, 2>(md, integ, dt);
    } else {
        if (md->P.dim == 3) md_cell_launch<LAW_SOFT, 3>(md, integ, dt);
        else md_cell_launch<LAW_SOFT, 2>(md, integ, dt);
    }
}

void md_forces(gc_md *md)
{
    cudaStream_t s = md->ctx->stream;
    const int n = md->n;
    if (md->cell_path) {
        md_cell_forces(md, false, 0.0);
        return;
    }
    if (md->law == LAW_LJ) {
        if (md->P.dim == 3)
            md_force_kernel<LAW_LJ, 3><<<grid_for(n, MD_TPB), MD_TPB, 0, s>>>(n, md->spos.p, md->sidx.p,
                                                                              md->cell_start.p, md->scell.p, md->P,
                                                                              md->force.p);
        else
            md_force_kernel<LAW_LJ, 2><<<grid_for(n, MD_TPB), MD_TPB, 0, s>>>(n, md->spos.p, md->sidx.p,
                                                                              md->cell_start.p, md->scell.p, md->P,
                                                                              md->force.p);
    } else {
        if (md->P.dim == 3)
            md_force_kernel<LAW_SOFT, 3><<<grid_for(n, MD_TPB), MD_TPB, 0, s>>>(n, md->spos.p, md->sidx.p,
                                                                                md->cell_start.p, md->scell.p, md->P,
                                                                                md->force.p);
        else
            md_force_kernel<LAW_SOFT, 2><<<grid_for(n, MD_TPB), MD_TPB, 0, s>>>(n, md->spos.p, md->sidx.p,
                                                                                md->cell_start.p, md->scell.p, md->P,
                                                                                md->force.p);
    }
    check_launch("md_force_kernel");
}

// One md_step (md.py:166-190) on a sorted state whose counts are zero:
// forces + integrator + new cell + counting in the cell kernel, then the
// cell sort of the new positions (4 launches).
void md_step_once(gc_md *md, double dt)
{
    if (md->cell_path) {
        md_cell_forces(md, false, dt);
        md_integrate_assign_kernel<<<grid_for(md->n, MD_TPB), MD_TPB, 0, md->ctx->stream>>>(
            md->n, md->pos.p, md->vel.p, md->force.p, md->P, dt, md->use_npy, md->cell_of.p, md->count.p);
        check_launch("md_integrate_assign_kernel");
        md_sort_counted(md);
        return;
    }
    md_forces(md);
    md_integrate_kernel<<<grid_for(md->n, MD_TPB), MD_TPB, 0, md->ctx->stream>>>(md->n, md->pos.p, md->vel.p,
                                                                                  md->force.p, md->P, dt);
    check_launch("md_integrate_kernel");
    md_sort(md, true);
}

}  // namespace

extern "C" {

gc_status gc_md_create(gc_ctx *ctx, gc_md **out)
{
    return guard([&] {
        GC_REQUIRE(ctx && out, GC_E_VALUE, "null argument");
        gc_md *md = new gc_md();
        md->ctx = ctx;
        GC_CUDA(cudaEventCreate(&md->e0));
        GC_CUDA(cudaEventCreate(&md->e1));
        *out = md;
    });
}

gc_status gc_md_destroy(gc_md *md)
{
    return guard([&] { delete md; });
}

gc_status gc_md_set_system(gc_md *md, int64_t n, int32_t dim, const double *pos, const double *vel,
                           const int64_t *cell_of, const int64_t dims[3], double cell_size, int32_t periodic,
                           int32_t law, const double params[3])
{
    return guard([&] {
        GC_REQUIRE(md && pos && n >= 0 && n < (1ll << 31), GC_E_VALUE, "bad argument");
        GC_REQUIRE(dim == 2 || dim == 3, GC_E_VALUE, "dim must be 2 or 3");
        GC_REQUIRE(law == LAW_SOFT || law == LAW_LJ, GC_E_VALUE, "unknown force law");
        GC_REQUIRE(dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1, GC_E_VALUE, "bad grid");
        GC_REQUIRE(dim == 3 || dims[2] == 1, GC_E_VALUE, "2-D grids have one layer");
        if (periodic)
            for (int k = 0; k < dim; ++k)
                GC_REQUIRE(dims[k] >= 3, GC_E_VALUE, "periodic cell grids need >= 3 cells per dimension");
        GC_REQUIRE(cell_size >= params[0], GC_E_VALUE, "patch size must cover the cutoff distance");
        MDParams &P = md->P;
        P.dim = dim;
        P.nx = (int)dims[0];
        P.ny = (int)dims[1];
        P.nz = (int)dims[2];
        P.cell = cell_size;
        P.bx = dims[0] * cell_size;
        P.by = dims[1] * cell_size;
        P.bz = dim == 3 ? dims[2] * cell_size : 0.0;
        P.periodic = periodic;
        P.cutoff = params[0];
        P.c2 = params[0] * params[0];
        P.stiffness = params[1];
        P.eps = params[1];
        P.sig2 = params[2] * params[2];
        P.slab = 0;
        P.gx0 = 1;
        P.gnx = P.nx;
        P.gbx = P.bx;
        md->law = law;
        md->use_npy = law == LAW_SOFT;
        md->n = (int)n;
        md->n_owned = (int)n;
        md->ncell = P.nx * P.ny * P.nz;
        std::vector<double4> hp(n), hv(n);
        for (int64_t i = 0; i < n; ++i) {
            hp[i] = make_double4(pos[i * dim], pos[i * dim + 1], dim == 3 ? pos[i * dim + 2] : 0.0, 0.0);
            hv[i] = vel ? make_double4(vel[i * dim], vel[i * dim + 1], dim == 3 ? vel[i * dim + 2] : 0.0, 0.0)
                        : make_double4(0, 0, 0, 0);
        }
        cudaStream_t s = md->ctx->stream;
        md->pos.upload(hp.data(), n, s);
        md->vel.upload(hv.data(), n, s);
        md->spos.resize(n);
        md->force.resize(n);
        md->cell_of.resize(n);
        md->scell.resize(n);
        md->sidx.resize(n);
        md->perm.resize(n);
        {
            std::vector<long long> g(n);
            for (int64_t i = 0; i < n; ++i) g[i] = i;
            md->gid.upload(g.data(), n, s);
        }
        md->count.resize(md->ncell + 1);
        md->cell_start.resize(md->ncell + 1);
        if (cell_of) {  // the caller's patch assignment (md.py PatchGrid.patch_of)
            std::vector<int> c(n);
            for (int64_t i = 0; i < n; ++i) {
                GC_REQUIRE(cell_of[i] >= 0 && cell_of[i] < md->ncell, GC_E_VALUE, "cell id out of range");
                c[i] = (int)cell_of[i];
            }
            md->cell_of.upload(c.data(), n, s);
            md_sort(md, false);
        } else {
            md_sort(md, true);
        }
        if (md->graph) {
            cudaGraphExecDestroy(md->graph);
            md->graph = nullptr;
        }
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_md_forces(gc_md *md, double *forces, double *energy)
{
    return guard([&] {
        GC_REQUIRE(md && md->n > 0, GC_E_STATE, "no system set");
        cudaStream_t s = md->ctx->stream;
        GC_CUDA(cudaEventRecord(md->e0, s));
        md_forces(md);
        GC_CUDA(cudaEventRecord(md->e1, s));
        std::vector<double4> f(md->n);
        md->force.download(f.data(), md->n, s);
        GC_CUDA(cudaStreamSynchronize(s));
        const int d = md->P.dim;
        for (int i = 0; i < md->n; ++i) {
            if (forces) {
                forces[i * d] = f[i].x;
                forces[i * d + 1] = f[i].y;
                if (d == 3) forces[i * d + 2] = f[i].z;
            }
            if (energy) energy[i] = f[i].w;
        }
    });
}

// `steps` md_step iterations on the device (one CUDA graph per step count)
gc_status gc_md_run(gc_md *md, int32_t steps, double dt)
{
    return guard([&] {
        GC_REQUIRE(md && md->n > 0 && steps >= 0, GC_E_STATE, "no system set");
        cudaStream_t s = md->ctx->stream;
        if (!md->graph || md->graph_steps != steps || md->graph_dt != dt) {
            if (md->graph) cudaGraphExecDestroy(md->graph);
            md->graph = nullptr;
            // make sure cub's temp storage is allocated before capture
            md_sort(md, true);
            GC_CUDA(cudaStreamSynchronize(s));
            cudaGraph_t g;
            GC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            for (int k = 0; k < steps; ++k) md_step_once(md, dt);
            GC_CUDA(cudaStreamEndCapture(s, &g));
            GC_CUDA(cudaGraphInstantiate(&md->graph, g, 0));
            cudaGraphDestroy(g);
            md->graph_steps = steps;
            md->graph_dt = dt;
        }
        GC_CUDA(cudaEventRecord(md->e0, s));
        GC_CUDA(cudaGraphLaunch(md->graph, s));
        GC_CUDA(cudaEventRecord(md->e1, s));
        GC_CUDA(cudaStreamSynchronize(s));  // every step ends with the cell sort of its new positions
    });
}

gc_status gc_md_get_state(gc_md *md, double *pos, double *vel, int64_t *cell_of)
{
    return guard([&] {
        GC_REQUIRE(md, GC_E_VALUE, "null argument");
        cudaStream_t s = md->ctx->stream;
        const int n = md->n, d = md->P.dim;
        std::vector<double4> p(n), v(n);
        std::vector<int> c(n);
        md->pos.download(p.data(), n, s);
        md->vel.download(v.data(), n, s);
        md->cell_of.download(c.data(), n, s);
        GC_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < n; ++i) {
            const double pp[3] = {p[i].x, p[i].y, p[i].z}, vv[3] = {v[i].x, v[i].y, v[i].z};
            for (int k = 0; k < d; ++k) {
                if (pos) pos[i * d + k] = pp[k];
                if (vel) vel[i * d + k] = vv[k];
            }
            if (cell_of) cell_of[i] = c[i];
        }
    });
}

gc_status gc_md_elapsed(gc_md *md, double *ms)
{
    return guard([&] {
        float t = 0.f;
        GC_CUDA(cudaEventElapsedTime(&t, md->e0, md->e1));
        *ms = t;
    });
}

// ---- slab decomposition (multi-GPU MD; orchestration in md_dist.py) ---------
static void md_grow(gc_md *md, int n)
{
    cudaStream_t s = md->ctx->stream;
    md->pos.grow(n, s);
    md->vel.grow(n, s);
    md->gid.grow(n, s);
    md->cell_of.grow(n, s);
    md->spos.resize(n);
    md->force.resize(n);
    md->scell.resize(n);
    md->sidx.resize(n);
    md->perm.resize(n);
}

gc_status gc_md_set_slab(gc_md *md, int64_t gx0, int64_t gnx, const int64_t *gid)
{
    return guard([&] {
        GC_REQUIRE(md && md->n > 0 || (md && md->ncell > 0), GC_E_STATE, "no system set");
        MDParams &P = md->P;
        GC_REQUIRE(P.dim == 3 && P.periodic, GC_E_VALUE, "slabs decompose a periodic 3-D grid");
        GC_REQUIRE(P.nx >= 3 && gnx >= P.nx - 2 && gx0 >= 0 && gx0 + P.nx - 2 <= gnx, GC_E_VALUE,
                   "slab must be local x cells = owned + 2 ghost planes inside the global grid");
        P.slab = 1;
        P.gx0 = (int)gx0;
        P.gnx = (int)gnx;
        P.gbx = (double)gnx * P.cell;
        cudaStream_t s = md->ctx->stream;
        if (gid) {
            std::vector<long long> g(md->n_owned);
            for (int i = 0; i < md->n_owned; ++i) {
                GC_REQUIRE(gid[i] >= 0 && gid[i] < INT_MAX, GC_E_VALUE, "global atom ids must be in [0, 2^31)");
                g[i] = gid[i];
            }
            md->gid.upload(g.data(), md->n_owned, s);
        }
        md->n = md->n_owned;
        if (md->graph) {
            cudaGraphExecDestroy(md->graph);
            md->graph = nullptr;
        }
        md_sort(md, true);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_md_pack(gc_md *md, int32_t what, void *out, int64_t cap, int64_t *count)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab && count, GC_E_STATE, "not a slab");
        GC_REQUIRE(what >= 0 && what <= 3, GC_E_VALUE, "what: 0/1 ghost planes, 2/3 migrants");
        cudaStream_t s = md->ctx->stream;
        const int nx = md->P.nx, pc = md->P.ny * md->P.nz;
        const int plane = what == 0 ? 1 : what == 1 ? nx - 2 : what == 2 ? 0 : nx - 1;
        md->nsel.resize(1);
        md->nsel.zero(s);
        if (md->n_owned > 0)
            md_pack_kernel<<<grid_for(md->n_owned, MD_TPB), MD_TPB, 0, s>>>(
                md->n_owned, md->cell_of.p, pc, plane, md->pos.p, md->vel.p, md->gid.p, what >= 2,
                (double4 *)out, out ? cap : 0, md->nsel.p);
        check_launch("md_pack_kernel");
        int c = 0;
        md->nsel.download(&c, 1, s);
        GC_CUDA(cudaStreamSynchronize(s));
        *count = c;
        GC_REQUIRE(!out || c <= cap, GC_E_CAPACITY, "pack buffer too small (count returned)");
    });
}

gc_status gc_md_set_ghosts(gc_md *md, const void *left, int64_t nl, const void *right, int64_t nr)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab, GC_E_STATE, "not a slab");
        cudaStream_t s = md->ctx->stream;
        const int n = md->n_owned + (int)(nl + nr);
        md_grow(md, n);
        if (nl > 0)
            md_unpack_kernel<<<grid_for(nl, MD_TPB), MD_TPB, 0, s>>>((int)nl, (const double4 *)left, 0, md->n_owned,
                                                                     md->pos.p, md->vel.p, md->gid.p);
        if (nr > 0)
            md_unpack_kernel<<<grid_for(nr, MD_TPB), MD_TPB, 0, s>>>((int)nr, (const double4 *)right, 0,
                                                                     md->n_owned + (int)nl, md->pos.p, md->vel.p,
                                                                     md->gid.p);
        check_launch("md_unpack_kernel");
        md->n = n;
        const int nc = md->ncell, no = md->n_owned;
        GC_CUDA(cudaMemsetAsync(md->count.p, 0, sizeof(int) * (nc + 1), s));
        if (no > 0)
            md_assign_kernel<<<grid_for(no, MD_TPB), MD_TPB, 0, s>>>(no, md->pos.p, md->P, md->use_npy, md->cell_of.p,
                                                                     md->count.p);
        if (nl > 0)
            md_ghost_assign_kernel<<<grid_for(nl, MD_TPB), MD_TPB, 0, s>>>((int)nl, no, 0, md->pos.p, md->P,
                                                                           md->cell_of.p, md->count.p);
        if (nr > 0)
            md_ghost_assign_kernel<<<grid_for(nr, MD_TPB), MD_TPB, 0, s>>>((int)nr, no + (int)nl, md->P.nx - 1,
                                                                           md->pos.p, md->P, md->cell_of.p,
                                                                           md->count.p);
        check_launch("md ghost cells");
        md_sort_counted(md);
    });
}

gc_status gc_md_migrate(gc_md *md, const void *in_left, int64_t nl, const void *in_right, int64_t nr)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab, GC_E_STATE, "not a slab");
        cudaStream_t s = md->ctx->stream;
        const int nown = md->n_owned;
        md->tmp4.resize(2 * (size_t)std::max(nown, 1));
        md->tmp8.resize(std::max(nown, 1));
        md->nsel.resize(1);
        md->nsel.zero(s);
        if (nown > 0)
            md_keep_kernel<<<grid_for(nown, MD_TPB), MD_TPB, 0, s>>>(
                nown, md->cell_of.p, md->P.ny * md->P.nz, md->P.nx, md->pos.p, md->vel.p, md->gid.p, md->tmp4.p,
                md->tmp4.p + nown, md->tmp8.p, md->nsel.p);
        check_launch("md_keep_kernel");
        int kept = 0;
        md->nsel.download(&kept, 1, s);
        GC_CUDA(cudaStreamSynchronize(s));
        const int n = kept + (int)(nl + nr);
        md_grow(md, std::max(n, nown));
        GC_CUDA(cudaMemcpyAsync(md->pos.p, md->tmp4.p, sizeof(double4) * kept, cudaMemcpyDeviceToDevice, s));
        GC_CUDA(cudaMemcpyAsync(md->vel.p, md->tmp4.p + nown, sizeof(double4) * kept, cudaMemcpyDeviceToDevice, s));
        GC_CUDA(cudaMemcpyAsync(md->gid.p, md->tmp8.p, sizeof(long long) * kept, cudaMemcpyDeviceToDevice, s));
        if (nl > 0)
            md_unpack_kernel<<<grid_for(nl, MD_TPB), MD_TPB, 0, s>>>((int)nl, (const double4 *)in_left, 1, kept,
                                                                     md->pos.p, md->vel.p, md->gid.p);
        if (nr > 0)
            md_unpack_kernel<<<grid_for(nr, MD_TPB), MD_TPB, 0, s>>>((int)nr, (const double4 *)in_right, 1,
                                                                     kept + (int)nl, md->pos.p, md->vel.p, md->gid.p);
        check_launch("md_unpack_kernel");
        md->n_owned = md->n = n;
        md_grow(md, n);
        md_sort(md, true);  // cells of the owned atoms (ghosts are refreshed before the next step)
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_md_slab_step(gc_md *md, double dt)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab, GC_E_STATE, "not a slab");
        cudaStream_t s = md->ctx->stream;
        GC_CUDA(cudaEventRecord(md->e0, s));
        md_cell_forces(md, false, dt);  // forces on the owned cells
        if (md->n_owned > 0)  // integrator + new cells of the owned atoms (ghosts are never advanced)
            md_integrate_assign_kernel<<<grid_for(md->n_owned, MD_TPB), MD_TPB, 0, s>>>(
                md->n_owned, md->pos.p, md->vel.p, md->force.p, md->P, dt, md->use_npy, md->cell_of.p, md->count.p);
        check_launch("md_integrate_assign_kernel");
        GC_CUDA(cudaEventRecord(md->e1, s));
    });
}

// ---- column work requests (configs[4] arrivals through the batcher) --------
// out = {columns (0: the column kernel does not apply), home cells per column
// (KZ), columns along z}
gc_status gc_md_columns(gc_md *md, int64_t out[3])
{
    return guard([&] {
        GC_REQUIRE(md && out, GC_E_VALUE, "null argument");
        const MDParams &P = md->P;
        const bool ok = md->law == LAW_LJ && P.dim == 3 && md->lj_fast && md->lj_column && !P.slab && P.nx >= 3 &&
                        P.ny >= 3 && P.nz >= 3;
        const int ncz = (P.nz + MDK_KZ - 1) / MDK_KZ;
        out[0] = ok ? (int64_t)P.nx * P.ny * ncz : 0;
        out[1] = MDK_KZ;
        out[2] = ncz;
    });
}

// forces of the home cells of columns cols[0..n) (device int32 list; the
// current cell order), asynchronous: one combined launch of n column requests
gc_status gc_md_forces_columns(gc_md *md, const int32_t *cols, int64_t n)
{
    return guard([&] {
        GC_REQUIRE(md && md->n > 0 && (cols || n == 0), GC_E_STATE, "no system set / null argument");
        int64_t c[3];
        const gc_status st = gc_md_columns(md, c);
        GC_REQUIRE(st == GC_OK && c[0] > 0, GC_E_STATE, "the column kernel does not apply to this system");
        if (n == 0) return;
        const double extc = (MDK_KZ + 2) * md->P.cell;
        const float bandc = (float)(md->P.c2 + 1e-5 * extc * extc + 1e-6);
        GC_CUDA(cudaFuncSetAttribute(md_lj3c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MDK_SMEM));
        md_lj3c_kernel<<<(unsigned)n, MDK_THREADS, MDK_SMEM, md->ctx->stream>>>(
            md->spos.p, md->sidx.p, md->cell_start.p, md->P, bandc, (int)c[2], md->force.p, cols);
        check_launch("md_lj3c_kernel (columns)");
    });
}

// the force array as it stands (no evaluation): forces (n, dim), energy (n)
gc_status gc_md_get_forces(gc_md *md, double *forces, double *energy)
{
    return guard([&] {
        GC_REQUIRE(md && md->n > 0, GC_E_STATE, "no system set");
        cudaStream_t s = md->ctx->stream;
        std::vector<double4> f(md->n);
        md->force.download(f.data(), md->n, s);
        GC_CUDA(cudaStreamSynchronize(s));
        const int d = md->P.dim;
        for (int i = 0; i < md->n; ++i) {
            if (forces)
                for (int k = 0; k < d; ++k) forces[i * d + k] = k == 0 ? f[i].x : (k == 1 ? f[i].y : f[i].z);
            if (energy) energy[i] = f[i].w;
        }
    });
}

// ---- device-count slab path (multi-GPU MD without host round trips) --------
namespace {
void mdv_enter(gc_md *md)
{
    if (md->dev_counts) return;
    cudaStream_t s = md->ctx->stream;
    const int cap = std::max(2 * md->n_owned + 4096, md->n);
    md_grow(md, cap);
    md->tmp4.resize(2 * (size_t)cap);
    md->tmp8.resize(cap);
    md->atom_cap = cap;
    md->dn.resize(4);
    const int h[4] = {md->n_owned, md->n, 0, 0};
    md->dn.upload(h, 4, s);
    GC_CUDA(cudaStreamSynchronize(s));
    md->dev_counts = true;
}

void mdv_sort(gc_md *md)
{
    cudaStream_t s = md->ctx->stream;
    const int nc = md->ncell, cap = md->atom_cap;
    size_t bytes = 0;
    GC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, md->count.p, md->cell_start.p, nc + 1, s));
    md->ctx->scratch.resize(std::max(bytes, md->ctx->scratch.n));
    GC_CUDA(cub::DeviceScan::ExclusiveSum(md->ctx->scratch.p, bytes, md->count.p, md->cell_start.p, nc + 1, s));
    mdv_scatter_kernel<<<grid_for(cap, MD_TPB), MD_TPB, 0, s>>>(md->dn.p, md->cell_start.p, md->cell_of.p,
                                                                md->count.p, md->perm.p);
    md_sortgather_kernel<<<grid_for((nc + 1) / 2, MD_TPB / 32), MD_TPB, 0, s>>>(nc, md->cell_start.p, md->perm.p, md->pos.p,
                                                                      md->gid.p, md->spos.p, md->sidx.p, md->scell.p);
    check_launch("mdv sort");
}
}  // namespace

gc_status gc_md_pack_dev(gc_md *md, int32_t what, void *out, int64_t cap, int32_t *count)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab && out && count && cap >= 0, GC_E_STATE, "not a slab / null argument");
        GC_REQUIRE(what >= 0 && what <= 3, GC_E_VALUE, "what: 0/1 ghost planes, 2/3 migrants");
        mdv_enter(md);
        cudaStream_t s = md->ctx->stream;
        const int nx = md->P.nx, pc = md->P.ny * md->P.nz;
        const int plane = what == 0 ? 1 : what == 1 ? nx - 2 : what == 2 ? 0 : nx - 1;
        GC_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), s));
        mdv_pack_kernel<<<grid_for(md->atom_cap, MD_TPB), MD_TPB, 0, s>>>(
            md->dn.p, md->cell_of.p, pc, plane, md->pos.p, md->vel.p, md->gid.p, what >= 2, (double4 *)out, (int)cap,
            count, md->dn.p + 2);
        check_launch("mdv_pack_kernel");
    });
}

gc_status gc_md_set_ghosts_dev(gc_md *md, const void *left, const int32_t *n_left, const void *right,
                               const int32_t *n_right, int64_t cap)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab && left && right && n_left && n_right, GC_E_STATE, "not a slab / null argument");
        mdv_enter(md);
        cudaStream_t s = md->ctx->stream;
        const int c = (int)cap, ac = md->atom_cap;
        mdv_unpack_kernel<<<grid_for(c, MD_TPB), MD_TPB, 0, s>>>(n_left, c, (const double4 *)left, 0, md->dn.p, 0,
                                                                 nullptr, ac, md->pos.p, md->vel.p, md->gid.p,
                                                                 md->dn.p + 2);
        mdv_unpack_kernel<<<grid_for(c, MD_TPB), MD_TPB, 0, s>>>(n_right, c, (const double4 *)right, 0, md->dn.p, 0,
                                                                 n_left, ac, md->pos.p, md->vel.p, md->gid.p,
                                                                 md->dn.p + 2);
        mdv_counts_kernel<<<1, 1, 0, s>>>(md->dn.p, n_left, n_right, c, 0, ac);
        GC_CUDA(cudaMemsetAsync(md->count.p, 0, sizeof(int) * (md->ncell + 1), s));
        mdv_assign_kernel<<<grid_for(ac, MD_TPB), MD_TPB, 0, s>>>(md->dn.p, -1, 0, n_left, c, md->pos.p, md->P,
                                                                  md->use_npy, md->cell_of.p, md->count.p);
        mdv_assign_kernel<<<grid_for(ac, MD_TPB), MD_TPB, 0, s>>>(md->dn.p, 0, 1, n_left, c, md->pos.p, md->P,
                                                                  md->use_npy, md->cell_of.p, md->count.p);
        check_launch("mdv ghosts");
        mdv_sort(md);
    });
}

gc_status gc_md_slab_step_dev(gc_md *md, double dt)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab, GC_E_STATE, "not a slab");
        mdv_enter(md);
        cudaStream_t s = md->ctx->stream;
        GC_CUDA(cudaEventRecord(md->e0, s));
        md_cell_forces(md, false, dt);  // forces on the owned cells
        mdv_integrate_assign_kernel<<<grid_for(md->atom_cap, MD_TPB), MD_TPB, 0, s>>>(
            md->dn.p, md->pos.p, md->vel.p, md->force.p, md->P, dt, md->use_npy, md->cell_of.p, md->count.p);
        check_launch("mdv_integrate_assign_kernel");
        GC_CUDA(cudaEventRecord(md->e1, s));
    });
}

gc_status gc_md_migrate_dev(gc_md *md, const void *in_left, const int32_t *n_left, const void *in_right,
                            const int32_t *n_right, int64_t cap)
{
    return guard([&] {
        GC_REQUIRE(md && md->P.slab && in_left && in_right && n_left && n_right, GC_E_STATE,
                   "not a slab / null argument");
        mdv_enter(md);
        cudaStream_t s = md->ctx->stream;
        const int c = (int)cap, ac = md->atom_cap;
        GC_CUDA(cudaMemsetAsync(md->dn.p + 3, 0, sizeof(int), s));
        mdv_keep_kernel<<<grid_for(ac, MD_TPB), MD_TPB, 0, s>>>(md->dn.p, md->cell_of.p, md->P.ny * md->P.nz,
                                                                md->P.nx, md->pos.p, md->vel.p, md->gid.p, md->tmp4.p,
                                                                md->tmp4.p + ac, md->tmp8.p);
        mdv_copy_kept_kernel<<<grid_for(ac, MD_TPB), MD_TPB, 0, s>>>(md->dn.p, md->tmp4.p, md->tmp4.p + ac,
                                                                     md->tmp8.p, md->pos.p, md->vel.p, md->gid.p);
        mdv_unpack_kernel<<<grid_for(c, MD_TPB), MD_TPB, 0, s>>>(n_left, c, (const double4 *)in_left, 1, md->dn.p, 3,
                                                                 nullptr, ac, md->pos.p, md->vel.p, md->gid.p,
                                                                 md->dn.p + 2);
        mdv_unpack_kernel<<<grid_for(c, MD_TPB), MD_TPB, 0, s>>>(n_right, c, (const double4 *)in_right, 1, md->dn.p,
                                                                 3, n_left, ac, md->pos.p, md->vel.p, md->gid.p,
                                                                 md->dn.p + 2);
        mdv_counts_kernel<<<1, 1, 0, s>>>(md->dn.p, n_left, n_right, c, 1, ac);
        GC_CUDA(cudaMemsetAsync(md->count.p, 0, sizeof(int) * (md->ncell + 1), s));
        mdv_assign_kernel<<<grid_for(ac, MD_TPB), MD_TPB, 0, s>>>(md->dn.p, -1, 0, n_left, c, md->pos.p, md->P,
                                                                  md->use_npy, md->cell_of.p, md->count.p);
        check_launch("mdv migrate");
        mdv_sort(md);
    });
}

// host view of the device counts (synchronises): out = {owned, all atoms, overflow flags}
gc_status gc_md_slab_counts(gc_md *md, int64_t out[3])
{
    return guard([&] {
        GC_REQUIRE(md && out, GC_E_VALUE, "null argument");
        if (!md->dev_counts) {
            out[0] = md->n_owned;
            out[1] = md->n;
            out[2] = 0;
            return;
        }
        int h[4];
        md->dn.download(h, 4, md->ctx->stream);
        GC_CUDA(cudaStreamSynchronize(md->ctx->stream));
        out[0] = h[0];
        out[1] = h[1];
        out[2] = h[2];
        md->n_owned = h[0];
        md->n = h[1];
    });
}

gc_status gc_md_owned(gc_md *md, int64_t *n_owned, double *pos, double *vel, int64_t *gid)
{
    return guard([&] {
        GC_REQUIRE(md && n_owned, GC_E_VALUE, "null argument");
        if (md->dev_counts) {  // refresh the host counts from the device path
            int64_t c[3];
            const gc_status st = gc_md_slab_counts(md, c);
            GC_REQUIRE(st == GC_OK, st, gc_last_error());
            GC_REQUIRE(c[2] == 0, GC_E_CAPACITY, "slab message / atom capacity exceeded (device-count path)");
        }
        const int n = md->n_owned;
        *n_owned = n;
        if (!pos && !vel && !gid) return;
        cudaStream_t s = md->ctx->stream;
        std::vector<double4> p(n), v(n);
        std::vector<long long> g(n);
        md->pos.download(p.data(), n, s);
        md->vel.download(v.data(), n, s);
        md->gid.download(g.data(), n, s);
        GC_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < n; ++i) {
            const double pp[3] = {p[i].x, p[i].y, p[i].z}, vv[3] = {v[i].x, v[i].y, v[i].z};
            for (int k = 0; k < 3; ++k) {
                if (pos) pos[3 * i + k] = pp[k];
                if (vel) vel[3 * i + k] = vv[k];
            }
            if (gid) gid[i] = g[i];
        }
    });
}

}  // extern "C"


namespace gc {
void md_kernel_spec(const char *cls, int64_t out[5])
{
    if (!strcmp(cls, "md_column")) {  // the LJ column kernel: one work request (column of home cells) per block
        cudaFuncAttributes a;
        GC_CUDA(cudaFuncGetAttributes(&a, md_lj3c_kernel));
        GC_CUDA(cudaFuncSetAttribute(md_lj3c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MDK_SMEM));
        int blocks = 0;
        GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, md_lj3c_kernel, MDK_THREADS, MDK_SMEM));
        out[0] = MDK_THREADS;
        out[1] = a.numRegs;
        out[2] = (int64_t)a.sharedSizeBytes + MDK_SMEM;
        out[3] = 1;
        out[4] = blocks;
        return;
    }
    const void *fn = (const void *)md_force_kernel<LAW_LJ, 3>;
    cudaFuncAttributes a;
    GC_CUDA(cudaFuncGetAttributes(&a, fn));
    int blocks = 0;
    GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, MD_TPB, 0));
    out[0] = MD_TPB;
    out[1] = a.numRegs;
    out[2] = (int64_t)a.sharedSizeBytes;
    out[3] = MD_TPB;  // one atom (one cell-pair row) per thread
    out[4] = blocks;
}
}  // namespace gc
