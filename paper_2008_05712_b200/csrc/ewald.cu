// ewald.cu -- Ewald correction entry points (see ewald.cuh): root multipole
// moments by a deterministic two-pass device reduction, the correction at
// arbitrary points (one warp per point), and the bh handle's moments / output.
// The member kernel of the "ewald" kernel class (reading bucket particles
// from their data-manager slots) lives in dm.cu next to the slot pool.
#include <cub/cub.cuh>

#include "bh_state.h"
#include "common.cuh"
#include "ewald.cuh"

namespace gc {

constexpr int EW_RED_BLOCKS = 296, EW_RED_TPB = 256, EW_TPB = 256;

// pass 0: (m, m x, m y, m z); pass 1: traceless Q about mom[1..3]
__global__ void __launch_bounds__(EW_RED_TPB) ew_moments_partial(int64_t n, const double *__restrict__ pos,
                                                                 const double *__restrict__ mass, int pass,
                                                                 const double *__restrict__ mom,
                                                                 double *__restrict__ part)
{
    double v[6] = {0, 0, 0, 0, 0, 0};
    const double c0 = pass ? mom[1] : 0.0, c1 = pass ? mom[2] : 0.0, c2 = pass ? mom[3] : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)EW_RED_TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * EW_RED_TPB) {
        const double m = mass[i];
        if (!pass) {
            v[0] += m;
            v[1] += m * pos[3 * i];
            v[2] += m * pos[3 * i + 1];
            v[3] += m * pos[3 * i + 2];
        } else {
            const double y0 = pos[3 * i] - c0, y1 = pos[3 * i + 1] - c1, y2 = pos[3 * i + 2] - c2;
            const double y2s = y0 * y0 + y1 * y1 + y2 * y2;
            v[0] += m * (3.0 * y0 * y0 - y2s);
            v[1] += m * (3.0 * y1 * y1 - y2s);
            v[2] += m * (3.0 * y2 * y2 - y2s);
            v[3] += m * 3.0 * y0 * y1;
            v[4] += m * 3.0 * y0 * y2;
            v[5] += m * 3.0 * y1 * y2;
        }
    }
    typedef cub::BlockReduce<double, EW_RED_TPB> Red;
    __shared__ typename Red::TempStorage ts;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double s = Red(ts).Sum(v[k]);
        if (threadIdx.x == 0) part[blockIdx.x * 6 + k] = s;
        __syncthreads();
    }
}

__global__ void ew_moments_final(int nb, const double *__restrict__ part, int pass, double *__restrict__ mom)
{
    if (threadIdx.x != 0) return;
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int b = 0; b < nb; ++b)
        for (int k = 0; k < 6; ++k) v[k] += part[b * 6 + k];
    if (!pass) {
        mom[0] = v[0];
        for (int k = 0; k < 3; ++k) mom[1 + k] = v[0] > 0 ? v[1 + k] / v[0] : 0.0;
    } else {
        for (int k = 0; k < 6; ++k) mom[4 + k] = v[k];
    }
}

void ewald_moments_device(int64_t n, const double *pos, const double *mass, double *mom, double *part, cudaStream_t s)
{
    for (int pass = 0; pass < 2; ++pass) {
        ew_moments_partial<<<EW_RED_BLOCKS, EW_RED_TPB, 0, s>>>(n, pos, mass, pass, mom, part);
        check_launch("ew_moments_partial");
        ew_moments_final<<<1, 32, 0, s>>>(EW_RED_BLOCKS, part, pass, mom);
        check_launch("ew_moments_final");
    }
}

__global__ void __launch_bounds__(EW_TPB) ewald_points_kernel(int64_t n, const double *__restrict__ pos,
                                                              const double *__restrict__ mom, const EwaldParams P,
                                                              const double4 *__restrict__ real,
                                                              const double4 *__restrict__ kv, double *__restrict__ acc,
                                                              double *__restrict__ pot)
{
    const int64_t i = (blockIdx.x * (int64_t)EW_TPB + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const double d[3] = {pos[3 * i] - mom[1], pos[3 * i + 1] - mom[2], pos[3 * i + 2] - mom[3]};
    double a[3], phi;
    ewald_warp(d, mom, P, real, kv, lane, a, phi);
    if (lane == 0) {
        acc[3 * i] = a[0];
        acc[3 * i + 1] = a[1];
        acc[3 * i + 2] = a[2];
        if (pot) pot[i] = phi;
    }
}

}  // namespace gc

using namespace gc;

extern "C" {

gc_status gc_ewald_moments(gc_ctx *ctx, int64_t n, const double *pos, const double *mass, double out[10])
{
    return guard([&] {
        GC_REQUIRE(ctx && pos && mass && out && n >= 1, GC_E_VALUE, "bad argument");
        cudaStream_t s = ctx->stream;
        DBuf<double> p, m, part, mom;
        p.upload(pos, 3 * n, s);
        m.upload(mass, n, s);
        part.resize(6 * EW_RED_BLOCKS);
        mom.resize(10);
        ewald_moments_device(n, p.p, m.p, mom.p, part.p, s);
        mom.download(out, 10, s);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

gc_status gc_ewald_correction(gc_ctx *ctx, int64_t n, const double *pos, const double moments[10],
                              const double params[5], double *acc, double *pot)
{
    return guard([&] {
        GC_REQUIRE(ctx && pos && moments && params && acc && n >= 0, GC_E_VALUE, "bad argument");
        GC_REQUIRE(params[0] > 0 && params[2] >= 0 && params[3] > 0 && params[4] > 0, GC_E_VALUE, "bad Ewald parameters");
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        std::vector<double4> real, kv;
        const EwaldParams P = ewald_setup(params, real, kv);
        DBuf<double4> dr, dk;
        DBuf<double> p, mom, a, ph;
        dr.upload(real.data(), real.size(), s);
        dk.upload(kv.data(), std::max<size_t>(kv.size(), 1), s);
        p.upload(pos, 3 * n, s);
        mom.upload(moments, 10, s);
        a.resize(3 * n);
        ph.resize(n);
        ewald_points_kernel<<<grid_for(32 * n, EW_TPB), EW_TPB, 0, s>>>(n, p.p, mom.p, P, dr.p, dk.p, a.p, ph.p);
        check_launch("ewald_points_kernel");
        a.download(acc, 3 * n, s);
        if (pot) ph.download(pot, n, s);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

// root multipole of the handle's particles (3-D), cached until the next set_particles
gc_status gc_bh_ewald_moments(gc_bh *bh, double out[10])
{
    return guard([&] {
        GC_REQUIRE(bh && bh->have_tree, GC_E_STATE, "no tree");
        GC_REQUIRE(bh->dim == 3, GC_E_VALUE, "Ewald summation needs dim = 3");
        GC_REQUIRE(bh->ws.pos.n == (size_t)(3 * bh->n) && bh->ws.mass.n == (size_t)bh->n, GC_E_STATE,
                   "float64 particles not resident");
        cudaStream_t s = bh->ctx->stream;
        if (!bh->ew_mom_valid) {
            if (bh->side) GC_CUDA(cudaStreamWaitEvent(s, bh->side_done, 0));  // masses uploaded on the side stream
            bh->d_ew_mom.resize(10);
            bh->d_ew_part.resize(6 * EW_RED_BLOCKS);
            ewald_moments_device(bh->n, bh->ws.pos.p, bh->ws.mass.p, bh->d_ew_mom.p, bh->d_ew_part.p, s);
            bh->ew_mom_valid = true;
        }
        if (out) {
            bh->d_ew_mom.download(out, 10, s);
            GC_CUDA(cudaStreamSynchronize(s));
        }
    });
}

gc_status gc_bh_get_ewald(gc_bh *bh, double *forces, double *pot)
{
    return guard([&] {
        GC_REQUIRE(bh && bh->d_ewf.n >= (size_t)(3 * bh->n), GC_E_STATE, "no Ewald forces");
        cudaStream_t s = bh->ctx->stream;
        if (forces) bh->d_ewf.download(forces, 3 * bh->n, s);
        if (pot) bh->d_ewp.download(pot, bh->n, s);
        GC_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
