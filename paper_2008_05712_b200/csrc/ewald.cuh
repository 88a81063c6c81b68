// ewald.cuh -- the "ewald" kernel class on sm_100a.
//
// The reference only MODELS this class: NBodyWorkload submits one request per
// bucket, buffers [bucket], item_count max(1, n_b) (hr/workloads/nbody.py:
// 317-323), and the simulator charges its cost (hr/devicesim.py:92-99).  Here
// it computes what a ChaNGa-style code computes for it: the periodic (Ewald)
// correction of every particle of the bucket from the root multipole
// (monopole + traceless quadrupole about the centre of mass), Hernquist,
// Bouchet & Suto (1991) as in PKDGRAV / ChaNGa.  Float64 throughout; the
// restatement it is checked against is oracle/gcharm_oracle.c
// (orc_ewald_correction, same formulas and term order per lane-free sum).
//
// Work decomposition: one warp per particle (or per member bucket, looping
// over its particles); the lanes split the term list -- real-space replicas
// then Fourier vectors, host-built tables in HBM -- and the warp reduces with
// a fixed xor tree, so results are deterministic.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

namespace gc {

constexpr int EW_SERIES = 12;

struct EwaldParams {
    double L, alpha, a2, ka, L3, cut2, inner2, k0;  // k0: pi M / (alpha^2 L^3) per unit M
    int nreal, nk;
    double ser[4][EW_SERIES];  // power series of B_0..B_3 near r = 0 (central replica)
};

// params[5] = L, alpha (<= 0: 2 / L), nrep, ewcut, hcut
inline EwaldParams ewald_setup(const double params[5], std::vector<double4> &real, std::vector<double4> &kv)
{
    EwaldParams P{};
    P.L = params[0];
    P.alpha = params[1] > 0 ? params[1] : 2.0 / P.L;
    const int nrep = (int)params[2];
    const double ewcut = params[3], hcut = params[4];
    P.a2 = P.alpha * P.alpha;
    P.ka = 2.0 * P.alpha / std::sqrt(M_PI);
    P.L3 = P.L * P.L * P.L;
    P.cut2 = ewcut * P.L * ewcut * P.L;
    P.inner2 = 0.04 / P.a2;
    P.k0 = M_PI / (P.a2 * P.L3);
    real.clear();
    kv.clear();
    for (int ix = -nrep; ix <= nrep; ++ix)
        for (int iy = -nrep; iy <= nrep; ++iy)
            for (int iz = -nrep; iz <= nrep; ++iz)
                real.push_back(make_double4(ix * P.L, iy * P.L, iz * P.L, (ix == 0 && iy == 0 && iz == 0) ? 1.0 : 0.0));
    const int hrep = (int)std::ceil(hcut);
    for (int mx = -hrep; mx <= hrep; ++mx)
        for (int my = -hrep; my <= hrep; ++my)
            for (int mz = -hrep; mz <= hrep; ++mz) {
                const int m2 = mx * mx + my * my + mz * mz;
                if (m2 == 0 || m2 > hcut * hcut) continue;
                const double k[3] = {2.0 * M_PI * mx / P.L, 2.0 * M_PI * my / P.L, 2.0 * M_PI * mz / P.L};
                const double k2 = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
                kv.push_back(make_double4(k[0], k[1], k[2], 4.0 * M_PI / P.L3 * std::exp(-k2 / (4.0 * P.a2)) / k2));
            }
    P.nreal = (int)real.size();
    P.nk = (int)kv.size();
    // t_{0,j} = -(-1)^j / (j! (2j+1)),  t_{l+1,j} = -(j+1) t_{l,j+1}
    double t[EW_SERIES + 4];
    double fact = 1.0;
    for (int j = 0; j < EW_SERIES + 4; ++j) {
        if (j > 0) fact *= j;
        t[j] = -((j & 1) ? -1.0 : 1.0) / (fact * (2 * j + 1));
    }
    double scale = P.ka;
    for (int l = 0; l < 4; ++l) {
        for (int j = 0; j < EW_SERIES; ++j) P.ser[l][j] = scale * t[j];
        for (int j = 0; j < EW_SERIES + 3 - l; ++j) t[j] = -(j + 1) * t[j + 1];
        scale *= 2.0 * P.a2;
    }
    return P;
}

// The correction at offset d (= x - com) from moments mom = [M, com(3),
// Q xx yy zz xy xz yz]; every lane returns the warp total (a[3], phi).
__device__ __forceinline__ void ewald_warp(const double d[3], const double *__restrict__ mom, const EwaldParams &P,
                                           const double4 *__restrict__ real, const double4 *__restrict__ kv, int lane,
                                           double a[3], double &phi)
{
    const double M = mom[0];
    const double Q00 = mom[4], Q11 = mom[5], Q22 = mom[6], Q01 = mom[7], Q02 = mom[8], Q12 = mom[9];
    a[0] = a[1] = a[2] = 0.0;
    phi = 0.0;
    for (int t = lane; t < P.nreal; t += 32) {
        const double4 n = real[t];
        const bool hole = n.w != 0.0;
        const double y0 = d[0] + n.x, y1 = d[1] + n.y, y2 = d[2] + n.z;
        const double r2 = y0 * y0 + y1 * y1 + y2 * y2;
        if (!hole && r2 > P.cut2) continue;
        double B0, B1, B2, B3;
        if (hole && r2 < P.inner2) {
            const double s = P.a2 * r2;
            double b[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                double acc = 0.0;
#pragma unroll
                for (int j = EW_SERIES - 1; j >= 0; --j) acc = acc * s + P.ser[l][j];
                b[l] = acc;
            }
            B0 = b[0];
            B1 = b[1];
            B2 = b[2];
            B3 = b[3];
        } else {
            const double r = sqrt(r2), e = P.ka * exp(-P.a2 * r2);
            B0 = (hole ? -erf(P.alpha * r) : erfc(P.alpha * r)) / r;
            B1 = (B0 + e) / r2;
            B2 = (3.0 * B1 + 2.0 * P.a2 * e) / r2;
            B3 = (5.0 * B2 + 4.0 * P.a2 * P.a2 * e) / r2;
        }
        const double q0 = Q00 * y0 + Q01 * y1 + Q02 * y2;
        const double q1 = Q01 * y0 + Q11 * y1 + Q12 * y2;
        const double q2 = Q02 * y0 + Q12 * y1 + Q22 * y2;
        const double yQy = y0 * q0 + y1 * q1 + y2 * q2;
        a[0] += -M * y0 * B1 + (-y0 * yQy * B3 + 2.0 * q0 * B2) / 6.0;
        a[1] += -M * y1 * B1 + (-y1 * yQy * B3 + 2.0 * q1 * B2) / 6.0;
        a[2] += -M * y2 * B1 + (-y2 * yQy * B3 + 2.0 * q2 * B2) / 6.0;
        phi += -M * B0 - yQy * B2 / 6.0;
    }
    for (int t = lane; t < P.nk; t += 32) {
        const double4 k = kv[t];
        const double kQk = k.x * (Q00 * k.x + Q01 * k.y + Q02 * k.z) + k.y * (Q01 * k.x + Q11 * k.y + Q12 * k.z) +
                           k.z * (Q02 * k.x + Q12 * k.y + Q22 * k.z);
        const double kd = k.x * d[0] + k.y * d[1] + k.z * d[2];
        const double coef = k.w * (kQk / 6.0 - M);
        double sn, cs;
        sincos(kd, &sn, &cs);
        a[0] += k.x * sn * coef;
        a[1] += k.y * sn * coef;
        a[2] += k.z * sn * coef;
        phi += cs * coef;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
        a[1] += __shfl_xor_sync(0xffffffffu, a[1], o);
        a[2] += __shfl_xor_sync(0xffffffffu, a[2], o);
        phi += __shfl_xor_sync(0xffffffffu, phi, o);
    }
    phi += M * P.k0;
}

}  // namespace gc
