// d2q37_device.cuh -- device-side building blocks of the D2Q37 hot path (sm_100a).
//
// HBM layout: the reference's padded SoA / CSoA
// storage (layout.hpp:46-98) generalised with a column pitch, so that one
// code path serves both layouts (SoA is CSoA with vl = 1):
//
//   elem(p, X, j, k) = lead + p*plane + (X*pitch + j)*vl + k
//
//   X in [0, lx+6)        padded column (3 ghost columns each side)
//   j in [0, strip+6)     padded row of a lane strip (3 halo rows each end)
//   k in [0, vl)          lane; lattice y = k*strip + (j - 3)
//
// pitch >= sy = strip + 6 and lead are chosen so that every column's first
// physical element (j = 3, k = 0) starts a 256-byte segment: one warp of
// consecutive q = (j-3)*vl + k stores two whole 128-byte lines.
#pragma once

#include <cstdint>

#include "d2q37_velocities.h"

namespace d2q37 {

struct DevGeo {
    int lx, ly;     // lattice (or slab) extents
    int vl, strip;  // lanes, rows per lane strip (strip = ly / vl)
    int sy;         // strip + 6 (reference padded rows per lane)
    int pitch;      // device rows per padded column (>= sy)
    int px;         // lx + 6
    int pad_;
    long long lead;   // element offset of population plane 0
    long long plane;  // elements per population plane
};

__host__ __device__ __forceinline__ long long elem_of(const DevGeo& g, int p, int X, int j, int k) {
    return g.lead + (long long)p * g.plane + ((long long)X * g.pitch + j) * g.vl + k;
}
// Element of physical q (q = (j-3)*vl + k, 0 <= q < ly) of column X, population 0.
__host__ __device__ __forceinline__ long long col_base(const DevGeo& g, int X) {
    return g.lead + ((long long)X * g.pitch + kHalo) * g.vl;
}

// Model constants travel as kernel parameters (constant bank 0, broadcast to
// every lane), so lattices with different models never race on __constant__.
struct ModelParams {
    double eq[kNpop][kNmom];
    double w[kNpop];
    double t0;
};

struct Offsets {
    long long o[kNpop];
};

// FP helpers: FAST lets nvcc contract a*b+c into DFMA; STRICT rounds every op.
template <bool STRICT>
struct Arith;
template <>
struct Arith<false> {
    static __device__ __forceinline__ double add(double a, double b) { return a + b; }
    static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
    static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
    static __device__ __forceinline__ double madd(double acc, double a, double b) { return fma(a, b, acc); }
    static __device__ __forceinline__ double rcp(double a) { return 1.0 / a; }
};
template <>
struct Arith<true> {
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double madd(double acc, double a, double b) {
        return __dadd_rn(acc, __dmul_rn(a, b));
    }
    static __device__ __forceinline__ double rcp(double a) { return __ddiv_rn(1.0, a); }
};

// VelocityModel::collide_site (model.cpp:293-298) = macros_of (:242-257) +
// equilibrium (:259-291) + relaxation, in place on f[37].  Reductions keep the
// reference's canonical population order; terms that are zero by the
// structure of the velocity set (cx = 0 or cy = 0 rows) are skipped, which is
// exact for finite inputs.  Returns true when !(rho > 0) (NonPhysicalError).
template <bool STRICT>
__device__ __forceinline__ bool collide_site(double (&f)[kNpop], double omega, const ModelParams& mp) {
    using A = Arith<STRICT>;
    double rho = 0.0;
#pragma unroll
    for (int i = 0; i < kNpop; ++i) rho = A::add(rho, f[i]);
    const bool bad = !(rho > 0.0);
    double jx = 0.0, jy = 0.0, e2 = 0.0;
#pragma unroll
    for (int i = 0; i < kNpop; ++i)
        if (cx_of(i) != 0) jx = A::madd(jx, (double)cx_of(i), f[i]);
#pragma unroll
    for (int i = 0; i < kNpop; ++i)
        if (cy_of(i) != 0) jy = A::madd(jy, (double)cy_of(i), f[i]);
#pragma unroll
    for (int i = 0; i < kNpop; ++i)
        if (cx_of(i) != 0 || cy_of(i) != 0)
            e2 = A::madd(e2, (double)(cx_of(i) * cx_of(i) + cy_of(i) * cy_of(i)), f[i]);
    const double inv_rho = A::rcp(rho);
    const double ux = A::mul(jx, inv_rho);
    const double uy = A::mul(jy, inv_rho);
    const double temp = A::mul(0.5, A::sub(A::mul(e2, inv_rho), A::add(A::mul(ux, ux), A::mul(uy, uy))));

    const double dt = A::sub(temp, mp.t0);
    const double ux2 = A::mul(ux, ux), uy2 = A::mul(uy, uy), uxuy = A::mul(ux, uy);
    const double dt3 = A::mul(3.0, dt);
    const double dt6 = A::mul(6.0, dt);
    const double dt2 = A::mul(dt, dt);
    const double dt2x3 = A::mul(3.0, dt2);
    double mom[kNmom];
    mom[0] = ux;
    mom[1] = uy;
    mom[2] = A::add(ux2, dt);
    mom[3] = uxuy;
    mom[4] = A::add(uy2, dt);
    mom[5] = A::mul(ux, A::add(ux2, dt3));
    mom[6] = A::mul(uy, A::add(ux2, dt));
    mom[7] = A::mul(ux, A::add(uy2, dt));
    mom[8] = A::mul(uy, A::add(uy2, dt3));
    mom[9] = A::add(A::mul(ux2, A::add(ux2, dt6)), dt2x3);
    mom[10] = A::mul(uxuy, A::add(ux2, dt3));
    mom[11] = A::add(A::add(A::mul(uxuy, uxuy), A::mul(dt, A::add(ux2, uy2))), dt2);
    mom[12] = A::mul(uxuy, A::add(uy2, dt3));
    mom[13] = A::add(A::mul(uy2, A::add(uy2, dt6)), dt2x3);

#pragma unroll
    for (int i = 0; i < kNpop; ++i) {
        double s = 1.0;
#pragma unroll
        for (int k = 0; k < kNmom; ++k)
            if (!eq_structural_zero(i, k)) s = A::madd(s, mp.eq[i][k], mom[k]);
        const double feq = A::mul(A::mul(rho, mp.w[i]), s);
        f[i] = A::madd(f[i], omega, A::sub(feq, f[i]));
    }
    return bad;
}

}  // namespace d2q37
