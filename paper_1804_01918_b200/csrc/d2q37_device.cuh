// d2q37_device.cuh -- device-side building blocks of the D2Q37 hot path (sm_100a).
//
// HBM layout: the reference's padded storage
// (layout.hpp:46-98) for all four layouts, generalised with a column pitch
// and expressed with three strides so one code path serves every layout:
//
//   elem(p, X, j, k) = lead + p*pstride + X*cstride + j*rstride + k
//   SoA/CSoA:   pstride = plane, rstride = vl      (SoA: vl = 1)
//   AoS/CAoSoA: pstride = vl,    rstride = 37*vl   (AoS: vl = 1)
//
//   X in [0, lx+6)        padded column (3 ghost columns each side)
//   j in [0, strip+6)     padded row of a lane strip (3 halo rows each end)
//   k in [0, vl)          lane; lattice y = k*strip + (j - 3)
//
// pitch >= sy = strip + 6 and lead are chosen so that every column's first
// physical element (j = 3, k = 0, p = 0) starts a 256-byte segment: for the
// SoA-type layouts one warp of consecutive q = (j-3)*vl + k stores two whole
// 128-byte lines, for CAoSoA (vl = 32) every population cluster is one.
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
    int lvl;        // log2(vl)
    int tr;         // 1: y-major storage (storage column = lattice y, storage row = lattice x)
    int deep;       // 1: x-major SoA with 6 ghost rows per side (j = -3 .. strip+8; FUSED2 slab halos)
    long long lead;     // element offset of (p, X, j, k) = (0, 0, 0, 0)
    long long pstride;  // between populations of one site: plane (SoA/CSoA) or vl (AoS/CAoSoA)
    long long rstride;  // between padded rows j of a lane: vl (SoA/CSoA) or 37*vl (AoS/CAoSoA)
    long long cstride;  // between padded columns X: pitch * rstride
    // band-blocked store (layout D2Q37_BANDED, d2q37_banded.cu): band = 1; nbt
    // bands of kBandRows rows
    int band, nbt;
};

// Reference Descriptor::elem (layout.hpp:67-79) for all four layouts.
__host__ __device__ __forceinline__ long long elem_of(const DevGeo& g, int p, int X, int j, int k) {
    return g.lead + (long long)p * g.pstride + (long long)X * g.cstride + (long long)j * g.rstride + k;
}
// Population-0 element of the site at memory position q = (j-3)*vl + k of column X.
__host__ __device__ __forceinline__ long long site_of(const DevGeo& g, int X, int q) {
    return g.lead + (long long)X * g.cstride + (long long)(kHalo + (q >> g.lvl)) * g.rstride + (q & (g.vl - 1));
}

// Storage velocity components: y-major storage (g.tr) swaps the lattice axes.
template <bool TR>
__host__ __device__ __forceinline__ constexpr int scx(int p) { return TR ? cy_of(p) : cx_of(p); }
template <bool TR>
__host__ __device__ __forceinline__ constexpr int scy(int p) { return TR ? cx_of(p) : cy_of(p); }

// Index in a canonical population plane ((x*ly + y), dump.hpp:19-21) of the
// storage site (column xs, storage y ys = lane*strip + row).
__host__ __device__ __forceinline__ long long canon_index(const DevGeo& g, int xs, int ys) {
    return g.tr ? (long long)ys * g.lx + xs : (long long)xs * g.ly + ys;
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
    int o32[kNpop];  // o as 32-bit (valid when w32)
    int ps32;        // pstride as 32-bit (valid when w32)
    int w32;         // every o and 36 * pstride fit in int32: one IMAD.WIDE per address
    int canonical;   // o are the pull offsets of the geometry (no corrupt_population hook)
};

// Fills o32 / ps32 / w32 from o and pstride (call after every change of o).
inline void finish_offsets(Offsets& off, long long pstride, bool canonical) {
    off.canonical = canonical ? 1 : 0;
    const long long lim = 0x7fffffffLL;
    bool fits = 36 * pstride <= lim;
    for (int p = 0; p < kNpop; ++p) {
        fits = fits && off.o[p] <= lim && off.o[p] >= -lim;
        off.o32[p] = int(off.o[p]);
    }
    off.ps32 = int(pstride);
    off.w32 = fits ? 1 : 0;
}

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

// ---------------------------------------------------------------------------
// FAST collide with the sign symmetry of the velocity set.
//
// Hermite coefficient k has a definite parity in cx and in cy (model.cpp:
// 200-232), so for the four velocities (+-a, +-b) the table rows are the row
// of (a, b) with signs flipped on the odd terms, exactly.  Per quadruple the
// equilibrium sum splits into four partial sums over the parity classes
//   EE = {2,4,9,11,13}  OE = {0,5,7}  EO = {1,6,8}  OO = {3,10,12}
// and s(+-a, +-b) = EE +- OE +- EO + (sign) OO.  Axis velocities (a,0)/(0,b)
// pair the same way.  221 FP64 ops instead of 436 for the equilibrium sums;
// same result as the reference up to summation-order rounding (~1e-16).
// d2q37_set_model verifies the table has the exact symmetry this relies on.

D2Q37_HD constexpr int vel_index(int cx, int cy) {
    for (int p = 0; p < kNpop; ++p)
        if (cx_of(p) == cx && cy_of(p) == cy) return p;
    return -1;
}

template <int A, int B>
__device__ __forceinline__ void eq_quad(double (&f)[kNpop], const double* mom, const ModelParams& mp, double rho,
                                        double omega) {
    constexpr int ipp = vel_index(A, B), imp = vel_index(-A, B), ipm = vel_index(A, -B), imm = vel_index(-A, -B);
    const double* g = mp.eq[ipp];
    double ee = fma(g[2], mom[2], 1.0);
    ee = fma(g[4], mom[4], ee);
    ee = fma(g[9], mom[9], ee);
    ee = fma(g[11], mom[11], ee);
    ee = fma(g[13], mom[13], ee);
    double oe = g[0] * mom[0];
    oe = fma(g[5], mom[5], oe);
    oe = fma(g[7], mom[7], oe);
    double eo = g[1] * mom[1];
    eo = fma(g[6], mom[6], eo);
    eo = fma(g[8], mom[8], eo);
    double oo = g[3] * mom[3];
    oo = fma(g[10], mom[10], oo);
    oo = fma(g[12], mom[12], oo);
    const double P = ee + oo, Q = ee - oo, S = oe + eo, T = oe - eo;
    const double rw = rho * mp.w[ipp];
    f[ipp] = fma(omega, fma(rw, P + S, -f[ipp]), f[ipp]);
    f[imm] = fma(omega, fma(rw, P - S, -f[imm]), f[imm]);
    f[ipm] = fma(omega, fma(rw, Q + T, -f[ipm]), f[ipm]);
    f[imp] = fma(omega, fma(rw, Q - T, -f[imp]), f[imp]);
}

template <int A>
__device__ __forceinline__ void eq_axis(double (&f)[kNpop], const double* mom, const ModelParams& mp, double rho,
                                        double omega) {
    // x-axis pair (+-A, 0) and y-axis pair (0, +-A) share a shell weight.
    constexpr int xp = vel_index(A, 0), xm = vel_index(-A, 0), yp = vel_index(0, A), ym = vel_index(0, -A);
    const double rw = rho * mp.w[xp];
    {
        const double* g = mp.eq[xp];
        double ee = fma(g[2], mom[2], 1.0);
        ee = fma(g[4], mom[4], ee);
        ee = fma(g[9], mom[9], ee);
        ee = fma(g[11], mom[11], ee);
        ee = fma(g[13], mom[13], ee);
        double o = g[0] * mom[0];
        o = fma(g[5], mom[5], o);
        o = fma(g[7], mom[7], o);
        f[xp] = fma(omega, fma(rw, ee + o, -f[xp]), f[xp]);
        f[xm] = fma(omega, fma(rw, ee - o, -f[xm]), f[xm]);
    }
    {
        const double* g = mp.eq[yp];
        double ee = fma(g[2], mom[2], 1.0);
        ee = fma(g[4], mom[4], ee);
        ee = fma(g[9], mom[9], ee);
        ee = fma(g[11], mom[11], ee);
        ee = fma(g[13], mom[13], ee);
        double o = g[1] * mom[1];
        o = fma(g[6], mom[6], o);
        o = fma(g[8], mom[8], o);
        f[yp] = fma(omega, fma(rw, ee + o, -f[yp]), f[yp]);
        f[ym] = fma(omega, fma(rw, ee - o, -f[ym]), f[ym]);
    }
}

// collide_site_sym in two parts -- the moments (consume all 37 inputs) and the
// relaxation -- so a caller can issue independent work in between (k_step2
// issues the next column's loads there).
struct SymMoments {
    double rho;
    double mom[kNmom];
};

// Population halves of the FAST collide.  Half 0 ("A"): the rest velocity and
// the quadruples (+-1, +-1), (+-2, +-1), (+-1, +-2), (+-2, +-2) (17
// populations); half 1 ("B"): the three axis shells and the quadruples
// (+-3, +-1), (+-1, +-3) (20) -- about equal moment and relaxation work
// (65 / 68 and ~116 / ~129 FP64 operations).  Each half's relaxation is closed
// (eq_axis / eq_quad groups), so the two-threads-per-site sweep
// (d2q37_pair.cu) gives each thread of a pair one half; the moments are
// summed per half (canonical order inside a half) and the halves added A + B,
// the same order in every FAST kernel, so all of them stay bit-identical.
D2Q37_HD constexpr int pop_half(int p) {
    return (cx_of(p) == 0 && cy_of(p) == 0) ||
                   (cx_of(p) != 0 && cy_of(p) != 0 && cx_of(p) * cx_of(p) <= 4 && cy_of(p) * cy_of(p) <= 4)
               ? 0
               : 1;
}

// Partial moment sums {rho, jx, jy, e2} of half H, group by group: a quadruple
// (+-a, +-b) adds u1 - u2 (the cx = +a pair minus the cx = -a pair) to jx,
// v1 - v2 to jy and their total S to rho and (a^2 + b^2) S to e2 -- 11 FP64
// operations instead of 16 -- and an axis group (+-a, 0), (0, +-a) the same
// in 9 instead of 12; per site 94 instead of ~145.  Fixed group order per
// half: A = rest, (1,1), (2,1), (1,2), (2,2); B = axes 1, 2, 3, (3,1), (1,3).
template <int A, int B>
__device__ __forceinline__ void part_quad(const double (&f)[kNpop], double (&s)[4]) {
    constexpr int pp = vel_index(A, B), mp = vel_index(-A, B), pm = vel_index(A, -B), mm = vel_index(-A, -B);
    const double u1 = f[pp] + f[pm], u2 = f[mp] + f[mm];
    const double v1 = f[pp] + f[mp], v2 = f[pm] + f[mm];
    const double t = u1 + u2;
    s[0] += t;
    s[1] = fma(double(A), u1 - u2, s[1]);
    s[2] = fma(double(B), v1 - v2, s[2]);
    s[3] = fma(double(A * A + B * B), t, s[3]);
}
template <int A>
__device__ __forceinline__ void part_axis(const double (&f)[kNpop], double (&s)[4]) {
    constexpr int xp = vel_index(A, 0), xm = vel_index(-A, 0), yp = vel_index(0, A), ym = vel_index(0, -A);
    const double t = (f[xp] + f[xm]) + (f[yp] + f[ym]);
    s[0] += t;
    s[1] = fma(double(A), f[xp] - f[xm], s[1]);
    s[2] = fma(double(A), f[yp] - f[ym], s[2]);
    s[3] = fma(double(A * A), t, s[3]);
}
template <int H>
__device__ __forceinline__ void sym_partials(const double (&f)[kNpop], double (&s)[4]) {
    if (H == 0) {
        s[0] = f[0];
        s[1] = s[2] = s[3] = 0.0;
        part_quad<1, 1>(f, s);
        part_quad<2, 1>(f, s);
        part_quad<1, 2>(f, s);
        part_quad<2, 2>(f, s);
    } else {
        s[0] = s[1] = s[2] = s[3] = 0.0;
        part_axis<1>(f, s);
        part_axis<2>(f, s);
        part_axis<3>(f, s);
        part_quad<3, 1>(f, s);
        part_quad<1, 3>(f, s);
    }
}

// the Hermite moment vector from the summed {rho, jx, jy, e2} (half A + half B)
__device__ __forceinline__ bool sym_macros(const double (&a)[4], const double (&b)[4], const ModelParams& mp,
                                           SymMoments& m) {
    const double rho = a[0] + b[0];
    const bool bad = !(rho > 0.0);
    const double jx = a[1] + b[1], jy = a[2] + b[2], e2 = a[3] + b[3];
    const double inv_rho = 1.0 / rho;
    const double ux = jx * inv_rho;
    const double uy = jy * inv_rho;
    const double temp = 0.5 * (e2 * inv_rho - (ux * ux + uy * uy));
    const double dt = temp - mp.t0;
    const double ux2 = ux * ux, uy2 = uy * uy, uxuy = ux * uy;
    const double dt3 = 3.0 * dt, dt6 = 6.0 * dt, dt2 = dt * dt, dt2x3 = 3.0 * dt2;
    double* mom = m.mom;
    mom[0] = ux;
    mom[1] = uy;
    mom[2] = ux2 + dt;
    mom[3] = uxuy;
    mom[4] = uy2 + dt;
    mom[5] = ux * (ux2 + dt3);
    mom[6] = uy * (ux2 + dt);
    mom[7] = ux * (uy2 + dt);
    mom[8] = uy * (uy2 + dt3);
    mom[9] = ux2 * (ux2 + dt6) + dt2x3;
    mom[10] = uxuy * (ux2 + dt3);
    mom[11] = uxuy * uxuy + dt * (ux2 + uy2) + dt2;
    mom[12] = uxuy * (uy2 + dt3);
    mom[13] = uy2 * (uy2 + dt6) + dt2x3;
    m.rho = rho;
    return bad;
}

__device__ __forceinline__ bool sym_moments(const double (&f)[kNpop], const ModelParams& mp, SymMoments& m) {
    double a[4], b[4];
    sym_partials<0>(f, a);
    sym_partials<1>(f, b);
    return sym_macros(a, b, mp, m);
}

// relaxation of the populations of half H (sym_relax = both halves)
template <int H>
__device__ __forceinline__ void sym_relax_half(double (&f)[kNpop], const SymMoments& m, double omega,
                                               const ModelParams& mp) {
    const double* mom = m.mom;
    const double rho = m.rho;
    if (H == 0) {
        {  // rest velocity: even terms only
            const double* g = mp.eq[0];
            double ee = fma(g[2], mom[2], 1.0);
            ee = fma(g[4], mom[4], ee);
            ee = fma(g[9], mom[9], ee);
            ee = fma(g[11], mom[11], ee);
            ee = fma(g[13], mom[13], ee);
            f[0] = fma(omega, fma(rho * mp.w[0], ee, -f[0]), f[0]);
        }
        eq_quad<1, 1>(f, mom, mp, rho, omega);
        eq_quad<2, 1>(f, mom, mp, rho, omega);
        eq_quad<1, 2>(f, mom, mp, rho, omega);
        eq_quad<2, 2>(f, mom, mp, rho, omega);
    } else {
        eq_axis<1>(f, mom, mp, rho, omega);
        eq_axis<2>(f, mom, mp, rho, omega);
        eq_axis<3>(f, mom, mp, rho, omega);
        eq_quad<3, 1>(f, mom, mp, rho, omega);
        eq_quad<1, 3>(f, mom, mp, rho, omega);
    }
}

__device__ __forceinline__ void sym_relax(double (&f)[kNpop], const SymMoments& m, double omega,
                                          const ModelParams& mp) {
    sym_relax_half<0>(f, m, omega, mp);
    sym_relax_half<1>(f, m, omega, mp);
}

__device__ __forceinline__ bool collide_site_sym(double (&f)[kNpop], double omega, const ModelParams& mp) {
    SymMoments m;
    const bool bad = sym_moments(f, mp, m);
    sym_relax(f, m, omega, mp);
    return bad;
}

}  // namespace d2q37
