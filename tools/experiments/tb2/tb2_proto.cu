// tb2_proto.cu -- experiment: two D2Q37 time steps per HBM sweep (temporal blocking).
//
// Standalone timing/bit-exactness probe, not part of the library.  Lattice in
// the canonical population-major order (p*lx + x)*ly + y, periodic in x and y.
//
//   ref : one fused pull+collide step per launch (one thread per site), run twice
//   tb2 : persistent CTAs, each owning a band of W output rows (y) and marching
//         along x.  Step 1 (pull from HBM + collide) is computed on W+6 rows of
//         column r and kept in a shared-memory ring; step 2 for column r-3
//         pulls from the ring (lattice rows y-cy of columns r-3-cx) and is
//         written to HBM.  Population p of a step-1 column lives cx_p+3
//         iterations, so the ring holds sum_p (cx_p + 4) = 148 population
//         columns of W+6 doubles (222 KB at W+6 = 192).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I../../../include -I../../../paper_1804_01918_b200/csrc tb2_proto.cu \
//        -L../../../paper_1804_01918_b200/lib -ld2q37_b200 -o tb2_proto
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "d2q37_b200.h"
#include "d2q37_device.cuh"

using namespace d2q37;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ int wrap(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// Split-sum variant of collide_site_sym: the four moment sums run as 4 / 2
// interleaved partial chains (shorter FP64 dependency chains).
__device__ __forceinline__ bool collide_site_sym2(double (&f)[kNpop], double omega, const ModelParams& mp) {
    double r4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < kNpop; ++i) r4[i & 3] += f[i];
    const double rho = (r4[0] + r4[1]) + (r4[2] + r4[3]);
    const bool bad = !(rho > 0.0);
    double jx2[2] = {0.0, 0.0}, jy2[2] = {0.0, 0.0}, e22[2] = {0.0, 0.0};
    int kx = 0, ky = 0, ke = 0;
#pragma unroll
    for (int i = 0; i < kNpop; ++i) {
        if (cx_of(i) != 0) { jx2[kx & 1] = fma((double)cx_of(i), f[i], jx2[kx & 1]); ++kx; }
        if (cy_of(i) != 0) { jy2[ky & 1] = fma((double)cy_of(i), f[i], jy2[ky & 1]); ++ky; }
        if (cx_of(i) != 0 || cy_of(i) != 0) {
            e22[ke & 1] = fma((double)(cx_of(i) * cx_of(i) + cy_of(i) * cy_of(i)), f[i], e22[ke & 1]);
            ++ke;
        }
    }
    const double jx = jx2[0] + jx2[1], jy = jy2[0] + jy2[1], e2 = e22[0] + e22[1];
    const double inv_rho = 1.0 / rho;
    const double ux = jx * inv_rho;
    const double uy = jy * inv_rho;
    const double temp = 0.5 * (e2 * inv_rho - (ux * ux + uy * uy));
    const double dt = temp - mp.t0;
    const double ux2 = ux * ux, uy2 = uy * uy, uxuy = ux * uy;
    const double dt3 = 3.0 * dt, dt6 = 6.0 * dt, dt2 = dt * dt, dt2x3 = 3.0 * dt2;
    double mom[kNmom];
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
    {
        const double* g = mp.eq[0];
        double ee = fma(g[2], mom[2], 1.0);
        ee = fma(g[4], mom[4], ee);
        ee = fma(g[9], mom[9], ee);
        ee = fma(g[11], mom[11], ee);
        ee = fma(g[13], mom[13], ee);
        f[0] = fma(omega, fma(rho * mp.w[0], ee, -f[0]), f[0]);
    }
    eq_axis<1>(f, mom, mp, rho, omega);
    eq_axis<2>(f, mom, mp, rho, omega);
    eq_axis<3>(f, mom, mp, rho, omega);
    eq_quad<1, 1>(f, mom, mp, rho, omega);
    eq_quad<2, 1>(f, mom, mp, rho, omega);
    eq_quad<1, 2>(f, mom, mp, rho, omega);
    eq_quad<2, 2>(f, mom, mp, rho, omega);
    eq_quad<3, 1>(f, mom, mp, rho, omega);
    eq_quad<1, 3>(f, mom, mp, rho, omega);
    return bad;
}
#ifdef SPLIT
#define COLLIDE collide_site_sym2
#else
#define COLLIDE collide_site_sym
#endif

// ---- reference: one step per launch ------------------------------------------------
__global__ void __launch_bounds__(128, 4) k_ref(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                int ly, ModelParams mp, double omega) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x, x = blockIdx.y;
    if (y >= ly) return;
    const long long plane = (long long)lx * ly;
    double f[kNpop];
#pragma unroll
    for (int p = 0; p < kNpop; ++p)
        f[p] = __ldg(in + p * plane + (long long)wrap(x - cx_of(p), lx) * ly + wrap(y - cy_of(p), ly));
    COLLIDE(f, omega, mp);
    const long long e = (long long)x * ly + y;
#pragma unroll
    for (int p = 0; p < kNpop; ++p) __stcs(out + p * plane + e, f[p]);
}

// ---- two steps per sweep -------------------------------------------------------------
D2Q37_HD constexpr int depth_of(int p) { return cx_of(p) + 4; }
D2Q37_HD constexpr int ring_base(int p) {  // in units of population columns
    int s = 0;
    for (int q = 0; q < p; ++q) s += depth_of(q);
    return s;
}
constexpr int kRingCols = ring_base(kNpop);  // 148

// Compile-time loop over the 37 populations (keeps ring_base a constant).
template <typename F, int... Ps>
__device__ __forceinline__ void for_pops_(F&& f, std::integer_sequence<int, Ps...>) {
    (f(std::integral_constant<int, Ps>{}), ...);
}
template <typename F>
__device__ __forceinline__ void for_pops(F&& f) {
    for_pops_(f, std::make_integer_sequence<int, kNpop>{});
}

template <int T, int MINB, bool PF>
__global__ void __launch_bounds__(T, MINB) k_tb2(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                 int ly, ModelParams mp, double omega, int nbands, long long per_cta) {
    constexpr int W = T - 6;
    extern __shared__ double ring[];
    const int tid = threadIdx.x;
    const long long plane = (long long)lx * ly;
    const long long total = (long long)nbands * lx;
    long long item = (long long)blockIdx.x * per_cta;
    const long long item_end = min(total, item + per_cta);
    while (item < item_end) {
        const int band = (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * W;
        const int y1 = wrap(y0 - 3 + tid, ly);  // this thread's step-1 row (periodic)
        const int ny = min(W, ly - y0);          // output rows of this band
        int ys[7];
#pragma unroll
        for (int d = 0; d < 7; ++d) ys[d] = wrap(y1 - (d - 3), ly);  // y1 - cy for cy = d - 3
        const int niter = xe - xs + 6;
        double f[kNpop];
        auto load = [&](int r) {
#pragma unroll
            for (int p = 0; p < kNpop; ++p)
                f[p] = __ldg(in + p * plane + (long long)wrap(r - cx_of(p), lx) * ly + ys[cy_of(p) + 3]);
        };
        if (PF) load(xs - 3);
#pragma unroll 1
        for (int t = 0; t < niter; ++t) {
            const int r = xs - 3 + t;
            if (!PF) load(r);
            COLLIDE(f, omega, mp);
            for_pops([&](auto P) {
                constexpr int p = decltype(P)::value, rb = ring_base(p), dp = depth_of(p);
                ring[(rb + t % dp) * T + tid] = f[p];
            });
            __syncthreads();
            if (PF && t + 1 < niter) load(r + 1);
            if (t >= 6 && tid < ny) {
                double g[kNpop];
                for_pops([&](auto P) {
                    constexpr int p = decltype(P)::value, rb = ring_base(p), dp = depth_of(p);
                    g[p] = ring[(rb + (t + 1) % dp) * T + tid + 3 - cy_of(p)];
                });
                COLLIDE(g, omega, mp);
                const long long e = (long long)wrap(r - 3 + lx, lx) * ly + y0 + tid;
#pragma unroll
                for (int p = 0; p < kNpop; ++p) __stcs(out + p * plane + e, g[p]);
            }
            __syncthreads();
        }
    }
}

// Warp-specialised: NB producer threads compute step 1 of column r while NB
// consumer threads compute step 2 of column r-4 (one column behind), so each
// SMSP interleaves a load-bound and a compute-bound warp.  Ring depth cx+5.
D2Q37_HD constexpr int depth5_of(int p) { return cx_of(p) + 5; }
D2Q37_HD constexpr int ring5_base(int p) {
    int s = 0;
    for (int q = 0; q < p; ++q) s += depth5_of(q);
    return s;
}
constexpr int kRing5Cols = ring5_base(kNpop);  // 185

template <int NB, int PF>
__global__ void __launch_bounds__(2 * NB, 1) k_tb2ws(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                     int ly, ModelParams mp, double omega, int nbands,
                                                     long long per_cta) {
    constexpr int W = NB - 6;
    extern __shared__ double ring[];
    const bool prod = threadIdx.x < NB;
    const int tid = threadIdx.x & (NB - 1);
    const long long plane = (long long)lx * ly;
    const long long total = (long long)nbands * lx;
    long long item = (long long)blockIdx.x * per_cta;
    const long long item_end = min(total, item + per_cta);
    while (item < item_end) {
        const int band = (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * W;
        const int ny = min(W, ly - y0);
        const int niter = xe - xs + 7;
        if (prod) {
            const int y1 = wrap(y0 - 3 + tid, ly);
            int ys[7];
#pragma unroll
            for (int d = 0; d < 7; ++d) ys[d] = wrap(y1 - (d - 3), ly);
            double f[kNpop], fn[kNpop];
            auto load = [&](double(&v)[kNpop], int r) {
#pragma unroll
                for (int p = 0; p < kNpop; ++p)
                    v[p] = __ldg(in + p * plane + (long long)wrap(r - cx_of(p), lx) * ly + ys[cy_of(p) + 3]);
            };
            if (PF == 1) load(f, xs - 3);
            if (PF == 2) load(fn, xs - 3);
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t < niter - 1) {
                    const int r = xs - 3 + t;
                    if (PF == 0) load(f, r);
                    if (PF == 2) {
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) f[p] = fn[p];
                        if (t < niter - 2) load(fn, r + 1);
                    }
                    COLLIDE(f, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        ring[(rb + t % dp) * NB + tid] = f[p];
                    });
                    if (PF == 1 && t < niter - 2) load(f, r + 1);
                }
                __syncthreads();
            }
        } else {
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t >= 7 && tid < ny) {
                    double g[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        g[p] = ring[(rb + (t + 1) % dp) * NB + tid + 3 - cy_of(p)];
                    });
                    COLLIDE(g, omega, mp);
                    const long long e = (long long)(xs - 7 + t) * ly + y0 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(out + p * plane + e, g[p]);
                }
                __syncthreads();
            }
        }
    }
}

// v3: warp-specialised + register prefetch one column ahead (ping-pong, no
// copies) + interior addressing from per-population offsets in the constant
// bank (one 64-bit add per load/store); the x / y wrap only on edge columns /
// edge threads.
struct PullOffs {
    long long o[kNpop];  // p*plane - cx*ly - cy
    long long s[kNpop];  // p*plane
};

template <int NB, bool FA, bool PP, int PFD = 0>
__global__ void __launch_bounds__(2 * NB, 1) k_tb2v3(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                     int ly, ModelParams mp, PullOffs po, double omega, int nbands,
                                                     long long per_cta) {
    constexpr int W = NB - 6;
    extern __shared__ double ring[];
    const bool prod = threadIdx.x < NB;
    const int tid = threadIdx.x & (NB - 1);
    const long long plane = (long long)lx * ly;
    const long long total = (long long)nbands * lx;
    long long item = (long long)blockIdx.x * per_cta;
    const long long item_end = min(total, item + per_cta);
    while (item < item_end) {
        const int band = (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * W;
        const int ny = min(W, ly - y0);
        const int niter = xe - xs + 7;
        if (prod) {
            const int yraw = y0 - 3 + tid;
            const int y1 = wrap(yraw, ly);
            const bool yin = yraw >= 3 && yraw + 3 < ly;
            auto load = [&](double(&v)[kNpop], int r) {
                if (FA && yin && r >= 3 && r < lx - 3) {
                    const char* b = reinterpret_cast<const char*>(in + (long long)r * ly + yraw);
                    asm("" : "+l"(b));  // keep the per-load address a single 64-bit add
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) v[p] = __ldg(reinterpret_cast<const double*>(b + po.o[p]));
                } else {
#pragma unroll
                    for (int p = 0; p < kNpop; ++p)
                        v[p] = __ldg(in + p * plane + (long long)wrap(wrap(r, lx) - cx_of(p), lx) * ly +
                                     wrap(y1 - cy_of(p), ly));
                }
            };
            auto body = [&](double(&f)[kNpop], double(&fn)[kNpop], int t) {
                if (t < niter - 1) {
                    const int r = xs - 3 + t;
                    if (PFD > 0 && tid < kNpop && t + PFD < niter - 1) {
                        // L2 prefetch of population tid of step-1 input column r + PFD
                        const int cxp = cx_of(tid), cyp = cy_of(tid);
                        const int c = wrap(wrap(r + PFD, lx) - cxp, lx);
                        int ya = max(0, (y0 - 3 - cyp) & ~1);
                        int yb = min(ly, y0 + NB - 3 - cyp + 1);
                        const unsigned bytes = (unsigned)(((yb - ya) * 8 + 15) & ~15);
                        const double* a = in + tid * plane + (long long)c * ly + ya;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
                    }
                    if (t < niter - 2) load(fn, r + 1);
                    COLLIDE(f, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        ring[(rb + t % dp) * NB + tid] = f[p];
                    });
                }
                __syncthreads();
            };
            double fa[kNpop], fb[kNpop];
            load(fa, xs - 3);
            int t = 0;
            if (PP) {
#pragma unroll 1
                for (; t + 1 < niter; t += 2) {
                    body(fa, fb, t);
                    body(fb, fa, t + 1);
                }
                if (t < niter) body(fa, fb, t);
            } else {
#pragma unroll 1
                for (; t < niter; ++t) {
                    body(fa, fb, t);
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) fa[p] = fb[p];
                }
            }
        } else {
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t >= 7 && tid < ny) {
                    double g[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        g[p] = ring[(rb + (t + 1) % dp) * NB + tid + 3 - cy_of(p)];
                    });
                    COLLIDE(g, omega, mp);
                    const long long e = (long long)(xs - 7 + t) * ly + y0 + tid;
                    if (FA) {
                        double* o = out + e;
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) __stcs(o + po.s[p], g[p]);
                    } else {
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) __stcs(out + p * plane + e, g[p]);
                    }
                }
                __syncthreads();
            }
        }
    }
}

// v4: three warp groups.  L (loader) keeps two columns of step-1 inputs in
// flight in registers and writes the current one to a shared staging column;
// P (producer) collides it (step 1) into the ring; C (consumer) collides step
// 2 from the ring and stores to HBM.  Ring depth cx+5, staging 37*NB doubles.
__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int NB>
__global__ void __launch_bounds__(4 * NB, 1) k_tb2v4(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                     int ly, ModelParams mp, PullOffs po, double omega, int nbands,
                                                     long long per_cta) {
    constexpr int W = NB - 6;
    extern __shared__ double ring[];
    double* stage = ring + kRing5Cols * NB;
    const int grp = threadIdx.x / NB;  // 0, 1 loaders (even / odd rows), 2 producer, 3 consumer
    const int tid = threadIdx.x % NB;
    const long long plane = (long long)lx * ly;
    const long long total = (long long)nbands * lx;
    long long item = (long long)blockIdx.x * per_cta;
    const long long item_end = min(total, item + per_cta);
    while (item < item_end) {
        const int band = (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * W;
        const int ny = min(W, ly - y0);
        const int niter = xe - xs + 7;
        const int nprod = niter - 1;  // producer rows t = 0 .. nprod-1 (r = xs-3+t)
        if (grp < 2) {
            const int y1 = wrap(y0 - 3 + tid, ly);
            double v[kNpop];
            auto load = [&](int t) {
                const int r = xs - 3 + t;
#pragma unroll
                for (int p = 0; p < kNpop; ++p)
                    v[p] = __ldg(in + p * plane + (long long)wrap(wrap(r, lx) - cx_of(p), lx) * ly +
                                 wrap(y1 - cy_of(p), ly));
            };
            if (grp < nprod) load(grp);
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if ((t & 1) == grp) {
                    if (t < nprod) {
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) stage[p * NB + tid] = v[p];
                    }
                    bar_named(1, 2 * NB);
                    if (t + 2 < nprod) load(t + 2);
                }
                __syncthreads();
            }
        } else if (grp == 2) {
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                bar_named(1, 2 * NB);
                if (t < nprod) {
                    double f[kNpop];
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) f[p] = stage[p * NB + tid];
                    COLLIDE(f, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        ring[(rb + t % dp) * NB + tid] = f[p];
                    });
                }
                __syncthreads();
            }
        } else {
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t >= 7 && tid < ny) {
                    double g[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        g[p] = ring[(rb + (t + 1) % dp) * NB + tid + 3 - cy_of(p)];
                    });
                    COLLIDE(g, omega, mp);
                    double* o = out + (long long)(xs - 7 + t) * ly + y0 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + po.s[p], g[p]);
                }
                __syncthreads();
            }
        }
    }
}

// v5: producer collides step 1 from a shared staging column (no global
// loads); the consumer, idle ~40 % in v3, loads the step-1 inputs one column
// ahead in registers and writes them to staging besides doing step 2.
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int NB>
__global__ void __launch_bounds__(2 * NB, 1) k_tb2v5(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                     int ly, ModelParams mp, PullOffs po, double omega, int nbands,
                                                     long long per_cta) {
    constexpr int W = NB - 6;
    extern __shared__ double ring[];
    double* stage = ring + kRing5Cols * NB;
    const bool prod = threadIdx.x < NB;
    const int tid = threadIdx.x & (NB - 1);
    const long long plane = (long long)lx * ly;
    const long long total = (long long)nbands * lx;
    long long item = (long long)blockIdx.x * per_cta;
    const long long item_end = min(total, item + per_cta);
    while (item < item_end) {
        const int band = (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * W;
        const int ny = min(W, ly - y0);
        const int niter = xe - xs + 7;
        const int nprod = niter - 1;
        if (prod) {
            __syncthreads();
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                double f[kNpop];
                if (t < nprod) {
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) f[p] = stage[p * NB + tid];
                }
                bar_arrive(1, 2 * NB);
                if (t < nprod) {
                    COLLIDE(f, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        ring[(rb + t % dp) * NB + tid] = f[p];
                    });
                }
                __syncthreads();
            }
        } else {
            const int y1 = wrap(y0 - 3 + tid, ly);
            double h[kNpop];
            auto load = [&](int t) {
                const int r = xs - 3 + t;
#pragma unroll
                for (int p = 0; p < kNpop; ++p)
                    h[p] = __ldg(in + p * plane + (long long)wrap(wrap(r, lx) - cx_of(p), lx) * ly +
                                 wrap(y1 - cy_of(p), ly));
            };
            auto put = [&]() {
#pragma unroll
                for (int p = 0; p < kNpop; ++p) stage[p * NB + tid] = h[p];
            };
            load(0);
            put();
            if (1 < nprod) load(1);
            __syncthreads();
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                bar_named(1, 2 * NB);
                if (t + 1 < nprod) {
                    put();
                    if (t + 2 < nprod) load(t + 2);
                }
                if (t >= 7 && tid < ny) {
                    double g[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        g[p] = ring[(rb + (t + 1) % dp) * NB + tid + 3 - cy_of(p)];
                    });
                    COLLIDE(g, omega, mp);
                    double* o = out + (long long)(xs - 7 + t) * ly + y0 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + po.s[p], g[p]);
                }
                __syncthreads();
            }
        }
    }
}

// v6: the step-1 loads are split -- the producer prefetches populations
// [0, KS) into registers one column ahead, the consumer loads [KS, 37) one
// column ahead and hands them over through a shared staging column.
template <int NB, int KS>
__global__ void __launch_bounds__(2 * NB, 1) k_tb2v6(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                     int ly, ModelParams mp, PullOffs po, double omega, int nbands,
                                                     long long per_cta) {
    constexpr int W = NB - 6;
    constexpr int NS = kNpop - KS;
    extern __shared__ double ring[];
    double* stage = ring + kRing5Cols * NB;  // NS populations x NB
    const bool prod = threadIdx.x < NB;
    const int tid = threadIdx.x & (NB - 1);
    const long long plane = (long long)lx * ly;
    const long long total = (long long)nbands * lx;
    long long item = (long long)blockIdx.x * per_cta;
    const long long item_end = min(total, item + per_cta);
    while (item < item_end) {
        const int band = (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * W;
        const int ny = min(W, ly - y0);
        const int niter = xe - xs + 7;
        const int nprod = niter - 1;
        const int y1 = wrap(y0 - 3 + tid, ly);
        auto ldp = [&](int p, int t) {
            const int r = xs - 3 + t;
            return __ldg(in + p * plane + (long long)wrap(wrap(r, lx) - cx_of(p), lx) * ly + wrap(y1 - cy_of(p), ly));
        };
        if (prod) {
            double fa[KS], fb[KS];
#pragma unroll
            for (int p = 0; p < KS; ++p) fa[p] = ldp(p, 0);
            __syncthreads();
            auto body = [&](double(&cur)[KS], double(&nxt)[KS], int t) {
                double f[kNpop];
                if (t < nprod) {
#pragma unroll
                    for (int p = KS; p < kNpop; ++p) f[p] = stage[(p - KS) * NB + tid];
                }
                bar_arrive(1, 2 * NB);
                if (t < nprod) {
                    if (t + 1 < nprod) {
#pragma unroll
                        for (int p = 0; p < KS; ++p) nxt[p] = ldp(p, t + 1);
                    }
#pragma unroll
                    for (int p = 0; p < KS; ++p) f[p] = cur[p];
                    COLLIDE(f, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        ring[(rb + t % dp) * NB + tid] = f[p];
                    });
                }
                __syncthreads();
            };
            int t = 0;
#pragma unroll 1
            for (; t + 1 < niter; t += 2) {
                body(fa, fb, t);
                body(fb, fa, t + 1);
            }
            if (t < niter) body(fa, fb, t);
        } else {
            double h[NS];
            auto load = [&](int t) {
#pragma unroll
                for (int p = KS; p < kNpop; ++p) h[p - KS] = ldp(p, t);
            };
            auto put = [&]() {
#pragma unroll
                for (int p = 0; p < NS; ++p) stage[p * NB + tid] = h[p];
            };
            load(0);
            put();
            if (1 < nprod) load(1);
            __syncthreads();
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                bar_named(1, 2 * NB);
                if (t + 1 < nprod) {
                    put();
                    if (t + 2 < nprod) load(t + 2);
                }
                if (t >= 7 && tid < ny) {
                    double g[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = ring5_base(p), dp = depth5_of(p);
                        g[p] = ring[(rb + (t + 1) % dp) * NB + tid + 3 - cy_of(p)];
                    });
                    COLLIDE(g, omega, mp);
                    double* o = out + (long long)(xs - 7 + t) * ly + y0 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + po.s[p], g[p]);
                }
                __syncthreads();
            }
        }
    }
}

__global__ void k_cmp(const double* a, const double* b, long long n, unsigned long long* nd) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += __double_as_longlong(a[i]) != __double_as_longlong(b[i]);
    if (c) atomicAdd(nd, c);
}

__global__ void k_init(double* f, long long n, unsigned long long seed, const double* w, long long plane) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const double u = (z >> 11) * 0x1.0p-53;
        f[i] = w[i / plane] * (1.0 + 0.02 * (u - 0.5));
    }
}

int main(int argc, char** argv) {
    const int lx = argc > 1 ? atoi(argv[1]) : 4096;
    const int ly = argc > 2 ? atoi(argv[2]) : 16384;
    const int reps = argc > 3 ? atoi(argv[3]) : 10;
    const double omega = 0.8;
    constexpr int T = 192;
    d2q37_model m;
    if (d2q37_model_d2q37(&m) != 0) return 1;
    ModelParams mp{};
    for (int i = 0; i < kNpop; ++i) {
        for (int k = 0; k < kNmom; ++k) mp.eq[i][k] = m.eq[i * kNmom + k];
        mp.w[i] = m.w[i];
    }
    mp.t0 = m.t0;
    const long long plane = (long long)lx * ly, n = plane * kNpop;
    double *a, *b, *c, *d, *w;
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&b, n * 8));
    CK(cudaMalloc(&c, n * 8));
    CK(cudaMalloc(&d, n * 8));
    CK(cudaMalloc(&w, kNpop * 8));
    CK(cudaMemcpy(w, m.w, kNpop * 8, cudaMemcpyHostToDevice));
    k_init<<<4096, 256>>>(a, n, 12345, w, plane);
    CK(cudaGetLastError());

    PullOffs po;
    for (int p = 0; p < kNpop; ++p) {
        po.o[p] = 8 * (p * plane - (long long)cx_of(p) * ly - cy_of(p));
        po.s[p] = p * plane;
    }
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    unsigned long long* nd;
    CK(cudaMalloc(&nd, 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](const char* name, auto&& fn, double sweeps) {
        for (int i = 0; i < 2; ++i) fn();
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) fn();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double per2 = ms / reps;
        printf("%-14s %8.3f ms per 2 steps = %8.1f MLUPS, %7.1f GB/s (592 B/site per sweep)\n", name, per2,
               2.0 * plane / (per2 * 1e3), sweeps * plane * 592.0 / (per2 * 1e6));
    };
    dim3 rg((ly + 127) / 128, lx);
    auto ref2 = [&]() {
        k_ref<<<rg, 128>>>(a, b, lx, ly, mp, omega);
        k_ref<<<rg, 128>>>(b, c, lx, ly, mp, omega);
    };
    ref2();
    CK(cudaDeviceSynchronize());
    if (argc <= 5) timeit("ref", ref2, 2.0);
    int bad = 0;
    auto run = [&](auto kern, int T, int minb, const char* name, int ws = 0) {
        const size_t smem = (size_t)(ws ? kRing5Cols + (ws == 6 || ws == 7 ? kNpop : ws == 8 ? kNpop - 18 : ws == 9 ? kNpop - 24 : 0) : kRingCols) * T * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int W = T - 6;
        const int nbands = (ly + W - 1) / W;
        const long long total = (long long)nbands * lx;
        const int grid = nsm * minb;
        const long long per_cta = (total + grid - 1) / grid;
        auto fn = [&]() {
            if (ws == 3)
                k_tb2v3<128, true, true><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 4)
                k_tb2v3<128, false, true><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 6)
                k_tb2v4<128><<<grid, T * 4, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 7)
                k_tb2v5<128><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 8)
                k_tb2v6<128, 18><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 9)
                k_tb2v6<128, 24><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 10)
                k_tb2v3<128, false, true, 2><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 11)
                k_tb2v3<128, false, true, 3><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 12)
                k_tb2v3<128, false, true, 5><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else if (ws == 5)
                k_tb2v3<128, true, false><<<grid, T * 2, smem>>>(a, d, lx, ly, mp, po, omega, nbands, per_cta);
            else
                kern<<<grid, T * (ws ? 2 : 1), smem>>>(a, d, lx, ly, mp, omega, nbands, per_cta);
        };
        CK(cudaMemset(d, 0, n * 8));
        CK(cudaMemset(nd, 0, 8));
        fn();
        CK(cudaGetLastError());
        k_cmp<<<4096, 256>>>(c, d, n, nd);
        unsigned long long h = 0;
        CK(cudaMemcpy(&h, nd, 8, cudaMemcpyDeviceToHost));
        printf("%-14s T=%d W=%d bands=%d smem=%zu grid=%d items/cta=%lld  bit-exact: %s (%llu diff)\n", name, T, W,
               nbands, smem, grid, per_cta, h ? "NO" : "yes", h);
        bad |= h != 0;
        if (argc <= 5) timeit(name, fn, 1.0);
    };
    const char* only = argc > 4 ? argv[4] : "";
    auto want = [&](const char* nm) { return !*only || !strcmp(only, nm); };
    if (want("t192")) run(k_tb2<192, 1, false>, 192, 1, "t192");
    if (want("t192pf")) run(k_tb2<192, 1, true>, 192, 1, "t192pf");
    if (want("t96x2")) run(k_tb2<96, 2, false>, 96, 2, "t96x2");
    if (want("t96x2pf")) run(k_tb2<96, 2, true>, 96, 2, "t96x2pf");
    if (want("t128pf")) run(k_tb2<128, 1, true>, 128, 1, "t128pf");
    if (want("ws128")) run(k_tb2ws<128, 0>, 128, 1, "ws128", 1);
    if (want("ws128pf")) run(k_tb2ws<128, 1>, 128, 1, "ws128pf", 1);
    if (want("ws128pf2")) run(k_tb2ws<128, 2>, 128, 1, "ws128pf2", 1);
    CK(cudaFuncSetAttribute(k_tb2v3<128, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing5Cols * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v3<128, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing5Cols * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v3<128, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing5Cols * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v4<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (kRing5Cols + kNpop) * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v5<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (kRing5Cols + kNpop) * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v6<128, 18>, cudaFuncAttributeMaxDynamicSharedMemorySize, (kRing5Cols + kNpop) * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v6<128, 24>, cudaFuncAttributeMaxDynamicSharedMemorySize, (kRing5Cols + kNpop) * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v3<128, false, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing5Cols * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v3<128, false, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing5Cols * 128 * 8));
    CK(cudaFuncSetAttribute(k_tb2v3<128, false, true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing5Cols * 128 * 8));
    if (want("pf2")) run(k_tb2ws<128, 2>, 128, 1, "pfd2", 10);
    if (want("pf3")) run(k_tb2ws<128, 2>, 128, 1, "pfd3", 11);
    if (want("pf5")) run(k_tb2ws<128, 2>, 128, 1, "pfd5", 12);
    if (want("v6")) run(k_tb2ws<128, 2>, 128, 1, "v6", 8);
    if (want("v6b")) run(k_tb2ws<128, 2>, 128, 1, "v6b", 9);
    if (want("v5")) run(k_tb2ws<128, 2>, 128, 1, "v5", 7);
    if (want("v4")) run(k_tb2ws<128, 2>, 128, 1, "v4", 6);
    if (want("v3")) run(k_tb2ws<128, 2>, 128, 1, "v3", 3);
    if (want("v3pp")) run(k_tb2ws<128, 2>, 128, 1, "v3pp", 4);
    if (want("v3fa")) run(k_tb2ws<128, 2>, 128, 1, "v3fa", 5);
    return bad ? 2 : 0;
}
