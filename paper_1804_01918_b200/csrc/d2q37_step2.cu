// d2q37_step2.cu -- two D2Q37 time steps per HBM sweep (temporal blocking, FUSED2).
//
// The single-step kernel (k_collide<.., SHIFT>) moves the algorithmic 592 B per
// site and step at ~105 % of the measured copy bandwidth, so past it a step
// has to cost fewer HBM bytes.  A FUSED2 sweep reads the state once and writes
// the state two steps later: 592 B per site per TWO steps.
//
// Storage: SoA (layout.hpp:74-75, vl = 1, x-major), the padded buffer of the
// other kernels; physical sites only are read and written, the boundary is
// resolved in the kernel (x periodic; y periodic, specular wall, or -- on a
// y-slab -- the 6 deep ghost rows per face that k_pack6 / NCCL / k_unpack6
// fill before every sweep).
//
// Schedule (persistent CTAs, one per SM):
//   * the lattice is cut into bands of kT2Out = 122 rows; a CTA walks a
//     contiguous range of (band, column) items in band-major order, marching
//     along x;
//   * producer warps (threads 0-127) compute step 1 -- the pull of
//     kernels.cpp:50-63 from HBM plus collide, model.cpp:293-298 -- for the 128
//     rows y0-3 .. y0+124 of column r and park the result in a shared-memory
//     ring; the next column's 37 loads are issued before this column's
//     collide (register double buffer);
//   * consumer warps (threads 128-255) compute step 2 for the 122 rows of
//     column r-4, pulling every population from the ring, and stream it to
//     HBM;
//   * population p of a step-1 column is read by step 2 of column r + cx_p,
//     i.e. it lives cx_p + 4 iterations (+1: producer and consumer run
//     concurrently), so the ring holds sum_p (cx_p + 5) = 185 population
//     columns of 128 doubles = 185 KB.
// Two code forms of that schedule: sweep_plain (per-population index
// arithmetic; every band of a periodic lattice, bands away from a wall, slab
// ghost faces) and sweep_general (per-thread row tables; wall bands and
// degenerate extents).  k_step2_split runs both in one launch, on disjoint CTA
// groups.  Every site is updated with the same gathered values and the same
// collide_site_sym as the single-step kernel, so a sweep is bit for bit two
// steps of k_collide<FAST, SHIFT> (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <utility>

#include "d2q37_device.cuh"
#include "d2q37_fused2.cuh"
#include "d2q37_kernels.cuh"

namespace d2q37 {


// Plain sweep: bands whose pulls stay inside the lattice rows (or any band
// of a y-periodic lattice), lx >= 3.  Every address is per-population index
// arithmetic with a one-step wrap; this form measured ~9 % faster than the
// table-driven general form.
// WRAPY: y-periodic lattice (rows wrap); otherwise rows are read unwrapped --
// inside [0, ly) for bands away from the faces, and down to -6 / up to ly+5
// (the deep ghost rows a slab's halo exchange fills) at ghost faces.
template <bool WRAPY, class Sched>
__device__ __forceinline__ void sweep_plain(const double* __restrict__ src, double* __restrict__ dst, const DevGeo& g,
                                            const ModelParams& mp, double omega, Sched sched,
                                            int* __restrict__ flag, double* __restrict__ send_lo = nullptr,
                                            double* __restrict__ send_hi = nullptr) {
    extern __shared__ double ring[];
    const bool prod = threadIdx.x < kT2Band;
    const int tid = threadIdx.x & (kT2Band - 1);
    const int lx = g.lx, ly = g.ly;
    const double* __restrict__ sb = src + g.lead + kHalo * g.cstride + kHalo;
    double* __restrict__ db = dst + g.lead + kHalo * g.cstride + kHalo;
    const long long plane = g.pstride, cs = g.cstride;
    auto wr = [](int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); };
    bool bad = false;
    int band, xs, xe;
    while (sched.next(band, xs, xe)) {
        const int y0 = band * kT2Out;
        const int ny = min(kT2Out, ly - y0);
        const int niter = xe - xs + 7;  // producer rows t = 0 .. niter-2, consumer t = 7 .. niter-1
        if (prod) {
            // step-1 row of this thread (rows past ly + 2 of the last band are never read)
            const int y1 = WRAPY ? wrap_mod(y0 - kHalo + tid, ly) : min(y0 - kHalo + tid, ly + kHalo - 1);
            auto load = [&](double(&v)[kNpop], int r) {
#pragma unroll
                for (int p = 0; p < kNpop; ++p)
                    v[p] = __ldg(sb + p * plane + (long long)wr(wr(r, lx) - cx_of(p), lx) * cs +
                                 (WRAPY ? wr(y1 - cy_of(p), ly) : y1 - cy_of(p)));
            };
            // the next column's loads issue before this column's collide (register double buffer)
            auto body = [&](double(&f)[kNpop], double(&fn)[kNpop], int t) {
                if (t < niter - 1) {
                    const int r = xs - kHalo + t;
                    if (t < niter - 2) load(fn, r + 1);
                    bad |= collide_site_sym(f, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2_base(p), dp = t2_depth(p);
                        ring[(rb + t % dp) * kT2Band + tid] = f[p];
                    });
                }
                __syncthreads();
            };
            double fa[kNpop], fb[kNpop];
            load(fa, xs - kHalo);
            int t = 0;
#pragma unroll 1
            for (; t + 1 < niter; t += 2) {
                body(fa, fb, t);
                body(fb, fa, t + 1);
            }
            if (t < niter) body(fa, fb, t);
        } else {
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t >= 7 && tid < ny) {
                    double v[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2_base(p), dp = t2_depth(p);
                        v[p] = ring[(rb + (t + 1) % dp) * kT2Band + tid + kHalo - cy_of(p)];
                    });
                    bad |= collide_site_sym(v, omega, mp);
                    const long long e = (long long)(xs - 7 + t) * cs + y0 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(db + p * plane + e, v[p]);
                    // fused pack of a slab's 6-row halos ([p][x][6], the k_pack6 layout)
                    const int y = y0 + tid;
                    if (send_lo && y < 2 * kHalo) {
                        double* __restrict__ sl = send_lo + (long long)(xs - 7 + t) * (2 * kHalo) + y;
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) sl[(long long)p * lx * (2 * kHalo)] = v[p];
                    }
                    if (send_hi && y >= ly - 2 * kHalo) {
                        double* __restrict__ sh = send_hi + (long long)(xs - 7 + t) * (2 * kHalo) + y - (ly - 2 * kHalo);
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) sh[(long long)p * lx * (2 * kHalo)] = v[p];
                    }
                }
                __syncthreads();
            }
        }
    }
    if (bad) atomicOr(flag, 1);
}

// Bulk-copy sweep: the plain form's schedule with the producer's 37 pulls of
// a column staged in shared memory by the copy engine instead of per-thread
// loads.  After the producers have consumed column r's stage (its moments
// need all 37 values), the four producer warps issue the 37 one-dimensional
// bulk copies of column r + 1 (cp.async.bulk, 1040 B each: rows y0-3-cy_p ..
// y0+124-cy_p of source column r - cx_p, 16-byte aligned) into the single
// stage, completion counted on one mbarrier; the copies are in flight during
// column r's relaxation, ring stores and barrier.  No per-thread address
// arithmetic, no register double buffer, no L1 for the pulls.
// Rows are read unwrapped: bands whose pull rows y0-6 .. y0+127 lie inside
// the stored rows (the lattice, or the deep ghost rows of a slab face).
// GHOST: the band may reach a slab ghost face; step-1 rows past ly + 2 are
// never read, so those threads collide row ly + 2 (finite) instead.
template <bool GHOST, bool EARLY>
__device__ __forceinline__ void sweep_tma(const double* __restrict__ src, double* __restrict__ dst, const DevGeo& g,
                                          const ModelParams& mp, double omega, int band0, int nbands,
                                          long long item_begin, long long item_end_, int* __restrict__ flag) {
    extern __shared__ double ring[];
    double* stage = ring + kT2RingCols * kT2Band;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(stage + kNpop * kStageRows);
    const bool prod = threadIdx.x < kT2Band;
    const int tid = threadIdx.x & (kT2Band - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = g.lx, ly = g.ly;
    const double* __restrict__ sb = src + g.lead + kHalo * g.cstride + kHalo;
    double* __restrict__ db = dst + g.lead + kHalo * g.cstride + kHalo;
    const long long plane = g.pstride, cs = g.cstride;
    const long long total = (long long)nbands * lx;
    long long item = item_begin;
    const long long item_end = min(total, item_end_);
    auto wr = [](int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); };
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // copy issue: producer warp w, lane l < 10 -> population 10 w + l
    const int ip = warp * 10 + lane;
    const bool issuer = prod && lane < 10 && ip < kNpop;
    const int icx = issuer ? c_cx[ip] : 0, icy = issuer ? c_cy[ip] : 0;
    double* const idst = stage + (issuer ? ip : 0) * kStageRows;
    unsigned phase = 0;
    bool bad = false;
    while (item < item_end) {
        const int band = band0 + (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * kT2Out;
        const int ny = min(kT2Out, ly - y0);
        const int niter = xe - xs + 7;  // producer rows t = 0 .. niter-2, consumer t = 7 .. niter-1
        if (prod) {
            const double* const isrc = sb + ip * plane + ((y0 - kHalo - icy) & ~1);
            auto issue = [&](int r) {
                if (issuer) {
                    const int col = wr(wr(r, lx) - icx, lx);
                    bulk_g2s(idst, isrc + (long long)col * cs, kStageRows * sizeof(double), full);
                }
                if (threadIdx.x == 0) mbar_arrive_expect_tx(full, kStageBytes);
            };
            if (issuer || threadIdx.x == 0) issue(xs - kHalo);
            // stage offset of this thread's step-1 row (y1 - cy_p - row0_p = yo + ((y0-3-cy_p) & 1))
            const int yo = GHOST ? min(tid, ly + kHalo - 1 - (y0 - kHalo)) : tid;
            const int par = (y0 - kHalo) & 1;
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t < niter - 1) {
                    mbar_wait(full, phase);
                    phase ^= 1;
                    double f[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value;
                        f[p] = stage[p * kStageRows + yo + (par ^ (cy_of(p) & 1))];
                    });
                    if (EARLY) {
                        // the 37 values are in registers (an empty asm consumes them): refill the stage now
#pragma unroll
                        for (int p = 0; p < kNpop; p += 6)
                            asm volatile("" ::"d"(f[p]), "d"(f[min(p + 1, kNpop - 1)]), "d"(f[min(p + 2, kNpop - 1)]),
                                         "d"(f[min(p + 3, kNpop - 1)]), "d"(f[min(p + 4, kNpop - 1)]),
                                         "d"(f[min(p + 5, kNpop - 1)]));
                        if (t < niter - 2) {
                            prod_bar_sync();
                            issue(xs - kHalo + t + 1);
                        }
                    }
                    SymMoments m;
                    bad |= sym_moments(f, mp, m);
                    // every producer has its 37 values (the moments consumed them): refill the stage
                    if (!EARLY && t < niter - 2) {
                        prod_bar_sync();
                        issue(xs - kHalo + t + 1);
                    }
                    sym_relax(f, m, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2_base(p), dp = t2_depth(p);
                        ring[(rb + t % dp) * kT2Band + tid] = f[p];
                    });
                }
                __syncthreads();
            }
        } else {
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t >= 7 && tid < ny) {
                    double v[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2_base(p), dp = t2_depth(p);
                        v[p] = ring[(rb + (t + 1) % dp) * kT2Band + tid + kHalo - cy_of(p)];
                    });
                    bad |= collide_site_sym(v, omega, mp);
                    const long long e = (long long)(xs - 7 + t) * cs + y0 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(db + p * plane + e, v[p]);
                }
                __syncthreads();
            }
        }
    }
    if (bad) atomicOr(flag, 1);
}

// Two-stage bulk-copy sweep (form kStep2Bulk2): the bulk-copy staging of
// sweep_tma with TWO stages in flight -- column r + 2 is copied while column r
// is collided and column r + 1 is landing -- which fits beside a 148-column
// ring (t2n_depth: cx_p + 4) because producers and consumers hand the ring
// over with named barriers instead of __syncthreads: the consumers read an
// iteration's slots first (barrier 2 -> the producers may overwrite them),
// the producers publish a step-1 column with barrier 3.  Stages: 2 x 38.5 KB;
// ring 148 KB; 228.5 KB of shared memory.  Rows are read unwrapped (as
// sweep_tma).  Bit-identical to the other forms (same gathered values, same
// collide_site_sym).
template <bool GHOST, class Sched>
__device__ __forceinline__ void sweep_tma2(const double* __restrict__ src, double* __restrict__ dst, const DevGeo& g,
                                           const ModelParams& mp, double omega, Sched sched,
                                           int* __restrict__ flag) {
    extern __shared__ double ring[];
    double* const stage0 = ring + kT2NRingCols * kT2Band;  // 2 stages [37][130]
    unsigned long long* const full = reinterpret_cast<unsigned long long*>(stage0 + 2 * kNpop * kStageRows);
    const bool prod = threadIdx.x < kT2Band;
    const int tid = threadIdx.x & (kT2Band - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = g.lx, ly = g.ly;
    const double* __restrict__ sb = src + g.lead + kHalo * g.cstride + kHalo;
    double* __restrict__ db = dst + g.lead + kHalo * g.cstride + kHalo;
    const long long plane = g.pstride, cs = g.cstride;
    auto wr = [](int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); };
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        mbar_init(full + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // copy issue: producer warp w, lane l < 10 -> population 10 w + l
    const int ip = warp * 10 + lane;
    const bool issuer = prod && lane < 10 && ip < kNpop;
    const int icx = issuer ? c_cx[ip] : 0, icy = issuer ? c_cy[ip] : 0;
    unsigned issued = 0, used = 0;  // stage columns issued / consumed (stage = n & 1)
    bool bad = false;
    int band, xs, xe;
    while (sched.next(band, xs, xe)) {
        const int y0 = band * kT2Out;
        const int ny = min(kT2Out, ly - y0);
        const int niter = xe - xs + 7;  // producer columns xs-3 .. xe+2 at t = 0 .. niter-2; outputs at t >= 7
        if (prod) {
            const double* const isrc = sb + ip * plane + ((y0 - kHalo - icy) & ~1);
            auto issue = [&](int r) {
                const unsigned st = issued & 1u;
                if (issuer) {
                    const int col = wr(wr(r, lx) - icx, lx);
                    bulk_g2s(stage0 + (st * kNpop + ip) * kStageRows, isrc + (long long)col * cs,
                             kStageRows * sizeof(double), full + st);
                }
                if (threadIdx.x == 0) mbar_arrive_expect_tx(full + st, kStageBytes);
                ++issued;
            };
            for (int k = 0; k < 2 && k < niter - 1; ++k) issue(xs - kHalo + k);
            // stage offset of this thread's step-1 row (y1 - cy_p - row0_p = yo + ((y0-3-cy_p) & 1))
            const int yo = GHOST ? min(tid, ly + kHalo - 1 - (y0 - kHalo)) : tid;
            const int par = (y0 - kHalo) & 1;
#pragma unroll 1
            for (int t = 0; t < niter - 1; ++t) {
                const unsigned st = used & 1u;
                mbar_wait(full + st, (used >> 1) & 1u);
                ++used;
                const double* const sg = stage0 + st * kNpop * kStageRows;
                double f[kNpop];
                for_pops([&](auto P) {
                    constexpr int p = decltype(P)::value;
                    f[p] = sg[p * kStageRows + yo + (par ^ (cy_of(p) & 1))];
                });
                // the 37 values are in registers (an empty asm consumes them): the stage is free
#pragma unroll
                for (int p = 0; p < kNpop; p += 6)
                    asm volatile("" ::"d"(f[p]), "d"(f[min(p + 1, kNpop - 1)]), "d"(f[min(p + 2, kNpop - 1)]),
                                 "d"(f[min(p + 3, kNpop - 1)]), "d"(f[min(p + 4, kNpop - 1)]),
                                 "d"(f[min(p + 5, kNpop - 1)]));
                bad |= collide_site_sym(f, omega, mp);
                // the consumers have read this iteration's slots -- and every producer has read the
                // stage (before its collide): refill it with column t + 2
                nbar_sync(2);
                if (t + 2 < niter - 1) issue(xs - kHalo + t + 2);
                for_pops([&](auto P) {
                    constexpr int p = decltype(P)::value, rb = t2n_base(p), dp = t2n_depth(p);
                    ring[(rb + t % dp) * kT2Band + tid] = f[p];
                });
                nbar_arrive(3);
            }
            nbar_sync(2);  // the consumers' last iteration
        } else {
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t > 0) nbar_sync(3);  // step-1 column t - 1 is in the ring
                const bool work = t >= 7 && tid < ny;
                double v[kNpop];
                if (work) {  // column c - cx_p, produced at t - 4 - cx_p: slot t % depth
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2n_base(p), dp = t2n_depth(p);
                        v[p] = ring[(rb + t % dp) * kT2Band + tid + kHalo - cy_of(p)];
                    });
#pragma unroll
                    for (int p = 0; p < kNpop; p += 6)
                        asm volatile("" ::"d"(v[p]), "d"(v[min(p + 1, kNpop - 1)]), "d"(v[min(p + 2, kNpop - 1)]),
                                     "d"(v[min(p + 3, kNpop - 1)]), "d"(v[min(p + 4, kNpop - 1)]),
                                     "d"(v[min(p + 5, kNpop - 1)]));
                }
                nbar_arrive(2);
                if (work) {
                    bad |= collide_site_sym(v, omega, mp);
                    const long long e = (long long)(xs - 7 + t) * cs + y0 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(db + p * plane + e, v[p]);
                }
            }
        }
    }
    if (bad) atomicOr(flag, 1);
}

// General sweep: any band, every face kind (periodic wrap, wall image, slab
// ghost rows) through per-thread row tables.  Launched on the face bands only
// (k_step2_plain covers the rest).
__device__ __forceinline__ void sweep_general(const double* __restrict__ src, double* __restrict__ dst,
                                              const DevGeo& g, const Faces& fc, const ModelParams& mp, double omega,
                                              int band0, int nbands, long long item_begin, long long item_end_,
                                              int* __restrict__ flag, double* __restrict__ send_lo = nullptr,
                                              double* __restrict__ send_hi = nullptr) {
    extern __shared__ double ring[];
    const bool prod = threadIdx.x < kT2Band;
    const int tid = threadIdx.x & (kT2Band - 1);
    const int lx = g.lx, ly = g.ly;
    const bool wall_lo = fc.lo == kFaceWall, wall_hi = fc.hi == kFaceWall;
    // ghost faces (y-slabs): rows -6..-1 / ly..ly+5 hold the neighbours' rows (k_unpack6)
    const bool ghost_lo = fc.lo == kFaceGhost, ghost_hi = fc.hi == kFaceGhost;
    // element of (p = 0, x = 0, y = 0); site (x, y) of population p at + p*plane + x*cs + y
    const double* __restrict__ sb = src + g.lead + kHalo * g.cstride + kHalo;
    double* __restrict__ db = dst + g.lead + kHalo * g.cstride + kHalo;
    const long long plane = g.pstride, cs = g.cstride;
    const long long total = (long long)nbands * lx;
    long long item = item_begin;
    const long long item_end = min(total, item_end_);
    bool bad = false;
    while (item < item_end) {
        const int band = band0 + (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * kT2Out;
        const int ny = min(kT2Out, ly - y0);
        const int niter = xe - xs + 7;  // producer rows t = 0 .. niter-2, consumer t = 7 .. niter-1
        if (prod) {
            // Step-1 row of this thread: y0 - 3 + tid, periodic image; beyond a
            // wall the value is never read (step 2 mirrors into the lattice).
            const int yr = y0 - kHalo + tid;
            int y1;
            if (yr >= 0 && yr < ly)
                y1 = yr;
            else if ((yr < 0 && wall_lo) || (yr >= ly && wall_hi))
                y1 = min(max(yr, 0), ly - 1);
            else if (yr < 0 && ghost_lo)
                y1 = yr;  // >= -3: its pulls reach row -6
            else if (yr >= ly && ghost_hi)
                y1 = min(yr, ly + kHalo - 1);  // rows past ly + 2 are never read
            else
                y1 = wrap_mod(yr, ly);
            // pull row of y1 - cy (k = cy + 3) and whether it is a wall image
            // (then population ybar(p) is read: specular reflection)
            int yo[2 * kHalo + 1];
            unsigned mirm = 0;
#pragma unroll
            for (int k = 0; k < 2 * kHalo + 1; ++k) {
                int ys = y1 - (k - kHalo);
                const bool m = (ys < 0 && wall_lo) || (ys >= ly && wall_hi);
                if (m)
                    ys = ys < 0 ? -1 - ys : 2 * ly - 1 - ys;
                else if (!((ys < 0 && ghost_lo) || (ys >= ly && ghost_hi)))
                    ys = wrap_mod(ys, ly);
                mirm |= unsigned(m) << k;
                yo[k] = ys;
            }
            auto load = [&](double(&v)[kNpop], int r) {
                const int rw = wrap_mod(r, lx);
                int col[2 * kHalo + 1];  // element offset of source column cx = k - 3 (< 2^31: one plane)
#pragma unroll
                for (int k = 0; k < 2 * kHalo + 1; ++k) col[k] = wrap_mod(rw - (k - kHalo), lx) * int(cs);
#pragma unroll
                for (int p = 0; p < kNpop; ++p) {
                    const int k = cy_of(p) + kHalo;
                    const int pp = (mirm >> k) & 1u ? ybar_of(p) : p;
                    v[p] = __ldg(sb + pp * plane + (col[cx_of(p) + kHalo] + yo[k]));
                }
            };
            auto body = [&](double(&f)[kNpop], double(&fn)[kNpop], int t) {
                if (t < niter - 1) {
                    const int r = xs - kHalo + t;
                    // moments first (they consume all 37 loads of this column), then
                    // the next column's loads, then the relaxation: the loads stay
                    // in flight for the relaxation, the ring stores and the barrier
                    SymMoments m;
                    bad |= sym_moments(f, mp, m);
                    asm volatile("" ::"d"(m.rho), "d"(m.mom[0]), "d"(m.mom[13]) : "memory");
                    if (t < niter - 2) load(fn, r + 1);
                    sym_relax(f, m, omega, mp);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2_base(p), dp = t2_depth(p);
                        ring[(rb + t % dp) * kT2Band + tid] = f[p];
                    });
                }
                __syncthreads();
            };
            double fa[kNpop], fb[kNpop];
            load(fa, xs - kHalo);
            int t = 0;
#pragma unroll 1
            for (; t + 1 < niter; t += 2) {
                body(fa, fb, t);
                body(fb, fa, t + 1);
            }
            if (t < niter) body(fa, fb, t);
        } else {
            const int y = y0 + tid;
            const bool active = tid < ny;
            // ring position of y - cy (k = cy + 3) and whether it is a wall image
            int pos[2 * kHalo + 1];
            unsigned mirm = 0;
#pragma unroll
            for (int k = 0; k < 2 * kHalo + 1; ++k) {
                int ys = y - (k - kHalo);
                const bool m = (ys < 0 && wall_lo) || (ys >= ly && wall_hi);
                if (m) ys = ys < 0 ? -1 - ys : 2 * ly - 1 - ys;
                mirm |= unsigned(m) << k;
                pos[k] = ys - (y0 - kHalo);
            }
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t >= 7 && active) {
                    double v[kNpop];
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, dp = t2_depth(p);
                        constexpr int k = cy_of(p) + kHalo, rb = t2_base(p), rbb = t2_base(ybar_of(p));
                        const int base = (mirm >> k) & 1u ? rbb : rb;
                        v[p] = ring[(base + (t + 1) % dp) * kT2Band + pos[k]];
                    });
                    bad |= collide_site_sym(v, omega, mp);
                    double* __restrict__ o = db + (long long)(xs - 7 + t) * cs + y;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + p * plane, v[p]);
                    // fused pack of a slab's 6-row halos ([p][x][6], the k_pack6 layout)
                    if (send_lo && y < 2 * kHalo) {
                        double* __restrict__ sl = send_lo + (long long)(xs - 7 + t) * (2 * kHalo) + y;
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) sl[(long long)p * lx * (2 * kHalo)] = v[p];
                    }
                    if (send_hi && y >= ly - 2 * kHalo) {
                        double* __restrict__ sh = send_hi + (long long)(xs - 7 + t) * (2 * kHalo) + y - (ly - 2 * kHalo);
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) sh[(long long)p * lx * (2 * kHalo)] = v[p];
                    }
                }
                __syncthreads();
            }
        }
    }
    if (bad) atomicOr(flag, 1);
}

template <bool WRAPY>
__global__ void __launch_bounds__(2 * kT2Band, 1)
    k_step2_plain(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, ModelParams mp, double omega,
                  int band0, int nbands, long long per_cta, int* __restrict__ flag) {
    sweep_plain<WRAPY>(src, dst, g, mp, omega, RangeSched(band0, nbands, g.lx, blockIdx.x * per_cta, (blockIdx.x + 1) * per_cta),
                       flag);
}

__global__ void __launch_bounds__(2 * kT2Band, 1)
    k_step2(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, Faces fc, ModelParams mp,
            double omega, int band0, int nbands, long long per_cta, int* __restrict__ flag) {
    sweep_general(src, dst, g, fc, mp, omega, band0, nbands, blockIdx.x * per_cta, (blockIdx.x + 1) * per_cta, flag);
}

// One launch, three CTA groups: the interior bands (plain form, or the
// bulk-copy form) beside the low and high face bands (general form); every
// CTA runs one form throughout, so an SM's instruction cache holds one loop.
struct Step2Split {
    int band0[3], nb[3], ctas[3];
    long long per_cta[3];
    int form;  // interior bands: 0 = sweep_plain, 1 = sweep_tma
    int lock;  // interior bands of the plain form: the lockstep schedule (LockSched)
    Lockstep ls;
};

__global__ void __launch_bounds__(2 * kT2Band, 1)
    k_step2_split(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, Faces fc, ModelParams mp,
                  double omega, Step2Split sp, int* __restrict__ flag) {
    int cta = blockIdx.x;
    if (cta < sp.ctas[0]) {
        if (sp.form == kStep2Bulk2) {
            const PartSched ps{sp.lock != 0,
                               RangeSched(sp.band0[0], sp.nb[0], g.lx, cta * sp.per_cta[0], (cta + 1) * sp.per_cta[0]),
                               LockSched(sp.band0[0], g.lx, sp.ctas[0], cta, sp.ls)};
            if (fc.hi == kFaceGhost)
                sweep_tma2<true>(src, dst, g, mp, omega, ps, flag);
            else
                sweep_tma2<false>(src, dst, g, mp, omega, ps, flag);
        } else if (sp.form == kStep2Bulk) {
            if (fc.hi == kFaceGhost)
                sweep_tma<true, false>(src, dst, g, mp, omega, sp.band0[0], sp.nb[0], cta * sp.per_cta[0], (cta + 1) * sp.per_cta[0], flag);
            else
                sweep_tma<false, false>(src, dst, g, mp, omega, sp.band0[0], sp.nb[0], cta * sp.per_cta[0], (cta + 1) * sp.per_cta[0], flag);
        } else if (sp.form == kStep2BulkEarly) {
            if (fc.hi == kFaceGhost)
                sweep_tma<true, true>(src, dst, g, mp, omega, sp.band0[0], sp.nb[0], cta * sp.per_cta[0], (cta + 1) * sp.per_cta[0], flag);
            else
                sweep_tma<false, true>(src, dst, g, mp, omega, sp.band0[0], sp.nb[0], cta * sp.per_cta[0], (cta + 1) * sp.per_cta[0], flag);
        } else {
            const PartSched ps{sp.lock != 0,
                               RangeSched(sp.band0[0], sp.nb[0], g.lx, cta * sp.per_cta[0], (cta + 1) * sp.per_cta[0]),
                               LockSched(sp.band0[0], g.lx, sp.ctas[0], cta, sp.ls)};
            if (fc.lo == kFacePeriodic && fc.hi == kFacePeriodic)
                sweep_plain<true>(src, dst, g, mp, omega, ps, flag);
            else
                sweep_plain<false>(src, dst, g, mp, omega, ps, flag);
        }
        return;
    }
    cta -= sp.ctas[0];
    const int part = cta < sp.ctas[1] ? 1 : 2;
    if (part == 2) cta -= sp.ctas[1];
    sweep_general(src, dst, g, fc, mp, omega, sp.band0[part], sp.nb[part], cta * sp.per_cta[part],
                  (cta + 1) * sp.per_cta[part], flag);
}

// One overlapped sweep of a FUSED2 y-slab (k_step2_slab): the first nf_lo +
// nf_hi CTAs sweep the face bands first -- the bands whose pulls reach the
// ghost rows or a wall -- writing the slab's 6 edge rows of the new state into
// the send buffers as they go (fused pack), then bump the sweep counter; every
// CTA then sweeps its share of the interior bands.  The host queues the halo
// exchange on the comm stream behind a stream wait on that counter, so the
// exchange runs while the interior is being swept.
constexpr int kSlabMaxCtas = 256;
struct SlabPlan {
    int nf_lo, nf_hi;  // CTAs [0, nf_lo): the low face bands; [nf_lo, nf_lo + nf_hi): the high ones
    int lo_band0, lo_nb, hi_band0, hi_nb, in_band0, in_nb;
    long long lo_per, hi_per;
    long long in_off[kSlabMaxCtas + 1];  // interior items of CTA c: [in_off[c], in_off[c + 1])
};

__global__ void __launch_bounds__(2 * kT2Band, 1)
    k_step2_slab(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, Faces fc, ModelParams mp,
                 double omega, SlabPlan sp, int* __restrict__ flag, unsigned* __restrict__ counter,
                 double* __restrict__ send_lo, double* __restrict__ send_hi) {
    const int cta = blockIdx.x;
    if (cta < sp.nf_lo + sp.nf_hi) {
        const bool lo = cta < sp.nf_lo;
        const long long c = lo ? cta : cta - sp.nf_lo, per = lo ? sp.lo_per : sp.hi_per;
        const int b0 = lo ? sp.lo_band0 : sp.hi_band0, nb = lo ? sp.lo_nb : sp.hi_nb;
        if ((lo ? fc.lo : fc.hi) == kFaceWall)  // a global wall: the general form mirrors
            sweep_general(src, dst, g, fc, mp, omega, b0, nb, c * per, (c + 1) * per, flag, send_lo, send_hi);
        else  // ghost rows: read unwrapped by the plain form
            sweep_plain<false>(src, dst, g, mp, omega, RangeSched(b0, nb, g.lx, c * per, (c + 1) * per), flag, send_lo,
                               send_hi);
        __syncthreads();  // every consumer's face rows (lattice and send buffers) are stored
        if (threadIdx.x == 0) {
            __threadfence_system();
            atomicAdd(counter, 1u);
        }
    }
    if (sp.in_off[cta] < sp.in_off[cta + 1])
        sweep_plain<false>(src, dst, g, mp, omega, RangeSched(sp.in_band0, sp.in_nb, g.lx, sp.in_off[cta], sp.in_off[cta + 1]),
                           flag);
}

// 6-row slab halos of FUSED2: rows 0..5 / ly-6..ly-1 of every physical column
// and population -> send buffers [p][x][6]; received buffers -> ghost rows
// -6..-1 / ly..ly+5 (a null buffer skips that face).
__global__ void __launch_bounds__(256) k_pack6(const double* __restrict__ buf, DevGeo g, double* __restrict__ send_lo,
                                               double* __restrict__ send_hi) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = int(i % (2 * kHalo));
    const long long px = i / (2 * kHalo);
    const int x = int(px % g.lx), p = int(px / g.lx);
    const long long base = elem_of(g, p, x + kHalo, kHalo, 0);  // row y = 0
    if (send_lo) send_lo[i] = buf[base + r];
    if (send_hi) send_hi[i] = buf[base + g.ly - 2 * kHalo + r];
}

__global__ void __launch_bounds__(256) k_unpack6(double* __restrict__ buf, DevGeo g, const double* __restrict__ recv_lo,
                                                 const double* __restrict__ recv_hi) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = int(i % (2 * kHalo));
    const long long px = i / (2 * kHalo);
    const int x = int(px % g.lx), p = int(px / g.lx);
    const long long base = elem_of(g, p, x + kHalo, kHalo, 0);  // row y = 0
    if (recv_lo) buf[base - 2 * kHalo + r] = recv_lo[i];  // rows -6 .. -1
    if (recv_hi) buf[base + g.ly + r] = recv_hi[i];       // rows ly .. ly+5
}

// Periodic images in the deep ghost rows of a y-periodic single domain: rows -6..-1 <- ly-6..ly-1 and
// ly..ly+5 <- 0..5 of every physical column and population (the pair form then sweeps it like a 1-rank
// slab ring, every band in one launch).
__global__ void __launch_bounds__(256) k_wrap6(double* __restrict__ buf, DevGeo g) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = int(i % (2 * kHalo));
    const long long px = i / (2 * kHalo);
    const int x = int(px % g.lx), p = int(px / g.lx);
    double* const col = buf + elem_of(g, p, x + kHalo, kHalo, 0);  // row y = 0
    col[r - 2 * kHalo] = col[g.ly - 2 * kHalo + r];
    col[g.ly + r] = col[r];
}

// Specular-wall images in the deep ghost rows: population p at ghost row -1-r holds ybar(p)
// = (cx, -cy) at row r, at row ly+r holds ybar(p) at row ly-1-r (r = 0..5).  An unwrapped pull into
// them is then the wall's mirrored pull, and the sweep's step-1 values on the ghost rows come out as
// the mirror images of rows 0..2 / ly-3..ly-1 (the FAST collide is exactly reflection-equivariant:
// the pair-sum moments flip jy by an exact subtraction, the sign-symmetric equilibrium swaps P +- S /
// Q +- T), so a wall sweep needs no mirror tables.
__global__ void __launch_bounds__(256) k_mirror6(double* __restrict__ buf, DevGeo g, Faces fc, int mask) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = int(i % (2 * kHalo));
    const long long px = i / (2 * kHalo);
    const int x = int(px % g.lx), p = int(px / g.lx);
    double* const col = buf + elem_of(g, p, x + kHalo, kHalo, 0);  // row y = 0 of population p
    const double* const img = buf + elem_of(g, fc.ybar[p], x + kHalo, kHalo, 0);
    if (mask & 1) col[-1 - r] = img[r];
    if (mask & 2) col[g.ly + r] = img[g.ly - 1 - r];
}

cudaError_t launch_mirror6(double* buf, const DevGeo& g, const Faces& fc, cudaStream_t s, int mask) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    k_mirror6<<<unsigned((n + 255) / 256), 256, 0, s>>>(buf, g, fc, mask);
    return cudaGetLastError();
}

cudaError_t launch_wrap6(double* buf, const DevGeo& g, cudaStream_t s) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    k_wrap6<<<unsigned((n + 255) / 256), 256, 0, s>>>(buf, g);
    return cudaGetLastError();
}

size_t halo6_count(const DevGeo& g) { return size_t(kNpop) * g.lx * 2 * kHalo; }

cudaError_t launch_pack6(const double* buf, const DevGeo& g, double* send_lo, double* send_hi, cudaStream_t s) {
    if (g.band) return launch_band_pack6(buf, g, send_lo, send_hi, s);
    const long long n = (long long)halo6_count(g);
    k_pack6<<<unsigned((n + 255) / 256), 256, 0, s>>>(buf, g, send_lo, send_hi);
    return cudaGetLastError();
}

cudaError_t launch_unpack6(double* buf, const DevGeo& g, const double* recv_lo, const double* recv_hi,
                           cudaStream_t s) {
    if (g.band) return launch_band_unpack6(buf, g, recv_lo, recv_hi, s);
    const long long n = (long long)halo6_count(g);
    k_unpack6<<<unsigned((n + 255) / 256), 256, 0, s>>>(buf, g, recv_lo, recv_hi);
    return cudaGetLastError();
}

bool step2_supported(const DevGeo& g, const Faces& fc) {
    if (g.band) return fc.col_lo == kFacePeriodic && fc.col_hi == kFacePeriodic;  // every y face kind
    auto ok = [&](int f) { return f == kFacePeriodic || f == kFaceWall || (f == kFaceGhost && g.deep); };
    const bool face_ok = ok(fc.lo) && ok(fc.hi) && (fc.lo != kFaceGhost && fc.hi != kFaceGhost ? true : g.ly >= 2 * kHalo);
    return g.vl == 1 && !g.tr && g.pstride != g.vl && face_ok && fc.col_lo == kFacePeriodic &&
           fc.col_hi == kFacePeriodic && g.lx >= 1 && g.ly >= kHalo &&
           (long long)(g.lx + 2 * kHalo) * g.cstride < 0x7fffffffLL;  // 32-bit offsets inside a plane
}

size_t step2_smem_bytes(int form) {
    const size_t ring = (size_t)kT2RingCols * kT2Band * sizeof(double);
    if (form == kStep2Bulk2)  // 148-column ring + two stages and their mbarriers
        return (size_t)kT2NRingCols * kT2Band * sizeof(double) + 2 * size_t(kStageBytes) + 16;
    return form != kStep2Plain ? ring + kStageBytes + 16 : ring;  // + the stage and its mbarrier
}

namespace {
int g_form = -1;  // interior-band form of every FUSED2 sweep (step2_form)
}  // namespace

int step2_band_rows() { return kT2Out; }

int step2_form() {
    if (g_form < 0) {
        const char* v = std::getenv("D2Q37_STEP2_FORM");
        g_form = v && *v ? std::min(4, std::max(0, std::atoi(v))) : kStep2Pair;  // measured fastest (DESIGN 3.1)
    }
    return g_form;
}

int set_step2_form(int form) {
    const int prev = step2_form();
    g_form = std::min(4, std::max(0, form));
    return prev;
}

namespace {
int g_sched = -1;  // interior schedule of the plain form: 0 = band-major ranges, 1 = lockstep
}  // namespace

int step2_sched() {
    if (g_sched < 0) {
        const char* v = std::getenv("D2Q37_STEP2_SCHED");
        g_sched = v && *v ? (std::atoi(v) != 0) : 1;
    }
    return g_sched;
}

int set_step2_sched(int sched) {
    const int prev = step2_sched();
    g_sched = sched != 0;
    return prev;
}

// Single-domain walls through wall images in the deep ghost rows (k_mirror6, the sweep reads them like a
// ghost face): D2Q37_STEP2_GHOST_WALLS=0 turns it off (then the mirror tables below, or the side launch).
bool step2_ghost_walls() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("D2Q37_STEP2_GHOST_WALLS");
        v = !(e && *e == '0');
    }
    return v != 0;
}

// Single-domain wall bands in the pair form itself (mirror tables, one launch per sweep) or, with
// D2Q37_STEP2_PAIR_WALLS=0, in a general-form launch beside it.  Measured with the mirror tables:
// 4096 x 4096 +8.7 %, 4096 x 8192 +16 %, 4096 x 16384 within run-to-run noise (DESIGN 3.1.1).
bool step2_pair_walls() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("D2Q37_STEP2_PAIR_WALLS");
        v = !(e && *e == '0');
    }
    return v != 0;
}

namespace {
int g_face_pct = -1;  // 0: the form's default
}  // namespace

int step2_face_pct() {
    if (g_face_pct < 0) {
        const char* v = std::getenv("D2Q37_STEP2_FACE_PCT");
        g_face_pct = v ? std::max(0, std::atoi(v)) : 0;
    }
    return g_face_pct > 0 ? g_face_pct : (step2_form() != kStep2Plain ? 135 : 115);
}

void set_step2_face_pct(int pct) { g_face_pct = std::max(0, pct); }

namespace {
// Band split of one sweep: plain bands [b_lo, b_hi) -- every pull row (y0 - 6 ..
// y0 + 127) inside the stored rows [0, ly) (or, at a slab ghost face, the deep
// ghost rows), or with the per-thread form any band of a y-periodic lattice --
// and the face bands [0, b_lo) / [b_hi, nbands), which take the general kernel.
// The bulk-copy form reads rows unwrapped, so the wrapping first and last bands
// of a y-periodic lattice are face bands for it.
void step2_bands(const DevGeo& g, const Faces& fc, int form, int* nbands, int* b_lo, int* b_hi) {
    *nbands = (g.ly + kT2Out - 1) / kT2Out;
    const bool per_lo = fc.lo == kFacePeriodic, per_hi = fc.hi == kFacePeriodic;
    int lo = 0, hi = *nbands;
    const int inside_hi = g.ly >= kT2Band ? (g.ly - kT2Band) / kT2Out + 1 : 0;  // bands with rows < ly
    if (per_lo && per_hi) {
        if (form != kStep2Plain) lo = 1, hi = inside_hi;  // the bulk-copy forms read rows unwrapped
    } else if (form == kStep2Pair && !per_lo && !per_hi && g.ly >= kT2Band &&
               ((fc.lo != kFaceWall && fc.hi != kFaceWall) || step2_pair_walls())) {
        // the pair form reads ghost faces' deep ghost rows unwrapped and mirrors at walls: every band is
        // interior
    } else {
        // ghost faces read the deep ghost rows unwrapped; wall bands need the general form
        lo = fc.lo == kFaceWall ? 1 : 0;
        hi = fc.hi == kFaceWall ? inside_hi : *nbands;
        if (per_lo != per_hi) lo = 0, hi = 0;  // one periodic face with a wall / ghost one: all general
    }
    hi = std::min(hi, *nbands);
    if (g.lx < kHalo || hi <= lo) lo = hi = 0;  // degenerate: every band general
    *b_lo = lo;
    *b_hi = hi;
}

void part_range(const DevGeo& g, const Faces& fc, int form, int part, int* band0, int* nb) {
    int nbands, b_lo, b_hi;
    step2_bands(g, fc, form, &nbands, &b_lo, &b_hi);
    *band0 = part == 0 ? b_lo : part == 1 ? 0 : part == 2 ? b_hi : 0;
    *nb = part == 0 ? b_hi - b_lo : part == 1 ? b_lo : part == 2 ? nbands - b_hi : nbands;
}

// per-device SM count, set once with the kernels' shared-memory attributes
int device_nsm(cudaError_t* err) {
    constexpr int kMaxDev = 64;
    static int nsm_of[kMaxDev] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    int nsm = (e == cudaSuccess && dev < kMaxDev) ? nsm_of[dev] : 0;
    if (e == cudaSuccess && nsm == 0) {
        e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int ring = (int)step2_smem_bytes(kStep2Plain),
                  bulk = (int)std::max(step2_smem_bytes(kStep2Bulk), step2_smem_bytes(kStep2Bulk2));
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k_step2, cudaFuncAttributeMaxDynamicSharedMemorySize, ring);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_step2_plain<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ring);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_step2_plain<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ring);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_step2_split, cudaFuncAttributeMaxDynamicSharedMemorySize, bulk);
        if (e == cudaSuccess && dev < kMaxDev) nsm_of[dev] = nsm;
    }
    *err = e;
    return e == cudaSuccess ? nsm : 0;
}
}  // namespace

long long step2_items(const DevGeo& g, const Faces& fc, int part) {
    int band0, nb;
    part_range(g, fc, step2_form(), part, &band0, &nb);
    return (long long)nb * g.lx;
}

cudaError_t launch_step2(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                         double omega, int* flag, cudaStream_t s, int part, int max_ctas) {
    cudaError_t e;
    const int nsm = device_nsm(&e);
    if (e != cudaSuccess) return e;
    int band0, nb;
    part_range(g, fc, kStep2Plain, part, &band0, &nb);
    if (nb <= 0) return cudaSuccess;
    const long long total = (long long)nb * g.lx;
    const int grid = (int)std::min<long long>(max_ctas > 0 ? std::min(max_ctas, nsm) : nsm, total);
    const long long per_cta = (total + grid - 1) / grid;
    const size_t smem = step2_smem_bytes(kStep2Plain);
    if (part == 0 && fc.lo == kFacePeriodic && fc.hi == kFacePeriodic)
        k_step2_plain<true><<<grid, 2 * kT2Band, smem, s>>>(src, dst, g, mp, omega, band0, nb, per_cta, flag);
    else if (part == 0)
        k_step2_plain<false><<<grid, 2 * kT2Band, smem, s>>>(src, dst, g, mp, omega, band0, nb, per_cta, flag);
    else
        k_step2<<<grid, 2 * kT2Band, smem, s>>>(src, dst, g, fc, mp, omega, band0, nb, per_cta, flag);
    return cudaGetLastError();
}

void step2_interior_bands(const DevGeo& g, int* nbands, int* b_lo, int* b_hi) {
    interior_bands(g.lx, g.ly, nbands, b_lo, b_hi);
}

cudaError_t launch_step2_parts(const double* src, double* dst, const DevGeo& g, const Faces& fc,
                               const ModelParams& mp, double omega, int* flag, cudaStream_t s, const int band0[3],
                               const int nb[3], const int ctas[3]) {
    cudaError_t e;
    device_nsm(&e);
    if (e != cudaSuccess) return e;
    Step2Split sp{};
    sp.form = kStep2Plain;  // part 0 reads rows unwrapped (slab interiors): the per-thread form
    int grid = 0;
    for (int part = 0; part < 3; ++part) {
        sp.band0[part] = band0[part];
        sp.nb[part] = nb[part];
        const long long total = (long long)std::max(0, nb[part]) * g.lx;
        sp.ctas[part] = total > 0 ? (int)std::min<long long>(ctas[part], total) : 0;
        if (total > 0 && sp.ctas[part] < 1) return cudaErrorInvalidValue;
        sp.per_cta[part] = sp.ctas[part] ? (total + sp.ctas[part] - 1) / sp.ctas[part] : 0;
        grid += sp.ctas[part];
    }
    if (grid == 0) return cudaSuccess;
    if (nb[0] > 0 && fc.lo == kFacePeriodic && fc.hi == kFacePeriodic) return cudaErrorInvalidValue;  // nowrap only
    k_step2_split<<<grid, 2 * kT2Band, step2_smem_bytes(sp.form), s>>>(src, dst, g, fc, mp, omega, sp, flag);
    return cudaGetLastError();
}

int launch_step2_slab(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                      double omega, int* flag, cudaStream_t s, int grid, unsigned* counter, double* send_lo,
                      double* send_hi, cudaError_t* err) {
    *err = cudaSuccess;
    int nbands, b_lo, b_hi;
    step2_interior_bands(g, &nbands, &b_lo, &b_hi);
    if (b_hi - b_lo < 1 || grid < 8 || grid > kSlabMaxCtas || fc.lo == kFacePeriodic || fc.hi == kFacePeriodic)
        return 0;  // no overlapped form: the caller runs the serial schedule
    static bool attr[64] = {};
    *err = once_per_device(attr, [] {
        return cudaFuncSetAttribute(k_step2_slab, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)step2_smem_bytes(kStep2Plain));
    });
    if (*err != cudaSuccess) return 0;
    SlabPlan sp{};
    sp.lo_band0 = 0;
    sp.lo_nb = b_lo;
    sp.hi_band0 = b_hi;
    sp.hi_nb = nbands - b_hi;
    sp.in_band0 = b_lo;
    sp.in_nb = b_hi - b_lo;
    // cost per item relative to the plain interior form: the general form at a wall
    const double cfl = fc.lo == kFaceWall ? step2_face_pct() / 100.0 : 1.0;
    const double cfh = fc.hi == kFaceWall ? step2_face_pct() / 100.0 : 1.0;
    const double lo_items = double(sp.lo_nb) * g.lx, hi_items = double(sp.hi_nb) * g.lx;
    const long long in_items = (long long)sp.in_nb * g.lx;
    const double per = (cfl * lo_items + cfh * hi_items + double(in_items)) / grid;  // work per CTA
    // face CTAs: enough that a face share is at most half of a CTA's work (the exchange then has
    // the other half of the sweep to hide under)
    auto nface = [&](double items, double cf) {
        if (items <= 0) return 0;
        return std::max(1, std::min(grid / 4, int(std::ceil(2.0 * cf * items / per))));
    };
    sp.nf_lo = nface(lo_items, cfl);
    sp.nf_hi = nface(hi_items, cfh);
    sp.lo_per = sp.nf_lo ? (long long)std::ceil(lo_items / sp.nf_lo) : 0;
    sp.hi_per = sp.nf_hi ? (long long)std::ceil(hi_items / sp.nf_hi) : 0;
    // interior shares: what is left of each CTA's work, scaled to the interior items
    std::vector<double> share(grid);
    double tot = 0.0;
    for (int c = 0; c < grid; ++c) {
        double face = 0.0;
        if (c < sp.nf_lo) face = cfl * std::min<double>(sp.lo_per, std::max(0.0, lo_items - double(c) * sp.lo_per));
        else if (c < sp.nf_lo + sp.nf_hi)
            face = cfh * std::min<double>(sp.hi_per, std::max(0.0, hi_items - double(c - sp.nf_lo) * sp.hi_per));
        share[c] = std::max(0.0, per - face);
        tot += share[c];
    }
    double acc = 0.0;
    sp.in_off[0] = 0;
    for (int c = 0; c < grid; ++c) {
        acc += share[c];
        sp.in_off[c + 1] = c + 1 == grid ? in_items : std::min<long long>(in_items, llround(acc / tot * in_items));
    }
    k_step2_slab<<<grid, 2 * kT2Band, step2_smem_bytes(kStep2Plain), s>>>(src, dst, g, fc, mp, omega, sp, flag,
                                                                         counter, send_lo, send_hi);
    *err = cudaGetLastError();
    return *err == cudaSuccess ? sp.nf_lo + sp.nf_hi : 0;
}

cudaError_t launch_step2_split(const double* src, double* dst, const DevGeo& g, const Faces& fc,
                               const ModelParams& mp, double omega, int* flag, cudaStream_t s, const int ctas[3]) {
    cudaError_t e;
    device_nsm(&e);
    if (e != cudaSuccess) return e;
    Step2Split sp{};
    sp.form = step2_form();
    sp.lock = (sp.form == kStep2Plain || sp.form == kStep2Bulk2) && step2_sched();
    int grid = 0;
    for (int part = 0; part < 3; ++part) {
        part_range(g, fc, sp.form, part, &sp.band0[part], &sp.nb[part]);
        const long long total = (long long)std::max(0, sp.nb[part]) * g.lx;
        sp.ctas[part] = total > 0 ? (int)std::min<long long>(ctas[part], total) : 0;
        if (total > 0 && sp.ctas[part] < 1) return cudaErrorInvalidValue;  // a part with items and no CTA
        sp.per_cta[part] = sp.ctas[part] ? (total + sp.ctas[part] - 1) / sp.ctas[part] : 0;
        grid += sp.ctas[part];
    }
    if (grid == 0) return cudaSuccess;
    if (sp.lock && sp.ctas[0] > 0) sp.ls = lockstep_plan(sp.nb[0], sp.ctas[0], g.lx);
    k_step2_split<<<grid, 2 * kT2Band, step2_smem_bytes(sp.form), s>>>(src, dst, g, fc, mp, omega, sp, flag);
    return cudaGetLastError();
}

cudaError_t launch_step2_pair_split(const double* src, double* dst, const DevGeo& g, const Faces& fc,
                                    const ModelParams& mp, double omega, int* flag, cudaStream_t s, cudaStream_t side,
                                    cudaEvent_t ev_fork, cudaEvent_t ev_join, const int ctas[3]) {
    cudaError_t e;
    device_nsm(&e);
    if (e != cudaSuccess) return e;
    Step2Split sp{};
    sp.form = kStep2Plain;  // unused: part 0 has no CTA in the face launch
    int band0 = 0, nb0 = 0, grid = 0;
    part_range(g, fc, kStep2Pair, 0, &band0, &nb0);
    for (int part = 1; part < 3; ++part) {
        part_range(g, fc, kStep2Pair, part, &sp.band0[part], &sp.nb[part]);
        const long long total = (long long)std::max(0, sp.nb[part]) * g.lx;
        sp.ctas[part] = total > 0 ? (int)std::min<long long>(ctas[part], total) : 0;
        if (total > 0 && sp.ctas[part] < 1) return cudaErrorInvalidValue;
        sp.per_cta[part] = sp.ctas[part] ? (total + sp.ctas[part] - 1) / sp.ctas[part] : 0;
        grid += sp.ctas[part];
    }
    if (grid > 0) {
        if ((e = cudaEventRecord(ev_fork, s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(side, ev_fork, 0)) != cudaSuccess) return e;
        k_step2_split<<<grid, 2 * kT2Band, step2_smem_bytes(kStep2Plain), side>>>(src, dst, g, fc, mp, omega, sp, flag);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (nb0 > 0 && (e = launch_step2_pair(src, dst, g, fc, mp, omega, flag, s, band0, nb0, ctas[0], step2_sched() != 0)) !=
                       cudaSuccess)
        return e;
    if (grid > 0) {
        if ((e = cudaEventRecord(ev_join, side)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(s, ev_join, 0)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace d2q37
