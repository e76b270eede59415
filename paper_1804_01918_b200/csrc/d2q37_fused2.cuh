// d2q37_fused2.cuh -- shared pieces of the two-steps-per-sweep kernels
// (d2q37_step2.cu on the SoA store, d2q37_banded.cu on the band-blocked store):
// the step-1 ring geometry, a compile-time population loop and the
// bulk-copy / mbarrier PTX wrappers.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <utility>

#include "d2q37_device.cuh"

namespace d2q37 {
namespace {

#ifndef D2Q37_T2_OUT
#define D2Q37_T2_OUT 120
#endif
constexpr int kT2Band = 128;        // producer threads per band column (ring rows)
constexpr int kT2Out = D2Q37_T2_OUT;  // step-2 (output) rows per band: 120 keeps every band's stores 32-byte sectors
static_assert(kT2Out % 2 == 0 && kT2Out + 2 * kHalo <= kT2Band, "band rows");
D2Q37_HD constexpr int t2_depth(int p) { return cx_of(p) + 5; }
D2Q37_HD constexpr int t2_base(int p) {
    int s = 0;
    for (int q = 0; q < p; ++q) s += t2_depth(q);
    return s;
}
constexpr int kT2RingCols = t2_base(kNpop);  // 185
// The two-stage bulk-copy sweep (sweep_tma2) orders the consumers' ring reads of
// an iteration before the producers' writes (named barriers), so population p
// of a step-1 column lives cx_p + 4 iterations: 148 columns, 148 KB.
D2Q37_HD constexpr int t2n_depth(int p) { return cx_of(p) + 4; }
D2Q37_HD constexpr int t2n_base(int p) {
    int s = 0;
    for (int q = 0; q < p; ++q) s += t2n_depth(q);
    return s;
}
constexpr int kT2NRingCols = t2n_base(kNpop);  // 148
D2Q37_HD constexpr int ybar_of(int p) { return vel_index(cx_of(p), -cy_of(p)); }

// Item schedules: the (band, column range) segments one persistent CTA marches.
// RangeSched: the band-major items [item, end) of bands band0, band0 + 1, ...
struct RangeSched {
    int band0, lx;
    long long item, end;
    __device__ RangeSched(int band0_, int nbands, int lx_, long long b, long long e)
        : band0(band0_), lx(lx_), item(b), end(min((long long)nbands * lx_, e)) {}
    __device__ __forceinline__ bool next(int& band, int& xs, int& xe) {
        if (item >= end) return false;
        band = band0 + (int)(item / lx);
        xs = (int)(item % lx);
        xe = (int)min((long long)lx, xs + (end - item));
        item += xe - xs;
        return true;
    }
};

// LockSched: CTA c of G marches whole bands c, c + G, ... from column 0, so at
// any moment the CTAs of neighbouring bands work on the same columns: the
// rows a band pulls from its neighbours (6 + 6 of its 132-row window) are L2
// hits, and each population plane is read and written as a few contiguous
// column-long streams instead of 1 KB pieces scattered over the plane.  The
// last round (rem < G bands) runs columns [0, cut) of its bands on CTAs
// 0 .. rem-1 and the remaining columns, band-major, on the other G - rem CTAs
// (cut balances the two, counting the 7-iteration start of every segment).
struct Lockstep {
    int full;  // whole rounds of G bands
    int rem;   // bands of the last round
    int cut;   // columns [0, cut) of a last-round band on its own CTA
    long long tail_per;  // items of [cut, lx) x rem bands per tail CTA
};
struct LockSched {
    int band0, lx, G, c, k;
    Lockstep ls;
    long long j, jend;
    __device__ LockSched(int band0_, int lx_, int G_, int c_, const Lockstep& l)
        : band0(band0_), lx(lx_), G(G_), c(c_), k(0), ls(l), j(0), jend(0) {
        if (c >= ls.rem && ls.rem > 0) {
            const long long w = lx - ls.cut;
            j = (long long)(c - ls.rem) * ls.tail_per;
            jend = min(j + ls.tail_per, (long long)ls.rem * w);
        }
    }
    __device__ __forceinline__ bool next(int& band, int& xs, int& xe) {
        if (k < ls.full) {
            band = band0 + c + k * G;
            xs = 0;
            xe = lx;
            ++k;
            return true;
        }
        const int base = band0 + ls.full * G;
        if (c < ls.rem) {  // own last-round band, columns [0, cut)
            if (k > ls.full || ls.cut <= 0) return false;
            ++k;
            band = base + c;
            xs = 0;
            xe = ls.cut;
            return true;
        }
        if (j >= jend) return false;
        const int w = lx - ls.cut;
        band = base + (int)(j / w);
        xs = ls.cut + (int)(j % w);
        xe = (int)min((long long)lx, xs + (jend - j));
        j += xe - xs;
        return true;
    }
};

// LockSched of G CTAs over nb bands of lx columns
inline Lockstep lockstep_plan(int nb, int G, int lx) {
    Lockstep ls{};
    ls.full = nb / G;
    ls.rem = nb % G;
    if (ls.rem > 0) {
        const long long T = G - ls.rem;  // tail CTAs
        // cut + 7 = rem (lx - cut) / T + 7 rem / T: a tail CTA's columns and segment starts
        long long cut = ((long long)ls.rem * lx + 7LL * (ls.rem - T) + G - 1) / G;
        cut = std::max<long long>(1, std::min<long long>(lx, cut));
        ls.cut = (int)cut;
        ls.tail_per = (ls.rem * (lx - cut) + T - 1) / T;
    }
    return ls;
}
// Part 0 of k_step2_split: band-major ranges or the lockstep schedule.
struct PartSched {
    bool lock;
    RangeSched r;
    LockSched l;
    __device__ __forceinline__ bool next(int& band, int& xs, int& xe) {
        return lock ? l.next(band, xs, xe) : r.next(band, xs, xe);
    }
};

// Kernel attributes (the dynamic shared-memory opt-in) are per device: set them once per device.
// Returns cudaSuccess once `set` has succeeded on the current device.
template <typename F>
inline cudaError_t once_per_device(bool (&done)[64], F&& set) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
    e = set();
    if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
    return e;
}

// Compile-time loop over the populations (keeps ring offsets constants).
template <typename F, int... Ps>
__device__ __forceinline__ void for_pops_(F&& f, std::integer_sequence<int, Ps...>) {
    (f(std::integral_constant<int, Ps>{}), ...);
}
template <typename F>
__device__ __forceinline__ void for_pops(F&& f) {
    for_pops_(f, std::make_integer_sequence<int, kNpop>{});
}

__device__ __forceinline__ int wrap_mod(int v, int n) {
    if (v < 0) v += n;
    else if (v >= n) v -= n;
    if (v < 0 || v >= n) {  // degenerate extents (n < 7)
        v %= n;
        if (v < 0) v += n;
    }
    return v;
}

// ---- bulk-copy staging of the producer's pulls (sweep_tma) -----------------
// Per population a 16-byte-aligned superset of the 128 source rows: 130 doubles
// from the even row at or below y0 - 3 - cy_p (1040 B, a multiple of 16).
constexpr int kStageRows = kT2Band + 2;
constexpr unsigned kStageBytes = unsigned(kNpop) * kStageRows * sizeof(double);  // 38 480 B per column

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared 1-D bulk copy (SASS UBLKCP), completion counted on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
// velocity components by runtime index (the copy-issuing lanes)
__constant__ signed char c_cx[kNpop] = {0,  -1, 0,  0,  1,  -1, -1, 1,  1,  -2, 0,  0,  2,  -2, -2, -1, -1, 1, 1,
                                        2,  2,  -2, -2, 2,  2,  -3, 0,  0,  3,  -3, -3, -1, -1, 1,  1,  3,  3};
__constant__ signed char c_cy[kNpop] = {0,  0,  -1, 1,  0,  -1, 1,  -1, 1,  0,  -2, 2,  0,  -1, 1,  -2, 2, -2, 2,
                                        -1, 1,  -2, 2,  -2, 2,  0,  -3, 3,  0,  -1, 1,  -3, 3,  -3, 3,  -1, 1};
// named barrier 1 among the 128 producer threads
__device__ __forceinline__ void prod_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void prod_bar_arrive() { asm volatile("bar.arrive 1, 128;" ::: "memory"); }
// named barriers of all 256 threads (producer / consumer hand-off without __syncthreads)
__device__ __forceinline__ void nbar_sync(int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id) { asm volatile("bar.arrive %0, 256;" ::"r"(id) : "memory"); }

}  // namespace

}  // namespace d2q37
