// d2q37_fused2.cuh -- shared pieces of the two-steps-per-sweep kernels
// (d2q37_step2.cu on the SoA store, d2q37_banded.cu on the band-blocked store):
// the step-1 ring geometry, a compile-time population loop and the
// bulk-copy / mbarrier PTX wrappers.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
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
    D2Q37_HD RangeSched(int band0_, int nbands, int lx_, long long b, long long e)
        : band0(band0_), lx(lx_), item(b), end((long long)nbands * lx_ < e ? (long long)nbands * lx_ : e) {}
    D2Q37_HD __forceinline__ bool next(int& band, int& xs, int& xe) {
        if (item >= end) return false;
        band = band0 + (int)(item / lx);
        xs = (int)(item % lx);
        xe = (int)((long long)lx < xs + (end - item) ? (long long)lx : xs + (end - item));
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
    // even split (q > 0, only without whole rounds): each band on q CTAs, CTA i of a band marching
    // columns [i w, (i + 1) w) -- every band's CTAs start on the same columns, so neighbouring bands
    // stay in lockstep over the whole sweep (few bands on many CTAs: the streamed run's chunks)
    int q, w;
};
struct LockSched {
    int band0, lx, G, c, k;
    Lockstep ls;
    long long j, jend;
    D2Q37_HD LockSched(int band0_, int lx_, int G_, int c_, const Lockstep& l)
        : band0(band0_), lx(lx_), G(G_), c(c_), k(0), ls(l), j(0), jend(0) {
        if (c >= ls.rem && ls.rem > 0) {
            const long long w = lx - ls.cut;
            j = (long long)(c - ls.rem) * ls.tail_per;
            jend = j + ls.tail_per < (long long)ls.rem * w ? j + ls.tail_per : (long long)ls.rem * w;
        }
    }
    D2Q37_HD __forceinline__ bool next(int& band, int& xs, int& xe) {
        if (k < ls.full) {
            band = band0 + c + k * G;
            xs = 0;
            xe = lx;
            ++k;
            return true;
        }
        const int base = band0 + ls.full * G;
        if (ls.q > 0) {
            if (k > ls.full || c >= ls.q * ls.rem) return false;
            ++k;
            band = base + c / ls.q;
            xs = (c % ls.q) * ls.w;
            xe = lx < xs + ls.w ? lx : xs + ls.w;
            return xs < xe;
        }
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
        xe = (int)((long long)lx < xs + (jend - j) ? (long long)lx : xs + (jend - j));
        j += xe - xs;
        return true;
    }
};

// LockSched of G CTAs over nb bands of lx columns
inline Lockstep lockstep_plan(int nb, int G, int lx) {
    Lockstep ls{};
    ls.full = nb / G;
    ls.rem = nb % G;
    // few bands on many CTAs: the even split when it idles at most 1 CTA in 32
    if (ls.full == 0 && ls.rem > 0 && G >= 2 * ls.rem && (G % ls.rem) * 32 <= G && lx >= 8 * (G / ls.rem)) {
        ls.q = G / ls.rem;
        ls.w = (lx + ls.q - 1) / ls.q;
        return ls;
    }
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
// Bands of a sweep: [b_lo, b_hi) pull only rows inside [0, ly) (band 0 pulls rows down to -6, the bands
// from (ly - 128) / 120 + 1 on reach past ly); degenerate extents: none.
inline void interior_bands(int lx, int ly, int* nbands, int* b_lo, int* b_hi) {
    *nbands = (ly + kT2Out - 1) / kT2Out;
    *b_lo = 1;
    *b_hi = std::min(*nbands, ly >= kT2Band ? (ly - kT2Band) / kT2Out + 1 : 0);
    if (lx < kHalo || *b_hi <= *b_lo) *b_lo = *b_hi = 0;
}

// Item schedule of a y-slab face CTA (k_step2_pair_slab): its share of the face band(s) -- whose new
// edge rows go to the send buffers and, once stored, are announced on the sweep counter -- then its
// share of the interior bands next to them.
struct FaceSched {
    RangeSched face, adj;
    bool in_face;
    D2Q37_HD __forceinline__ bool next(int& band, int& xs, int& xe) {
        if (in_face) {
            if (face.next(band, xs, xe)) return true;
            in_face = false;
        }
        return adj.next(band, xs, xe);
    }
};

// One overlapped FUSED2 slab sweep in the pair form (k_step2_pair_slab).  CTAs [0, nf_lo) /
// [nf_lo, nf_lo + nf_hi) sweep the ghost-face band(s) of the low / high face first -- packing the new
// edge rows into the send buffers and announcing them on the sweep counter -- then the interior bands
// next to them; the other CTAs march the remaining bands in lockstep, a global wall's band among them
// (mirror tables).
struct PairSlabPlan {
    int nf_lo, nf_hi;
    int lo_face0, lo_face_nb, lo_adj0, lo_adj_nb;  // bands
    int hi_face0, hi_face_nb, hi_adj0, hi_adj_nb;
    long long lo_face_per, lo_adj_per, hi_face_per, hi_adj_per;  // items per face CTA
    int main_band0, main_nb;
    Lockstep ls;  // main CTAs: grid - nf_lo - nf_hi
    int walls;    // bit 0 / 1: the low / high face is a global wall (its band is a main band)
};

// The plan of one slab sweep on `grid` CTAs (face kinds kFaceGhost = 3 / kFaceWall = 1); false: no
// overlapped pair form for this slab (no ghost face, too few bands, edge rows outside the face bands).
inline bool pair_slab_plan(int lx, int ly, int face_lo, int face_hi, int grid, PairSlabPlan* out) {
    constexpr int kGhost = 3, kWall = 1;
    int nbands, b_lo, b_hi;
    interior_bands(lx, ly, &nbands, &b_lo, &b_hi);
    const bool ghost_lo = face_lo == kGhost, ghost_hi = face_hi == kGhost;
    const bool wall_lo = face_lo == kWall, wall_hi = face_hi == kWall;
    // the new edge rows must lie in the face bands: a full first band, >= 6 rows in the last one
    if (!(ghost_lo || ghost_hi) || !(ghost_lo || wall_lo) || !(ghost_hi || wall_hi) || b_lo != 1 ||
        b_hi - b_lo < 3 || grid < 16 || ly - (nbands - 1) * kT2Out < 2 * kHalo || ly < kT2Out)
        return false;
    const long long lo_items = (long long)b_lo * lx, hi_items = (long long)(nbands - b_hi) * lx;
    const double per = double(nbands) * lx / grid;  // items per CTA
    PairSlabPlan sp{};
    sp.walls = (wall_lo ? 1 : 0) | (wall_hi ? 2 : 0);
    // ghost faces: enough CTAs that a face share is at most a third of a CTA's work (the exchange then
    // starts a third into the sweep and hides under the rest: tools/slab_timeline.py), topped up with whole
    // interior bands next to the face; a wall face's band is an ordinary main band
    auto face_ctas = [&](long long items) {
        return std::max(1, std::min(grid / 8, (int)std::ceil(3.0 * items / per)));
    };
    int k_lo = 0, k_hi = 0;
    if (ghost_lo) {
        sp.nf_lo = face_ctas(lo_items);
        k_lo = std::max(0, (int)std::floor(sp.nf_lo * per / lx) - b_lo);
    }
    if (ghost_hi) {
        sp.nf_hi = face_ctas(hi_items);
        k_hi = std::max(0, (int)std::floor(sp.nf_hi * per / lx) - (nbands - b_hi));
    }
    while (k_lo + k_hi > b_hi - b_lo - 1) (k_lo >= k_hi ? k_lo : k_hi)--;  // keep >= 1 main band
    sp.lo_face0 = 0;
    sp.lo_face_nb = ghost_lo ? b_lo : 0;
    sp.lo_adj0 = b_lo;
    sp.lo_adj_nb = k_lo;
    sp.hi_face0 = b_hi;
    sp.hi_face_nb = ghost_hi ? nbands - b_hi : 0;
    sp.hi_adj0 = b_hi - k_hi;
    sp.hi_adj_nb = k_hi;
    auto share = [](long long items, int n) { return n ? (items + n - 1) / n : 0LL; };
    sp.lo_face_per = share(lo_items, sp.nf_lo);
    sp.lo_adj_per = share((long long)k_lo * lx, sp.nf_lo);
    sp.hi_face_per = share(hi_items, sp.nf_hi);
    sp.hi_adj_per = share((long long)k_hi * lx, sp.nf_hi);
    sp.main_band0 = ghost_lo ? b_lo + k_lo : 0;
    sp.main_nb = (ghost_hi ? b_hi - k_hi : nbands) - sp.main_band0;
    const int gmain = grid - sp.nf_lo - sp.nf_hi;
    if (gmain < 1 || sp.main_nb < 1) return false;
    sp.ls = lockstep_plan(sp.main_nb, gmain, lx);
    *out = sp;
    return true;
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
