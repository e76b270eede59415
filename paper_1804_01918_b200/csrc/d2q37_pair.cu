// d2q37_pair.cu -- FUSED2 interior sweep with two threads per site (form kStep2Pair).
//
// The two-steps-per-sweep schedule of d2q37_step2.cu (persistent CTAs marching
// along x over 120-row bands, producers computing step 1 of column r into a
// shared-memory ring, consumers computing step 2 of column r - 4 from it; the
// producers' pulls staged by two bulk-copy stages -- sweep_tma2), with every
// site update split over TWO threads: thread half 0 holds the 17 populations
// of the rest velocity and the quadruples with |cx|, |cy| <= 2, half 1 the 20
// of the axis shells and the (3, 1) / (1, 3) quadruples (pop_half,
// d2q37_device.cuh; about equal FP64 work).  Each
// thread sums the moments of its half; the pair swaps the four partial sums
// {rho, jx, jy, e2} through tensor memory (tcgen05.st / tcgen05.ld: the two
// warps of a pair own the same TMEM lanes) and both form rho = A + B, ...;
// each then relaxes and stores its own half.
//
// Why: the one-thread-per-site sweep runs 2 warps per scheduler (255
// registers x 256 threads) and is latency bound (ncu: 63 % of cycles with no
// eligible warp; stalls on FP64 dependency chains and on the producer /
// consumer hand-off).  Half a site per thread needs < 128 registers, so the
// CTA runs 512 threads -- 4 warps per scheduler -- with half the dependent
// work per warp, on the same shared memory (148-column ring + 2 stages).
//
// Warps 0-7 produce, 8-15 consume; warp w handles rows 32 (w & 3) .. +31 of
// the band column, half (w >> 2) & 1.  Named barriers: 2 consumers ->
// producers (ring slots read; the producers have all read the stage, which
// is then refilled), 3 producers ->
// consumers (step-1 column published), 4-7 / 8-11 the producer / consumer
// pairs (w, w + 4) around the TMEM swap.
//
// Results are bit-identical to every other FAST kernel (same gathered values,
// same per-half summation order, same relaxation).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>

#include "d2q37_device.cuh"
#include "d2q37_fused2.cuh"
#include "d2q37_kernels.cuh"

namespace d2q37 {

namespace {

constexpr int kPairThreads = 4 * kT2Band;  // 512
// who refills a stage with column t + 2, and when: 0 the producers right after barrier 2 of iteration t,
// 1 the producers after publishing column t (barrier 3), 2 the consumers once they hold column t,
// 3 the half-0 consumers at the end of their iteration t, behind an "empty" mbarrier the producer warps
// arrive on when their stage reads of iteration t have landed
#ifndef D2Q37_PAIR_ISSUE_MODE
#define D2Q37_PAIR_ISSUE_MODE 1
#endif
static_assert(kFaceGhost == 3 && kFaceWall == 1, "pair_slab_plan's face kinds (d2q37_fused2.cuh)");
constexpr int kTmemCols = 64;              // [role][parity][half] x 8 32-bit columns (4 doubles)

__device__ __forceinline__ void tmem_st8(unsigned taddr, const double (&v)[4]) {
    unsigned r[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) asm("mov.b64 {%0, %1}, %2;" : "=r"(r[2 * i]), "=r"(r[2 * i + 1]) : "d"(v[i]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_ld8(unsigned taddr, double (&v)[4]) {
    unsigned r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) asm("mov.b64 %0, {%1, %2};" : "=d"(v[i]) : "r"(r[2 * i]), "r"(r[2 * i + 1]));
}

// The pair's partial sums: this warp's half into its columns, barrier with the
// partner warp (64 threads), the partner's half back.  Columns alternate with
// the swap count's parity (and the role barriers 2 / 3 separate consecutive
// swaps of a role), so a fast warp's next store never overwrites values its
// partner has not read yet.
__device__ __forceinline__ void pair_swap(unsigned tbase, int role, int par, int half, int barid,
                                          const double (&mine)[4], double (&other)[4]) {
    const unsigned lane_base = unsigned((threadIdx.x >> 5) & 3) * 32u << 16;
    const unsigned col = unsigned(role * 32 + par * 16);
    tmem_st8(tbase + lane_base + col + unsigned(half * 8), mine);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync %0, 64;" ::"r"(barid) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tmem_ld8(tbase + lane_base + col + unsigned((1 - half) * 8), other);
}

// One half-site update: moments of half H, swap, macros, relaxation of half H.
template <int H>
__device__ __forceinline__ bool pair_collide(double (&f)[kNpop], const ModelParams& mp, double omega,
                                             unsigned tbase, int role, int par, int barid) {
    double mine[4], other[4];
    sym_partials<H>(f, mine);
    pair_swap(tbase, role, par, H, barid, mine, other);
    SymMoments m;
    const bool bad = H == 0 ? sym_macros(mine, other, mp, m) : sym_macros(other, mine, mp, m);
    sym_relax_half<H>(f, m, omega, mp);
    return bad;
}

// t % d for the ring depths d = 1 .. 7 (t2n_depth), advanced once per iteration instead of seven
// divisions by constants per iteration
struct SlotClock {
    int s[7];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int i = 0; i < 7; ++i) s[i] = 0;
    }
    __device__ __forceinline__ void tick() {
#pragma unroll
        for (int i = 1; i < 7; ++i) s[i] = s[i] == i ? 0 : s[i] + 1;
    }
    __device__ __forceinline__ int operator[](int depth) const { return s[depth - 1]; }
};

template <typename F>
__device__ __forceinline__ void consume_regs(const double (&v)[kNpop], F&& in_set) {
    // an empty asm per value of the set: the loads have landed (the stage / ring slots may be reused)
    for_pops([&](auto P) {
        constexpr int p = decltype(P)::value;
        if (in_set(p)) asm volatile("" ::"d"(v[p]));
    });
}

// Bulk-copy staging of the producers' pulls: copy n (a whole column, 37 x 1040 B, completion counted on
// full[n & 1]) fills the stage of producer use n.  Producer warps 0-3 issue the copies of column t + 2
// right after the hand-off barrier 2 of iteration t -- every producer has read the stage of iteration t
// before its collide.  (Measured against earlier refills -- a producer-wide barrier after the stage
// reads, an "empty" mbarrier with one issuing warp or with the consumers issuing: all slower, DESIGN 3.1.1.)
struct StageIssuer {
    const double* sb;
    double* stage0;
    unsigned long long* full;
    long long plane, cs;
    int lx, ip, icx, icy;
    bool issuer, leader;
    unsigned issued;
    const double* isrc;
    __device__ __forceinline__ void set_band(int y0) { isrc = sb + ip * plane + ((y0 - kHalo - icy) & ~1); }
    __device__ __forceinline__ void issue(int r, bool active = true, unsigned long long* empty = nullptr) {
        const unsigned st = issued & 1u;
        // mode 3: the use this copy overwrites (two copies back) has been read by every producer warp
        if (empty && active && (issuer || leader)) mbar_wait(empty + st, ((issued - 2u) >> 1) & 1u);
        if (issuer && active) {
            int col = r < 0 ? r + lx : (r >= lx ? r - lx : r);
            col -= icx;
            col = col < 0 ? col + lx : (col >= lx ? col - lx : col);
            bulk_g2s(stage0 + (st * kNpop + ip) * kStageRows, isrc + (long long)col * cs, kStageRows * sizeof(double),
                     full + st);
#ifdef D2Q37_PAIR_PREFETCH  // L2 prefetch of the column D2Q37_PAIR_PREFETCH further on
            int pc = col + D2Q37_PAIR_PREFETCH;
            pc = pc >= lx ? pc - lx : pc;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(isrc + (long long)pc * cs),
                         "r"(unsigned(kStageRows * sizeof(double)))
                         : "memory");
#endif
        }
        if (leader && active) mbar_arrive_expect_tx(full + st, kStageBytes);
        ++issued;
    }
};

__device__ __forceinline__ StageIssuer make_issuer(const double* sb, const DevGeo& g, double* stage0,
                                                   unsigned long long* full, int warp0 = 0) {
    StageIssuer is;
    const int warp = (threadIdx.x >> 5) - warp0, lane = threadIdx.x & 31;
    is.sb = sb;
    is.stage0 = stage0;
    is.full = full;
    is.plane = g.pstride;
    is.cs = g.cstride;
    is.lx = g.lx;
#ifndef D2Q37_PAIR_ISSUE_WARPS
#define D2Q37_PAIR_ISSUE_WARPS 4
#endif
    // warps 0 .. W-1, lane l < 40 / W -> population (40 / W) w + l
    constexpr int kPer = 40 / D2Q37_PAIR_ISSUE_WARPS;
    is.ip = warp * kPer + lane;
    is.issuer = warp >= 0 && warp < D2Q37_PAIR_ISSUE_WARPS && lane < kPer && is.ip < kNpop;
    is.leader = warp == 0 && lane == 0;
    if (!is.issuer) is.ip = 0;
    is.icx = is.issuer ? c_cx[is.ip] : 0;
    is.icy = is.issuer ? c_cy[is.ip] : 0;
    is.issued = 0;
    is.isrc = sb;
    return is;
}

// Send-buffer packing and the sweep counter of a face CTA (null: none)
struct SlabPack {
    double* send_lo;
    double* send_hi;
    unsigned* counter;
};

template <class Sched>
__device__ __forceinline__ bool sched_in_face(const Sched&) { return false; }
__device__ __forceinline__ bool sched_in_face(const FaceSched& s) { return s.in_face; }

// Wall bands (specular reflection): a pull of row y - cy beyond a wall reads population
// ybar(p) = (cx, -cy) at the mirror row -1 - (y - cy) / 2 ly - 1 - (y - cy).  walls: bit 0 the low face
// is a wall, bit 1 the high one; a band needs the mirror tables when its producer rows reach row 0 /
// row ly - 1 within the pull distance.
__device__ __forceinline__ bool wall_lo_band(int walls, int band) { return (walls & 1) && band == 0; }
__device__ __forceinline__ bool wall_hi_band(int walls, int y0, int ly) { return (walls & 2) && y0 + kT2Band - 1 >= ly; }
__device__ __forceinline__ int mirror_row(int ys, int ly, bool wlo, bool whi) {
    return (wlo && ys < 0) ? -1 - ys : (whi && ys >= ly) ? 2 * ly - 1 - ys : INT_MIN;
}

template <int H, bool GHOST, class Sched>
__device__ __forceinline__ void pair_producer(const double* __restrict__ sb, const DevGeo& g, const ModelParams& mp,
                                              double omega, Sched sched, int walls, double* ring, double* stage0,
                                              unsigned long long* full, unsigned tbase, bool& bad) {
    const int tid = threadIdx.x & (kT2Band - 1);
    const int warp = threadIdx.x >> 5;
    const int ly = g.ly;
    const int pbar = 4 + (warp & 3);
    StageIssuer is = make_issuer(sb, g, stage0, full);
    unsigned used = 0;
    int band, xs, xe;
    while (sched.next(band, xs, xe)) {
        const int y0 = band * kT2Out;
        const int niter = xe - xs + 7;
        is.set_band(y0);
        for (int k = 0; k < 2 && k < niter - 1; ++k) is.issue(xs - kHalo + k);  // (every mode: by the producers)
        // step-1 row of this thread, clamped: rows beyond a wall are never read (step 2 mirrors into the
        // lattice), rows past ly + 2 never (their pulls would leave a slab's deep ghost rows)
        const bool wlo = wall_lo_band(walls, band), whi = wall_hi_band(walls, y0, ly);
        int y1 = y0 - kHalo + tid;
        if (wlo) y1 = max(y1, 0);
        if (whi) y1 = min(y1, ly - 1);
        if (GHOST) y1 = min(y1, ly + kHalo - 1);
        const int yo = y1 - (y0 - kHalo);
        const int par = (y0 - kHalo) & 1;
        // wall bands: per k = cy + 3, the stage offset of the mirrored pull (population ybar, whose stage
        // starts at row (y0 - 3 + cy) & ~1) or none
        unsigned mirm = 0;
        int moff[2 * kHalo + 1];
#pragma unroll
        for (int k = 0; k < 2 * kHalo + 1; ++k) {
            const int cy = k - kHalo, m = mirror_row(y1 - cy, ly, wlo, whi);
            mirm |= unsigned(m != INT_MIN) << k;
            moff[k] = m - ((y0 - kHalo + cy) & ~1);
        }
        SlotClock clk;
        clk.reset();
#pragma unroll 1
        for (int t = 0; t < niter - 1; ++t) {
            const unsigned st = used & 1u;
            mbar_wait(full + st, (used >> 1) & 1u);
            ++used;
            const double* const sg = stage0 + st * kNpop * kStageRows;
            double f[kNpop];
            if (!mirm) {
                for_pops([&](auto P) {
                    constexpr int p = decltype(P)::value;
                    if (pop_half(p) == H) f[p] = sg[p * kStageRows + yo + (par ^ (cy_of(p) & 1))];
                });
            } else {
                for_pops([&](auto P) {
                    constexpr int p = decltype(P)::value, k = cy_of(p) + kHalo, q = ybar_of(p);
                    if (pop_half(p) == H)
                        f[p] = (mirm >> k) & 1u ? sg[q * kStageRows + moff[k]]
                                                : sg[p * kStageRows + yo + (par ^ (cy_of(p) & 1))];
                });
            }
            consume_regs(f, [](int p) { return pop_half(p) == H; });
#if D2Q37_PAIR_ISSUE_MODE == 3
            if ((threadIdx.x & 31) == 0) mbar_arrive(full + 2 + st);  // empty[st]: this warp's stage reads landed
#endif
            bad |= pair_collide<H>(f, mp, omega, tbase, 0, int(used & 1u), pbar);  // parity: runs across segments
            // the consumers have read this iteration's slots -- and every producer has read the stage
            // (before its collide): refill it with column t + 2
#ifdef D2Q37_PAIR_PRESYNC  // measured -2 %: the producers do not wait at this barrier
            // The barrier number depends on every relaxed value (or'ed high words, masked by a run-time
            // zero), so the relaxation is complete before the hand-off barrier: ptxas otherwise sinks its
            // tail (~25 FP64 operations, a 10-deep dependent chain) below the barrier, between it and the
            // ring stores the consumers wait for.
            unsigned dep = 0;
            for_pops([&](auto P) {
                constexpr int p = decltype(P)::value;
                if (pop_half(p) == H) dep |= unsigned(__double2hiint(f[p]));
            });
            asm volatile("bar.sync %0, 512;" ::"r"(2u + (dep & unsigned(g.band))) : "memory");  // g.band == 0 here
#else
            asm volatile("bar.sync 2, 512;" ::: "memory");
#endif
#if D2Q37_PAIR_ISSUE_MODE == 0
            if (t + 2 < niter - 1) is.issue(xs - kHalo + t + 2);
#endif
            for_pops([&](auto P) {
                constexpr int p = decltype(P)::value, rb = t2n_base(p), dp = t2n_depth(p);
                if (pop_half(p) == H) ring[(rb + clk[dp]) * kT2Band + tid] = f[p];
            });
            asm volatile("bar.arrive 3, 512;" ::: "memory");
#if D2Q37_PAIR_ISSUE_MODE == 1
            if (t + 2 < niter - 1) is.issue(xs - kHalo + t + 2);
#elif D2Q37_PAIR_ISSUE_MODE >= 2
            if (t + 2 < niter - 1) is.issue(xs - kHalo + t + 2, false);  // the consumers issue it; count it
#endif
            clk.tick();
        }
        asm volatile("bar.sync 2, 512;" ::: "memory");  // the consumers' last iteration
    }
}

template <int H, class Sched>
__device__ __forceinline__ void pair_consumer(const double* __restrict__ sb, double* __restrict__ db, const DevGeo& g,
                                              const ModelParams& mp, double omega, Sched sched, int walls,
                                              const double* ring, double* stage0, unsigned long long* full,
                                              unsigned tbase, const SlabPack& pk, bool& bad) {
    const int tid = threadIdx.x & (kT2Band - 1);
    const int warp = threadIdx.x >> 5;
    const int lx = g.lx, ly = g.ly;
    const long long plane = g.pstride, cs = g.cstride;
    const int cbar = 8 + (warp & 3);
    unsigned swaps = 0;  // TMEM column parity of the pair swaps, running across segments
#if D2Q37_PAIR_ISSUE_MODE == 2
    StageIssuer is = make_issuer(sb, g, stage0, full, 8);
#elif D2Q37_PAIR_ISSUE_MODE == 3
    StageIssuer is = make_issuer(sb, g, stage0, full, H == 0 ? 8 : 64);  // half 1: no issuing lane
#else
    (void)sb, (void)stage0, (void)full;
#endif
    int band, xs, xe;
    bool was_face = sched_in_face(sched);
    while (sched.next(band, xs, xe)) {
        const bool face = sched_in_face(sched);
        if (was_face && !face) {
            // every consumer's face rows (lattice and send buffers) are stored: announce them
            asm volatile("bar.sync 12, 256;" ::: "memory");
            if (threadIdx.x == 2 * kT2Band) {
                __threadfence_system();
                atomicAdd(pk.counter, 1u);
            }
        }
        was_face = face;
        const int y0 = band * kT2Out;
        const int ny = min(kT2Out, ly - y0);
        const int niter = xe - xs + 7;
        const bool active = tid < ny;
        const bool wlo = wall_lo_band(walls, band), whi = wall_hi_band(walls, y0, ly);
        // idle lanes (rows >= ny) collide a copy of the band's last row
        const int row = min(tid, (wlo || whi ? ny : kT2Out) - 1);
        const int y = y0 + tid;
        // wall bands: per k = cy + 3, the ring row of the mirrored pull (population ybar) or none
        unsigned mirm = 0;
        int mpos[2 * kHalo + 1];
#pragma unroll
        for (int k = 0; k < 2 * kHalo + 1; ++k) {
            const int m = mirror_row(y0 + row - (k - kHalo), ly, wlo, whi);
            mirm |= unsigned(m != INT_MIN) << k;
            mpos[k] = m - (y0 - kHalo);
        }
        // face segments: rows 0..5 / ly-6..ly-1 of the new state also go to the send buffers ([p][x][6])
        double* __restrict__ sl = face && pk.send_lo && y < 2 * kHalo ? pk.send_lo + y : nullptr;
        double* __restrict__ sh = face && pk.send_hi && y >= ly - 2 * kHalo && active ? pk.send_hi + (y - (ly - 2 * kHalo))
                                                                                    : nullptr;
        SlotClock clk;  // t % depth
        clk.reset();
#if D2Q37_PAIR_ISSUE_MODE == 2
        is.set_band(y0);
        for (int k = 0; k < 2 && k < niter - 1; ++k) is.issue(xs - kHalo + k, false);  // (the producers' prologue)
#elif D2Q37_PAIR_ISSUE_MODE == 3
        if (H == 0) {
            is.set_band(y0);
            for (int k = 0; k < 2 && k < niter - 1; ++k) is.issue(xs - kHalo + k, false);
        }
#endif
#pragma unroll 1
        for (int t = 0; t < niter; ++t) {
            if (t > 0) asm volatile("bar.sync 3, 512;" ::: "memory");  // step-1 column t - 1 is in the ring
            double v[kNpop];
            if (t >= 7) {  // column c - cx_p, produced at t - 4 - cx_p: slot t % depth
                if (!mirm) {
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2n_base(p), dp = t2n_depth(p);
                        if (pop_half(p) == H) v[p] = ring[(rb + clk[dp]) * kT2Band + row + kHalo - cy_of(p)];
                    });
                } else {  // ybar(p) has p's cx, hence p's ring depth
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, rb = t2n_base(p), dp = t2n_depth(p);
                        constexpr int k = cy_of(p) + kHalo, rbb = t2n_base(ybar_of(p));
                        if (pop_half(p) == H)
                            v[p] = (mirm >> k) & 1u ? ring[(rbb + clk[dp]) * kT2Band + mpos[k]]
                                                    : ring[(rb + clk[dp]) * kT2Band + row + kHalo - cy_of(p)];
                    });
                }
                consume_regs(v, [](int p) { return pop_half(p) == H; });
            }
            asm volatile("bar.arrive 2, 512;" ::: "memory");
#if D2Q37_PAIR_ISSUE_MODE == 2
            // every producer has passed barrier 2 of iteration t - 1, hence read its stage: refill it
            if (t >= 1 && t + 1 < niter - 1) is.issue(xs - kHalo + t + 1);
#endif
            if (t >= 7) {
                const bool b = pair_collide<H>(v, mp, omega, tbase, 1, int(swaps++ & 1u), cbar);
                if (active) {
                    bad |= b;
                    const int x = xs - 7 + t;
                    double* __restrict__ o = db + ((long long)x * cs + y);
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value;
                        if (pop_half(p) == H) __stcs(o + p * plane, v[p]);
                    });
                    if (sl) {
                        for_pops([&](auto P) {
                            constexpr int p = decltype(P)::value;
                            if (pop_half(p) == H) sl[((long long)p * lx + x) * (2 * kHalo)] = v[p];
                        });
                    }
                    if (sh) {
                        for_pops([&](auto P) {
                            constexpr int p = decltype(P)::value;
                            if (pop_half(p) == H) sh[((long long)p * lx + x) * (2 * kHalo)] = v[p];
                        });
                    }
                }
            }
            clk.tick();
#if D2Q37_PAIR_ISSUE_MODE == 3
            // the producers' iteration t runs beside this one and read its stage at its start: refill it
            if (H == 0 && t + 2 < niter - 1) is.issue(xs - kHalo + t + 2, true, full + 2);
#endif
        }
    }
    if (was_face) {  // the schedule ended inside the face bands
        asm volatile("bar.sync 12, 256;" ::: "memory");
        if (threadIdx.x == 2 * kT2Band) {
            __threadfence_system();
            atomicAdd(pk.counter, 1u);
        }
    }
}

// Shared-memory layout, TMEM allocation and the role split of every pair kernel; `sched` gives this
// CTA's segments.
template <bool GHOST, class Sched>
__device__ __forceinline__ void pair_sweep(const double* __restrict__ src, double* __restrict__ dst, const DevGeo& g,
                                           const ModelParams& mp, double omega, const Sched& sched, int walls,
                                           const SlabPack& pk, int* __restrict__ flag) {
    extern __shared__ double ring[];
    double* const stage0 = ring + kT2NRingCols * kT2Band;  // 2 stages [37][130]
    unsigned long long* const full = reinterpret_cast<unsigned long long*>(stage0 + 2 * kNpop * kStageRows);
    unsigned* const tslot = reinterpret_cast<unsigned*>(full + 4);  // full[2], empty[2] (issue mode 3)
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tslot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        mbar_init(full + 1, 1);
        mbar_init(full + 2, 8);  // one arrival per producer warp
        mbar_init(full + 3, 8);
        asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tbase = *tslot;
    const double* __restrict__ sb = src + g.lead + kHalo * g.cstride + kHalo;
    double* __restrict__ db = dst + g.lead + kHalo * g.cstride + kHalo;
    bool bad = false;
    const bool half = (warp >> 2) & 1;
    if (warp < 8) {
        if (!half)
            pair_producer<0, GHOST>(sb, g, mp, omega, sched, walls, ring, stage0, full, tbase, bad);
        else
            pair_producer<1, GHOST>(sb, g, mp, omega, sched, walls, ring, stage0, full, tbase, bad);
    } else {
        if (!half)
            pair_consumer<0>(sb, db, g, mp, omega, sched, walls, ring, stage0, full, tbase, pk, bad);
        else
            pair_consumer<1>(sb, db, g, mp, omega, sched, walls, ring, stage0, full, tbase, pk, bad);
    }
    if (bad) atomicOr(flag, 1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols) : "memory");
}

template <bool GHOST>
__global__ void __launch_bounds__(kPairThreads, 1)
    k_step2_pair(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, ModelParams mp, double omega,
                 int band0, int nbands, long long per_cta, int lock, Lockstep ls, int walls, int* __restrict__ flag) {
    const int cta = blockIdx.x;
    const PartSched sched{lock != 0, RangeSched(band0, nbands, g.lx, cta * per_cta, (cta + 1) * per_cta),
                          LockSched(band0, g.lx, (int)gridDim.x, cta, ls)};
    pair_sweep<GHOST>(src, dst, g, mp, omega, sched, walls, SlabPack{nullptr, nullptr, nullptr}, flag);
}

// One overlapped FUSED2 sweep of a y-slab in the pair form.  CTAs [0, nf_lo) / [nf_lo, nf_lo + nf_hi)
// sweep the ghost-face band(s) of the low / high face first -- packing the new edge rows into the send
// buffers and announcing them on the sweep counter -- then the interior bands next to them; the other
// CTAs march the remaining bands in lockstep, a global wall's band among them (mirror tables).

__global__ void __launch_bounds__(kPairThreads, 1)
    k_step2_pair_slab(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, ModelParams mp,
                      double omega, PairSlabPlan sp, int* __restrict__ flag, unsigned* __restrict__ counter,
                      double* __restrict__ send_lo, double* __restrict__ send_hi) {
    const int cta = blockIdx.x, lx = g.lx;
    if (cta < sp.nf_lo + sp.nf_hi) {
        const bool lo = cta < sp.nf_lo;
        const long long c = lo ? cta : cta - sp.nf_lo;
        const FaceSched fs =
            lo ? FaceSched{RangeSched(sp.lo_face0, sp.lo_face_nb, lx, c * sp.lo_face_per, (c + 1) * sp.lo_face_per),
                           RangeSched(sp.lo_adj0, sp.lo_adj_nb, lx, c * sp.lo_adj_per, (c + 1) * sp.lo_adj_per), true}
               : FaceSched{RangeSched(sp.hi_face0, sp.hi_face_nb, lx, c * sp.hi_face_per, (c + 1) * sp.hi_face_per),
                           RangeSched(sp.hi_adj0, sp.hi_adj_nb, lx, c * sp.hi_adj_per, (c + 1) * sp.hi_adj_per), true};
        pair_sweep<true>(src, dst, g, mp, omega, fs, sp.walls,
                         SlabPack{lo ? send_lo : nullptr, lo ? nullptr : send_hi, counter}, flag);
    } else {
        const int G = (int)gridDim.x - sp.nf_lo - sp.nf_hi;
        const LockSched ls(sp.main_band0, lx, G, cta - sp.nf_lo - sp.nf_hi, sp.ls);
        pair_sweep<true>(src, dst, g, mp, omega, ls, sp.walls, SlabPack{nullptr, nullptr, nullptr}, flag);
    }
}

size_t pair_smem_bytes() {
    return (size_t)kT2NRingCols * kT2Band * sizeof(double) + 2 * size_t(kStageBytes) + 32 + 16;  // + mbarriers, TMEM slot
}

}  // namespace

cudaError_t launch_step2_pair(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                              double omega, int* flag, cudaStream_t s, int band0, int nb, int ctas, bool lock) {
    static bool attr[64] = {};
    cudaError_t e = once_per_device(attr, [] {
        cudaError_t r = cudaFuncSetAttribute(k_step2_pair<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pair_smem_bytes());
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(k_step2_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pair_smem_bytes());
        return r;
    });
    if (e != cudaSuccess) return e;
    const long long total = (long long)std::max(0, nb) * g.lx;
    if (total == 0) return cudaSuccess;
    ctas = (int)std::min<long long>(ctas, total);
    if (ctas < 1) return cudaErrorInvalidValue;
    const long long per_cta = (total + ctas - 1) / ctas;
    const Lockstep ls = lockstep_plan(nb, ctas, g.lx);
    const int walls = (fc.lo == kFaceWall ? 1 : 0) | (fc.hi == kFaceWall ? 2 : 0);
    if (fc.hi == kFaceGhost)
        k_step2_pair<true><<<ctas, kPairThreads, pair_smem_bytes(), s>>>(src, dst, g, mp, omega, band0, nb, per_cta,
                                                                       lock, ls, walls, flag);
    else
        k_step2_pair<false><<<ctas, kPairThreads, pair_smem_bytes(), s>>>(src, dst, g, mp, omega, band0, nb, per_cta,
                                                                        lock, ls, walls, flag);
    return cudaGetLastError();
}

int launch_step2_pair_slab(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                           double omega, int* flag, cudaStream_t s, int grid, unsigned* counter, double* send_lo,
                           double* send_hi, cudaError_t* err) {
    *err = cudaSuccess;
    PairSlabPlan sp{};
    if (!pair_slab_plan(g.lx, g.ly, fc.lo, fc.hi, grid, &sp)) return 0;
    static bool attr[64] = {};
    *err = once_per_device(attr, [] {
        return cudaFuncSetAttribute(k_step2_pair_slab, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)pair_smem_bytes());
    });
    if (*err != cudaSuccess) return 0;
    k_step2_pair_slab<<<grid, kPairThreads, pair_smem_bytes(), s>>>(src, dst, g, mp, omega, sp, flag, counter, send_lo,
                                                                    send_hi);
    if ((*err = cudaGetLastError()) != cudaSuccess) return 0;
    return sp.nf_lo + sp.nf_hi;
}

}  // namespace d2q37
