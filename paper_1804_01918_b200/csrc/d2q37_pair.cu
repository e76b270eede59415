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

#include "d2q37_device.cuh"
#include "d2q37_fused2.cuh"
#include "d2q37_kernels.cuh"

namespace d2q37 {

namespace {

constexpr int kPairThreads = 4 * kT2Band;  // 512
// Who refills a stage with column t + 2, and when (A/B experiment): 0 the producers after the hand-off
// barrier (no extra barrier), 1 the producers after a producer-wide barrier right after the stage reads,
// 3 the consumer warps 8-11 once every producer warp has arrived on the stage's "empty" mbarrier, 4 the
// consumer warps 8-11 right after the hand-off barrier 3 (the producers have passed barrier 2).
#ifndef D2Q37_PAIR_REFILL
#define D2Q37_PAIR_REFILL 0
#endif
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
// the iteration parity, so a fast thread's next store never overwrites
// values its partner has not read yet.
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

template <typename F>
__device__ __forceinline__ void consume_regs(const double (&v)[kNpop], F&& in_set) {
    // an empty asm per value of the set: the loads have landed (the stage / ring slots may be reused)
    for_pops([&](auto P) {
        constexpr int p = decltype(P)::value;
        if (in_set(p)) asm volatile("" ::"d"(v[p]));
    });
}

// Bulk-copy staging of the producers' pulls: copy n (a whole column, 37 x 1040 B, completion counted on
// full[n & 1]) fills the stage of producer use n.  With D2Q37_PAIR_REFILL 3 the consumer warps issue the
// copies, waiting first until use n - 2 of that stage is released on empty[n & 1] (one arrival per producer
// warp); otherwise producer warps issue them at the point the variant fixes.
struct StageIssuer {
    const double* sb;
    double* stage0;
    unsigned long long* full;
    unsigned long long* empty;
    long long plane, cs;
    int lx, ip, icx, icy;
    bool issuer, leader;
    unsigned issued;
    const double* isrc;
    __device__ __forceinline__ void set_band(int y0) { isrc = sb + ip * plane + ((y0 - kHalo - icy) & ~1); }
    __device__ __forceinline__ void issue(int r, bool wait_empty) {
        const unsigned st = issued & 1u;
        if (wait_empty && issued >= 2) mbar_wait(empty + st, ((issued >> 1) + 1) & 1u);
        if (issuer) {
            int col = r < 0 ? r + lx : (r >= lx ? r - lx : r);
            col -= icx;
            col = col < 0 ? col + lx : (col >= lx ? col - lx : col);
            bulk_g2s(stage0 + (st * kNpop + ip) * kStageRows, isrc + (long long)col * cs, kStageRows * sizeof(double),
                     full + st);
        }
        if (leader) mbar_arrive_expect_tx(full + st, kStageBytes);
        ++issued;
    }
};

__device__ __forceinline__ StageIssuer make_issuer(const double* sb, const DevGeo& g, double* stage0,
                                                   unsigned long long* full, int first_warp) {
    StageIssuer is;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    is.sb = sb;
    is.stage0 = stage0;
    is.full = full;
    is.empty = full + 2;
    is.plane = g.pstride;
    is.cs = g.cstride;
    is.lx = g.lx;
    // warps first_warp .. +3, lane l < 10 -> population 10 (w - first_warp) + l
    is.ip = (warp - first_warp) * 10 + lane;
    is.issuer = warp >= first_warp && warp < first_warp + 4 && lane < 10 && is.ip < kNpop;
    is.leader = (int)threadIdx.x == first_warp * 32;
    if (!is.issuer) is.ip = 0;
    is.icx = is.issuer ? c_cx[is.ip] : 0;
    is.icy = is.issuer ? c_cy[is.ip] : 0;
    is.issued = 0;
    is.isrc = sb;
    return is;
}

template <int H, bool GHOST, class Sched>
__device__ __forceinline__ void pair_producer(const double* __restrict__ sb, const DevGeo& g, const ModelParams& mp,
                                              double omega, Sched sched, double* ring, double* stage0,
                                              unsigned long long* full, unsigned tbase, bool& bad) {
    unsigned long long* const empty = full + 2;
    const int tid = threadIdx.x & (kT2Band - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ly = g.ly;
    const int pbar = 4 + (warp & 3);
    constexpr bool kProdIssue = D2Q37_PAIR_REFILL < 3;
    StageIssuer is = make_issuer(sb, g, stage0, full, 0);
    unsigned used = 0;
    int band, xs, xe;
    while (sched.next(band, xs, xe)) {
        const int y0 = band * kT2Out;
        const int niter = xe - xs + 7;
        if (kProdIssue) {
            is.set_band(y0);
            for (int k = 0; k < 2 && k < niter - 1; ++k) is.issue(xs - kHalo + k, false);
        }
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
                if (pop_half(p) == H) f[p] = sg[p * kStageRows + yo + (par ^ (cy_of(p) & 1))];
            });
            consume_regs(f, [](int p) { return pop_half(p) == H; });
#if D2Q37_PAIR_REFILL == 1
            if (t + 2 < niter - 1) {
                asm volatile("bar.sync 1, 256;" ::: "memory");  // every producer has its values: refill
                is.issue(xs - kHalo + t + 2, false);
            }
#elif D2Q37_PAIR_REFILL == 3
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);  // this warp has read the stage
#endif
            bad |= pair_collide<H>(f, mp, omega, tbase, 0, t & 1, pbar);
            asm volatile("bar.sync 2, 512;" ::: "memory");  // the consumers have read this iteration's slots
#if D2Q37_PAIR_REFILL == 0
            // ... and every producer has read the stage (before its collide): refill it with column t + 2
            if (t + 2 < niter - 1) is.issue(xs - kHalo + t + 2, false);
#endif
            for_pops([&](auto P) {
                constexpr int p = decltype(P)::value, rb = t2n_base(p), dp = t2n_depth(p);
                if (pop_half(p) == H) ring[(rb + t % dp) * kT2Band + tid] = f[p];
            });
            asm volatile("bar.arrive 3, 512;" ::: "memory");
        }
        asm volatile("bar.sync 2, 512;" ::: "memory");  // the consumers' last iteration
    }
}

template <int H, class Sched>
__device__ __forceinline__ void pair_consumer(const double* __restrict__ sb, double* __restrict__ db, const DevGeo& g,
                                              const ModelParams& mp, double omega, Sched sched, const double* ring,
                                              double* stage0, unsigned long long* full, unsigned tbase, bool& bad) {
    const int tid = threadIdx.x & (kT2Band - 1);
    const int warp = threadIdx.x >> 5;
    const int ly = g.ly;
    const long long plane = g.pstride, cs = g.cstride;
    const int cbar = 8 + (warp & 3);
    constexpr bool kConsIssue = (D2Q37_PAIR_REFILL == 3 || D2Q37_PAIR_REFILL == 4) && H == 0;  // warps 8-11
    StageIssuer is = make_issuer(sb, g, stage0, full, 8);
    int band, xs, xe;
    while (sched.next(band, xs, xe)) {
        const int y0 = band * kT2Out;
        const int ny = min(kT2Out, ly - y0);
        const int niter = xe - xs + 7;
        const bool active = tid < ny;
        const int row = min(tid, kT2Out - 1);  // idle lanes (rows >= 120) collide a copy of row 119
        if (kConsIssue) {
            is.set_band(y0);
            for (int k = 0; k < 2 && k < niter - 1; ++k) is.issue(xs - kHalo + k, D2Q37_PAIR_REFILL == 3);
        }
#pragma unroll 1
        for (int t = 0; t < niter; ++t) {
            if (t > 0) asm volatile("bar.sync 3, 512;" ::: "memory");  // step-1 column t - 1 is in the ring
#if D2Q37_PAIR_REFILL == 4
            // ... so the producers have read their iteration-(t-1) stage: refill it for iteration t + 1
            if (kConsIssue && t >= 1 && t + 1 < niter - 1) is.issue(xs - kHalo + t + 1, false);
#endif
            double v[kNpop];
            if (t >= 7) {  // column c - cx_p, produced at t - 4 - cx_p: slot t % depth
                for_pops([&](auto P) {
                    constexpr int p = decltype(P)::value, rb = t2n_base(p), dp = t2n_depth(p);
                    if (pop_half(p) == H) v[p] = ring[(rb + t % dp) * kT2Band + row + kHalo - cy_of(p)];
                });
                consume_regs(v, [](int p) { return pop_half(p) == H; });
            }
            asm volatile("bar.arrive 2, 512;" ::: "memory");
#if D2Q37_PAIR_REFILL == 3
            // the producers' iteration-t stage is released once they have read it: refill it (column t + 2)
            if (kConsIssue && t + 2 < niter - 1) is.issue(xs - kHalo + t + 2, true);
#endif
            if (t >= 7) {
                const bool b = pair_collide<H>(v, mp, omega, tbase, 1, t & 1, cbar);
                if (active) {
                    bad |= b;
                    const long long e = (long long)(xs - 7 + t) * cs + y0 + tid;
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value;
                        if (pop_half(p) == H) __stcs(db + p * plane + e, v[p]);
                    });
                }
            }
        }
    }
}

template <bool GHOST>
__global__ void __launch_bounds__(kPairThreads, 1)
    k_step2_pair(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, ModelParams mp, double omega,
                 int band0, int nbands, long long per_cta, int lock, Lockstep ls, int* __restrict__ flag) {
    extern __shared__ double ring[];
    double* const stage0 = ring + kT2NRingCols * kT2Band;  // 2 stages [37][130]
    unsigned long long* const full = reinterpret_cast<unsigned long long*>(stage0 + 2 * kNpop * kStageRows);
    unsigned* const tslot = reinterpret_cast<unsigned*>(full + 4);  // full[2], empty[2], TMEM address
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
        mbar_init(full + 2, 8);
        mbar_init(full + 3, 8);
        asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tbase = *tslot;
    const double* __restrict__ sb = src + g.lead + kHalo * g.cstride + kHalo;
    double* __restrict__ db = dst + g.lead + kHalo * g.cstride + kHalo;
    const int cta = blockIdx.x;
    const PartSched sched{lock != 0, RangeSched(band0, nbands, g.lx, cta * per_cta, (cta + 1) * per_cta),
                          LockSched(band0, g.lx, (int)gridDim.x, cta, ls)};
    bool bad = false;
    const bool half = (warp >> 2) & 1;
    if (warp < 8) {
        if (!half)
            pair_producer<0, GHOST>(sb, g, mp, omega, sched, ring, stage0, full, tbase, bad);
        else
            pair_producer<1, GHOST>(sb, g, mp, omega, sched, ring, stage0, full, tbase, bad);
    } else {
        if (!half)
            pair_consumer<0>(sb, db, g, mp, omega, sched, ring, stage0, full, tbase, bad);
        else
            pair_consumer<1>(sb, db, g, mp, omega, sched, ring, stage0, full, tbase, bad);
    }
    if (bad) atomicOr(flag, 1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols) : "memory");
}

size_t pair_smem_bytes() {
    return (size_t)kT2NRingCols * kT2Band * sizeof(double) + 2 * size_t(kStageBytes) + 32 + 16;  // + mbarriers, TMEM slot
}

}  // namespace

cudaError_t launch_step2_pair(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                              double omega, int* flag, cudaStream_t s, int band0, int nb, int ctas, bool lock) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_step2_pair<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pair_smem_bytes());
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_step2_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pair_smem_bytes());
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const long long total = (long long)std::max(0, nb) * g.lx;
    if (total == 0) return cudaSuccess;
    ctas = (int)std::min<long long>(ctas, total);
    if (ctas < 1) return cudaErrorInvalidValue;
    const long long per_cta = (total + ctas - 1) / ctas;
    const Lockstep ls = lockstep_plan(nb, ctas, g.lx);
    if (fc.hi == kFaceGhost)
        k_step2_pair<true><<<ctas, kPairThreads, pair_smem_bytes(), s>>>(src, dst, g, mp, omega, band0, nb, per_cta,
                                                                       lock, ls, flag);
    else
        k_step2_pair<false><<<ctas, kPairThreads, pair_smem_bytes(), s>>>(src, dst, g, mp, omega, band0, nb, per_cta,
                                                                        lock, ls, flag);
    return cudaGetLastError();
}

}  // namespace d2q37
