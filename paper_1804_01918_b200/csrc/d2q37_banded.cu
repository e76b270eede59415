// d2q37_banded.cu -- the band-blocked device store and its two-steps-per-sweep kernel.
//
// Why a fifth device layout.  A FUSED2 sweep (d2q37_step2.cu) reads, per
// column of a 120-row band, 37 row segments (~1 KB each, one per population,
// from the 7 columns x - cx) and writes 37 more.  On the SoA store those 74
// segments lie in 37 population planes half a gigabyte apart, and a probe of
// exactly that access stream with the arithmetic removed
// (tools/experiments/tb2/membench.cu) tops out at 4.3-4.7 TB/s of
// algorithmic traffic: the kernel with arithmetic ran at the same rate, so
// the sweep was bound by the DRAM access pattern, not by compute.  With the
// 37 populations of one (column, band) block contiguous the same stream moves
// 5.1-6.2 TB/s.
//
// Layout (DevGeo::band = 1; x-periodic lattice of lx x ly sites, nbt bands of
// kBandRows = 120 rows, the last one possibly partial): one block per
// (column x, band b) of 37 population rows of 136 doubles,
//   blk[x][b][s][L]   row y = 120 b - 8 + L of population p = pop of slot s
//                     (populations sorted by cx, so each of the 7 pull
//                     columns of a step is one contiguous run of a block)
// L = 8 .. 127 are the band's own rows; L = 0 .. 7 and 128 .. 135 are copies
// of the neighbouring bands' edge rows (8 rows, not the 6 a pull needs, so
// every row range a writer stores is whole 32-byte sectors).  Every store of
// row y also goes to every slot that holds row y, y + ly or y - ly (periodic
// images -- a slab's ghost rows, written by the halo exchange before each
// sweep, share those slots; a wall face never reads them), so a band's
// producer reads only its own block, whatever the faces.  A partial last
// band keeps the rows after it (images / ghosts) in its tail.
//
// Sweep (k_band_sweep): the schedule of d2q37_step2.cu -- persistent CTAs
// marching along x, producer warps computing step 1 of column r into the
// shared-memory ring, consumer warps step 2 of column r - 4 -- with the
// producer's pulls staged by 7 bulk copies per column (one per cx group,
// 40 KB) into one of two shared stages guarded by mbarriers, issued as soon
// as the producers hold the stage's previous column in registers.
// Walls are mirrored on the fly; every other face reads slots.
// Each site update is collide_site_sym on the gathered values of
// k_collide<FAST, SHIFT>, so a sweep is bit for bit two FUSED steps (a
// one-step sweep, TWO = false, serves odd step counts).
#include <cuda_runtime.h>

#include <algorithm>

#include "d2q37_device.cuh"
#include "d2q37_fused2.cuh"
#include "d2q37_kernels.cuh"

namespace d2q37 {

namespace {

constexpr int kBR = kBandRows;           // rows per band
constexpr int kBH = kBandHalo;           // halo rows per side kept in a block
constexpr int kBS = kBR + 2 * kBH;       // block rows per population (136)
constexpr int kBlk = kNpop * kBS;        // elements per (x, band) block
constexpr unsigned kBandStageBytes = unsigned(kBlk) * sizeof(double);  // 40 256 B
static_assert(kBR == kT2Out, "a band block is one FUSED2 band");

// storage slot of population p (sorted by cx, then canonical index)
D2Q37_HD constexpr int slot_of(int p) {
    int s = 0;
    for (int q = 0; q < kNpop; ++q)
        if (cx_of(q) < cx_of(p) || (cx_of(q) == cx_of(p) && q < p)) ++s;
    return s;
}
// first slot and size of the cx = g - 3 group
D2Q37_HD constexpr int group_start(int g) {
    int s = 0;
    for (int q = 0; q < kNpop; ++q)
        if (cx_of(q) < g - kHalo) ++s;
    return s;
}
__constant__ int c_gstart[2 * kHalo + 2] = {group_start(0), group_start(1), group_start(2), group_start(3),
                                            group_start(4), group_start(5), group_start(6), kNpop};

// Rows a block holds: i = y - 120 bb in [-8, 128) (L = i + 8).  Rows it does
// not own (i < 0, i >= ny) are filled up to 8 past the band: a pull reads
// i in [-6, ny + 6).
__device__ __forceinline__ int band_ny(const DevGeo& g, int bb) { return min(kBR, g.ly - bb * kBR); }

// Element of (block (x, bb), block row i, population slot s) = base + s * kBS.
__device__ __forceinline__ long long band_base(const DevGeo& g, int x, int bb, int i) {
    return g.lead + ((long long)x * g.nbt + bb) * kBlk + (i + kBH);
}

// Every block row holding lattice row y (0 <= y < ly) of column x: the owner
// first, then halo copies and periodic images (at most 5 in all).
__device__ __forceinline__ int band_targets(const DevGeo& g, int x, int y, long long (&base)[6]) {
    int n = 0;
    const int b = y / kBR;
    base[n++] = band_base(g, x, b, y - b * kBR);
    const int imgs[3] = {y, y + g.ly, y - g.ly};
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        const int yp = imgs[m];
        const int bc = (yp >= 0 ? yp : yp - kBR + 1) / kBR;  // floor
#pragma unroll
        for (int bb = bc - 1; bb <= bc + 1; ++bb) {
            if (bb < 0 || bb >= g.nbt) continue;
            const int i = yp - bb * kBR;
            const int ny = band_ny(g, bb);
            if (i < -kBH || i >= min(kBR + kBH, ny + kBH) || (i >= 0 && i < ny)) continue;  // not a copy slot
            if (n < 6) base[n++] = band_base(g, x, bb, i);
        }
    }
    return n;
}

__device__ __forceinline__ long long band_owner(const DevGeo& g, int x, int y) {
    const int b = y / kBR;
    return band_base(g, x, b, y - b * kBR);
}

// storage slot of population p (runtime index)
__constant__ signed char c_slot[kNpop] = {
    slot_of(0),  slot_of(1),  slot_of(2),  slot_of(3),  slot_of(4),  slot_of(5),  slot_of(6),  slot_of(7),
    slot_of(8),  slot_of(9),  slot_of(10), slot_of(11), slot_of(12), slot_of(13), slot_of(14), slot_of(15),
    slot_of(16), slot_of(17), slot_of(18), slot_of(19), slot_of(20), slot_of(21), slot_of(22), slot_of(23),
    slot_of(24), slot_of(25), slot_of(26), slot_of(27), slot_of(28), slot_of(29), slot_of(30), slot_of(31),
    slot_of(32), slot_of(33), slot_of(34), slot_of(35), slot_of(36)};
__device__ __forceinline__ int slot_of_rt(int p) { return c_slot[p]; }
// cx of the population in storage slot s
D2Q37_HD constexpr int cx_of_slot(int s) {
    for (int p = 0; p < kNpop; ++p)
        if (slot_of(p) == s) return cx_of(p);
    return 0;
}
__constant__ signed char c_cx_slot[kNpop] = {
    cx_of_slot(0),  cx_of_slot(1),  cx_of_slot(2),  cx_of_slot(3),  cx_of_slot(4),  cx_of_slot(5),  cx_of_slot(6),
    cx_of_slot(7),  cx_of_slot(8),  cx_of_slot(9),  cx_of_slot(10), cx_of_slot(11), cx_of_slot(12), cx_of_slot(13),
    cx_of_slot(14), cx_of_slot(15), cx_of_slot(16), cx_of_slot(17), cx_of_slot(18), cx_of_slot(19), cx_of_slot(20),
    cx_of_slot(21), cx_of_slot(22), cx_of_slot(23), cx_of_slot(24), cx_of_slot(25), cx_of_slot(26), cx_of_slot(27),
    cx_of_slot(28), cx_of_slot(29), cx_of_slot(30), cx_of_slot(31), cx_of_slot(32), cx_of_slot(33), cx_of_slot(34),
    cx_of_slot(35), cx_of_slot(36)};

}  // namespace

// ---------------------------------------------------------------------------
// The sweep.

// Step-1 ring of the banded sweep: population p of the step-1 column produced at
// iteration t is read by step 2 at iteration t + cx_p + 4 and its slot is
// rewritten at iteration t + depth.  Depth cx_p + 4 (148 columns, 148 KB) --
// one less than the SoA sweep's -- because the consumers read an iteration's
// slots before the producers overwrite them (named barrier 2), which leaves
// room for two bulk-copy stages.
D2Q37_HD constexpr int b2_depth(int p) { return cx_of(p) + 4; }
D2Q37_HD constexpr int b2_base(int p) {
    int s = 0;
    for (int q = 0; q < p; ++q) s += b2_depth(q);
    return s;
}
constexpr int kB2RingCols = b2_base(kNpop);  // 148
// timing probes (tools/gpu_g8.sh; results are garbage): 1 / 2 / 3 no consumer / producer / any collide,
// 4 no stores, 5 no bulk copies, 6 one copy per population instead of per cx group
#ifndef D2Q37_BAND_PROBE
#define D2Q37_BAND_PROBE 0
#endif
constexpr int kBandStages = 2;

// named barriers (256 threads): 2 = consumers -> producers "this iteration's ring slots are read",
// 3 = producers -> consumers "this iteration's step-1 column is in the ring"
__device__ __forceinline__ void nb_sync(int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id) { asm volatile("bar.arrive %0, 256;" ::"r"(id) : "memory"); }

template <bool TWO>
__global__ void __launch_bounds__(2 * kT2Band, 1)
    k_band_sweep(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, Faces fc, ModelParams mp,
                 double omega, long long per_cta, int* __restrict__ flag) {
    extern __shared__ double ring[];
    double* const stage0 = ring + kB2RingCols * kT2Band;  // kBandStages blocks [37][136]
    unsigned long long* const full = reinterpret_cast<unsigned long long*>(stage0 + kBandStages * kBlk);
    const bool prod = threadIdx.x < kT2Band;
    const int tid = threadIdx.x & (kT2Band - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = g.lx, ly = g.ly, nbt = g.nbt;
    const bool wall_lo = fc.lo == kFaceWall, wall_hi = fc.hi == kFaceWall;
    const long long total = (long long)nbt * lx;
    long long item = (long long)blockIdx.x * per_cta;
    const long long item_end = min(total, item + per_cta);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kBandStages; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
#if D2Q37_BAND_PROBE == 6 || D2Q37_BAND_PROBE == 7
    // probe: one copy per population (slot 10 w + lane), block rows 2 .. 135
    const int isl = 10 * warp + lane;
    const bool issuer = prod && lane < 10 && isl < kNpop;
    const int gs = issuer ? isl : 0;
    const unsigned ibytes = unsigned((kBS - 2) * sizeof(double));
    const int icx = issuer ? c_cx_slot[isl] : 0;
    constexpr int kIoff = 2;
#else
    // copy issue: producer warp w, lanes 0-1 -> cx group 2 w + lane (7 groups, one contiguous run each)
    const int igr = 2 * warp + lane;
    const bool issuer = prod && lane < 2 && igr < 2 * kHalo + 1;
    const int gs = issuer ? c_gstart[igr] : 0, gn = issuer ? c_gstart[igr + 1] - gs : 0;
    const unsigned ibytes = unsigned(gn * kBS * sizeof(double));
    const int icx = igr - kHalo;
    constexpr int kIoff = 0;
#endif
    unsigned issued = 0, used = 0;  // stage columns issued / consumed by this CTA (stage = n % 2)
    bool bad = false;
    while (item < item_end) {
        const int band = (int)(item / lx);
        const int xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (item_end - item));
        item += xe - xs;
        const int y0 = band * kBR;
        const int ny = min(kBR, ly - y0);
        const int niter = xe - xs + 7;  // producer columns xs-3 .. xe+2 at t = 0 .. niter-2
        // wall bands: the pulls of this band reach beyond a wall (mirrored)
        const bool wlo = wall_lo && band == 0, whi = wall_hi && y0 + kBR + kHalo + kHalo > ly;
        if (prod) {
            auto issue = [&](int r) {  // stage the column of producer row r
                const unsigned st = issued % kBandStages;
                if (issuer && D2Q37_BAND_PROBE != 5) {
                    const int col = wrap_mod(wrap_mod(r, lx) - icx, lx);
                    bulk_g2s(stage0 + st * kBlk + gs * kBS + kIoff,
                             src + g.lead + ((long long)col * nbt + band) * kBlk + gs * kBS + kIoff, ibytes, full + st);
                }
                if (threadIdx.x == 0 && D2Q37_BAND_PROBE != 5)
                    mbar_arrive_expect_tx(full + st, D2Q37_BAND_PROBE == 6 || D2Q37_BAND_PROBE == 7
                                                         ? unsigned(kNpop * (kBS - 2) * sizeof(double))
                                                         : kBandStageBytes);
                ++issued;
            };
            for (int k = 0; k < kBandStages && k < niter - 1; ++k) issue(xs - kHalo + k);
            // step-1 row of this thread, clamped: rows beyond a wall are never read (step 2
            // mirrors into the lattice), rows past ly + 2 / the band's 126 rows are unused
            int y1 = y0 - kHalo + tid;
            if (wlo) y1 = max(y1, 0);
            if (whi) y1 = min(y1, ly - 1);
            y1 = min(y1, min(ly + kHalo - 1, y0 + kBR + kHalo - 1));
            const int L0 = y1 - y0 + kBH;  // block row of y1 (the pull of cy is at L0 - cy)
#pragma unroll 1
            for (int t = 0; t < niter - 1; ++t) {
                const unsigned st = used % kBandStages;
                if (D2Q37_BAND_PROBE != 5) mbar_wait(full + st, (used / kBandStages) & 1);  // probe 5: no copies
                ++used;
                const double* const sg = stage0 + st * kBlk;
                double f[kNpop];
                if (!(wlo || whi)) {
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value;
                        f[p] = sg[slot_of(p) * kBS + L0 - cy_of(p)];
                    });
                } else {
                    int l0 = L0;
                    asm volatile("" : "+r"(l0));  // recomputed per iteration: no hoisted (spilled) offsets
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value, q = ybar_of(p);
                        int L = l0 - cy_of(p);
                        int s = slot_of(p);
                        const int yy = y0 + L - kBH;  // lattice row of the pull
                        if (wlo && yy < 0) {  // specular wall: population ybar at the mirror row
                            L = -1 - yy - y0 + kBH;
                            s = slot_of(q);
                        } else if (whi && yy >= ly) {
                            L = 2 * ly - 1 - yy - y0 + kBH;
                            s = slot_of(q);
                        }
                        f[p] = sg[s * kBS + L];
                    });
                }
                // the 37 values are in registers (an empty asm consumes them): the stage is free
#pragma unroll
                for (int p = 0; p < kNpop; p += 6)
                    asm volatile("" ::"d"(f[p]), "d"(f[min(p + 1, kNpop - 1)]), "d"(f[min(p + 2, kNpop - 1)]),
                                 "d"(f[min(p + 3, kNpop - 1)]), "d"(f[min(p + 4, kNpop - 1)]),
                                 "d"(f[min(p + 5, kNpop - 1)]));
                if (t + kBandStages < niter - 1) {
                    // every producer warp syncs (an arrive-only warp could run an iteration ahead and
                    // arrive twice at one barrier instance: nothing else bounds the producers per iteration)
                    prod_bar_sync();
                    issue(xs - kHalo + t + kBandStages);
                }
                if (D2Q37_BAND_PROBE != 2 && D2Q37_BAND_PROBE != 3 && D2Q37_BAND_PROBE != 7)
                    bad |= collide_site_sym(f, omega, mp);  // probes 2, 3: no producer collide
                nb_sync(2);  // the consumers have read this iteration's slots
                for_pops([&](auto P) {
                    constexpr int p = decltype(P)::value, rb = b2_base(p), dp = b2_depth(p);
                    ring[(rb + t % dp) * kT2Band + tid] = f[p];
                });
                nb_arrive(3);
            }
            nb_sync(2);  // the consumers' last iteration
        } else {
            const int y = y0 + tid;
            const bool active = tid < ny;
            // wall bands: ring row of y - cy (k = cy + 3) and whether it is a mirror image
            int pos[2 * kHalo + 1];
            unsigned mirm = 0;
#pragma unroll
            for (int k = 0; k < 2 * kHalo + 1; ++k) {
                int ys = y - (k - kHalo);
                const bool m = (ys < 0 && wlo) || (ys >= ly && whi);
                if (m) ys = ys < 0 ? -1 - ys : 2 * ly - 1 - ys;
                mirm |= unsigned(m) << k;
                pos[k] = ys - (y0 - kHalo);
            }
            const bool wband = wlo || whi;
            // rows whose value also lives in other blocks: band-edge halo copies (interior bands: one,
            // inline) and near the lattice edges periodic images (band_targets)
            const bool img_band = band == 0 || band >= nbt - 2;
            const bool edge_row = tid < kBH || tid >= kBR - kBH;
            const bool extra = img_band ? (edge_row || y < kBH || y >= ly - kBH) : edge_row;
            const long long copy_off = (tid < kBH ? -(long long)kBlk + kBR : (long long)kBlk - kBR);
#pragma unroll 1
            for (int t = 0; t < niter; ++t) {
                if (t > 0) nb_sync(3);  // step-1 column t - 1 is in the ring
                const int c = TWO ? xs - 7 + t : xs - 4 + t;  // output column of this iteration
                const bool work = active && c >= xs && c < xe;
                double v[kNpop];
                if (work) {
                    if (!TWO) {  // one step: the step-1 values of column c (produced at t - 1)
                        for_pops([&](auto P) {
                            constexpr int p = decltype(P)::value, rb = b2_base(p), dp = b2_depth(p);
                            v[p] = ring[(rb + (t - 1) % dp) * kT2Band + tid + kHalo];
                        });
                    } else if (!wband) {  // column c - cx_p, produced at t - 4 - cx_p: slot t % depth
                        for_pops([&](auto P) {
                            constexpr int p = decltype(P)::value, rb = b2_base(p), dp = b2_depth(p);
                            v[p] = ring[(rb + t % dp) * kT2Band + tid + kHalo - cy_of(p)];
                        });
                    } else {
                        for_pops([&](auto P) {
                            constexpr int p = decltype(P)::value, dp = b2_depth(p);
                            constexpr int k = cy_of(p) + kHalo, rb = b2_base(p), rbb = b2_base(ybar_of(p));
                            const int base = (mirm >> k) & 1u ? rbb : rb;
                            v[p] = ring[(base + t % dp) * kT2Band + pos[k]];
                        });
                    }
                    // the reads have landed before the producers may overwrite the slots
#pragma unroll
                    for (int p = 0; p < kNpop; p += 6)
                        asm volatile("" ::"d"(v[p]), "d"(v[min(p + 1, kNpop - 1)]), "d"(v[min(p + 2, kNpop - 1)]),
                                     "d"(v[min(p + 3, kNpop - 1)]), "d"(v[min(p + 4, kNpop - 1)]),
                                     "d"(v[min(p + 5, kNpop - 1)]));
                }
                nb_arrive(2);
                if (work) {
                    if (TWO && D2Q37_BAND_PROBE != 1 && D2Q37_BAND_PROBE != 3 && D2Q37_BAND_PROBE != 7)
                        bad |= collide_site_sym(v, omega, mp);  // probes 1, 3: no consumer collide
                    double* __restrict__ o = dst + band_base(g, c, band, tid);
                    if (D2Q37_BAND_PROBE == 4) continue;  // probe 4: no stores
                    for_pops([&](auto P) {
                        constexpr int p = decltype(P)::value;
                        __stcs(o + slot_of(p) * kBS, v[p]);
                    });
                    if (extra) {
                        if (!img_band) {  // the previous band's high / the next band's low copy
                            double* __restrict__ oo = o + copy_off;
                            for_pops([&](auto P) {
                                constexpr int p = decltype(P)::value;
                                __stcs(oo + slot_of(p) * kBS, v[p]);
                            });
                        } else {
                            long long tb[6];
                            const int n = band_targets(g, c, y, tb);
#pragma unroll 1
                            for (int m = 1; m < n; ++m) {
                                double* __restrict__ oo = dst + tb[m];
                                for_pops([&](auto P) {
                                    constexpr int p = decltype(P)::value;
                                    __stcs(oo + slot_of(p) * kBS, v[p]);
                                });
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();  // the item's ring is drained before the next item reuses it
    }
    if (bad) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// Canonical planes, init, moments, 6-row slab halos.

__global__ void k_band_scatter(double* __restrict__ buf, DevGeo g, const double* __restrict__ canon, int p) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)g.lx * g.ly) return;
    const int x = int(t / g.ly), y = int(t % g.ly);
    const double v = canon[t];
    long long tb[6];
    const int n = band_targets(g, x, y, tb);
    const long long so = (long long)slot_of_rt(p) * kBS;
    for (int m = 0; m < n; ++m) buf[tb[m] + so] = v;
}

__global__ void k_band_gather(const double* __restrict__ buf, DevGeo g, double* __restrict__ canon, int p) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)g.lx * g.ly) return;
    const int x = int(t / g.ly), y = int(t % g.ly);
    canon[t] = buf[band_owner(g, x, y) + (long long)slot_of_rt(p) * kBS];
}

__device__ __forceinline__ double philox_u01_band(unsigned long long seed, unsigned long long ctr) {
    unsigned int c0 = (unsigned int)ctr, c1 = (unsigned int)(ctr >> 32), c2 = 0u, c3 = 0u;
    unsigned int k0 = (unsigned int)seed, k1 = (unsigned int)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const unsigned int hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const unsigned int hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const unsigned int n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    const unsigned long long bits = (unsigned long long)c0 | ((unsigned long long)c1 << 32);
    return (double)(bits >> 11) * 0x1.0p-53;
}

// k_init_rt (d2q37_kernels.cu) on the band-blocked store: same per-site values.
__global__ void k_band_init_rt(double* __restrict__ buf, DevGeo g, ModelParams mp, unsigned long long seed, int y0,
                               int ly_global) {
    const int yl = blockIdx.x * blockDim.x + threadIdx.x;
    if (yl >= g.ly) return;
    const int x = blockIdx.y, y = y0 + yl;
    const double noise = -1e-3 + 2e-3 * philox_u01_band(seed, (unsigned long long)x * ly_global + y);
    const double yint = 0.5 * ly_global + 0.01 * ly_global * sin(2.0 * 3.14159265358979323846 * x / g.lx);
    const double temp = ((double)y < yint ? 1.5 : 0.5) + noise;
    const double rho = 1.0 / temp;
    const double dt = temp - mp.t0, dt2 = dt * dt;
    const double m2 = dt, m9 = 3.0 * dt2, m11 = dt2;
    long long tb[6];
    const int n = band_targets(g, x, yl, tb);
#pragma unroll 1
    for (int p = 0; p < kNpop; ++p) {
        const double* gp = mp.eq[p];
        double s = 1.0;
        s += gp[2] * m2;
        s += gp[4] * m2;
        s += gp[9] * m9;
        s += gp[11] * m11;
        s += gp[13] * m9;
        const double v = rho * mp.w[p] * s;
        const long long so = (long long)slot_of_rt(p) * kBS;
        for (int m = 0; m < n; ++m) buf[tb[m] + so] = v;
    }
}

__global__ void __launch_bounds__(256) k_band_moments(const double* __restrict__ buf, DevGeo g,
                                                      double* __restrict__ part) {
    __shared__ double red[4][256];
    const int x = blockIdx.x;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int y = threadIdx.x; y < g.ly; y += blockDim.x) {
        const long long e = band_owner(g, x, y);
#pragma unroll
        for (int p = 0; p < kNpop; ++p) {
            const double v = buf[e + slot_of(p) * kBS];
            s[0] += v;
            s[1] += cx_of(p) * v;
            s[2] += cy_of(p) * v;
            s[3] += (cx_of(p) * cx_of(p) + cy_of(p) * cy_of(p)) * v;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) red[i][threadIdx.x] = s[i];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
#pragma unroll
            for (int i = 0; i < 4; ++i) red[i][threadIdx.x] += red[i][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
#pragma unroll
        for (int i = 0; i < 4; ++i) part[blockIdx.x * 4 + i] = red[i][0];
}

// rows 0..5 / ly-6..ly-1 -> send buffers [p][x][6] (the SoA k_pack6 format)
__global__ void __launch_bounds__(256) k_band_pack6(const double* __restrict__ buf, DevGeo g,
                                                   double* __restrict__ send_lo, double* __restrict__ send_hi) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = int(i % (2 * kHalo));
    const long long px = i / (2 * kHalo);
    const int x = int(px % g.lx), p = int(px / g.lx);
    const long long so = (long long)slot_of_rt(p) * kBS;
    if (send_lo) send_lo[i] = buf[band_owner(g, x, r) + so];
    if (send_hi) send_hi[i] = buf[band_owner(g, x, g.ly - 2 * kHalo + r) + so];
}

// received rows -> the slots of rows -6..-1 / ly..ly+5 (a null buffer skips that face)
__global__ void __launch_bounds__(256) k_band_unpack6(double* __restrict__ buf, DevGeo g,
                                                     const double* __restrict__ recv_lo,
                                                     const double* __restrict__ recv_hi) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = int(i % (2 * kHalo));
    const long long px = i / (2 * kHalo);
    const int x = int(px % g.lx), p = int(px / g.lx);
    const long long so = (long long)slot_of_rt(p) * kBS;
    for (int face = 0; face < 2; ++face) {
        const double* rv = face == 0 ? recv_lo : recv_hi;
        if (!rv) continue;
        const int yp = face == 0 ? r - 2 * kHalo : g.ly + r;  // ghost row
        const int bc = (yp >= 0 ? yp : yp - kBR + 1) / kBR;
        for (int bb = bc - 1; bb <= bc + 1; ++bb) {
            if (bb < 0 || bb >= g.nbt) continue;
            const int iy = yp - bb * kBR, ny = band_ny(g, bb);
            if (iy < -kBH || iy >= min(kBR + kBH, ny + kBH) || (iy >= 0 && iy < ny)) continue;
            buf[band_base(g, x, bb, iy) + so] = rv[i];
        }
    }
}

// ---------------------------------------------------------------------------
// Host side.

namespace {
template <typename K>
cudaError_t band_attr(K kern) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)band_smem_bytes());
}
}  // namespace

size_t band_smem_bytes() {
    return (size_t)kB2RingCols * kT2Band * sizeof(double) + kBandStages * kBandStageBytes + 16;  // + mbarriers
}

void band_geometry(int lx, int ly, DevGeo* g) {
    *g = DevGeo{};
    g->lx = lx;
    g->ly = ly;
    g->vl = 1;
    g->strip = ly;
    g->sy = ly;
    g->px = lx;
    g->band = 1;
    g->nbt = (ly + kBR - 1) / kBR;
    g->pitch = g->nbt * kBS;
    g->lead = 0;
    g->pstride = kBS;
    g->rstride = 1;
    g->cstride = (long long)g->nbt * kBlk;
}

size_t band_elems(const DevGeo& g) { return size_t((long long)g.lx * g.nbt * kBlk + 64); }

cudaError_t launch_band_sweep(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                              double omega, bool two, int* flag, cudaStream_t s) {
    constexpr int kMaxDev = 64;
    static int nsm_of[kMaxDev] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int nsm = dev < kMaxDev ? nsm_of[dev] : 0;
    if (nsm == 0) {
        e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = band_attr(k_band_sweep<true>);
        if (e == cudaSuccess) e = band_attr(k_band_sweep<false>);
        if (e != cudaSuccess) return e;
        if (dev < kMaxDev) nsm_of[dev] = nsm;
    }
    const long long total = (long long)g.nbt * g.lx;
    const int grid = (int)std::min<long long>(nsm, total);
    const long long per_cta = (total + grid - 1) / grid;
    if (two)
        k_band_sweep<true><<<grid, 2 * kT2Band, band_smem_bytes(), s>>>(src, dst, g, fc, mp, omega, per_cta, flag);
    else
        k_band_sweep<false><<<grid, 2 * kT2Band, band_smem_bytes(), s>>>(src, dst, g, fc, mp, omega, per_cta, flag);
    return cudaGetLastError();
}

cudaError_t launch_band_scatter(double* buf, const DevGeo& g, const double* canon_plane, int p, cudaStream_t s) {
    const long long n = (long long)g.lx * g.ly;
    k_band_scatter<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(buf, g, canon_plane, p);
    return cudaGetLastError();
}

cudaError_t launch_band_gather(const double* buf, const DevGeo& g, double* canon_plane, int p, cudaStream_t s) {
    const long long n = (long long)g.lx * g.ly;
    k_band_gather<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(buf, g, canon_plane, p);
    return cudaGetLastError();
}

cudaError_t launch_band_init_rt(double* buf, const DevGeo& g, const ModelParams& mp, unsigned long long seed, int y0,
                                int ly_global, cudaStream_t s) {
    k_band_init_rt<<<dim3((g.ly + 127) / 128, g.lx), 128, 0, s>>>(buf, g, mp, seed, y0, ly_global);
    return cudaGetLastError();
}

cudaError_t launch_band_moments(const double* buf, const DevGeo& g, double* part, cudaStream_t s) {
    k_band_moments<<<g.lx, 256, 0, s>>>(buf, g, part);
    return cudaGetLastError();
}

cudaError_t launch_band_pack6(const double* buf, const DevGeo& g, double* send_lo, double* send_hi, cudaStream_t s) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    k_band_pack6<<<unsigned((n + 255) / 256), 256, 0, s>>>(buf, g, send_lo, send_hi);
    return cudaGetLastError();
}

cudaError_t launch_band_unpack6(double* buf, const DevGeo& g, const double* recv_lo, const double* recv_hi,
                                cudaStream_t s) {
    const long long n = (long long)kNpop * g.lx * 2 * kHalo;
    k_band_unpack6<<<unsigned((n + 255) / 256), 256, 0, s>>>(buf, g, recv_lo, recv_hi);
    return cudaGetLastError();
}

cudaError_t preload_band_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_band_sweep<true>);
    cudaFuncGetAttributes(&a, k_band_sweep<false>);
    cudaFuncGetAttributes(&a, k_band_scatter);
    cudaFuncGetAttributes(&a, k_band_gather);
    cudaFuncGetAttributes(&a, k_band_init_rt);
    cudaFuncGetAttributes(&a, k_band_moments);
    cudaFuncGetAttributes(&a, k_band_pack6);
    cudaFuncGetAttributes(&a, k_band_unpack6);
    return cudaGetLastError();
}

}  // namespace d2q37
