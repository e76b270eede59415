// membench.cu -- experiment: the memory side of a FUSED2 sweep without the arithmetic.
//
// Persistent CTAs (one per SM) march along x over bands of 128 rows of a SoA
// lattice (37 population planes, column pitch ly + 12), exactly like
// k_step2_split: per column, 37 one-dimensional bulk copies of 1040 B (rows
// y0-3-cy .. y0+126-cy of column x-cx, 16-byte aligned) land in a shared-memory
// stage; 128 "producer" threads read the stage, 128 "consumer" threads store
// 37 x 122 doubles of the column x-4 (st.global.cs).  NST stages are kept in
// flight (the library kernel can afford one next to its 185 KB ring), and
// each iteration spins DELAY cycles to stand in for the two collides.
// Prints GB/s of algorithmic traffic (592 B per output site) per variant.
//
// Build: SRC=membench ./build.sh   Run: ./membench [lx ly]
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

constexpr int kNpop = 37, kBand = 128, kRows = 136;
__constant__ signed char c_cx[kNpop] = {0, -1, 0, 0, 1, -1, -1, 1, 1, -2, 0, 0, 2, -2, -2, -1, -1, 1, 1,
                                        2, 2, -2, -2, 2, 2, -3, 0, 0, 3, -3, -3, -1, -1, 1, 1, 3, 3};
__constant__ signed char c_cy[kNpop] = {0, 0, -1, 1, 0, -1, 1, -1, 1, 0, -2, 2, 0, -1, 1, -2, 2, -2, 2,
                                        -1, 1, -2, 2, -2, 2, 0, -3, 3, 0, -1, 1, -3, 3, -3, 3, -1, 1};

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__constant__ int c_gs[8] = {0, 3, 8, 15, 22, 29, 34, 37};
__constant__ int c_slot[kNpop];  // cx-sorted position of population p (MODE 11)

// MODE 0: SoA planes (the library's FUSED2 store): element (p, x, y) at p*plane + x*cs + y.
// MODE 2: SoA reads, band-blocked writes.  MODE 3: band-blocked reads, SoA writes.
// MODE 9: exact 120-row blocks; the 6-row halos read straight from the neighbouring blocks (per
//         population, 48 B each: 7 group copies + 74 small copies per column), exact writes.
// MODE 8: exact 120-row blocks plus separate halo arrays LO/HI[x][b][s][8] (contiguous per column):
//         21 copies per column (main, lo, hi of each cx group), halo copies written as contiguous runs.
// MODE 5: MODE 4 without the halo copies.  MODE 6: MODE 4 reads, MODE 1 writes.
// MODE 4: the library's banded store (csrc/d2q37_banded.cu): blocks of 37 x 136 rows, 7 copies per
//         column (one per cx group), writes of the 120 own rows plus 8-row halo copies.
// MODE 1: band-blocked: element (p, x, y) of band b at ((x*nb + b)*37 + p)*kOut + y - y0 -- one
//         column's 37 populations x kOut rows contiguous (reads approximate: each population's
//         1040 B taken from inside its own block).
template <int NST, int MODE, int kOut>
__global__ void __launch_bounds__(256, 1) k_mem(const double* __restrict__ src, double* __restrict__ dst, int lx,
                                                int ly, long long cs, long long plane, int nbands, long long per_cta,
                                                int delay, unsigned long long* waitcyc, int lock) {
    extern __shared__ double sm[];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + NST * kNpop * kRows);
    const bool prod = threadIdx.x < kBand;
    const int tid = threadIdx.x & 127, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < NST) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar + threadIdx.x)));
    asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int ip = MODE == 9 ? warp * 32 + lane : MODE == 8 ? lane : (MODE >= 4) ? 2 * warp + lane : warp * 10 + lane;
    const bool issuer = MODE == 9 ? (prod && ip < 7 + 2 * kNpop)
                      : MODE == 8 ? (prod && warp < 3 && lane < 7)
                                  : (MODE >= 4) ? (prod && lane < 2 && ip < 7) : (prod && lane < 10 && ip < kNpop);
    const long long hsz = (long long)(lx + 8) * nbands * kNpop * 8;  // one halo array (doubles)
    const long long mainsz = (long long)(lx + 8) * nbands * kNpop * 120;
    const int icx = (MODE >= 4) ? ip - 3 : (issuer ? c_cx[ip] : 0), icy = (MODE >= 4) ? 0 : (issuer ? c_cy[ip] : 0);
    // lock: CTA b marches band b over every column (lockstep: neighbouring bands at the same columns)
    long long item = lock ? (long long)blockIdx.x * lx : (long long)blockIdx.x * per_cta;
    const long long end = min((long long)nbands * lx, item + (lock ? lx : per_cta));
    unsigned ph[NST > 0 ? NST : 1] = {};
    unsigned long long waited = 0;
    double acc = 0.0;
    int issued = 0, used = 0;
    while (item < end) {
        const int band = (int)(item / lx), xs = (int)(item % lx);
        const int xe = (int)min((long long)lx, xs + (end - item));
        item += xe - xs;
        const int y0 = band * kOut;
        const int niter = xe - xs + 7;
        auto wr = [&](int v) { return v < 0 ? v + lx : (v >= lx ? v - lx : v); };
        auto issue = [&](int t) {
            const int st = issued % NST;
            if (issuer && MODE == 9) {
                const int k = ip < 7 ? ip : (ip - 7) % kNpop;  // group (main) or population (halo)
                const int cxk = ip < 7 ? k - 3 : c_cx[k];
                const int col = wr(wr(xs - 3 + t) - cxk);
                const long long blk = (long long)col * nbands + band;
                const double* s;
                double* d;
                unsigned bytes;
                if (ip < 7) {
                    const int gs = c_gs[k], gn = c_gs[k + 1] - gs;
                    s = src + (blk * kNpop + gs) * 120;
                    d = sm + st * kNpop * kRows + gs * 120;
                    bytes = gn * 120 * 8;
                } else {
                    const bool lo = ip - 7 < kNpop;
                    const long long nb = lo ? (band > 0 ? blk - 1 : blk) : (band + 1 < nbands ? blk + 1 : blk);
                    s = src + (nb * kNpop + k) * 120 + (lo ? 114 : 0);
                    d = sm + st * kNpop * kRows + kNpop * 120 + (lo ? 0 : kNpop * 6) + k * 6;
                    bytes = 48;
                }
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa(d)),
                    "l"(s), "r"(bytes), "r"(sa(bar + st))
                    : "memory");
            } else if (issuer && MODE == 8) {
                const int col = wr(wr(xs - 3 + t) - icx);
                const int gs = c_gs[ip], gn = c_gs[ip + 1] - gs;
                const long long blk = (long long)col * nbands + band;
                const double* s = warp == 0 ? src + (blk * kNpop + gs) * 120
                                            : src + mainsz + (warp - 1) * hsz + (blk * kNpop + gs) * 8;
                double* d = sm + st * kNpop * kRows + (warp == 0 ? gs * 120 : kNpop * 120 + (warp - 1) * kNpop * 8 + gs * 8);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa(d)),
                    "l"(s), "r"(gn * (warp == 0 ? 120 : 8) * 8), "r"(sa(bar + st))
                    : "memory");
            } else if (issuer && MODE >= 4) {
                const int col = wr(wr(xs - 3 + t) - icx);
                const int gs = c_gs[ip], gn = c_gs[ip + 1] - gs;
                const double* s = src + (((long long)col * nbands + band) * kNpop + gs) * 136;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa(sm + st * kNpop * kRows + gs * 136)),
                    "l"(s), "r"(gn * 136 * 8), "r"(sa(bar + st))
                    : "memory");
            } else if (issuer) {
                const int col = wr(wr(xs - 3 + t) - icx);
                const double* s = (MODE == 0 || MODE == 2) ? src + ip * plane + col * cs + ((y0 + 3 - icy) & ~1)
                                  : (MODE >= 10) ? src + ((long long)col * kNpop + (MODE == 11 ? c_slot[ip] : ip)) * cs +
                                                       ((y0 + 3 - icy) & ~1)
                                                 : src + (((long long)col * nbands + band) * kNpop + ip) * kOut;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa(sm + (st * kNpop + ip) * kRows)),
                    "l"(s), "r"(kRows * 8), "r"(sa(bar + st))
                    : "memory");
            }
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar + st)),
                             "r"(MODE == 9 ? kNpop * 132 * 8 : (MODE >= 4) ? kNpop * 136 * 8 : kNpop * kRows * 8)
                             : "memory");
            ++issued;
        };
        if (prod)
            for (int t = 0; t < NST && t < niter - 1; ++t) issue(t);
        for (int t = 0; t < niter; ++t) {
            if (prod && t < niter - 1) {
                const int st = used % NST;
                const long long c0 = clock64();
                asm volatile(
                    "{\n\t.reg .pred p;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra "
                    "W%=;\n}" ::"r"(sa(bar + st)),
                    "r"(ph[st])
                    : "memory");
                waited += clock64() - c0;
                ph[st] ^= 1;
                double v = 0.0;
#pragma unroll
                for (int p = 0; p < kNpop; ++p) v += sm[(st * kNpop + p) * kRows + tid + 1];
                acc += v;
                ++used;
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (t + NST < niter - 1) issue(t + NST);
            }
            if (!prod && t >= 7 && tid < kOut && xs - 7 + t < lx) {
                if (MODE == 0 || MODE == 3) {
                    double* o = dst + (long long)(xs - 7 + t) * cs + y0 + (kOut == 120 ? 4 : 6) + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + p * plane, acc + p);
                } else if (MODE >= 10) {  // column-major [x][p][y] (11: populations sorted by cx)
                    double* o = dst + (long long)(xs - 7 + t) * kNpop * cs + y0 + 4 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + (long long)(MODE == 11 ? c_slot[p] : p) * cs, acc + p);
                } else if (MODE == 8) {
                    const long long blk = (long long)(xs - 7 + t) * nbands + band;
                    double* o = dst + blk * kNpop * 120 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + p * 120, acc + p);
                    if ((tid < 8 && band > 0) || (tid >= 112 && band + 1 < nbands)) {
                        double* oo = tid < 8 ? dst + mainsz + hsz + ((blk - 1) * kNpop) * 8 + tid
                                             : dst + mainsz + ((blk + 1) * kNpop) * 8 + tid - 112;
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) __stcs(oo + p * 8, acc + p);
                    }
                } else if (MODE == 4 || MODE == 5) {  // 5: no halo copies
                    double* o = dst + ((long long)(xs - 7 + t) * nbands + band) * kNpop * 136 + 8 + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + p * 136, acc + p);
                    if (MODE == 4 && ((tid < 8 && band > 0) || (tid >= 112 && band + 1 < nbands))) {
                        double* oo = o + (tid < 8 ? -kNpop * 136 + 120 : kNpop * 136 - 120);
#pragma unroll
                        for (int p = 0; p < kNpop; ++p) __stcs(oo + p * 136, acc + p);
                    }
                } else {
                    double* o = dst + ((long long)(xs - 7 + t) * nbands + band) * kNpop * kOut + tid;
#pragma unroll
                    for (int p = 0; p < kNpop; ++p) __stcs(o + p * kOut, acc + p);
                }
            }
            const long long c1 = clock64();
            while (clock64() - c1 < delay) {
            }
            __syncthreads();
        }
    }
    if (acc == 12345.678) dst[0] = acc;
    if (threadIdx.x == 0) atomicAdd(waitcyc, waited);
}

int main(int argc, char** argv) {
    const int lx = argc > 1 ? atoi(argv[1]) : 4096, ly = argc > 2 ? atoi(argv[2]) : 16384;
    const long long cs = ly + 12 + 128, plane = (long long)(lx + 8) * cs;  // padded like the lattice
    const size_t bytes = std::max((size_t)plane * kNpop * 8, (size_t)(lx + 8) * (ly / 120 + 2) * kNpop * 136 * 8);
    double *a, *b;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes));
    unsigned long long* wc;
    CK(cudaMalloc(&wc, 8));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));

    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](auto kern, int nst, int delay, int kOut, int mode, int lock = 0) {
        const int nbands = ly / kOut - 1;
        const long long items = (long long)nbands * lx, per = (items + nsm - 1) / nsm;
        const int smem = nst * kNpop * kRows * 8 + 64;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
            CK(cudaMemset(wc, 0, 8));
            CK(cudaEventRecord(e0));
            kern<<<lock ? std::min(nbands, nsm) : nsm, 256, smem>>>(a + 8, b + 8, lx, ly, cs, plane, nbands, per, delay, wc, lock);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (r) best = ms < best ? ms : best;
        }
        unsigned long long w = 0;
        CK(cudaMemcpy(&w, wc, 8, cudaMemcpyDeviceToHost));
        const double sites = (double)nbands * kOut * lx;
        printf("lock %d mode %d out %d stages %d delay %5d: %7.3f ms  %7.1f GB/s algorithmic (592 B/site)  %6.2f ns/column  producer wait "
               "%.1f%%\n",
               lock, mode, kOut, nst, delay, best, sites * 592 / (best * 1e6), best * 1e6 / (double)(per + 7),
               100.0 * w / (double)nsm / ((double)best * 1e-3 * 1.9e9));
    };
    // round 2: which side of the SoA stream costs -- reads (modes 0 / 2) or writes (0 / 3) -- in lockstep
    {
        int slot[kNpop];
        signed char cx[kNpop];
        CK(cudaMemcpyFromSymbol(cx, c_cx, sizeof cx));
        for (int p = 0; p < kNpop; ++p) {
            int n = 0;
            for (int q = 0; q < kNpop; ++q) n += (cx[q] < cx[p]) || (cx[q] == cx[p] && q < p);
            slot[p] = n;
        }
        CK(cudaMemcpyToSymbol(c_slot, slot, sizeof slot));
    }
    for (int lock : {1, 0}) {
        run(k_mem<2, 10, 120>, 2, 0, 120, 10, lock);
        run(k_mem<2, 11, 120>, 2, 0, 120, 11, lock);
        run(k_mem<2, 0, 120>, 2, 0, 120, 0, lock);
        run(k_mem<2, 2, 120>, 2, 0, 120, 2, lock);
        run(k_mem<2, 1, 120>, 2, 0, 120, 1, lock);
    }
    return 0;
}
