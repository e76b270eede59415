// tb2x.cu -- temporal-blocking probe: split roles in time instead of warps.
//
// Every warp is a producer, then a consumer, in each march iteration: warps 0-3
// own populations {0..12, 25..28} (half 0), warps 4-7 the rest (half 1) of the
// same 128 rows; the halves exchange partial moment sums through shared memory
// (pairwise named barrier).  Phases are serialized by __syncthreads, so the
// ring depth is cx+4 (148 population columns = 151.5 KB: the 164 KB carveout,
// ~92 KB of L1).  Layout: canonical SoA (p*lx + x)*ly + y, periodic.
// Bit-exact against k_ref (collide_split order) by construction.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "d2q37_b200.h"
#include "d2q37_device.cuh"

using namespace d2q37;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ int wrap(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

__host__ __device__ __forceinline__ long long idx(int p, int x, int y, int lx, int ly) {
    return ((long long)p * lx + x) * ly + y;  // canonical population-major SoA
}

D2Q37_HD constexpr bool in_half(int p, int h) { return ((p <= 12) || (p >= 25 && p <= 28)) == (h == 0); }

struct Part {
    double rho, jx, jy, e2;
};

template <int H>
__device__ __forceinline__ Part half_sums(const double (&f)[kNpop]) {
    Part s{0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < kNpop; ++i)
        if (in_half(i, H)) s.rho += f[i];
#pragma unroll
    for (int i = 0; i < kNpop; ++i)
        if (in_half(i, H) && cx_of(i) != 0) s.jx = fma((double)cx_of(i), f[i], s.jx);
#pragma unroll
    for (int i = 0; i < kNpop; ++i)
        if (in_half(i, H) && cy_of(i) != 0) s.jy = fma((double)cy_of(i), f[i], s.jy);
#pragma unroll
    for (int i = 0; i < kNpop; ++i)
        if (in_half(i, H) && (cx_of(i) != 0 || cy_of(i) != 0))
            s.e2 = fma((double)(cx_of(i) * cx_of(i) + cy_of(i) * cy_of(i)), f[i], s.e2);
    return s;
}

__device__ __forceinline__ void moments(const Part& a, const Part& b, const ModelParams& mp, double& rho,
                                        double (&mom)[kNmom]) {
    rho = a.rho + b.rho;
    const double jx = a.jx + b.jx, jy = a.jy + b.jy, e2 = a.e2 + b.e2;
    const double inv_rho = 1.0 / rho;
    const double ux = jx * inv_rho;
    const double uy = jy * inv_rho;
    const double temp = 0.5 * (e2 * inv_rho - (ux * ux + uy * uy));
    const double dt = temp - mp.t0;
    const double ux2 = ux * ux, uy2 = uy * uy, uxuy = ux * uy;
    const double dt3 = 3.0 * dt, dt6 = 6.0 * dt, dt2 = dt * dt, dt2x3 = 3.0 * dt2;
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
}

template <int H>
__device__ __forceinline__ void half_relax(double (&f)[kNpop], const double (&mom)[kNmom], const ModelParams& mp,
                                           double rho, double omega) {
    if (H == 0) {
        const double* g = mp.eq[0];
        double ee = fma(g[2], mom[2], 1.0);
        ee = fma(g[4], mom[4], ee);
        ee = fma(g[9], mom[9], ee);
        ee = fma(g[11], mom[11], ee);
        ee = fma(g[13], mom[13], ee);
        f[0] = fma(omega, fma(rho * mp.w[0], ee, -f[0]), f[0]);
        eq_axis<1>(f, mom, mp, rho, omega);
        eq_axis<2>(f, mom, mp, rho, omega);
        eq_axis<3>(f, mom, mp, rho, omega);
        eq_quad<1, 1>(f, mom, mp, rho, omega);
    } else {
        eq_quad<2, 1>(f, mom, mp, rho, omega);
        eq_quad<1, 2>(f, mom, mp, rho, omega);
        eq_quad<2, 2>(f, mom, mp, rho, omega);
        eq_quad<3, 1>(f, mom, mp, rho, omega);
        eq_quad<1, 3>(f, mom, mp, rho, omega);
    }
}

// Whole-site collide with the split summation order (one thread).
__device__ __forceinline__ void collide_split(double (&f)[kNpop], double omega, const ModelParams& mp) {
    const Part a = half_sums<0>(f), b = half_sums<1>(f);
    double rho, mom[kNmom];
    moments(a, b, mp, rho, mom);
    half_relax<0>(f, mom, mp, rho, omega);
    half_relax<1>(f, mom, mp, rho, omega);
}

__global__ void __launch_bounds__(128, 4) k_ref(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                int ly, ModelParams mp, double omega) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x, x = blockIdx.y;
    if (y >= ly) return;
    double f[kNpop];
#pragma unroll
    for (int p = 0; p < kNpop; ++p) f[p] = __ldg(in + idx(p, wrap(x - cx_of(p), lx), wrap(y - cy_of(p), ly), lx, ly));
    collide_split(f, omega, mp);
#pragma unroll
    for (int p = 0; p < kNpop; ++p) __stcs(out + idx(p, x, y, lx, ly), f[p]);
}

D2Q37_HD constexpr int depth_of(int p) { return cx_of(p) + 4; }
D2Q37_HD constexpr int ring_base(int p) {
    int s = 0;
    for (int q = 0; q < p; ++q) s += depth_of(q);
    return s;
}
constexpr int kRingCols = ring_base(kNpop);  // 148

template <typename F, int... Ps>
__device__ __forceinline__ void for_pops_(F&& f, std::integer_sequence<int, Ps...>) {
    (f(std::integral_constant<int, Ps>{}), ...);
}
template <typename F>
__device__ __forceinline__ void for_pops(F&& f) {
    for_pops_(f, std::make_integer_sequence<int, kNpop>{});
}

__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

constexpr int NB = 128;

template <int H>
__device__ __forceinline__ void run_half(const double* __restrict__ in, double* __restrict__ out, double* ring,
                                         double* xch, int lx, int ly, const ModelParams& mp, double omega, int xs,
                                         int xe, int y0, int ny, int site, int pair) {
    const long long plane = (long long)lx * ly;
    const int niter = xe - xs + 6;
    const int y1 = wrap(y0 - 3 + site, ly);
    auto wr = [](int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); };
    auto load = [&](double(&v)[kNpop], int r) {
#pragma unroll
        for (int p = 0; p < kNpop; ++p)
            if (in_half(p, H)) v[p] = __ldg(in + p * plane + (long long)wr(wr(r, lx) - cx_of(p), lx) * ly + wr(y1 - cy_of(p), ly));
    };
    auto exchange = [&](const Part& mine, double& rho, double (&mom)[kNmom]) {
        double* xs_ = xch + H * 4 * NB + site;
        xs_[0] = mine.rho;
        xs_[NB] = mine.jx;
        xs_[2 * NB] = mine.jy;
        xs_[3 * NB] = mine.e2;
        bar_named(1 + pair, 64);
        const double* xo = xch + (1 - H) * 4 * NB + site;
        const Part other{xo[0], xo[NB], xo[2 * NB], xo[3 * NB]};
        if (H == 0)
            moments(mine, other, mp, rho, mom);
        else
            moments(other, mine, mp, rho, mom);
    };
    auto body = [&](double(&f)[kNpop], double(&fn)[kNpop], int t) {
        const int r = xs - 3 + t;
        {  // producer phase: step 1 of column r, own populations
            double rho, mom[kNmom];
            exchange(half_sums<H>(f), rho, mom);
            if (t + 1 < niter) load(fn, r + 1);
            half_relax<H>(f, mom, mp, rho, omega);
            for_pops([&](auto P) {
                constexpr int p = decltype(P)::value, rb = ring_base(p), dp = depth_of(p);
                if (in_half(p, H)) ring[(rb + t % dp) * NB + site] = f[p];
            });
        }
        __syncthreads();
        if (t >= 6) {  // consumer phase: step 2 of column r - 3, own populations
            double g[kNpop];
            for_pops([&](auto P) {
                constexpr int p = decltype(P)::value, rb = ring_base(p), dp = depth_of(p);
                if (in_half(p, H)) g[p] = ring[(rb + (t + 1) % dp) * NB + site + 3 - cy_of(p)];
            });
            double rho, mom[kNmom];
            exchange(half_sums<H>(g), rho, mom);
            half_relax<H>(g, mom, mp, rho, omega);
            if (site < ny) {
                const long long e = (long long)(r - 3) * ly + y0 + site;
#pragma unroll
                for (int p = 0; p < kNpop; ++p)
                    if (in_half(p, H)) __stcs(out + p * plane + e, g[p]);
            }
        }
        __syncthreads();
    };
    double fa[kNpop], fb[kNpop];
    load(fa, xs - 3);
    int t = 0;
#pragma unroll 1
    for (; t + 1 < niter; t += 2) {
        body(fa, fb, t);
        body(fb, fa, t + 1);
    }
    if (t < niter) body(fa, fb, t);
}

__global__ void __launch_bounds__(2 * NB, 1) k_tb2x(const double* __restrict__ in, double* __restrict__ out, int lx,
                                                    int ly, ModelParams mp, double omega, int nbands, long long per_cta) {
    constexpr int W = NB - 6;
    extern __shared__ double ring[];
    double* xch = ring + kRingCols * NB;  // [2 halves][4 sums][NB]
    const int h = threadIdx.x / NB;
    const int site = threadIdx.x % NB;
    const int pair = (threadIdx.x / 32) & 3;
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
        if (h == 0)
            run_half<0>(in, out, ring, xch, lx, ly, mp, omega, xs, xe, y0, ny, site, pair);
        else
            run_half<1>(in, out, ring, xch, lx, ly, mp, omega, xs, xe, y0, ny, site, pair);
    }
}

__global__ void k_init(double* f, int lx, int ly, unsigned long long seed, const double* w) {
    const long long n = (long long)lx * ly;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n; s += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(s / ly), y = (int)(s % ly);
        for (int p = 0; p < kNpop; ++p) {
            unsigned long long z = ((s * kNpop + p) + 1) * 0x9E3779B97F4A7C15ull ^ seed;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            f[idx(p, x, y, lx, ly)] = w[p] * (1.0 + 0.02 * ((z >> 11) * 0x1.0p-53 - 0.5));
        }
    }
}

__global__ void k_cmp(const double* a, const double* b, long long n, unsigned long long* nd) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += __double_as_longlong(a[i]) != __double_as_longlong(b[i]);
    if (c) atomicAdd(nd, c);
}

int main(int argc, char** argv) {
    const int lx = argc > 1 ? atoi(argv[1]) : 4096;
    const int ly = argc > 2 ? atoi(argv[2]) : 16384;
    const int reps = argc > 3 ? atoi(argv[3]) : 10;
    const double omega = 0.8;
    d2q37_model m;
    if (d2q37_model_d2q37(&m) != 0) return 1;
    ModelParams mp{};
    for (int i = 0; i < kNpop; ++i) {
        for (int k = 0; k < kNmom; ++k) mp.eq[i][k] = m.eq[i * kNmom + k];
        mp.w[i] = m.w[i];
    }
    mp.t0 = m.t0;
    const long long S = (long long)lx * ly, n = S * kNpop;
    double *a, *b, *c, *d, *w;
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&b, n * 8));
    CK(cudaMalloc(&c, n * 8));
    CK(cudaMalloc(&d, n * 8));
    CK(cudaMalloc(&w, kNpop * 8));
    CK(cudaMemcpy(w, m.w, kNpop * 8, cudaMemcpyHostToDevice));
    unsigned long long* nd;
    CK(cudaMalloc(&nd, 8));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    k_init<<<4096, 256>>>(a, lx, ly, 12345, w);
    dim3 rg((ly + 127) / 128, lx);
    auto ref2 = [&]() {
        k_ref<<<rg, 128>>>(a, b, lx, ly, mp, omega);
        k_ref<<<rg, 128>>>(b, c, lx, ly, mp, omega);
    };
    const size_t smem = (size_t)(kRingCols + 8) * NB * 8;
    CK(cudaFuncSetAttribute(k_tb2x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int W = NB - 6;
    const int nbands = (ly + W - 1) / W;
    const int grid = nsm;
    const long long per_cta = ((long long)nbands * lx + grid - 1) / grid;
    auto tb2 = [&]() { k_tb2x<<<grid, 2 * NB, smem>>>(a, d, lx, ly, mp, omega, nbands, per_cta); };
    if (getenv("TB2_PROF")) {
        tb2();
        CK(cudaDeviceSynchronize());
        return 0;
    }
    ref2();
    tb2();
    CK(cudaGetLastError());
    CK(cudaMemset(nd, 0, 8));
    k_cmp<<<4096, 256>>>(c, d, n, nd);
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, nd, 8, cudaMemcpyDeviceToHost));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](auto&& fn) {
        fn();
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) fn();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms / reps;
    };
    const double tr = timeit(ref2), tt = timeit(tb2);
    printf("split roles: ref %.3f ms/2 steps = %.0f MLUPS | tb2x %.3f ms = %.0f MLUPS (%.2fx) | bit-exact %s (%llu)\n",
           tr, 2.0 * S / (tr * 1e3), tt, 2.0 * S / (tt * 1e3), tr / tt, h ? "NO" : "yes", h);
    return h ? 2 : 0;
}
