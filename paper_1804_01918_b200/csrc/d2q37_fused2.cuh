// d2q37_fused2.cuh -- shared pieces of the two-steps-per-sweep kernels
// (d2q37_step2.cu on the SoA store, d2q37_banded.cu on the band-blocked store):
// the step-1 ring geometry, a compile-time population loop and the
// bulk-copy / mbarrier PTX wrappers.
#pragma once

#include <cuda_runtime.h>

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
D2Q37_HD constexpr int ybar_of(int p) { return vel_index(cx_of(p), -cy_of(p)); }

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

}  // namespace

}  // namespace d2q37
