// d2q37_velocities.h -- the D2Q37 velocity set, shared by host and device code.
#pragma once

#ifdef __CUDACC__
#define D2Q37_HD __host__ __device__
#else
#define D2Q37_HD
#endif

namespace d2q37 {

constexpr int kNpop = 37;
constexpr int kNmom = 14;
constexpr int kHalo = 3;

// Canonical D2Q37 velocity order (model.cpp:81-99: sorted by |c|^2, then cx,
// then cy).  Integer, build-independent; d2q37_set_model checks the caller's
// model against it.
D2Q37_HD constexpr int cx_of(int p) {
    constexpr int t[kNpop] = {0,  -1, 0,  0,  1,  -1, -1, 1,  1,  -2, 0,  0,  2,  -2, -2, -1, -1, 1, 1,
                              2,  2,  -2, -2, 2,  2,  -3, 0,  0,  3,  -3, -3, -1, -1, 1,  1,  3,  3};
    return t[p];
}
D2Q37_HD constexpr int cy_of(int p) {
    constexpr int t[kNpop] = {0,  0,  -1, 1,  0,  -1, 1,  -1, 1,  0,  -2, 2,  0,  -1, 1,  -2, 2, -2, 2,
                              -1, 1,  -2, 2,  -2, 2,  0,  -3, 3,  0,  -1, 1,  -3, 3,  -3, 3,  -1, 1};
    return t[p];
}
// Hermite coefficient k carries a factor cx (resp. cy): zero for cx == 0
// (resp. cy == 0) rows of the table (model.cpp:211-232).
D2Q37_HD constexpr bool mom_has_cx(int k) {
    return k == 0 || k == 3 || k == 5 || k == 7 || k == 10 || k == 12;
}
D2Q37_HD constexpr bool mom_has_cy(int k) {
    return k == 1 || k == 3 || k == 6 || k == 8 || k == 10 || k == 12;
}
D2Q37_HD constexpr bool eq_structural_zero(int i, int k) {
    return (cx_of(i) == 0 && mom_has_cx(k)) || (cy_of(i) == 0 && mom_has_cy(k));
}

}  // namespace d2q37
