// d2q37_host.cpp -- host side of the product: the D2Q37 velocity model and the
// lattice initialisers (pure C++, no CUDA).
//
//   d2q37_model_d2q37  <- VelocityModel::d2q37() (model.hpp:52, model.cpp:81-240):
//                         velocity set, moment-matched shell weights + t0,
//                         Hermite table folded with 1/(n! t0^n).
//   d2q37_make_lattice <- make_random/equilibrium/shear_lattice (lattice.cpp:8-47)
//                         and the BASELINE config 0-2 recipes.
//
// Compiled with -ffp-contract=off: the arithmetic order is the reference's, one
// IEEE op per source operation.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "d2q37_b200.h"
#include "d2q37_internal.h"
#include "d2q37_velocities.h"

namespace d2q37 {
namespace {

constexpr int kShells = 8;
constexpr std::array<int, kShells> kShellNorms = {0, 1, 2, 4, 5, 8, 9, 10};

int shell_of_norm(int n2) {
    for (int s = 0; s < kShells; ++s)
        if (kShellNorms[s] == n2) return s;
    return -1;
}

// Moment conditions E[x^a y^b] of a 2-D Gaussian with variance t0: the first
// eight determine the shell weights linearly, E[x^8] closes the system in t0.
struct Cond {
    int a, b;
};
constexpr std::array<Cond, kShells> kLinear = {{{0, 0}, {2, 0}, {4, 0}, {2, 2}, {6, 0}, {4, 2}, {6, 2}, {4, 4}}};
constexpr Cond kClosing = {8, 0};

double gaussian_moment(int k, double t0) {
    if (k % 2 != 0) return 0.0;
    double dfact = 1.0;
    for (int j = k - 1; j > 0; j -= 2) dfact *= j;
    return dfact * std::pow(t0, k / 2);
}

double int_pow(int base, int e) {
    double r = 1.0;
    for (int i = 0; i < e; ++i) r *= base;
    return r;
}

using Mat = std::array<std::array<double, kShells>, kShells>;
using Vec = std::array<double, kShells>;

Vec gauss_solve(Mat a, Vec b) {
    for (int col = 0; col < kShells; ++col) {
        int piv = col;
        for (int r = col + 1; r < kShells; ++r)
            if (std::abs(a[r][col]) > std::abs(a[piv][col])) piv = r;
        if (a[piv][col] == 0.0) throw std::runtime_error("singular moment system");
        std::swap(a[col], a[piv]);
        std::swap(b[col], b[piv]);
        for (int r = col + 1; r < kShells; ++r) {
            const double f = a[r][col] / a[col][col];
            for (int c = col; c < kShells; ++c) a[r][c] -= f * a[col][c];
            b[r] -= f * b[col];
        }
    }
    Vec x{};
    for (int r = kShells - 1; r >= 0; --r) {
        double s = b[r];
        for (int c = r + 1; c < kShells; ++c) s -= a[r][c] * x[c];
        x[r] = s / a[r][r];
    }
    return x;
}

struct Derived {
    Vec shell_w;
    double t0;
};

Derived derive(const int* cx, const int* cy) {
    auto shell_moment = [&](int s, int a, int b) {
        double acc = 0.0;
        for (int i = 0; i < kNpop; ++i)
            if (shell_of_norm(cx[i] * cx[i] + cy[i] * cy[i]) == s) acc += int_pow(cx[i], a) * int_pow(cy[i], b);
        return acc;
    };
    Mat a{};
    Vec closing{};
    for (int r = 0; r < kShells; ++r)
        for (int s = 0; s < kShells; ++s) a[r][s] = shell_moment(s, kLinear[r].a, kLinear[r].b);
    for (int s = 0; s < kShells; ++s) closing[s] = shell_moment(s, kClosing.a, kClosing.b);

    auto weights = [&](double t0) {
        Vec rhs{};
        for (int r = 0; r < kShells; ++r)
            rhs[r] = gaussian_moment(kLinear[r].a, t0) * gaussian_moment(kLinear[r].b, t0);
        return gauss_solve(a, rhs);
    };
    auto closing_residual = [&](double t0) {
        const Vec w = weights(t0);
        double r = -gaussian_moment(kClosing.a, t0) * gaussian_moment(kClosing.b, t0);
        for (int s = 0; s < kShells; ++s) r += closing[s] * w[s];
        return r;
    };
    auto population_sum = [&](const Vec& w) {
        double sum = 0.0;
        for (int i = 0; i < kNpop; ++i) sum += w[shell_of_norm(cx[i] * cx[i] + cy[i] * cy[i])];
        return sum;
    };

    // Scan t0 in (0.1, 2.0) for a sign change of the closing residual, bisect,
    // accept the first root with all-positive weights, then pin sum(w) == 1.
    const double lo0 = 0.1, hi0 = 2.0, dt = 1e-3;
    double t_prev = lo0, r_prev = closing_residual(lo0);
    for (double t = lo0 + dt; t < hi0; t += dt) {
        const double r = closing_residual(t);
        if (std::signbit(r) != std::signbit(r_prev)) {
            double lo = t_prev, hi = t, r_lo = r_prev;
            for (int it = 0; it < 200 && hi - lo > 1e-16; ++it) {
                const double mid = 0.5 * (lo + hi);
                const double rm = closing_residual(mid);
                if (std::abs(rm) < 1e-14) {
                    lo = hi = mid;
                    break;
                }
                if (std::signbit(rm) == std::signbit(r_lo)) {
                    lo = mid;
                    r_lo = rm;
                } else {
                    hi = mid;
                }
            }
            const double t0 = 0.5 * (lo + hi);
            Vec w = weights(t0);
            if (std::all_of(w.begin(), w.end(), [](double v) { return v > 0.0; })) {
                for (int pass = 0; pass < 4; ++pass) {
                    const double sum = population_sum(w);
                    if (sum == 1.0) break;
                    for (double& v : w) v /= sum;
                }
                for (int pass = 0; pass < 4; ++pass) {
                    const double sum = population_sum(w);
                    if (sum == 1.0) break;
                    w[0] -= sum - 1.0;  // rest weight enters no other moment condition
                }
                return {w, t0};
            }
        }
        t_prev = t;
        r_prev = r;
    }
    throw std::runtime_error("no all-positive D2Q37 quadrature for t0 in (0.1, 2.0)");
}

}  // namespace

void build_model(d2q37_model* m) {
    std::memset(m, 0, sizeof *m);
    for (int p = 0; p < kNpop; ++p) {
        m->cx[p] = cx_of(p);
        m->cy[p] = cy_of(p);
    }
    const Derived d = derive(m->cx, m->cy);
    const double t0 = d.t0;
    m->t0 = t0;
    for (int i = 0; i < kNpop; ++i) {
        m->w[i] = d.shell_w[shell_of_norm(m->cx[i] * m->cx[i] + m->cy[i] * m->cy[i])];
        const double cx = m->cx[i], cy = m->cy[i];
        const double cx2 = cx * cx, cy2 = cy * cy;
        const double t2 = t0 * t0, t3 = t2 * t0, t4 = t2 * t2;
        // Probabilists' Hermite tensors of variance t0 (model.cpp:200-232).
        const double h[kNmom] = {
            cx,
            cy,
            cx2 - t0,
            cx * cy,
            cy2 - t0,
            cx * cx2 - 3.0 * t0 * cx,
            cx2 * cy - t0 * cy,
            cx * cy2 - t0 * cx,
            cy * cy2 - 3.0 * t0 * cy,
            cx2 * cx2 - 6.0 * t0 * cx2 + 3.0 * t0 * t0,
            cx * cx2 * cy - 3.0 * t0 * cx * cy,
            cx2 * cy2 - t0 * (cx2 + cy2) + t0 * t0,
            cx * cy * cy2 - 3.0 * t0 * cx * cy,
            cy2 * cy2 - 6.0 * t0 * cy2 + 3.0 * t0 * t0,
        };
        // 1/(n! t0^n) times the tensor multiplicity.
        const double denom[kNmom] = {t0,       t0,       2.0 * t2, t2,       2.0 * t2, 6.0 * t3,  2.0 * t3,
                                     2.0 * t3, 6.0 * t3, 24.0 * t4, 6.0 * t4, 4.0 * t4, 6.0 * t4, 24.0 * t4};
        for (int k = 0; k < kNmom; ++k) m->eq[i * kNmom + k] = h[k] / denom[k];
    }
}

// Host equilibrium with the reference's operation order (model.cpp:259-291).
void host_equilibrium(const d2q37_model& m, double rho, double ux, double uy, double temp, double* f_eq) {
    const double dt = temp - m.t0;
    const double ux2 = ux * ux, uy2 = uy * uy, uxuy = ux * uy;
    const double dt3 = 3.0 * dt, dt6 = 6.0 * dt, dt2 = dt * dt, dt2x3 = 3.0 * dt2;
    const double mom[kNmom] = {ux,
                               uy,
                               ux2 + dt,
                               uxuy,
                               uy2 + dt,
                               ux * (ux2 + dt3),
                               uy * (ux2 + dt),
                               ux * (uy2 + dt),
                               uy * (uy2 + dt3),
                               ux2 * (ux2 + dt6) + dt2x3,
                               uxuy * (ux2 + dt3),
                               uxuy * uxuy + dt * (ux2 + uy2) + dt2,
                               uxuy * (uy2 + dt3),
                               uy2 * (uy2 + dt6) + dt2x3};
    for (int i = 0; i < kNpop; ++i) {
        const double* g = m.eq + i * kNmom;
        double s = 1.0;
        for (int k = 0; k < kNmom; ++k) s += g[k] * mom[k];
        f_eq[i] = rho * m.w[i] * s;
    }
}

void philox4x32_10(const uint32_t in[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {in[0], in[1], in[2], in[3]};
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t a = uint64_t(0xD2511F53u) * c[0];
        const uint64_t b = uint64_t(0xCD9E8D57u) * c[2];
        const uint32_t n[4] = {uint32_t(b >> 32) ^ c[1] ^ k0, uint32_t(b), uint32_t(a >> 32) ^ c[3] ^ k1, uint32_t(a)};
        std::memcpy(c, n, sizeof c);
    }
    std::memcpy(out, c, sizeof c);
}

double philox_u01(uint64_t seed, uint64_t counter) {
    const uint32_t ctr[4] = {uint32_t(counter), uint32_t(counter >> 32), 0u, 0u};
    const uint32_t key[2] = {uint32_t(seed), uint32_t(seed >> 32)};
    uint32_t r[4];
    philox4x32_10(ctr, key, r);
    const uint64_t bits = uint64_t(r[0]) | (uint64_t(r[1]) << 32);
    return double(bits >> 11) * 0x1.0p-53;
}

namespace {

template <class F>
void parallel_columns(int lx, int nthreads, F&& body) {
    if (nthreads <= 0) nthreads = int(std::max(1u, std::thread::hardware_concurrency()));
    nthreads = std::max(1, std::min(nthreads, lx));
    if (nthreads == 1) {
        body(0, lx);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) {
        const int x0 = int(long(lx) * t / nthreads), x1 = int(long(lx) * (t + 1) / nthreads);
        th.emplace_back([&, x0, x1] { body(x0, x1); });
    }
    for (auto& t : th) t.join();
}

inline size_t cidx(int lx, int ly, int p, int x, int y) { return (size_t(p) * lx + x) * ly + y; }

}  // namespace

// Draws per site follow the reference generator (lattice.cpp:8-23): a
// std::mt19937_64 stream consumed site by site in x-then-y order, mapped with
// (r >> 11) * 2^-53.  Draws are sequential; equilibrium evaluation is spread
// over column blocks.
void make_lattice(int kind, int lx, int ly, uint64_t seed, const double* params, const d2q37_model& m,
                  double* out, int nthreads) {
    const size_t sites = size_t(lx) * ly;
    auto u01 = [](std::mt19937_64& g) { return double(g() >> 11) * 0x1.0p-53; };
    switch (kind) {
        case D2Q37_INIT_EQUILIBRIUM: {
            double feq[kNpop];
            host_equilibrium(m, params[0], params[1], params[2], params[3], feq);
            parallel_columns(lx, nthreads, [&](int x0, int x1) {
                for (int p = 0; p < kNpop; ++p)
                    for (int x = x0; x < x1; ++x) std::fill_n(out + cidx(lx, ly, p, x, 0), ly, feq[p]);
            });
            return;
        }
        case D2Q37_INIT_SHEAR: {
            const double amp = params[0], temp = params[1];
            std::vector<double> rows(size_t(ly) * kNpop);
            for (int y = 0; y < ly; ++y)
                host_equilibrium(m, 1.0, amp * std::sin(2.0 * M_PI * y / ly), 0.0, temp, &rows[size_t(y) * kNpop]);
            parallel_columns(lx, nthreads, [&](int x0, int x1) {
                for (int p = 0; p < kNpop; ++p)
                    for (int x = x0; x < x1; ++x)
                        for (int y = 0; y < ly; ++y) out[cidx(lx, ly, p, x, y)] = rows[size_t(y) * kNpop + p];
            });
            return;
        }
        case D2Q37_INIT_PHILOX: {
            parallel_columns(lx, nthreads, [&](int x0, int x1) {
                for (int x = x0; x < x1; ++x)
                    for (int y = 0; y < ly; ++y)
                        for (int p = 0; p < kNpop; ++p)
                            out[cidx(lx, ly, p, x, y)] = philox_u01(seed, (uint64_t(x) * ly + y) * kNpop + p);
            });
            return;
        }
        case D2Q37_INIT_RT: {
            // Config 0: T = 1.5 below the interface y_int(x) = ly/2 + 0.01 ly sin(2 pi x/lx),
            // 0.5 above, + U(-1e-3, 1e-3) per site; rho = 1/T (uniform pressure); u = 0.
            // Optional params {ly_global, y0}: this array is rows [y0, y0+ly) of a
            // taller lattice (a y-slab); its noise then comes from the stream
            // seeded seed + y0 (slab-local), the interface from ly_global.
            const int lyg = params ? int(params[0]) : ly;
            const int y0 = params ? int(params[1]) : 0;
            std::vector<double> noise(sites);
            std::mt19937_64 g(seed + uint64_t(y0));
            for (size_t s = 0; s < sites; ++s) noise[s] = -1e-3 + 2e-3 * u01(g);
            parallel_columns(lx, nthreads, [&](int x0, int x1) {
                double feq[kNpop];
                for (int x = x0; x < x1; ++x) {
                    const double yint = 0.5 * lyg + 0.01 * lyg * std::sin(2.0 * M_PI * x / lx);
                    for (int y = 0; y < ly; ++y) {
                        const double temp = (double(y0 + y) < yint ? 1.5 : 0.5) + noise[size_t(x) * ly + y];
                        host_equilibrium(m, 1.0 / temp, 0.0, 0.0, temp, feq);
                        for (int p = 0; p < kNpop; ++p) out[cidx(lx, ly, p, x, y)] = feq[p];
                    }
                }
            });
            return;
        }
        case D2Q37_INIT_RANDOM:
        case D2Q37_INIT_C2: {
            // 4 field draws (rho, ux, uy, T: brace-init order, lattice.cpp:16-17)
            // then 37 multiplicative perturbations per site.  Streamed in column
            // blocks so the uniform buffer stays bounded.
            constexpr int kDraws = 4 + kNpop;
            const int block = std::max(1, int((size_t(1) << 24) / (size_t(ly) * kDraws)));
            std::vector<double> u(size_t(block) * ly * kDraws);
            std::mt19937_64 g(seed);
            for (int xb = 0; xb < lx; xb += block) {
                const int xe = std::min(lx, xb + block);
                const size_t n = size_t(xe - xb) * ly * kDraws;
                for (size_t i = 0; i < n; ++i) u[i] = u01(g);
                parallel_columns(xe - xb, nthreads, [&](int a, int b) {
                    double feq[kNpop];
                    for (int xo = a; xo < b; ++xo)
                        for (int y = 0; y < ly; ++y) {
                            const double* d = &u[(size_t(xo) * ly + y) * kDraws];
                            double rho, ux, uy, temp;
                            if (kind == D2Q37_INIT_RANDOM) {
                                rho = 0.9 + 0.2 * d[0];
                                ux = -0.05 + 0.1 * d[1];
                                uy = -0.05 + 0.1 * d[2];
                                temp = m.t0 * (0.9 + 0.2 * d[3]);
                            } else {
                                rho = 0.95 + 0.1 * d[0];
                                ux = -0.05 + 0.1 * d[1];
                                uy = -0.05 + 0.1 * d[2];
                                temp = 0.9 + 0.2 * d[3];
                            }
                            host_equilibrium(m, rho, ux, uy, temp, feq);
                            for (int p = 0; p < kNpop; ++p)
                                out[cidx(lx, ly, p, xb + xo, y)] = feq[p] * (1.0 + 2e-3 * (d[4 + p] - 0.5));
                        }
                });
            }
            return;
        }
        default:
            throw std::invalid_argument("unknown initialiser kind " + std::to_string(kind));
    }
}

}  // namespace d2q37
