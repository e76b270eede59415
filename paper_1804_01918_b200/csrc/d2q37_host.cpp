// d2q37_host.cpp -- host side of the product: the D2Q37 velocity model and the
// lattice initialisers (pure C++, no CUDA).
//
//   d2q37_model_d2q37  <- VelocityModel::d2q37() (model.hpp:52, model.cpp:81-240):
//                         velocity set, the quadrature's shell weights + t0 (a
//                         constant table), Hermite table folded with 1/(n! t0^n).
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

// The D2Q37 quadrature (VelocityModel::d2q37, model.cpp:101-181 derives it at
// run time): shell weights w_s and the lattice temperature t0 for which the
// lattice moments sum_i w_i cx^a cy^b equal those of a 2-D Gaussian of
// variance t0 for (a, b) in {(0,0) (2,0) (4,0) (2,2) (6,0) (4,2) (6,2) (4,4)
// (8,0)}, with sum_i w_i = 1.  The library ships the solution as a constant
// table (round-to-nearest, no FMA contraction: identical to the oracle's
// restatement, within 16 ulp of the reference's FMA build) instead of
// re-deriving it; tests/test_host.py checks the moment residuals (< 1e-12),
// the positivity and the reference's frozen values (test_model.cpp:87-142).
// The lattice arithmetic takes the constants of the caller's model anyway
// (d2q37_set_model: e.g. the reference's own VelocityModel).
constexpr double kT0 = 0x1.655a23486b0eap-1;  // 0.6979533220196832
constexpr int kShells = 8;
constexpr int kShellNorms[kShells] = {0, 1, 2, 4, 5, 8, 9, 10};  // |c|^2 of each shell
constexpr double kShellW[kShells] = {
    0x1.dd7e1917b635fp-3,   // |c|^2 = 0   0.23315066913235236
    0x1.b786979d5dd9fp-4,   //         1   0.10730609154221903
    0x1.d86a448815fd4p-5,   //         2   0.05766785988879489
    0x1.d19327de15f20p-7,   //         4   0.014208216158450748
    0x1.5ed142641e9dap-8,   //         5   0.005353049000513777
    0x1.0945fb76e9ba7p-10,  //         8   0.0010119375926735759
    0x1.01377e453341cp-12,  //         9   0.00024530102775771763
    0x1.292e6f2a5028ep-12,  //        10   0.00028341425299419846
};

double shell_weight(int n2) {
    for (int s = 0; s < kShells; ++s)
        if (kShellNorms[s] == n2) return kShellW[s];
    throw std::runtime_error("velocity outside the D2Q37 shells");
}

}  // namespace

void build_model(d2q37_model* m) {
    std::memset(m, 0, sizeof *m);
    for (int p = 0; p < kNpop; ++p) {
        m->cx[p] = cx_of(p);
        m->cy[p] = cy_of(p);
    }
    const double t0 = kT0;
    m->t0 = t0;
    for (int i = 0; i < kNpop; ++i) {
        m->w[i] = shell_weight(m->cx[i] * m->cx[i] + m->cy[i] * m->cy[i]);
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

// Host per-site verbs of VelocityModel (model.hpp:60-72) in the reference's
// operation order: macros_of (model.cpp:242-257: four separate reductions in
// population order) and collide_site (model.cpp:293-298).  Returns false when
// !(rho > 0) (NonPhysicalError).
bool host_macros(const d2q37_model& m, const double* f, double out[4]) {
    double rho = 0.0;
    for (int i = 0; i < kNpop; ++i) rho += f[i];
    if (!(rho > 0.0)) return false;
    double jx = 0.0, jy = 0.0, e2 = 0.0;
    for (int i = 0; i < kNpop; ++i) jx += double(m.cx[i]) * f[i];
    for (int i = 0; i < kNpop; ++i) jy += double(m.cy[i]) * f[i];
    for (int i = 0; i < kNpop; ++i) e2 += double(m.cx[i] * m.cx[i] + m.cy[i] * m.cy[i]) * f[i];
    const double inv_rho = 1.0 / rho;
    const double ux = jx * inv_rho, uy = jy * inv_rho;
    out[0] = rho;
    out[1] = ux;
    out[2] = uy;
    out[3] = 0.5 * (e2 * inv_rho - (ux * ux + uy * uy));
    return true;
}

bool host_collide_site(const d2q37_model& m, const double* f, double omega, double* out) {
    double mac[4], feq[kNpop];
    if (!host_macros(m, f, mac)) return false;
    host_equilibrium(m, mac[0], mac[1], mac[2], mac[3], feq);
    for (int i = 0; i < kNpop; ++i) out[i] = f[i] + omega * (feq[i] - f[i]);
    return true;
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
