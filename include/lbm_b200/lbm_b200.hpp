// lbm_b200.hpp -- C++ host API mirroring the reference lbmbench operator API
// (proj/include/lbm/{model,layout,dump,lattice,kernels,metrics}.hpp) on top of
// the C-ABI in d2q37_b200.h.  Header-only; link libd2q37_b200.so.
//
// Same verbs, argument meaning and error behaviour as the reference:
//   VelocityModel::d2q37()                  model.hpp:52
//   LatticeState{Descriptor}.load / dump    lattice.hpp:13-24
//   halo_exchange(state)                    kernels.hpp:29   (+ Boundary::Wall)
//   propagate(state)                        kernels.hpp:33   (prv -> nxt)
//   collide(state, model, omega)            kernels.hpp:40   (nxt -> prv)
//   step(state, model, omega)               kernels.hpp:45
//   run(state, model, in, out, omega, n)    load + n x step + dump in one (streamed) call
//   mlups / propagate_gbps / collide_gflops metrics.hpp:27-33
// Every verb blocks until the device work is done (the reference is
// synchronous); std::invalid_argument and NonPhysicalError are thrown where
// the reference throws them.  State lives in device memory (HBM); the
// ThreadPool / KernelOptions arguments of the reference have no counterpart.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "d2q37_b200.h"

namespace lbm_b200 {

inline constexpr int kNpop = D2Q37_NPOP;
inline constexpr int kHaloExtent = D2Q37_HALO;

struct NonPhysicalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == D2Q37_OK) return;
    const std::string msg = d2q37_last_error();
    switch (rc) {
        case D2Q37_ERR_NON_PHYSICAL: throw NonPhysicalError(msg);
        case D2Q37_ERR_INVALID_ARGUMENT:
        case D2Q37_ERR_UNSUPPORTED: throw std::invalid_argument(msg);
        case D2Q37_ERR_CUDA: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

// Banded: the device store of the two-step sweep (no reference counterpart; FUSED2 / FUSED steps,
// load / dump / files / convert only -- see d2q37_b200.h).
enum class LayoutKind { AoS = D2Q37_AOS, SoA = D2Q37_SOA, CSoA = D2Q37_CSOA, CAoSoA = D2Q37_CAOSOA, Banded = D2Q37_BANDED };
enum class Boundary { Periodic = D2Q37_BC_PERIODIC, Wall = D2Q37_BC_WALL };
enum class StepVariant { Unfused = D2Q37_UNFUSED, Fused = D2Q37_FUSED, Fused2 = D2Q37_FUSED2 };
enum class Math { Fast = D2Q37_MATH_FAST, Strict = D2Q37_MATH_STRICT };

struct IVec2 {
    int x = 0;
    int y = 0;
};

/// Per-site macroscopic fields (model.hpp:21-26).
struct Macros {
    double rho = 0.0;
    double ux = 0.0;
    double uy = 0.0;
    double temp = 0.0;
};

/// VelocityModel (model.hpp:50-100): the constants the kernels need.
class VelocityModel {
  public:
    static const VelocityModel& d2q37() {
        static const VelocityModel m = [] {
            VelocityModel v;
            check(d2q37_model_d2q37(&v.raw_));
            return v;
        }();
        return m;
    }
    /// From another VelocityModel's tables (e.g. the reference's own).
    static VelocityModel from_raw(const d2q37_model& raw) {
        VelocityModel v;
        v.raw_ = raw;
        return v;
    }
    IVec2 velocity(int i) const { return {raw_.cx[i], raw_.cy[i]}; }
    double weight(int i) const { return raw_.w[i]; }
    std::array<IVec2, kNpop> velocities() const {
        std::array<IVec2, kNpop> v{};
        for (int i = 0; i < kNpop; ++i) v[i] = velocity(i);
        return v;
    }
    std::array<double, kNpop> weights() const {
        std::array<double, kNpop> w{};
        for (int i = 0; i < kNpop; ++i) w[i] = raw_.w[i];
        return w;
    }
    double t0() const { return raw_.t0; }
    int halo_extent() const { return kHaloExtent; }
    const d2q37_model& raw() const { return raw_; }
    /// Per-site verbs (model.hpp:60-72), host arithmetic in the reference's order.
    Macros macros_of(const double* f) const {
        double m[4];
        check(d2q37_macros_of(&raw_, f, m));
        return {m[0], m[1], m[2], m[3]};
    }
    void equilibrium(const Macros& m, double* f_eq) const {
        const double mac[4] = {m.rho, m.ux, m.uy, m.temp};
        check(d2q37_equilibrium(&raw_, mac, f_eq));
    }
    void collide_site(const double* f, double omega, double* out) const {
        check(d2q37_collide_site(&raw_, f, omega, out));
    }
    static constexpr int kCollideFlopsPerSite = 1522;
    static constexpr int kEqMoments = D2Q37_NMOM;

  private:
    d2q37_model raw_{};
};

struct Geometry {
    int lx = 0;
    int ly = 0;
    int hx = kHaloExtent;
    int hy = kHaloExtent;
    int vl = 1;
};

/// CanonicalLattice (dump.hpp:13-24): index (p*lx + x)*ly + y.
struct CanonicalLattice {
    int lx = 0;
    int ly = 0;
    int npop = kNpop;
    std::vector<double> values;

    std::size_t index(int x, int y, int p) const { return (std::size_t(p) * lx + x) * ly + y; }
    double& at(int x, int y, int p) { return values[index(x, y, p)]; }
    double at(int x, int y, int p) const { return values[index(x, y, p)]; }
};

inline CanonicalLattice make_canonical(int lx, int ly) {
    CanonicalLattice c;
    c.lx = lx;
    c.ly = ly;
    c.values.assign(std::size_t(kNpop) * lx * ly, 0.0);
    return c;
}

/// make_random_lattice / make_equilibrium_lattice / make_shear_lattice (lattice.cpp:8-47).
inline CanonicalLattice make_random_lattice(int lx, int ly, std::uint64_t seed,
                                            const VelocityModel& m = VelocityModel::d2q37()) {
    CanonicalLattice c = make_canonical(lx, ly);
    check(d2q37_make_lattice(D2Q37_INIT_RANDOM, lx, ly, seed, nullptr, &m.raw(), c.values.data(), c.values.size(), 0));
    return c;
}
inline CanonicalLattice make_equilibrium_lattice(int lx, int ly, const VelocityModel& m, double rho, double ux,
                                                 double uy, double temp) {
    CanonicalLattice c = make_canonical(lx, ly);
    const double par[4] = {rho, ux, uy, temp};
    check(d2q37_make_lattice(D2Q37_INIT_EQUILIBRIUM, lx, ly, 0, par, &m.raw(), c.values.data(), c.values.size(), 0));
    return c;
}
inline CanonicalLattice make_shear_lattice(int lx, int ly, const VelocityModel& m, double amp, double temp) {
    CanonicalLattice c = make_canonical(lx, ly);
    const double par[2] = {amp, temp};
    check(d2q37_make_lattice(D2Q37_INIT_SHEAR, lx, ly, 0, par, &m.raw(), c.values.data(), c.values.size(), 0));
    return c;
}
/// BASELINE config-0 Rayleigh-Taylor-like init.
inline CanonicalLattice make_rt_lattice(int lx, int ly, std::uint64_t seed,
                                        const VelocityModel& m = VelocityModel::d2q37()) {
    CanonicalLattice c = make_canonical(lx, ly);
    check(d2q37_make_lattice(D2Q37_INIT_RT, lx, ly, seed, nullptr, &m.raw(), c.values.data(), c.values.size(), 0));
    return c;
}

/// LatticeState (lattice.hpp:13-24) resident in device memory: prv holds the
/// state between steps, nxt is the propagate target.
class LatticeState {
  public:
    LatticeState(LayoutKind kind, Geometry g, int device = 0) : geom_(g) {
        if (g.hx != kHaloExtent || g.hy != kHaloExtent)
            throw std::invalid_argument("halos narrower than the velocity reach");
        check(d2q37_create(int(kind), g.lx, g.ly, g.vl, device, &h_));
    }
    ~LatticeState() { d2q37_destroy(h_); }
    LatticeState(const LatticeState&) = delete;
    LatticeState& operator=(const LatticeState&) = delete;
    LatticeState(LatticeState&& o) noexcept : h_(std::exchange(o.h_, nullptr)), geom_(o.geom_) {}

    const Geometry& geom() const { return geom_; }
    d2q37_lattice* handle() const { return h_; }
    long time_step() const { return d2q37_time_step(h_); }

    void set_model(const VelocityModel& m) { check(d2q37_set_model(h_, &m.raw())); }
    void set_math(Math m) { check(d2q37_set_math(h_, int(m))); }

    void load(const CanonicalLattice& c) { load_into(0, c); }
    CanonicalLattice dump() const { return dump_from(0); }
    /// from_canonical / to_canonical on prv (0) or nxt (1) (dump.hpp:28-29).
    void load_into(int which, const CanonicalLattice& c) {
        if (c.lx != geom_.lx || c.ly != geom_.ly || c.npop != kNpop)
            throw std::invalid_argument("from_canonical: dimension mismatch");
        check(d2q37_load_buffer(h_, which, c.values.data(), c.values.size()));
    }
    CanonicalLattice dump_from(int which) const {
        CanonicalLattice c = make_canonical(geom_.lx, geom_.ly);
        check(d2q37_dump_buffer(h_, which, c.values.data(), c.values.size()));
        return c;
    }
    void sync() { check(d2q37_sync(h_)); }

  private:
    d2q37_lattice* h_ = nullptr;
    Geometry geom_;
};

/// convert(src, to) (layout.hpp:148, layout.cpp:105-116): a new device lattice
/// with layout `kind` / geometry `to` holding src's physical sites.
inline LatticeState convert(const LatticeState& src, LayoutKind kind, Geometry to, int device = 0) {
    if (to.lx != src.geom().lx || to.ly != src.geom().ly || to.hx != src.geom().hx || to.hy != src.geom().hy)
        throw std::invalid_argument("convert: geometry mismatch");
    LatticeState dst(kind, to, device);
    check(d2q37_convert(src.handle(), dst.handle()));
    return dst;
}

/// The scalar device reference of run_validation (validation.hpp:36-42):
/// nsteps of propagate then collide on a halo-free canonical array, periodic.
inline CanonicalLattice scalar_steps(const VelocityModel& m, const CanonicalLattice& in, double omega, int nsteps,
                                     Math math = Math::Fast, int device = 0) {
    CanonicalLattice out = make_canonical(in.lx, in.ly);
    check(d2q37_scalar_steps(&m.raw(), in.lx, in.ly, in.values.data(), out.values.data(), in.values.size(), omega,
                             nsteps, int(math), device));
    return out;
}

/// One lattice as P2P y-slabs on several GPUs of this process
/// (d2q37_create_multi): slab r holds rows [r*ly/n, (r+1)*ly/n) on devices[r].
/// load / dump take the whole canonical lattice; step advances every slab in
/// lockstep through the peer-memory halo protocol.
class MultiGpuLattice {
  public:
    MultiGpuLattice(LayoutKind kind, Geometry g, const std::vector<int>& devices) : geom_(g), h_(devices.size()) {
        if (g.hx != kHaloExtent || g.hy != kHaloExtent)
            throw std::invalid_argument("halos narrower than the velocity reach");
        check(d2q37_create_multi(int(kind), g.lx, g.ly, g.vl, int(devices.size()), devices.data(), h_.data()));
    }
    ~MultiGpuLattice() {
        for (d2q37_lattice* h : h_) d2q37_destroy(h);
    }
    MultiGpuLattice(const MultiGpuLattice&) = delete;
    MultiGpuLattice& operator=(const MultiGpuLattice&) = delete;

    int slabs() const { return int(h_.size()); }

    void load(const CanonicalLattice& c) {
        if (c.lx != geom_.lx || c.ly != geom_.ly) throw std::invalid_argument("from_canonical: dimension mismatch");
        const int n = slabs(), ny = geom_.ly / n;
        std::vector<double> part(size_t(kNpop) * geom_.lx * ny);
        for (int r = 0; r < n; ++r) {
            for (int p = 0; p < kNpop; ++p)
                for (int x = 0; x < geom_.lx; ++x)
                    for (int y = 0; y < ny; ++y)
                        part[(size_t(p) * geom_.lx + x) * ny + y] = c.values[(size_t(p) * geom_.lx + x) * geom_.ly + r * ny + y];
            check(d2q37_load_canonical(h_[r], part.data(), part.size()));
        }
    }
    CanonicalLattice dump() const {
        CanonicalLattice c = make_canonical(geom_.lx, geom_.ly);
        const int n = slabs(), ny = geom_.ly / n;
        std::vector<double> part(size_t(kNpop) * geom_.lx * ny);
        for (int r = 0; r < n; ++r) {
            check(d2q37_dump_canonical(h_[r], part.data(), part.size()));
            for (int p = 0; p < kNpop; ++p)
                for (int x = 0; x < geom_.lx; ++x)
                    for (int y = 0; y < ny; ++y)
                        c.values[(size_t(p) * geom_.lx + x) * geom_.ly + r * ny + y] = part[(size_t(p) * geom_.lx + x) * ny + y];
        }
        return c;
    }
    void step(const VelocityModel& m, double omega, int nsteps = 1, StepVariant variant = StepVariant::Fused,
              Boundary bc = Boundary::Periodic) {
        for (d2q37_lattice* h : h_) check(d2q37_set_model(h, &m.raw()));
        check(d2q37_multi_step(h_.data(), slabs(), omega, nsteps, int(variant), int(bc)));
    }

  private:
    Geometry geom_;
    std::vector<d2q37_lattice*> h_;
};

inline void halo_exchange(LatticeState& s, Boundary bc = Boundary::Periodic) {
    check(d2q37_bc(s.handle(), int(bc)));
    s.sync();
}

inline void propagate(LatticeState& s) {
    check(d2q37_propagate(s.handle()));
    s.sync();
}

inline void collide(LatticeState& s, const VelocityModel& m, double omega) {
    s.set_model(m);
    check(d2q37_collide(s.handle(), omega));
    s.sync();
}

inline void step(LatticeState& s, const VelocityModel& m, double omega, int nsteps = 1,
                 StepVariant variant = StepVariant::Fused, Boundary bc = Boundary::Periodic) {
    s.set_model(m);
    check(d2q37_step(s.handle(), omega, nsteps, int(variant), int(bc)));
    s.sync();
}

/// load(in) + step x nsteps + dump as one call (d2q37_run_canonical): the result of LatticeState::load,
/// nsteps x step (kernels.hpp:45) and LatticeState::dump (lattice.hpp:18-19), bit for bit.  On a single
/// SoA wall domain with StepVariant::Fused2 and an even nsteps the upload, the sweeps and the download
/// are pipelined in y-chunks, so the host copies hide under the sweeps.  `out` may be `in` itself.
inline void run(LatticeState& s, const VelocityModel& m, const CanonicalLattice& in, CanonicalLattice& out,
                double omega, int nsteps, StepVariant variant = StepVariant::Fused, Boundary bc = Boundary::Periodic) {
    if (in.lx != s.geom().lx || in.ly != s.geom().ly || in.npop != kNpop)
        throw std::invalid_argument("from_canonical: dimension mismatch");
    if (&out != &in) {
        out.lx = in.lx;
        out.ly = in.ly;
        out.npop = in.npop;
        out.values.resize(in.values.size());
    }
    s.set_model(m);
    check(d2q37_run_canonical(s.handle(), in.values.data(), out.values.data(), in.values.size(), omega, nsteps,
                              int(variant), int(bc)));
}

// metrics.cpp:50-63
inline double mlups(int lx, int ly, double t) {
    if (!(t > 0.0)) throw std::invalid_argument("iteration time must be positive");
    return double(lx) * ly / (t * 1e6);
}
inline double propagate_gbps(int lx, int ly, int npop, double t, bool nontemporal = true) {
    if (!(t > 0.0)) throw std::invalid_argument("iteration time must be positive");
    return double(lx) * ly * npop * 8.0 * (nontemporal ? 2 : 3) / (t * 1e9);
}
inline double collide_gflops(int lx, int ly, double flops_per_site, double t) {
    if (!(t > 0.0)) throw std::invalid_argument("iteration time must be positive");
    return double(lx) * ly * flops_per_site / (t * 1e9);
}

}  // namespace lbm_b200
