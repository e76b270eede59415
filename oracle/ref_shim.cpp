// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference library compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/.  It lets
// the Python tests, the golden-fixture generator and bench.py's reference arm
// drive the reference's own code path (LatticeState, halo_exchange,
// propagate, collide, step, ThreadPool, time_kernel) through ctypes.  No
// reference source is copied; this file only includes the reference headers.
//
// Exceptions are mapped to the same status codes as the product C-ABI
// (include/d2q37_b200.h): 1 invalid_argument/out_of_range, 2 NonPhysicalError,
// 9 anything else.

// Standard headers first, so the access-specifier override below only reaches
// the reference's own class definitions.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <functional>
#include <iosfwd>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <utility>
#include <vector>

// Test-only: VelocityModel keeps its Hermite table private (model.hpp:97) and
// the product must be fed the exact table of the binary that computes the
// reference answer, so expose it for reading.
#define private public
#include "lbm/model.hpp"
#undef private

#include "lbm/dump.hpp"
#include "lbm/kernels.hpp"
#include "lbm/lattice.hpp"
#include "lbm/layout.hpp"
#include "lbm/metrics.hpp"
#include "lbm/thread_pool.hpp"
#include "lbm/validation.hpp"

using namespace lbm;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const NonPhysicalError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

struct RefSim {
    LatticeState state;
    std::unique_ptr<ThreadPool> pool;
    RefSim(const Descriptor& d, int workers) : state(d), pool(new ThreadPool(workers)) {}
};

CanonicalLattice canon_from(int lx, int ly, const double* v) {
    CanonicalLattice c = make_canonical(lx, ly);
    std::memcpy(c.values.data(), v, c.values.size() * sizeof(double));
    return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// VelocityModel::d2q37() accessors (model.hpp:52-59) + the private eq_table_.
int ref_model(int* cx, int* cy, double* w, double* t0, double* eq) {
    return guard([&] {
        const VelocityModel& m = VelocityModel::d2q37();
        for (int i = 0; i < kNpop; ++i) {
            cx[i] = m.velocities()[i].x;
            cy[i] = m.velocities()[i].y;
            w[i] = m.weights()[i];
            for (int k = 0; k < VelocityModel::kEqMoments; ++k)
                eq[i * VelocityModel::kEqMoments + k] = m.eq_table_[i][k];
        }
        *t0 = m.t0();
    });
}

int ref_macros(const double* f, double* mac) {
    return guard([&] {
        const Macros m = VelocityModel::d2q37().macros_of(f);
        mac[0] = m.rho;
        mac[1] = m.ux;
        mac[2] = m.uy;
        mac[3] = m.temp;
    });
}

int ref_equilibrium(const double* mac, double* feq) {
    return guard([&] { VelocityModel::d2q37().equilibrium({mac[0], mac[1], mac[2], mac[3]}, feq); });
}

int ref_collide_site(const double* f, double omega, double* out) {
    return guard([&] { VelocityModel::d2q37().collide_site(f, omega, out); });
}

// lattice.cpp initialisers -> canonical arrays
int ref_random_lattice(int lx, int ly, std::uint64_t seed, double* out) {
    return guard([&] {
        const CanonicalLattice c = make_random_lattice(lx, ly, seed);
        std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
    });
}

int ref_equilibrium_lattice(int lx, int ly, const double* mac, double* out) {
    return guard([&] {
        const CanonicalLattice c = make_equilibrium_lattice(lx, ly, VelocityModel::d2q37(),
                                                            {mac[0], mac[1], mac[2], mac[3]});
        std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
    });
}

int ref_shear_lattice(int lx, int ly, double amp, double temp, double* out) {
    return guard([&] {
        const CanonicalLattice c = make_shear_lattice(lx, ly, VelocityModel::d2q37(), amp, temp);
        std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
    });
}

// validation.cpp oracle functions on canonical arrays
int ref_oracle_propagate(int lx, int ly, const double* in, double* out) {
    return guard([&] {
        const VelocityModel& m = VelocityModel::d2q37();
        OracleLattice a(lx, ly), b(lx, ly);
        oracle_from_canonical(canon_from(lx, ly, in), a);
        oracle_propagate(a, b, m.velocities());
        const CanonicalLattice c = oracle_to_canonical(b);
        std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
    });
}

int ref_oracle_collide(int lx, int ly, double omega, const double* in, double* out) {
    return guard([&] {
        const VelocityModel& m = VelocityModel::d2q37();
        OracleLattice a(lx, ly), b(lx, ly);
        oracle_from_canonical(canon_from(lx, ly, in), a);
        oracle_collide(a, b, m, omega);
        const CanonicalLattice c = oracle_to_canonical(b);
        std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
    });
}

// LatticeState + ThreadPool: the reference's layout kernels.
// layout: 0 AoS, 1 SoA, 2 CSoA, 3 CAoSoA (LayoutKind order, layout.hpp:12).
void* ref_sim_create(int layout, int lx, int ly, int vl, int workers) {
    RefSim* s = nullptr;
    const int rc = guard([&] {
        Geometry g{lx, ly};
        g.vl = vl;
        s = new RefSim(Descriptor(static_cast<LayoutKind>(layout), g), workers);
    });
    return rc == 0 ? s : nullptr;
}

void ref_sim_destroy(void* h) { delete static_cast<RefSim*>(h); }

std::size_t ref_sim_elems(void* h) { return static_cast<RefSim*>(h)->state.prv.size(); }

int ref_sim_load(void* h, const double* canon) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        const Geometry& g = s->state.desc().geom();
        s->state.load(canon_from(g.lx, g.ly, canon));
    });
}

// which: 0 = prv, 1 = nxt
int ref_sim_load_into(void* h, int which, const double* canon) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        const Geometry& g = s->state.desc().geom();
        from_canonical(canon_from(g.lx, g.ly, canon), which ? s->state.nxt : s->state.prv);
    });
}

int ref_sim_dump(void* h, int which, double* out) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        const CanonicalLattice c = to_canonical(which ? s->state.nxt : s->state.prv);
        std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
    });
}

int ref_sim_read_raw(void* h, int which, double* out) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        const Field& f = which ? s->state.nxt : s->state.prv;
        std::memcpy(out, f.data(), f.size() * sizeof(double));
    });
}

int ref_sim_halo_exchange(void* h) {
    return guard([&] { halo_exchange(static_cast<RefSim*>(h)->state.prv); });
}

int ref_sim_propagate(void* h, int nt_stores) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        KernelOptions o;
        o.nt_stores = nt_stores != 0;
        propagate(s->state.prv, s->state.nxt, build_offset_table(s->state.desc(), VelocityModel::d2q37()),
                  *s->pool, o);
    });
}

int ref_sim_collide(void* h, double omega) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        collide(s->state.nxt, s->state.prv, VelocityModel::d2q37(), omega, *s->pool);
    });
}

int ref_sim_step(void* h, double omega, int nsteps, int nt_stores) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        KernelOptions o;
        o.nt_stores = nt_stores != 0;
        for (int n = 0; n < nsteps; ++n) step(s->state, VelocityModel::d2q37(), omega, *s->pool, o);
    });
}

long ref_sim_time_step_counter(void* h) { return static_cast<RefSim*>(h)->state.time_step; }

// metrics.cpp time_kernel around one of the reference verbs (0 propagate,
// 1 collide, 2 step); returns the median seconds per call in *median_s.
int ref_sim_time(void* h, int kernel, double omega, int iterations, int warmup, int nt_stores,
                 double* median_s, double* min_s) {
    return guard([&] {
        RefSim* s = static_cast<RefSim*>(h);
        const VelocityModel& m = VelocityModel::d2q37();
        KernelOptions o;
        o.nt_stores = nt_stores != 0;
        const OffsetTable off = build_offset_table(s->state.desc(), m);
        std::function<void()> body;
        if (kernel == 0)
            body = [&] { propagate(s->state.prv, s->state.nxt, off, *s->pool, o); };
        else if (kernel == 1)
            body = [&] { collide(s->state.nxt, s->state.prv, m, omega, *s->pool, o); };
        else
            body = [&] { step(s->state, m, omega, *s->pool, o); };
        const TimingResult t = time_kernel(body, iterations, warmup);
        *median_s = t.median_s;
        *min_s = t.min_s;
    });
}

int ref_hardware_concurrency() { return int(std::thread::hardware_concurrency()); }

// dump.cpp:44-70 (LBDUMP01 files)
int ref_save_dump(int lx, int ly, const double* canon, const char* path) {
    return guard([&] { save_dump(path, canon_from(lx, ly, canon)); });
}

// dims: {lx, ly, npop}; out may be null to query the dims only.
int ref_load_dump(const char* path, int* dims, double* out, std::size_t n) {
    return guard([&] {
        const CanonicalLattice c = load_dump(path);
        dims[0] = c.lx;
        dims[1] = c.ly;
        dims[2] = c.npop;
        if (out) {
            if (n != c.values.size()) throw std::invalid_argument("ref_load_dump: buffer size mismatch");
            std::memcpy(out, c.values.data(), n * sizeof(double));
        }
    });
}

}  // extern "C"
