// parity_main.cpp -- C++ drop-in parity program (TEST INFRASTRUCTURE).
//
// Links the UNMODIFIED reference library (oracle/_ref/liblbmref.so, built from
// /root/reference/proj/src by oracle/Makefile) and drives the B200 path through
// the reference-shaped C++ API (include/lbm_b200/lbm_b200.hpp), criterion by
// criterion like the reference's own acceptance suite (proj/tests/
// acceptance.cpp): one PASS/FAIL line each, exit status = number of failures.
//
//   G1  model constants: device model == VelocityModel::d2q37()      (C1, C2)
//   G2  halo_exchange + propagate bitwise == oracle_propagate, 4 layouts x vl (C3)
//   G3  collide <= 1e-12 vs oracle_collide with the reference's own table;
//       100 steps conserve mass, momentum, energy to 1e-11               (C4)
//   G4  identical dumps after 10 steps across the four layouts          (C5)
//   G5  10 steps <= 1e-12 vs the reference lbm::step                     (validation.cpp)
//   G6  metric formulas reproduce Table 1                                (C6)
//   G7  errors: invalid geometry -> std::invalid_argument,
//       rho <= 0 -> NonPhysicalError                                     (test_kernels.cpp:424-433)
//   G8  run_validation's scalar device reference <= 1e-12 vs the reference's
//       oracle_propagate + oracle_collide (5 steps); convert between device
//       layouts preserves every physical site                           (validation.cpp, layout.cpp:105-116)
//   G9  a MultiGpuLattice (P2P halos) <= 1e-12 vs the reference lbm::step over
//       6 periodic steps: one slab per device listed in D2Q37_G9_DEVICES
//       (default "0": a 1-slab ring that waits only on its own stream --
//       several slabs on one GPU would spin on each other's counters)
//   G10 StepVariant::Fused2 (two steps per HBM sweep) on SoA: 10 steps
//       <= 1e-12 vs the reference lbm::step, and bit for bit == 10 fused steps
//   G11 VelocityModel per-site verbs (model.hpp:60-72): macros_of,
//       equilibrium and collide_site <= 1e-14 vs the reference's on random
//       sites; macros_of of a non-positive density throws NonPhysicalError
//   G12 run(state, model, in, out, omega, n): the streamed load + step + dump
//       (walls, Fused2, y-chunks) bit for bit == load, step, dump; the periodic
//       call (three verbs inside) <= 1e-12 vs the reference load / lbm::step / dump
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#define private public  // read the reference's Hermite table (model.hpp:97), test-only
#include "lbm/model.hpp"
#undef private
#include "lbm/kernels.hpp"
#include "lbm/lattice.hpp"
#include "lbm/validation.hpp"
#include "lbm_b200/lbm_b200.hpp"

namespace {

using B = lbm_b200::LayoutKind;
const std::array<B, 4> kLayouts = {B::AoS, B::SoA, B::CSoA, B::CAoSoA};

lbm_b200::CanonicalLattice to_gpu(const lbm::CanonicalLattice& c) {
    lbm_b200::CanonicalLattice g = lbm_b200::make_canonical(c.lx, c.ly);
    g.values = c.values;
    return g;
}

lbm::CanonicalLattice oracle_run(const lbm::CanonicalLattice& init, const std::function<void(lbm::OracleLattice&, lbm::OracleLattice&)>& f) {
    lbm::OracleLattice a(init.lx, init.ly), b(init.lx, init.ly);
    lbm::oracle_from_canonical(init, a);
    f(a, b);
    return lbm::oracle_to_canonical(b);
}

double max_rel(const std::vector<double>& got, const std::vector<double>& want) {
    double m = 0.0;
    for (size_t i = 0; i < want.size(); ++i) m = std::max(m, std::abs(got[i] - want[i]) / std::abs(want[i]));
    return m;
}

// The reference model's own constants (the device gets the table
// of the binary it is compared with).
lbm_b200::VelocityModel reference_model() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    d2q37_model raw{};
    for (int i = 0; i < 37; ++i) {
        raw.cx[i] = m.velocities()[i].x;
        raw.cy[i] = m.velocities()[i].y;
        raw.w[i] = m.weights()[i];
        for (int k = 0; k < 14; ++k) raw.eq[i * 14 + k] = m.eq_table_[i][k];
    }
    raw.t0 = m.t0();
    return lbm_b200::VelocityModel::from_raw(raw);
}

bool g1() {
    const lbm::VelocityModel& r = lbm::VelocityModel::d2q37();
    const lbm_b200::VelocityModel& d = lbm_b200::VelocityModel::d2q37();
    if (d.t0() != r.t0()) return false;
    for (int i = 0; i < 37; ++i) {
        if (d.velocity(i).x != r.velocities()[i].x || d.velocity(i).y != r.velocities()[i].y) return false;
        // the reference build contracts into FMA: weights agree to a few ulp
        if (std::abs(d.weight(i) - r.weights()[i]) > 1e-14 * r.weights()[i]) return false;
    }
    return true;
}

bool g2() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    for (const auto& [lx, ly] : {std::pair{16, 32}, std::pair{64, 128}}) {
        const lbm::CanonicalLattice init = lbm::make_random_lattice(lx, ly, 1001 + lx);
        const lbm::CanonicalLattice want =
            oracle_run(init, [&](auto& a, auto& b) { lbm::oracle_propagate(a, b, m.velocities()); });
        for (const B kind : kLayouts)
            for (const int vl : {1, 2, 4, 8}) {
                lbm_b200::LatticeState s(kind, lbm_b200::Geometry{lx, ly, 3, 3, vl});
                s.load(to_gpu(init));
                lbm_b200::halo_exchange(s);
                lbm_b200::propagate(s);
                if (s.dump_from(1).values != want.values) return false;
            }
    }
    return true;
}

bool g3() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    const lbm_b200::VelocityModel dm = reference_model();
    const int lx = 64, ly = 128;
    const double omega = 1.3;
    const lbm::CanonicalLattice init = lbm::make_random_lattice(lx, ly, 2002);
    const lbm::CanonicalLattice want =
        oracle_run(init, [&](auto& a, auto& b) { lbm::oracle_collide(a, b, m, omega); });
    for (const B kind : kLayouts) {
        lbm_b200::LatticeState s(kind, lbm_b200::Geometry{lx, ly, 3, 3, 4});
        s.load_into(1, to_gpu(init));
        lbm_b200::collide(s, dm, omega);
        if (!(max_rel(s.dump().values, want.values) <= 1e-12)) return false;
    }
    auto totals = [&](const lbm_b200::CanonicalLattice& c) {
        std::array<double, 4> t{};
        for (int p = 0; p < 37; ++p)
            for (int x = 0; x < c.lx; ++x)
                for (int y = 0; y < c.ly; ++y) {
                    const double f = c.at(x, y, p);
                    const auto v = m.velocities()[p];
                    t[0] += f;
                    t[1] += v.x * f;
                    t[2] += v.y * f;
                    t[3] += (v.x * v.x + v.y * v.y) * f;
                }
        return t;
    };
    lbm_b200::LatticeState s(B::CAoSoA, lbm_b200::Geometry{lx, ly, 3, 3, 4});
    s.load(to_gpu(init));
    const auto t0 = totals(s.dump());
    for (int n = 0; n < 100; ++n) {
        lbm_b200::step(s, dm, omega);
        const auto t = totals(s.dump());
        if (!(std::abs(t[0] - t0[0]) / t0[0] < 1e-11)) return false;
        if (!(std::abs(t[1] - t0[1]) / t0[0] < 1e-11)) return false;
        if (!(std::abs(t[2] - t0[2]) / t0[0] < 1e-11)) return false;
        if (!(std::abs(t[3] - t0[3]) / t0[3] < 1e-11)) return false;
    }
    return true;
}

bool g4() {
    const lbm_b200::VelocityModel& m = lbm_b200::VelocityModel::d2q37();
    const lbm::CanonicalLattice init = lbm::make_random_lattice(64, 128, 3003);
    std::vector<double> reference;
    for (const B kind : kLayouts)
        for (const auto variant : {lbm_b200::StepVariant::Fused, lbm_b200::StepVariant::Unfused}) {
            lbm_b200::LatticeState s(kind, lbm_b200::Geometry{64, 128, 3, 3, 4});
            s.load(to_gpu(init));
            lbm_b200::step(s, m, 1.1, 10, variant);
            const auto out = s.dump();
            if (reference.empty())
                reference = out.values;
            else if (out.values != reference)
                return false;
        }
    return true;
}

bool g5() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    const lbm::CanonicalLattice init = lbm::make_random_lattice(32, 64, 88);
    lbm::LatticeState ref{lbm::Descriptor(lbm::LayoutKind::CSoA, [] {
        lbm::Geometry g{32, 64};
        g.vl = 4;
        return g;
    }())};
    ref.load(init);
    lbm::ThreadPool pool(4);
    for (int n = 0; n < 10; ++n) lbm::step(ref, m, 0.9, pool);
    lbm_b200::LatticeState s(B::CAoSoA, lbm_b200::Geometry{32, 64, 3, 3, 16});
    s.load(to_gpu(init));
    lbm_b200::step(s, reference_model(), 0.9, 10);
    return s.time_step() == ref.time_step && max_rel(s.dump().values, ref.dump().values) <= 1e-12;
}

bool g10() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    const lbm::CanonicalLattice init = lbm::make_random_lattice(40, 300, 89);
    lbm::LatticeState ref{lbm::Descriptor(lbm::LayoutKind::SoA, lbm::Geometry{40, 300})};
    ref.load(init);
    lbm::ThreadPool pool(4);
    for (int n = 0; n < 10; ++n) lbm::step(ref, m, 0.9, pool);
    lbm_b200::LatticeState two(B::SoA, lbm_b200::Geometry{40, 300});
    two.load(to_gpu(init));
    lbm_b200::step(two, reference_model(), 0.9, 10, lbm_b200::StepVariant::Fused2);
    lbm_b200::LatticeState one(B::SoA, lbm_b200::Geometry{40, 300});
    one.load(to_gpu(init));
    lbm_b200::step(one, reference_model(), 0.9, 10, lbm_b200::StepVariant::Fused);
    const auto a = two.dump().values, b = one.dump().values;
    return two.time_step() == ref.time_step && max_rel(a, ref.dump().values) <= 1e-12 &&
           std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

bool g6() {
    auto within = [](double got, double want, double tol) { return std::abs(got - want) / want <= tol; };
    return within(lbm_b200::propagate_gbps(1024, 8192, 37, 0.0125), 398.0, 0.01) &&
           within(lbm_b200::collide_gflops(1024, 8192, 6600.0, 0.0503), 1100.0, 0.01) &&
           within(lbm_b200::mlups(1024, 8192, 0.0503), 166.0, 0.01) &&
           within(lbm_b200::mlups(4608, 12288, 0.55025), 103.0, 0.01);
}

bool g7() {
    try {
        lbm_b200::LatticeState bad(B::CSoA, lbm_b200::Geometry{8, 16, 3, 3, 8});  // strip 2 < halo
        return false;
    } catch (const std::invalid_argument&) {
    }
    lbm_b200::LatticeState s(B::SoA, lbm_b200::Geometry{8, 16, 3, 3, 1});
    lbm_b200::CanonicalLattice neg = lbm_b200::make_canonical(8, 16);
    for (double& v : neg.values) v = -1.0;
    s.load_into(1, neg);
    try {
        lbm_b200::collide(s, lbm_b200::VelocityModel::d2q37(), 1.0);
        return false;
    } catch (const lbm_b200::NonPhysicalError&) {
    }
    return true;
}

bool g8() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    const lbm::CanonicalLattice init = lbm::make_random_lattice(24, 48, 808);
    const lbm::CanonicalLattice want = oracle_run(init, [&](lbm::OracleLattice& a, lbm::OracleLattice& b) {
        lbm::OracleLattice t(init.lx, init.ly);
        for (int n = 0; n < 5; ++n) {
            lbm::oracle_propagate(a, t, m.velocities());
            lbm::oracle_collide(t, a, m, 1.3);
        }
        b = a;
    });
    const auto got = lbm_b200::scalar_steps(reference_model(), to_gpu(init), 1.3, 5);
    if (!(max_rel(got.values, want.values) <= 1e-12)) return false;
    lbm_b200::LatticeState src(B::CAoSoA, lbm_b200::Geometry{24, 48, 3, 3, 8});
    src.load(to_gpu(init));
    for (const B kind : kLayouts) {
        const lbm_b200::LatticeState dst = lbm_b200::convert(src, kind, lbm_b200::Geometry{24, 48, 3, 3, 4});
        if (dst.dump().values != init.values) return false;
    }
    return true;
}

bool g9() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    const lbm::CanonicalLattice init = lbm::make_random_lattice(96, 256, 909);
    lbm::LatticeState ref{lbm::Descriptor(lbm::LayoutKind::CAoSoA, [] {
        lbm::Geometry g{96, 256};
        g.vl = 8;
        return g;
    }())};
    ref.load(init);
    lbm::ThreadPool pool(4);
    for (int n = 0; n < 6; ++n) lbm::step(ref, m, 1.05, pool);
    std::vector<int> devs;
    const char* env = std::getenv("D2Q37_G9_DEVICES");
    for (const char* c = env ? env : "0"; *c; ++c)
        if (*c >= '0' && *c <= '9') devs.push_back(*c - '0');
    lbm_b200::MultiGpuLattice gpu(B::CAoSoA, lbm_b200::Geometry{96, 256, 3, 3, 8}, devs);
    gpu.load(to_gpu(init));
    gpu.step(reference_model(), 1.05, 6);
    return max_rel(gpu.dump().values, ref.dump().values) <= 1e-12;
}

bool g11() {
    const lbm::VelocityModel& r = lbm::VelocityModel::d2q37();
    const lbm_b200::VelocityModel& d = lbm_b200::VelocityModel::d2q37();
    const lbm::CanonicalLattice lat = lbm::make_random_lattice(8, 16, 1111);
    auto rel = [](double a, double b) { return std::abs(a - b) / std::max(std::abs(b), 1e-300); };
    for (int site = 0; site < 8 * 16; ++site) {
        double f[37], outr[37], outd[37], feqr[37], feqd[37];
        for (int p = 0; p < 37; ++p) f[p] = lat.values[size_t(p) * 8 * 16 + site];
        const lbm::Macros mr = r.macros_of(f);
        const lbm_b200::Macros md = d.macros_of(f);
        if (rel(md.rho, mr.rho) > 1e-14 || rel(md.temp, mr.temp) > 1e-14) return false;
        if (std::abs(md.ux - mr.ux) > 1e-14 || std::abs(md.uy - mr.uy) > 1e-14) return false;
        r.equilibrium(mr, feqr);
        d.equilibrium(md, feqd);
        r.collide_site(f, 1.3, outr);
        d.collide_site(f, 1.3, outd);
        for (int p = 0; p < 37; ++p)
            if (rel(feqd[p], feqr[p]) > 1e-14 || rel(outd[p], outr[p]) > 1e-14) return false;
    }
    double bad[37] = {};
    bad[0] = -1.0;
    try {
        (void)d.macros_of(bad);
        return false;
    } catch (const lbm_b200::NonPhysicalError&) {
    }
    return true;
}

bool g12() {
    const lbm::VelocityModel& m = lbm::VelocityModel::d2q37();
    const lbm::CanonicalLattice init = lbm::make_random_lattice(64, 960, 1212);
    const lbm_b200::CanonicalLattice in = to_gpu(init);
    // walls (no reference counterpart: SURVEY A8): streamed in 120/240-row chunks vs the three verbs
    setenv("D2Q37_STREAM_ROWS", "240", 1);
    setenv("D2Q37_STREAM_FIRST", "120", 1);
    lbm_b200::LatticeState a(B::SoA, lbm_b200::Geometry{64, 960}), b(B::SoA, lbm_b200::Geometry{64, 960});
    lbm_b200::CanonicalLattice out;
    lbm_b200::run(a, reference_model(), in, out, 0.9, 6, lbm_b200::StepVariant::Fused2, lbm_b200::Boundary::Wall);
    unsetenv("D2Q37_STREAM_ROWS");
    unsetenv("D2Q37_STREAM_FIRST");
    b.load(in);
    lbm_b200::step(b, reference_model(), 0.9, 6, lbm_b200::StepVariant::Fused2, lbm_b200::Boundary::Wall);
    const auto want = b.dump().values;
    if (out.values.size() != want.size() || std::memcmp(out.values.data(), want.data(), want.size() * sizeof(double)) != 0)
        return false;
    if (a.time_step() != 6 || a.dump().values != want) return false;
    // periodic: against the reference's own load / step / dump
    lbm::LatticeState ref{lbm::Descriptor(lbm::LayoutKind::SoA, lbm::Geometry{64, 960})};
    ref.load(init);
    lbm::ThreadPool pool(4);
    for (int n = 0; n < 4; ++n) lbm::step(ref, m, 0.9, pool);
    lbm_b200::CanonicalLattice io = in;
    lbm_b200::run(a, reference_model(), io, io, 0.9, 4, lbm_b200::StepVariant::Fused2);  // in place
    return max_rel(io.values, ref.dump().values) <= 1e-12;
}

}  // namespace

int main(int argc, char** argv) {
    const std::array<std::pair<const char*, bool (*)()>, 12> all = {{{"G1", g1},
                                                                     {"G2", g2},
                                                                     {"G3", g3},
                                                                     {"G4", g4},
                                                                     {"G5", g5},
                                                                     {"G6", g6},
                                                                     {"G7", g7},
                                                                     {"G8", g8},
                                                                     {"G9", g9},
                                                                     {"G10", g10},
                                                                     {"G11", g11},
                                                                     {"G12", g12}}};
    int failures = 0;
    for (const auto& [name, fn] : all) {
        if (argc > 1 && std::strcmp(argv[1], name) != 0) continue;
        bool ok = false;
        try {
            ok = fn();
        } catch (const std::exception& e) {
            std::printf("%s exception: %s\n", name, e.what());
        }
        std::printf("%s %s\n", name, ok ? "PASS" : "FAIL");
        failures += ok ? 0 : 1;
    }
    return failures;
}
