/*
 * d2q37_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference lbmbench D2Q37 hot path
 * (/root/reference/proj, C++20).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library; the
 * product path (paper_1804_01918_b200) never links or calls it.
 *
 * Pinned against: the reference's own frozen weights / t0 and moment identities
 * (proj/tests/test_model.cpp:87-142), the delta-impulse / permutation /
 * periodicity known-answer tests (proj/tests/test_kernels.cpp:114-276), and the
 * compiled reference itself (oracle/_ref, built by oracle/Makefile) through the
 * golden fixtures in tests/golden/.  Wall bc, RT/c2/Philox initialisers have no
 * reference counterpart: those are "parity unpinned" and
 * are pinned only by the builder's own known-answer tests (tests/test_oracle.py).
 *
 * Canonical lattice order everywhere: index (p*lx + x)*ly + y
 * (proj/include/lbm/dump.hpp:19-21).
 */
#ifndef D2Q37_ORACLE_H
#define D2Q37_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_NPOP 37
#define ORC_NSHELL 8
#define ORC_NMOM 14
#define ORC_HALO 3

enum { ORC_BC_PERIODIC = 0, ORC_BC_WALL = 1 };

typedef struct {
    int cx[ORC_NPOP];
    int cy[ORC_NPOP];
    int shell[ORC_NPOP];
    double w[ORC_NPOP];
    double shell_w[ORC_NSHELL];
    double t0;
    double eq[ORC_NPOP * ORC_NMOM]; /* row-major [i][k] */
} orc_model;

/* model.cpp:81-99 / :101-181 / :183-234 */
int orc_model_d2q37(orc_model* m);
/* y-mirror index ybar(p): population with (cx, -cy) -- wall bc. */
void orc_ymirror(const orc_model* m, int out[ORC_NPOP]);

/* model.cpp:242-257; returns 0, or 1 when !(rho > 0) (NonPhysicalError). */
int orc_macros(const orc_model* m, const double* f, double mac[4]);
/* model.cpp:259-291; mac = {rho, ux, uy, temp}. */
void orc_equilibrium(const orc_model* m, const double mac[4], double* feq);
/* model.cpp:293-298 */
int orc_collide_site(const orc_model* m, const double* f, double omega, double* out);

/* validation.cpp:13-25 (periodic) + builder wall rule, canonical arrays. */
int orc_propagate(const orc_model* m, int lx, int ly, int bc, const double* in, double* out);
/* the same pull copy split over threads by canonical rows (a permutation: thread-count invariant) */
int orc_propagate_mt(const orc_model* m, int lx, int ly, int bc, const double* in, double* out, int nthreads);
/* validation.cpp:27-38; returns 1 if any site is non-physical. */
int orc_collide(const orc_model* m, int lx, int ly, double omega, const double* in, double* out,
                int nthreads);
/* kernels.cpp:276-283 semantics on a canonical state: nsteps x (propagate, collide). */
int orc_step(const orc_model* m, int lx, int ly, int bc, double omega, int nsteps, double* state,
             double* scratch, int nthreads);

/* Reference padded SoA/CSoA storage (layout.hpp:46-98, layout.cpp:50-59); vl=1 is SoA. */
size_t orc_padded_elems(int lx, int ly, int vl);
size_t orc_padded_index(int lx, int ly, int vl, int p, int X, int j, int k);
int orc_canonical_to_padded(int lx, int ly, int vl, const double* canon, double* padded);
int orc_padded_to_canonical(int lx, int ly, int vl, const double* padded, double* canon);
/* kernels.cpp:197-234 (periodic) and the builder wall variant on the outer faces. */
int orc_halo_fill(const orc_model* m, int lx, int ly, int vl, int bc, double* padded);
/* kernels.cpp:37-85 on a padded SoA/CSoA buffer (physical sites of out only). */
int orc_propagate_padded(const orc_model* m, int lx, int ly, int vl, const double* in,
                         double* out);

/* std::mt19937_64 (C++ [rand.predef]) and the reference's u01 mapping
 * (lattice.cpp:11-12): (r >> 11) * 2^-53. */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
double orc_mt64_u01(orc_mt64* g);
void orc_mt64_fill_u01(uint64_t seed, size_t n, double* out);

/* Philox4x32-10 (Salmon et al., SC'11), one block per counter. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Initialisers, all writing canonical arrays. */
/* lattice.cpp:8-23 */
void orc_random_lattice(const orc_model* m, int lx, int ly, uint64_t seed, double* out);
/* lattice.cpp:25-34 */
void orc_equilibrium_lattice(const orc_model* m, int lx, int ly, const double mac[4], double* out);
/* lattice.cpp:36-47 */
void orc_shear_lattice(const orc_model* m, int lx, int ly, double amp, double temp, double* out);
/* BASELINE config 0/3/4: Rayleigh-Taylor-like init (builder recipe). */
void orc_rt_lattice(const orc_model* m, int lx, int ly, uint64_t seed, double* out);
/* Same RT formulas with Philox noise keyed by the global site index x*ly_global + y_global,
 * for rows [y0, y0+ly) of an lx x ly_global lattice (the product's device-side init). */
void orc_rt_philox_lattice(const orc_model* m, int lx, int ly, int ly_global, int y0, uint64_t seed, double* out);
/* BASELINE config 2 recipe. */
void orc_c2_lattice(const orc_model* m, int lx, int ly, uint64_t seed, double* out);
/* BASELINE config 1: i.i.d. U[0,1) from Philox keyed by seed, counter = site-major index. */
void orc_philox_lattice(int lx, int ly, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
