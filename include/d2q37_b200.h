/*
 * d2q37_b200.h -- C-ABI of the B200-native D2Q37 hot path (sm_100a).
 *
 * Drop-in boundary for the reference lbmbench operator API
 * (/root/reference/proj/include/lbm/{kernels,lattice,dump,model}.hpp).  Every
 * entry point below names the reference interface it replaces.  Plain C types
 * only (no torch, no CUDA types); host arrays are borrowed for the duration of
 * the call; device state is owned by an opaque handle.
 *
 * Calls enqueue work on the handle's CUDA stream and return; d2q37_sync()
 * waits and reports deferred errors (D2Q37_ERR_NON_PHYSICAL from the collide
 * kernels' device flag).  load/dump/read calls are synchronous.  The C++
 * header include/lbm_b200/lbm_b200.hpp wraps this into the reference's
 * blocking, exception-throwing verbs.
 *
 * Canonical lattice order (all host arrays): (p*lx + x)*ly + y, p < 37
 * (proj/include/lbm/dump.hpp:19-21).
 */
#ifndef D2Q37_B200_H
#define D2Q37_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define D2Q37_NPOP 37
#define D2Q37_NMOM 14
#define D2Q37_HALO 3
#define D2Q37_NCCL_ID_BYTES 128
#define D2Q37_P2P_BLOB_BYTES 256

/* Status codes.  Reference exception types:
 *   INVALID_ARGUMENT  <- std::invalid_argument / std::out_of_range
 *                        (layout.cpp:14-23, kernels.cpp:181-183, :238-242, dump.cpp:37-38)
 *   NON_PHYSICAL      <- lbm::NonPhysicalError (model.hpp:28-30, model.cpp:245)       */
enum {
    D2Q37_OK = 0,
    D2Q37_ERR_INVALID_ARGUMENT = 1,
    D2Q37_ERR_NON_PHYSICAL = 2,
    D2Q37_ERR_CUDA = 3,
    D2Q37_ERR_NCCL = 4,
    D2Q37_ERR_UNSUPPORTED = 5
};

/* LayoutKind numbering of layout.hpp:12 {AoS, SoA, CSoA, CAoSoA}; all four are
 * device layouts (the reference's element order, with a device column pitch).
 * BANDED (no reference counterpart) is the device store of the two-step sweep:
 * per column, bands of 120 rows with the 37 populations of a band contiguous
 * (csrc/d2q37_banded.cu).  It supports load / dump (canonical order), the
 * device initialisers, moments, LBDUMP01 files, convert, and step() with
 * FUSED2 (FUSED = one step per sweep) in FAST math, single domain and NCCL /
 * group y-slabs; the padded-buffer verbs (bc, propagate, collide,
 * read/write_padded), UNFUSED steps, STRICT math and P2P slabs return
 * D2Q37_ERR_UNSUPPORTED.  Requires ly >= 12 (per slab). */
enum { D2Q37_AOS = 0, D2Q37_SOA = 1, D2Q37_CSOA = 2, D2Q37_CAOSOA = 3, D2Q37_BANDED = 4 };

/* Boundary condition of the y faces.  PERIODIC is the reference
 * halo_exchange (kernels.cpp:197-234); WALL is the specular top/bottom wall
 * of BASELINE config 0 (no reference counterpart).  x is always
 * periodic. */
enum { D2Q37_BC_PERIODIC = 0, D2Q37_BC_WALL = 1 };

/* step() variants: UNFUSED = bc, propagate, collide (kernels.cpp:276-283);
 * FUSED = bc, one pull-gather + collide kernel.
 * FUSED2 = two time steps per HBM sweep (temporal blocking, csrc/d2q37_step2.cu):
 * every pair of steps is one kernel that reads the state once and writes it two
 * steps later, bit-identical to two FUSED steps.  Used on SoA lattices with
 * FAST math: single domain (periodic / wall faces), NCCL y-slabs and slab
 * groups (6-row halos exchanged once per two steps); an odd last step and
 * every other case (other layouts, P2P-transport slabs, STRICT math) run FUSED
 * steps. */
enum { D2Q37_UNFUSED = 0, D2Q37_FUSED = 1, D2Q37_FUSED2 = 2 };

/* Arithmetic of the collide kernels.  FAST lets nvcc contract into DFMA (as the
 * reference's -march=native build does); STRICT performs every operation as a
 * separate IEEE op in the reference's source order (model.cpp:242-298), which
 * reproduces a no-contraction build of the reference bit for bit. */
enum { D2Q37_MATH_FAST = 0, D2Q37_MATH_STRICT = 1 };

/* Host initialisers (lattice.hpp:28-40 plus the BASELINE recipes). */
enum {
    D2Q37_INIT_RANDOM = 0,      /* make_random_lattice (lattice.cpp:8-23); params unused     */
    D2Q37_INIT_EQUILIBRIUM = 1, /* make_equilibrium_lattice (:25-34); params {rho,ux,uy,T}   */
    D2Q37_INIT_SHEAR = 2,       /* make_shear_lattice (:36-47); params {amp, temp}           */
    D2Q37_INIT_RT = 3,          /* BASELINE config 0/3/4 Rayleigh-Taylor-like init; optional   */
                                /* params {ly_global, y0} for one y-slab of a taller lattice  */
    D2Q37_INIT_C2 = 4,          /* BASELINE config 2 perturbed equilibrium                    */
    D2Q37_INIT_PHILOX = 5       /* BASELINE config 1 i.i.d. U[0,1) (Philox4x32-10)            */
};

/* Model constants (VelocityModel accessors, model.hpp:54-59, plus the Hermite
 * table eq_table_ of model.hpp:97 / model.cpp:197-234, row-major [i][k]). */
typedef struct d2q37_model {
    int cx[D2Q37_NPOP];
    int cy[D2Q37_NPOP];
    double w[D2Q37_NPOP];
    double t0;
    double eq[D2Q37_NPOP * D2Q37_NMOM];
} d2q37_model;

typedef struct d2q37_lattice d2q37_lattice;

/* Thread-local message of the last failing call. */
const char* d2q37_last_error(void);

/* VelocityModel::d2q37() (model.hpp:52, model.cpp:183-240): velocity set,
 * moment-matched weights and t0, Hermite table, derived on the host. */
int d2q37_model_d2q37(d2q37_model* out);

/* Descriptor(layout, Geometry{lx, ly, 3, 3, vl}) + LatticeState
 * (layout.hpp:46-98, layout.cpp:50-59, lattice.hpp:13-24): zero-initialised
 * double-buffered device storage.  vl is ignored for SoA. */
int d2q37_create(int layout, int lx, int ly, int vl, int device, d2q37_lattice** out);
int d2q37_destroy(d2q37_lattice* h);

/* Constants used by collide (take them from the caller's VelocityModel). */
int d2q37_set_model(d2q37_lattice* h, const d2q37_model* m);
int d2q37_set_math(d2q37_lattice* h, int math);
/* CUDA stream (cudaStream_t as void*) that all work of h is enqueued on; NULL = library-owned. */
int d2q37_set_stream(d2q37_lattice* h, void* stream);
void* d2q37_get_stream(d2q37_lattice* h);

/* Descriptor queries (layout.hpp:54-65): lx, ly, vl, strip, sy, px. */
int d2q37_geometry(const d2q37_lattice* h, int out[6]);
/* Bytes of device memory owned by h (both buffers + exchange buffers). */
size_t d2q37_device_bytes(const d2q37_lattice* h);
/* LatticeState::time_step (lattice.hpp:23). */
long d2q37_time_step(const d2q37_lattice* h);

/* LatticeState::load / dump (lattice.hpp:18-19, dump.cpp:26-42): canonical
 * host array of n = 37*lx*ly doubles into / out of the state buffer (prv). */
int d2q37_load_canonical(d2q37_lattice* h, const double* host, size_t n);
int d2q37_dump_canonical(d2q37_lattice* h, double* host, size_t n);
/* load(host_in) -> step x nsteps -> dump(host_out) as one call (lattice.hpp:18-19 + kernels.hpp:45): the
 * same result as d2q37_load_canonical + d2q37_step + d2q37_sync + d2q37_dump_canonical, bit for bit.
 * On a single-GPU SoA domain (wall or periodic bc), FUSED2, FAST math and an even nsteps the three phases
 * are pipelined in y-chunks: rows are uploaded, swept (each chunk as a parallelogram of sweeps, 8 rows
 * lower per sweep) and downloaded concurrently, so the PCIe copies hide under the sweeps (pinned
 * host arrays; pageable ones work but serialise).  host_out may be host_in.  Every other case runs
 * the three verbs one after another.  D2Q37_STREAM_RUN=0 forces that, D2Q37_STREAM_ROWS /
 * D2Q37_STREAM_FIRST / D2Q37_STREAM_LAST set the chunk heights, D2Q37_STREAM_SKEW the rows per sweep. */
int d2q37_run_canonical(d2q37_lattice* h, const double* host_in, double* host_out, size_t n, double omega,
                        int nsteps, int variant, int bc);
/* How the last d2q37_run_canonical on h ran: 0 the three verbs one after another, 1 pipelined between
 * walls, 2 pipelined on a y-periodic domain (-1: null handle). */
int d2q37_last_run_mode(const d2q37_lattice* h);
/* Test hook (no GPU needed): the operations a pipelined d2q37_run_canonical of an ly-row domain would
 * queue, 4 ints each {kind, a, b, c}: kind 0 upload rows [a, b) (upload index c), 1 the compute stream
 * waits for upload c, 2 sweep c (two steps) of rows [a, b), 3 wall images of the state after sweep c
 * (a: bit 0 low face, bit 1 high face), 4 periodic images of the state after sweep c, 5 download rows
 * [a, b) of the final state once everything before it has run.  Uploads come first (their own stream, in
 * order).  Returns the number of operations (0: the call would run the three verbs; < 0: minus an error
 * code), fills up to cap. */
int d2q37_debug_stream_plan(int ly, int nsteps, int bc, int* ops, int cap);
/* from_canonical / to_canonical on one buffer: which = 0 prv, 1 nxt (dump.hpp:28-29). */
int d2q37_load_buffer(d2q37_lattice* h, int which, const double* host, size_t n);
int d2q37_dump_buffer(d2q37_lattice* h, int which, double* host, size_t n);
/* Same with a canonical array already resident in device memory. */
int d2q37_load_buffer_device(d2q37_lattice* h, int which, const double* dev, size_t n);
int d2q37_dump_buffer_device(d2q37_lattice* h, int which, double* dev, size_t n);
/* Field::data() of one buffer in the reference Descriptor element order
 * elem(p,X,j,k) (layout.hpp:67-79), halos included: n = 37*(lx+6)*(ly/vl+6)*vl. */
int d2q37_read_padded(d2q37_lattice* h, int which, double* host, size_t n);
int d2q37_write_padded(d2q37_lattice* h, int which, const double* host, size_t n);

/* halo_exchange(prv) (kernels.hpp:29, kernels.cpp:197-234) as one fused edge
 * kernel; bc = D2Q37_BC_PERIODIC reproduces the reference bit for bit, WALL
 * mirrors the outer y faces (specular). */
int d2q37_bc(d2q37_lattice* h, int bc);
/* propagate(prv, nxt, offsets) (kernels.hpp:33, kernels.cpp:50-85).  Pass
 * corrupt_population >= 0 to add +1 to that population's pull offset (the
 * ValidationOptions::corrupt_population hook, validation.hpp:55-57). */
int d2q37_propagate(d2q37_lattice* h);
int d2q37_propagate_corrupt(d2q37_lattice* h, int corrupt_population);
/* collide(nxt, prv, model, omega) (kernels.hpp:40, kernels.cpp:120-156). */
int d2q37_collide(d2q37_lattice* h, double omega);
/* step(state, model, omega) x nsteps (kernels.hpp:45, kernels.cpp:276-283). */
int d2q37_step(d2q37_lattice* h, double omega, int nsteps, int variant, int bc);
/* std::swap(state.prv, state.nxt) (module.cpp:82, test_kernels.cpp:272): O(1). */
int d2q37_swap_buffers(d2q37_lattice* h);
/* Wait for h's stream; returns D2Q37_ERR_NON_PHYSICAL (and clears the flag) if
 * any collide since the last sync saw !(rho > 0) (model.cpp:245). */
int d2q37_sync(d2q37_lattice* h);

/* convert(src, to) (layout.hpp:148, layout.cpp:105-116): copy the
 * physical sites of src's state buffer into dst's state buffer, any layouts
 * and vl, same lx x ly, same device (dst is "Field dst(to)" of the reference,
 * created by the caller).  Ghost slots of dst are left as they were. */
int d2q37_convert(d2q37_lattice* src, d2q37_lattice* dst);

/* Scalar device reference of run_validation (validation.hpp:15-42,
 * validation.cpp:13-38 OracleLattice / oracle_propagate / oracle_collide):
 * nsteps of propagate then collide, periodic in x and y, on a halo-free
 * canonical array (dump.hpp:19-21 order) with explicit modulo indexing and no
 * layout machinery.  n = 37*lx*ly; m = NULL uses VelocityModel::d2q37();
 * math selects the collide arithmetic (compare like with like). */
int d2q37_scalar_steps(const d2q37_model* m, int lx, int ly, const double* host_in, double* host_out, size_t n,
                       double omega, int nsteps, int math, int device);

/* Global sums over the physical sites of the state buffer (prv):
 * out = {mass, x-momentum, y-momentum, energy sum |c|^2 f}; deterministic
 * for a given geometry.  Conservation checks at full size. */
int d2q37_moments(d2q37_lattice* h, double out[4]);

/* Per-site host verbs of VelocityModel (model.hpp:60-72), in the reference's
 * operation order on the host (no FMA contraction): macros_of -> {rho, ux,
 * uy, temp} (model.cpp:242-257; D2Q37_ERR_NON_PHYSICAL when !(rho > 0)),
 * equilibrium from {rho, ux, uy, temp} (model.cpp:259-291), collide_site
 * (model.cpp:293-298).  m = NULL uses d2q37_model_d2q37.  Inspection / test
 * helpers; the lattice-wide arithmetic runs on the GPU. */
int d2q37_macros_of(const d2q37_model* m, const double f[37], double out[4]);
int d2q37_equilibrium(const d2q37_model* m, const double macros[4], double f_eq[37]);
int d2q37_collide_site(const d2q37_model* m, const double f[37], double omega, double out[37]);

/* Host initialisers -> canonical array (n = 37*lx*ly); params per kind above;
 * nthreads host threads for the equilibrium evaluation (<= 0: all cores). */
int d2q37_make_lattice(int kind, int lx, int ly, uint64_t seed, const double* params,
                       const d2q37_model* m, double* out, size_t n, int nthreads);
/* Device-side D2Q37_INIT_PHILOX straight into one buffer (bit-identical to the host one). */
int d2q37_fill_philox(d2q37_lattice* h, int which, uint64_t seed);

/* save_dump / load_dump (dump.hpp:31-34, dump.cpp:44-70) of the state buffer:
 * "LBDUMP01", u64 lx, ly, npop, then the canonical values as little-endian
 * f64, streamed plane by plane through two 64 MB pinned chunks (no full host
 * copy of the lattice).  Errors as the reference: unopenable / short / not a
 * dump / truncated -> INVALID_ARGUMENT with the reference's message. */
int d2q37_save_dump(d2q37_lattice* h, const char* path);
int d2q37_load_dump(d2q37_lattice* h, const char* path);

/* Device-side config-0/3/4 RT init of the state buffer: the D2Q37_INIT_RT
 * formulas with the per-site noise drawn from Philox (key = seed, counter = the
 * global site index x*ly + y) instead of the sequential mt19937_64 stream, so
 * every y-slab initialises itself; equilibrium in the reference's op order. */
int d2q37_init_rt_device(d2q37_lattice* h, uint64_t seed);

/* ---- Multi-GPU: 1-D y-slab decomposition (BASELINE config 4) ------------- */

/* NCCL unique id for d2q37_create_slab (rank 0 creates, the caller broadcasts). */
int d2q37_nccl_unique_id(unsigned char id[D2Q37_NCCL_ID_BYTES]);
/* Rank `rank` of `nranks` owns global rows [rank*ly/nranks, (rank+1)*ly/nranks)
 * of an lx x ly lattice; load/dump take that slab's canonical array (lx x ly/nranks).
 * Halos travel by ncclSend/ncclRecv between y neighbours each step: the 3 face
 * columns of a y-major (AoS / CAoSoA) slab straight from / into the lattice
 * buffer, the 26 planned pop-rows of an SoA / CSoA slab through pack buffers.
 * nranks = 1 with a non-NULL id builds a one-rank NCCL ring: the periodic y
 * wrap goes through NCCL send/recv to self (the whole multi-GPU schedule on
 * one GPU); with id = NULL it is a plain single-domain lattice. */
int d2q37_create_slab(int layout, int lx, int ly, int vl, int device, int rank, int nranks,
                      const unsigned char id[D2Q37_NCCL_ID_BYTES], d2q37_lattice** out);
/* In-process emulation: nslabs slabs of one lx x ly lattice on one device whose
 * halos move by device copies.  Same pack / edge / interior / boundary kernels
 * as the NCCL path; used to prove slab invariance on a single GPU. */
int d2q37_create_group(int layout, int lx, int ly, int vl, int device, int nslabs,
                       d2q37_lattice** out);
/* step for every slab of a group created by d2q37_create_group; blocks until
 * every slab is done and reports a NonPhysicalError raised in any slab. */
int d2q37_group_step(d2q37_lattice** slabs, int nslabs, double omega, int nsteps, int variant, int bc);
/* The halo message layout: entry i of send_lo / recv_hi is (distance d, population p)
 * = (lo_d[i], lo_p[i]) with cy_p <= -d (the low neighbour's high ghost row d),
 * entry i of send_hi / recv_lo is (hi_d[i], hi_p[i]) with cy_p >= d.  Returns the
 * entry count (26 for D2Q37): 26 * lx doubles per face instead of 111 * lx. */
int d2q37_halo_plan(int lo_d[32], int lo_p[32], int hi_d[32], int hi_p[32]);
/* Peer ranks {lo, hi} of `rank` for a bc (-1 = wall / no neighbour). Host-only. */
int d2q37_slab_neighbors(int rank, int nranks, int bc, int out[2]);
/* rank, nranks, first global row, rows of this slab. */
int d2q37_slab_info(const d2q37_lattice* h, int out[4]);
/* Multi-GPU y-slabs without NCCL (the P2P transport), all four layouts: the
 * fused kernel of the face sites stores its results straight into the
 * neighbours' ghost slots through NVLink peer memory (site-major layouts in
 * y-major storage: 3 whole columns per face; SoA / CSoA: lane 0's first /
 * lane vl-1's last 3 rows), and per-step counters in peer memory order the
 * ranks.  create -> export a 256-byte blob -> exchange
 * the blobs (any host channel, e.g. torch.distributed) -> connect(lo
 * neighbour's blob, hi neighbour's blob); a 1-rank ring connects to its own
 * blob.  Neighbours in this process are used directly, others are mapped
 * with CUDA IPC.  All ranks must issue the same sequence of steps and
 * state-changing verbs (like NCCL collectives); a rank that waits longer than
 * D2Q37_P2P_TIMEOUT_S seconds (environment, default 60) for a neighbour
 * reports D2Q37_ERR_NCCL from d2q37_sync instead of hanging. */
int d2q37_create_slab_p2p(int layout, int lx, int ly, int vl, int device, int rank, int nranks,
                          d2q37_lattice** out);
int d2q37_p2p_export(const d2q37_lattice* h, unsigned char blob[D2Q37_P2P_BLOB_BYTES]);
int d2q37_p2p_connect(d2q37_lattice* h, const unsigned char lo[D2Q37_P2P_BLOB_BYTES],
                      const unsigned char hi[D2Q37_P2P_BLOB_BYTES]);
/* Single-process multi-GPU (SURVEY.md 8(b) "create_multi"): nslabs P2P
 * y-slabs of one lx x ly lattice, slab r on devices[r] (devices may repeat:
 * several slabs per GPU), connected as a ring; out[r] are ordinary slab
 * handles (load/dump their rows).  multi_step advances all of them in
 * lockstep and syncs. */
int d2q37_create_multi(int layout, int lx, int ly, int vl, int nslabs, const int* devices, d2q37_lattice** out);
int d2q37_multi_step(d2q37_lattice** slabs, int nslabs, double omega, int nsteps, int variant, int bc);
/* Per-kernel device timing (CUDA events recorded around each launch on the
 * handle's stream while profiling is on).  d2q37_kernel_times returns the
 * summed milliseconds and launch counts since the last call, per class:
 * 0 edge (bc), 1 propagate, 2 collide, 3 fused propagate+collide, 4 pack,
 * 5 fused face sites of a slab (after its halos arrived; P2P: with the peer
 * stores). */
int d2q37_set_profiling(d2q37_lattice* h, int on);
int d2q37_kernel_times(d2q37_lattice* h, double ms[6], long counts[6]);
/* Average device time (ms) of the last step's halo phase that was not hidden
 * behind interior compute (0 for single-domain lattices; one entry per
 * two-step sweep for FUSED2 slabs); see DESIGN.md.  d2q37_set_profiling(h, 1)
 * restarts the averaging window. */
double d2q37_exposed_halo_ms(const d2q37_lattice* h);

/* Timeline of the last overlapped FUSED2 slab sweep run with profiling on
 * (no reference counterpart): milliseconds after the sweep's launch point on
 * the lattice stream at which the halo exchange started (the sweep counter
 * released the comm stream), NCCL finished, the unpack finished, and the sweep
 * itself finished.  CUDA events on both streams; measurement only. */
int d2q37_slab_timeline(d2q37_lattice* h, double ms[4]);

/* FUSED2 tuning (no reference counterpart; process-wide).  form: how the
 * interior bands of a two-step sweep on the SoA store are swept -- 0
 * per-thread loads (one thread per site, 185-column ring), 1 one bulk-copy
 * stage (cp.async.bulk + mbarrier) issued after the moments, 2 the same
 * issued as soon as the stage is in registers, 3 two bulk-copy stages beside
 * a 148-column ring (named-barrier hand-off), 4 (default, measured fastest)
 * form 3 with two threads per site (512-thread CTAs, the pair's partial
 * moments swapped through tensor memory; the face bands then run in a
 * general-form launch beside it); all bit-identical.
 * face_pct: items per face-band CTA relative to an interior CTA, in percent
 * of the interior's cost (0 = the form's default: 115 / 135 for forms 0 / 1-4).
 * A negative argument leaves a setting unchanged; the previous values are
 * returned through prev_form / prev_face_pct when non-null.  Environment:
 * D2Q37_STEP2_FORM, D2Q37_STEP2_FACE_PCT. */
int d2q37_set_fused2_tuning(int form, int face_pct, int* prev_form, int* prev_face_pct);

/* FUSED2 interior schedule (no reference counterpart; process-wide; form 0
 * only): 1 (default) lockstep -- persistent CTA c marches whole bands c,
 * c + G, ... from column 0, so neighbouring bands sweep the same columns at
 * the same time (their shared pull rows are L2 hits, each population plane is
 * streamed as a few column-long runs); 0 band-major item ranges.  Both are
 * bit-identical.  A negative argument leaves it unchanged; the previous value
 * is returned through prev_sched when non-null.  Environment: D2Q37_STEP2_SCHED. */
int d2q37_set_fused2_schedule(int sched, int* prev_sched);

/* Test hooks (no reference counterpart).  d2q37_debug_step2_slab_sweep: one
 * overlapped FUSED2 slab sweep of h's current state with faces face_lo /
 * face_hi (1 = wall, 3 = ghost: the 6 deep ghost rows are read as they stand,
 * nothing is exchanged) in the pair form (form 4) or the one-thread form
 * (any other), the new edge rows packed into the halo send buffers;
 * d2q37_debug_read_halo6 copies send buffer `which` (0 low, 1 high; 37 x lx x 6
 * doubles, [p][x][row]) to host.  They let one GPU check the two slab sweeps
 * against each other on the face combinations of a multi-GPU run. */
int d2q37_debug_step2_slab_sweep(d2q37_lattice* h, double omega, int form, int face_lo, int face_hi);
int d2q37_debug_read_halo6(d2q37_lattice* h, int which, double* host, size_t n);

/* Measurement helper (no reference counterpart): the achieved FP64 rate of
 * independent DFMA chains on every SM of `device`, in TFLOP/s (2 FLOP per
 * DFMA) -- the FP64 roofline denominator at the clocks the GPU holds under
 * load (bench.py; MEASURED_PEAKS.json has no FP64 figure). */
int d2q37_fp64_peak(int device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* D2Q37_B200_H */
