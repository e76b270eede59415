// d2q37_kernels.cuh -- launch interface of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include "d2q37_device.cuh"

namespace d2q37 {

// 128-thread CTAs; the collide kernels keep f[37] in registers and are capped
// at 128 registers (no spills) so 4 CTAs (16 warps) are resident per SM: the
// load bursts of more warps overlap (+1.2 % CAoSoA, +7 % SoA over 3 CTAs).
constexpr int kStreamThreads = 128;
constexpr int kCollideMinBlocks = 4;

// Up to two q-ranges per launch (blockIdx.z selects one); each has nq sites
// per column at q = q0 + t*stride.  q indexes a column's physical elements in
// memory order (q = row*vl + lane).  skip_lo / skip_hi drop the sites whose
// pull reaches a remote face (lane 0's first 3 rows / lane vl-1's last 3):
// a slab computes those after its halos arrive.
// dense = 1 packs the segments of every column into one 1-D grid (a few sites
// per column: the slab boundary launch); otherwise grid = (nq/128, lx, nseg).
// nx > 0 makes segment z the box of storage columns x0[z] .. x0[z]+nx-1 by
// sites q0[z] + t*stride: the y-major slab's interior / boundary columns.
struct Segments {
    int q0[2];
    int nq;
    int stride;
    int skip_lo, skip_hi;
    int dense, nseg;
    int x0[2];
    int nx;
};

// Outer y-face treatment.  k_edge: periodic wrap, wall mirror, or remote (from
// the slab receive buffers).  Stream kernels: periodic / wall resolved
// in-kernel, ghost = read the ghost rows (filled by a bc verb or k_edge remote).
enum { kFacePeriodic = 0, kFaceWall = 1, kFaceRemote = 2, kFaceGhost = 3 };
enum { kEdgeLocal = 1, kEdgeRemote = 2, kEdgeAll = 3 };

// lo / hi: the storage-row faces (lane 0 low, lane vl-1 high); col_lo / col_hi:
// the storage-column faces (periodic x in the normal storage; the lattice y
// faces in y-major storage, where walls and slab neighbours sit).
struct Faces {
    int lo, hi;
    int col_lo, col_hi;
    signed char ybar[kNpop];  // y-mirror (cx, -cy)
};

struct EdgeParams {
    const double* recv_lo;  // [slot][x]: neighbour's rows ny-d for (d, p) with cy_p >= d
    const double* recv_hi;  // [slot][x]: neighbour's rows d-1 for (d, p) with cy_p <= -d
    int face_lo, face_hi;
    int filter;
    int lean;  // fill only lane 0's low / lane vl-1's high ghost rows (+ ghost columns)
    signed char lo_slot[kHalo][kNpop];  // (d-1, p) -> slot or -1
    signed char hi_slot[kHalo][kNpop];
    signed char ybar[kNpop];            // y-mirror (cx, -cy)
};

constexpr int kMaxSlots = 32;  // 26 for D2Q37

struct PackParams {
    double* send_lo;
    double* send_hi;
    int nslots;
    signed char lo_d[kMaxSlots], lo_p[kMaxSlots];  // entries of send_lo (cy_p <= -d)
    signed char hi_d[kMaxSlots], hi_p[kMaxSlots];  // entries of send_hi (cy_p >= d)
};

// Peer-memory halo push of a slab (P2P transport): the face kernel also
// stores the updated face sites straight into the neighbour's buffer (its
// ghost slots), over NVLink.  Element e of this slab lands at peer element
// e + shift (a constant per face: slabs share one geometry).
struct PeerStores {
    double* lo;  // lo neighbour's buffer, or null
    double* hi;  // hi neighbour's buffer, or null
    long long lo_shift, hi_shift;
};

cudaError_t launch_propagate(const double* src, double* dst, const DevGeo& g, const Offsets& off, const Faces& fc,
                             const Segments& seg, int nseg, cudaStream_t s);
cudaError_t launch_collide(const double* src, double* dst, const DevGeo& g, const Offsets& off, const Faces& fc,
                           const ModelParams& mp, double omega, bool strict, bool shift, const Segments& seg,
                           int nseg, int* flag, cudaStream_t s);
// The fused step on the face sites of (seg, nseg) with the peer stores.
cudaError_t launch_face(const double* src, double* dst, const DevGeo& g, const Offsets& off, const Faces& fc,
                        const ModelParams& mp, double omega, bool strict, const Segments& seg, int nseg,
                        const PeerStores& ps, int* flag, cudaStream_t s);
// Copies the face sites of (seg, nseg) of buf into the peers (same buffer index).
cudaError_t launch_face_prime(const double* buf, const DevGeo& g, const Offsets& off, const Segments& seg, int nseg,
                              const PeerStores& ps, cudaStream_t s);
// P2P step protocol: wait until the step counters the neighbours wrote into
// seq[0] (lo) / seq[1] (hi) reach `target` (system-scope acquire; gives up
// after timeout_ns and sets bit 2 of *flag); signal = system-scope release
// store of `value` into the neighbours' counter slots.
cudaError_t launch_p2p_wait(const unsigned long long* seq, bool need_lo, bool need_hi, unsigned long long target,
                            unsigned long long timeout_ns, int* flag, cudaStream_t s);
cudaError_t launch_copy(double* dst, const double* src, long long n, cudaStream_t s);
// Loads every kernel of this library on the current device (see d2q37_kernels.cu).
cudaError_t preload_kernels();
cudaError_t launch_p2p_signal(unsigned long long* lo_slot, unsigned long long* hi_slot, unsigned long long value,
                              cudaStream_t s);
cudaError_t launch_edge(double* buf, const DevGeo& g, const EdgeParams& ep, cudaStream_t s);
cudaError_t launch_pack(const double* buf, const DevGeo& g, const PackParams& pp, cudaStream_t s);
cudaError_t launch_scatter(double* buf, const DevGeo& g, const double* canon_plane, int p, cudaStream_t s);
cudaError_t launch_gather(const double* buf, const DevGeo& g, double* canon_plane, int p, cudaStream_t s);
cudaError_t launch_philox(double* buf, const DevGeo& g, unsigned long long seed, int y0, int ly_global,
                          cudaStream_t s);
cudaError_t launch_init_rt(double* buf, const DevGeo& g, const ModelParams& mp, unsigned long long seed, int y0,
                           int ly_global, cudaStream_t s);
// One scalar reference step (propagate then collide, periodic x and y) on a
// halo-free canonical array: in -> tmp -> out (validation.cpp:13-38).
cudaError_t launch_scalar_step(const double* in, double* tmp, double* out, int lx, int ly, const ModelParams& mp,
                               double omega, bool strict, int* flag, cudaStream_t s);
// Two fused steps in one sweep (d2q37_step2.cu): SoA (vl = 1), x-major storage,
// periodic x, periodic or wall y faces, FAST math.  src and dst must differ.
bool step2_supported(const DevGeo& g, const Faces& fc);
// One part of a sweep: 0 = the plain (interior) bands, 1 / 2 = the low / high
// face bands, 3 = every band (the last three through the general kernel);
// step2_items = its (band, column) items; at most max_ctas persistent CTAs
// (0: one per SM).
long long step2_items(const DevGeo& g, const Faces& fc, int part);
// Interior-band code form of a FUSED2 sweep: per-thread pulls (sweep_plain, the
// default: measured fastest) or bulk copies staged in shared memory (sweep_tma;
// 1 = issued after the moments, 2 = as soon as the stage is in registers).
// Environment D2Q37_STEP2_FORM selects one.  set_step2_form returns the previous form.
// 3 = two bulk-copy stages beside a 148-column ring (sweep_tma2).
// 4 = form 3 with two threads per site (k_step2_pair, d2q37_pair.cu).
enum { kStep2Plain = 0, kStep2Bulk = 1, kStep2BulkEarly = 2, kStep2Bulk2 = 3, kStep2Pair = 4 };
int step2_band_rows();  // output rows per band (kT2Out)
int step2_form();
int set_step2_form(int form);
// Interior schedule of the plain form: 1 = lockstep (CTAs of neighbouring bands
// march the same columns together; the default), 0 = band-major item ranges.
// Environment D2Q37_STEP2_SCHED selects one; set_step2_sched returns the previous.
int step2_sched();
bool step2_ghost_walls();
int set_step2_sched(int sched);
// percent cost of a face-band (general form) item relative to an interior item,
// which sizes the face CTA groups of k_step2_split (0 = the form's default)
int step2_face_pct();
void set_step2_face_pct(int pct);
size_t step2_smem_bytes(int form);
// Parts 0, 1, 2 in one launch with ctas[part] persistent CTAs each (every part
// with items needs at least one).
cudaError_t launch_step2_split(const double* src, double* dst, const DevGeo& g, const Faces& fc,
                               const ModelParams& mp, double omega, int* flag, cudaStream_t s, const int ctas[3]);
// The pair form (kStep2Pair): interior bands [band0, band0 + nb) by k_step2_pair on `ctas` CTAs (lock:
// the lockstep schedule) ...
cudaError_t launch_step2_pair(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                              double omega, int* flag, cudaStream_t s, int band0, int nb, int ctas, bool lock);
// ... and a whole sweep in that form: part 0 by k_step2_pair on s, the face parts 1 and 2 by the
// general form on `side` in the same interval (ev_fork / ev_join order it with s).
cudaError_t launch_step2_pair_split(const double* src, double* dst, const DevGeo& g, const Faces& fc,
                                    const ModelParams& mp, double omega, int* flag, cudaStream_t s, cudaStream_t side,
                                    cudaEvent_t ev_fork, cudaEvent_t ev_join, const int ctas[3]);
cudaError_t launch_step2(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                         double omega, int* flag, cudaStream_t s, int part, int max_ctas);
// Slab sweeps split in time (the overlapped FUSED2 slab schedule): bands
// [b_lo, b_hi) pull only rows inside [0, ly); the others reach a face.
void step2_interior_bands(const DevGeo& g, int* nbands, int* b_lo, int* b_hi);
// One overlapped FUSED2 slab sweep on `grid` CTAs (k_step2_slab): face bands
// first on a few CTAs, which write the 6-row halos of the new state into
// send_lo / send_hi and add one each to *counter; then the interior.  Returns
// the number of CTAs that signal (0: not launched -- no interior band, a
// periodic face, or a launch error in *err).
int launch_step2_slab(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                      double omega, int* flag, cudaStream_t s, int grid, unsigned* counter, double* send_lo,
                      double* send_hi, cudaError_t* err);
// The overlapped slab sweep in the pair form (k_step2_pair_slab): ghost-face bands first on a few CTAs
// (new edge rows into send_lo / send_hi, one counter increment per CTA once stored), the other bands --
// a global wall's among them -- in lockstep on the rest.  Returns the number of CTAs that signal (0: not
// launched -- no ghost face, too few bands, or an error in *err).
int launch_step2_pair_slab(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                           double omega, int* flag, cudaStream_t s, int grid, unsigned* counter, double* send_lo,
                           double* send_hi, cudaError_t* err);
// Explicit band ranges per part: part 0 in the per-thread plain form (rows read
// unwrapped: not for y-periodic faces), parts 1 and 2 in the general form.
cudaError_t launch_step2_parts(const double* src, double* dst, const DevGeo& g, const Faces& fc,
                               const ModelParams& mp, double omega, int* flag, cudaStream_t s, const int band0[3],
                               const int nb[3], const int ctas[3]);
// Band-blocked store (layout D2Q37_BANDED, d2q37_banded.cu): FUSED2 sweeps on
// blocks of 37 populations x (kBandRows + 2 kBandHalo) rows per (column, band),
// the halo rows kept as copies.  band_geometry fills a DevGeo (band = 1), band_elems its buffer size.
constexpr int kBandRows = 120;
constexpr int kBandHalo = 8;
void band_geometry(int lx, int ly, DevGeo* g);
size_t band_elems(const DevGeo& g);
size_t band_smem_bytes();
// one sweep: two steps (two = true) or one
cudaError_t launch_band_sweep(const double* src, double* dst, const DevGeo& g, const Faces& fc, const ModelParams& mp,
                              double omega, bool two, int* flag, cudaStream_t s);
cudaError_t launch_band_scatter(double* buf, const DevGeo& g, const double* canon_plane, int p, cudaStream_t s);
cudaError_t launch_band_gather(const double* buf, const DevGeo& g, double* canon_plane, int p, cudaStream_t s);
cudaError_t launch_band_init_rt(double* buf, const DevGeo& g, const ModelParams& mp, unsigned long long seed, int y0,
                                int ly_global, cudaStream_t s);
cudaError_t launch_band_moments(const double* buf, const DevGeo& g, double* part, cudaStream_t s);
cudaError_t launch_band_pack6(const double* buf, const DevGeo& g, double* send_lo, double* send_hi, cudaStream_t s);
cudaError_t launch_band_unpack6(double* buf, const DevGeo& g, const double* recv_lo, const double* recv_hi,
                                cudaStream_t s);
cudaError_t preload_band_kernels();
// FUSED2 slab halos (deep SoA geometry): 6 rows per face and population,
// buffers of halo6_count(g) doubles laid out [p][x][6].
size_t halo6_count(const DevGeo& g);
// periodic images of rows ly-6..ly-1 / 0..5 into the deep ghost rows -6..-1 / ly..ly+5 (y-periodic single domain)
cudaError_t launch_wrap6(double* buf, const DevGeo& g, cudaStream_t s);
// specular-wall images (population ybar at the mirror row) into the deep ghost rows (walls at both faces);
// mask: bit 0 the low face's rows -6..-1, bit 1 the high face's rows ly..ly+5
cudaError_t launch_mirror6(double* buf, const DevGeo& g, const Faces& fc, cudaStream_t s, int mask = 3);
cudaError_t launch_pack6(const double* buf, const DevGeo& g, double* send_lo, double* send_hi, cudaStream_t s);
cudaError_t launch_unpack6(double* buf, const DevGeo& g, const double* recv_lo, const double* recv_hi,
                           cudaStream_t s);
cudaError_t launch_moments(const double* buf, const DevGeo& g, double* part, cudaStream_t s);

}  // namespace d2q37
