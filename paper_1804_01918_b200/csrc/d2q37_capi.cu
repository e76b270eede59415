// d2q37_capi.cu -- the C-ABI of include/d2q37_b200.h: device lattice handle,
// storage, the per-step schedule (single domain and y-slab), load/dump.
#include <cuda.h>  // CUresult / CUstream for the driver's stream wait-value operation
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include <unistd.h>

#include "d2q37_b200.h"
#include "d2q37_device.cuh"
#include "d2q37_internal.h"
#include "d2q37_kernels.cuh"

using namespace d2q37;

namespace {

thread_local std::string g_last_error;

constexpr int kTransportNone = 0;
constexpr int kTransportNccl = 1;
constexpr int kTransportGroup = 2;
constexpr int kTransportP2P = 3;  // y-major slabs pushing halos through NVLink peer memory
constexpr int kEventRing = 64;
constexpr int kGraphSteps = 10;  // even, so a replay leaves the state in the same buffer

}  // namespace

namespace d2q37 {
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace d2q37

struct d2q37_lattice {
    int layout = D2Q37_SOA;
    int device = 0;
    DevGeo g{};
    size_t buf_elems = 0;
    double* buf[2] = {nullptr, nullptr};
    int cur = 0;  // index of the state buffer ("prv"); 1 - cur is "nxt"
    ModelParams mp{};
    int math = D2Q37_MATH_FAST;
    Offsets off_pull{};
    cudaStream_t stream = nullptr;
    std::shared_ptr<CUstream_st> stream_owner;  // shared by the slabs of a group
    int* d_flag = nullptr;
    int* h_flag = nullptr;
    double* d_part = nullptr;
    double* stage = nullptr;
    // host <-> device canonical transfers: a second staging plane, a copy
    // stream and events, so one plane's PCIe copy overlaps the next one's
    // scatter / gather kernel
    double* stage2 = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaStream_t copy_stream2 = nullptr;  // streamed run (d2q37_run_canonical): downloads beside the uploads
    int last_run_mode = 0;  // last d2q37_run_canonical: 0 three verbs, 1 pipelined (walls), 2 pipelined (y-periodic)
    cudaEvent_t ev_io[4] = {};
    long time_step = 0;

    // y-slab decomposition
    int rank = 0, nranks = 1, y0 = 0, ly_global = 0;
    int transport = kTransportNone;
    int nslots = 0;
    double* send_lo = nullptr;
    double* send_hi = nullptr;
    double* recv_lo = nullptr;
    double* recv_hi = nullptr;
    // FUSED2 slab halos: 6 rows x 37 populations per face, [send lo, send hi, recv lo, recv hi]
    double* h6[4] = {nullptr, nullptr, nullptr, nullptr};
    int nsm = 0;  // SM count of the device (FUSED2 CTA split)
    void* comm = nullptr;
    cudaStream_t comm_stream = nullptr;
    // NCCL slabs: pack / unpack / boundary sites run on a high-priority stream
    // concurrently with the interior kernel (disjoint sites), joined per step.
    cudaStream_t halo_stream = nullptr;
    // FUSED2 pair form: the face bands' general-form launch runs beside the interior one
    cudaStream_t side_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // overlapped FUSED2 slab sweep timeline (profiling on): sweep launch, exchange start (the counter
    // wait released), NCCL done, unpack done, sweep done
    cudaEvent_t tl[5] = {};
    bool tl_valid = false;
    cudaEvent_t ev_start = nullptr, ev_bnd = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_recv = nullptr;
    cudaEvent_t ev_int[kEventRing] = {}, ev_wait[kEventRing] = {};
    int ev_count = 0;
    PackParams pack{};
    EdgeParams edge_base{};
    // optional per-kernel timing (d2q37_set_profiling): event pairs around launches
    bool prof_on = false;
    struct ProfEntry {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<ProfEntry> prof_pending;
    std::vector<cudaEvent_t> prof_free;
    std::vector<d2q37_lattice*> group;  // transport == group: all slabs, in rank order
    // P2P transport: the neighbours' state buffers and step counters, mapped
    // into this process (CUDA IPC across processes, direct pointers within one)
    unsigned long long* d_seq = nullptr;        // [0]: last step of the lo neighbour, [1]: of the hi one
    double* peer_buf[2][2] = {};                // [lo / hi][buffer]
    unsigned long long* peer_seq_slot[2] = {};  // my slot in the lo / hi neighbour's counters
    std::vector<void*> ipc_mapped;              // opened with cudaIpcOpenMemHandle
    unsigned long long p2p_seq = 0;             // steps (and primes) issued
    bool p2p_connected = false;
    bool p2p_dirty = true;  // prv changed outside a step: ghost columns must be re-primed
    bool h6_valid = false;  // FUSED2 slab: prv's 6-row ghost rows hold the neighbours' current rows
    int h6_kind = -1;       // single domain: what they hold -- periodic images (0) or wall images (1)
    int bc_filled = -1;  // y-major slab: boundary mode of the last bc verb while prv is unchanged (else -1)
    unsigned* d_sweep_counter = nullptr;  // overlapped FUSED2 slab sweeps: face CTAs done (k_step2_slab)
    unsigned sweep_target = 0;            // its value once the last queued sweep's face CTAs are done
    // cached CUDA graph of kGraphSteps single-domain steps (d2q37_step)
    struct StepGraph {
        cudaGraphExec_t exec = nullptr;
        double omega = 0.0;
        int variant = -1, bc = -1, cur = -1, math = -1, form = -1;
        unsigned long model_gen = 0;
        cudaStream_t stream = nullptr;
    } graph;
    unsigned long model_gen = 0;  // bumped by every set_model
};

namespace {

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        const cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                                     \
            return fail(D2Q37_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                                 \
    } while (0)

#define RET(call)                          \
    do {                                   \
        const int r_ = (call);             \
        if (r_ != D2Q37_OK) return r_;     \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int now = -1;
        cudaGetDevice(&now);
        if (prev >= 0 && now != prev) cudaSetDevice(prev);
    }
};

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// Geometry checks of layout.cpp:12-24 plus the device limits.
bool clustered(int layout) { return layout == D2Q37_CSOA || layout == D2Q37_CAOSOA; }
bool site_major(int layout) { return layout == D2Q37_AOS || layout == D2Q37_CAOSOA; }

int make_geometry(int layout, int lx, int ly, int vl, DevGeo* g) {
    if (layout < D2Q37_AOS || layout > D2Q37_BANDED) return fail(D2Q37_ERR_INVALID_ARGUMENT, "unknown layout %d", layout);
    if (lx < 1 || ly < 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "lattice extents must be positive");
    if (lx > 65535) return fail(D2Q37_ERR_INVALID_ARGUMENT, "lx > 65535 not supported");
    if (layout == D2Q37_BANDED) {
        // halo slots hold single periodic images: 12 rows at least
        if (ly < 4 * kHalo) return fail(D2Q37_ERR_INVALID_ARGUMENT, "banded store needs ly >= 12 (per slab)");
        band_geometry(lx, ly, g);
        return D2Q37_OK;
    }
    if (!clustered(layout)) vl = 1;  // Descriptor::evl (layout.cpp:55)
    if (clustered(layout)) {
        if (!is_pow2(vl)) return fail(D2Q37_ERR_INVALID_ARGUMENT, "vl must be a power of two");
        if (ly % vl != 0) return fail(D2Q37_ERR_INVALID_ARGUMENT, "ly divisible by vl");
        if (ly / vl < kHalo) return fail(D2Q37_ERR_INVALID_ARGUMENT, "lane strip shorter than its halo (ly/vl < hy)");
    }
    g->lx = lx;
    g->ly = ly;
    g->vl = vl;
    g->strip = ly / vl;
    g->sy = g->strip + 2 * kHalo;
    g->px = lx + 2 * kHalo;
    g->lvl = 0;
    while ((1 << g->lvl) < vl) ++g->lvl;
    // 256-byte alignment of every column's first physical element: the column
    // stride is a multiple of 32 doubles and lead puts (p=0, X=0, j=3, k=0) on
    // a 32-double boundary.
    g->rstride = site_major(layout) ? (long long)kNpop * vl : vl;
    const int per = int(32 / std::gcd(g->rstride, 32LL));
    // SoA: room for 3 more ghost rows on each side of a column (rows j = -3..-1
    // sit in the previous column's unused tail): the 6-row halos of two-step
    // (FUSED2) slab sweeps; the reference's 3-row ghost rows are unchanged.
    g->deep = layout == D2Q37_SOA ? 1 : 0;
    g->pitch = (g->sy + (g->deep ? 2 * kHalo : 0) + per - 1) / per * per;
    g->cstride = (long long)g->pitch * g->rstride;
    g->lead = (32 - (kHalo * g->rstride) % 32) % 32;
    g->pstride = site_major(layout) ? vl : (g->px * g->cstride + 31) / 32 * 32;
    return D2Q37_OK;
}

void fill_offsets(d2q37_lattice* h, int corrupt = -1) {
    const DevGeo& g = h->g;
    for (int p = 0; p < kNpop; ++p) {
        // build_offset_table (kernels.cpp:180-195): pull from (x - cx, y - cy).
        const int sx = g.tr ? scx<true>(p) : scx<false>(p), sy = g.tr ? scy<true>(p) : scy<false>(p);
        h->off_pull.o[p] = (long long)p * g.pstride - (long long)sx * g.cstride - (long long)sy * g.rstride;
        if (p == corrupt) h->off_pull.o[p] += 1;
    }
    finish_offsets(h->off_pull, g.pstride, corrupt < 0);
}

// Validates a host model against the device velocity set and the symmetry the
// FAST kernels rely on, and packs it into kernel parameters.
int model_params(const d2q37_model* m, ModelParams* mp) {
    for (int p = 0; p < kNpop; ++p)
        if (m->cx[p] != cx_of(p) || m->cy[p] != cy_of(p))
            return fail(D2Q37_ERR_INVALID_ARGUMENT,
                        "model velocity %d is (%d,%d), the device velocity set expects (%d,%d)", p, m->cx[p],
                        m->cy[p], cx_of(p), cy_of(p));
    for (int i = 0; i < kNpop; ++i)
        for (int k = 0; k < kNmom; ++k) {
            const double v = m->eq[i * kNmom + k];
            if (eq_structural_zero(i, k) && v != 0.0)
                return fail(D2Q37_ERR_INVALID_ARGUMENT, "Hermite table entry (%d,%d) must be zero", i, k);
            mp->eq[i][k] = v;
        }
    // The FAST kernels evaluate one Hermite row per (+-a, +-b) group and take
    // the other rows' signs from the parity of each coefficient; require that
    // symmetry (and equal weights within a group) to hold exactly.
    for (int i = 0; i < kNpop; ++i)
        for (int j = 0; j < kNpop; ++j) {
            if (std::abs(cx_of(i)) != std::abs(cx_of(j)) || std::abs(cy_of(i)) != std::abs(cy_of(j))) continue;
            if (m->w[i] != m->w[j]) return fail(D2Q37_ERR_INVALID_ARGUMENT, "weights %d and %d differ", i, j);
            const bool fx = (cx_of(i) < 0) != (cx_of(j) < 0), fy = (cy_of(i) < 0) != (cy_of(j) < 0);
            for (int k = 0; k < kNmom; ++k) {
                const double s = ((fx && mom_has_cx(k)) != (fy && mom_has_cy(k))) ? -1.0 : 1.0;
                if (m->eq[j * kNmom + k] != s * m->eq[i * kNmom + k])
                    return fail(D2Q37_ERR_INVALID_ARGUMENT,
                                "Hermite table rows %d and %d are not sign-symmetric at term %d", i, j, k);
            }
        }
    for (int i = 0; i < kNpop; ++i) mp->w[i] = m->w[i];
    mp->t0 = m->t0;
    return D2Q37_OK;
}

int upload_model(d2q37_lattice* h, const d2q37_model* m) {
    ModelParams mp{};
    RET(model_params(m, &mp));
    if (std::memcmp(&mp, &h->mp, sizeof mp) == 0) return D2Q37_OK;  // same constants: keep the cached graphs
    h->mp = mp;
    ++h->model_gen;  // captured step graphs carry the old constants
    return D2Q37_OK;
}

void make_slot_tables(d2q37_lattice* h) {
    // Ghost row at distance d below the slab (gy = -d) is read only by
    // populations with cy >= d (15 + 8 + 3 = 26 pop-rows); symmetric above.
    EdgeParams& ep = h->edge_base;
    std::memset(ep.lo_slot, -1, sizeof ep.lo_slot);
    std::memset(ep.hi_slot, -1, sizeof ep.hi_slot);
    int nlo = 0, nhi = 0;
    for (int d = 1; d <= kHalo; ++d)
        for (int p = 0; p < kNpop; ++p) {
            if (cy_of(p) >= d) {
                ep.lo_slot[d - 1][p] = (signed char)nlo;
                h->pack.hi_d[nlo] = (signed char)d;  // our rows ny-d feed the hi neighbour's low ghosts
                h->pack.hi_p[nlo] = (signed char)p;
                ++nlo;
            }
            if (cy_of(p) <= -d) {
                ep.hi_slot[d - 1][p] = (signed char)nhi;
                h->pack.lo_d[nhi] = (signed char)d;
                h->pack.lo_p[nhi] = (signed char)p;
                ++nhi;
            }
        }
    h->nslots = nlo;  // == nhi by the y-symmetry of the velocity set
    h->pack.nslots = nlo;
    for (int p = 0; p < kNpop; ++p)
        for (int q = 0; q < kNpop; ++q)
            if (cx_of(q) == cx_of(p) && cy_of(q) == -cy_of(p)) ep.ybar[p] = (signed char)q;
}

int new_stream(d2q37_lattice* h) {
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    h->stream_owner = std::shared_ptr<CUstream_st>(s, [](cudaStream_t p) { cudaStreamDestroy(p); });
    h->stream = s;
    return D2Q37_OK;
}

int alloc_lattice(d2q37_lattice* h) {
    DeviceGuard dg(h->device);
    const DevGeo& g = h->g;
    h->buf_elems = g.band ? band_elems(g)
                          : size_t(g.lead + (site_major(h->layout) ? g.px * g.cstride : kNpop * g.pstride) + 32);
    for (int b = 0; b < 2; ++b) {
        CK(cudaMalloc(&h->buf[b], h->buf_elems * sizeof(double)));
        CK(cudaMemset(h->buf[b], 0, h->buf_elems * sizeof(double)));  // AlignedBuffer is zeroed (layout.cpp:101)
    }
    CK(cudaMalloc(&h->d_flag, sizeof(int)));
    CK(cudaMemset(h->d_flag, 0, sizeof(int)));
    CK(cudaMallocHost(&h->h_flag, sizeof(int)));
    CK(cudaMalloc(&h->d_part, size_t(g.lx) * 4 * sizeof(double)));
    if (!h->stream) RET(new_stream(h));
    make_slot_tables(h);
    fill_offsets(h);
    return D2Q37_OK;
}

int alloc_exchange(d2q37_lattice* h) {
    DeviceGuard dg(h->device);
    const size_t n = size_t(h->nslots) * h->g.lx;
    CK(cudaMalloc(&h->send_lo, n * sizeof(double)));
    CK(cudaMalloc(&h->send_hi, n * sizeof(double)));
    CK(cudaMalloc(&h->recv_lo, n * sizeof(double)));
    CK(cudaMalloc(&h->recv_hi, n * sizeof(double)));
    CK(cudaMemset(h->recv_lo, 0, n * sizeof(double)));
    CK(cudaMemset(h->recv_hi, 0, n * sizeof(double)));
    h->pack.send_lo = h->send_lo;
    h->pack.send_hi = h->send_hi;
    CK(cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_recv, cudaEventDisableTiming));
    for (int i = 0; i < kEventRing; ++i) {
        CK(cudaEventCreate(&h->ev_int[i]));
        CK(cudaEventCreate(&h->ev_wait[i]));
    }
    return D2Q37_OK;
}

void free_lattice(d2q37_lattice* h) {
    DeviceGuard dg(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->comm_stream) cudaStreamSynchronize(h->comm_stream);
    if (h->halo_stream) cudaStreamSynchronize(h->halo_stream);
    if (h->side_stream) cudaStreamSynchronize(h->side_stream);
    if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
    if (h->copy_stream2) cudaStreamSynchronize(h->copy_stream2);
    for (double* p : {h->buf[0], h->buf[1], h->d_part, h->stage, h->stage2, h->send_lo, h->send_hi, h->recv_lo,
                      h->recv_hi, h->h6[0], h->h6[1], h->h6[2], h->h6[3]})
        if (p) cudaFree(p);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->copy_stream2) cudaStreamDestroy(h->copy_stream2);
    for (cudaEvent_t e : h->ev_io)
        if (e) cudaEventDestroy(e);
    if (h->d_flag) cudaFree(h->d_flag);
    if (h->d_seq) cudaFree(h->d_seq);
    if (h->d_sweep_counter) cudaFree(h->d_sweep_counter);
    for (void* p : h->ipc_mapped) cudaIpcCloseMemHandle(p);
    if (h->h_flag) cudaFreeHost(h->h_flag);
    if (h->ev_pack) cudaEventDestroy(h->ev_pack);
    if (h->ev_recv) cudaEventDestroy(h->ev_recv);
    for (int i = 0; i < kEventRing; ++i) {
        if (h->ev_int[i]) cudaEventDestroy(h->ev_int[i]);
        if (h->ev_wait[i]) cudaEventDestroy(h->ev_wait[i]);
    }
    for (auto& e : h->prof_pending) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    for (cudaEvent_t e : h->prof_free) cudaEventDestroy(e);
    if (h->graph.exec) cudaGraphExecDestroy(h->graph.exec);
    if (h->comm) nccl_comm_destroy(h->comm);
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->halo_stream) cudaStreamDestroy(h->halo_stream);
    if (h->side_stream) cudaStreamDestroy(h->side_stream);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    for (cudaEvent_t e : h->tl)
        if (e) cudaEventDestroy(e);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->ev_start) cudaEventDestroy(h->ev_start);
    if (h->ev_bnd) cudaEventDestroy(h->ev_bnd);
    h->stream_owner.reset();
    (void)cudaGetLastError();  // teardown errors must not leak into later launches
}

size_t canon_count(const d2q37_lattice* h) { return size_t(kNpop) * h->g.lx * h->g.ly; }

int check_handle(const d2q37_lattice* h) {
    if (!h) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null lattice handle");
    return D2Q37_OK;
}

// The padded-buffer verbs (halo_exchange, propagate-after-halo, Field::data())
// speak the reference's x-major element order; y-major slab storage has none.
int padded_verbs_ok(const d2q37_lattice* h, const char* verb) {
    if (h->g.band)
        return fail(D2Q37_ERR_UNSUPPORTED, "%s: not available on the banded store (use FUSED2 steps / load / dump)", verb);
    if (h->g.tr)
        return fail(D2Q37_ERR_UNSUPPORTED, "%s: not available on y-major slab storage (use step / load / dump)", verb);
    return D2Q37_OK;
}

cudaEvent_t prof_event(d2q37_lattice* h) {
    if (h->prof_free.empty()) {
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    cudaEvent_t e = h->prof_free.back();
    h->prof_free.pop_back();
    return e;
}

// Records an event pair around the launches in its scope when profiling is on.
struct ProfScope {
    d2q37_lattice* h;
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(d2q37_lattice* h_, int cls_, cudaStream_t st_ = nullptr) : h(h_), cls(cls_), st(st_ ? st_ : h_->stream) {
        if (h->prof_on) {
            a = prof_event(h);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = prof_event(h);
            cudaEventRecord(b, st);
            h->prof_pending.push_back({cls, a, b});
        }
    }
};

enum { kProfEdge = 0, kProfPropagate = 1, kProfCollide = 2, kProfFused = 3, kProfPack = 4, kProfBoundary = 5, kProfClasses = 6 };

Segments all_sites(const DevGeo& g) {
    Segments s{};
    s.nq = g.ly;
    s.stride = 1;
    return s;
}

// A single rank with an NCCL communicator (d2q37_create_slab with nranks = 1
// and an id) routes its periodic y wrap through NCCL to itself: the full
// multi-GPU schedule on one GPU.
bool local_only(const d2q37_lattice* h) {
    return h->nranks == 1 && h->transport != kTransportNccl && h->transport != kTransportP2P;
}

int face_lo_of(const d2q37_lattice* h, int bc) {
    if (local_only(h)) return bc == D2Q37_BC_WALL ? kFaceWall : kFacePeriodic;
    if (h->rank == 0 && bc == D2Q37_BC_WALL) return kFaceWall;  // global low wall
    return kFaceRemote;
}
int face_hi_of(const d2q37_lattice* h, int bc) {
    if (local_only(h)) return bc == D2Q37_BC_WALL ? kFaceWall : kFacePeriodic;
    if (h->rank == h->nranks - 1 && bc == D2Q37_BC_WALL) return kFaceWall;
    return kFaceRemote;
}
int lo_peer_of(const d2q37_lattice* h, int bc) {
    return face_lo_of(h, bc) == kFaceRemote ? (h->rank - 1 + h->nranks) % h->nranks : -1;
}
int hi_peer_of(const d2q37_lattice* h, int bc) {
    return face_hi_of(h, bc) == kFaceRemote ? (h->rank + 1) % h->nranks : -1;
}

int validate_bc(const d2q37_lattice* h, int bc) {
    if (bc != D2Q37_BC_PERIODIC && bc != D2Q37_BC_WALL) return fail(D2Q37_ERR_INVALID_ARGUMENT, "unknown bc %d", bc);
    if (bc == D2Q37_BC_WALL && h->ly_global < kHalo)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "wall bc needs ly >= 3 (single specular image)");
    if (h->nranks > 1 && h->g.strip < kHalo)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "slab lane strip shorter than the halo");
    return D2Q37_OK;
}

// lean = true inside steps: the stream kernels read inner lane rows directly,
// so only the outer faces' ghost rows are needed; the bc verb fills all ghosts
// (the reference's halo_exchange semantics).
int edge(d2q37_lattice* h, int bc, int filter, bool lean = true) {
    EdgeParams ep = h->edge_base;
    ep.lean = lean ? 1 : 0;
    ep.face_lo = face_lo_of(h, bc);
    ep.face_hi = face_hi_of(h, bc);
    ep.filter = filter;
    ep.recv_lo = h->recv_lo;
    ep.recv_hi = h->recv_hi;
    ProfScope ps(h, kProfEdge);
    CK(launch_edge(h->buf[h->cur], h->g, ep, h->stream));
    return D2Q37_OK;
}

bool remote_faces(const d2q37_lattice* h, int bc) {
    return face_lo_of(h, bc) == kFaceRemote || face_hi_of(h, bc) == kFaceRemote;
}

// Pack the slab's boundary rows and (NCCL) start the exchange on the comm
// stream.  Group transport moves the data in group_exchange().
int exchange_begin(d2q37_lattice* h, int bc) {
    {
        ProfScope ps(h, kProfPack);
        CK(launch_pack(h->buf[h->cur], h->g, h->pack, h->stream));
    }
    if (h->transport == kTransportNccl) {
        CK(cudaEventRecord(h->ev_pack, h->stream));
        CK(cudaStreamWaitEvent(h->comm_stream, h->ev_pack, 0));
        std::string why;
        const int rc = nccl_exchange(h->comm, h->comm_stream, h->send_lo, h->recv_lo, lo_peer_of(h, bc), h->send_hi,
                                     h->recv_hi, hi_peer_of(h, bc), size_t(h->nslots) * h->g.lx, &why);
        if (rc != D2Q37_OK) return fail(rc, "%s", why.c_str());
        CK(cudaEventRecord(h->ev_recv, h->comm_stream));
    }
    return D2Q37_OK;
}

int exchange_wait(d2q37_lattice* h) {
    if (h->transport == kTransportNccl) CK(cudaStreamWaitEvent(h->stream, h->ev_recv, 0));
    return D2Q37_OK;
}

int group_exchange(std::vector<d2q37_lattice*>& slabs, int bc) {
    const int n = int(slabs.size());
    for (int r = 0; r < n; ++r) {
        d2q37_lattice* h = slabs[r];
        const size_t bytes = size_t(h->nslots) * h->g.lx * sizeof(double);
        const int lo = lo_peer_of(h, bc), hi = hi_peer_of(h, bc);
        if (lo >= 0) CK(cudaMemcpyAsync(h->recv_lo, slabs[lo]->send_hi, bytes, cudaMemcpyDeviceToDevice, h->stream));
        if (hi >= 0) CK(cudaMemcpyAsync(h->recv_hi, slabs[hi]->send_lo, bytes, cudaMemcpyDeviceToDevice, h->stream));
    }
    return D2Q37_OK;
}

bool can_split(const d2q37_lattice* h) { return h->g.strip >= 2 * kHalo; }

// Every site whose pull does not reach a remote face: all sites but lane 0's
// first 3 rows (remote low face) and lane vl-1's last 3 rows (remote high face).
Segments interior(const d2q37_lattice* h, int bc) {
    Segments s = all_sites(h->g);
    s.skip_lo = face_lo_of(h, bc) == kFaceRemote;
    s.skip_hi = face_hi_of(h, bc) == kFaceRemote;
    return s;
}

// The sites interior() skips, 3 per remote face and column; *nseg = 1 or 2.
Segments boundary(const d2q37_lattice* h, int bc, int* nseg) {
    const DevGeo& g = h->g;
    Segments s{};
    s.nq = kHalo;
    s.stride = g.vl;
    int n = 0;
    if (face_lo_of(h, bc) == kFaceRemote) s.q0[n++] = 0;  // rows 0..2 of lane 0
    if (face_hi_of(h, bc) == kFaceRemote) s.q0[n++] = (g.strip - kHalo) * g.vl + g.vl - 1;  // lane vl-1's last rows
    *nseg = n;
    s.dense = 1;  // 3 or 6 sites per column: one 1-D grid over all columns
    s.nseg = n;
    return s;
}

// Outer-face handling of the pull kernels for a step with boundary `bc`: local
// faces (periodic wrap, wall) are resolved inside the kernel, faces shared with
// another slab read the ghost rows k_edge fills from the receive buffers.
// In y-major storage the y faces are the storage-column faces and the storage
// rows (lattice x) are periodic.
Faces step_faces(const d2q37_lattice* h, int bc) {
    Faces fc;
    const int lo = face_lo_of(h, bc), hi = face_hi_of(h, bc);
    const int ylo = lo == kFaceRemote ? kFaceGhost : lo;
    const int yhi = hi == kFaceRemote ? kFaceGhost : hi;
    if (h->g.tr) {
        fc.lo = fc.hi = kFacePeriodic;
        fc.col_lo = ylo;
        fc.col_hi = yhi;
    } else {
        fc.lo = ylo;
        fc.hi = yhi;
        fc.col_lo = fc.col_hi = kFacePeriodic;
    }
    std::memcpy(fc.ybar, h->edge_base.ybar, sizeof fc.ybar);
    return fc;
}

// The propagate verb reads whatever the preceding bc verb left in the ghost rows
// (kernels.hpp:33: "Requires halo_exchange(prv) first"); x is always periodic.
Faces ghost_faces(const d2q37_lattice* h) {
    Faces fc;
    fc.lo = fc.hi = kFaceGhost;
    fc.col_lo = fc.col_hi = kFacePeriodic;
    std::memcpy(fc.ybar, h->edge_base.ybar, sizeof fc.ybar);
    return fc;
}

int collide_launch(d2q37_lattice* h, int src, int dst, double omega, bool shift, const Segments& seg, int nseg,
                   const Faces& fc, bool boundary = false) {
    ProfScope ps(h, !shift ? kProfCollide : (boundary || seg.dense) ? kProfBoundary : kProfFused);
    CK(launch_collide(h->buf[src], h->buf[dst], h->g, h->off_pull, fc, h->mp, omega, h->math == D2Q37_MATH_STRICT,
                      shift, seg, nseg, h->d_flag, h->stream));
    return D2Q37_OK;
}

int propagate_launch(d2q37_lattice* h, const Offsets& off, const Faces& fc) {
    ProfScope ps(h, kProfPropagate);
    CK(launch_propagate(h->buf[h->cur], h->buf[1 - h->cur], h->g, off, fc, all_sites(h->g), 1, h->stream));
    return D2Q37_OK;
}

// One time step on a single domain: one fused kernel (or propagate + collide);
// the boundary is resolved inside the pull, no bc pass.
int step_local(d2q37_lattice* h, double omega, int variant, int bc) {
    const Faces fc = step_faces(h, bc);
    if (h->g.band) {  // one step = a one-step sweep of the banded store
        {
            ProfScope ps(h, kProfFused);
            CK(launch_band_sweep(h->buf[h->cur], h->buf[1 - h->cur], h->g, fc, h->mp, omega, false, h->d_flag,
                                 h->stream));
        }
        h->cur = 1 - h->cur;
        ++h->time_step;
        return D2Q37_OK;
    }
    const Segments all = all_sites(h->g);
    if (variant == D2Q37_FUSED) {
        RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, all, 1, fc));
        h->cur = 1 - h->cur;
    } else {
        RET(propagate_launch(h, h->off_pull, fc));
        RET(collide_launch(h, 1 - h->cur, h->cur, omega, false, all, 1, fc));
    }
    ++h->time_step;
    return D2Q37_OK;
}

// the side stream of the pair form's general-form launches (face / wall bands beside the pair launch)
int ensure_side_stream(d2q37_lattice* h) {
    if (h->side_stream) return D2Q37_OK;
    CK(cudaStreamCreateWithFlags(&h->side_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    return D2Q37_OK;
}

// Two time steps in one HBM sweep (D2Q37_FUSED2, d2q37_step2.cu).
// One sweep.  The interior bands (plain form) and the face bands (general
// form) write disjoint rows, so on a large lattice one launch runs them side
// by side, each face part on as many SMs as keep its items per CTA at the
// interior's (k_step2_split).  Small lattices (a few persistent-CTA waves of
// items) run every band in one general launch.
int step2_local(d2q37_lattice* h, double omega, const Faces& fc) {
    const double* src = h->buf[h->cur];
    double* dst = h->buf[1 - h->cur];
    if (h->g.band) {
        {
            ProfScope ps(h, kProfFused);
            CK(launch_band_sweep(src, dst, h->g, fc, h->mp, omega, true, h->d_flag, h->stream));
        }
        h->cur = 1 - h->cur;
        h->time_step += 2;
        return D2Q37_OK;
    }
    if (!h->nsm) CK(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->device));
    const long long n_in = step2_items(h->g, fc, 0), n_lo = step2_items(h->g, fc, 1),
                    n_hi = step2_items(h->g, fc, 2);
    const long long n_faces = n_lo + n_hi;
    // CTAs per face part: items per CTA no more than the interior's (+ the general
    // form's extra cost per iteration, step2_face_pct)
    const int pct = step2_face_pct();
    auto share = [&](long long n) {
        return n == 0 ? 0 : int(std::max<long long>(1, (pct * n * h->nsm + 100 * n_in - 1) / (100 * n_in)));
    };
    const int c_lo = n_in ? share(n_lo) : 0, c_hi = n_in ? share(n_hi) : 0;
    const bool single = fc.lo != kFaceGhost && fc.hi != kFaceGhost;
    const bool per = fc.lo == kFacePeriodic && fc.hi == kFacePeriodic, walls = fc.lo == kFaceWall && fc.hi == kFaceWall;
    if (step2_form() == kStep2Pair && (per || (walls && step2_ghost_walls())) && h->g.deep && h->g.ly >= 128 &&
        n_in + n_faces > 256LL * h->nsm) {  // >= one producer band of rows
        // single domain in the pair form: the periodic images (k_wrap6) or the specular-wall images
        // (k_mirror6) live in the deep ghost rows, valid across sweeps, so every band is swept in one
        // launch like a 1-rank slab ring's (ghost rows read unwrapped)
        Faces gf = fc;
        gf.lo = gf.hi = kFaceGhost;
        const int kind = per ? 0 : 1;
        auto fill = [&](double* buf) { return per ? launch_wrap6(buf, h->g, h->stream) : launch_mirror6(buf, h->g, fc, h->stream); };
        int nbands, b_lo, b_hi;
        step2_interior_bands(h->g, &nbands, &b_lo, &b_hi);
        if (!h->h6_valid || h->h6_kind != kind) CK(fill(h->buf[h->cur]));
        {
            ProfScope ps(h, kProfFused);
            CK(launch_step2_pair(src, dst, h->g, gf, h->mp, omega, h->d_flag, h->stream, 0, nbands, h->nsm,
                                 step2_sched() != 0));
            CK(fill(dst));
        }
        h->cur = 1 - h->cur;
        h->time_step += 2;
        h->h6_valid = true;
        h->h6_kind = kind;
        return D2Q37_OK;
    }
    if (single) h->h6_valid = false;
    ProfScope ps(h, kProfFused);
    if (n_in == 0 || n_in + n_faces <= 256LL * h->nsm || c_lo + c_hi > h->nsm / 2) {
        // small lattices (a few persistent-CTA waves of items), or face bands too large a
        // share to split off: every band through the general form
        CK(launch_step2(src, dst, h->g, fc, h->mp, omega, h->d_flag, h->stream, 3, 0));
    } else if (step2_form() == kStep2Pair) {
        // two threads per site (512-thread CTAs) on the interior, the face bands' general form
        // (256-thread CTAs) in a launch beside it on the side stream
        RET(ensure_side_stream(h));
        const int ctas[3] = {h->nsm - c_lo - c_hi, c_lo, c_hi};
        CK(launch_step2_pair_split(src, dst, h->g, fc, h->mp, omega, h->d_flag, h->stream, h->side_stream,
                                   h->ev_fork, h->ev_join, ctas));
    } else {
        const int ctas[3] = {h->nsm - c_lo - c_hi, c_lo, c_hi};  // interior >= nsm / 2
        CK(launch_step2_split(src, dst, h->g, fc, h->mp, omega, h->d_flag, h->stream, ctas));
    }
    h->cur = 1 - h->cur;
    h->time_step += 2;
    return D2Q37_OK;
}

int ensure_halo6(d2q37_lattice* h) {
    if (h->h6[0]) return D2Q37_OK;
    DeviceGuard dg(h->device);
    const size_t bytes = halo6_count(h->g) * sizeof(double);
    for (double*& p : h->h6) {
        CK(cudaMalloc(&p, bytes));
        CK(cudaMemset(p, 0, bytes));
    }
    return D2Q37_OK;
}

// FUSED2 on a y-slab: 6-row halos of the current state (pack, NCCL to / from
// both neighbours, unpack into the deep ghost rows), then one two-step sweep
// reading them.  Everything on the lattice stream; the exchange is ~7 MB per
// face per two steps, tens of microseconds against a ~10 ms sweep.
int step2_slab_exchange_nccl(d2q37_lattice* h, int bc) {
    RET(ensure_halo6(h));
    const int lo = lo_peer_of(h, bc), hi = hi_peer_of(h, bc);
    CK(cudaEventRecord(h->ev_int[h->ev_count % kEventRing], h->stream));
    {
        ProfScope ps(h, kProfPack);
        CK(launch_pack6(h->buf[h->cur], h->g, h->h6[0], h->h6[1], h->stream));
        std::string why;
        const int rc = nccl_exchange(h->comm, h->stream, h->h6[0], h->h6[2], lo, h->h6[1], h->h6[3], hi,
                                     halo6_count(h->g), &why);
        if (rc != D2Q37_OK) return fail(rc, "%s", why.c_str());
    }
    {
        ProfScope ps(h, kProfEdge);
        CK(launch_unpack6(h->buf[h->cur], h->g, lo >= 0 ? h->h6[2] : nullptr, hi >= 0 ? h->h6[3] : nullptr,
                          h->stream));
    }
    CK(cudaEventRecord(h->ev_wait[h->ev_count % kEventRing], h->stream));
    ++h->ev_count;
    return D2Q37_OK;
}

// SMs the interior launch of an overlapped FUSED2 slab sweep leaves to the halo
// pipeline (pack, NCCL, unpack on the comm stream): the persistent interior
// CTAs take every register and all shared memory of their SM, so the halo
// kernels only run beside them on SMs left free.  D2Q37_STEP2_HALO_SMS.
// D2Q37_STEP2_OVERLAP=0 selects the serial exchange-then-sweep schedule (A/B).
bool step2_overlap() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("D2Q37_STEP2_OVERLAP");
        v = (e && *e == '0') ? 0 : 1;
    }
    return v != 0;
}

int step2_halo_sms() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("D2Q37_STEP2_HALO_SMS");
        v = e ? std::max(0, std::atoi(e)) : 1;
    }
    return v;
}

// The driver's cuStreamWaitValue32 (stream memory operation; 32-bit waits need
// no device attribute), looked up once through the runtime.
using WaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32 wait_value32() {
    static WaitValue32 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WaitValue32>(p);
        (void)cudaGetLastError();
    }
    return fn;
}

// One FUSED2 sweep of an NCCL y-slab with its 6-row halo exchange overlapped
// (north_star: "overlapped with interior compute"); prv's ghost rows are
// current (h6_valid).  One launch (k_step2_slab): a few CTAs sweep the face
// bands first and pack the new state's 6 edge rows into the send buffers as
// they write them, then bump a device counter; all CTAs then sweep the
// interior.  On the comm stream a wait on that counter gates the NCCL
// exchange and the unpack into the new state's ghost rows, which run on the
// step2_halo_sms() SMs the sweep leaves free (its persistent CTAs take every
// register and all shared memory of their SM) while the interior is swept.
// The lattice stream waits for the exchange before the next sweep.  Every
// band sees the same inputs as in the serial exchange-then-sweep schedule, so
// the two are bit-identical.
int step2_sweep_overlapped(d2q37_lattice* h, double omega, int bc, const Faces& fc) {
    if (!h->nsm) CK(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->device));
    WaitValue32 wait = wait_value32();
    RET(ensure_halo6(h));
    if (!h->d_sweep_counter) {
        CK(cudaMalloc(&h->d_sweep_counter, sizeof(unsigned)));
        CK(cudaMemset(h->d_sweep_counter, 0, sizeof(unsigned)));
        h->sweep_target = 0;
    }
    const double* src = h->buf[h->cur];
    double* dst = h->buf[1 - h->cur];
    const int grid = h->nsm - std::min(step2_halo_sms(), h->nsm / 4);
    int nsig = 0;
    const bool tl = h->prof_on;
    if (tl) {
        for (cudaEvent_t& e : h->tl)
            if (!e) CK(cudaEventCreate(&e));
        CK(cudaEventRecord(h->tl[0], h->stream));
    }
    if (wait) {
        ProfScope ps(h, kProfFused);
        cudaError_t err = cudaSuccess;
        if (step2_form() == kStep2Pair) {  // the two-threads-per-site form (wall faces beside it)
            nsig = launch_step2_pair_slab(src, dst, h->g, fc, h->mp, omega, h->d_flag, h->stream, grid,
                                          h->d_sweep_counter, h->h6[0], h->h6[1], &err);
            CK(err);
        }
        if (nsig == 0) {
            nsig = launch_step2_slab(src, dst, h->g, fc, h->mp, omega, h->d_flag, h->stream, grid,
                                     h->d_sweep_counter, h->h6[0], h->h6[1], &err);
            CK(err);
        }
    }
    if (nsig == 0) {  // no overlapped form for this slab (small, periodic face): the serial schedule
        RET(step2_local(h, omega, fc));
        h->h6_valid = false;
        return D2Q37_OK;
    }
    h->sweep_target += unsigned(nsig);
    {  // the halo pipeline of the new state, beside the interior
        const int lo = lo_peer_of(h, bc), hi = hi_peer_of(h, bc);
        if (wait(reinterpret_cast<CUstream>(h->comm_stream), reinterpret_cast<CUdeviceptr>(h->d_sweep_counter),
                 h->sweep_target, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return fail(D2Q37_ERR_CUDA, "cuStreamWaitValue32 failed");
        if (tl) CK(cudaEventRecord(h->tl[1], h->comm_stream));
        std::string why;
        const int rc = nccl_exchange(h->comm, h->comm_stream, h->h6[0], h->h6[2], lo, h->h6[1], h->h6[3], hi,
                                     halo6_count(h->g), &why);
        if (rc != D2Q37_OK) return fail(rc, "%s", why.c_str());
        if (tl) CK(cudaEventRecord(h->tl[2], h->comm_stream));
        {
            ProfScope ps(h, kProfEdge, h->comm_stream);
            CK(launch_unpack6(dst, h->g, lo >= 0 ? h->h6[2] : nullptr, hi >= 0 ? h->h6[3] : nullptr,
                              h->comm_stream));
        }
        if (tl) CK(cudaEventRecord(h->tl[3], h->comm_stream));
        CK(cudaEventRecord(h->ev_recv, h->comm_stream));
    }
    if (tl) {
        CK(cudaEventRecord(h->tl[4], h->stream));
        h->tl_valid = true;
    }
    // exposed halo: from the end of the sweep to the end of the exchange
    CK(cudaEventRecord(h->ev_int[h->ev_count % kEventRing], h->stream));
    CK(cudaStreamWaitEvent(h->stream, h->ev_recv, 0));
    CK(cudaEventRecord(h->ev_wait[h->ev_count % kEventRing], h->stream));
    ++h->ev_count;
    h->cur = 1 - h->cur;
    h->time_step += 2;
    h->h6_valid = true;
    return D2Q37_OK;
}

int step2_group_exchange(std::vector<d2q37_lattice*>& slabs, int bc) {
    for (d2q37_lattice* h : slabs) {
        RET(ensure_halo6(h));
        ProfScope ps(h, kProfPack);
        CK(launch_pack6(h->buf[h->cur], h->g, h->h6[0], h->h6[1], h->stream));
    }
    for (d2q37_lattice* h : slabs) {
        const size_t bytes = halo6_count(h->g) * sizeof(double);
        const int lo = lo_peer_of(h, bc), hi = hi_peer_of(h, bc);
        if (lo >= 0) CK(cudaMemcpyAsync(h->h6[2], slabs[lo]->h6[1], bytes, cudaMemcpyDeviceToDevice, h->stream));
        if (hi >= 0) CK(cudaMemcpyAsync(h->h6[3], slabs[hi]->h6[0], bytes, cudaMemcpyDeviceToDevice, h->stream));
    }
    for (d2q37_lattice* h : slabs) {
        const int lo = lo_peer_of(h, bc), hi = hi_peer_of(h, bc);
        ProfScope ps(h, kProfEdge);
        CK(launch_unpack6(h->buf[h->cur], h->g, lo >= 0 ? h->h6[2] : nullptr, hi >= 0 ? h->h6[3] : nullptr,
                          h->stream));
    }
    return D2Q37_OK;
}

void drop_step_graph(d2q37_lattice* h) {
    if (h->graph.exec) cudaGraphExecDestroy(h->graph.exec);
    h->graph = d2q37_lattice::StepGraph{};
}

// Captures kGraphSteps single-domain steps (edge + fused, or edge + propagate +
// collide) into one executable graph, keyed by everything the kernels bake in.
// On any capture failure (e.g. a legacy default stream) graphs stay off and
// d2q37_step launches directly.
int ensure_step_graph(d2q37_lattice* h, double omega, int variant, int bc) {
    auto& gr = h->graph;
    if (gr.exec && gr.omega == omega && gr.variant == variant && gr.bc == bc && gr.cur == h->cur &&
        gr.math == h->math && gr.model_gen == h->model_gen && gr.stream == h->stream && gr.form == 2 * step2_form() + step2_sched())
        return D2Q37_OK;
    drop_step_graph(h);
    const int cur0 = h->cur;
    const long ts0 = h->time_step;
    if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        (void)cudaGetLastError();
        return D2Q37_OK;
    }
    int rc = D2Q37_OK;
    if (variant == D2Q37_FUSED2) {  // kGraphSteps two-step sweeps (an even number: cur is unchanged)
        const Faces fc = step_faces(h, bc);
        for (int i = 0; i < kGraphSteps && rc == D2Q37_OK; ++i) rc = step2_local(h, omega, fc);
    } else {
        for (int i = 0; i < kGraphSteps && rc == D2Q37_OK; ++i) rc = step_local(h, omega, variant, bc);
    }
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(h->stream, &graph);
    h->cur = cur0;  // capture only recorded the launches
    h->time_step = ts0;
    if (rc != D2Q37_OK || ec != cudaSuccess || !graph) {
        if (graph) cudaGraphDestroy(graph);
        (void)cudaGetLastError();
        return rc;
    }
    const cudaError_t ei = cudaGraphInstantiate(&gr.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        gr.exec = nullptr;
        (void)cudaGetLastError();
        return D2Q37_OK;
    }
    gr.omega = omega;
    gr.variant = variant;
    gr.bc = bc;
    gr.cur = h->cur;
    gr.math = h->math;
    gr.model_gen = h->model_gen;
    gr.stream = h->stream;
    gr.form = 2 * step2_form() + step2_sched();
    return D2Q37_OK;
}

// Launches in scope go to `s` (the kernels and ProfScope use h->stream).
struct OnStream {
    d2q37_lattice* h;
    cudaStream_t saved;
    OnStream(d2q37_lattice* h_, cudaStream_t s) : h(h_), saved(h_->stream) { h->stream = s; }
    ~OnStream() { h->stream = saved; }
};

// One fused slab step with the halo work hidden behind the interior:
//   compute stream:  interior sites (everything whose pull stays local) ... join
//   halo stream (high priority): pack -> | wait halos -> remote ghost rows -> boundary sites
//   comm stream:                          NCCL send/recv
// The interior and the boundary write disjoint sites of the next buffer; the
// interior reads no ghost row the halo stream writes.
int slab_step_overlapped(d2q37_lattice* h, double omega, int bc) {
    CK(cudaEventRecord(h->ev_start, h->stream));
    CK(cudaStreamWaitEvent(h->halo_stream, h->ev_start, 0));
    {
        OnStream on(h, h->halo_stream);
        RET(exchange_begin(h, bc));  // pack on the halo stream, NCCL on the comm stream
    }
    RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, interior(h, bc), 1, step_faces(h, bc)));
    const int ring = h->ev_count % kEventRing;
    CK(cudaEventRecord(h->ev_int[ring], h->stream));
    {
        OnStream on(h, h->halo_stream);
        RET(exchange_wait(h));
        RET(edge(h, bc, kEdgeRemote));
        int nseg = 0;
        const Segments bnd = boundary(h, bc, &nseg);
        RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, bnd, nseg, step_faces(h, bc)));
        CK(cudaEventRecord(h->ev_bnd, h->halo_stream));
    }
    CK(cudaStreamWaitEvent(h->stream, h->ev_bnd, 0));
    CK(cudaEventRecord(h->ev_wait[ring], h->stream));  // exposed halo: interior done -> boundary done
    ++h->ev_count;
    h->cur = 1 - h->cur;
    ++h->time_step;
    return D2Q37_OK;
}

// ---- y-major slabs: the slab faces are whole storage columns ---------------
//
// A neighbour needs our 3 physical columns next to the shared face; they
// arrive in our 3 ghost columns.  Both are contiguous runs of the state buffer
// (site-major layouts keep a column's 37 populations together), so NCCL sends
// and receives straight from / into the lattice: no pack, no unpack.

double* ycols(d2q37_lattice* h, int X) { return h->buf[h->cur] + h->g.lead + (long long)X * h->g.cstride; }
size_t ycols_count(const d2q37_lattice* h) { return size_t(kHalo) * size_t(h->g.cstride); }

int ymajor_exchange_nccl(d2q37_lattice* h, int bc) {
    const int lx = h->g.lx;
    std::string why;
    const int rc = nccl_exchange(h->comm, h->comm_stream, ycols(h, kHalo), ycols(h, 0), lo_peer_of(h, bc),
                                 ycols(h, lx), ycols(h, lx + kHalo), hi_peer_of(h, bc), ycols_count(h), &why);
    if (rc != D2Q37_OK) return fail(rc, "%s", why.c_str());
    CK(cudaEventRecord(h->ev_recv, h->comm_stream));
    return D2Q37_OK;
}

int ymajor_group_exchange(std::vector<d2q37_lattice*>& slabs, int bc) {
    for (d2q37_lattice* h : slabs) {
        const size_t bytes = ycols_count(h) * sizeof(double);
        const int lo = lo_peer_of(h, bc), hi = hi_peer_of(h, bc);
        if (lo >= 0)
            CK(cudaMemcpyAsync(ycols(h, 0), ycols(slabs[lo], slabs[lo]->g.lx), bytes, cudaMemcpyDeviceToDevice,
                               h->stream));
        if (hi >= 0)
            CK(cudaMemcpyAsync(ycols(h, h->g.lx + kHalo), ycols(slabs[hi], kHalo), bytes, cudaMemcpyDeviceToDevice,
                               h->stream));
    }
    return D2Q37_OK;
}

// Columns whose pull stays inside the slab: all but the 3 next to a remote face.
Segments ycols_interior(const d2q37_lattice* h, int bc) {
    Segments s = all_sites(h->g);
    const bool lo = face_lo_of(h, bc) == kFaceRemote, hi = face_hi_of(h, bc) == kFaceRemote;
    s.x0[0] = lo ? kHalo : 0;
    s.nx = h->g.lx - (lo ? kHalo : 0) - (hi ? kHalo : 0);
    return s;
}

Segments ycols_boundary(const d2q37_lattice* h, int bc, int* nseg) {
    Segments s = all_sites(h->g);
    int n = 0;
    if (face_lo_of(h, bc) == kFaceRemote) s.x0[n++] = 0;
    if (face_hi_of(h, bc) == kFaceRemote) s.x0[n++] = h->g.lx - kHalo;
    s.nx = kHalo;
    *nseg = n;
    return s;
}

// Fused y-major slab step over NCCL: the interior columns on the compute
// stream while the halo columns travel, the 3 + 3 boundary columns on the
// high-priority halo stream once they landed.
int ymajor_step_nccl(d2q37_lattice* h, double omega, int bc) {
    CK(cudaEventRecord(h->ev_start, h->stream));
    CK(cudaStreamWaitEvent(h->comm_stream, h->ev_start, 0));
    RET(ymajor_exchange_nccl(h, bc));
    const Faces fc = step_faces(h, bc);
    RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, ycols_interior(h, bc), 1, fc));
    const int ring = h->ev_count % kEventRing;
    CK(cudaEventRecord(h->ev_int[ring], h->stream));
    {
        OnStream on(h, h->halo_stream);
        CK(cudaStreamWaitEvent(h->halo_stream, h->ev_recv, 0));
        int nseg = 0;
        const Segments bnd = ycols_boundary(h, bc, &nseg);
        RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, bnd, nseg, fc, true));
        CK(cudaEventRecord(h->ev_bnd, h->halo_stream));
    }
    CK(cudaStreamWaitEvent(h->stream, h->ev_bnd, 0));
    CK(cudaEventRecord(h->ev_wait[ring], h->stream));
    ++h->ev_count;
    h->cur = 1 - h->cur;
    ++h->time_step;
    return D2Q37_OK;
}

// Unfused y-major slab step over NCCL: exchange, then propagate + collide.
int ymajor_step_nccl_unfused(d2q37_lattice* h, double omega, int bc) {
    CK(cudaEventRecord(h->ev_start, h->stream));
    CK(cudaStreamWaitEvent(h->comm_stream, h->ev_start, 0));
    RET(ymajor_exchange_nccl(h, bc));
    CK(cudaStreamWaitEvent(h->stream, h->ev_recv, 0));
    return step_local(h, omega, D2Q37_UNFUSED, bc);
}

// ---- P2P y-major slabs: halos pushed through peer memory ------------------
//
// Step k (counter seq = k) of every rank, with ping-pong buffers in lockstep:
//   compute stream: interior columns (no ghost reads, no remote writes)
//   halo stream:    wait until both neighbours finished step k-1 (their
//                   counters >= seq-1: my ghost columns hold their step k-1
//                   faces, and they no longer read the ghost columns of the
//                   buffer I am about to write) -> the 3 + 3 face columns, whose
//                   fused kernel also stores its results into the neighbours'
//                   next buffers (ghost columns) over NVLink -> signal seq.
// No NCCL, no pack, no exchange buffers: the halo travels with the kernel's
// own stores.  A prime (after load / init / swap) pushes the current face
// columns with peer copies under the same counter protocol.

// How long a rank waits for a neighbour before reporting instead of hanging:
// D2Q37_P2P_TIMEOUT_S (default 60 s).
unsigned long long p2p_timeout_ns() {
    static const unsigned long long ns = [] {
        const char* v = std::getenv("D2Q37_P2P_TIMEOUT_S");
        const double sec = v ? std::atof(v) : 60.0;
        return (unsigned long long)((sec > 0 ? sec : 60.0) * 1e9);
    }();
    return ns;
}

int p2p_wait(d2q37_lattice* h, int bc, unsigned long long target) {
    CK(launch_p2p_wait(h->d_seq, face_lo_of(h, bc) == kFaceRemote, face_hi_of(h, bc) == kFaceRemote, target,
                       p2p_timeout_ns(), h->d_flag, h->halo_stream));
    return D2Q37_OK;
}

int p2p_signal(d2q37_lattice* h, int bc, unsigned long long value) {
    CK(launch_p2p_signal(face_lo_of(h, bc) == kFaceRemote ? h->peer_seq_slot[0] : nullptr,
                         face_hi_of(h, bc) == kFaceRemote ? h->peer_seq_slot[1] : nullptr, value, h->halo_stream));
    return D2Q37_OK;
}

// The face sites of a P2P slab for bc (both orientations) and the element
// shifts that map each face site onto the neighbour's ghost slot for it.
//   y-major: 3 storage columns per face; my column x < 3 is the lo
//            neighbour's ghost column lx + 3 + x (shift +lx*cstride), my column
//            lx - 3 + c is the hi neighbour's ghost column c (-lx*cstride).
//   x-major: lane 0's rows r < 3 are the lo neighbour's lane vl-1 ghost rows
//            strip + 3 + r (shift +strip*rstride + vl-1); lane vl-1's last rows
//            are the hi neighbour's lane-0 ghost rows (the negative shift).
Segments p2p_faces(const d2q37_lattice* h, int bc, int* nseg) {
    return h->g.tr ? ycols_boundary(h, bc, nseg) : boundary(h, bc, nseg);
}

PeerStores p2p_peers(const d2q37_lattice* h, int bc, int buffer) {
    const DevGeo& g = h->g;
    const long long span = g.tr ? (long long)g.lx * g.cstride : (long long)g.strip * g.rstride + (g.vl - 1);
    PeerStores ps{};
    if (face_lo_of(h, bc) == kFaceRemote) {
        ps.lo = h->peer_buf[0][buffer];
        ps.lo_shift = span;
    }
    if (face_hi_of(h, bc) == kFaceRemote) {
        ps.hi = h->peer_buf[1][buffer];
        ps.hi_shift = -span;
    }
    return ps;
}

// Pushes the current state's face sites into the neighbours' current ghost
// slots, then signals; waits for the neighbours' pushes into mine.  Invariant
// of the counters: a neighbour's counter >= s means its operation s has
// finished both its pushes and its reads of its own ghost slots, so waiting
// for s - 1 before writing into its buffers is safe.
int p2p_prime(d2q37_lattice* h, int bc) {
    const unsigned long long seq = ++h->p2p_seq;
    CK(cudaEventRecord(h->ev_start, h->stream));
    CK(cudaStreamWaitEvent(h->halo_stream, h->ev_start, 0));
    RET(p2p_wait(h, bc, seq - 1));
    int nseg = 0;
    const Segments faces = p2p_faces(h, bc, &nseg);
    CK(launch_face_prime(h->buf[h->cur], h->g, h->off_pull, faces, nseg, p2p_peers(h, bc, h->cur), h->halo_stream));
    RET(p2p_signal(h, bc, seq));
    RET(p2p_wait(h, bc, seq));  // the neighbours' pushes into my ghost slots
    CK(cudaEventRecord(h->ev_bnd, h->halo_stream));
    CK(cudaStreamWaitEvent(h->stream, h->ev_bnd, 0));
    h->p2p_dirty = false;
    return D2Q37_OK;
}

int p2p_step(d2q37_lattice* h, double omega, int variant, int bc) {
    if (!h->p2p_connected) return fail(D2Q37_ERR_INVALID_ARGUMENT, "p2p slab is not connected to its neighbours");
    if (h->p2p_dirty) RET(p2p_prime(h, bc));
    if (variant != D2Q37_FUSED) {
        // unfused: push the faces (counter c1), run the local verbs, then signal c1 + 1 once
        // they are done reading the ghost slots -- the state stays in the same buffer, so a
        // neighbour's next push must not land while propagate is still reading
        RET(p2p_prime(h, bc));
        RET(step_local(h, omega, D2Q37_UNFUSED, bc));
        const unsigned long long done = ++h->p2p_seq;
        CK(cudaEventRecord(h->ev_start, h->stream));
        CK(cudaStreamWaitEvent(h->halo_stream, h->ev_start, 0));
        RET(p2p_signal(h, bc, done));
        return D2Q37_OK;
    }
    const unsigned long long seq = ++h->p2p_seq;
    const Faces fc = step_faces(h, bc);
    CK(cudaEventRecord(h->ev_start, h->stream));
    CK(cudaStreamWaitEvent(h->halo_stream, h->ev_start, 0));
    // interior: every site whose pull stays inside the slab (no ghost reads, no remote writes)
    RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, h->g.tr ? ycols_interior(h, bc) : interior(h, bc), 1,
                       fc));
    const int ring = h->ev_count % kEventRing;
    CK(cudaEventRecord(h->ev_int[ring], h->stream));
    {
        OnStream on(h, h->halo_stream);
        RET(p2p_wait(h, bc, seq - 1));
        int nseg = 0;
        const Segments faces = p2p_faces(h, bc, &nseg);
        {
            ProfScope prof(h, kProfBoundary);
            CK(launch_face(h->buf[h->cur], h->buf[1 - h->cur], h->g, h->off_pull, fc, h->mp, omega,
                           h->math == D2Q37_MATH_STRICT, faces, nseg, p2p_peers(h, bc, 1 - h->cur), h->d_flag,
                           h->stream));
        }
        RET(p2p_signal(h, bc, seq));
        CK(cudaEventRecord(h->ev_bnd, h->halo_stream));
    }
    CK(cudaStreamWaitEvent(h->stream, h->ev_bnd, 0));
    CK(cudaEventRecord(h->ev_wait[ring], h->stream));
    ++h->ev_count;
    h->cur = 1 - h->cur;
    ++h->time_step;
    return D2Q37_OK;
}

// Slab step, phase 1 (before the halos are needed): the interior rows, whose
// pull stencil stays inside the slab (x wrap and lane shifts in-kernel).
int slab_phase1(d2q37_lattice* h, double omega, int variant, int bc) {
    if (variant == D2Q37_FUSED && can_split(h)) {
        RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, interior(h, bc), 1, step_faces(h, bc)));
        if (h->transport == kTransportNccl) CK(cudaEventRecord(h->ev_int[h->ev_count % kEventRing], h->stream));
    }
    return D2Q37_OK;
}

// Slab step, phase 2 (after the halos landed): remote ghost rows + boundary rows.
int slab_phase2(d2q37_lattice* h, double omega, int variant, int bc) {
    RET(exchange_wait(h));
    const bool split = variant == D2Q37_FUSED && can_split(h);
    if (h->transport == kTransportNccl && split) {
        CK(cudaEventRecord(h->ev_wait[h->ev_count % kEventRing], h->stream));
        ++h->ev_count;
    }
    RET(edge(h, bc, kEdgeRemote));
    const Faces fc = step_faces(h, bc);
    const Segments all = all_sites(h->g);
    if (variant == D2Q37_FUSED) {
        int nseg = 0;
        const Segments bnd = boundary(h, bc, &nseg);
        if (split)
            RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, bnd, nseg, fc));
        else
            RET(collide_launch(h, h->cur, 1 - h->cur, omega, true, all, 1, fc));
        h->cur = 1 - h->cur;
    } else {
        RET(propagate_launch(h, h->off_pull, fc));
        RET(collide_launch(h, 1 - h->cur, h->cur, omega, false, all, 1, fc));
    }
    ++h->time_step;
    return D2Q37_OK;
}

// Two staging planes, a copy stream and 4 events for pipelined host transfers.
int ensure_io_pipeline(d2q37_lattice* h, size_t plane_vals) {
    if (!h->stage) CK(cudaMalloc(&h->stage, plane_vals * sizeof(double)));
    if (!h->stage2) CK(cudaMalloc(&h->stage2, plane_vals * sizeof(double)));
    if (!h->copy_stream) CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : h->ev_io)
        if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return D2Q37_OK;
}

int load_canonical_impl(d2q37_lattice* h, int which, const double* src, size_t n, bool src_device) {
    if (h) h->p2p_dirty = true, h->h6_valid = false, h->bc_filled = -1;
    RET(check_handle(h));
    if (which != 0 && which != 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "buffer index must be 0 (prv) or 1 (nxt)");
    if (n != canon_count(h)) return fail(D2Q37_ERR_INVALID_ARGUMENT, "from_canonical: dimension mismatch");
    if (!src) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null canonical array");
    DeviceGuard dg(h->device);
    const DevGeo& g = h->g;
    double* dst = h->buf[which == 0 ? h->cur : 1 - h->cur];
    const size_t plane_vals = size_t(g.lx) * g.ly;
    if (h->layout == D2Q37_SOA && !src_device) {
        // SoA: one pitched copy per population straight from the host array.
        for (int p = 0; p < kNpop; ++p)
            CK(cudaMemcpy2DAsync(dst + site_of(g, kHalo, 0) + p * g.pstride, size_t(g.cstride) * sizeof(double),
                                 src + p * plane_vals, size_t(g.ly) * sizeof(double), size_t(g.ly) * sizeof(double),
                                 size_t(g.lx), cudaMemcpyHostToDevice, h->stream));
    } else if (src_device) {
        for (int p = 0; p < kNpop; ++p) CK(launch_scatter(dst, g, src + p * plane_vals, p, h->stream));
    } else {
        // plane p's H2D copy (copy stream) overlaps plane p-1's scatter (compute stream)
        RET(ensure_io_pipeline(h, plane_vals));
        double* stage[2] = {h->stage, h->stage2};
        cudaEvent_t* copied = h->ev_io;        // [2]
        cudaEvent_t* consumed = h->ev_io + 2;  // [2]
        CK(cudaEventRecord(consumed[0], h->stream));  // orders the copies after prior work on the lattice
        CK(cudaEventRecord(consumed[1], h->stream));
        for (int p = 0; p < kNpop; ++p) {
            const int b = p & 1;
            CK(cudaStreamWaitEvent(h->copy_stream, consumed[b], 0));
            CK(cudaMemcpyAsync(stage[b], src + p * plane_vals, plane_vals * sizeof(double), cudaMemcpyHostToDevice,
                               h->copy_stream));
            CK(cudaEventRecord(copied[b], h->copy_stream));
            CK(cudaStreamWaitEvent(h->stream, copied[b], 0));
            CK(launch_scatter(dst, g, stage[b], p, h->stream));
            CK(cudaEventRecord(consumed[b], h->stream));
        }
    }
    CK(cudaStreamSynchronize(h->stream));
    return D2Q37_OK;
}

int dump_canonical_impl(d2q37_lattice* h, int which, double* out, size_t n, bool out_device) {
    RET(check_handle(h));
    if (which != 0 && which != 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "buffer index must be 0 (prv) or 1 (nxt)");
    if (n != canon_count(h)) return fail(D2Q37_ERR_INVALID_ARGUMENT, "to_canonical: dimension mismatch");
    if (!out) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null canonical array");
    DeviceGuard dg(h->device);
    const DevGeo& g = h->g;
    const double* src = h->buf[which == 0 ? h->cur : 1 - h->cur];
    const size_t plane_vals = size_t(g.lx) * g.ly;
    if (h->layout == D2Q37_SOA && !out_device) {
        for (int p = 0; p < kNpop; ++p)
            CK(cudaMemcpy2DAsync(out + p * plane_vals, size_t(g.ly) * sizeof(double),
                                 src + site_of(g, kHalo, 0) + p * g.pstride, size_t(g.cstride) * sizeof(double),
                                 size_t(g.ly) * sizeof(double), size_t(g.lx),
                                 cudaMemcpyDeviceToHost, h->stream));
    } else if (out_device) {
        for (int p = 0; p < kNpop; ++p) CK(launch_gather(src, g, out + p * plane_vals, p, h->stream));
    } else {
        // plane p's gather (compute stream) overlaps plane p-1's D2H copy (copy stream)
        RET(ensure_io_pipeline(h, plane_vals));
        double* stage[2] = {h->stage, h->stage2};
        cudaEvent_t* gathered = h->ev_io;     // [2]
        cudaEvent_t* drained = h->ev_io + 2;  // [2]
        CK(cudaEventRecord(drained[0], h->copy_stream));
        CK(cudaEventRecord(drained[1], h->copy_stream));
        for (int p = 0; p < kNpop; ++p) {
            const int b = p & 1;
            CK(cudaStreamWaitEvent(h->stream, drained[b], 0));
            CK(launch_gather(src, g, stage[b], p, h->stream));
            CK(cudaEventRecord(gathered[b], h->stream));
            CK(cudaStreamWaitEvent(h->copy_stream, gathered[b], 0));
            CK(cudaMemcpyAsync(out + p * plane_vals, stage[b], plane_vals * sizeof(double), cudaMemcpyDeviceToHost,
                               h->copy_stream));
            CK(cudaEventRecord(drained[b], h->copy_stream));
        }
        CK(cudaStreamSynchronize(h->copy_stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    return D2Q37_OK;
}

// ---- streamed run: load -> nsteps FUSED2 steps -> dump, pipelined in y-chunks -------------------
//
// d2q37_run_canonical on a single SoA domain (walls; y-periodic: stream_plan).  The canonical host array
// is [p][x][y] (dump.hpp:19-21), so rows [r0, r1) of every population are one pitched copy each; chunk k
// of the input is uploaded on the copy stream while the compute stream sweeps the chunks before it, and
// finished rows are downloaded on a second copy stream (the other DMA direction) while later chunks
// are still being swept.  A FUSED2 sweep s (two steps) of rows [a, b) needs sweep s - 1 on rows
// [a - 6, b + 6), so chunk k is swept as a parallelogram: sweep s covers rows
//     [edge[k] - d s, edge[k+1] - d s),  d >= 6   (clipped at row 0; the last chunk ends at ly)
// and every sweep's input rows are then final when it is launched (all in stream order on the compute
// stream).  The two state buffers still alternate (X_s = sweep s's output; X_s and X_{s-2} share a
// buffer): sweep s on chunk k overwrites X_{s-2} rows below edge[k+1] - d s, and the only reader of
// X_{s-2} still to come -- sweep s - 1 on chunk k + 1 -- reads rows from edge[k+1] - d s + d - 6 on.  The
// sweep of a row range is the pair form on a pointer-shifted geometry with ghost faces
// (k_step2_pair<true>, rows beyond the range read as they stand, like a slab's deep ghost rows); the
// walls stay the wall images of step2_local (k_mirror6 once a sweep's rows 0..5 / ly-6..ly-1 are
// complete).  Results are bit-identical to load + step + dump (same kernel, same values).  The schedule
// is built as a list of operations (stream_plan) that run_streamed executes and
// tests/test_stream_plan.py replays on a model of the two buffers.
int seam_rows(int S, int skew);
int stream_skew();

bool can_stream_run(const d2q37_lattice* h, int nsteps, int variant, int bc, const Faces& fc) {
    const bool walls = bc == D2Q37_BC_WALL && fc.lo == kFaceWall && fc.hi == kFaceWall && step2_ghost_walls();
    const bool per = bc == D2Q37_BC_PERIODIC && fc.lo == kFacePeriodic && fc.hi == kFacePeriodic;
    if (!(h->layout == D2Q37_SOA && !h->g.band && h->g.deep && !h->g.tr && h->g.vl == 1 && local_only(h) &&
          h->math == D2Q37_MATH_FAST && variant == D2Q37_FUSED2 && (walls || per) && step2_form() == kStep2Pair &&
          step2_supported(h->g, fc) && nsteps >= 2 && nsteps % 2 == 0 && h->g.ly >= 4 * step2_band_rows() &&
          !h->prof_on))
        return false;
    // y-periodic: room for the two seam pieces and a wave between them
    return !per || h->g.ly >= 2 * seam_rows(nsteps / 2, stream_skew()) + 4 * step2_band_rows();
}

// Chunk edges (multiples of 4 rows).  The sweeps take longer than the copies, so only the first upload
// and the last download are exposed: the chunk heights double from D2Q37_STREAM_FIRST (2 bands) while
// they stay within half of D2Q37_STREAM_ROWS (37 bands: 4 CTAs per band on 148 SMs, the lockstep
// plan's even split) -- the upload stays ahead of the sweeps as long as a chunk is little more than
// twice the rows before it -- and halve again down to D2Q37_STREAM_LAST (1 band) at the top wall, whose
// last chunk (plus the d rows per sweep the parallelograms lean back) is downloaded after the last
// sweep.  Band counts of 2^n and 37 divide the 148 CTAs (almost) evenly.
std::vector<int> stream_edges(int ly) {
    const int band = step2_band_rows();
    auto env_rows = [](const char* name, int dflt) {
        const char* e = std::getenv(name);
        const int v = e ? std::atoi(e) : dflt;
        return std::max(2 * kHalo, v) & ~1;
    };
    const int rows = env_rows("D2Q37_STREAM_ROWS", 37 * band);
    const int first = std::min(rows, env_rows("D2Q37_STREAM_FIRST", 2 * band));
    const int last = std::min(rows, env_rows("D2Q37_STREAM_LAST", band));
    std::vector<int> head, tail;
    long long used = 0;
    for (int h = first, t = last; used + h + t <= ly && (2 * h <= rows || 2 * t <= rows);) {
        if (2 * h <= rows) head.push_back(h), used += h, h *= 2;
        if (used + t <= ly && 2 * t <= rows) tail.push_back(t), used += t, t *= 2;
        if (head.size() + tail.size() > 64) break;
    }
    std::vector<int> edge{0};
    for (int h : head) edge.push_back(edge.back() + h);
    const int mid_end = ly - int(std::accumulate(tail.begin(), tail.end(), 0LL));
    // the middle: whole `rows` chunks, the remainder spread as one shorter chunk in front of them
    const int mid = mid_end - edge.back();
    if (mid > 0) {
        const int rem = mid % rows;
        if (rem >= 2 * kHalo) edge.push_back(edge.back() + (rem & ~1));
        while (mid_end - edge.back() > rows) edge.push_back(edge.back() + rows);
        if (edge.back() < mid_end) edge.push_back(mid_end);
    }
    for (auto t = tail.rbegin(); t != tail.rend(); ++t) edge.push_back(edge.back() + *t);
    edge.back() = ly;
    // no sliver (< 6 rows) and no empty chunk anywhere
    std::vector<int> out{0};
    for (size_t i = 1; i < edge.size(); ++i) {
        const int e = edge[i] == ly ? ly : edge[i] & ~3;  // inner edges on 32-byte sectors (even: 16-byte bulk copies)
        if (e - out.back() >= 2 * kHalo && (ly - e >= 2 * kHalo || e == ly)) out.push_back(e);
    }
    if (out.back() != ly) out.back() == 0 ? out.push_back(ly) : void(out.back() = ly);
    return out;
}

// Rows the seam pieces of a y-periodic streamed run need beyond the d rows per sweep they lose
// (the seam's wrap images mirror 6 rows on each side; two bands of margin keep the launches useful)
int seam_rows(int S, int skew) { return skew * S + 2 * step2_band_rows(); }

// The streamed run as a list of operations (also exported to the host-side schedule test,
// d2q37_debug_stream_plan): uploads first (copy stream, in order), then the compute stream's operations in
// order; a download follows everything before it on the compute stream (second copy stream).
enum { kOpUpload = 0, kOpWaitUpload = 1, kOpSweep = 2, kOpMirror = 3, kOpWrap = 4, kOpDownload = 5 };
struct StreamOp {
    int kind;
    int a, b;  // rows [a, b) (upload, sweep, download); mirror: a = face mask
    int c;     // upload / wait: upload index; sweep / mirror / wrap: the sweep s whose output (or, s = 0,
               // the uploaded state) it writes / completes
};

int stream_skew() {
    // rows a chunk's range moves down per sweep: at least the 6 a sweep reaches; 8 keeps the bands'
    // 960-byte column stores on 32-byte sectors (D2Q37_STREAM_SKEW)
    const char* skew_env = std::getenv("D2Q37_STREAM_SKEW");
    return std::max(2 * kHalo, skew_env ? std::atoi(skew_env) & ~1 : 8);
}

int stream_min_download_rows() {
    const char* e = std::getenv("D2Q37_STREAM_MIN_DOWNLOAD");
    return e ? std::max(1, std::atoi(e)) : 240;
}

std::vector<StreamOp> stream_plan(int ly, int S, bool per) {
    const int skew = stream_skew();
    // y-periodic: the two pieces at the seam, BOT = [0, base) and TOP = [top0, ly), are uploaded first and
    // swept together -- sweep s on [0, base - d s) and [top0 + d s, ly), then the periodic images of the
    // new state's rows 0..5 / ly-6..ly-1 (k_wrap6) -- losing d rows per sweep on their far sides; the wave
    // of chunks then runs over [base, top0) as between walls, its last chunk growing into the rows TOP
    // lost: sweep s up to top0 + d s.  Walls: base = 0, top0 = ly, no seam pieces.
    const int base = per ? seam_rows(S, skew) & ~3 : 0, top0 = per ? (ly - seam_rows(S, skew)) & ~3 : ly;
    std::vector<int> edge = stream_edges(top0 - base);
    for (int& e : edge) e += base;
    const int K = int(edge.size()) - 1;
    std::vector<StreamOp> ops;
    int nup = 0;
    if (per) {
        ops.push_back({kOpUpload, top0, ly, nup});
        ops.push_back({kOpUpload, 0, base, nup++});  // (one event after both)
    }
    const int up0 = nup;
    for (int k = 0; k < K; ++k) ops.push_back({kOpUpload, edge[k], edge[k + 1], nup++});
    auto sweep = [&](int s, int lo, int hi) {
        if (hi > lo) ops.push_back({kOpSweep, lo, hi, s});
    };
    if (per) {
        ops.push_back({kOpWaitUpload, 0, 0, 0});
        ops.push_back({kOpWrap, 0, 0, 0});
        for (int s = 1; s <= S; ++s) {
            sweep(s, top0 + skew * s, ly);
            sweep(s, 0, base - skew * s);
            ops.push_back({kOpWrap, 0, 0, s});
        }
        ops.push_back({kOpDownload, top0 + skew * S, ly, 0});
        ops.push_back({kOpDownload, 0, base - skew * S, 0});
    }
    // final rows narrower than this wait for the next chunk's download (a first download of a few dozen
    // rows -- e.g. 170 or 400 steps on 4096 x 16384 -- measured 0.5-1 s slower per run; DESIGN 3.3)
    const int min_dl = stream_min_download_rows();
    int dl_lo = -1;
    for (int k = 0; k < K; ++k) {
        const bool last = k == K - 1;
        ops.push_back({kOpWaitUpload, 0, 0, up0 + k});
        if (!per && k == 0) ops.push_back({kOpMirror, 1, 0, 0});
        if (!per && last) ops.push_back({kOpMirror, 2, 0, 0});
        int lo = 0, hi = 0;
        for (int s = 1; s <= S; ++s) {
            lo = !per && k == 0 ? 0 : std::max(0, edge[k] - skew * s);
            hi = last ? (per ? top0 + skew * s : ly) : std::max(0, edge[k + 1] - skew * s);
            sweep(s, lo, hi);
            if (!per && hi > lo) {
                // wall images once the six rows they mirror are complete: the launch that wrote row 5 (a
                // range clipped at row 0 may end below it; the chunk above then finishes the rows) / the
                // last chunk's (it always reaches from below ly - 6 to ly)
                const int mask = (lo < 2 * kHalo && hi >= 2 * kHalo ? 1 : 0) | (hi == ly ? 2 : 0);
                if (mask) ops.push_back({kOpMirror, mask, 0, s});
            }
        }
        if (hi > lo) {
            const int from = dl_lo >= 0 ? dl_lo : lo;
            if (!last && hi - from < min_dl) {
                dl_lo = from;
            } else {
                ops.push_back({kOpDownload, from, hi, 0});
                dl_lo = -1;
            }
        }
    }
    return ops;
}

int run_streamed(d2q37_lattice* h, const double* in, double* out, double omega, int nsteps, const Faces& fc) {
    DeviceGuard dg(h->device);
    const DevGeo& g = h->g;
    if (!h->nsm) CK(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->device));
    if (!h->copy_stream) CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    if (!h->copy_stream2) CK(cudaStreamCreateWithFlags(&h->copy_stream2, cudaStreamNonBlocking));
    const int S = nsteps / 2;
    const bool per = fc.lo == kFacePeriodic;
    const std::vector<StreamOp> ops = stream_plan(g.ly, S, per);
    size_t nev = 1;
    for (const StreamOp& op : ops) nev += op.kind == kOpUpload || op.kind == kOpDownload;
    std::vector<cudaEvent_t> ev(nev, nullptr);
    struct EventsGuard {
        std::vector<cudaEvent_t>& e;
        ~EventsGuard() {
            for (cudaEvent_t x : e)
                if (x) cudaEventDestroy(x);
        }
    } guard{ev};
    for (cudaEvent_t& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t& start = ev[0];
    cudaEvent_t* const uploaded = ev.data() + 1;  // by upload index (two seam uploads share one)
    size_t next_ev = 1;
    for (const StreamOp& op : ops)
        if (op.kind == kOpUpload) next_ev = std::max(next_ev, size_t(op.c) + 2);
    double* const X[2] = {h->buf[h->cur], h->buf[1 - h->cur]};  // X[s & 1]: the state after sweep s
    const size_t plane_vals = size_t(g.lx) * g.ly;
    const long long row0 = site_of(g, kHalo, 0);
    // timing probes (results are then meaningless): 1 = no copies, 2 = no sweeps, 3 = no downloads, 4 = no uploads
    const char* probe_env = std::getenv("D2Q37_STREAM_PROBE");
    const int probe = probe_env ? std::atoi(probe_env) : 0;
    auto copy_rows = [&](bool up, double* dev, int r0, int r1, cudaStream_t st) -> int {
        for (int p = 0; p < kNpop && r1 > r0 && probe != 1 && probe != (up ? 4 : 3); ++p) {
            double* const d = dev + row0 + p * g.pstride + r0;
            if (up)
                CK(cudaMemcpy2DAsync(d, size_t(g.cstride) * sizeof(double), in + p * plane_vals + r0,
                                     size_t(g.ly) * sizeof(double), size_t(r1 - r0) * sizeof(double), size_t(g.lx),
                                     cudaMemcpyHostToDevice, st));
            else
                CK(cudaMemcpy2DAsync(out + p * plane_vals + r0, size_t(g.ly) * sizeof(double), d,
                                     size_t(g.cstride) * sizeof(double), size_t(r1 - r0) * sizeof(double),
                                     size_t(g.lx), cudaMemcpyDeviceToHost, st));
        }
        return D2Q37_OK;
    };
    Faces gf = fc;
    gf.lo = gf.hi = kFaceGhost;
    const bool lock = step2_sched() != 0;
    cudaStream_t st = h->stream;
    // the copies start after whatever the lattice's stream still has queued
    CK(cudaEventRecord(start, st));
    CK(cudaStreamWaitEvent(h->copy_stream, start, 0));
    CK(cudaStreamWaitEvent(h->copy_stream2, start, 0));
    for (size_t i = 0; i < ops.size(); ++i) {
        const StreamOp& op = ops[i];
        switch (op.kind) {
            case kOpUpload:
                RET(copy_rows(true, X[0], op.a, op.b, h->copy_stream));
                if (i + 1 == ops.size() || ops[i + 1].kind != kOpUpload || ops[i + 1].c != op.c)
                    CK(cudaEventRecord(uploaded[op.c], h->copy_stream));
                break;
            case kOpWaitUpload: CK(cudaStreamWaitEvent(st, uploaded[op.c], 0)); break;
            case kOpSweep: {
                if (probe == 2) break;
                // rows [a, b) of sweep c: the pair form on the pointer-shifted range, ghost faces
                DevGeo gs = g;
                gs.ly = op.b - op.a;
                const int nb = (gs.ly + step2_band_rows() - 1) / step2_band_rows();
                CK(launch_step2_pair(X[(op.c - 1) & 1] + op.a, X[op.c & 1] + op.a, gs, gf, h->mp, omega, h->d_flag, st, 0,
                                     nb, h->nsm, lock));
                break;
            }
            case kOpMirror: CK(launch_mirror6(X[op.c & 1], g, fc, st, op.a)); break;
            case kOpWrap: CK(launch_wrap6(X[op.c & 1], g, st)); break;
            case kOpDownload:
                CK(cudaEventRecord(ev[next_ev], st));
                CK(cudaStreamWaitEvent(h->copy_stream2, ev[next_ev], 0));
                ++next_ev;
                RET(copy_rows(false, X[S & 1], op.a, op.b, h->copy_stream2));
                break;
        }
    }
    h->cur = S & 1 ? 1 - h->cur : h->cur;
    h->time_step += nsteps;
    h->h6_valid = true;
    h->h6_kind = per ? 0 : 1;
    CK(cudaStreamSynchronize(h->copy_stream2));
    CK(cudaStreamSynchronize(h->copy_stream));
    return D2Q37_OK;
}

// ymajor: store the lattice transposed (storage columns along y, rows along x)
// -- the y-slab layout of the site-major layouts, whose slab faces are then
// whole contiguous storage columns.
int create_impl(int layout, int lx, int ly, int vl, int device, d2q37_lattice** out, int rank, int nranks,
                bool ymajor = false) {
    if (!out) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null output handle");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(D2Q37_ERR_INVALID_ARGUMENT, "bad rank %d / %d", rank, nranks);
    if (ly % nranks != 0) return fail(D2Q37_ERR_INVALID_ARGUMENT, "ly=%d not divisible by %d slabs", ly, nranks);
    std::unique_ptr<d2q37_lattice> h(new (std::nothrow) d2q37_lattice());
    if (!h) return fail(D2Q37_ERR_CUDA, "out of host memory");
    if (ymajor) {
        if (ly / nranks < 2 * kHalo + 1)
            return fail(D2Q37_ERR_INVALID_ARGUMENT, "y-major slab needs at least 7 rows per slab");
        RET(make_geometry(layout, ly / nranks, lx, vl, &h->g));
        h->g.tr = 1;
    } else {
        RET(make_geometry(layout, lx, ly / nranks, vl, &h->g));
    }
    h->layout = layout;
    h->device = device;
    h->rank = rank;
    h->nranks = nranks;
    h->y0 = rank * (ly / nranks);
    h->ly_global = ly;
    d2q37_model m;
    build_model(&m);
    RET(upload_model(h.get(), &m));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(D2Q37_ERR_INVALID_ARGUMENT, "device %d of %d", device, ndev);
    const int rc = alloc_lattice(h.get());
    if (rc != D2Q37_OK) {
        free_lattice(h.get());
        return rc;
    }
    *out = h.release();
    return D2Q37_OK;
}

}  // namespace

// =========================================================================
extern "C" {

const char* d2q37_last_error(void) { return g_last_error.c_str(); }

int d2q37_model_d2q37(d2q37_model* out) {
    if (!out) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null model");
    try {
        build_model(out);
    } catch (const std::exception& e) {
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "%s", e.what());
    }
    return D2Q37_OK;
}

int d2q37_create(int layout, int lx, int ly, int vl, int device, d2q37_lattice** out) {
    return create_impl(layout, lx, ly, vl, device, out, 0, 1);
}

int d2q37_destroy(d2q37_lattice* h) {
    if (!h) return D2Q37_OK;
    free_lattice(h);
    delete h;
    return D2Q37_OK;
}

int d2q37_set_model(d2q37_lattice* h, const d2q37_model* m) {
    RET(check_handle(h));
    if (!m) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null model");
    return upload_model(h, m);
}

int d2q37_set_math(d2q37_lattice* h, int math) {
    RET(check_handle(h));
    if (math != D2Q37_MATH_FAST && math != D2Q37_MATH_STRICT) return fail(D2Q37_ERR_INVALID_ARGUMENT, "unknown math mode");
    h->math = math;
    return D2Q37_OK;
}

int d2q37_set_stream(d2q37_lattice* h, void* stream) {
    RET(check_handle(h));
    DeviceGuard dg(h->device);
    CK(cudaStreamSynchronize(h->stream));
    h->stream_owner.reset();
    h->stream = static_cast<cudaStream_t>(stream);
    if (!h->stream) RET(new_stream(h));
    return D2Q37_OK;
}

void* d2q37_get_stream(d2q37_lattice* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int d2q37_geometry(const d2q37_lattice* h, int out[6]) {
    RET(check_handle(h));
    out[0] = h->g.tr ? h->g.ly : h->g.lx;  // lattice extents (y-major storage is transposed)
    out[1] = h->g.tr ? h->g.lx : h->g.ly;
    out[2] = h->g.vl;
    out[3] = h->g.strip;
    out[4] = h->g.sy;
    out[5] = h->g.px;
    return D2Q37_OK;
}

size_t d2q37_device_bytes(const d2q37_lattice* h) {
    if (!h) return 0;
    return 2 * h->buf_elems * sizeof(double) + 4 * size_t(h->nslots) * h->g.lx * sizeof(double) * (h->send_lo ? 1 : 0);
}

long d2q37_time_step(const d2q37_lattice* h) { return h ? h->time_step : -1; }

int d2q37_load_canonical(d2q37_lattice* h, const double* host, size_t n) {
    return load_canonical_impl(h, 0, host, n, false);
}
int d2q37_dump_canonical(d2q37_lattice* h, double* host, size_t n) { return dump_canonical_impl(h, 0, host, n, false); }

int d2q37_run_canonical(d2q37_lattice* h, const double* host_in, double* host_out, size_t n, double omega, int nsteps,
                        int variant, int bc) {
    RET(check_handle(h));
    if (n != canon_count(h)) return fail(D2Q37_ERR_INVALID_ARGUMENT, "run_canonical: dimension mismatch");
    if (!host_in || !host_out) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null canonical array");
    if (nsteps < 0) return fail(D2Q37_ERR_INVALID_ARGUMENT, "nsteps must be >= 0");
    if (variant != D2Q37_FUSED && variant != D2Q37_UNFUSED && variant != D2Q37_FUSED2)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "unknown variant");
    RET(validate_bc(h, bc));
    const Faces fc = step_faces(h, bc);
    const char* off = std::getenv("D2Q37_STREAM_RUN");
    if (!(off && std::atoi(off) == 0) && can_stream_run(h, nsteps, variant, bc, fc)) {
        h->p2p_dirty = true, h->h6_valid = false, h->bc_filled = -1;
        h->last_run_mode = fc.lo == kFacePeriodic ? 2 : 1;
        RET(run_streamed(h, host_in, host_out, omega, nsteps, fc));
        return d2q37_sync(h);
    }
    h->last_run_mode = 0;
    RET(load_canonical_impl(h, 0, host_in, n, false));
    RET(d2q37_step(h, omega, nsteps, variant, bc));
    RET(d2q37_sync(h));
    return dump_canonical_impl(h, 0, host_out, n, false);
}
int d2q37_last_run_mode(const d2q37_lattice* h) { return h ? h->last_run_mode : -1; }

int d2q37_debug_stream_plan(int ly, int nsteps, int bc, int* ops, int cap) {
    if (ly < 1 || nsteps < 2 || nsteps % 2 != 0 || (bc != D2Q37_BC_WALL && bc != D2Q37_BC_PERIODIC))
        return -fail(D2Q37_ERR_INVALID_ARGUMENT, "stream plan: ly >= 1, an even nsteps >= 2, wall or periodic bc");
    const bool per = bc == D2Q37_BC_PERIODIC;
    if (per && ly < 2 * seam_rows(nsteps / 2, stream_skew()) + 4 * step2_band_rows()) return 0;  // three verbs
    const std::vector<StreamOp> plan = stream_plan(ly, nsteps / 2, per);
    for (size_t i = 0; i < plan.size() && int(i) < cap && ops; ++i) {
        ops[4 * i] = plan[i].kind;
        ops[4 * i + 1] = plan[i].a;
        ops[4 * i + 2] = plan[i].b;
        ops[4 * i + 3] = plan[i].c;
    }
    return int(plan.size());
}

int d2q37_load_buffer(d2q37_lattice* h, int which, const double* host, size_t n) {
    return load_canonical_impl(h, which, host, n, false);
}
int d2q37_dump_buffer(d2q37_lattice* h, int which, double* host, size_t n) {
    return dump_canonical_impl(h, which, host, n, false);
}
int d2q37_load_buffer_device(d2q37_lattice* h, int which, const double* dev, size_t n) {
    return load_canonical_impl(h, which, dev, n, true);
}
int d2q37_dump_buffer_device(d2q37_lattice* h, int which, double* dev, size_t n) {
    return dump_canonical_impl(h, which, dev, n, true);
}

static size_t padded_count(const d2q37_lattice* h) {
    return size_t(kNpop) * h->g.px * h->g.sy * h->g.vl;
}

// Element index of the reference Descriptor for this layout (layout.hpp:67-79).
static size_t ref_index(const d2q37_lattice* h, int p, int X, int j, int k) {
    const DevGeo& g = h->g;
    const size_t cluster = site_major(h->layout) ? (size_t(X) * g.sy + j) * kNpop + p
                                                 : (size_t(p) * g.px + X) * g.sy + j;
    return cluster * size_t(g.vl) + size_t(k);
}

int d2q37_read_padded(d2q37_lattice* h, int which, double* host, size_t n) {
    RET(check_handle(h));
    RET(padded_verbs_ok(h, "read_padded"));
    if (which != 0 && which != 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "buffer index must be 0 or 1");
    if (n != padded_count(h)) return fail(D2Q37_ERR_INVALID_ARGUMENT, "padded size mismatch (want %zu)", padded_count(h));
    DeviceGuard dg(h->device);
    std::vector<double> dev(h->buf_elems);
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(dev.data(), h->buf[which == 0 ? h->cur : 1 - h->cur], h->buf_elems * sizeof(double),
                  cudaMemcpyDeviceToHost));
    const DevGeo& g = h->g;
    for (int p = 0; p < kNpop; ++p)
        for (int X = 0; X < g.px; ++X)
            for (int j = 0; j < g.sy; ++j)
                for (int k = 0; k < g.vl; ++k) host[ref_index(h, p, X, j, k)] = dev[size_t(elem_of(g, p, X, j, k))];
    return D2Q37_OK;
}

int d2q37_write_padded(d2q37_lattice* h, int which, const double* host, size_t n) {
    if (h) h->p2p_dirty = true, h->h6_valid = false, h->bc_filled = -1;
    RET(check_handle(h));
    RET(padded_verbs_ok(h, "write_padded"));
    if (which != 0 && which != 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "buffer index must be 0 or 1");
    if (n != padded_count(h)) return fail(D2Q37_ERR_INVALID_ARGUMENT, "padded size mismatch (want %zu)", padded_count(h));
    DeviceGuard dg(h->device);
    double* d = h->buf[which == 0 ? h->cur : 1 - h->cur];
    std::vector<double> dev(h->buf_elems);
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(dev.data(), d, h->buf_elems * sizeof(double), cudaMemcpyDeviceToHost));
    const DevGeo& g = h->g;
    for (int p = 0; p < kNpop; ++p)
        for (int X = 0; X < g.px; ++X)
            for (int j = 0; j < g.sy; ++j)
                for (int k = 0; k < g.vl; ++k) dev[size_t(elem_of(g, p, X, j, k))] = host[ref_index(h, p, X, j, k)];
    CK(cudaMemcpy(d, dev.data(), h->buf_elems * sizeof(double), cudaMemcpyHostToDevice));
    return D2Q37_OK;
}

// halo_exchange (kernels.cpp:197-234) on y-major slab storage, which has no
// reference padded order: the neighbours' face columns come into the ghost
// columns (NCCL or, in a group, device copies) and the boundary mode is
// recorded; the propagate verb then resolves the faces in the kernel (x
// periodic, y wall / periodic / the exchanged ghost columns) -- the same
// pulls the reference makes from its filled ghost cells.
int ymajor_bc(d2q37_lattice* h, int bc) {
    if (!local_only(h) && remote_faces(h, bc)) {
        if (h->transport == kTransportGroup) {
            RET(ymajor_group_exchange(h->group, bc));
            for (d2q37_lattice* s : h->group) s->bc_filled = bc;
            return D2Q37_OK;
        }
        if (h->transport != kTransportNccl)
            return fail(D2Q37_ERR_UNSUPPORTED, "bc: not available on P2P y-major slabs (use step)");
        CK(cudaEventRecord(h->ev_start, h->stream));
        CK(cudaStreamWaitEvent(h->comm_stream, h->ev_start, 0));
        RET(ymajor_exchange_nccl(h, bc));
        CK(cudaStreamWaitEvent(h->stream, h->ev_recv, 0));
    }
    h->bc_filled = bc;
    return D2Q37_OK;
}

int d2q37_bc(d2q37_lattice* h, int bc) {
    RET(check_handle(h));
    h->h6_valid = false;  // the reference's 3 ghost rows share storage with the 6-row FUSED2 ghosts
    RET(validate_bc(h, bc));
    if (h->g.tr) {
        DeviceGuard dg(h->device);
        return ymajor_bc(h, bc);
    }
    RET(padded_verbs_ok(h, "bc"));
    RET(validate_bc(h, bc));
    DeviceGuard dg(h->device);
    if (!local_only(h) && remote_faces(h, bc)) {
        if (h->transport == kTransportGroup) {
            // every slab of the group packs, then halos move, then edges run
            for (d2q37_lattice* s : h->group) RET(exchange_begin(s, bc));
            RET(group_exchange(h->group, bc));
            for (d2q37_lattice* s : h->group) RET(edge(s, bc, kEdgeAll, false));
            return D2Q37_OK;
        }
        RET(exchange_begin(h, bc));
        RET(exchange_wait(h));
    }
    return edge(h, bc, kEdgeAll, false);
}

int d2q37_propagate(d2q37_lattice* h) { return d2q37_propagate_corrupt(h, -1); }

int d2q37_propagate_corrupt(d2q37_lattice* h, int corrupt_population) {
    RET(check_handle(h));
    h->h6_valid = false;
    if (!h->g.tr) RET(padded_verbs_ok(h, "propagate"));
    if (h->g.tr && h->bc_filled < 0)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "propagate on a y-major slab: call bc (halo_exchange) first");
    DeviceGuard dg(h->device);
    if (corrupt_population >= kNpop) return fail(D2Q37_ERR_INVALID_ARGUMENT, "corrupt_population out of range");
    Offsets off = h->off_pull;
    if (corrupt_population >= 0) off.o[corrupt_population] += 1;  // bites on the flat-offset (interior) sites
    finish_offsets(off, h->g.pstride, corrupt_population < 0);
    // y-major slabs: the faces of the last bc, resolved in the pull (see ymajor_bc)
    return propagate_launch(h, off, h->g.tr ? step_faces(h, h->bc_filled) : ghost_faces(h));
}

int d2q37_collide(d2q37_lattice* h, double omega) {
    RET(check_handle(h));
    h->h6_valid = false;
    h->bc_filled = -1;
    if (h->g.band) return fail(D2Q37_ERR_UNSUPPORTED, "collide: not available on the banded store (use FUSED2 steps)");
    DeviceGuard dg(h->device);
    return collide_launch(h, 1 - h->cur, h->cur, omega, false, all_sites(h->g), 1, ghost_faces(h));
}

int d2q37_step(d2q37_lattice* h, double omega, int nsteps, int variant, int bc) {
    RET(check_handle(h));
    h->bc_filled = -1;
    RET(validate_bc(h, bc));
    if (nsteps < 0) return fail(D2Q37_ERR_INVALID_ARGUMENT, "nsteps must be >= 0");
    if (variant != D2Q37_FUSED && variant != D2Q37_UNFUSED && variant != D2Q37_FUSED2)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "unknown variant");
    if (h->g.band && (variant == D2Q37_UNFUSED || h->math != D2Q37_MATH_FAST))
        return fail(D2Q37_ERR_UNSUPPORTED, "banded store: FUSED2 / FUSED steps in FAST math only");
    DeviceGuard dg(h->device);
    if (h->transport == kTransportGroup) {
        d2q37_lattice** slabs = h->group.data();
        return d2q37_group_step(slabs, int(h->group.size()), omega, nsteps, variant, bc);
    }
    const bool slab = !local_only(h) && remote_faces(h, bc);
    int s = 0;
    if (variant == D2Q37_FUSED2) {
        const Faces fc = step_faces(h, bc);
        if (h->math == D2Q37_MATH_FAST && step2_supported(h->g, fc)) {
            if (!slab) {
                if (!h->prof_on && nsteps - s >= 4 * kGraphSteps) {
                    // launch-bound small lattices: one direct sweep (kernel attributes, SM
                    // count), then graphs of kGraphSteps sweeps
                    RET(step2_local(h, omega, fc));
                    s += 2;
                    RET(ensure_step_graph(h, omega, D2Q37_FUSED2, bc));
                    if (h->graph.exec) {
                        for (; s + 2 * kGraphSteps <= nsteps; s += 2 * kGraphSteps) {
                            CK(cudaGraphLaunch(h->graph.exec, h->stream));
                            h->time_step += 2 * kGraphSteps;
                        }
                    }
                }
                for (; s + 2 <= nsteps; s += 2) RET(step2_local(h, omega, fc));
            } else if (h->transport == kTransportNccl && h->comm_stream && step2_overlap() && !h->g.band) {
                // (the overlapped sweep k_step2_slab is the SoA store's; the banded store exchanges first)
                for (; s + 2 <= nsteps; s += 2) {
                    if (!h->h6_valid) RET(step2_slab_exchange_nccl(h, bc));
                    RET(step2_sweep_overlapped(h, omega, bc, fc));
                }
            } else if (h->transport == kTransportNccl) {
                for (; s + 2 <= nsteps; s += 2) {
                    RET(step2_slab_exchange_nccl(h, bc));
                    RET(step2_local(h, omega, fc));
                }
            }
        }
        variant = D2Q37_FUSED;  // the odd last step, and every layout / case k_step2 does not cover
    }
    if (s < nsteps) h->h6_valid = false;  // the remaining steps change prv without refreshing its 6-row ghosts
    if (!slab && !h->prof_on && nsteps - s >= kGraphSteps) {
        // Launch-bound small lattices: replay kGraphSteps steps as one CUDA graph.
        RET(ensure_step_graph(h, omega, variant, bc));
        if (h->graph.exec) {
            for (; s + kGraphSteps <= nsteps; s += kGraphSteps) {
                CK(cudaGraphLaunch(h->graph.exec, h->stream));
                h->time_step += kGraphSteps;  // kGraphSteps is even: cur is unchanged
            }
        }
    }
    for (; s < nsteps; ++s) {
        if (slab && h->g.band) {  // 6-row halos, then a one-step sweep
            RET(step2_slab_exchange_nccl(h, bc));
            RET(step_local(h, omega, variant, bc));
        } else if (slab && h->transport == kTransportP2P) {
            RET(p2p_step(h, omega, variant, bc));
        } else if (slab && h->g.tr) {
            RET(variant == D2Q37_FUSED ? ymajor_step_nccl(h, omega, bc) : ymajor_step_nccl_unfused(h, omega, bc));
        } else if (slab && h->halo_stream && variant == D2Q37_FUSED && can_split(h)) {
            RET(slab_step_overlapped(h, omega, bc));
        } else if (slab) {
            RET(exchange_begin(h, bc));
            RET(slab_phase1(h, omega, variant, bc));
            RET(slab_phase2(h, omega, variant, bc));
        } else {
            RET(step_local(h, omega, variant, bc));
        }
    }
    return D2Q37_OK;
}

int d2q37_swap_buffers(d2q37_lattice* h) {
    if (h) h->p2p_dirty = true, h->h6_valid = false, h->bc_filled = -1;
    RET(check_handle(h));
    h->cur = 1 - h->cur;
    return D2Q37_OK;
}

int d2q37_sync(d2q37_lattice* h) {
    RET(check_handle(h));
    DeviceGuard dg(h->device);
    CK(cudaMemcpyAsync(h->h_flag, h->d_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (h->comm_stream) CK(cudaStreamSynchronize(h->comm_stream));
    if (h->halo_stream) CK(cudaStreamSynchronize(h->halo_stream));
    if (*h->h_flag) {
        const int f = *h->h_flag;
        *h->h_flag = 0;
        CK(cudaMemsetAsync(h->d_flag, 0, sizeof(int), h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (f & 2) return fail(D2Q37_ERR_NCCL, "p2p halo: a neighbour did not reach the step in time (D2Q37_P2P_TIMEOUT_S)");
        return fail(D2Q37_ERR_NON_PHYSICAL, "non-positive density");
    }
    return D2Q37_OK;
}

int d2q37_moments(d2q37_lattice* h, double out[4]) {
    RET(check_handle(h));
    DeviceGuard dg(h->device);
    CK(launch_moments(h->buf[h->cur], h->g, h->d_part, h->stream));
    std::vector<double> part(size_t(h->g.lx) * 4);
    CK(cudaMemcpyAsync(part.data(), h->d_part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (int i = 0; i < 4; ++i) out[i] = 0.0;
    for (int x = 0; x < h->g.lx; ++x)
        for (int i = 0; i < 4; ++i) out[i] += part[size_t(x) * 4 + i];
    return D2Q37_OK;
}

int d2q37_scalar_steps(const d2q37_model* m, int lx, int ly, const double* host_in, double* host_out, size_t n,
                       double omega, int nsteps, int math, int device) {
    if (lx < 1 || ly < 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "lattice extents must be positive");
    if (!host_in || !host_out || n != size_t(kNpop) * lx * ly)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "canonical array size mismatch");
    if (nsteps < 0) return fail(D2Q37_ERR_INVALID_ARGUMENT, "nsteps must be >= 0");
    if (math != D2Q37_MATH_FAST && math != D2Q37_MATH_STRICT)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "unknown math mode");
    d2q37_model local;
    if (!m) {
        build_model(&local);
        m = &local;
    }
    ModelParams mp{};
    RET(model_params(m, &mp));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(D2Q37_ERR_INVALID_ARGUMENT, "no CUDA device %d", device);
    DeviceGuard dg(device);
    const size_t bytes = n * sizeof(double);
    double *a = nullptr, *b = nullptr;
    int* flag = nullptr;
    int rc = D2Q37_OK;
    cudaStream_t st = nullptr;
    auto run = [&]() -> int {
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        CK(cudaMalloc(&a, bytes));
        CK(cudaMalloc(&b, bytes));
        CK(cudaMalloc(&flag, sizeof(int)));
        CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
        CK(cudaMemcpyAsync(a, host_in, bytes, cudaMemcpyHostToDevice, st));
        for (int i = 0; i < nsteps; ++i)  // a -> b (propagate) -> a (collide)
            CK(launch_scalar_step(a, b, a, lx, ly, mp, omega, math == D2Q37_MATH_STRICT, flag, st));
        int hflag = 0;
        CK(cudaMemcpyAsync(host_out, a, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hflag) return fail(D2Q37_ERR_NON_PHYSICAL, "non-positive density");
        return D2Q37_OK;
    };
    rc = run();
    if (a) cudaFree(a);
    if (b) cudaFree(b);
    if (flag) cudaFree(flag);
    if (st) cudaStreamDestroy(st);
    return rc;
}

int d2q37_convert(d2q37_lattice* src, d2q37_lattice* dst) {
    RET(check_handle(src));
    RET(check_handle(dst));
    if (src == dst) return fail(D2Q37_ERR_INVALID_ARGUMENT, "convert: source and destination alias");
    int gs[6], gd[6];
    RET(d2q37_geometry(src, gs));
    RET(d2q37_geometry(dst, gd));
    if (gs[0] != gd[0] || gs[1] != gd[1]) return fail(D2Q37_ERR_INVALID_ARGUMENT, "convert: geometry mismatch");
    if (src->device != dst->device) return fail(D2Q37_ERR_INVALID_ARGUMENT, "convert: lattices on different devices");
    DeviceGuard dg(src->device);
    const size_t plane = size_t(src->g.lx) * src->g.ly;
    double* tmp = nullptr;
    CK(cudaStreamSynchronize(dst->stream));
    CK(cudaMallocAsync(&tmp, plane * sizeof(double), src->stream));
    for (int p = 0; p < kNpop; ++p) {
        CK(launch_gather(src->buf[src->cur], src->g, tmp, p, src->stream));
        CK(launch_scatter(dst->buf[dst->cur], dst->g, tmp, p, src->stream));
    }
    CK(cudaFreeAsync(tmp, src->stream));
    CK(cudaStreamSynchronize(src->stream));
    dst->time_step = src->time_step;
    dst->p2p_dirty = true;
    dst->h6_valid = false;
    dst->bc_filled = -1;
    return D2Q37_OK;
}

namespace {
const d2q37_model& model_or_default(const d2q37_model* m) {
    static const d2q37_model def = [] {
        d2q37_model d;
        build_model(&d);
        return d;
    }();
    return m ? *m : def;
}
}  // namespace

int d2q37_macros_of(const d2q37_model* m, const double f[37], double out[4]) {
    if (!f || !out) return fail(D2Q37_ERR_INVALID_ARGUMENT, "macros_of: null array");
    if (!host_macros(model_or_default(m), f, out)) return fail(D2Q37_ERR_NON_PHYSICAL, "non-positive density");
    return D2Q37_OK;
}

int d2q37_equilibrium(const d2q37_model* m, const double macros[4], double f_eq[37]) {
    if (!macros || !f_eq) return fail(D2Q37_ERR_INVALID_ARGUMENT, "equilibrium: null array");
    host_equilibrium(model_or_default(m), macros[0], macros[1], macros[2], macros[3], f_eq);
    return D2Q37_OK;
}

int d2q37_collide_site(const d2q37_model* m, const double f[37], double omega, double out[37]) {
    if (!f || !out) return fail(D2Q37_ERR_INVALID_ARGUMENT, "collide_site: null array");
    if (!host_collide_site(model_or_default(m), f, omega, out))
        return fail(D2Q37_ERR_NON_PHYSICAL, "non-positive density");
    return D2Q37_OK;
}

int d2q37_make_lattice(int kind, int lx, int ly, uint64_t seed, const double* params, const d2q37_model* m,
                       double* out, size_t n, int nthreads) {
    if (lx < 1 || ly < 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "lattice extents must be positive");
    if (!out || n != size_t(kNpop) * lx * ly) return fail(D2Q37_ERR_INVALID_ARGUMENT, "output size mismatch");
    if ((kind == D2Q37_INIT_EQUILIBRIUM || kind == D2Q37_INIT_SHEAR) && !params)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "initialiser needs params");
    d2q37_model local;
    if (!m) {
        build_model(&local);
        m = &local;
    }
    try {
        make_lattice(kind, lx, ly, seed, params, *m, out, nthreads);
    } catch (const std::exception& e) {
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "%s", e.what());
    }
    return D2Q37_OK;
}

int d2q37_fill_philox(d2q37_lattice* h, int which, uint64_t seed) {
    if (h) h->p2p_dirty = true, h->h6_valid = false, h->bc_filled = -1;
    RET(check_handle(h));
    if (which != 0 && which != 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "buffer index must be 0 or 1");
    if (h->g.band) return fail(D2Q37_ERR_UNSUPPORTED, "fill_philox: not available on the banded store");
    DeviceGuard dg(h->device);
    CK(launch_philox(h->buf[which == 0 ? h->cur : 1 - h->cur], h->g, seed, h->y0, h->ly_global, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return D2Q37_OK;
}

int d2q37_init_rt_device(d2q37_lattice* h, uint64_t seed) {
    if (h) h->p2p_dirty = true, h->h6_valid = false, h->bc_filled = -1;
    RET(check_handle(h));
    DeviceGuard dg(h->device);
    CK(launch_init_rt(h->buf[h->cur], h->g, h->mp, seed, h->y0, h->ly_global, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return D2Q37_OK;
}

// ---- LBDUMP01 snapshots streamed from / to device memory (dump.cpp:44-70) ----

namespace {

constexpr char kDumpMagic[8] = {'L', 'B', 'D', 'U', 'M', 'P', '0', '1'};
constexpr size_t kDumpChunk = size_t(1) << 23;  // doubles per pinned staging chunk (64 MB)

struct FileCloser {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};

// Two pinned chunks so file I/O of one overlaps the copy of the other.
struct PinnedPair {
    double* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~PinnedPair() {
        for (int i = 0; i < 2; ++i) {
            if (buf[i]) cudaFreeHost(buf[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
    }
    int init(size_t n) {
        for (int i = 0; i < 2; ++i) {
            CK(cudaMallocHost(&buf[i], n * sizeof(double)));
            CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        return D2Q37_OK;
    }
};

}  // namespace

int d2q37_save_dump(d2q37_lattice* h, const char* path) {
    RET(check_handle(h));
    if (!path) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null path");
    DeviceGuard dg(h->device);
    std::unique_ptr<std::FILE, FileCloser> f(std::fopen(path, "wb"));
    if (!f) return fail(D2Q37_ERR_INVALID_ARGUMENT, "cannot open dump file for writing: %s", path);
    const DevGeo& g = h->g;
    const uint64_t dims[3] = {uint64_t(g.lx), uint64_t(g.ly), uint64_t(kNpop)};
    if (std::fwrite(kDumpMagic, 1, 8, f.get()) != 8 || std::fwrite(dims, 8, 3, f.get()) != 3)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "short write to dump file: %s", path);
    const size_t plane = size_t(g.lx) * g.ly;
    if (!h->stage) CK(cudaMalloc(&h->stage, plane * sizeof(double)));
    PinnedPair pin;
    const size_t chunk = std::min(plane, kDumpChunk);
    RET(pin.init(chunk));
    CK(cudaStreamSynchronize(h->stream));
    int slot = 0;
    bool pending[2] = {false, false};
    size_t pending_n[2] = {0, 0};
    auto drain = [&](int s) -> int {
        if (!pending[s]) return D2Q37_OK;
        CK(cudaEventSynchronize(pin.ev[s]));
        if (std::fwrite(pin.buf[s], sizeof(double), pending_n[s], f.get()) != pending_n[s])
            return fail(D2Q37_ERR_INVALID_ARGUMENT, "short write to dump file: %s", path);
        pending[s] = false;
        return D2Q37_OK;
    };
    for (int p = 0; p < kNpop; ++p) {
        CK(launch_gather(h->buf[h->cur], g, h->stage, p, h->stream));
        for (size_t off = 0; off < plane; off += chunk) {
            const size_t n = std::min(chunk, plane - off);
            RET(drain(slot));  // the chunk we are about to overwrite is on disk
            CK(cudaMemcpyAsync(pin.buf[slot], h->stage + off, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
            CK(cudaEventRecord(pin.ev[slot], h->stream));
            pending[slot] = true;
            pending_n[slot] = n;
            slot ^= 1;
        }
    }
    RET(drain(slot));
    RET(drain(slot ^ 1));
    return D2Q37_OK;
}

int d2q37_load_dump(d2q37_lattice* h, const char* path) {
    if (h) h->p2p_dirty = true, h->h6_valid = false, h->bc_filled = -1;
    RET(check_handle(h));
    if (!path) return fail(D2Q37_ERR_INVALID_ARGUMENT, "null path");
    DeviceGuard dg(h->device);
    std::unique_ptr<std::FILE, FileCloser> f(std::fopen(path, "rb"));
    if (!f) return fail(D2Q37_ERR_INVALID_ARGUMENT, "cannot open dump file: %s", path);
    char magic[8];
    uint64_t dims[3];
    if (std::fread(magic, 1, 8, f.get()) != 8 || std::fread(dims, 8, 3, f.get()) != 3 ||
        std::memcmp(magic, kDumpMagic, 8) != 0)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "not a lattice dump: %s", path);
    const DevGeo& g = h->g;
    if (dims[0] != uint64_t(g.lx) || dims[1] != uint64_t(g.ly) || dims[2] != uint64_t(kNpop))
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "from_canonical: dimension mismatch (dump %llu x %llu x %llu)",
                    (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2]);
    const size_t plane = size_t(g.lx) * g.ly;
    if (!h->stage) CK(cudaMalloc(&h->stage, plane * sizeof(double)));
    PinnedPair pin;
    const size_t chunk = std::min(plane, kDumpChunk);
    RET(pin.init(chunk));
    CK(cudaStreamSynchronize(h->stream));
    double* dst = h->buf[h->cur];
    int slot = 0;
    for (int p = 0; p < kNpop; ++p) {
        for (size_t off = 0; off < plane; off += chunk) {
            const size_t n = std::min(chunk, plane - off);
            CK(cudaEventSynchronize(pin.ev[slot]));  // previous copy out of this chunk finished
            if (std::fread(pin.buf[slot], sizeof(double), n, f.get()) != n)
                return fail(D2Q37_ERR_INVALID_ARGUMENT, "truncated dump file: %s", path);
            CK(cudaMemcpyAsync(h->stage + off, pin.buf[slot], n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
            CK(cudaEventRecord(pin.ev[slot], h->stream));
            slot ^= 1;
        }
        CK(launch_scatter(dst, g, h->stage, p, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    return D2Q37_OK;
}

// ---- multi-GPU ------------------------------------------------------------

int d2q37_nccl_unique_id(unsigned char id[D2Q37_NCCL_ID_BYTES]) {
    std::string why;
    const int rc = nccl_unique_id(id, &why);
    if (rc != D2Q37_OK) return fail(rc, "%s", why.c_str());
    return D2Q37_OK;
}

int d2q37_create_slab(int layout, int lx, int ly, int vl, int device, int rank, int nranks,
                      const unsigned char id[D2Q37_NCCL_ID_BYTES], d2q37_lattice** out) {
    // site-major layouts (AoS, CAoSoA) slab in y-major storage: faces = contiguous columns
    const bool ymajor = site_major(layout) && (nranks > 1 || id != nullptr);
    RET(create_impl(layout, lx, ly, vl, device, out, rank, nranks, ymajor));
    d2q37_lattice* h = *out;
    if (nranks == 1 && !id) return D2Q37_OK;
    auto bail = [&](int rc) {
        d2q37_destroy(h);
        *out = nullptr;
        return rc;
    };
    if (!id) return bail(fail(D2Q37_ERR_INVALID_ARGUMENT, "null NCCL id"));
    int rc = alloc_exchange(h);
    if (rc != D2Q37_OK) return bail(rc);
    {
        DeviceGuard dg(device);
        // Both side streams get the highest priority: NCCL's kernels and the
        // boundary work must get SMs while the interior kernel is running.
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        if (cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess)
            return bail(fail(D2Q37_ERR_CUDA, "comm stream creation failed"));
        if (cudaStreamCreateWithPriority(&h->halo_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(D2Q37_ERR_CUDA, "halo stream creation failed"));
        std::string why;
        rc = nccl_comm_init(&h->comm, nranks, id, rank, &why);
        if (rc != D2Q37_OK) return bail(fail(rc, "%s", why.c_str()));
        // no lazy kernel load while NCCL kernels wait on the other ranks
        if (preload_kernels() != cudaSuccess) return bail(fail(D2Q37_ERR_CUDA, "kernel preload failed"));
    }
    h->transport = kTransportNccl;
    return D2Q37_OK;
}

namespace {
struct P2PBlob {
    uint32_t magic;
    int32_t pid, device, rank, nranks, layout, cols, rows, vl;
    uint64_t buf0, buf1, seq;  // pointers, valid in the exporting process
    cudaIpcMemHandle_t hbuf0, hbuf1, hseq;
};
static_assert(sizeof(P2PBlob) <= D2Q37_P2P_BLOB_BYTES, "P2P blob too large");
constexpr uint32_t kP2PMagic = 0x50373344u;  // "D37P"
}  // namespace

int d2q37_create_slab_p2p(int layout, int lx, int ly, int vl, int device, int rank, int nranks,
                          d2q37_lattice** out) {
    if (layout == D2Q37_BANDED) return fail(D2Q37_ERR_UNSUPPORTED, "p2p slabs: not available on the banded store");
    // site-major layouts slab in y-major storage (faces = contiguous columns), the others x-major
    if (!site_major(layout) && nranks > 0 && ly % nranks == 0 && !clustered(layout) && ly / nranks < 2 * kHalo)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "p2p SoA slab needs at least 6 rows per slab");
    RET(create_impl(layout, lx, ly, vl, device, out, rank, nranks, site_major(layout)));
    d2q37_lattice* h = *out;
    auto bail = [&](int rc) {
        d2q37_destroy(h);
        *out = nullptr;
        return rc;
    };
    DeviceGuard dg(device);
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&h->halo_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&h->d_seq, 2 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(h->d_seq, 0, 2 * sizeof(unsigned long long)) != cudaSuccess)
        return bail(fail(D2Q37_ERR_CUDA, "p2p slab setup failed"));
    for (int i = 0; i < kEventRing; ++i)
        if (cudaEventCreate(&h->ev_int[i]) != cudaSuccess || cudaEventCreate(&h->ev_wait[i]) != cudaSuccess)
            return bail(fail(D2Q37_ERR_CUDA, "p2p slab event creation failed"));
    if (preload_kernels() != cudaSuccess) return bail(fail(D2Q37_ERR_CUDA, "kernel preload failed"));
    h->transport = kTransportP2P;
    return D2Q37_OK;
}

int d2q37_p2p_export(const d2q37_lattice* h, unsigned char blob[D2Q37_P2P_BLOB_BYTES]) {
    RET(check_handle(h));
    if (h->transport != kTransportP2P) return fail(D2Q37_ERR_INVALID_ARGUMENT, "not a p2p slab");
    DeviceGuard dg(h->device);
    P2PBlob b{};
    b.magic = kP2PMagic;
    b.pid = int32_t(getpid());
    b.device = h->device;
    b.rank = h->rank;
    b.nranks = h->nranks;
    b.layout = h->layout;
    b.cols = h->g.lx;
    b.rows = h->g.ly;
    b.vl = h->g.vl;
    b.buf0 = reinterpret_cast<uint64_t>(h->buf[0]);
    b.buf1 = reinterpret_cast<uint64_t>(h->buf[1]);
    b.seq = reinterpret_cast<uint64_t>(h->d_seq);
    CK(cudaIpcGetMemHandle(&b.hbuf0, h->buf[0]));
    CK(cudaIpcGetMemHandle(&b.hbuf1, h->buf[1]));
    CK(cudaIpcGetMemHandle(&b.hseq, h->d_seq));
    std::memset(blob, 0, D2Q37_P2P_BLOB_BYTES);
    std::memcpy(blob, &b, sizeof b);
    return D2Q37_OK;
}

namespace {
// Maps a neighbour's allocation into this process: its own pointer when it
// lives in this process, else a CUDA IPC mapping (reused if already open).
int map_peer(d2q37_lattice* h, const P2PBlob& b, uint64_t ptr, const cudaIpcMemHandle_t& ipc, void** out) {
    if (b.pid == int32_t(getpid())) {
        if (b.device != h->device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return fail(D2Q37_ERR_CUDA, "peer access to device %d: %s", b.device, cudaGetErrorString(e));
            (void)cudaGetLastError();
        }
        *out = reinterpret_cast<void*>(ptr);
        return D2Q37_OK;
    }
    CK(cudaIpcOpenMemHandle(out, ipc, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_mapped.push_back(*out);
    return D2Q37_OK;
}
}  // namespace

int d2q37_p2p_connect(d2q37_lattice* h, const unsigned char lo[D2Q37_P2P_BLOB_BYTES],
                      const unsigned char hi[D2Q37_P2P_BLOB_BYTES]) {
    RET(check_handle(h));
    if (h->transport != kTransportP2P) return fail(D2Q37_ERR_INVALID_ARGUMENT, "not a p2p slab");
    if (h->p2p_connected) return fail(D2Q37_ERR_INVALID_ARGUMENT, "p2p slab already connected");
    DeviceGuard dg(h->device);
    P2PBlob nb[2];
    const unsigned char* in[2] = {lo, hi};
    for (int side = 0; side < 2; ++side) {
        if (!in[side]) continue;
        std::memcpy(&nb[side], in[side], sizeof(P2PBlob));
        const P2PBlob& b = nb[side];
        if (b.magic != kP2PMagic) return fail(D2Q37_ERR_INVALID_ARGUMENT, "not a p2p slab blob");
        if (b.layout != h->layout || b.vl != h->g.vl || b.rows != h->g.ly || b.cols != h->g.lx ||
            b.nranks != h->nranks)
            return fail(D2Q37_ERR_INVALID_ARGUMENT, "p2p neighbour has a different slab geometry");
        const int want = side == 0 ? (h->rank - 1 + h->nranks) % h->nranks : (h->rank + 1) % h->nranks;
        if (b.rank != want) return fail(D2Q37_ERR_INVALID_ARGUMENT, "p2p blob of rank %d, expected %d", b.rank, want);
    }
    // the same neighbour on both sides (2 ranks, or a 1-rank ring) is mapped once
    for (int side = 0; side < 2; ++side) {
        if (!in[side]) continue;
        const P2PBlob& b = nb[side];
        void *p0 = nullptr, *p1 = nullptr, *ps = nullptr;
        if (side == 1 && in[0] && std::memcmp(&nb[0], &nb[1], sizeof(P2PBlob)) == 0) {
            p0 = h->peer_buf[0][0];
            p1 = h->peer_buf[0][1];
            ps = h->peer_seq_slot[0] - 1;
        } else {
            RET(map_peer(h, b, b.buf0, b.hbuf0, &p0));
            RET(map_peer(h, b, b.buf1, b.hbuf1, &p1));
            RET(map_peer(h, b, b.seq, b.hseq, &ps));
        }
        h->peer_buf[side][0] = static_cast<double*>(p0);
        h->peer_buf[side][1] = static_cast<double*>(p1);
        // I am my lo neighbour's hi neighbour (its slot 1) and my hi neighbour's lo one (slot 0)
        h->peer_seq_slot[side] = static_cast<unsigned long long*>(ps) + (side == 0 ? 1 : 0);
    }
    h->p2p_connected = true;
    h->p2p_dirty = true;
    h->h6_valid = false;
    return D2Q37_OK;
}

int d2q37_create_multi(int layout, int lx, int ly, int vl, int nslabs, const int* devices, d2q37_lattice** out) {
    if (!out || !devices || nslabs < 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "bad multi-GPU arguments");
    std::vector<d2q37_lattice*> slabs(nslabs, nullptr);
    auto bail = [&](int rc) {
        for (d2q37_lattice* sl : slabs) d2q37_destroy(sl);
        for (int r = 0; r < nslabs; ++r) out[r] = nullptr;
        return rc;
    };
    std::vector<std::vector<unsigned char>> blobs(nslabs, std::vector<unsigned char>(D2Q37_P2P_BLOB_BYTES));
    for (int r = 0; r < nslabs; ++r) {
        int rc = d2q37_create_slab_p2p(layout, lx, ly, vl, devices[r], r, nslabs, &slabs[r]);
        if (rc == D2Q37_OK) rc = d2q37_p2p_export(slabs[r], blobs[r].data());
        if (rc != D2Q37_OK) {
            const std::string why = g_last_error;
            bail(rc);
            return fail(rc, "%s", why.c_str());
        }
    }
    for (int r = 0; r < nslabs; ++r) {
        const int rc = d2q37_p2p_connect(slabs[r], blobs[(r - 1 + nslabs) % nslabs].data(),
                                         blobs[(r + 1) % nslabs].data());
        if (rc != D2Q37_OK) {
            const std::string why = g_last_error;
            bail(rc);
            return fail(rc, "%s", why.c_str());
        }
    }
    for (int r = 0; r < nslabs; ++r) out[r] = slabs[r];
    return D2Q37_OK;
}

int d2q37_multi_step(d2q37_lattice** slabs, int nslabs, double omega, int nsteps, int variant, int bc) {
    if (!slabs || nslabs < 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "bad multi-GPU slabs");
    for (int r = 0; r < nslabs; ++r) {
        RET(check_handle(slabs[r]));
        if (slabs[r]->transport != kTransportP2P || slabs[r]->nranks != nslabs)
            return fail(D2Q37_ERR_INVALID_ARGUMENT, "not the slabs of one d2q37_create_multi lattice");
    }
    // lockstep: every slab's step k is enqueued before any slab's step k + 1, so no
    // slab's counter wait depends on work the host has not issued yet
    for (int k = 0; k < nsteps; ++k)
        for (int r = 0; r < nslabs; ++r) RET(d2q37_step(slabs[r], omega, 1, variant, bc));
    for (int r = 0; r < nslabs; ++r) RET(d2q37_sync(slabs[r]));
    return D2Q37_OK;
}

int d2q37_create_group(int layout, int lx, int ly, int vl, int device, int nslabs, d2q37_lattice** out) {
    if (!out || nslabs < 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "bad group arguments");
    std::vector<d2q37_lattice*> slabs(nslabs, nullptr);
    auto bail = [&](int rc) {
        for (d2q37_lattice* s : slabs) d2q37_destroy(s);
        return rc;
    };
    for (int r = 0; r < nslabs; ++r) {
        int rc = create_impl(layout, lx, ly, vl, device, &slabs[r], r, nslabs, site_major(layout) && nslabs > 1);
        if (rc != D2Q37_OK) return bail(rc);
        if (nslabs > 1) {
            rc = alloc_exchange(slabs[r]);
            if (rc != D2Q37_OK) return bail(rc);
        }
    }
    // One stream for the whole group: slabs never wait on each other inside a kernel.
    for (int r = 1; r < nslabs; ++r) {
        cudaStreamSynchronize(slabs[r]->stream);
        slabs[r]->stream_owner = slabs[0]->stream_owner;
        slabs[r]->stream = slabs[0]->stream;
    }
    for (int r = 0; r < nslabs; ++r) {
        if (nslabs > 1) slabs[r]->transport = kTransportGroup;
        slabs[r]->group = slabs;
        out[r] = slabs[r];
    }
    return D2Q37_OK;
}

int d2q37_group_step(d2q37_lattice** slabs_in, int nslabs, double omega, int nsteps, int variant, int bc) {
    if (!slabs_in || nslabs < 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "bad group");
    std::vector<d2q37_lattice*> slabs(slabs_in, slabs_in + nslabs);
    for (d2q37_lattice* h : slabs) {
        RET(check_handle(h));
        RET(validate_bc(h, bc));
    }
    if (variant != D2Q37_FUSED && variant != D2Q37_UNFUSED && variant != D2Q37_FUSED2)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "unknown variant");
    if (slabs[0]->g.band && (variant == D2Q37_UNFUSED || slabs[0]->math != D2Q37_MATH_FAST))
        return fail(D2Q37_ERR_UNSUPPORTED, "banded store: FUSED2 / FUSED steps in FAST math only");
    DeviceGuard dg(slabs[0]->device);
    int s = 0;
    if (variant == D2Q37_FUSED2) {
        bool ok = true;
        for (d2q37_lattice* h : slabs) ok = ok && h->math == D2Q37_MATH_FAST && step2_supported(h->g, step_faces(h, bc));
        if (ok) {
            const bool remote = nslabs > 1 && remote_faces(slabs[0], bc);
            for (; s + 2 <= nsteps; s += 2) {
                if (remote) RET(step2_group_exchange(slabs, bc));
                for (d2q37_lattice* h : slabs) RET(step2_local(h, omega, step_faces(h, bc)));
            }
        }
        variant = D2Q37_FUSED;
    }
    for (; s < nsteps; ++s) {
        if (nslabs == 1 || !remote_faces(slabs[0], bc)) {
            for (d2q37_lattice* h : slabs) RET(step_local(h, omega, variant, bc));
            continue;
        }
        if (slabs[0]->g.band) {  // 6-row halos, then one-step sweeps
            RET(step2_group_exchange(slabs, bc));
            for (d2q37_lattice* h : slabs) RET(step_local(h, omega, variant, bc));
            continue;
        }
        if (slabs[0]->g.tr) {  // y-major: ghost columns <- neighbours' columns, then local steps
            RET(ymajor_group_exchange(slabs, bc));
            for (d2q37_lattice* h : slabs) RET(step_local(h, omega, variant, bc));
            continue;
        }
        for (d2q37_lattice* h : slabs) RET(exchange_begin(h, bc));
        for (d2q37_lattice* h : slabs) RET(slab_phase1(h, omega, variant, bc));
        RET(group_exchange(slabs, bc));
        for (d2q37_lattice* h : slabs) RET(slab_phase2(h, omega, variant, bc));
    }
    // like the reference's blocking step (and d2q37_multi_step): every slab's deferred
    // non-physical flag is collected, so an error in any slab surfaces here
    int rc = D2Q37_OK;
    for (d2q37_lattice* h : slabs) {
        const int r = d2q37_sync(h);
        if (rc == D2Q37_OK) rc = r;
    }
    return rc;
}

int d2q37_set_fused2_tuning(int form, int face_pct, int* prev_form, int* prev_face_pct) {
    if (prev_form) *prev_form = step2_form();
    if (prev_face_pct) *prev_face_pct = step2_face_pct();
    if (form > 4 || face_pct > 1000) return fail(D2Q37_ERR_INVALID_ARGUMENT, "fused2 tuning: form %d, face_pct %d", form, face_pct);
    if (form >= 0) set_step2_form(form);
    if (face_pct >= 0) set_step2_face_pct(face_pct);
    return D2Q37_OK;
}

// Test hook: one overlapped FUSED2 slab sweep of this lattice's current state with the given faces
// (1 wall, 3 ghost: the deep ghost rows are read as they stand; no exchange), interior form `form`
// (kStep2Pair: k_step2_pair_slab, else k_step2_slab), the new edge rows packed into the halo buffers.
int d2q37_debug_step2_slab_sweep(d2q37_lattice* h, double omega, int form, int face_lo, int face_hi) {
    RET(check_handle(h));
    auto face_ok = [](int f) { return f == kFaceWall || f == kFaceGhost; };
    if (!face_ok(face_lo) || !face_ok(face_hi) || h->layout != D2Q37_SOA || !h->g.deep)
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "debug slab sweep: SoA lattice with deep ghost rows, faces 1 / 3");
    DeviceGuard dg(h->device);
    if (!h->nsm) CK(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->device));
    RET(ensure_halo6(h));
    if (!h->d_sweep_counter) {
        CK(cudaMalloc(&h->d_sweep_counter, sizeof(unsigned)));
        CK(cudaMemset(h->d_sweep_counter, 0, sizeof(unsigned)));
    }
    Faces fc = step_faces(h, D2Q37_BC_PERIODIC);
    fc.lo = face_lo;
    fc.hi = face_hi;
    const double* src = h->buf[h->cur];
    double* dst = h->buf[1 - h->cur];
    const int grid = h->nsm - std::min(step2_halo_sms(), h->nsm / 4);
    cudaError_t err = cudaSuccess;
    int nsig = 0;
    if (form == kStep2Pair)
        nsig = launch_step2_pair_slab(src, dst, h->g, fc, h->mp, omega, h->d_flag, h->stream, grid,
                                      h->d_sweep_counter, h->h6[0], h->h6[1], &err);
    else
        nsig = launch_step2_slab(src, dst, h->g, fc, h->mp, omega, h->d_flag, h->stream, grid, h->d_sweep_counter,
                                 h->h6[0], h->h6[1], &err);
    CK(err);
    if (nsig == 0) return fail(D2Q37_ERR_UNSUPPORTED, "debug slab sweep: no overlapped form for this lattice");
    h->cur = 1 - h->cur;
    h->time_step += 2;
    h->h6_valid = false;
    return d2q37_sync(h);
}

// Test hook: the FUSED2 halo send buffers ([p][x][6] doubles; which = 0 low face, 1 high face).
int d2q37_debug_read_halo6(d2q37_lattice* h, int which, double* host, size_t n) {
    RET(check_handle(h));
    if (!h->h6[0] || (which != 0 && which != 1) || n != halo6_count(h->g))
        return fail(D2Q37_ERR_INVALID_ARGUMENT, "debug read halo6: no buffers or size mismatch");
    DeviceGuard dg(h->device);
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(host, h->h6[which], n * sizeof(double), cudaMemcpyDeviceToHost));
    return D2Q37_OK;
}

int d2q37_set_fused2_schedule(int sched, int* prev_sched) {
    if (prev_sched) *prev_sched = step2_sched();
    if (sched > 1) return fail(D2Q37_ERR_INVALID_ARGUMENT, "fused2 schedule %d", sched);
    if (sched >= 0) set_step2_sched(sched);
    return D2Q37_OK;
}

int d2q37_set_profiling(d2q37_lattice* h, int on) {
    RET(check_handle(h));
    h->prof_on = on != 0;
    if (h->prof_on) {  // a new measurement window: the exposed-halo ring restarts too (no warm-up exchanges)
        DeviceGuard dg(h->device);
        CK(cudaStreamSynchronize(h->stream));
        h->ev_count = 0;
    }
    return D2Q37_OK;
}

int d2q37_kernel_times(d2q37_lattice* h, double ms[6], long counts[6]) {
    RET(check_handle(h));
    DeviceGuard dg(h->device);
    CK(cudaStreamSynchronize(h->stream));
    for (int i = 0; i < kProfClasses; ++i) {
        ms[i] = 0.0;
        counts[i] = 0;
    }
    for (auto& e : h->prof_pending) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, e.a, e.b));
        ms[e.cls] += t;
        counts[e.cls] += 1;
        h->prof_free.push_back(e.a);
        h->prof_free.push_back(e.b);
    }
    h->prof_pending.clear();
    return D2Q37_OK;
}

int d2q37_halo_plan(int lo_d[32], int lo_p[32], int hi_d[32], int hi_p[32]) {
    int n_lo = 0, n_hi = 0;
    for (int d = 1; d <= kHalo; ++d)
        for (int p = 0; p < kNpop; ++p) {
            if (cy_of(p) <= -d) {
                lo_d[n_lo] = d;
                lo_p[n_lo++] = p;
            }
            if (cy_of(p) >= d) {
                hi_d[n_hi] = d;
                hi_p[n_hi++] = p;
            }
        }
    return n_lo == n_hi ? n_lo : -1;
}

int d2q37_slab_neighbors(int rank, int nranks, int bc, int out[2]) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(D2Q37_ERR_INVALID_ARGUMENT, "bad rank");
    d2q37_lattice tmp;
    tmp.rank = rank;
    tmp.nranks = nranks;
    out[0] = lo_peer_of(&tmp, bc);
    out[1] = hi_peer_of(&tmp, bc);
    return D2Q37_OK;
}

int d2q37_slab_info(const d2q37_lattice* h, int out[4]) {
    RET(check_handle(h));
    out[0] = h->rank;
    out[1] = h->nranks;
    out[2] = h->y0;
    out[3] = h->g.tr ? h->g.lx : h->g.ly;  // y-major: lattice y runs along the storage columns
    return D2Q37_OK;
}

int d2q37_slab_timeline(d2q37_lattice* h, double ms[4]) {
    RET(check_handle(h));
    if (!h->tl_valid) return fail(D2Q37_ERR_INVALID_ARGUMENT, "slab timeline: no overlapped sweep with profiling on");
    DeviceGuard dg(h->device);
    CK(cudaStreamSynchronize(h->stream));
    for (int i = 0; i < 4; ++i) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, h->tl[0], h->tl[i + 1]));
        ms[i] = t;
    }
    return D2Q37_OK;
}

double d2q37_exposed_halo_ms(const d2q37_lattice* h) {
    if (!h || (h->transport != kTransportNccl && h->transport != kTransportP2P) || h->ev_count == 0) return 0.0;
    DeviceGuard dg(h->device);
    cudaStreamSynchronize(h->stream);
    const int n = std::min(h->ev_count, kEventRing);
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, h->ev_int[i], h->ev_wait[i]) == cudaSuccess) sum += std::max(0.f, ms);
    }
    return sum / n;
}

}  // extern "C"
