// d2q37_kernels.cu -- sm_100a kernels of the D2Q37 hot path.
//
//   k_propagate        propagate (kernels.cpp:50-85): per site, 37 pull loads
//                      from up to 3 sites away, 37 streaming stores.
//   k_collide<S,SHIFT> collide (kernels.cpp:120-156, model.cpp:242-298) and,
//                      with SHIFT, the fused propagate+collide step kernel.
//   k_edge             bc: every ghost slot of the padded store in one pass
//                      (kernels.cpp:197-234 periodic, or specular walls, or
//                      slab halos received from the neighbour ranks).
//   k_pack             slab boundary rows -> contiguous send buffers.
//   k_scatter/k_gather canonical plane <-> padded layout (dump.cpp:26-42).
//   k_philox           BASELINE config-1 input generation on the device.
//   k_moments          global mass / momentum / energy sums per column.
//
// All of them are HBM-streaming kernels (no tensor-core-shaped work: collide
// is 2.57 FLOP/B, below the FP64 ridge).
#include <cuda_runtime.h>

#include <algorithm>

#include "d2q37_device.cuh"
#include "d2q37_kernels.cuh"

namespace d2q37 {

// ---------------------------------------------------------------------------
// Streaming loads / stores.  Inputs are read once per launch (ld.global.nc);
// outputs are not re-read before the lattice (GBs) has cycled through the
// 126 MB L2, so they are written evict-first (st.global.cs).

__device__ __forceinline__ double ld_stream(const double* p) { return __ldg(p); }
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }

// ---------------------------------------------------------------------------

__device__ __forceinline__ int wrapi(int v, int n) {
    const int r = v % n;
    return r < 0 ? r + n : r;
}

// Source element of population p for the site (column x, lane row `row`, lane
// k) of a pull step, for sites within 3 of a column end or a lane-strip end
// (everything else uses the flat offsets).  The boundary is resolved here
// instead of through ghost copies:
//   * x is periodic: the source column wraps (no ghost columns are read);
//   * a lane reads rows beyond its strip ends from the neighbouring lane
//     (CSoA/CAoSoA, vl > 1), so inner lane halos are never read;
//   * the outer y faces (lane 0 low, lane vl-1 high) are periodic (wrap to the
//     opposite face), wall (specular image f(mirror y, ybar p)) or
//     ghost (read the ghost rows: after a bc verb, or halos received by a slab).
//   * in y-major storage (TR) the roles swap: rows are periodic lattice x and the
//     storage columns carry the y faces (periodic wrap, wall mirror, or ghost
//     columns received from a slab neighbour).
// Periodic wrap of an index at most one period outside [0, n) (the modulo
// only runs for degenerate extents n < 3).
__device__ __forceinline__ int wrap_near(int v, int n) {
    if (v < 0) v += n;
    else if (v >= n) v -= n;
    return (v < 0 || v >= n) ? wrapi(v, n) : v;
}

template <bool TR>
__device__ __forceinline__ long long edge_source(const DevGeo& g, const Faces& fc, int p, int x, int row, int k) {
    int xs = x - scx<TR>(p), pp = p;
    if (!TR) {  // normal storage: the columns are lattice x, always periodic
        xs = wrap_near(xs, g.lx);
    } else if (xs < 0) {
        if (fc.col_lo == kFacePeriodic)
            xs = wrap_near(xs, g.lx);
        else if (fc.col_lo == kFaceWall) {
            xs = -1 - xs;
            pp = fc.ybar[p];
        }  // kFaceGhost: ghost column X = 3 + xs
    } else if (xs >= g.lx) {
        if (fc.col_hi == kFacePeriodic)
            xs = wrap_near(xs, g.lx);
        else if (fc.col_hi == kFaceWall) {
            xs = 2 * g.lx - 1 - xs;
            pp = fc.ybar[p];
        }
    }
    // y-major storage: the rows are lattice x, periodic (lane 0 low <-> lane vl-1 high)
    const int face_lo = TR ? int(kFacePeriodic) : fc.lo, face_hi = TR ? int(kFacePeriodic) : fc.hi;
    int r = row - scy<TR>(p), kk = k;
    if (r < 0) {
        if (k > 0) {
            r += g.strip;
            kk = k - 1;
        } else if (face_lo == kFacePeriodic) {
            if (g.vl == 1) {
                r = wrap_near(r, g.strip);
            } else {
                r += g.strip;
                kk = g.vl - 1;
            }
        } else if (face_lo == kFaceWall) {
            r = -1 - r;
            pp = fc.ybar[p];
        }  // kFaceGhost: ghost row j = 3 + r of lane 0
    } else if (r >= g.strip) {
        if (k < g.vl - 1) {
            r -= g.strip;
            kk = k + 1;
        } else if (face_hi == kFacePeriodic) {
            if (g.vl == 1) {
                r = wrap_near(r, g.strip);
            } else {
                r -= g.strip;
                kk = 0;
            }
        } else if (face_hi == kFaceWall) {
            r = 2 * g.strip - 1 - r;
            pp = fc.ybar[p];
        }
    }
    return elem_of(g, pp, xs + kHalo, r + kHalo, kk);
}

// Column x and site q of this thread in the launch's segments; false if none.
__device__ __forceinline__ bool segment_site(const DevGeo& g, const Segments& seg, int& x, int& q) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (seg.dense) {
        const int per_col = seg.nq * seg.nseg;
        if (t >= per_col * g.lx) return false;
        x = t / per_col;
        const int i = t - x * per_col;
        q = seg.q0[i / seg.nq] + (i % seg.nq) * seg.stride;
    } else if (seg.nx > 0) {  // segment z: columns x0[z] .. +nx, sites q0[z] .. +nq
        if (t >= seg.nq) return false;
        x = seg.x0[blockIdx.z] + blockIdx.y;
        q = seg.q0[blockIdx.z] + t * seg.stride;
    } else {
        if (t >= seg.nq) return false;
        x = blockIdx.y;
        q = seg.q0[blockIdx.z] + t * seg.stride;
    }
    const int row = q >> g.lvl, k = q & (g.vl - 1);
    if (seg.skip_lo && k == 0 && row < kHalo) return false;
    if (seg.skip_hi && k == g.vl - 1 && row >= g.strip - kHalo) return false;
    return true;
}

// True if the site is within 3 of a column end or a lane-strip end, i.e. its
// pull needs the in-kernel boundary (edge_source).  Per thread: a per-CTA test
// sends whole CTAs of flat sites down the slower edge path (measured -2 %).
__device__ __forceinline__ bool edge_site(const DevGeo& g, const Segments& seg, int x, int q) {
    if (seg.dense) return true;
    const int row = q >> g.lvl;
    return x < kHalo || x >= g.lx - kHalo || row < kHalo || row >= g.strip - kHalo;
}

enum { kPullNone = 0, kPullFlat = 1, kPullEdge = 2 };

// Hides how a pointer was formed, so nvcc adds each offset to it (one IMAD.WIDE)
// instead of re-associating base + (e + o) * 8 per population.
template <typename T>
__device__ __forceinline__ T* opaque(T* p) {
    asm("" : "+l"(p));
    return p;
}

// Address modes of the flat (edge-free) site paths:
//   kAddr64: 64-bit offsets (any geometry);
//   kAddr32: 32-bit offsets, one IMAD.WIDE per address off the site pointer;
//   VL > 0:  site-major store (AoS / CAoSoA) with vl = VL known at compile time:
//            7 column base pointers, every load / store an immediate offset.
enum { kAddr64 = -1, kAddr32 = 0 };

// Gathers the 37 populations of site e: from itself (collide), from the flat
// pull offsets, or through edge_source (in-kernel boundary).
template <int PULL, bool TR, int AM>
__device__ __forceinline__ void gather_site(double (&f)[kNpop], const double* __restrict__ src, long long e,
                                            const DevGeo& g, const Offsets& off, const Faces& fc, int x, int q) {
    const double* __restrict__ s = AM == kAddr64 ? src + e : opaque(src + e);
    if (PULL == kPullNone) {
#pragma unroll
        for (int p = 0; p < kNpop; ++p)
            f[p] = ld_stream(AM > 0 ? s + p * AM : AM == kAddr32 ? s + p * off.ps32 : s + p * g.pstride);
    } else if (PULL == kPullFlat) {
        if (AM > 0) {
            // pull offset p*vl - sx*cstride - sy*37*vl (fill_offsets): a base per source column
            const double* b[2 * kHalo + 1];
#pragma unroll
            for (int c = -kHalo; c <= kHalo; ++c) b[c + kHalo] = opaque(s - (long long)c * g.cstride);
#pragma unroll
            for (int p = 0; p < kNpop; ++p)
                f[p] = ld_stream(b[scx<TR>(p) + kHalo] + (p * AM - scy<TR>(p) * kNpop * AM));
        } else {
#pragma unroll
            for (int p = 0; p < kNpop; ++p) f[p] = ld_stream(AM == kAddr32 ? s + off.o32[p] : s + off.o[p]);
        }
    } else {  // unrolled: f[] must stay in registers (a rolled address loop costs 16 %)
        const int row = q >> g.lvl, k = q & (g.vl - 1);
#pragma unroll
        for (int p = 0; p < kNpop; ++p) f[p] = ld_stream(src + edge_source<TR>(g, fc, p, x, row, k));
    }
}

template <int AM>
__device__ __forceinline__ void store_site(double* __restrict__ dst, long long e, const DevGeo& g, const Offsets& off,
                                           const double (&f)[kNpop]) {
    double* __restrict__ d = AM == kAddr64 ? dst + e : opaque(dst + e);
#pragma unroll
    for (int p = 0; p < kNpop; ++p)
        st_stream(AM > 0 ? d + p * AM : AM == kAddr32 ? d + p * off.ps32 : d + p * g.pstride, f[p]);
}

// Gathers the pulled populations of a site: flat offsets (address mode AM) for
// sites away from every column / strip end, edge_source (64-bit) otherwise.
// One gather per thread and a single collide after it: a duplicated collide
// per path measured -13 % on config 0, where edge and flat warps share every
// SM (likely the larger hot code footprint; full size was unaffected).
template <bool TR, int AM>
__device__ __forceinline__ void pull_site(double (&f)[kNpop], const double* __restrict__ src, long long e,
                                          const DevGeo& g, const Offsets& off, const Faces& fc, const Segments& seg,
                                          int x, int q) {
    if (edge_site(g, seg, x, q))
        gather_site<kPullEdge, TR, kAddr64>(f, src, e, g, off, fc, x, q);
    else
        gather_site<kPullFlat, TR, AM>(f, src, e, g, off, fc, x, q);
}

template <bool TR, int AM>
__global__ void __launch_bounds__(kStreamThreads) k_propagate(const double* __restrict__ src,
                                                              double* __restrict__ dst, DevGeo g, Offsets off,
                                                              Faces fc, Segments seg) {
    int x, q;
    if (!segment_site(g, seg, x, q)) return;
    const long long e = site_of(g, x + kHalo, q);
    double f[kNpop];
    pull_site<TR, AM>(f, src, e, g, off, fc, seg, x, q);
    store_site<AM>(dst, e, g, off, f);
}

template <bool STRICT, bool SHIFT, bool TR, int AM>
__global__ void __launch_bounds__(kStreamThreads, kCollideMinBlocks)
    k_collide(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, Offsets off, Faces fc,
              ModelParams mp, double omega, Segments seg, int* __restrict__ flag) {
    int x, q;
    if (!segment_site(g, seg, x, q)) return;
    const long long e = site_of(g, x + kHalo, q);
    double f[kNpop];
    if (SHIFT)
        pull_site<TR, AM>(f, src, e, g, off, fc, seg, x, q);
    else
        gather_site<kPullNone, TR, AM>(f, src, e, g, off, fc, x, q);
    const bool bad = STRICT ? collide_site<true>(f, omega, mp) : collide_site_sym(f, omega, mp);
    if (bad) atomicOr(flag, 1);  // keeps other status bits (P2P timeout = 2)
    store_site<AM>(dst, e, g, off, f);
}

// ---------------------------------------------------------------------------
// P2P slab faces.  A face site is within 3 sites of a face shared with a
// neighbour: y-major storage, the 3 storage columns next to the face; x-major,
// lane 0's first 3 rows (lo) / lane vl-1's last 3 rows (hi).

template <bool TR>
__device__ __forceinline__ int face_side(const DevGeo& g, int x, int q) {
    if (TR) return x < kHalo ? 0 : x >= g.lx - kHalo ? 1 : -1;
    const int row = q >> g.lvl, k = q & (g.vl - 1);
    if (k == 0 && row < kHalo) return 0;
    if (k == g.vl - 1 && row >= g.strip - kHalo) return 1;
    return -1;
}

// The fused step on face sites that also stores each result into the
// neighbour's next buffer (its ghost slots for this site): the halo travels
// with the kernel's own stores over NVLink.
template <bool STRICT, bool TR>
__global__ void __launch_bounds__(kStreamThreads, kCollideMinBlocks)
    k_face(const double* __restrict__ src, double* __restrict__ dst, DevGeo g, Offsets off, Faces fc,
           ModelParams mp, double omega, Segments seg, int* __restrict__ flag, PeerStores ps) {
    int x, q;
    if (!segment_site(g, seg, x, q)) return;
    const long long e = site_of(g, x + kHalo, q);
    double f[kNpop];
    gather_site<kPullEdge, TR, kAddr64>(f, src, e, g, off, fc, x, q);
    const bool bad = STRICT ? collide_site<true>(f, omega, mp) : collide_site_sym(f, omega, mp);
    if (bad) atomicOr(flag, 1);  // keeps other status bits (P2P timeout = 2)
    store_site<kAddr64>(dst, e, g, off, f);
    const int side = face_side<TR>(g, x, q);
    double* peer = side == 0 ? ps.lo : side == 1 ? ps.hi : nullptr;
    if (peer) {
        store_site<kAddr64>(peer, e + (side == 0 ? ps.lo_shift : ps.hi_shift), g, off, f);
        __threadfence_system();  // performed before the step counter is released
    }
}

// Prime: copies the current state's face sites into the neighbours' current
// ghost slots (after a load / init / swap).
template <bool TR>
__global__ void __launch_bounds__(kStreamThreads) k_face_prime(const double* __restrict__ buf, DevGeo g, Offsets off,
                                                               Segments seg, PeerStores ps) {
    int x, q;
    if (!segment_site(g, seg, x, q)) return;
    const int side = face_side<TR>(g, x, q);
    double* peer = side == 0 ? ps.lo : side == 1 ? ps.hi : nullptr;
    if (!peer) return;
    const long long e = site_of(g, x + kHalo, q);
    const long long shift = side == 0 ? ps.lo_shift : ps.hi_shift;
#pragma unroll
    for (int p = 0; p < kNpop; ++p) peer[e + shift + p * g.pstride] = buf[e + p * g.pstride];
    __threadfence_system();
}

// ---------------------------------------------------------------------------
// P2P step counters (one thread each).

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}

__global__ void k_p2p_wait(const unsigned long long* seq, int need_lo, int need_hi, unsigned long long target,
                           unsigned long long timeout_ns, int* flag) {
    const unsigned long long t0 = global_ns();
    for (;;) {
        const bool lo = !need_lo || ld_acquire_sys(&seq[0]) >= target;
        const bool hi = !need_hi || ld_acquire_sys(&seq[1]) >= target;
        if (lo && hi) return;
        if (global_ns() - t0 > timeout_ns) {  // a neighbour never arrived: report, do not hang
            atomicOr(flag, 2);
            return;
        }
        __nanosleep(256);
    }
}

__global__ void k_p2p_signal(unsigned long long* lo_slot, unsigned long long* hi_slot, unsigned long long value) {
    __threadfence_system();
    if (lo_slot) st_release_sys(lo_slot, value);
    if (hi_slot) st_release_sys(hi_slot, value);
}

// ---------------------------------------------------------------------------
// Scalar device reference (validation.hpp:15-42, validation.cpp:13-38): a
// halo-free canonical array ((p*lx + x)*ly + y, dump.hpp:19-21) stepped with
// explicit modulo indexing and no layout machinery, so that run_validation
// can point a divergence at a layout or offset bug.  One thread per site.

__global__ void __launch_bounds__(256) k_scalar_propagate(const double* __restrict__ in, double* __restrict__ out,
                                                          int lx, int ly) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)lx * ly) return;
    const int x = int(t / ly), y = int(t - (long long)x * ly);
    const long long plane = (long long)lx * ly;
    for (int p = 0; p < kNpop; ++p) {
        const int xs = ((x - cx_of(p)) % lx + lx) % lx;
        const int ys = ((y - cy_of(p)) % ly + ly) % ly;
        out[p * plane + (long long)x * ly + y] = in[p * plane + (long long)xs * ly + ys];
    }
}

template <bool STRICT>
__global__ void __launch_bounds__(256) k_scalar_collide(const double* __restrict__ in, double* __restrict__ out,
                                                        int lx, int ly, ModelParams mp, double omega,
                                                        int* __restrict__ flag) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long plane = (long long)lx * ly;
    if (t >= plane) return;
    double f[kNpop];
#pragma unroll
    for (int p = 0; p < kNpop; ++p) f[p] = in[p * plane + t];
    const bool bad = STRICT ? collide_site<true>(f, omega, mp) : collide_site_sym(f, omega, mp);
    if (bad) atomicOr(flag, 1);  // keeps other status bits (P2P timeout = 2)
#pragma unroll
    for (int p = 0; p < kNpop; ++p) out[p * plane + t] = f[p];
}

// ---------------------------------------------------------------------------
// Edge (bc) kernel.  Thread t < nrows covers the ghost rows of every padded
// column (6 rows x vl lanes per (p, X)); t >= nrows covers the physical rows of
// the 6 ghost columns.  Every ghost slot is computed from its final physical
// source directly (ghost-column images of ghost rows included), so one pass
// reproduces the reference's y-then-x fill order.

__global__ void __launch_bounds__(256) k_edge(double* __restrict__ buf, DevGeo g, EdgeParams ep) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // lean: only the outer faces' ghost rows (lane 0 low, lane vl-1 high)
    const int nk = ep.lean ? 1 : g.vl;
    const long long nrows = (long long)kNpop * g.px * 6 * nk;
    if (t < nrows) {
        const int r = int((t / nk) % 6);
        const int k = ep.lean ? (r < 3 ? 0 : g.vl - 1) : int(t % nk);
        const int X = int((t / (6LL * nk)) % g.px);
        const int p = int(t / (6LL * nk * g.px));
        const int xs = wrapi(X - kHalo, g.lx);
        const int Xs = xs + kHalo;
        int j, y, q = p;
        bool remote = false;
        const double* rbuf = nullptr;
        int slot = -1;
        if (r < 3) {  // low-y ghost rows of lane k
            j = r;
            const int yraw = k * g.strip + r - kHalo;
            if (k > 0) {
                y = yraw;
            } else if (ep.face_lo == kFacePeriodic) {
                y = wrapi(yraw, g.ly);
            } else if (ep.face_lo == kFaceWall) {
                y = -1 - yraw;
                q = ep.ybar[p];
            } else {
                remote = true;
                slot = ep.lo_slot[kHalo - r - 1][p];
                rbuf = ep.recv_lo;
                y = 0;
            }
        } else {  // high-y ghost rows of lane k
            const int h = r - 3;
            j = g.strip + kHalo + h;
            const int yraw = (k + 1) * g.strip + h;
            if (k < g.vl - 1) {
                y = yraw;
            } else if (ep.face_hi == kFacePeriodic) {
                y = yraw % g.ly;
            } else if (ep.face_hi == kFaceWall) {
                y = 2 * g.ly - 1 - yraw;
                q = ep.ybar[p];
            } else {
                remote = true;
                slot = ep.hi_slot[h][p];
                rbuf = ep.recv_hi;
                y = 0;
            }
        }
        if (remote) {
            if (!(ep.filter & kEdgeRemote) || slot < 0) return;
            buf[elem_of(g, p, X, j, k)] = rbuf[(long long)slot * g.lx + xs];
        } else {
            if (!(ep.filter & kEdgeLocal)) return;
            buf[elem_of(g, p, X, j, k)] = buf[elem_of(g, q, Xs, y % g.strip + kHalo, y / g.strip)];
        }
        return;
    }
    if (!(ep.filter & kEdgeLocal)) return;
    const long long u = t - nrows;
    const long long ncols = (long long)kNpop * 6 * g.ly;
    if (u >= ncols) return;
    const int qq = int(u % g.ly);
    const int c = int((u / g.ly) % 6);
    const int p = int(u / (6LL * g.ly));
    const int X = c < 3 ? c : g.lx + kHalo + (c - 3);
    const int Xs = wrapi(X - kHalo, g.lx) + kHalo;
    buf[site_of(g, X, qq) + p * g.pstride] = buf[site_of(g, Xs, qq) + p * g.pstride];
}

// Slab boundary rows -> send buffers, [slot][x] contiguous.  send_hi carries
// rows ny-d of the (d, p) entries with cy_p >= d (the receiver's low ghosts),
// send_lo rows d-1 of the entries with cy_p <= -d.
__global__ void k_pack(const double* __restrict__ buf, DevGeo g, PackParams pp) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int total = pp.nslots * g.lx;
    if (t >= 2 * total) return;
    const bool hi = t >= total;
    const int u = hi ? t - total : t;
    const int slot = u / g.lx, x = u % g.lx;
    const int d = hi ? pp.hi_d[slot] : pp.lo_d[slot];
    const int p = hi ? pp.hi_p[slot] : pp.lo_p[slot];
    const int y = hi ? g.ly - d : d - 1;
    const double v = buf[elem_of(g, p, x + kHalo, y % g.strip + kHalo, y / g.strip)];
    (hi ? pp.send_hi : pp.send_lo)[u] = v;
}

// canonical plane p (x-major, y-minor, lx*ly values) <-> padded store
__global__ void k_scatter(double* __restrict__ buf, DevGeo g, const double* __restrict__ canon, int p) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)g.lx * g.ly) return;
    const int x = int(t / g.ly), q = int(t % g.ly);
    const int y = (q % g.vl) * g.strip + q / g.vl;
    buf[site_of(g, x + kHalo, q) + p * g.pstride] = canon[canon_index(g, x, y)];
}

__global__ void k_gather(const double* __restrict__ buf, DevGeo g, double* __restrict__ canon, int p) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)g.lx * g.ly) return;
    const int x = int(t / g.ly), q = int(t % g.ly);
    const int y = (q % g.vl) * g.strip + q / g.vl;
    canon[canon_index(g, x, y)] = buf[site_of(g, x + kHalo, q) + p * g.pstride];
}

// Lattice (x, y_local) of the storage site (column xs, storage y ys).
__device__ __forceinline__ void lattice_xy(const DevGeo& g, int xs, int ys, int& x, int& y) {
    x = g.tr ? ys : xs;
    y = g.tr ? xs : ys;
}

// Philox4x32-10, key = seed, counter = site-major index (x*ly_global + y)*37 + p.
__device__ __forceinline__ double philox_u01_dev(unsigned long long seed, unsigned long long ctr) {
    unsigned int c0 = (unsigned int)ctr, c1 = (unsigned int)(ctr >> 32), c2 = 0u, c3 = 0u;
    unsigned int k0 = (unsigned int)seed, k1 = (unsigned int)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const unsigned int hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const unsigned int hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const unsigned int n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    const unsigned long long bits = (unsigned long long)c0 | ((unsigned long long)c1 << 32);
    return (double)(bits >> 11) * 0x1.0p-53;
}

__global__ void k_philox(double* __restrict__ buf, DevGeo g, unsigned long long seed, int y0, int ly_global) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= g.ly) return;
    const int xs = blockIdx.y;
    int x, y;
    lattice_xy(g, xs, (q % g.vl) * g.strip + q / g.vl, x, y);
    const unsigned long long site = (unsigned long long)x * ly_global + (unsigned long long)(y0 + y);
    const long long e = site_of(g, xs + kHalo, q);
#pragma unroll 1
    for (int p = 0; p < kNpop; ++p) buf[e + p * g.pstride] = philox_u01_dev(seed, site * kNpop + p);
}

// BASELINE config-0/3/4 Rayleigh-Taylor-like init on the device: T = 1.5 below
// y_int(x) = ly_g/2 + 0.01 ly_g sin(2 pi x / lx), 0.5 above, plus U(-1e-3, 1e-3)
// noise from Philox keyed by the global site index x*ly_g + y; rho = 1/T, u = 0;
// f = equilibrium (model.cpp:259-291 operation order, DFMA-contracted).
__global__ void k_init_rt(double* __restrict__ buf, DevGeo g, ModelParams mp, unsigned long long seed, int y0,
                          int ly_global) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= g.ly) return;
    const int xs = blockIdx.y;
    int x, y;
    lattice_xy(g, xs, (q % g.vl) * g.strip + q / g.vl, x, y);
    y += y0;
    const int lx = g.tr ? g.ly : g.lx;
    const double noise = -1e-3 + 2e-3 * philox_u01_dev(seed, (unsigned long long)x * ly_global + y);
    const double yint = 0.5 * ly_global + 0.01 * ly_global * sin(2.0 * 3.14159265358979323846 * x / lx);
    const double temp = ((double)y < yint ? 1.5 : 0.5) + noise;
    const double rho = 1.0 / temp;
    const double dt = temp - mp.t0, dt2 = dt * dt;
    // u = 0: only the pure-temperature Hermite terms survive (mom 2, 4, 9, 11, 13)
    const double m2 = dt, m9 = 3.0 * dt2, m11 = dt2;
    const long long e = site_of(g, xs + kHalo, q);
#pragma unroll 1
    for (int p = 0; p < kNpop; ++p) {
        const double* gp = mp.eq[p];
        double s = 1.0;
        s += gp[2] * m2;
        s += gp[4] * m2;
        s += gp[9] * m9;
        s += gp[11] * m11;
        s += gp[13] * m9;
        buf[e + p * g.pstride] = rho * mp.w[p] * s;
    }
}

// Per-column sums {mass, jx, jy, sum |c|^2 f} in a fixed order (deterministic).
__global__ void __launch_bounds__(256) k_moments(const double* __restrict__ buf, DevGeo g, double* __restrict__ part) {
    __shared__ double red[4][256];
    const int X = blockIdx.x + kHalo;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = threadIdx.x; q < g.ly; q += blockDim.x) {
        const long long e = site_of(g, X, q);
#pragma unroll
        for (int p = 0; p < kNpop; ++p) {
            const double v = buf[e + p * g.pstride];
            s[0] += v;
            s[1] += cx_of(p) * v;
            s[2] += cy_of(p) * v;
            s[3] += (cx_of(p) * cx_of(p) + cy_of(p) * cy_of(p)) * v;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) red[i][threadIdx.x] = s[i];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
#pragma unroll
            for (int i = 0; i < 4; ++i) red[i][threadIdx.x] += red[i][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
#pragma unroll
        for (int i = 0; i < 4; ++i) part[blockIdx.x * 4 + i] = red[i][0];
}

// ---------------------------------------------------------------------------
// Launchers

static dim3 stream_grid(const DevGeo& g, const Segments& seg, int nseg) {
    if (seg.dense) {
        const long long n = (long long)seg.nq * nseg * g.lx;
        return dim3(unsigned((n + kStreamThreads - 1) / kStreamThreads), 1, 1);
    }
    return dim3((seg.nq + kStreamThreads - 1) / kStreamThreads, seg.nx > 0 ? seg.nx : g.lx, nseg);
}

// Address mode of a launch (see gather_site): the compile-time site-major
// store for the canonical pull offsets at vl = 32 / 16 / 1 (CAoSoA, AoS), else
// 32-bit or 64-bit offsets.
int addr_mode(const DevGeo& g, const Offsets& off) {
    if (off.canonical && g.pstride == g.vl && g.rstride == (long long)kNpop * g.vl && off.w32 &&
        (g.vl == 32 || g.vl == 16 || g.vl == 1))
        return g.vl;
    return off.w32 ? kAddr32 : kAddr64;
}

#define D2Q37_BY_ADDR(am, LAUNCH)             \
    switch (am) {                             \
        case 32: LAUNCH(32); break;           \
        case 16: LAUNCH(16); break;           \
        case 1: LAUNCH(1); break;             \
        case kAddr32: LAUNCH(kAddr32); break; \
        default: LAUNCH(kAddr64); break;      \
    }

cudaError_t launch_propagate(const double* src, double* dst, const DevGeo& g, const Offsets& off, const Faces& fc,
                             const Segments& seg, int nseg, cudaStream_t s) {
    if (seg.nq <= 0 || nseg <= 0) return cudaSuccess;
    const dim3 grid = stream_grid(g, seg, nseg);
    (void)cudaGetLastError();
#define D2Q37_PROP_T(AM) k_propagate<true, AM><<<grid, kStreamThreads, 0, s>>>(src, dst, g, off, fc, seg)
#define D2Q37_PROP_N(AM) k_propagate<false, AM><<<grid, kStreamThreads, 0, s>>>(src, dst, g, off, fc, seg)
    if (g.tr) {
        D2Q37_BY_ADDR(addr_mode(g, off), D2Q37_PROP_T)
    } else {
        D2Q37_BY_ADDR(addr_mode(g, off), D2Q37_PROP_N)
    }
#undef D2Q37_PROP_T
#undef D2Q37_PROP_N
    return cudaGetLastError();
}

namespace {
template <bool S, bool SH, bool TR>
void collide_am(dim3 grid, cudaStream_t s, const double* src, double* dst, const DevGeo& g, const Offsets& off,
                const Faces& fc, const ModelParams& mp, double omega, const Segments& seg, int* flag) {
#define D2Q37_COLL(AM) \
    k_collide<S, SH, TR, AM><<<grid, kStreamThreads, 0, s>>>(src, dst, g, off, fc, mp, omega, seg, flag)
    D2Q37_BY_ADDR(addr_mode(g, off), D2Q37_COLL)
#undef D2Q37_COLL
}
}  // namespace

cudaError_t launch_collide(const double* src, double* dst, const DevGeo& g, const Offsets& off, const Faces& fc,
                           const ModelParams& mp, double omega, bool strict, bool shift, const Segments& seg,
                           int nseg, int* flag, cudaStream_t s) {
    if (seg.nq <= 0 || nseg <= 0) return cudaSuccess;
    const dim3 grid = stream_grid(g, seg, nseg);
#define D2Q37_COLLIDE(S, SH, TR) collide_am<S, SH, TR>(grid, s, src, dst, g, off, fc, mp, omega, seg, flag)
    (void)cudaGetLastError();
    if (!shift) {  // no pull: the storage orientation does not matter
        if (strict)
            D2Q37_COLLIDE(true, false, false);
        else
            D2Q37_COLLIDE(false, false, false);
    } else if (strict) {
        if (g.tr)
            D2Q37_COLLIDE(true, true, true);
        else
            D2Q37_COLLIDE(true, true, false);
    } else {
        if (g.tr)
            D2Q37_COLLIDE(false, true, true);
        else
            D2Q37_COLLIDE(false, true, false);
    }
#undef D2Q37_COLLIDE
    return cudaGetLastError();
}
#undef D2Q37_BY_ADDR

// Plain device copy (also peer memory): the P2P prime uses it instead of
// cudaMemcpyAsync so that every GPU operation of the protocol is a kernel of
// this library, loaded up front.
__global__ void __launch_bounds__(256) k_copy(double* __restrict__ dst, const double* __restrict__ src, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t launch_copy(double* dst, const double* src, long long n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    (void)cudaGetLastError();
    const long long blocks = std::min<long long>((n + 255) / 256, 4096);
    k_copy<<<unsigned(blocks), 256, 0, s>>>(dst, src, n);
    return cudaGetLastError();
}

// With CUDA's lazy module loading (the default), the first launch of a kernel
// loads it, which can wait for the device to go idle.  A spin-waiting
// k_p2p_wait of another slab never lets it go idle, so the P2P transport loads
// every kernel up front (cudaFuncGetAttributes forces the load).
namespace {
template <typename F>
void load_kernel(F f) {
    cudaFuncAttributes a{};
    (void)cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f));
}
template <bool S, bool SH, bool TR>
void load_collide() {
    load_kernel(k_collide<S, SH, TR, 32>);
    load_kernel(k_collide<S, SH, TR, 16>);
    load_kernel(k_collide<S, SH, TR, 1>);
    load_kernel(k_collide<S, SH, TR, kAddr32>);
    load_kernel(k_collide<S, SH, TR, kAddr64>);
}
template <bool TR>
void load_propagate() {
    load_kernel(k_propagate<TR, 32>);
    load_kernel(k_propagate<TR, 16>);
    load_kernel(k_propagate<TR, 1>);
    load_kernel(k_propagate<TR, kAddr32>);
    load_kernel(k_propagate<TR, kAddr64>);
}
}  // namespace

cudaError_t preload_kernels() {
    load_collide<false, false, false>();
    load_collide<true, false, false>();
    load_collide<false, true, false>();
    load_collide<true, true, false>();
    load_collide<false, true, true>();
    load_collide<true, true, true>();
    load_propagate<false>();
    load_propagate<true>();
    load_kernel(k_p2p_wait);
    load_kernel(k_p2p_signal);
    load_kernel(k_copy);
    load_kernel(k_face<false, false>);
    load_kernel(k_face<true, false>);
    load_kernel(k_face<false, true>);
    load_kernel(k_face<true, true>);
    load_kernel(k_face_prime<false>);
    load_kernel(k_face_prime<true>);
    load_kernel(k_edge);
    load_kernel(k_pack);
    load_kernel(k_scatter);
    load_kernel(k_gather);
    load_kernel(k_philox);
    load_kernel(k_init_rt);
    load_kernel(k_moments);
    load_kernel(k_scalar_propagate);
    load_kernel(k_scalar_collide<false>);
    load_kernel(k_scalar_collide<true>);
    preload_band_kernels();
    return cudaGetLastError();
}

cudaError_t launch_face(const double* src, double* dst, const DevGeo& g, const Offsets& off, const Faces& fc,
                        const ModelParams& mp, double omega, bool strict, const Segments& seg, int nseg,
                        const PeerStores& ps, int* flag, cudaStream_t s) {
    if (seg.nq <= 0 || nseg <= 0) return cudaSuccess;
    const dim3 grid = stream_grid(g, seg, nseg);
    (void)cudaGetLastError();
#define D2Q37_FACE(S, TR) k_face<S, TR><<<grid, kStreamThreads, 0, s>>>(src, dst, g, off, fc, mp, omega, seg, flag, ps)
    if (g.tr) {
        if (strict)
            D2Q37_FACE(true, true);
        else
            D2Q37_FACE(false, true);
    } else {
        if (strict)
            D2Q37_FACE(true, false);
        else
            D2Q37_FACE(false, false);
    }
#undef D2Q37_FACE
    return cudaGetLastError();
}

cudaError_t launch_face_prime(const double* buf, const DevGeo& g, const Offsets& off, const Segments& seg, int nseg,
                              const PeerStores& ps, cudaStream_t s) {
    if (seg.nq <= 0 || nseg <= 0) return cudaSuccess;
    const dim3 grid = stream_grid(g, seg, nseg);
    (void)cudaGetLastError();
    if (g.tr)
        k_face_prime<true><<<grid, kStreamThreads, 0, s>>>(buf, g, off, seg, ps);
    else
        k_face_prime<false><<<grid, kStreamThreads, 0, s>>>(buf, g, off, seg, ps);
    return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const unsigned long long* seq, bool need_lo, bool need_hi, unsigned long long target,
                            unsigned long long timeout_ns, int* flag, cudaStream_t s) {
    if (!need_lo && !need_hi) return cudaSuccess;
    (void)cudaGetLastError();
    k_p2p_wait<<<1, 1, 0, s>>>(seq, need_lo ? 1 : 0, need_hi ? 1 : 0, target, timeout_ns, flag);
    return cudaGetLastError();
}

cudaError_t launch_p2p_signal(unsigned long long* lo_slot, unsigned long long* hi_slot, unsigned long long value,
                              cudaStream_t s) {
    if (!lo_slot && !hi_slot) return cudaSuccess;
    (void)cudaGetLastError();
    k_p2p_signal<<<1, 1, 0, s>>>(lo_slot, hi_slot, value);
    return cudaGetLastError();
}

cudaError_t launch_edge(double* buf, const DevGeo& g, const EdgeParams& ep, cudaStream_t s) {
    long long total = (long long)kNpop * g.px * 6 * (ep.lean ? 1 : g.vl);
    if (ep.filter & kEdgeLocal) total += (long long)kNpop * 6 * g.ly;
    const long long blocks = (total + 255) / 256;
    (void)cudaGetLastError();
    k_edge<<<(unsigned)blocks, 256, 0, s>>>(buf, g, ep);
    return cudaGetLastError();
}

cudaError_t launch_pack(const double* buf, const DevGeo& g, const PackParams& pp, cudaStream_t s) {
    const int total = 2 * pp.nslots * g.lx;
    if (total == 0) return cudaSuccess;
    (void)cudaGetLastError();
    k_pack<<<(total + 255) / 256, 256, 0, s>>>(buf, g, pp);
    return cudaGetLastError();
}

cudaError_t launch_scatter(double* buf, const DevGeo& g, const double* canon_plane, int p, cudaStream_t s) {
    if (g.band) return launch_band_scatter(buf, g, canon_plane, p, s);
    const long long n = (long long)g.lx * g.ly;
    (void)cudaGetLastError();
    k_scatter<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(buf, g, canon_plane, p);
    return cudaGetLastError();
}

cudaError_t launch_gather(const double* buf, const DevGeo& g, double* canon_plane, int p, cudaStream_t s) {
    if (g.band) return launch_band_gather(buf, g, canon_plane, p, s);
    const long long n = (long long)g.lx * g.ly;
    (void)cudaGetLastError();
    k_gather<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(buf, g, canon_plane, p);
    return cudaGetLastError();
}

cudaError_t launch_philox(double* buf, const DevGeo& g, unsigned long long seed, int y0, int ly_global,
                          cudaStream_t s) {
    (void)cudaGetLastError();
    k_philox<<<dim3((g.ly + 255) / 256, g.lx), 256, 0, s>>>(buf, g, seed, y0, ly_global);
    return cudaGetLastError();
}

cudaError_t launch_init_rt(double* buf, const DevGeo& g, const ModelParams& mp, unsigned long long seed, int y0,
                           int ly_global, cudaStream_t s) {
    if (g.band) return launch_band_init_rt(buf, g, mp, seed, y0, ly_global, s);
    (void)cudaGetLastError();
    k_init_rt<<<dim3((g.ly + 127) / 128, g.lx), 128, 0, s>>>(buf, g, mp, seed, y0, ly_global);
    return cudaGetLastError();
}

cudaError_t launch_scalar_step(const double* in, double* tmp, double* out, int lx, int ly, const ModelParams& mp,
                               double omega, bool strict, int* flag, cudaStream_t s) {
    const long long n = (long long)lx * ly;
    const unsigned blocks = unsigned((n + 255) / 256);
    (void)cudaGetLastError();
    k_scalar_propagate<<<blocks, 256, 0, s>>>(in, tmp, lx, ly);
    if (strict)
        k_scalar_collide<true><<<blocks, 256, 0, s>>>(tmp, out, lx, ly, mp, omega, flag);
    else
        k_scalar_collide<false><<<blocks, 256, 0, s>>>(tmp, out, lx, ly, mp, omega, flag);
    return cudaGetLastError();
}

cudaError_t launch_moments(const double* buf, const DevGeo& g, double* part, cudaStream_t s) {
    if (g.band) return launch_band_moments(buf, g, part, s);
    (void)cudaGetLastError();
    k_moments<<<g.lx, 256, 0, s>>>(buf, g, part);
    return cudaGetLastError();
}

}  // namespace d2q37
