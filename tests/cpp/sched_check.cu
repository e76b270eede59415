// sched_check.cu -- host-side check of the FUSED2 sweep schedules (test infrastructure, no GPU needed).
//
// Every (band, column) item of a sweep must be swept by exactly one persistent CTA, whatever the extents
// and CTA counts: the lockstep schedule (LockSched over lockstep_plan: whole rounds, the last round's
// own-band prefixes and the band-major tail, or the even split of few bands over many CTAs), the band-major ranges (RangeSched), and the overlapped slab
// plan of the pair form (pair_slab_plan: ghost-face CTAs' face + adjacent bands, main CTAs in lockstep).
// Also checks the balance the plans promise (no CTA more than one band-width plus the segment starts
// above the mean) and that a face CTA's schedule starts with its face items.
// Build: nvcc -std=c++17 -I../../paper_1804_01918_b200/csrc sched_check.cu -o _build/sched_check
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "d2q37_fused2.cuh"

using namespace d2q37;

static int failures = 0;
#define CHECK(c, ...)                              \
    do {                                           \
        if (!(c)) {                                \
            if (failures < 20) {                   \
                std::printf("FAIL %s: ", #c);      \
                std::printf(__VA_ARGS__);          \
                std::printf("\n");                 \
            }                                      \
            ++failures;                            \
        }                                          \
    } while (0)

// marks the items of one CTA's schedule; returns its work in iterations (columns + 7 per segment)
template <class S>
static long long walk(S s, int nb_total, int lx, std::vector<int>& hits, bool* first_face = nullptr) {
    long long work = 0;
    int band, xs, xe;
    while (s.next(band, xs, xe)) {
        CHECK(band >= 0 && band < nb_total && xs >= 0 && xe <= lx && xs < xe, "segment band %d [%d, %d)", band, xs,
              xe);
        if (!(band >= 0 && band < nb_total && xs >= 0 && xe <= lx && xs < xe)) return work;
        for (int x = xs; x < xe; ++x) ++hits[(size_t)band * lx + x];
        work += xe - xs + 7;
    }
    (void)first_face;
    return work;
}

static void check_lockstep(int nb, int G, int lx) {
    std::vector<int> hits((size_t)nb * lx, 0);
    const Lockstep ls = lockstep_plan(nb, G, lx);
    long long maxw = 0;
    for (int c = 0; c < G; ++c) {
        const long long w = walk(LockSched(0, lx, G, c, ls), nb, lx, hits);
        maxw = w > maxw ? w : maxw;
    }
    for (size_t i = 0; i < hits.size(); ++i) CHECK(hits[i] == 1, "lockstep nb %d G %d lx %d item %zu hit %d", nb, G, lx, i, hits[i]);
    const double mean = double(nb) * lx / G;
    CHECK(maxw <= mean + lx + 7.0 * (nb / G + 2) + 7.0 * (double(nb % G) / std::max(1, G - nb % G) + 2),
          "lockstep nb %d G %d lx %d: max work %lld vs mean %.0f", nb, G, lx, maxw, mean);
}

static void check_range(int nb, int G, int lx) {
    std::vector<int> hits((size_t)nb * lx, 0);
    const long long total = (long long)nb * lx, per = (total + G - 1) / G;
    for (int c = 0; c < G; ++c) walk(RangeSched(0, nb, lx, c * per, (c + 1) * per), nb, lx, hits);
    for (size_t i = 0; i < hits.size(); ++i) CHECK(hits[i] == 1, "range nb %d G %d lx %d item %zu", nb, G, lx, i);
}

static void check_slab(int lx, int ly, int flo, int fhi, int grid) {
    PairSlabPlan sp;
    if (!pair_slab_plan(lx, ly, flo, fhi, grid, &sp)) return;
    const int nbands = (ly + kT2Out - 1) / kT2Out;
    std::vector<int> hits((size_t)nbands * lx, 0);
    for (int cta = 0; cta < sp.nf_lo + sp.nf_hi; ++cta) {
        const bool lo = cta < sp.nf_lo;
        const long long c = lo ? cta : cta - sp.nf_lo;
        FaceSched fs = lo ? FaceSched{RangeSched(sp.lo_face0, sp.lo_face_nb, lx, c * sp.lo_face_per, (c + 1) * sp.lo_face_per),
                                      RangeSched(sp.lo_adj0, sp.lo_adj_nb, lx, c * sp.lo_adj_per, (c + 1) * sp.lo_adj_per), true}
                          : FaceSched{RangeSched(sp.hi_face0, sp.hi_face_nb, lx, c * sp.hi_face_per, (c + 1) * sp.hi_face_per),
                                      RangeSched(sp.hi_adj0, sp.hi_adj_nb, lx, c * sp.hi_adj_per, (c + 1) * sp.hi_adj_per), true};
        // face items first: once the schedule leaves the face bands it never returns
        FaceSched probe = fs;
        int band, xs, xe;
        bool left = false;
        while (probe.next(band, xs, xe)) {
            const bool face = lo ? band < sp.lo_face0 + sp.lo_face_nb : band >= sp.hi_face0;
            CHECK(!(left && face), "slab %dx%d: face CTA %d returns to a face band", lx, ly, cta);
            left = left || !face;
        }
        walk(fs, nbands, lx, hits);
    }
    const int G = grid - sp.nf_lo - sp.nf_hi;
    for (int c = 0; c < G; ++c) walk(LockSched(sp.main_band0, lx, G, c, sp.ls), nbands, lx, hits);
    for (size_t i = 0; i < hits.size(); ++i)
        CHECK(hits[i] == 1, "slab %dx%d faces %d/%d grid %d: band %zu col %zu hit %d", lx, ly, flo, fhi, grid,
              i / lx, i % lx, hits[i]);
    // the face bands' 6 edge rows are in the face CTAs' face items
    if (flo == 3) CHECK(sp.lo_face_nb >= 1 && sp.lo_face0 == 0, "slab %dx%d: low face band", lx, ly);
    if (fhi == 3) CHECK(sp.hi_face0 * kT2Out <= ly - 2 * kHalo, "slab %dx%d: high edge rows outside face bands", lx, ly);
}

int main() {
    const int lxs[] = {3, 7, 64, 256, 1000, 4096};
    const int nbs[] = {1, 2, 4, 5, 8, 9, 16, 35, 37, 69, 74, 135, 137, 147, 148, 149, 274, 300};
    const int Gs[] = {1, 4, 100, 135, 144, 147, 148};
    int n = 0;
    for (int lx : lxs)
        for (int nb : nbs)
            for (int G : Gs) {
                check_lockstep(nb, G, lx);
                check_range(nb, G, lx);
                ++n;
            }
    const int lys[] = {128, 480, 600, 1024, 1205, 2048, 4096, 8192, 16384, 40000};
    for (int lx : {128, 512, 4096})
        for (int ly : lys)
            for (int f : {0, 1, 2})
                for (int grid : {16, 100, 147}) {
                    const int flo = f == 1 ? 1 : 3, fhi = f == 2 ? 1 : 3;
                    check_slab(lx, ly, flo, fhi, grid);
                    ++n;
                }
    if (failures) {
        std::printf("sched_check: %d failures in %d configurations\n", failures, n);
        return 1;
    }
    std::printf("sched_check: OK (%d configurations, every item swept exactly once)\n", n);
    return 0;
}
