/*
 * d2q37_oracle.c -- TEST INFRASTRUCTURE ONLY (see d2q37_oracle.h).
 *
 * CPU restatement of the reference D2Q37 hot path in plain C.  Built with
 * -ffp-contract=off so every floating-point operation is one IEEE basic op in
 * the reference's source order; the product's STRICT math mode performs the
 * same operations with __dmul_rn/__dadd_rn and is checked against this file
 * bit for bit.  The reference's own release build contracts into FMA
 * (SURVEY.md 0.7), so against oracle/_ref the bar is the BASELINE tolerance.
 */
#include "d2q37_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------------- */
/* Model: model.cpp:14-19 (shell norms), :81-99 (velocity set)               */

static const int k_shell_norms[ORC_NSHELL] = {0, 1, 2, 4, 5, 8, 9, 10};

static int shell_index(int n2) {
    for (int s = 0; s < ORC_NSHELL; ++s)
        if (k_shell_norms[s] == n2) return s;
    return -1;
}

static int vel_less(int ax, int ay, int bx, int by) {
    const int na = ax * ax + ay * ay, nb = bx * bx + by * by;
    if (na != nb) return na < nb;
    if (ax != bx) return ax < bx;
    return ay < by;
}

static int build_velocity_set(int* cx, int* cy) {
    int n = 0;
    for (int x = -ORC_HALO; x <= ORC_HALO; ++x)
        for (int y = -ORC_HALO; y <= ORC_HALO; ++y)
            if (shell_index(x * x + y * y) >= 0) {
                if (n >= ORC_NPOP) return -1;
                cx[n] = x;
                cy[n] = y;
                ++n;
            }
    if (n != ORC_NPOP) return -1;
    /* insertion sort on (norm2, cx, cy) -- model.cpp:89-94 */
    for (int i = 1; i < n; ++i) {
        const int bx = cx[i], by = cy[i];
        int j = i - 1;
        while (j >= 0 && vel_less(bx, by, cx[j], cy[j])) {
            cx[j + 1] = cx[j];
            cy[j + 1] = cy[j];
            --j;
        }
        cx[j + 1] = bx;
        cy[j + 1] = by;
    }
    return 0;
}

/* model.cpp:23-29 */
static double gauss_moment_1d(int k, double t0) {
    if (k % 2 != 0) return 0.0;
    double df = 1.0;
    for (int j = k - 1; j > 0; j -= 2) df *= j;
    return df * pow(t0, (double)(k / 2));
}

/* model.cpp:65-70 */
static double ipow_d(int base, int e) {
    double r = 1.0;
    for (int i = 0; i < e; ++i) r *= base;
    return r;
}

/* model.cpp:36-44: solve conditions and the x^8 residual condition */
static const int k_solve_a[ORC_NSHELL] = {0, 2, 4, 2, 6, 4, 6, 4};
static const int k_solve_b[ORC_NSHELL] = {0, 0, 0, 2, 0, 2, 2, 4};
static const int k_res_a = 8, k_res_b = 0;

/* model.cpp:47-63: Gaussian elimination with partial pivoting */
static int solve_linear8(double a_in[ORC_NSHELL][ORC_NSHELL], const double* b_in, double* x) {
    double a[ORC_NSHELL][ORC_NSHELL], b[ORC_NSHELL];
    memcpy(a, a_in, sizeof a);
    memcpy(b, b_in, sizeof b);
    for (int col = 0; col < ORC_NSHELL; ++col) {
        int piv = col;
        for (int r = col + 1; r < ORC_NSHELL; ++r)
            if (fabs(a[r][col]) > fabs(a[piv][col])) piv = r;
        if (a[piv][col] == 0.0) return -1;
        for (int c = 0; c < ORC_NSHELL; ++c) {
            const double t = a[col][c];
            a[col][c] = a[piv][c];
            a[piv][c] = t;
        }
        {
            const double t = b[col];
            b[col] = b[piv];
            b[piv] = t;
        }
        for (int r = col + 1; r < ORC_NSHELL; ++r) {
            const double f = a[r][col] / a[col][col];
            for (int c = col; c < ORC_NSHELL; ++c) a[r][c] -= f * a[col][c];
            b[r] -= f * b[col];
        }
    }
    for (int r = ORC_NSHELL - 1; r >= 0; --r) {
        double s = b[r];
        for (int c = r + 1; c < ORC_NSHELL; ++c) s -= a[r][c] * x[c];
        x[r] = s / a[r][r];
    }
    return 0;
}

typedef struct {
    const int* cx;
    const int* cy;
    double a[ORC_NSHELL][ORC_NSHELL];
    double res_row[ORC_NSHELL];
} weight_ctx;

static double shell_sum(const weight_ctx* c, int s, int a, int b) {
    double acc = 0.0;
    for (int i = 0; i < ORC_NPOP; ++i)
        if (shell_index(c->cx[i] * c->cx[i] + c->cy[i] * c->cy[i]) == s)
            acc += ipow_d(c->cx[i], a) * ipow_d(c->cy[i], b);
    return acc;
}

static int weights_at(weight_ctx* c, double t0, double* w) {
    double b[ORC_NSHELL];
    for (int r = 0; r < ORC_NSHELL; ++r)
        b[r] = gauss_moment_1d(k_solve_a[r], t0) * gauss_moment_1d(k_solve_b[r], t0);
    return solve_linear8(c->a, b, w);
}

static double residual(weight_ctx* c, double t0) {
    double w[ORC_NSHELL];
    weights_at(c, t0, w);
    double r = -gauss_moment_1d(k_res_a, t0) * gauss_moment_1d(k_res_b, t0);
    for (int s = 0; s < ORC_NSHELL; ++s) r += c->res_row[s] * w[s];
    return r;
}

static double canonical_sum(const weight_ctx* c, const double* w) {
    double sum = 0.0;
    for (int i = 0; i < ORC_NPOP; ++i) sum += w[shell_index(c->cx[i] * c->cx[i] + c->cy[i] * c->cy[i])];
    return sum;
}

/* model.cpp:101-181 derive_weights */
static int derive_weights(const int* cx, const int* cy, double* shell_w, double* t0_out) {
    weight_ctx c;
    c.cx = cx;
    c.cy = cy;
    for (int r = 0; r < ORC_NSHELL; ++r)
        for (int s = 0; s < ORC_NSHELL; ++s) c.a[r][s] = shell_sum(&c, s, k_solve_a[r], k_solve_b[r]);
    for (int s = 0; s < ORC_NSHELL; ++s) c.res_row[s] = shell_sum(&c, s, k_res_a, k_res_b);

    const double lo0 = 0.1, hi0 = 2.0, step = 1e-3;
    double prev_t = lo0;
    double prev_r = residual(&c, lo0);
    for (double t = lo0 + step; t < hi0; t += step) {
        const double r = residual(&c, t);
        if (signbit(r) != signbit(prev_r)) {
            double lo = prev_t, hi = t, rlo = prev_r;
            for (int it = 0; it < 200 && hi - lo > 1e-16; ++it) {
                const double mid = 0.5 * (lo + hi);
                const double rm = residual(&c, mid);
                if (fabs(rm) < 1e-14) {
                    lo = hi = mid;
                    break;
                }
                if ((signbit(rm) != 0) == (signbit(rlo) != 0)) {
                    lo = mid;
                    rlo = rm;
                } else {
                    hi = mid;
                }
            }
            const double t0 = 0.5 * (lo + hi);
            double w[ORC_NSHELL];
            if (weights_at(&c, t0, w) != 0) return -1;
            int allpos = 1;
            for (int s = 0; s < ORC_NSHELL; ++s)
                if (!(w[s] > 0.0)) allpos = 0;
            if (allpos) {
                for (int pass = 0; pass < 4; ++pass) {
                    const double sum = canonical_sum(&c, w);
                    if (sum == 1.0) break;
                    for (int s = 0; s < ORC_NSHELL; ++s) w[s] /= sum;
                }
                for (int pass = 0; pass < 4; ++pass) {
                    const double sum = canonical_sum(&c, w);
                    if (sum == 1.0) break;
                    w[0] -= sum - 1.0;
                }
                memcpy(shell_w, w, sizeof w);
                *t0_out = t0;
                return 0;
            }
        }
        prev_t = t;
        prev_r = r;
    }
    return -1;
}

/* model.cpp:183-234 constructor: weights per population + Hermite table */
int orc_model_d2q37(orc_model* m) {
    memset(m, 0, sizeof *m);
    if (build_velocity_set(m->cx, m->cy) != 0) return -1;
    if (derive_weights(m->cx, m->cy, m->shell_w, &m->t0) != 0) return -1;
    const double t0 = m->t0;
    for (int i = 0; i < ORC_NPOP; ++i) {
        m->shell[i] = shell_index(m->cx[i] * m->cx[i] + m->cy[i] * m->cy[i]);
        m->w[i] = m->shell_w[m->shell[i]];
        const double cx = m->cx[i], cy = m->cy[i];
        const double cx2 = cx * cx, cy2 = cy * cy;
        const double h_x = cx;
        const double h_y = cy;
        const double h_xx = cx2 - t0;
        const double h_xy = cx * cy;
        const double h_yy = cy2 - t0;
        const double h_xxx = cx * cx2 - 3.0 * t0 * cx;
        const double h_xxy = cx2 * cy - t0 * cy;
        const double h_xyy = cx * cy2 - t0 * cx;
        const double h_yyy = cy * cy2 - 3.0 * t0 * cy;
        const double h_xxxx = cx2 * cx2 - 6.0 * t0 * cx2 + 3.0 * t0 * t0;
        const double h_xxxy = cx * cx2 * cy - 3.0 * t0 * cx * cy;
        const double h_xxyy = cx2 * cy2 - t0 * (cx2 + cy2) + t0 * t0;
        const double h_xyyy = cx * cy * cy2 - 3.0 * t0 * cx * cy;
        const double h_yyyy = cy2 * cy2 - 6.0 * t0 * cy2 + 3.0 * t0 * t0;
        const double t2 = t0 * t0, t3 = t2 * t0, t4 = t2 * t2;
        double* g = m->eq + i * ORC_NMOM;
        g[0] = h_x / t0;
        g[1] = h_y / t0;
        g[2] = h_xx / (2.0 * t2);
        g[3] = h_xy / t2;
        g[4] = h_yy / (2.0 * t2);
        g[5] = h_xxx / (6.0 * t3);
        g[6] = h_xxy / (2.0 * t3);
        g[7] = h_xyy / (2.0 * t3);
        g[8] = h_yyy / (6.0 * t3);
        g[9] = h_xxxx / (24.0 * t4);
        g[10] = h_xxxy / (6.0 * t4);
        g[11] = h_xxyy / (4.0 * t4);
        g[12] = h_xyyy / (6.0 * t4);
        g[13] = h_yyyy / (24.0 * t4);
    }
    return 0;
}

void orc_ymirror(const orc_model* m, int out[ORC_NPOP]) {
    for (int p = 0; p < ORC_NPOP; ++p) {
        out[p] = -1;
        for (int q = 0; q < ORC_NPOP; ++q)
            if (m->cx[q] == m->cx[p] && m->cy[q] == -m->cy[p]) out[p] = q;
    }
}

/* ------------------------------------------------------------------------- */
/* Per-site arithmetic: model.cpp:242-298                                    */

int orc_macros(const orc_model* m, const double* f, double mac[4]) {
    double rho = 0.0;
    for (int i = 0; i < ORC_NPOP; ++i) rho += f[i];
    const int bad = !(rho > 0.0);
    double jx = 0.0;
    for (int i = 0; i < ORC_NPOP; ++i) jx += (double)m->cx[i] * f[i];
    double jy = 0.0;
    for (int i = 0; i < ORC_NPOP; ++i) jy += (double)m->cy[i] * f[i];
    double e2 = 0.0;
    for (int i = 0; i < ORC_NPOP; ++i) e2 += (double)(m->cx[i] * m->cx[i] + m->cy[i] * m->cy[i]) * f[i];
    const double inv_rho = 1.0 / rho;
    const double ux = jx * inv_rho;
    const double uy = jy * inv_rho;
    const double temp = 0.5 * (e2 * inv_rho - (ux * ux + uy * uy));
    mac[0] = rho;
    mac[1] = ux;
    mac[2] = uy;
    mac[3] = temp;
    return bad;
}

void orc_equilibrium(const orc_model* m, const double mac[4], double* f_eq) {
    const double rho = mac[0], ux = mac[1], uy = mac[2];
    const double dt = mac[3] - m->t0;
    const double ux2 = ux * ux, uy2 = uy * uy, uxuy = ux * uy;
    const double dt3 = 3.0 * dt;
    const double dt6 = 6.0 * dt;
    const double dt2 = dt * dt;
    const double dt2x3 = 3.0 * dt2;
    double mom[ORC_NMOM];
    mom[0] = ux;
    mom[1] = uy;
    mom[2] = ux2 + dt;
    mom[3] = uxuy;
    mom[4] = uy2 + dt;
    mom[5] = ux * (ux2 + dt3);
    mom[6] = uy * (ux2 + dt);
    mom[7] = ux * (uy2 + dt);
    mom[8] = uy * (uy2 + dt3);
    mom[9] = ux2 * (ux2 + dt6) + dt2x3;
    mom[10] = uxuy * (ux2 + dt3);
    mom[11] = uxuy * uxuy + dt * (ux2 + uy2) + dt2;
    mom[12] = uxuy * (uy2 + dt3);
    mom[13] = uy2 * (uy2 + dt6) + dt2x3;
    for (int i = 0; i < ORC_NPOP; ++i) {
        const double* g = m->eq + i * ORC_NMOM;
        double s = 1.0;
        for (int k = 0; k < ORC_NMOM; ++k) s += g[k] * mom[k];
        f_eq[i] = rho * m->w[i] * s;
    }
}

int orc_collide_site(const orc_model* m, const double* f, double omega, double* out) {
    double mac[4], feq[ORC_NPOP];
    const int bad = orc_macros(m, f, mac);
    orc_equilibrium(m, mac, feq);
    for (int i = 0; i < ORC_NPOP; ++i) out[i] = f[i] + omega * (feq[i] - f[i]);
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Lattice level on canonical arrays                                        */

static inline size_t cidx(int lx, int ly, int p, int x, int y) {
    return ((size_t)p * lx + x) * ly + y;
}

static inline int wrap(int v, int n) { return ((v % n) + n) % n; }

typedef struct {
    const orc_model* m;
    int lx, ly, bc, r0, r1; /* rows r = p * lx + x of the canonical array, [r0, r1) */
    const int* ybar;
    const double* in;
    double* out;
} propagate_job;

static void* propagate_worker(void* arg) {
    const propagate_job* j = (const propagate_job*)arg;
    const orc_model* m = j->m;
    const int lx = j->lx, ly = j->ly, bc = j->bc;
    for (int r = j->r0; r < j->r1; ++r) {
        const int p = r / lx, x = r % lx;
        const int xs = wrap(x - m->cx[p], lx);
        for (int y = 0; y < ly; ++y) {
            const int gy = y - m->cy[p];
            int ys = gy, q = p;
            if (bc == ORC_BC_PERIODIC) {
                ys = wrap(gy, ly);
            } else if (gy < 0) {
                ys = -1 - gy;
                q = j->ybar[p];
            } else if (gy >= ly) {
                ys = 2 * ly - 1 - gy;
                q = j->ybar[p];
            }
            j->out[cidx(lx, ly, p, x, y)] = j->in[cidx(lx, ly, q, xs, ys)];
        }
    }
    return NULL;
}

/* The pull copy is a pure permutation of values, so the result does not depend on the thread count. */
int orc_propagate_mt(const orc_model* m, int lx, int ly, int bc, const double* in, double* out, int nthreads) {
    if (lx < 1 || ly < 1) return -1;
    if (bc == ORC_BC_WALL && ly < ORC_HALO) return -1;
    int ybar[ORC_NPOP];
    orc_ymirror(m, ybar);
    const long rows = (long)ORC_NPOP * lx;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads > rows) nthreads = (int)rows;
    if ((long)lx * ly < 65536) nthreads = 1; /* small lattices: not worth the thread start */
    propagate_job jobs[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].m = m;
        jobs[t].lx = lx;
        jobs[t].ly = ly;
        jobs[t].bc = bc;
        jobs[t].r0 = (int)(rows * t / nthreads);
        jobs[t].r1 = (int)(rows * (t + 1) / nthreads);
        jobs[t].ybar = ybar;
        jobs[t].in = in;
        jobs[t].out = out;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, propagate_worker, &jobs[t]);
    propagate_worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    return 0;
}

int orc_propagate(const orc_model* m, int lx, int ly, int bc, const double* in, double* out) {
    return orc_propagate_mt(m, lx, ly, bc, in, out, 1);
}

typedef struct {
    const orc_model* m;
    int lx, ly, x0, x1;
    double omega;
    const double* in;
    double* out;
    int bad;
} collide_job;

static void* collide_worker(void* arg) {
    collide_job* j = (collide_job*)arg;
    double f[ORC_NPOP], fpost[ORC_NPOP];
    for (int x = j->x0; x < j->x1; ++x)
        for (int y = 0; y < j->ly; ++y) {
            for (int p = 0; p < ORC_NPOP; ++p) f[p] = j->in[cidx(j->lx, j->ly, p, x, y)];
            j->bad |= orc_collide_site(j->m, f, j->omega, fpost);
            for (int p = 0; p < ORC_NPOP; ++p) j->out[cidx(j->lx, j->ly, p, x, y)] = fpost[p];
        }
    return NULL;
}

int orc_collide(const orc_model* m, int lx, int ly, double omega, const double* in, double* out,
                int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > lx) nthreads = lx;
    collide_job jobs[256];
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].m = m;
        jobs[t].lx = lx;
        jobs[t].ly = ly;
        jobs[t].x0 = (int)((long)lx * t / nthreads);
        jobs[t].x1 = (int)((long)lx * (t + 1) / nthreads);
        jobs[t].omega = omega;
        jobs[t].in = in;
        jobs[t].out = out;
        jobs[t].bad = 0;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, collide_worker, &jobs[t]);
    collide_worker(&jobs[0]);
    int bad = jobs[0].bad;
    for (int t = 1; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        bad |= jobs[t].bad;
    }
    return bad ? 1 : 0;
}

int orc_step(const orc_model* m, int lx, int ly, int bc, double omega, int nsteps, double* state,
             double* scratch, int nthreads) {
    int bad = 0;
    for (int s = 0; s < nsteps; ++s) {
        if (orc_propagate_mt(m, lx, ly, bc, state, scratch, nthreads) != 0) return -1;
        bad |= orc_collide(m, lx, ly, omega, scratch, state, nthreads);
    }
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Reference padded layouts (layout.hpp:46-98): vl == 1 is SoA, vl > 1 CSoA   */

static int padded_ok(int lx, int ly, int vl) {
    if (lx < 1 || ly < 1 || vl < 1 || (vl & (vl - 1)) != 0) return 0;
    if (vl > 1 && (ly % vl != 0 || ly / vl < ORC_HALO)) return 0;
    return 1;
}

size_t orc_padded_elems(int lx, int ly, int vl) {
    if (!padded_ok(lx, ly, vl)) return 0;
    const size_t strip = (size_t)(ly / vl), sy = strip + 2 * ORC_HALO, px = (size_t)lx + 2 * ORC_HALO;
    return px * sy * ORC_NPOP * (size_t)vl;
}

size_t orc_padded_index(int lx, int ly, int vl, int p, int X, int j, int k) {
    const size_t sy = (size_t)(ly / vl) + 2 * ORC_HALO, px = (size_t)lx + 2 * ORC_HALO;
    return (((size_t)p * px * sy) + (size_t)X * sy + (size_t)j) * (size_t)vl + (size_t)k;
}

int orc_canonical_to_padded(int lx, int ly, int vl, const double* canon, double* padded) {
    if (!padded_ok(lx, ly, vl)) return -1;
    const int strip = ly / vl;
    for (int p = 0; p < ORC_NPOP; ++p)
        for (int x = 0; x < lx; ++x)
            for (int y = 0; y < ly; ++y)
                padded[orc_padded_index(lx, ly, vl, p, x + ORC_HALO, y % strip + ORC_HALO, y / strip)] =
                    canon[cidx(lx, ly, p, x, y)];
    return 0;
}

int orc_padded_to_canonical(int lx, int ly, int vl, const double* padded, double* canon) {
    if (!padded_ok(lx, ly, vl)) return -1;
    const int strip = ly / vl;
    for (int p = 0; p < ORC_NPOP; ++p)
        for (int x = 0; x < lx; ++x)
            for (int y = 0; y < ly; ++y)
                canon[cidx(lx, ly, p, x, y)] =
                    padded[orc_padded_index(lx, ly, vl, p, x + ORC_HALO, y % strip + ORC_HALO, y / strip)];
    return 0;
}

/* kernels.cpp:197-234; in WALL mode the two outer faces (lane 0 top, lane
 * vl-1 bottom) take the specular image f(X, mirror(y), ybar(p)) instead of the
 * periodic wrap.  Inner lane-strip halos are unchanged. */
int orc_halo_fill(const orc_model* m, int lx, int ly, int vl, int bc, double* a) {
    if (!padded_ok(lx, ly, vl)) return -1;
    if (bc == ORC_BC_WALL && ly < ORC_HALO) return -1;
    int ybar[ORC_NPOP];
    orc_ymirror(m, ybar);
    const int strip = ly / vl, sy = strip + 2 * ORC_HALO;
    for (int x = 0; x < lx; ++x) {
        const int X = x + ORC_HALO;
        for (int p = 0; p < ORC_NPOP; ++p)
            for (int k = 0; k < vl; ++k)
                for (int h = 0; h < ORC_HALO; ++h) {
                    /* top ghost row j = h */
                    int yraw = k * strip + h - ORC_HALO, ys, q = p;
                    if (bc == ORC_BC_WALL && yraw < 0) {
                        ys = -1 - yraw;
                        q = ybar[p];
                    } else {
                        ys = wrap(yraw, ly);
                    }
                    a[orc_padded_index(lx, ly, vl, p, X, h, k)] =
                        a[orc_padded_index(lx, ly, vl, q, X, ys % strip + ORC_HALO, ys / strip)];
                    /* bottom ghost row j = strip + 3 + h */
                    yraw = (k + 1) * strip + h;
                    q = p;
                    if (bc == ORC_BC_WALL && yraw >= ly) {
                        ys = 2 * ly - 1 - yraw;
                        q = ybar[p];
                    } else {
                        ys = yraw % ly;
                    }
                    a[orc_padded_index(lx, ly, vl, p, X, strip + ORC_HALO + h, k)] =
                        a[orc_padded_index(lx, ly, vl, q, X, ys % strip + ORC_HALO, ys / strip)];
                }
    }
    for (int side = 0; side < 2; ++side)
        for (int h = 0; h < ORC_HALO; ++h) {
            const int X = side == 0 ? h : lx + ORC_HALO + h;
            const int x = side == 0 ? h - ORC_HALO : lx + h;
            const int Xs = wrap(x, lx) + ORC_HALO;
            for (int p = 0; p < ORC_NPOP; ++p)
                for (int j = 0; j < sy; ++j)
                    for (int k = 0; k < vl; ++k)
                        a[orc_padded_index(lx, ly, vl, p, X, j, k)] = a[orc_padded_index(lx, ly, vl, p, Xs, j, k)];
        }
    return 0;
}

/* kernels.cpp:50-85 + build_offset_table kernels.cpp:180-195 */
int orc_propagate_padded(const orc_model* m, int lx, int ly, int vl, const double* in, double* out) {
    if (!padded_ok(lx, ly, vl)) return -1;
    const int strip = ly / vl;
    const long sy = strip + 2 * ORC_HALO;
    for (int p = 0; p < ORC_NPOP; ++p) {
        const long off = -((long)m->cx[p] * sy + m->cy[p]);
        for (int x = 0; x < lx; ++x)
            for (int j = ORC_HALO; j < ORC_HALO + strip; ++j)
                for (int k = 0; k < vl; ++k) {
                    const size_t e = orc_padded_index(lx, ly, vl, p, x + ORC_HALO, j, k);
                    out[e] = in[(size_t)((long)e + off * vl)];
                }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* std::mt19937_64: w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555
 * s=17 b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005 */

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

double orc_mt64_u01(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }

void orc_mt64_fill_u01(uint64_t seed, size_t n, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) out[i] = orc_mt64_u01(&g);
}

/* Philox4x32-10 */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* ------------------------------------------------------------------------- */
/* Initialisers                                                              */

void orc_random_lattice(const orc_model* m, int lx, int ly, uint64_t seed, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    double feq[ORC_NPOP], mac[4];
    for (int x = 0; x < lx; ++x)
        for (int y = 0; y < ly; ++y) {
            /* brace-init order rho, ux, uy, temp (lattice.cpp:16-17) */
            mac[0] = 0.9 + 0.2 * orc_mt64_u01(&g);
            mac[1] = -0.05 + 0.1 * orc_mt64_u01(&g);
            mac[2] = -0.05 + 0.1 * orc_mt64_u01(&g);
            mac[3] = m->t0 * (0.9 + 0.2 * orc_mt64_u01(&g));
            orc_equilibrium(m, mac, feq);
            for (int p = 0; p < ORC_NPOP; ++p)
                out[cidx(lx, ly, p, x, y)] = feq[p] * (1.0 + 2e-3 * (orc_mt64_u01(&g) - 0.5));
        }
}

void orc_equilibrium_lattice(const orc_model* m, int lx, int ly, const double mac[4], double* out) {
    double feq[ORC_NPOP];
    orc_equilibrium(m, mac, feq);
    for (int p = 0; p < ORC_NPOP; ++p)
        for (int x = 0; x < lx; ++x)
            for (int y = 0; y < ly; ++y) out[cidx(lx, ly, p, x, y)] = feq[p];
}

void orc_shear_lattice(const orc_model* m, int lx, int ly, double amp, double temp, double* out) {
    double feq[ORC_NPOP];
    for (int y = 0; y < ly; ++y) {
        const double mac[4] = {1.0, amp * sin(2.0 * ORC_PI * y / ly), 0.0, temp};
        orc_equilibrium(m, mac, feq);
        for (int x = 0; x < lx; ++x)
            for (int p = 0; p < ORC_NPOP; ++p) out[cidx(lx, ly, p, x, y)] = feq[p];
    }
}

void orc_rt_lattice(const orc_model* m, int lx, int ly, uint64_t seed, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    double feq[ORC_NPOP], mac[4];
    for (int x = 0; x < lx; ++x) {
        const double yint = 0.5 * ly + 0.01 * ly * sin(2.0 * ORC_PI * x / lx);
        for (int y = 0; y < ly; ++y) {
            const double noise = -1e-3 + 2e-3 * orc_mt64_u01(&g);
            const double temp = ((double)y < yint ? 1.5 : 0.5) + noise;
            mac[0] = 1.0 / temp;
            mac[1] = 0.0;
            mac[2] = 0.0;
            mac[3] = temp;
            orc_equilibrium(m, mac, feq);
            for (int p = 0; p < ORC_NPOP; ++p) out[cidx(lx, ly, p, x, y)] = feq[p];
        }
    }
}

static double philox_u01(uint64_t seed, uint64_t counter) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const uint32_t ctr[4] = {(uint32_t)counter, (uint32_t)(counter >> 32), 0u, 0u};
    uint32_t r[4];
    orc_philox4x32_10(ctr, key, r);
    return (double)((((uint64_t)r[1] << 32) | r[0]) >> 11) * 0x1.0p-53;
}

void orc_rt_philox_lattice(const orc_model* m, int lx, int ly, int ly_global, int y0, uint64_t seed, double* out) {
    double feq[ORC_NPOP], mac[4];
    for (int x = 0; x < lx; ++x) {
        const double yint = 0.5 * ly_global + 0.01 * ly_global * sin(2.0 * ORC_PI * x / lx);
        for (int y = 0; y < ly; ++y) {
            const int yg = y0 + y;
            const double noise = -1e-3 + 2e-3 * philox_u01(seed, (uint64_t)x * (uint64_t)ly_global + (uint64_t)yg);
            const double temp = ((double)yg < yint ? 1.5 : 0.5) + noise;
            mac[0] = 1.0 / temp;
            mac[1] = 0.0;
            mac[2] = 0.0;
            mac[3] = temp;
            orc_equilibrium(m, mac, feq);
            for (int p = 0; p < ORC_NPOP; ++p) out[cidx(lx, ly, p, x, y)] = feq[p];
        }
    }
}

void orc_c2_lattice(const orc_model* m, int lx, int ly, uint64_t seed, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    double feq[ORC_NPOP], mac[4];
    for (int x = 0; x < lx; ++x)
        for (int y = 0; y < ly; ++y) {
            mac[0] = 0.95 + 0.1 * orc_mt64_u01(&g);
            mac[1] = -0.05 + 0.1 * orc_mt64_u01(&g);
            mac[2] = -0.05 + 0.1 * orc_mt64_u01(&g);
            mac[3] = 0.9 + 0.2 * orc_mt64_u01(&g);
            orc_equilibrium(m, mac, feq);
            for (int p = 0; p < ORC_NPOP; ++p)
                out[cidx(lx, ly, p, x, y)] = feq[p] * (1.0 + 2e-3 * (orc_mt64_u01(&g) - 0.5));
        }
}

void orc_philox_lattice(int lx, int ly, uint64_t seed, double* out) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int x = 0; x < lx; ++x)
        for (int y = 0; y < ly; ++y)
            for (int p = 0; p < ORC_NPOP; ++p) {
                const uint64_t idx = ((uint64_t)x * (uint64_t)ly + (uint64_t)y) * ORC_NPOP + (uint64_t)p;
                const uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), 0u, 0u};
                uint32_t r[4];
                orc_philox4x32_10(ctr, key, r);
                const uint64_t bits = (uint64_t)r[0] | ((uint64_t)r[1] << 32);
                out[cidx(lx, ly, p, x, y)] = (double)(bits >> 11) * 0x1.0p-53;
            }
}
