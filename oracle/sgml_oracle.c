/*
 * sgml_oracle.c — CPU restatement of the reference SGML solve path.
 *
 * TEST INFRASTRUCTURE ONLY (see sgml_oracle.h).  Not part of the product:
 * the B200 path never links or calls this file.  Parity is pinned against
 * the reference (SURVEY.md 6.2 histories, tests/golden, oracle/_ref).
 *
 * Build: gcc -std=c11 -O2 -fopenmp -ffp-contract=off -fPIC (no -march:
 * FMA contraction changes bits).
 *
 * Citations are to /root/reference/proj/core/{src,include/sgml}.
 */
#include "sgml_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OG_NEU 1

/* ---------------------------------------------------------------- grid -- */

/* grid.cpp:10-23 */
int og_make_grid(int dim, int n, og_grid* out) {
    if (dim != 2 && dim != 3) return OG_INVALID;
    if (n < 1 || n > 13) return OG_INVALID;
    out->dim = dim;
    out->n = n;
    out->N = (1 << n) + 1;
    out->pad_ = 0;
    out->h = 1.0 / (out->N - 1);
    out->total = 1;
    for (int d = 0; d < dim; ++d) out->total *= (uint64_t)out->N;
    return OG_OK;
}

/* grid.cpp:44-51 */
int og_on_dirichlet(const og_bc* bc, int dim, int N, int i, int j, int k) {
    const int c[3] = {i, j, k};
    for (int a = 0; a < dim; ++a) {
        if (c[a] == 0 && bc->kind[2 * a] != OG_NEU) return 1;
        if (c[a] == N - 1 && bc->kind[2 * a + 1] != OG_NEU) return 1;
    }
    return 0;
}

/* grid.cpp:53-62: lowest Dirichlet face id wins */
double og_dirichlet_value(const og_bc* bc, int dim, int N, int i, int j, int k) {
    const int c[3] = {i, j, k};
    for (int a = 0; a < dim; ++a) {
        if (c[a] == 0 && bc->kind[2 * a] != OG_NEU) return bc->value[2 * a];
        if (c[a] == N - 1 && bc->kind[2 * a + 1] != OG_NEU) return bc->value[2 * a + 1];
    }
    return NAN; /* reference throws std::logic_error; never reached by callers */
}

static inline size_t lin(int N, int i, int j, int k) {
    return (size_t)i + (size_t)N * ((size_t)j + (size_t)N * (size_t)k);
}

/* grid.hpp:63-69 */
static inline int mirror_index(int i, int N) {
    if (i < 0) i = -i;
    else if (i > N - 1) i = 2 * (N - 1) - i;
    return i;
}

/* ------------------------------------------------------------- stencil -- */

/* stencil.cpp:13-25: offsets in order r, q, p (skip the centre) */
typedef struct { int p, q, r; double inv_l2; } og_off;
static og_off OFF2[8], OFF3[26], CMP2[4], CMP3[6];
static int offs_ready = 0;

/* Stencil family.  0: the reference's radial 9/27-point form (stencil.cpp).
 * 1: the compact 5/7-point form the north star names and the reference does
 * not implement (parity UNPINNED, no reference): the
 * axis offsets only, in the same r, q, p order, inv_l2 = 1, prefactor 1,
 * step constant K = 1/(2d) (the Gershgorin bound, which reproduces the
 * reference's K_2 = 1/3 and K_3 = 13/44 for the radial form); same sigma
 * face average and ghosts. */
static int og_stencil_mode = 0;
void og_set_stencil(int mode) { og_stencil_mode = mode; }
int og_get_stencil(void) { return og_stencil_mode; }

static void build_offsets(void) {
    if (offs_ready) return;
    int c2 = 0, c3 = 0, k2 = 0, k3 = 0;
    for (int r = -1; r <= 1; ++r)
        for (int q = -1; q <= 1; ++q)
            for (int p = -1; p <= 1; ++p) {
                if (p == 0 && q == 0 && r == 0) continue;
                const int l2i = p * p + q * q + r * r;
                const double l2 = (double)l2i;
                OFF3[c3++] = (og_off){p, q, r, 1.0 / l2};
                if (r == 0) OFF2[c2++] = (og_off){p, q, 0, 1.0 / l2};
                if (l2i == 1) {
                    CMP3[k3++] = (og_off){p, q, r, 1.0};
                    if (r == 0) CMP2[k2++] = (og_off){p, q, 0, 1.0};
                }
            }
    offs_ready = 1;
}

static inline const og_off* offsets(int dim, int* count) {
    build_offsets();
    if (og_stencil_mode == 1) {
        *count = dim == 2 ? 4 : 6;
        return dim == 2 ? CMP2 : CMP3;
    }
    *count = dim == 2 ? 8 : 26;
    return dim == 2 ? OFF2 : OFF3;
}

/* stencil.hpp:49,52 (radial); compact: 1 and 1/(2d) */
static inline double prefactor(int dim) {
    if (og_stencil_mode == 1) return 1.0;
    return dim == 2 ? 0.5 : 3.0 / 13.0;
}
static inline double step_constant(int dim) {
    if (og_stencil_mode == 1) return dim == 2 ? 1.0 / 4.0 : 1.0 / 6.0;
    return dim == 2 ? 1.0 / 3.0 : 13.0 / 44.0;
}
/* stencil.hpp:65 / kernels.cpp:22 */
static const double AXW[3] = {0.25, 0.5, 0.25};

/* stencil.cpp:52-85: resolve x, then y, then z; Neumann even, Dirichlet odd
 * about the stored face value (mirror term evaluated before the face term). */
double og_ghost_value(const og_grid* g, const og_bc* bc, const double* u, int i, int j, int k) {
    const int N = g->N;
    if (i < 0) {
        const double m = og_ghost_value(g, bc, u, -i, j, k);
        if (bc->kind[0] == OG_NEU) return m;
        return 2.0 * og_ghost_value(g, bc, u, 0, j, k) - m;
    }
    if (i > N - 1) {
        const double m = og_ghost_value(g, bc, u, 2 * (N - 1) - i, j, k);
        if (bc->kind[1] == OG_NEU) return m;
        return 2.0 * og_ghost_value(g, bc, u, N - 1, j, k) - m;
    }
    if (j < 0) {
        const double m = og_ghost_value(g, bc, u, i, -j, k);
        if (bc->kind[2] == OG_NEU) return m;
        return 2.0 * og_ghost_value(g, bc, u, i, 0, k) - m;
    }
    if (j > N - 1) {
        const double m = og_ghost_value(g, bc, u, i, 2 * (N - 1) - j, k);
        if (bc->kind[3] == OG_NEU) return m;
        return 2.0 * og_ghost_value(g, bc, u, i, N - 1, k) - m;
    }
    if (k < 0) {
        const double m = og_ghost_value(g, bc, u, i, j, -k);
        if (bc->kind[4] == OG_NEU) return m;
        return 2.0 * og_ghost_value(g, bc, u, i, j, 0) - m;
    }
    if (k > N - 1) {
        const double m = og_ghost_value(g, bc, u, i, j, 2 * (N - 1) - k);
        if (bc->kind[5] == OG_NEU) return m;
        return 2.0 * og_ghost_value(g, bc, u, i, j, N - 1) - m;
    }
    return u[lin(N, i, j, k)];
}

/* stencil.cpp:87-90: sigma is always the even mirror */
static inline double mirror_value(const og_grid* g, const double* u, int i, int j, int k) {
    const int N = g->N;
    return u[lin(N, mirror_index(i, N), mirror_index(j, N), mirror_index(k, N))];
}

/* stencil.cpp:98-119 */
double og_restrict_at(const og_grid* g, const og_bc* bc, const double* f, int i, int j, int k, int lam) {
    double acc = 0.0;
    if (g->dim == 2) {
        for (int q = -1; q <= 1; ++q)
            for (int p = -1; p <= 1; ++p) {
                const double w = AXW[p + 1] * AXW[q + 1];
                acc += w * og_ghost_value(g, bc, f, i + p * lam, j + q * lam, 0);
            }
    } else {
        for (int r = -1; r <= 1; ++r)
            for (int q = -1; q <= 1; ++q)
                for (int p = -1; p <= 1; ++p) {
                    const double w = AXW[p + 1] * AXW[q + 1] * AXW[r + 1];
                    acc += w * og_ghost_value(g, bc, f, i + p * lam, j + q * lam, k + r * lam);
                }
    }
    return acc;
}

/* stencil.cpp:121-137 */
double og_apply_operator(const og_grid* g, const og_bc* bc, const double* u,
                         const double* sig, double a, int i, int j, int k, int lam) {
    const double s = lam * g->h;
    const size_t pos = lin(g->N, i, j, k);
    const double uc = u[pos];
    const double sc = sig ? sig[pos] : 1.0;
    int no;
    const og_off* off = offsets(g->dim, &no);
    double acc = 0.0;
    for (int o = 0; o < no; ++o) {
        const int ni = i + off[o].p * lam, nj = j + off[o].q * lam, nk = k + off[o].r * lam;
        const double un = og_ghost_value(g, bc, u, ni, nj, nk);
        const double sn = sig ? mirror_value(g, sig, ni, nj, nk) : 1.0;
        acc += 0.5 * (sn + sc) * (un - uc) * off[o].inv_l2;
    }
    return acc * prefactor(g->dim) / (s * s) + a * uc;
}

/* ------------------------------------------------------------- kernels -- */

/* kernels.cpp:28-81: one averaging pass at spacing lam */
void og_restrict_pass(const og_grid* g, const og_bc* bc, const double* in, double* out, int lam) {
    const int N = g->N, dim = g->dim;
    const int lo = lam, hi = N - 1 - lam;
    const ptrdiff_t sx = lam, sy = (ptrdiff_t)N * lam, sz = (ptrdiff_t)N * N * lam;
    const int KMAX = dim == 2 ? 1 : N;
#pragma omp parallel for collapse(2) schedule(static)
    for (int k = 0; k < KMAX; ++k)
        for (int j = 0; j < N; ++j) {
            const int zin = dim == 2 || (k >= lo && k <= hi);
            const int yin = j >= lo && j <= hi;
            for (int i = 0; i < N; ++i) {
                const size_t pos = lin(N, i, j, k);
                if (zin && yin && i >= lo && i <= hi) {
                    const double* c = in + pos;
                    double acc = 0.0;
                    if (dim == 2) {
                        for (int q = -1; q <= 1; ++q)
                            for (int p = -1; p <= 1; ++p)
                                acc += AXW[p + 1] * AXW[q + 1] * c[q * sy + p * sx];
                    } else {
                        for (int r = -1; r <= 1; ++r)
                            for (int q = -1; q <= 1; ++q)
                                for (int p = -1; p <= 1; ++p)
                                    acc += AXW[p + 1] * AXW[q + 1] * AXW[r + 1] *
                                           c[r * sz + q * sy + p * sx];
                    }
                    out[pos] = acc;
                } else {
                    out[pos] = og_restrict_at(g, bc, in, i, j, k, lam);
                }
            }
        }
}

/* kernels.cpp:305-325: v nested passes, lam = 1..2^(v-1), ping-pong ending in out */
void og_restriction_into(const og_grid* g, const og_bc* bc, const double* f, int v,
                         double* out, double* scratch, uint64_t* work) {
    if (v == 0) {
        memcpy(out, f, g->total * sizeof(double));
        return;
    }
    const double* src = f;
    double* dst = (v % 2 == 1) ? out : scratch;
    for (int m = 0; m < v; ++m) {
        og_restrict_pass(g, bc, src, dst, 1 << m);
        src = dst;
        dst = (dst == out) ? scratch : out;
    }
    if (work) *work += (uint64_t)v;
}

/* kernels.cpp:94-137: relax update at one subset node */
static double relax_node(const og_grid* gr, const og_bc* bc, const double* up, const double* sig,
                         const double* gsrc, int i, int j, int k, int lam, double inv_s2,
                         double pref, double kdim, double a, double safety, double* diag) {
    const int N = gr->N, dim = gr->dim;
    const size_t pos = lin(N, i, j, k);
    const double uc = up[pos];
    const double sc = sig ? sig[pos] : 1.0;
    const int fast = i >= lam && i <= N - 1 - lam && j >= lam && j <= N - 1 - lam &&
                     (dim == 2 || (k >= lam && k <= N - 1 - lam));
    int no;
    const og_off* off = offsets(dim, &no);
    double acc = 0.0, smax = 0.0;
    for (int o = 0; o < no; ++o) {
        double un, sbar;
        if (fast) {
            const ptrdiff_t dd = (((ptrdiff_t)off[o].r * N + off[o].q) * N + off[o].p) * lam;
            un = up[(ptrdiff_t)pos + dd];
            sbar = sig ? 0.5 * (sig[(ptrdiff_t)pos + dd] + sc) : 1.0;
        } else {
            const int ni = i + off[o].p * lam, nj = j + off[o].q * lam, nk = k + off[o].r * lam;
            un = og_ghost_value(gr, bc, up, ni, nj, nk);
            sbar = sig ? 0.5 * (mirror_value(gr, sig, ni, nj, nk) + sc) : 1.0;
        }
        acc += sbar * (un - uc) * off[o].inv_l2;
        smax = smax < sbar ? sbar : smax; /* std::max(smax, sbar) */
    }
    const double op = acc * pref * inv_s2;
    const double gc = gsrc[pos];
    *diag = fabs(op + a * uc - gc);
    const double dtau = safety * kdim / (inv_s2 * smax);
    if (!(dtau > 0.0)) return NAN;
    return (uc + dtau * (op - gc)) / (1.0 - dtau * a);
}

/* kernels.cpp:140-174: multilinear gather of du_prev.  Zero-weight corners on
 * non-Dirichlet high faces index past the row/plane; inside the
 * array the read is reproduced exactly, past its end it reads 0 (the
 * reference is undefined there). */
static double interp_node(const og_grid* g, const double* dup, int i, int j, int k, int lam,
                          double inv_lam) {
    const int m = lam - 1;
    const int i0 = i & ~m, j0 = j & ~m, k0 = k & ~m;
    const double fx = (i - i0) * inv_lam;
    const double fy = (j - j0) * inv_lam;
    const double wx[2] = {1.0 - fx, fx};
    const double wy[2] = {1.0 - fy, fy};
    const size_t N = (size_t)g->N;
    const size_t total = g->total;
    if (g->dim == 2) {
        const size_t b = lin((int)N, i0, j0, 0);
        double acc = 0.0;
        for (int q = 0; q < 2; ++q)
            for (int p = 0; p < 2; ++p) {
                const size_t idx = b + (size_t)q * lam * N + (size_t)p * lam;
                acc += wy[q] * wx[p] * (idx < total ? dup[idx] : 0.0);
            }
        return acc;
    } else {
        const double fz = (k - k0) * inv_lam;
        const double wz[2] = {1.0 - fz, fz};
        const size_t b = lin((int)N, i0, j0, k0);
        const size_t NN = N * N;
        double acc = 0.0;
        for (int r = 0; r < 2; ++r)
            for (int q = 0; q < 2; ++q)
                for (int p = 0; p < 2; ++p) {
                    const size_t idx = b + (size_t)r * lam * NN + (size_t)q * lam * N + (size_t)p * lam;
                    acc += wz[r] * wy[q] * wx[p] * (idx < total ? dup[idx] : 0.0);
                }
        return acc;
    }
}

/* kernels.cpp:176-237 + 334-349 */
int og_relaxation_interpolation(const og_grid* gr, const og_bc* bc, double* un, const double* up,
                                double* dun, const double* dup, int level, const double* gsrc,
                                const double* sig, double a, double safety, int homogeneous,
                                double* diag_out, uint64_t* work) {
    const int N = gr->N, dim = gr->dim;
    const int lam = 1 << level;
    const int mask = lam - 1;
    const double s = lam * gr->h;
    const double inv_s2 = 1.0 / (s * s);
    const double inv_lam = 1.0 / lam;
    const double pref = prefactor(dim);
    const double kdim = step_constant(dim);
    double diag_max = 0.0;
    int nonfinite = 0;
    const int badstep = !(safety > 0.0);
    const int KMAX = dim == 2 ? 1 : N;
    build_offsets();
#pragma omp parallel for collapse(2) schedule(static) reduction(max : diag_max) reduction(| : nonfinite)
    for (int k = 0; k < KMAX; ++k)
        for (int j = 0; j < N; ++j) {
            const int jk_face = j == 0 || j == N - 1 || (dim == 3 && (k == 0 || k == N - 1));
            const int jk_bits = j | (dim == 3 ? k : 0);
            for (int i = 0; i < N; ++i) {
                const size_t pos = lin(N, i, j, k);
                double value, du_value = 0.0;
                const int on_face = jk_face || i == 0 || i == N - 1;
                if (on_face && og_on_dirichlet(bc, dim, N, i, j, k)) {
                    value = homogeneous ? 0.0 : og_dirichlet_value(bc, dim, N, i, j, k);
                    du_value = value - up[pos];
                } else if (((i | jk_bits) & mask) == 0) {
                    double diag;
                    value = relax_node(gr, bc, up, sig, gsrc, i, j, k, lam, inv_s2, pref, kdim, a,
                                       safety, &diag);
                    diag_max = diag_max < diag ? diag : diag_max;
                    du_value = value - up[pos];
                } else {
                    value = up[pos] + interp_node(gr, dup, i, j, k, lam, inv_lam);
                }
                nonfinite |= !isfinite(value);
                un[pos] = value;
                dun[pos] = du_value;
            }
        }
    *diag_out = diag_max;
    if (badstep) return OG_BADSTEP;
    if (nonfinite) return OG_NONFINITE;
    if (work) *work += 1;
    return OG_OK;
}

/* kernels.cpp:243-286 (lam = 1) and 288-297, composed as in 351-358 */
void og_residual_update(const og_grid* g, const og_bc* bc, double* r, const double* e,
                        const double* sig, double a) {
    const int N = g->N, dim = g->dim;
    const double inv_h2 = 1.0 / (g->h * g->h);
    const double pref = prefactor(dim);
    int no;
    const og_off* off = offsets(dim, &no);
    const int KMAX = dim == 2 ? 1 : N;
#pragma omp parallel for collapse(2) schedule(static)
    for (int k = 0; k < KMAX; ++k)
        for (int j = 0; j < N; ++j) {
            const int jk_in = j >= 1 && j <= N - 2 && (dim == 2 || (k >= 1 && k <= N - 2));
            for (int i = 0; i < N; ++i) {
                const size_t pos = lin(N, i, j, k);
                const double ec = e[pos];
                const double sc = sig ? sig[pos] : 1.0;
                double acc = 0.0;
                if (jk_in && i >= 1 && i <= N - 2) {
                    for (int o = 0; o < no; ++o) {
                        const ptrdiff_t d = ((ptrdiff_t)off[o].r * N + off[o].q) * N + off[o].p;
                        const double sbar = sig ? 0.5 * (sig[(ptrdiff_t)pos + d] + sc) : 1.0;
                        acc += sbar * (e[(ptrdiff_t)pos + d] - ec) * off[o].inv_l2;
                    }
                } else {
                    for (int o = 0; o < no; ++o) {
                        const int ni = i + off[o].p, nj = j + off[o].q, nk = k + off[o].r;
                        const double en = og_ghost_value(g, bc, e, ni, nj, nk);
                        const double sbar = sig ? 0.5 * (mirror_value(g, sig, ni, nj, nk) + sc) : 1.0;
                        acc += sbar * (en - ec) * off[o].inv_l2;
                    }
                }
                r[pos] -= acc * pref * inv_h2 + a * ec;
            }
        }
    /* zero_dirichlet_faces */
    int anyd = 0;
    for (int f = 0; f < 2 * dim; ++f) anyd |= bc->kind[f] != OG_NEU;
    if (!anyd) return;
    for (int k = 0; k < KMAX; ++k)
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i)
                if (og_on_dirichlet(bc, dim, N, i, j, k)) r[lin(N, i, j, k)] = 0.0;
}

/* kernels.cpp:407-415 */
double og_max_abs(const double* f, uint64_t total) {
    double m = 0.0;
#pragma omp parallel for schedule(static) reduction(max : m)
    for (int64_t p = 0; p < (int64_t)total; ++p) {
        const double a = fabs(f[p]);
        m = m < a ? a : m;
    }
    return m;
}

/* kernels.cpp:367-386: serial Kahan sum in linear order */
double og_trapezoid_mean(const og_grid* g, const double* f) {
    const int N = g->N;
    double sum = 0.0, comp = 0.0;
    for (uint64_t pos = 0; pos < g->total; ++pos) {
        const int i = (int)(pos % (uint64_t)N);
        const int j = (int)((pos / (uint64_t)N) % (uint64_t)N);
        const int k = (int)(pos / ((uint64_t)N * N));
        double w = 1.0;
        if (i == 0 || i == N - 1) w *= 0.5;
        if (j == 0 || j == N - 1) w *= 0.5;
        if (g->dim == 3 && (k == 0 || k == N - 1)) w *= 0.5;
        const double y = w * f[pos] - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    double wsum = 1.0;
    for (int d = 0; d < g->dim; ++d) wsum *= (double)(N - 1);
    return sum / wsum;
}

/* kernels.cpp:388-395 */
void og_zero_mean_projection(const og_grid* g, double* f) {
    const double mean = og_trapezoid_mean(g, f);
    for (uint64_t p = 0; p < g->total; ++p) f[p] -= mean;
}

/* kernels.cpp:397-405 */
void og_apply_boundary(const og_grid* g, const og_bc* bc, double* u, int homogeneous) {
    const int N = g->N, dim = g->dim;
    const int KMAX = dim == 2 ? 1 : N;
    for (int k = 0; k < KMAX; ++k)
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i)
                if (og_on_dirichlet(bc, dim, N, i, j, k))
                    u[lin(N, i, j, k)] = homogeneous ? 0.0 : og_dirichlet_value(bc, dim, N, i, j, k);
}

/* ------------------------------------------------------------ schedule -- */

/* cycle.cpp:21-24 */
static int relax_count(int n, int n_r, int v1) {
    const long long doubling = 1LL << (n - v1);
    return (int)(n_r < doubling ? n_r : doubling);
}

/* cycle.cpp:28-45; kinds: 0 = restrict_source, 1 = relax */
int og_build_schedule(int n, int n_r, int* kinds, int* levels, int* counts, int cap) {
    if (n < 1 || n_r < 1) return -1;
    int c = 0;
#define PUSH(K, L, C)                                                   \
    do {                                                                \
        if (c < cap) { kinds[c] = (K); levels[c] = (L); counts[c] = (C); } \
        ++c;                                                            \
    } while (0)
    for (int v1 = n - 1; v1 >= 0; --v1) {
        const int cnt = relax_count(n, n_r, v1);
        for (int v = v1; v >= 0; --v) {
            PUSH(0, v, 1);
            PUSH(1, v, cnt);
        }
    }
    const long long tail_cap = n < 62 ? (1LL << n) : (long long)1 << 62;
    PUSH(1, 0, (int)(n_r < tail_cap ? n_r : tail_cap));
#undef PUSH
    return c;
}

/* cycle.cpp:47-59 */
uint64_t og_closed_form_work_units(int n, int n_r) {
    uint64_t total = 0;
    for (int v1 = 0; v1 <= n - 1; ++v1) {
        total += (uint64_t)v1 * (v1 + 1) / 2;
        total += (uint64_t)(v1 + 1) * relax_count(n, n_r, v1);
    }
    const long long tail_cap = n < 62 ? (1LL << n) : (long long)1 << 62;
    total += (uint64_t)(n_r < tail_cap ? n_r : tail_cap);
    return total;
}

/* -------------------------------------------------------------- driver -- */

static void push_sample(og_report* rep, int cycle, int pass, int level, double value) {
    if (rep->n_trace < rep->trace_cap) {
        og_sample* s = &rep->trace[rep->n_trace];
        s->cycle = cycle;
        s->pass = pass;
        s->level = level;
        s->pad_ = 0;
        s->value = value;
    }
    rep->n_trace++;
}

/* cycle.cpp:76-111.  State buffers swap by pointer, as std::swap of vectors
 * does; on return the final pass output is copied into u (state.u). */
int og_single_cycle(const og_grid* g, const og_bc* bc, double* u, double* u_prev, double* du,
                    double* du_prev, const double* source, const double* sigma_levels, double a,
                    int homogeneous, int n_r, double safety, int cycle_index, double normalization,
                    og_report* rep, uint64_t* work) {
    const size_t T = g->total;
    double* gbuf = (double*)calloc(T, sizeof(double));
    double* scratch = (double*)calloc(T, sizeof(double));
    double *bu = u, *bup = u_prev, *bdu = du, *bdup = du_prev;
    int kinds[512], levels[512], counts[512];
    const int ns = og_build_schedule(g->n, n_r, kinds, levels, counts, 512);
    int pass_index = 0, current_level = -1, status = OG_OK;
    const double inv_norm = normalization > 0.0 ? 1.0 / normalization : 1.0;
    for (int s = 0; s < ns && status == OG_OK; ++s) {
        if (kinds[s] == 0) {
            const uint64_t before = *work;
            og_restriction_into(g, bc, source, levels[s], gbuf, scratch, work);
            pass_index += (int)(*work - before);
        } else {
            if (levels[s] != current_level) { /* SolveState::reset_level */
                memset(bdu, 0, T * sizeof(double));
                memset(bdup, 0, T * sizeof(double));
                current_level = levels[s];
            }
            const double* sig = sigma_levels ? sigma_levels + (size_t)levels[s] * T : NULL;
            for (int c = 0; c < counts[s]; ++c) {
                double* t = bu; bu = bup; bup = t; /* swap_buffers */
                t = bdu; bdu = bdup; bdup = t;
                double diag = 0.0;
                status = og_relaxation_interpolation(g, bc, bu, bup, bdu, bdup, current_level, gbuf,
                                                     sig, a, safety, homogeneous, &diag, work);
                if (status != OG_OK) break;
                push_sample(rep, cycle_index, pass_index, current_level, diag * inv_norm);
                ++pass_index;
            }
        }
    }
    /* hand the buffers back in their roles */
    if (bu != u) {
        memcpy(u, bu, T * sizeof(double));
        memcpy(u_prev, bup, T * sizeof(double));
        memcpy(du, bdu, T * sizeof(double));
        memcpy(du_prev, bdup, T * sizeof(double));
    }
    free(gbuf);
    free(scratch);
    return status;
}

/* cycle.cpp:117-133: levels_out holds n fields of g->total doubles */
int og_restrict_sigma_levels(const og_grid* g, const double* sigma, double* levels_out) {
    og_bc even;
    for (int f = 0; f < 6; ++f) { even.kind[f] = OG_NEU; even.value[f] = 0.0; }
    const size_t T = g->total;
    double* scratch = (double*)malloc(T * sizeof(double));
    int status = OG_OK;
    for (int v = 0; v < g->n && status == OG_OK; ++v) {
        double* lv = levels_out + (size_t)v * T;
        og_restriction_into(g, &even, sigma, v, lv, scratch, NULL);
        for (size_t p = 0; p < T; ++p)
            if (!(lv[p] > 0.0)) { status = OG_INVALID; break; }
    }
    free(scratch);
    return status;
}

/* cycle.cpp:140-247 (problem.exact is not carried: the l1 column is off) */
int og_solve(const og_grid* g, const og_bc* bc, const double* f, const double* sigma, double a,
             int n_r, double tol, int max_cycles, double safety, double* u_total, og_report* rep) {
    if (!(tol > 0.0) || n_r < 1) return OG_INVALID;
    const size_t T = g->total;
    for (size_t p = 0; p < T; ++p)
        if (!isfinite(f[p])) return OG_INVALID;
    int all_neumann = 1;
    for (int fc = 0; fc < 2 * g->dim; ++fc) all_neumann &= bc->kind[fc] == OG_NEU;

    double* sigma_levels = NULL;
    if (sigma) {
        sigma_levels = (double*)malloc((size_t)g->n * T * sizeof(double));
        if (og_restrict_sigma_levels(g, sigma, sigma_levels) != OG_OK) {
            free(sigma_levels);
            return OG_INVALID;
        }
    }
    rep->n_rows = rep->n_trace = 0;
    rep->converged = rep->nan_detected = rep->stagnated = 0;
    rep->normalization = 0.0;
    rep->node_updates = 0;

    memset(u_total, 0, T * sizeof(double));
    double* r = (double*)malloc(T * sizeof(double));
    memcpy(r, f, T * sizeof(double));
    if (all_neumann) og_zero_mean_projection(g, r);
    double norm = og_max_abs(r, T);
    int norm_pending = norm == 0.0;

    double* su = (double*)calloc(T, sizeof(double));
    double* sup = (double*)calloc(T, sizeof(double));
    double* sdu = (double*)calloc(T, sizeof(double));
    double* sdup = (double*)calloc(T, sizeof(double));
    uint64_t work = 0, last_work = 0;
    double prev_res = INFINITY;
    int non_decreasing = 0;

    for (int cycle = 0; cycle < max_cycles; ++cycle) {
        const int homogeneous = cycle > 0;
        if (all_neumann && cycle > 0) og_zero_mean_projection(g, r);
        memset(su, 0, T * sizeof(double));
        memset(sup, 0, T * sizeof(double));
        const int64_t trace_mark = rep->n_trace;
        const int st = og_single_cycle(g, bc, su, sup, sdu, sdup, r, sigma_levels, a, homogeneous,
                                       n_r, safety, cycle, norm_pending ? 0.0 : norm, rep, &work);
        if (st != OG_OK) {
            rep->nan_detected = 1;
            rep->converged = 0;
            break;
        }
        rep->node_updates += (work - last_work) * T;
        last_work = work;
        for (size_t p = 0; p < T; ++p) u_total[p] += su[p];
        og_residual_update(g, bc, r, su, sigma, a);
        const double r_max = og_max_abs(r, T);
        if (norm_pending) {
            norm = r_max;
            norm_pending = 0;
            if (norm == 0.0) {
                if (rep->n_rows < rep->rows_cap)
                    rep->rows[rep->n_rows] = (og_row){cycle, 0, work, 0.0, 0.0};
                rep->n_rows++;
                rep->converged = 1;
                break;
            }
            for (int64_t t = trace_mark; t < rep->n_trace && t < rep->trace_cap; ++t)
                rep->trace[t].value /= norm;
        }
        const double res = r_max / norm;
        double diag_min = INFINITY;
        for (int64_t t = trace_mark; t < rep->n_trace && t < rep->trace_cap; ++t)
            diag_min = rep->trace[t].value < diag_min ? rep->trace[t].value : diag_min;
        if (rep->n_rows < rep->rows_cap)
            rep->rows[rep->n_rows] = (og_row){cycle, 0, work, res, diag_min};
        rep->n_rows++;
        if (!isfinite(res)) { rep->nan_detected = 1; break; }
        if (res <= tol) { rep->converged = 1; break; }
        if (res >= prev_res) {
            if (++non_decreasing >= 3) { rep->stagnated = 1; break; }
        } else {
            non_decreasing = 0;
        }
        prev_res = res;
    }
    rep->normalization = norm_pending ? 0.0 : norm;
    if (all_neumann && a == 0.0) og_zero_mean_projection(g, u_total); /* pure_neumann_pin */
    free(r); free(su); free(sup); free(sdu); free(sdup); free(sigma_levels);
    return OG_OK;
}

/* ------------------------------------------------------------ builders -- */

static const double OG_PI = 3.14159265358979323846;

/* problems.cpp:160-176 */
void og_fill_poisson2d(const og_grid* g, double* f) {
    const int N = g->N;
    for (uint64_t p = 0; p < g->total; ++p) {
        const int i = (int)(p % (uint64_t)N), j = (int)((p / (uint64_t)N) % (uint64_t)N);
        const double x = i * g->h, y = j * g->h;
        const double Px = x * x - x * x * x * x, Py = y * y - y * y * y * y;
        const double Dx = 2.0 - 12.0 * x * x, Dy = 2.0 - 12.0 * y * y;
        f[p] = -(Dx * Py + Px * Dy);
    }
}

/* problems.cpp:178-193 */
void og_fill_poisson3d(const og_grid* g, double* f) {
    const int N = g->N;
    for (uint64_t p = 0; p < g->total; ++p) {
        const int i = (int)(p % (uint64_t)N), j = (int)((p / (uint64_t)N) % (uint64_t)N);
        const int k = (int)(p / ((uint64_t)N * N));
        const double ex = sin(OG_PI * (i * g->h)) * sin(OG_PI * (j * g->h)) * sin(OG_PI * (k * g->h));
        f[p] = -3.0 * OG_PI * OG_PI * ex;
    }
}

/* BASELINE.json configs[0]: f = -2 pi^2 sin(pi x) sin(pi y), Dirichlet 0
 * (SURVEY.md 8(d) C1 literal form) */
void og_fill_sinsin2d(const og_grid* g, double* f) {
    const int N = g->N;
    for (uint64_t p = 0; p < g->total; ++p) {
        const int i = (int)(p % (uint64_t)N), j = (int)((p / (uint64_t)N) % (uint64_t)N);
        f[p] = -2.0 * OG_PI * OG_PI * sin(OG_PI * (i * g->h)) * sin(OG_PI * (j * g->h));
    }
}

/* problems.cpp:500-521 (sign = +1 "low", -1 "high") */
void og_fill_capacitor_sigma(const og_grid* g, double sign, double* sigma) {
    const int N = g->N;
    for (uint64_t p = 0; p < g->total; ++p) {
        const int i = (int)(p % (uint64_t)N), j = (int)((p / (uint64_t)N) % (uint64_t)N);
        const int k = (int)(p / ((uint64_t)N * N));
        const double dx = i * g->h - 0.5, dy = j * g->h - 0.5, dz = k * g->h - 0.5;
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        sigma[p] = 0.55 + sign * 0.45 * tanh((r - 0.2) / 0.1);
    }
}

/* kernels_tests.cpp:19-25 (the unit-test LCG: seed is pre-advanced once) */
void og_lcg_fill(double* f, uint64_t total, uint64_t seed) {
    uint64_t x = seed * 6364136223846793005ull + 1442695040888963407ull;
    for (uint64_t p = 0; p < total; ++p) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        f[p] = (double)(x >> 11) / (double)(1ull << 53) * 2.0 - 1.0;
    }
}

/* ======================================================================
 * Post-solve fields (problems.cpp:40-97, 327-455)
 * ====================================================================== */

/* problems.cpp:74-97: central differences inside, one-sided three-point
 * stencils on the two faces; inv2h = 1.0 / (2.0 * h) */
void og_axis_derivative(const og_grid* g, const double* u, int axis, double* out) {
    const int N = g->N;
    const ptrdiff_t s = axis == 0 ? 1 : (axis == 1 ? (ptrdiff_t)N : (ptrdiff_t)N * N);
    const double inv2h = 1.0 / (2.0 * g->h);
    for (uint64_t p = 0; p < g->total; ++p) {
        const int i = (int)(p % (uint64_t)N), j = (int)((p / (uint64_t)N) % (uint64_t)N),
                  k = (int)(p / ((uint64_t)N * (uint64_t)N));
        const int c = axis == 0 ? i : (axis == 1 ? j : k);
        double v;
        if (c == 0)
            v = (-3.0 * u[p] + 4.0 * u[p + s] - u[p + 2 * s]) * inv2h;
        else if (c == N - 1)
            v = (3.0 * u[p] - 4.0 * u[p - s] + u[p - 2 * s]) * inv2h;
        else
            v = (u[p + s] - u[p - s]) * inv2h;
        out[p] = v;
    }
}

/* problems.cpp:391-396 */
void og_gradient(const og_grid* g, const double* u, double* out) {
    for (int c = 0; c < g->dim; ++c) og_axis_derivative(g, u, c, out + (size_t)c * g->total);
}

/* problems.cpp:376-389 */
void og_curl(const og_grid* g, const double* psi, double* out) {
    const uint64_t T = g->total;
    double* d = (double*)malloc(6 * T * sizeof(double));
    double *dzy = d, *dyz = d + T, *dxz = d + 2 * T, *dzx = d + 3 * T, *dyx = d + 4 * T, *dxy = d + 5 * T;
    og_axis_derivative(g, psi + 2 * T, 1, dzy);
    og_axis_derivative(g, psi + 1 * T, 2, dyz);
    og_axis_derivative(g, psi + 0 * T, 2, dxz);
    og_axis_derivative(g, psi + 2 * T, 0, dzx);
    og_axis_derivative(g, psi + 1 * T, 0, dyx);
    og_axis_derivative(g, psi + 0 * T, 1, dxy);
    for (uint64_t p = 0; p < T; ++p) {
        out[p] = dzy[p] - dyz[p];
        out[T + p] = dxz[p] - dzx[p];
        out[2 * T + p] = dyx[p] - dxy[p];
    }
    free(d);
}

/* problems.cpp:398-405: d = 0; d += d_c v_c for c < dim */
void og_divergence(const og_grid* g, const double* v, double* out) {
    const uint64_t T = g->total;
    double* dc = (double*)malloc(T * sizeof(double));
    for (uint64_t p = 0; p < T; ++p) out[p] = 0.0;
    for (int c = 0; c < g->dim; ++c) {
        og_axis_derivative(g, v + (size_t)c * T, c, dc);
        for (uint64_t p = 0; p < T; ++p) out[p] += dc[p];
    }
    free(dc);
}

/* problems.cpp:327-341 */
int og_deformation_velocity(const og_grid* g, const double* u, const double* f_raw, double raw_integral,
                            double t, double* out) {
    og_gradient(g, u, out);
    for (int c = 0; c < g->dim; ++c) {
        double* comp = out + (size_t)c * g->total;
        for (uint64_t p = 0; p < g->total; ++p) {
            const double den = t * f_raw[p] + raw_integral;
            if (den == 0.0) return OG_INVALID;
            comp[p] = -comp[p] / den;
        }
    }
    return OG_OK;
}

/* std::clamp for doubles */
static double og_clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* problems.cpp:40-67 */
double og_sample_scalar(const og_grid* g, const double* f, const double* pt) {
    const int N = g->N;
    int idx[3] = {0, 0, 0};
    double frac[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < g->dim; ++c) {
        const double x = og_clampd(pt[c], 0.0, 1.0) / g->h;
        int i0 = (int)floor(x);
        i0 = i0 < 0 ? 0 : (N - 2 < i0 ? N - 2 : i0);
        idx[c] = i0;
        frac[c] = x - i0;
    }
    const double wx[2] = {1.0 - frac[0], frac[0]};
    const double wy[2] = {1.0 - frac[1], frac[1]};
    double acc = 0.0;
    if (g->dim == 2) {
        for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a)
                acc += wx[a] * wy[b] * f[(size_t)(idx[0] + a) + (size_t)N * (size_t)(idx[1] + b)];
    } else {
        const double wz[2] = {1.0 - frac[2], frac[2]};
        for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    acc += wx[a] * wy[b] * wz[c] *
                           f[(size_t)(idx[0] + a) + (size_t)N * ((size_t)(idx[1] + b) + (size_t)N * (size_t)(idx[2] + c))];
    }
    return acc;
}

/* problems.cpp:407-413 */
void og_sample_vector(const og_grid* g, const double* v, int nv, const double* pt, double* out) {
    out[0] = out[1] = out[2] = 0.0;
    for (int c = 0; c < nv; ++c) out[c] = og_sample_scalar(g, v + (size_t)c * g->total, pt);
}

/* problems.cpp:343-372 */
int og_move_nodes(const og_grid* g, const double* u, const double* f_raw, double raw_integral, double t,
                  int steps, double* pos) {
    if (steps < 1) return OG_INVALID;
    const uint64_t T = g->total;
    const int N = g->N;
    double* grad = (double*)malloc((size_t)g->dim * T * sizeof(double));
    og_gradient(g, u, grad);
    for (uint64_t p = 0; p < T; ++p) {
        const int i = (int)(p % (uint64_t)N), j = (int)((p / (uint64_t)N) % (uint64_t)N),
                  k = (int)(p / ((uint64_t)N * (uint64_t)N));
        pos[3 * p] = i * g->h;
        pos[3 * p + 1] = j * g->h;
        pos[3 * p + 2] = g->dim == 3 ? k * g->h : 0.0;
    }
    const double dt = t / steps;
    for (int s = 0; s < steps; ++s) {
        const double tau = s * dt;
        for (uint64_t p = 0; p < T; ++p) {
            double* x = pos + 3 * p;
            const double den = tau * og_sample_scalar(g, f_raw, x) + raw_integral;
            if (den == 0.0) continue;
            for (int c = 0; c < g->dim; ++c) {
                const double gc = og_sample_scalar(g, grad + (size_t)c * T, x);
                x[c] = og_clampd(x[c] - dt * gc / den, 0.0, 1.0);
            }
        }
    }
    free(grad);
    return OG_OK;
}

static int og_inside_unit(const double* p, int dim) {
    for (int c = 0; c < dim; ++c)
        if (!(p[c] >= 0.0 && p[c] <= 1.0)) return 0;
    return 1;
}

static double og_norm3(const double* a) { return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

/* problems.cpp:415-455 */
int og_integrate_streamline(const og_grid* g, const double* v, const double* seed, double step, int max_steps,
                            double* pts, int* stop) {
    int cnt = 0;
    double p[3] = {seed[0], seed[1], seed[2]};
#define OG_PUSH(q) do { pts[3 * cnt] = (q)[0]; pts[3 * cnt + 1] = (q)[1]; pts[3 * cnt + 2] = (q)[2]; ++cnt; } while (0)
    OG_PUSH(p);
    *stop = 0;
    if (!og_inside_unit(p, g->dim)) {
        *stop = 1;
        return cnt;
    }
    for (int s = 0; s < max_steps; ++s) {
        double k1[3], k2[3], k3[3], k4[3], q[3], nx[3];
        og_sample_vector(g, v, g->dim, p, k1);
        if (og_norm3(k1) < 1e-12) { *stop = 2; return cnt; }
        for (int c = 0; c < 3; ++c) q[c] = p[c] + 0.5 * step * k1[c];
        if (!og_inside_unit(q, g->dim)) { *stop = 1; return cnt; }
        og_sample_vector(g, v, g->dim, q, k2);
        for (int c = 0; c < 3; ++c) q[c] = p[c] + 0.5 * step * k2[c];
        if (!og_inside_unit(q, g->dim)) { *stop = 1; return cnt; }
        og_sample_vector(g, v, g->dim, q, k3);
        for (int c = 0; c < 3; ++c) q[c] = p[c] + step * k3[c];
        if (!og_inside_unit(q, g->dim)) { *stop = 1; return cnt; }
        og_sample_vector(g, v, g->dim, q, k4);
        for (int c = 0; c < 3; ++c) nx[c] = p[c];
        for (int c = 0; c < 3; ++c) nx[c] += step / 6.0 * (k1[c] + 2.0 * k2[c] + 2.0 * k3[c] + k4[c]);
        if (!og_inside_unit(nx, g->dim)) { *stop = 1; return cnt; }
        for (int c = 0; c < 3; ++c) p[c] = nx[c];
        OG_PUSH(p);
    }
#undef OG_PUSH
    return cnt;
}
