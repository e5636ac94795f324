/*
 * sgml_oracle.h — CPU restatement of the reference SGML solve path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 kernels in paper_1703_07206_b200/csrc.  Only tests/, the smoke()
 * check in __graft_entry__.py and the cpu_baseline / --impl reference legs
 * of bench.py may load it.  The product path never links or calls it.
 *
 * Every function restates the algorithm of the reference C++ core at
 * /root/reference/proj/core (cited file:line), in plain C, with the same
 * IEEE operation order (compile with -ffp-contract=off, no -march) so that
 * results are bit-identical to the reference built the same way.
 * Pinning: tests/test_oracle_pinning.py checks this restatement against
 *   (1) the residual histories measured from the reference,
 *   (2) golden vectors generated from the reference itself
 *       (tests/golden/make_golden.py, which drives oracle/_ref), and
 *   (3) the live reference build in oracle/_ref when present.
 */
#ifndef SGML_ORACLE_H
#define SGML_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* grid.hpp:31-39 */
typedef struct {
    int dim;
    int n;
    int N;
    int pad_;
    double h;
    uint64_t total;
} og_grid;

/* grid.hpp:125-157; kind 0 = dirichlet, 1 = neumann (BcKind order) */
typedef struct {
    int kind[6];
    double value[6];
} og_bc;

/* cycle.hpp:81-89 without the optional l1 column */
typedef struct {
    int cycle;
    int pad_;
    uint64_t work_units;
    double residual;
    double diag_min;
} og_row;

/* cycle.hpp:74-79 */
typedef struct {
    int cycle;
    int pass;
    int level;
    int pad_;
    double value;
} og_sample;

/* cycle.hpp:91-99 with caller-owned arrays */
typedef struct {
    og_row* rows;
    int64_t rows_cap;
    int64_t n_rows;
    og_sample* trace;
    int64_t trace_cap;
    int64_t n_trace;
    int converged;
    int nan_detected;
    int stagnated;
    int pad_;
    double normalization;
    uint64_t node_updates;
} og_report;

/* status codes shared with the product C-ABI */
enum { OG_OK = 0, OG_INVALID = 1, OG_BADSTEP = 2, OG_NONFINITE = 3 };

/* stencil family for every function below (test infrastructure switch):
 * 0 = the reference's radial form (default), 1 = compact 5/7-point (SURVEY.md
 * 8a row a23, parity unpinned: the reference has no such stencil) */
void og_set_stencil(int mode);
int og_get_stencil(void);

int og_make_grid(int dim, int n, og_grid* out);
int og_on_dirichlet(const og_bc* bc, int dim, int N, int i, int j, int k);
double og_dirichlet_value(const og_bc* bc, int dim, int N, int i, int j, int k);
double og_ghost_value(const og_grid* g, const og_bc* bc, const double* u, int i, int j, int k);

double og_restrict_at(const og_grid* g, const og_bc* bc, const double* f, int i, int j, int k, int lam);
void og_restrict_pass(const og_grid* g, const og_bc* bc, const double* in, double* out, int lam);
void og_restriction_into(const og_grid* g, const og_bc* bc, const double* f, int v,
                         double* out, double* scratch, uint64_t* work);
int og_relaxation_interpolation(const og_grid* g, const og_bc* bc, double* u, const double* u_prev,
                                double* du, const double* du_prev, int level, const double* gsrc,
                                const double* sigma_or_null, double a, double safety,
                                int homogeneous, double* diag_out, uint64_t* work);
void og_residual_update(const og_grid* g, const og_bc* bc, double* r, const double* e,
                        const double* sigma_or_null, double a);
double og_apply_operator(const og_grid* g, const og_bc* bc, const double* u,
                         const double* sigma_or_null, double a, int i, int j, int k, int lam);
double og_max_abs(const double* f, uint64_t total);
double og_trapezoid_mean(const og_grid* g, const double* f);
void og_zero_mean_projection(const og_grid* g, double* f);
void og_apply_boundary(const og_grid* g, const og_bc* bc, double* u, int homogeneous);

int og_build_schedule(int n, int n_r, int* kinds, int* levels, int* counts, int cap);
uint64_t og_closed_form_work_units(int n, int n_r);

int og_restrict_sigma_levels(const og_grid* g, const double* sigma, double* levels_out);
int og_single_cycle(const og_grid* g, const og_bc* bc, double* u, double* u_prev, double* du,
                    double* du_prev, const double* source, const double* sigma_levels_or_null,
                    double a, int homogeneous, int n_r, double safety, int cycle_index,
                    double normalization, og_report* rep, uint64_t* work);
int og_solve(const og_grid* g, const og_bc* bc, const double* f, const double* sigma_or_null,
             double a, int n_r, double tol, int max_cycles, double safety, double* u_out,
             og_report* rep);

/* problem builders used to pin the oracle against the reference's measured
 * residual histories (problems.cpp:160-193, 500-521) */
void og_fill_poisson2d(const og_grid* g, double* f);
void og_fill_poisson3d(const og_grid* g, double* f);
void og_fill_sinsin2d(const og_grid* g, double* f);
void og_fill_capacitor_sigma(const og_grid* g, double sign, double* sigma);
void og_lcg_fill(double* f, uint64_t total, uint64_t seed);

/* post-solve fields (problems.cpp:40-97, 327-455).  Vector fields are
 * component-major: comp c at v + c * total.  Points are xyz triples. */
void og_axis_derivative(const og_grid* g, const double* u, int axis, double* out);
void og_gradient(const og_grid* g, const double* u, double* out);            /* dim comps */
void og_curl(const og_grid* g, const double* psi, double* out);             /* 3D, 3 comps */
void og_divergence(const og_grid* g, const double* v, double* out);         /* dim comps in */
int og_deformation_velocity(const og_grid* g, const double* u, const double* f_raw, double raw_integral,
                            double t, double* out);                           /* OG_INVALID on den == 0 */
int og_move_nodes(const og_grid* g, const double* u, const double* f_raw, double raw_integral, double t,
                  int steps, double* pos);                                    /* total xyz triples */
double og_sample_scalar(const og_grid* g, const double* f, const double* p);
void og_sample_vector(const og_grid* g, const double* v, int nv, const double* p, double* out);
/* returns the number of points written (<= max_steps + 1); *stop = 0 max_steps,
 * 1 left_domain, 2 stagnation */
int og_integrate_streamline(const og_grid* g, const double* v, const double* seed, double step, int max_steps,
                            double* pts, int* stop);

#ifdef __cplusplus
}
#endif
#endif
