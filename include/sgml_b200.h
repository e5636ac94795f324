/*
 * sgml_b200.h — C ABI of the B200-native SGML solve path.
 *
 * This is the drop-in boundary for the reference's solve path
 * (/root/reference/proj/core).  Every entry point names the reference
 * interface it replaces (file:line under proj/core/include/sgml or src).
 * Plain pointers and sizes only; no C++ or torch types cross this line.
 * The C++ mirror of the reference API (include/sgml/*.hpp, namespace sgml)
 * and the Python package (paper_1703_07206_b200) are thin layers over it.
 *
 * Memory model: an sgml_field is a device-resident fp64 field of N^dim
 * nodes in the reference's x-fastest order (grid.hpp:78-119).  Host arrays
 * cross the boundary only through sgml_field_upload/download and the
 * host-buffer entry point sgml_solve.
 *
 * Errors: every function returns an sgml_status.  SGML_EINVAL maps to the
 * reference's std::invalid_argument, SGML_EBADSTEP / SGML_ENONFINITE to
 * sgml::kernel_error (kernels.hpp:38-40), SGML_ECUDA / SGML_ENCCL to
 * std::runtime_error.  sgml_last_error() returns the message of the last
 * failure on the calling thread.
 *
 * Numerics: all kernels are compiled without FMA contraction and follow the
 * reference's operation order, so results are bit-identical to the
 * reference CPU path up to the sign of exact zeros.
 */
#ifndef SGML_B200_H
#define SGML_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SGML_OK = 0,
    SGML_EINVAL = 1,     /* std::invalid_argument */
    SGML_EBADSTEP = 2,   /* kernel_error: non-positive pseudo-time step */
    SGML_ENONFINITE = 3, /* kernel_error: non-finite value produced */
    SGML_ECUDA = 4,      /* std::runtime_error (CUDA) */
    SGML_ENCCL = 5,      /* std::runtime_error (NCCL) */
    SGML_ELOGIC = 6,     /* std::logic_error / std::out_of_range */
    SGML_EIO = 7         /* io_error: a file cannot be opened / written */
} sgml_status;

typedef struct sgml_ctx sgml_ctx;       /* one device + one stream + buffer pool */
typedef struct sgml_field sgml_field;   /* device-resident fp64 field */
typedef struct sgml_solver sgml_solver; /* preallocated solve engine */

/* grid.hpp:31-39 (make_grid, grid.cpp:10-23) */
typedef struct {
    int dim;
    int n;
    int N;
    int pad_;
    double h;
    uint64_t total;
} sgml_grid;

/* grid.hpp:125-157: faces axis*2+side; kind 0 = dirichlet, 1 = neumann */
typedef struct {
    int kind[6];
    double value[6];
} sgml_bc;

/* cycle.hpp:66-71 */
typedef struct {
    int n_r;
    int max_cycles;
    double tol;
    double safety;
} sgml_solver_cfg;

/* Engine options that the reference has no counterpart for (kept out of
 * sgml_solver_cfg so the reference SolverConfig maps 1:1). */
typedef struct {
    int engine;     /* 0 = level-compact B200 engine (default), 1 = literal full-grid passes */
    int use_graph;  /* 0 / 1: single-GPU compact solves replay each cycle from a CUDA graph
                       (default); -1: launch eagerly */
    int timing;     /* record per-kernel-class device time in the report */
    int timing_classes; /* 0: every class; else a mask of (1 << SGML_CLASS_*) to time */
    int stencil;    /* SGML_STENCIL_RADIAL (0, the reference's 9/27-point form) or
                       SGML_STENCIL_COMPACT (1, 5/7-point, no
                       reference counterpart, parity unpinned) */
    int small_levels; /* 0 (default): a visit of a small level array (<= 6144 relaxed
                       nodes) runs all its passes in one CTA; -1: one TMA launch per
                       pass on every level (same bits either way) */
    int cluster_levels; /* 0 (default): operations on level arrays of <= 5000 nodes (3D
                       <= 17^3) and on 2D level arrays of <= 129^2 nodes run as batches
                       in one thread-block cluster launch each (single GPU);
                       -1: one kernel per operation (same bits either way) */
    int replicate_n;  /* z-slab solves: levels whose arrays hold at most this many nodes
                       per axis are replicated on every rank instead of exchanging
                       halos (0: SGML_REPLICATE_N = 65; levels also replicate once a
                       rank would hold fewer than 2 planes) */
} sgml_solver_opts;

enum { SGML_STENCIL_RADIAL = 0, SGML_STENCIL_COMPACT = 1 };

/* cycle.hpp:81-89 */
typedef struct {
    int cycle;
    int has_l1;
    uint64_t work_units;
    double residual;
    double diag_min;
    double l1_error;
} sgml_cycle_record;

/* cycle.hpp:74-79 */
typedef struct {
    int cycle;
    int pass;
    int level;
    int pad_;
    double value;
} sgml_diag_sample;

/* Per-cycle hook (the l1_error column, cycle.cpp:222): called after u_total
 * is accumulated; return 1 and set *l1 to record a value. */
typedef int (*sgml_cycle_hook)(void* user, int cycle, const sgml_field* u_total, double* l1);

/* cycle.hpp:91-99 with caller-owned arrays.  n_rows / n_trace count every
 * record produced even past the capacities. */
typedef struct {
    sgml_cycle_record* rows;
    int64_t rows_cap;
    int64_t n_rows;
    sgml_diag_sample* trace;
    int64_t trace_cap;
    int64_t n_trace;
    int converged;
    int nan_detected;
    int stagnated;
    int pad_;
    double normalization;
    uint64_t node_updates;
    sgml_cycle_hook hook;
    void* hook_user;
    /* device timing of the last solve (CUDA events on the ctx stream) */
    double device_ms;
    uint64_t kernel_launches;
    /* per kernel class (SGML_CLASS_*), filled when sgml_solver_opts.timing:
     * summed event time and launch count inside the solve */
    double class_ms[8];
    uint64_t class_launches[8];
} sgml_report;

/* kernel classes of sgml_report.class_ms */
enum {
    SGML_CLASS_RELAX0 = 0,      /* level-0 (full-grid) relaxation pass */
    SGML_CLASS_RELAX_COARSE = 1,/* level >= 1 compact relaxation pass */
    SGML_CLASS_MATERIALIZE = 2, /* lazy interpolation / next-level input */
    SGML_CLASS_PYRAMID = 3,     /* restriction pyramid step */
    SGML_CLASS_RESIDUAL = 4,    /* fused residual recurrence */
    SGML_CLASS_LITERAL = 5,     /* literal-engine restrict / relax passes */
    SGML_CLASS_OTHER = 6        /* reductions, projections, fills */
};

/* pinned host memory for end-to-end transfers (cudaMallocHost) */
int sgml_host_alloc(uint64_t bytes, void** out);
int sgml_host_free(void* p);

/* ---- library / context ------------------------------------------------ */
const char* sgml_last_error(void);
const char* sgml_version(void);
int sgml_device_count(int* count);
int sgml_ctx_create(int device, sgml_ctx** out);
int sgml_ctx_destroy(sgml_ctx* ctx);
int sgml_ctx_synchronize(sgml_ctx* ctx);
/* the stream every kernel of this ctx is launched on (cudaStream_t) */
void* sgml_ctx_stream(sgml_ctx* ctx);

/* ---- multi-GPU clique (z-slab solves) ---------------------
 * One context per rank.  A 3D compact-engine solve (sgml_solve, sgml_solver_*)
 * on a context that joined a clique of nranks > 1 runs the z-slab
 * decomposition: every rank passes the same full problem and receives the
 * full solution; the report is identical on all ranks and bit-identical to
 * the single-GPU solve (every reduction is a max).  nranks must be a power
 * of two with at least 2 level-0 planes per rank. */
typedef struct sgml_group sgml_group;
/* NCCL, one process per GPU: rank 0 creates the id, every rank joins with it
 * (libnccl.so.2 is opened at run time) */
int sgml_nccl_unique_id(unsigned char id[128]);
int sgml_ctx_join_nccl(sgml_ctx* ctx, int nranks, int rank, const unsigned char id[128]);
/* in-process ranks (one host thread per rank, devices may be shared): the
 * parity tests of the decomposition on one GPU */
int sgml_local_group_create(int nranks, sgml_group** out);
int sgml_local_group_destroy(sgml_group* g);
int sgml_ctx_join_local(sgml_ctx* ctx, sgml_group* g, int rank);
int sgml_ctx_clique(sgml_ctx* ctx, int* nranks, int* rank);
/* the z-slab plan (host only): levels < *vrep are z-slabs and rank `rank`
 * owns level-v planes [z0 >> v, (z0 >> v) + nz_v) with nz_v = (nz - last) >> v
 * + last, last = (rank == nranks - 1); level-0 planes [*z0, *z0 + *nz) */
int sgml_slab_plan(int n, int nranks, int rank, int* vrep, int* z0, int* nz);
/* the same with an explicit replicate_n (sgml_solver_opts; 0: the default) */
int sgml_slab_plan_ex(int n, int nranks, int rank, int replicate_n, int* vrep, int* z0, int* nz);
#define SGML_REPLICATE_N 65

/* ---- grid / schedule (host logic; no device needed) --------------------- */
int sgml_make_grid(int dim, int n, sgml_grid* out);                      /* grid.cpp:10-23 */
/* cycle.cpp:28-45: kinds 0 = restrict_source, 1 = relax; returns the step
 * count via *count (entries past cap are not written) */
int sgml_build_schedule(int n, int n_r, int* kinds, int* levels, int* counts, int cap, int* count);
uint64_t sgml_closed_form_work_units(int n, int n_r);                    /* cycle.cpp:47-59 */

/* ---- fields (grid.hpp:78-119) ------------------------------------------ */
int sgml_field_create(sgml_ctx* ctx, int dim, int n, sgml_field** out);
int sgml_field_destroy(sgml_field* f);
int sgml_field_upload(sgml_field* f, const double* host);
int sgml_field_download(const sgml_field* f, double* host);
int sgml_field_copy(sgml_field* dst, const sgml_field* src);
int sgml_field_fill(sgml_field* f, double value);
int sgml_field_grid(const sgml_field* f, sgml_grid* out);
void* sgml_field_device_ptr(sgml_field* f);

/* ---- kernels (kernels.hpp) ---------------------------------------------- */
/* kernels.hpp:79-87 / kernels.cpp:305-325: v literal passes, out != scratch */
int sgml_restriction_into(const sgml_field* f, int v, const sgml_bc* bc, sgml_field* out,
                          sgml_field* scratch, uint64_t* work);
/* kernels.hpp:89-104 / kernels.cpp:334-349: one pass at `level`, reads
 * u_prev/du_prev, writes u/du; diag_out = unnormalised diagnostic max */
int sgml_relaxation_interpolation(sgml_field* u, const sgml_field* u_prev, sgml_field* du,
                                  const sgml_field* du_prev, int level, const sgml_field* g,
                                  const sgml_field* sigma_or_null, double a, double safety,
                                  const sgml_bc* bc, int homogeneous, double* diag_out,
                                  uint64_t* work);
/* kernels.hpp:106-117 / kernels.cpp:351-358 */
int sgml_residual_update(sgml_field* r, const sgml_field* e, const sgml_field* sigma_or_null,
                         double a, const sgml_bc* bc);
int sgml_max_abs(const sgml_field* f, double* out);                      /* kernels.cpp:407-415 */
int sgml_trapezoid_mean(const sgml_field* f, double* out);               /* kernels.cpp:367-386 */
int sgml_zero_mean_projection(sgml_field* f);                            /* kernels.cpp:388-395 */
int sgml_apply_boundary(sgml_field* u, const sgml_bc* bc, int homogeneous); /* kernels.cpp:397-405 */
/* cycle.cpp:117-133: levels[v] <- sigma restricted to level v (even ghosts),
 * SGML_EINVAL if any level is not positive; levels holds n fields */
int sgml_restrict_sigma_levels(const sgml_field* sigma, sgml_field* const* levels);
/* cycle.cpp:135-138 */
int sgml_pure_neumann_pin(sgml_field* u);

/* ---- driver (cycle.hpp) ------------------------------------------------- */
/* cycle.hpp:121-136 / cycle.cpp:76-111: one cycle from the zero state of
 * `state_u`; sigma_levels is NULL or n fields; trace samples appended to
 * rep (rows untouched); *work advanced by the schedule's units.  On return
 * state_u holds the cycle's correction (SolveState::u). */
int sgml_single_cycle(sgml_ctx* ctx, sgml_field* state_u, const sgml_field* source,
                      sgml_field* const* sigma_levels, double a, const sgml_bc* bc,
                      int homogeneous, int n_r, double safety, int cycle_index,
                      double normalization, const sgml_solver_opts* opts, sgml_report* rep,
                      uint64_t* work);

/* single_cycle with the reference's full SolveState semantics
 * (cycle.cpp:76-111): the state's four buffers (u, u_prev, du, du_prev) and
 * *level are read and written exactly as the reference does (the cycle
 * starts from the caller's state.u; du / du_prev reset at every level change;
 * each pass swaps the buffers, which here swaps the fields' device storage),
 * an arbitrary schedule (nsteps steps: kind 0 restrict_source / 1 relax,
 * level, count) and caller-supplied sigma levels (sigma_levels[v] for every
 * level a step relaxes, or NULL for sigma == 1).  Runs the literal full-grid
 * kernels pass by pass; a failing pass stops the cycle there, with the trace
 * samples and work units of the steps before it recorded and the state as
 * the reference leaves it, and returns SGML_EBADSTEP / SGML_ENONFINITE. */
int sgml_single_cycle_state(sgml_ctx* ctx, sgml_field* u, sgml_field* u_prev, sgml_field* du,
                            sgml_field* du_prev, int* level, const sgml_field* source,
                            sgml_field* const* sigma_levels, double a, const sgml_bc* bc, int homogeneous,
                            const int* step_kinds, const int* step_levels, const int* step_counts, int nsteps,
                            double safety, int cycle_index, double normalization, sgml_report* rep,
                            uint64_t* work);

/* Preallocated engine for repeated solves on one grid/problem shape. */
int sgml_solver_create(sgml_ctx* ctx, int dim, int n, const sgml_bc* bc, double a,
                       const sgml_field* sigma_or_null, const sgml_solver_cfg* cfg,
                       const sgml_solver_opts* opts, sgml_solver** out);
int sgml_solver_destroy(sgml_solver* s);
/* cycle.cpp:140-247 with device-resident f and u_out */
int sgml_solver_run(sgml_solver* s, const sgml_field* f, sgml_field* u_out, sgml_report* rep);
/* bytes of device memory the engine holds */
int sgml_solver_footprint(const sgml_solver* s, uint64_t* bytes);

/* cycle.hpp:147 / cycle.cpp:140-247 end to end: host f (and sigma), host
 * u_out; uploads, solves on `ctx`'s device, downloads. */
int sgml_solve(sgml_ctx* ctx, int dim, int n, const sgml_bc* bc, const double* f_host,
               const double* sigma_host_or_null, double a, const sgml_solver_cfg* cfg,
               const sgml_solver_opts* opts_or_null, double* u_host_out, sgml_report* rep);
/* `count` solves of one problem shape (one sigma, different sources) end to
 * end, pipelined: solve k+1's source moves in and solve k-1's solution moves
 * out on a copy stream while solve k runs.  f_hosts[k] / u_hosts[k] host
 * buffers (pinned for full overlap), reps[k] one report each.  Results are
 * those of count sgml_solve calls. */
int sgml_solve_many(sgml_ctx* ctx, int dim, int n, const sgml_bc* bc, int count, const double* const* f_hosts,
                    const double* sigma_host_or_null, double a, const sgml_solver_cfg* cfg,
                    const sgml_solver_opts* opts_or_null, double* const* u_hosts, sgml_report* reps);

/* ---- post-solve fields (problems.hpp:100-148) ----------
 * Dense device fields in, dense device fields out; the reference's bits.
 * Vector fields are arrays of dim component fields (3 for curl). */
/* axis_derivative (problems.cpp:74-97): central inside, one-sided 3-point on faces */
int sgml_axis_derivative(const sgml_field* u, int axis, sgml_field* out);
/* gradient (problems.cpp:391-396): out[c] for c < dim */
int sgml_gradient(const sgml_field* u, sgml_field* const* out);
/* curl (problems.cpp:376-389); SGML_EINVAL unless 3D */
int sgml_curl(const sgml_field* const* psi, sgml_field* const* out);
/* divergence (problems.cpp:398-405): v[c] for c < dim */
int sgml_divergence(const sgml_field* const* v, sgml_field* out);
/* deformation_velocity (problems.cpp:327-341): -grad u / (t f_raw + raw_integral);
 * SGML_EINVAL on a zero denominator */
int sgml_deformation_velocity(const sgml_field* u, const sgml_field* f_raw, double raw_integral, double t,
                              sgml_field* const* out);
/* move_nodes (problems.cpp:343-372): node positions after `steps` Euler steps,
 * as coordinate fields pos[0..dim-1] (pos[2] optional in 2D: zeros) */
int sgml_move_nodes(const sgml_field* u, const sgml_field* f_raw, double raw_integral, double t, int steps,
                    sgml_field* const* pos);
/* sample_vector (problems.cpp:407-413) of nv component fields at host points
 * (3 doubles each) into host out (3 doubles each, unused components 0) */
int sgml_sample_vector(const sgml_field* const* v, int nv, const double* points, int count, double* out);
/* integrate_streamline (problems.cpp:415-455) for nseeds host seeds: points
 * [seed][max_steps + 1][3], counts[seed] points used, stops[seed] =
 * 0 max_steps, 1 left_domain, 2 stagnation (StreamlineStop order) */
int sgml_integrate_streamlines(const sgml_field* const* v, const double* seeds, int nseeds, double step,
                               int max_steps, double* points, int* counts, int* stops);

/* ---- problem builders --------------------------------
 * The reference's sources / coefficients assembled on the device, bit for bit
 * (the libm calls run on the host over their few distinct arguments; curve
 * deposits are summed on the host in the reference's sample order and
 * scattered).  Fields must be allocated on the target grid. */
int sgml_build_poisson2d_source(sgml_field* f);              /* problems.cpp:160-176 */
int sgml_build_poisson3d_source(sgml_field* f);              /* problems.cpp:178-193 */
int sgml_build_sinsin2d_source(sgml_field* f);               /* BASELINE configs[0]: -2 pi^2 sin sin */
int sgml_build_capacitor_sigma(sgml_field* sigma, int high); /* problems.cpp:500-521 (high: -, low: +) */
/* problems.cpp:374-398: the three psi sources -omega_c of trifoil_problem(n, r) */
int sgml_build_trifoil_sources(sgml_field* const* f3, double r);
/* problems.cpp:302-325 for a closed curve (xyz triples; z != 0 anywhere makes
 * it 3D): f_raw, the zero-mean source f and the raw trapezoid integral */
int sgml_build_deformation_sources(const double* points, int npts, sgml_field* f, sgml_field* f_raw,
                                   double* raw_integral);

/* problems.cpp:302-325 for any curve (closed flag; with_payload: the curve
 * carries a payload, so resampling also forms unit tangents and rejects
 * degenerate ones, as the reference does) */
int sgml_build_deformation_problem(const double* points, int npts, int closed, int with_payload, sgml_field* f,
                                   sgml_field* f_raw, double* raw_integral);

/* ---- curves (problems.cpp:217-300) -------------------------------------------
 * Host curve work (a few thousand samples) with the reference's arithmetic.
 * Points / payloads are xyz triples.  resample_curve writes min(count, cap)
 * samples and sets *count to the full count (call again with a larger cap
 * when *count > cap); out_payload may be NULL unless with_payload. */
int sgml_resample_curve(const double* points, int npts, int closed, int with_payload, double h, double* out_points,
                        double* out_payload, int cap, int* count);
/* deposit_delta: strength * arc element per sample, hat weights / h^dim,
 * into the device field f (zeroed first) */
int sgml_deposit_delta(const double* points, int npts, int closed, double strength, sgml_field* f);
/* deposit_delta_vector: payload * arc element into the 3 component fields */
int sgml_deposit_delta_vector(const double* points, const double* payload, int npts, int closed,
                              sgml_field* const* f3);
/* trifoil_problem's curve (problems.cpp:374-398): the 512-sample overhand
 * knot of scale r, checked inside the unit cube, resampled at spacing h with
 * unit tangents (same count / cap protocol as sgml_resample_curve) */
int sgml_trifoil_curve(double r, double h, double* out_points, double* out_payload, int cap, int* count);

/* ---- output (io.cpp:14-64) ------------------------------
 * The reference's legacy ASCII VTK files ("%.17g"), byte for byte, streamed
 * from the device in chunks and formatted on all host threads. */
int sgml_write_field_vtk(const sgml_field* f, const char* path, const char* name);
int sgml_write_vector_vtk(const sgml_field* const* v3, const char* path, const char* name); /* v3[2] may be NULL */
/* the same files from host arrays: ncomp 1 (SCALARS) or 3 (VECTORS; comps[2] may be NULL) */
int sgml_write_vtk_host(const double* const* comps, int ncomp, const sgml_grid* g, const char* path,
                        const char* name);

#ifdef __cplusplus
}
#endif
#endif /* SGML_B200_H */
