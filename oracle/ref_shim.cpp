// ref_shim.cpp — extern "C" view of the UNMODIFIED reference core.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with /root/reference/proj/core/src/{grid,stencil,kernels,cycle,problems,io}.cpp
// (in place, never copied) into oracle/_ref/libsgml_ref.so with
// -Dsgml=sgml_ref, so the reference's namespace cannot collide with
// anything else loaded in the process.  The functions mirror
// oracle/sgml_oracle.h (prefix ref_ instead of og_) so tests can run the
// restatement and the reference side by side on identical inputs.
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>

#include "sgml/cycle.hpp"
#include "sgml/kernels.hpp"
#include "sgml/io.hpp"
#include "sgml/problems.hpp"

extern "C" {
#include "sgml_oracle.h"
}

namespace R = sgml;  // expands to sgml_ref under -Dsgml=sgml_ref

// ---- zero-padded allocations for the reference's code in this library -----
// The reference's interpolation reads zero-weight corners past the end of
// du_prev on non-Dirichlet high faces (kernels.cpp:140-174):
// up to half an array past its end.  What those bytes decode to is heap
// layout (undefined behaviour); Inf/NaN there turns 0 * x non-finite and
// the reference reports nan_detected at random.  Every allocation the
// reference's code makes in this library is therefore followed by as many
// zero bytes as it holds (calloc; large blocks are fresh zero pages that are
// never touched), so the past-the-end reads see 0 -- the outcome the C
// restatement and the B200 engine implement.  The library is linked with
// -Bsymbolic-functions and loaded RTLD_LOCAL, so only this library's calls
// bind here; calloc/free stay compatible with the process's own
// operator new/delete.
#define SGML_REF_HIDDEN
SGML_REF_HIDDEN void* operator new(std::size_t n) {
    void* p = std::calloc(1, 2 * n + 64);
    if (!p) throw std::bad_alloc();
    return p;
}
SGML_REF_HIDDEN void* operator new[](std::size_t n) { return ::operator new(n); }
SGML_REF_HIDDEN void operator delete(void* p) noexcept { std::free(p); }
SGML_REF_HIDDEN void operator delete[](void* p) noexcept { std::free(p); }
SGML_REF_HIDDEN void operator delete(void* p, std::size_t) noexcept { std::free(p); }
SGML_REF_HIDDEN void operator delete[](void* p, std::size_t) noexcept { std::free(p); }

namespace {

R::BoundarySpec to_bc(const og_bc* bc) {
    R::BoundarySpec b;
    for (int f = 0; f < 6; ++f)
        b.faces[f] = {bc->kind[f] == 1 ? R::BcKind::neumann : R::BcKind::dirichlet, bc->value[f]};
    return b;
}

R::Field to_field(const R::Grid& g, const double* p) {
    R::Field f(g);
    std::memcpy(f.data(), p, g.total * sizeof(double));
    return f;
}

void from_field(const R::Field& f, double* p) { std::memcpy(p, f.data(), f.size() * sizeof(double)); }

R::Grid grid_of(const og_grid* g) { return R::make_grid(g->dim, g->n); }

}  // namespace

extern "C" {

void ref_restriction_into(const og_grid* g, const og_bc* bc, const double* f, int v, double* out,
                          uint64_t* work) {
    const R::Grid gr = grid_of(g);
    R::Field fo(gr), sc(gr);
    std::uint64_t w = work ? *work : 0;
    R::restriction_into(to_field(gr, f), v, to_bc(bc), fo, sc, &w);
    if (work) *work = w;
    from_field(fo, out);
}

int ref_relaxation_interpolation(const og_grid* g, const og_bc* bc, double* u, const double* u_prev,
                                 double* du, const double* du_prev, int level, const double* gsrc,
                                 const double* sigma, double a, double safety, int homogeneous,
                                 double* diag_out, uint64_t* work) {
    const R::Grid gr = grid_of(g);
    R::SolveState st(gr);
    st.level = level;
    std::memcpy(st.u_prev.data(), u_prev, gr.total * sizeof(double));
    std::memcpy(st.du_prev.data(), du_prev, gr.total * sizeof(double));
    R::Field gf = to_field(gr, gsrc);
    R::Field sf = sigma ? to_field(gr, sigma) : R::Field();
    std::uint64_t w = work ? *work : 0;
    int status = 0;
    try {
        *diag_out = R::relaxation_interpolation(st, gf, sigma ? &sf : nullptr, a, safety,
                                                to_bc(bc), homogeneous != 0, &w);
    } catch (const R::kernel_error& e) {
        status = std::strstr(e.what(), "step") ? OG_BADSTEP : OG_NONFINITE;
    }
    if (work) *work = w;
    from_field(st.u, u);
    from_field(st.du, du);
    return status;
}

void ref_residual_update(const og_grid* g, const og_bc* bc, double* r, const double* e,
                         const double* sigma, double a) {
    const R::Grid gr = grid_of(g);
    R::Field rf = to_field(gr, r);
    R::Field sf = sigma ? to_field(gr, sigma) : R::Field();
    R::residual_update(rf, to_field(gr, e), R::OperatorCoefficients{sigma ? &sf : nullptr, a},
                       to_bc(bc));
    from_field(rf, r);
}

double ref_max_abs(const og_grid* g, const double* f) {
    return R::max_abs(to_field(grid_of(g), f));
}

double ref_trapezoid_mean(const og_grid* g, const double* f) {
    return R::trapezoid_mean(to_field(grid_of(g), f));
}

uint64_t ref_closed_form_work_units(int n, int n_r) { return R::closed_form_work_units(n, n_r); }

int ref_single_cycle(const og_grid* g, const og_bc* bc, double* u_out, const double* source,
                     const double* sigma_levels, double a, int homogeneous, int n_r, double safety,
                     int cycle_index, double normalization, og_report* rep, uint64_t* work) {
    const R::Grid gr = grid_of(g);
    R::SolveState st(gr);
    std::vector<R::Field> levels;
    if (sigma_levels)
        for (int v = 0; v < gr.n; ++v) levels.push_back(to_field(gr, sigma_levels + (size_t)v * gr.total));
    R::SolveReport report;
    std::uint64_t w = work ? *work : 0;
    int status = 0;
    try {
        R::single_cycle(st, to_field(gr, source), levels, a, to_bc(bc), homogeneous != 0,
                        R::build_schedule(gr.n, n_r), safety, cycle_index, normalization, report, w);
    } catch (const R::kernel_error&) {
        status = OG_NONFINITE;
    }
    if (work) *work = w;
    from_field(st.u, u_out);
    rep->n_trace = 0;
    for (const auto& s : report.trace) {
        if (rep->n_trace < rep->trace_cap)
            rep->trace[rep->n_trace] = og_sample{s.cycle, s.pass, s.level, 0, s.value};
        rep->n_trace++;
    }
    return status;
}

// single_cycle with an arbitrary state, schedule and sigma levels (the
// reference's full SolveState semantics; cycle.cpp:76-111)
int ref_single_cycle_state(const og_grid* g, const og_bc* bc, double* u, double* u_prev, double* du,
                           double* du_prev, int* level, const double* source, const double* sigma_levels,
                           int nlevels, double a, int homogeneous, const int* kinds, const int* levels,
                           const int* counts, int nsteps, double safety, int cycle_index, double normalization,
                           og_report* rep, uint64_t* work) {
    const R::Grid gr = grid_of(g);
    R::SolveState st(gr);
    std::memcpy(st.u.data(), u, gr.total * sizeof(double));
    std::memcpy(st.u_prev.data(), u_prev, gr.total * sizeof(double));
    std::memcpy(st.du.data(), du, gr.total * sizeof(double));
    std::memcpy(st.du_prev.data(), du_prev, gr.total * sizeof(double));
    st.level = *level;
    std::vector<R::Field> lv;
    for (int v = 0; sigma_levels && v < nlevels; ++v) lv.push_back(to_field(gr, sigma_levels + (size_t)v * gr.total));
    R::CycleSchedule sch;
    sch.n = gr.n;
    for (int i = 0; i < nsteps; ++i)
        sch.steps.push_back({kinds[i] == 0 ? R::ScheduleStep::Kind::restrict_source : R::ScheduleStep::Kind::relax,
                             levels[i], counts[i]});
    R::SolveReport report;
    std::uint64_t w = *work;
    int status = 0;
    try {
        R::single_cycle(st, to_field(gr, source), lv, a, to_bc(bc), homogeneous != 0, sch, safety, cycle_index,
                        normalization, report, w);
    } catch (const R::kernel_error& e) {
        status = std::strstr(e.what(), "step") ? OG_BADSTEP : OG_NONFINITE;
    }
    *work = w;
    from_field(st.u, u);
    from_field(st.u_prev, u_prev);
    from_field(st.du, du);
    from_field(st.du_prev, du_prev);
    *level = st.level;
    rep->n_trace = 0;
    for (const auto& smp : report.trace) {
        if (rep->n_trace < rep->trace_cap)
            rep->trace[rep->n_trace] = og_sample{smp.cycle, smp.pass, smp.level, 0, smp.value};
        rep->n_trace++;
    }
    return status;
}

int ref_solve(const og_grid* g, const og_bc* bc, const double* f, const double* sigma, double a,
              int n_r, double tol, int max_cycles, double safety, double* u_out, og_report* rep) {
    const R::Grid gr = grid_of(g);
    R::ProblemSpec prob;
    prob.grid = gr;
    prob.f = to_field(gr, f);
    if (sigma) prob.sigma = to_field(gr, sigma);
    prob.a = a;
    prob.bc = to_bc(bc);
    R::SolverConfig cfg;
    cfg.n_r = n_r;
    cfg.tol = tol;
    cfg.max_cycles = max_cycles;
    cfg.safety = safety;
    R::SolveResult res;
    try {
        res = R::solve(prob, cfg);
    } catch (const std::invalid_argument&) {
        return OG_INVALID;
    }
    from_field(res.u, u_out);
    const R::SolveReport& r = res.report;
    rep->n_rows = 0;
    for (const auto& row : r.rows) {
        if (rep->n_rows < rep->rows_cap)
            rep->rows[rep->n_rows] = og_row{row.cycle, 0, row.work_units, row.residual, row.diag_min};
        rep->n_rows++;
    }
    rep->n_trace = 0;
    for (const auto& s : r.trace) {
        if (rep->n_trace < rep->trace_cap)
            rep->trace[rep->n_trace] = og_sample{s.cycle, s.pass, s.level, 0, s.value};
        rep->n_trace++;
    }
    rep->converged = r.converged;
    rep->nan_detected = r.nan_detected;
    rep->stagnated = r.stagnated;
    rep->normalization = r.normalization;
    rep->node_updates = r.node_updates;
    return 0;
}

// ---- timing sessions (bench.py --impl reference / cpu_baseline) ----------
// The reference's solve (cycle.cpp:140-247) driven one schedule step at a
// time through its own public functions, so a bounded part of a large solve
// can be timed: begin_cycle = the per-cycle set-up of solve + single_cycle
// (cycle.cpp:179-180, 83-84), step = one ScheduleStep exactly as
// single_cycle runs it (cycle.cpp:88-109: restriction_into, or reset_level
// on a level change + count x (swap_buffers, relaxation_interpolation)),
// recurrence = the rest of solve's cycle (u_total += e, residual_update,
// max_abs; cycle.cpp:191-198).
struct ref_session {
    R::Grid grid;
    R::BoundarySpec bc;
    R::Field r, u_total;
    R::SolveState state;
    R::Field g, scratch;
    R::CycleSchedule schedule;
    std::vector<R::Field> sigma_levels;
    R::Field sigma;
    double a = 0.0, safety = 0.9;
    int current_level = -1;
    std::uint64_t work = 0;
    bool homogeneous = false;
    explicit ref_session(const R::Grid& gr) : grid(gr), r(gr), u_total(gr), state(gr) {}
};

void* ref_session_create(const og_grid* g, const og_bc* bc, const double* f, const double* sigma, double a,
                         int n_r, double safety) {
    const R::Grid gr = grid_of(g);
    auto* s = new ref_session(gr);
    s->bc = to_bc(bc);
    s->r = to_field(gr, f);
    if (sigma) {
        s->sigma = to_field(gr, sigma);
        s->sigma_levels = R::restrict_sigma_levels(s->sigma, gr.n);
    }
    s->a = a;
    s->safety = safety;
    s->schedule = R::build_schedule(gr.n, n_r);
    return s;
}

void ref_session_destroy(void* p) { delete static_cast<ref_session*>(p); }

int ref_session_nsteps(void* p) { return (int)static_cast<ref_session*>(p)->schedule.steps.size(); }

void ref_session_begin_cycle(void* p, int homogeneous) {
    auto* s = static_cast<ref_session*>(p);
    s->state.u.fill(0.0);
    s->state.u_prev.fill(0.0);
    s->g = R::Field(s->grid);
    s->scratch = R::Field(s->grid);
    s->current_level = -1;
    s->homogeneous = homogeneous != 0;
}

// returns 0, or 1 when a pass throws kernel_error
int ref_session_step(void* p, int index, double* diag_max) {
    auto* s = static_cast<ref_session*>(p);
    const R::ScheduleStep& st = s->schedule.steps.at((size_t)index);
    try {
        if (st.kind == R::ScheduleStep::Kind::restrict_source) {
            R::restriction_into(s->r, st.level, s->bc, s->g, s->scratch, &s->work);
        } else {
            if (st.level != s->current_level) {
                s->state.reset_level(st.level);
                s->current_level = st.level;
            }
            const R::Field* sig = s->sigma_levels.empty() ? nullptr : &s->sigma_levels[(size_t)st.level];
            double dmax = 0.0;
            for (int c = 0; c < st.count; ++c) {
                s->state.swap_buffers();
                const double d = R::relaxation_interpolation(s->state, s->g, sig, s->a, s->safety, s->bc,
                                                             s->homogeneous, &s->work);
                dmax = d > dmax ? d : dmax;
            }
            if (diag_max) *diag_max = dmax;
        }
    } catch (const R::kernel_error&) {
        return 1;
    }
    return 0;
}

double ref_session_recurrence(void* p) {
    auto* s = static_cast<ref_session*>(p);
    const R::Field& e = s->state.u;
    for (std::size_t q = 0; q < s->u_total.size(); ++q) s->u_total[q] += e[q];
    R::residual_update(s->r, e, R::OperatorCoefficients{s->sigma.size() ? &s->sigma : nullptr, s->a}, s->bc);
    return R::max_abs(s->r);
}

// Reference problem builders: the exact source/coefficient bits the
// reference solves (used for golden vectors and the cpu baseline).
int ref_problem_fields(const char* name, int n, double* f_out, double* sigma_out, int* bc_kind,
                       double* bc_value, double* a_out) {
    R::ProblemSpec p;
    const std::string s(name);
    if (s == "poisson2d") p = R::poisson2d_problem(n);
    else if (s == "poisson3d") p = R::poisson3d_problem(n);
    else if (s == "capacitor_high") p = R::capacitor_problem(n, "high");
    else if (s == "capacitor_low") p = R::capacitor_problem(n, "low");
    else if (s == "trifoil_x" || s == "trifoil_y" || s == "trifoil_z") {
        const R::TrifoilSetup t = R::trifoil_problem(n, 0.14);
        p = t.psi[s == "trifoil_x" ? 0 : s == "trifoil_y" ? 1 : 2];
    } else if (s == "deformation_circle") {
        // the CLI smoke circle: 32 points, centre (1/2, 1/2), radius 1/4, closed
        R::Curve c;
        c.closed = true;
        for (int q = 0; q < 32; ++q) {
            const double t = 2.0 * 3.14159265358979323846 * q / 32.0;
            c.points.push_back({0.5 + 0.25 * std::cos(t), 0.5 + 0.25 * std::sin(t), 0.0});
        }
        p = R::deformation_problem(c, 0.1, n).problem;
    } else {
        return 1;
    }
    if (f_out) std::memcpy(f_out, p.f.data(), p.f.size() * sizeof(double));
    if (sigma_out && p.sigma.size()) std::memcpy(sigma_out, p.sigma.data(), p.sigma.size() * sizeof(double));
    for (int f = 0; f < 6; ++f) {
        bc_kind[f] = p.bc.faces[f].kind == R::BcKind::neumann ? 1 : 0;
        bc_value[f] = p.bc.faces[f].value;
    }
    *a_out = p.a;
    return p.sigma.size() ? 3 : 2;
}

// ---- post-solve fields (problems.hpp:100-148), component-major vectors ----

namespace {
R::VectorField to_vector(const R::Grid& g, const double* v, int nc) {
    R::VectorField f(g);
    for (int c = 0; c < nc; ++c) std::memcpy(f.comp[c].data(), v + (size_t)c * g.total, g.total * sizeof(double));
    return f;
}
void from_vector(const R::VectorField& f, int nc, double* out) {
    for (int c = 0; c < nc; ++c) std::memcpy(out + (size_t)c * f.comp[c].size(), f.comp[c].data(),
                                             f.comp[c].size() * sizeof(double));
}
}  // namespace

void ref_gradient(const og_grid* g, const double* u, double* out) {
    const R::Grid gr = grid_of(g);
    from_vector(R::gradient(to_field(gr, u)), g->dim, out);
}

void ref_curl(const og_grid* g, const double* psi, double* out) {
    const R::Grid gr = grid_of(g);
    from_vector(R::curl(to_vector(gr, psi, 3)), 3, out);
}

void ref_divergence(const og_grid* g, const double* v, double* out) {
    const R::Grid gr = grid_of(g);
    from_field(R::divergence(to_vector(gr, v, g->dim)), out);
}

int ref_deformation_velocity(const og_grid* g, const double* u, const double* f_raw, double raw_integral,
                             double t, double* out) {
    const R::Grid gr = grid_of(g);
    try {
        from_vector(R::deformation_velocity(to_field(gr, u), to_field(gr, f_raw), raw_integral, t), g->dim, out);
    } catch (const std::invalid_argument&) {
        return 1;
    }
    return 0;
}

int ref_move_nodes(const og_grid* g, const double* u, const double* f_raw, double raw_integral, double t,
                   int steps, double* pos) {
    const R::Grid gr = grid_of(g);
    try {
        const std::vector<R::Point> pts =
            R::move_nodes(to_field(gr, u), to_field(gr, f_raw), raw_integral, t, steps);
        for (size_t p = 0; p < pts.size(); ++p)
            for (int c = 0; c < 3; ++c) pos[3 * p + c] = pts[p][c];
    } catch (const std::invalid_argument&) {
        return 1;
    }
    return 0;
}

void ref_sample_vector(const og_grid* g, const double* v, const double* pt, double* out) {
    const R::Grid gr = grid_of(g);
    const R::Point s = R::sample_vector(to_vector(gr, v, g->dim), {pt[0], pt[1], pt[2]});
    for (int c = 0; c < 3; ++c) out[c] = s[c];
}

int ref_integrate_streamline(const og_grid* g, const double* v, const double* seed, double step, int max_steps,
                             double* pts, int* stop) {
    const R::Grid gr = grid_of(g);
    const R::Streamline line =
        R::integrate_streamline(to_vector(gr, v, g->dim), {seed[0], seed[1], seed[2]}, step, max_steps);
    for (size_t q = 0; q < line.points.size(); ++q)
        for (int c = 0; c < 3; ++c) pts[3 * q + c] = line.points[q][c];
    *stop = line.stop == R::StreamlineStop::max_steps ? 0 : (line.stop == R::StreamlineStop::left_domain ? 1 : 2);
    return (int)line.points.size();
}

// deformation_problem (problems.cpp:302-325) for a closed curve given as
// xyz triples: the raw deposited source, the projected source and the raw
// integral; returns the grid dimension
int ref_deformation_setup(const double* pts, int npts, double a, int n, double* f_raw, double* f,
                          double* raw_integral) {
    R::Curve c;
    c.closed = true;
    for (int q = 0; q < npts; ++q) c.points.push_back({pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]});
    const R::DeformationSetup s = R::deformation_problem(c, a, n);
    std::memcpy(f_raw, s.f_raw.data(), s.f_raw.size() * sizeof(double));
    std::memcpy(f, s.problem.f.data(), s.problem.f.size() * sizeof(double));
    *raw_integral = s.raw_integral;
    return s.problem.grid.dim;
}

// io.cpp:45-64 (byte reference for the streamed writers)
void ref_write_field_vtk(const og_grid* g, const double* f, const char* path, const char* name) {
    R::write_field_vtk(to_field(grid_of(g), f), path, name);
}
void ref_write_vector_vtk(const og_grid* g, const double* v, const char* path, const char* name) {
    const R::Grid gr = grid_of(g);
    R::VectorField vf(gr);
    for (int c = 0; c < g->dim; ++c) std::memcpy(vf.comp[c].data(), v + (size_t)c * g->total, g->total * sizeof(double));
    R::write_vector_vtk(vf, path, name);
}

}  // extern "C"
