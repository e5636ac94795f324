// sgml_cpp.cpp — the reference's C++ solver API (include/sgml/*.hpp) on top of
// the C-ABI (include/sgml_b200.h).  A reference caller recompiles against
// these headers, links libsgml_b200.so instead of proj/core, and every
// solve-path call runs on the B200.
//
// Error behaviour mirrors the reference: std::invalid_argument for bad
// inputs, sgml::kernel_error for non-finite values / non-positive steps,
// std::logic_error / std::out_of_range for misuse, std::runtime_error for
// device failures.
#include <cmath>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sgml/cycle.hpp"
#include "../../include/sgml/grid.hpp"
#include "../../include/sgml/kernels.hpp"
#include "../../include/sgml/problems.hpp"
#include "../../include/sgml_b200.h"
#include "sgml_cpp_internal.hpp"

namespace sgml {

using cabi::check;
using cabi::context;
using cabi::Dev;
using cabi::to_c;

// ---- grid.hpp --------------------------------------------------------------

Grid make_grid(int dim, int n) {
    sgml_grid g{};
    check(sgml_make_grid(dim, n, &g));
    return Grid{g.dim, g.n, g.N, g.h, static_cast<std::size_t>(g.total)};
}

BoundarySpec BoundarySpec::all_dirichlet(double value) {
    BoundarySpec b;
    for (auto& f : b.faces) f = FaceBc{BcKind::dirichlet, value};
    return b;
}

BoundarySpec BoundarySpec::all_neumann() {
    BoundarySpec b;
    for (auto& f : b.faces) f = FaceBc{BcKind::neumann, 0.0};
    return b;
}

bool BoundarySpec::any_dirichlet(int dim) const {
    for (int f = 0; f < 2 * dim; ++f)
        if (faces[f].kind == BcKind::dirichlet) return true;
    return false;
}

bool BoundarySpec::on_dirichlet(const NodeIndex& idx, int dim, int N) const {
    const int c[3] = {idx.i, idx.j, idx.k};
    for (int a = 0; a < dim; ++a)
        if ((c[a] == 0 && face(a, 0).kind == BcKind::dirichlet) ||
            (c[a] == N - 1 && face(a, 1).kind == BcKind::dirichlet))
            return true;
    return false;
}

double BoundarySpec::dirichlet_value(const NodeIndex& idx, int dim, int N) const {
    const int c[3] = {idx.i, idx.j, idx.k};
    for (int a = 0; a < dim; ++a) {
        if (c[a] == 0 && face(a, 0).kind == BcKind::dirichlet) return face(a, 0).value;
        if (c[a] == N - 1 && face(a, 1).kind == BcKind::dirichlet) return face(a, 1).value;
    }
    throw std::logic_error("dirichlet_value: node is not on a Dirichlet face");
}

// ---- kernels.hpp -----------------------------------------------------------

void restriction_into(const Field& f, int v, const BoundarySpec& bc, Field& out, Field& scratch,
                      std::uint64_t* work) {
    if (&out == &scratch) throw std::invalid_argument("restriction_into: out and scratch must differ");
    Dev df(f), dout(f.grid()), dscr(f.grid());
    const sgml_bc b = to_c(bc);
    check(sgml_restriction_into(df.f, v, &b, dout.f, dscr.f, work));
    if (out.grid() != f.grid() || out.size() != f.size()) out = Field(f.grid());
    dout.to(out);
}

Field restriction(const Field& f, int v, const BoundarySpec& bc, std::uint64_t* work) {
    Field out(f.grid()), scratch(f.grid());
    restriction_into(f, v, bc, out, scratch, work);
    return out;
}

double relaxation_interpolation(SolveState& state, const Field& g, const Field* sigma_level, double a,
                                double safety, const BoundarySpec& bc, bool homogeneous, std::uint64_t* work) {
    const Grid& gr = state.u_prev.grid();
    Dev u(gr), du(gr), up(state.u_prev), dup(state.du_prev), dg(g);
    std::unique_ptr<Dev> ds;
    if (sigma_level) ds = std::make_unique<Dev>(*sigma_level);
    const sgml_bc b = to_c(bc);
    double diag = 0.0;
    const int st = sgml_relaxation_interpolation(u.f, up.f, du.f, dup.f, state.level, dg.f, ds ? ds->f : nullptr,
                                                 a, safety, &b, homogeneous ? 1 : 0, &diag, work);
    if (st == SGML_OK || st == SGML_ENONFINITE || st == SGML_EBADSTEP) {  // outputs written either way
        u.to(state.u);
        du.to(state.du);
    }
    check(st);
    return diag;
}

void residual_update(Field& r, const Field& e, const OperatorCoefficients& coeff, const BoundarySpec& bc) {
    Dev dr(r), de(e);
    std::unique_ptr<Dev> ds;
    if (coeff.sigma) ds = std::make_unique<Dev>(*coeff.sigma);
    const sgml_bc b = to_c(bc);
    check(sgml_residual_update(dr.f, de.f, ds ? ds->f : nullptr, coeff.a, &b));
    dr.to(r);
}

Field residual(const Field& u, const Field& f, const OperatorCoefficients& coeff, const BoundarySpec& bc) {
    Field r = f;
    residual_update(r, u, coeff, bc);
    return r;
}

double trapezoid_mean(const Field& f) {
    Dev d(f);
    double m = 0.0;
    check(sgml_trapezoid_mean(d.f, &m));
    return m;
}

void zero_mean_projection(Field& f) {
    Dev d(f);
    check(sgml_zero_mean_projection(d.f));
    d.to(f);
}

void apply_boundary(Field& u, const BoundarySpec& bc, bool homogeneous) {
    Dev d(u);
    const sgml_bc b = to_c(bc);
    check(sgml_apply_boundary(d.f, &b, homogeneous ? 1 : 0));
    d.to(u);
}

double max_abs(const Field& f) {
    Dev d(f);
    double m = 0.0;
    check(sgml_max_abs(d.f, &m));
    return m;
}

// ---- cycle.hpp -------------------------------------------------------------

CycleSchedule build_schedule(int n, int n_r) {
    int count = 0;
    check(sgml_build_schedule(n, n_r, nullptr, nullptr, nullptr, 0, &count));
    std::vector<int> k(count), l(count), c(count);
    check(sgml_build_schedule(n, n_r, k.data(), l.data(), c.data(), count, &count));
    CycleSchedule s;
    s.n = n;
    s.n_r = n_r;
    for (int i = 0; i < count; ++i)
        s.steps.push_back(ScheduleStep{k[i] == 0 ? ScheduleStep::Kind::restrict_source : ScheduleStep::Kind::relax,
                                       l[i], c[i]});
    return s;
}

std::uint64_t closed_form_work_units(int n, int n_r) { return sgml_closed_form_work_units(n, n_r); }

std::uint64_t schedule_work_units(const CycleSchedule& schedule) {
    std::uint64_t total = 0;
    for (const ScheduleStep& st : schedule.steps)
        total += st.kind == ScheduleStep::Kind::restrict_source ? static_cast<std::uint64_t>(st.level)
                                                                 : static_cast<std::uint64_t>(st.count);
    return total;
}

namespace {

std::size_t relax_passes(int n, int n_r) {
    std::size_t p = 0;
    for (const ScheduleStep& st : build_schedule(n, n_r).steps)
        if (st.kind == ScheduleStep::Kind::relax) p += static_cast<std::size_t>(st.count);
    return p;
}

struct HookData {
    const ExactSolution* exact;
    Grid grid;
};

int l1_hook(void* user, int, const sgml_field* u_total, double* l1) {
    const HookData* hd = static_cast<const HookData*>(user);
    Field u(hd->grid);
    if (sgml_field_download(u_total, u.data()) != SGML_OK) return 0;
    *l1 = l1_error(u, *hd->exact);
    return 1;
}

}  // namespace

// cycle.cpp:76-111 with the reference's full SolveState semantics: the caller's
// state (all four buffers and the level) goes in and comes back as the
// reference leaves it, the schedule's own steps and the caller's sigma levels
// are used (sgml_single_cycle_state: literal full-grid kernels, pass by pass)
void single_cycle(SolveState& state, const Field& source, const std::vector<Field>& sigma_levels, double a,
                  const BoundarySpec& bc, bool homogeneous, const CycleSchedule& schedule, double safety,
                  int cycle_index, double normalization, SolveReport& report, std::uint64_t& work_units) {
    const Grid& g = source.grid();
    Dev u(state.u), up(state.u_prev), du(state.du), dup(state.du_prev), src(source);
    std::vector<std::unique_ptr<Dev>> lv;
    std::vector<sgml_field*> lvp;
    for (const Field& f : sigma_levels) {
        lv.push_back(std::make_unique<Dev>(f));
        lvp.push_back(lv.back()->f);
    }
    std::vector<int> kinds, levels, counts;
    std::size_t passes = 0;
    for (const ScheduleStep& st : schedule.steps) {
        if (st.kind == ScheduleStep::Kind::relax && !lvp.empty() && static_cast<std::size_t>(st.level) >= lvp.size())
            throw std::out_of_range("single_cycle: no sigma level for a relax step");
        kinds.push_back(st.kind == ScheduleStep::Kind::restrict_source ? 0 : 1);
        levels.push_back(st.level);
        counts.push_back(st.count);
        if (st.kind == ScheduleStep::Kind::relax) passes += static_cast<std::size_t>(st.count);
    }
    const sgml_bc b = to_c(bc);
    std::vector<sgml_diag_sample> trace(std::max<std::size_t>(passes, 1));
    sgml_report rep{};
    rep.trace = trace.data();
    rep.trace_cap = static_cast<int64_t>(trace.size());
    int level = state.level;
    const int st = sgml_single_cycle_state(context(), u.f, up.f, du.f, dup.f, &level, src.f,
                                           lvp.empty() ? nullptr : lvp.data(), a, &b, homogeneous ? 1 : 0,
                                           kinds.data(), levels.data(), counts.data(), static_cast<int>(kinds.size()),
                                           safety, cycle_index, normalization, &rep, &work_units);
    for (int64_t t = 0; t < std::min<int64_t>(rep.n_trace, rep.trace_cap); ++t)
        report.trace.push_back(DiagSample{trace[t].cycle, trace[t].pass, trace[t].level, trace[t].value});
    // the state as the reference leaves it (also when a pass throws)
    if (st == SGML_OK || st == SGML_EBADSTEP || st == SGML_ENONFINITE) {
        u.to(state.u);
        up.to(state.u_prev);
        du.to(state.du);
        dup.to(state.du_prev);
        state.level = level;
    }
    check(st);
}

SolveResult solve(const ProblemSpec& problem, const SolverConfig& config) {
    const Grid& g = problem.grid;
    if (problem.f.grid() != g) throw std::invalid_argument("solve: source grid mismatch");
    if (problem.sigma.size() && problem.sigma.grid() != g)
        throw std::invalid_argument("solve: sigma grid mismatch");
    if (!(config.tol > 0.0)) throw std::invalid_argument("solve: tol must be positive");
    if (config.n_r < 1) throw std::invalid_argument("solve: n_r must be >= 1");

    SolveResult result{Field(g), {}};
    const int max_rows = std::max(1, config.max_cycles);
    std::vector<sgml_cycle_record> rows(static_cast<std::size_t>(max_rows));
    std::vector<sgml_diag_sample> trace(static_cast<std::size_t>(max_rows) * relax_passes(g.n, config.n_r));
    sgml_report rep{};
    rep.rows = rows.data();
    rep.rows_cap = max_rows;
    rep.trace = trace.data();
    rep.trace_cap = static_cast<int64_t>(trace.size());
    HookData hd{&problem.exact, g};
    if (problem.exact) {
        rep.hook = &l1_hook;
        rep.hook_user = &hd;
    }
    const sgml_bc b = to_c(problem.bc);
    const sgml_solver_cfg cfg{config.n_r, config.max_cycles, config.tol, config.safety};
    check(sgml_solve(context(), g.dim, g.n, &b, problem.f.data(),
                     problem.sigma.size() ? problem.sigma.data() : nullptr, problem.a, &cfg, nullptr,
                     result.u.data(), &rep));
    SolveReport& out = result.report;
    for (int64_t i = 0; i < std::min<int64_t>(rep.n_rows, rep.rows_cap); ++i) {
        CycleRecord r{rows[i].cycle, rows[i].work_units, rows[i].residual, rows[i].diag_min, std::nullopt};
        if (rows[i].has_l1) r.l1_error = rows[i].l1_error;
        out.rows.push_back(r);
    }
    for (int64_t t = 0; t < std::min<int64_t>(rep.n_trace, rep.trace_cap); ++t)
        out.trace.push_back(DiagSample{trace[t].cycle, trace[t].pass, trace[t].level, trace[t].value});
    out.converged = rep.converged != 0;
    out.nan_detected = rep.nan_detected != 0;
    out.stagnated = rep.stagnated != 0;
    out.normalization = rep.normalization;
    out.node_updates = rep.node_updates;
    return result;
}

void pure_neumann_pin(Field& u) { zero_mean_projection(u); }

std::vector<Field> restrict_sigma_levels(const Field& sigma, int n) {
    std::vector<Field> levels;
    if (!sigma.size()) return levels;
    Dev ds(sigma);
    std::vector<std::unique_ptr<Dev>> lv;
    std::vector<sgml_field*> lvp;
    for (int v = 0; v < n; ++v) {
        lv.push_back(std::make_unique<Dev>(sigma.grid()));
        lvp.push_back(lv.back()->f);
    }
    check(sgml_restrict_sigma_levels(ds.f, lvp.data()));
    for (int v = 0; v < n; ++v) {
        levels.emplace_back(sigma.grid());
        lv[static_cast<std::size_t>(v)]->to(levels.back());
    }
    return levels;
}

// problems.cpp:195-215: serial compensated sums of w|u - exact| and w|exact|
// with trapezoid weights (1/2 per face axis).
double l1_error(const Field& v_h, const ExactSolution& exact) {
    if (!exact) throw std::invalid_argument("l1_error: no exact solution");
    const Grid& g = v_h.grid();
    double num = 0.0, cnum = 0.0, den = 0.0, cden = 0.0;
    for (std::size_t p = 0; p < v_h.size(); ++p) {
        const NodeIndex x = v_h.node_of(p);
        double w = (x.i == 0 || x.i == g.N - 1) ? 0.5 : 1.0;
        w *= (x.j == 0 || x.j == g.N - 1) ? 0.5 : 1.0;
        if (g.dim == 3) w *= (x.k == 0 || x.k == g.N - 1) ? 0.5 : 1.0;
        const double ue = exact(x.i * g.h, x.j * g.h, x.k * g.h);
        double y = w * std::abs(v_h[p] - ue) - cnum;
        double t = num + y;
        cnum = (t - num) - y;
        num = t;
        y = w * std::abs(ue) - cden;
        t = den + y;
        cden = (t - den) - y;
        den = t;
    }
    if (den == 0.0) throw std::invalid_argument("l1_error: exact solution is identically zero");
    return num / den;
}

// ---- problems.hpp (post-solve fields, problems.cpp:327-455) -----------------

namespace {

// device copies of the dim (or 3) components of a host vector field
struct DevVec {
    std::vector<std::unique_ptr<Dev>> c;
    std::vector<sgml_field*> h;
    DevVec(const VectorField& v, int n) {
        for (int k = 0; k < n; ++k) {
            c.push_back(std::make_unique<Dev>(v.comp[k]));
            h.push_back(c.back()->f);
        }
    }
    DevVec(const Grid& g, int n) {
        for (int k = 0; k < n; ++k) {
            c.push_back(std::make_unique<Dev>(g));
            h.push_back(c.back()->f);
        }
    }
    void to(VectorField& v, int n) const {
        for (int k = 0; k < n; ++k) c[k]->to(v.comp[k]);
    }
};

}  // namespace

VectorField gradient(const Field& u) {
    const Grid& g = u.grid();
    Dev du(u);
    DevVec out(g, g.dim);
    check(sgml_gradient(du.f, out.h.data()));
    VectorField v(g);
    out.to(v, g.dim);
    return v;
}

VectorField curl(const VectorField& psi) {
    if (psi.dim != 3) throw std::invalid_argument("curl: defined for 3D fields");
    const Grid& g = psi.grid();
    DevVec in(psi, 3), out(g, 3);
    check(sgml_curl(in.h.data(), out.h.data()));
    VectorField v(g);
    out.to(v, 3);
    return v;
}

Field divergence(const VectorField& v) {
    const Grid& g = v.grid();
    DevVec in(v, v.dim);
    Dev out(g);
    check(sgml_divergence(in.h.data(), out.f));
    Field d(g);
    out.to(d);
    return d;
}

VectorField deformation_velocity(const Field& u, const Field& f_raw, double raw_integral, double t) {
    const Grid& g = u.grid();
    Dev du(u), df(f_raw);
    DevVec out(g, g.dim);
    check(sgml_deformation_velocity(du.f, df.f, raw_integral, t, out.h.data()));
    VectorField v(g);
    out.to(v, g.dim);
    return v;
}

std::vector<Point> move_nodes(const Field& u, const Field& f_raw, double raw_integral, double t, int steps) {
    if (steps < 1) throw std::invalid_argument("move_nodes: steps must be >= 1");
    const Grid& g = u.grid();
    Dev du(u), df(f_raw);
    DevVec pos(g, 3);
    check(sgml_move_nodes(du.f, df.f, raw_integral, t, steps, pos.h.data()));
    VectorField p(g);
    pos.to(p, 3);
    std::vector<Point> out(g.total);
    for (std::size_t q = 0; q < g.total; ++q) out[q] = {p.comp[0][q], p.comp[1][q], p.comp[2][q]};
    return out;
}

Point sample_vector(const VectorField& v, const Point& p) {
    DevVec in(v, v.dim);
    Point out{0.0, 0.0, 0.0};
    check(sgml_sample_vector(in.h.data(), v.dim, p.data(), 1, out.data()));
    return out;
}

Streamline integrate_streamline(const VectorField& v, const Point& seed, double step, int max_steps) {
    if (!(step > 0.0)) throw std::invalid_argument("integrate_streamline: step must be positive");
    DevVec in(v, v.dim);
    std::vector<double> pts(3 * (static_cast<std::size_t>(max_steps > 0 ? max_steps : 0) + 1));
    int count = 0, stop = 0;
    check(sgml_integrate_streamlines(in.h.data(), seed.data(), 1, step, max_steps, pts.data(), &count, &stop));
    Streamline line;
    for (int q = 0; q < count; ++q) line.points.push_back({pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]});
    line.stop = static_cast<StreamlineStop>(stop);
    return line;
}

}  // namespace sgml
