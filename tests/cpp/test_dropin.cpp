// test_dropin.cpp — the reference's C++ API (include/sgml/*.hpp) exercised the
// way proj/tests/unit/{cycle,kernels}_tests.cpp use it, running on the B200
// through libsgml_b200.so, with bit-parity checks against the oracle
// (oracle/sgml_oracle.c, test infrastructure).  Exit code = failures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgml/cycle.hpp"
#include "sgml/grid.hpp"
#include "sgml/kernels.hpp"
#include "sgml/problems.hpp"

extern "C" {
#include "sgml_oracle.h"
}

using namespace sgml;

static int failures = 0;
#define EXPECT(cond)                                                             \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static og_grid og_of(const Grid& g) {
    og_grid o;
    og_make_grid(g.dim, g.n, &o);
    return o;
}

static og_bc og_of(const BoundarySpec& b) {
    og_bc o;
    for (int f = 0; f < 6; ++f) {
        o.kind[f] = b.faces[f].kind == BcKind::neumann ? 1 : 0;
        o.value[f] = b.faces[f].value;
    }
    return o;
}

static bool same_bits(const Field& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return false;
    for (std::size_t p = 0; p < a.size(); ++p) {
        const double x = a[p] == 0.0 ? 0.0 : a[p], y = b[p] == 0.0 ? 0.0 : b[p];
        if (std::memcmp(&x, &y, sizeof x) != 0) return false;
    }
    return true;
}

// reference problems.cpp:160-176 (u = -P(x)P(y), P = t^2 - t^4)
static ProblemSpec poisson2d(int n) {
    ProblemSpec p;
    p.grid = make_grid(2, n);
    p.f = Field(p.grid);
    p.bc = BoundarySpec::all_dirichlet(0.0);
    og_grid g = og_of(p.grid);
    og_fill_poisson2d(&g, p.f.data());
    p.exact = [](double x, double y, double) {
        const double px = x * x - x * x * x * x, py = y * y - y * y * y * y;
        return -px * py;
    };
    return p;
}

static void test_schedule() {
    // cycle_tests.cpp:16-60
    const CycleSchedule s = build_schedule(2, 1);
    EXPECT(s.steps.size() == 7);
    EXPECT(s.steps[0].kind == ScheduleStep::Kind::restrict_source && s.steps[0].level == 1);
    EXPECT(s.steps[6].kind == ScheduleStep::Kind::relax && s.steps[6].level == 0);
    EXPECT(schedule_work_units(s) == 5);
    EXPECT(closed_form_work_units(8, 2) == 158 && closed_form_work_units(6, 8) == 155);
    for (int n = 1; n <= 10; ++n)
        for (int nr : {1, 2, 3, 8}) EXPECT(closed_form_work_units(n, nr) == schedule_work_units(build_schedule(n, nr)));
    EXPECT(throws<std::invalid_argument>([] { build_schedule(0, 1); }));
    EXPECT(throws<std::invalid_argument>([] { make_grid(4, 3); }));
}

static void test_driver_converges() {
    // cycle_tests.cpp:74-103, plus bit parity of u and every row vs the oracle
    const ProblemSpec prob = poisson2d(4);
    SolverConfig cfg;
    cfg.tol = 1e-11;
    const SolveResult res = solve(prob, cfg);
    EXPECT(res.report.converged && !res.report.nan_detected && !res.report.stagnated);
    EXPECT(res.report.rows.size() >= 3 && res.report.rows.size() < 25);
    const std::uint64_t per = closed_form_work_units(4, cfg.n_r);
    double prev = 2.0;
    for (std::size_t i = 0; i < res.report.rows.size(); ++i) {
        EXPECT(res.report.rows[i].work_units == per * (i + 1));
        EXPECT(res.report.rows[i].residual < prev);
        prev = res.report.rows[i].residual;
        EXPECT(res.report.rows[i].l1_error.has_value());
    }
    EXPECT(res.report.rows.back().residual <= 1e-11);
    EXPECT(*res.report.rows.back().l1_error < 0.03);
    EXPECT(res.report.node_updates == res.report.rows.back().work_units * prob.grid.total);

    og_grid g = og_of(prob.grid);
    og_bc b = og_of(prob.bc);
    std::vector<double> u(prob.grid.total);
    std::vector<og_row> rows(64);
    std::vector<og_sample> trace(1 << 14);
    og_report rep{};
    rep.rows = rows.data();
    rep.rows_cap = 64;
    rep.trace = trace.data();
    rep.trace_cap = 1 << 14;
    og_solve(&g, &b, prob.f.data(), nullptr, 0.0, cfg.n_r, cfg.tol, cfg.max_cycles, cfg.safety, u.data(), &rep);
    EXPECT(same_bits(res.u, u));
    EXPECT(rep.n_rows == (int64_t)res.report.rows.size());
    for (std::size_t i = 0; i < res.report.rows.size() && (int64_t)i < rep.n_rows; ++i)
        EXPECT(rows[i].residual == res.report.rows[i].residual && rows[i].diag_min == res.report.rows[i].diag_min);
    EXPECT(rep.n_trace == (int64_t)res.report.trace.size());
    for (std::size_t t = 0; t < res.report.trace.size() && (int64_t)t < rep.n_trace; ++t)
        EXPECT(trace[t].value == res.report.trace[t].value && trace[t].pass == res.report.trace[t].pass);
}

static void test_capacitor_bitwise() {
    // heterogeneous sigma, mixed faces (reference capacitor_problem shape), 3D
    ProblemSpec p;
    p.grid = make_grid(3, 4);
    p.f = Field(p.grid);
    p.sigma = Field(p.grid);
    og_grid g = og_of(p.grid);
    og_fill_capacitor_sigma(&g, -1.0, p.sigma.data());
    p.bc = BoundarySpec::all_neumann();
    p.bc.face(2, 0) = {BcKind::dirichlet, -1.0};
    p.bc.face(2, 1) = {BcKind::dirichlet, 1.0};
    SolverConfig cfg;
    cfg.tol = 1e-10;
    const SolveResult res = solve(p, cfg);
    og_bc b = og_of(p.bc);
    std::vector<double> u(p.grid.total);
    std::vector<og_row> rows(64);
    std::vector<og_sample> trace(1 << 15);
    og_report rep{};
    rep.rows = rows.data();
    rep.rows_cap = 64;
    rep.trace = trace.data();
    rep.trace_cap = 1 << 15;
    og_solve(&g, &b, p.f.data(), p.sigma.data(), 0.0, 2, 1e-10, cfg.max_cycles, 0.9, u.data(), &rep);
    EXPECT(res.report.converged == (rep.converged != 0));
    EXPECT((int64_t)res.report.rows.size() == rep.n_rows);
    EXPECT(res.report.normalization == rep.normalization);
    EXPECT(same_bits(res.u, u));
}

static void test_kernels() {
    // kernels_tests.cpp:38-46, 116-132, 160-169, 171-189 (+ oracle parity)
    const Grid g = make_grid(2, 3);
    Field f(g);
    for (std::size_t p = 0; p < f.size(); ++p) f[p] = std::sin(0.37 * (double)p);
    std::uint64_t work = 0;
    EXPECT(restriction(f, 0, BoundarySpec::all_neumann(), &work) == f && work == 0);
    const Field r3 = restriction(f, 3, BoundarySpec::all_dirichlet(0.0), &work);
    EXPECT(work == 3);
    og_grid og = og_of(g);
    og_bc ob = og_of(BoundarySpec::all_dirichlet(0.0));
    std::vector<double> ro(g.total), rs(g.total);
    og_restriction_into(&og, &ob, f.data(), 3, ro.data(), rs.data(), nullptr);
    EXPECT(same_bits(r3, ro));

    BoundarySpec bc3 = BoundarySpec::all_dirichlet(3.0);
    SolveState st(make_grid(2, 2));
    st.reset_level(0);
    for (std::size_t p = 0; p < st.u_prev.size(); ++p) st.u_prev[p] = 0.1 * (double)p;
    Field gsrc(st.u.grid());
    relaxation_interpolation(st, gsrc, nullptr, 0.0, 0.9, bc3, false);
    EXPECT(st.u.at(0, 2) == 3.0 && st.u.at(4, 4) == 3.0);
    EXPECT(st.du.at(0, 2) == 3.0 - st.u_prev.at(0, 2));
    st.reset_level(0);
    relaxation_interpolation(st, gsrc, nullptr, 0.0, 0.9, bc3, true);
    EXPECT(st.u.at(0, 2) == 0.0);

    SolveState bad(make_grid(2, 2));
    bad.reset_level(0);
    bad.u_prev.at(2, 2) = std::nan("");
    EXPECT(throws<kernel_error>(
        [&] { relaxation_interpolation(bad, gsrc, nullptr, 0.0, 0.9, BoundarySpec::all_dirichlet(0.0), true); }));

    Field u(g), rhs(g);
    for (std::size_t p = 0; p < u.size(); ++p) {
        u[p] = std::cos(0.11 * (double)p);
        rhs[p] = std::sin(0.05 * (double)p);
    }
    const OperatorCoefficients coeff{nullptr, 0.3};
    const Field r1 = residual(u, rhs, coeff, BoundarySpec::all_dirichlet(0.0));
    Field r2 = rhs;
    residual_update(r2, u, coeff, BoundarySpec::all_dirichlet(0.0));
    EXPECT(r1 == r2);
    for (int i = 0; i < g.N; ++i) EXPECT(r1.at(i, 0) == 0.0);
    std::vector<double> rr(rhs.data(), rhs.data() + rhs.size());
    og_residual_update(&og, &ob, rr.data(), u.data(), nullptr, 0.3);
    EXPECT(same_bits(r1, rr));

    Field m(make_grid(2, 2));
    m.at(3, 1) = -7.5;
    m.at(1, 3) = 6.0;
    EXPECT(max_abs(m) == 7.5);
}

static void test_driver_edges() {
    // cycle_tests.cpp:126-202
    ProblemSpec p = poisson2d(4);
    SolverConfig one;
    one.tol = 1.0;
    const SolveResult r1 = solve(p, one);
    EXPECT(r1.report.converged && r1.report.rows.size() == 1);

    ProblemSpec z;
    z.grid = make_grid(2, 3);
    z.f = Field(z.grid);
    z.bc = BoundarySpec::all_dirichlet(1.0);
    SolverConfig c11;
    c11.tol = 1e-11;
    const SolveResult rz = solve(z, c11);
    EXPECT(rz.report.converged && rz.report.normalization > 0.0);
    for (std::size_t q = 0; q < rz.u.size(); ++q) EXPECT(std::abs(rz.u[q] - 1.0) <= 1e-9);

    ProblemSpec indef = poisson2d(3);
    indef.a = 100.0;
    SolverConfig c30;
    c30.max_cycles = 30;
    const SolveResult ri = solve(indef, c30);
    EXPECT(!ri.report.converged);
    EXPECT(ri.report.stagnated || ri.report.nan_detected || ri.report.rows.size() == 30);

    ProblemSpec bad = poisson2d(3);
    SolverConfig c;
    c.tol = 0.0;
    EXPECT(throws<std::invalid_argument>([&] { solve(bad, c); }));
    c.tol = 1e-10;
    c.n_r = 0;
    EXPECT(throws<std::invalid_argument>([&] { solve(bad, c); }));
    c.n_r = 2;
    bad.f.at(2, 2) = std::nan("");
    EXPECT(throws<std::invalid_argument>([&] { solve(bad, c); }));

    Field sigma(make_grid(2, 3), 1.0);
    sigma.at(4, 4) = 9.0;
    const std::vector<Field> lv = restrict_sigma_levels(sigma, 3);
    EXPECT(lv.size() == 3 && lv[0] == sigma);
    Field neg(make_grid(2, 3), 1.0);
    neg.at(3, 3) = -50.0;
    EXPECT(throws<std::invalid_argument>([&] { restrict_sigma_levels(neg, 3); }));
}

// problems_tests.cpp:165-309 through the drop-in header, bitwise against the oracle
static void test_post_solve_fields() {
    const Grid g = make_grid(3, 4);
    og_grid og = og_of(g);
    VectorField psi(g);
    std::vector<double> flat(3 * g.total);
    for (int c = 0; c < 3; ++c) {
        og_lcg_fill(psi.comp[c].data(), g.total, 500 + c);
        std::memcpy(flat.data() + c * g.total, psi.comp[c].data(), g.total * sizeof(double));
    }
    const VectorField v = curl(psi);
    std::vector<double> want(3 * g.total);
    og_curl(&og, flat.data(), want.data());
    for (int c = 0; c < 3; ++c)
        EXPECT(same_bits(v.comp[c], std::vector<double>(want.begin() + c * g.total, want.begin() + (c + 1) * g.total)));
    const Field d = divergence(v);
    std::vector<double> vflat(3 * g.total), dwant(g.total);
    for (int c = 0; c < 3; ++c) std::memcpy(vflat.data() + c * g.total, v.comp[c].data(), g.total * sizeof(double));
    og_divergence(&og, vflat.data(), dwant.data());
    EXPECT(same_bits(d, dwant));
    const VectorField gr = gradient(psi.comp[0]);
    std::vector<double> gwant(3 * g.total);
    og_gradient(&og, psi.comp[0].data(), gwant.data());
    EXPECT(same_bits(gr.comp[1], std::vector<double>(gwant.begin() + g.total, gwant.begin() + 2 * g.total)));
    EXPECT(throws<std::invalid_argument>([&] { curl(VectorField(make_grid(2, 3))); }));

    // deformation velocity and node motion (problems_tests.cpp:165-189)
    const Grid g2 = make_grid(2, 3);
    Field u(g2), f_raw(g2);
    for (std::size_t p = 0; p < u.size(); ++p) u[p] = 2.0 * u.node_of(p).i * g2.h;
    const VectorField dv = deformation_velocity(u, f_raw, 4.0, 0.7);
    EXPECT(std::abs(dv.comp[0].at(3, 3) + 0.5) <= 1e-13);
    EXPECT(throws<std::invalid_argument>([&] { deformation_velocity(u, f_raw, 0.0, 0.0); }));
    const std::vector<Point> pos = move_nodes(Field(g2), f_raw, 1.0, 0.5, 10);
    EXPECT(pos.size() == g2.total && pos[7][0] == 7 * g2.h);
    EXPECT(throws<std::invalid_argument>([&] { move_nodes(u, f_raw, 1.0, 0.5, 0); }));

    // streamline contract (problems_tests.cpp:281-309)
    VectorField drift(g2);
    drift.comp[0].fill(1.0);
    const Streamline out = integrate_streamline(drift, {0.75, 0.5, 0.0}, 0.1, 100);
    EXPECT(out.stop == StreamlineStop::left_domain && out.points.size() >= 2);
    EXPECT(std::abs(out.points[1][0] - 0.85) <= 1e-13);
    const Streamline stall = integrate_streamline(VectorField(g2), {0.5, 0.5, 0.0}, 0.1, 100);
    EXPECT(stall.stop == StreamlineStop::stagnation && stall.points.size() == 1);
    const Point s = sample_vector(drift, {0.317, 0.682, 0.0});
    EXPECT(s[0] == 1.0 && s[1] == 0.0 && s[2] == 0.0);
}

int main() {
    const std::vector<std::pair<const char*, void (*)()>> tests = {
        {"schedule", test_schedule},
        {"driver_converges", test_driver_converges},
        {"capacitor_bitwise", test_capacitor_bitwise},
        {"kernels", test_kernels},
        {"driver_edges", test_driver_edges},
        {"post_solve_fields", test_post_solve_fields},
    };
    for (const auto& [name, fn] : tests) {
        const int before = failures;
        try {
            fn();
        } catch (const std::exception& e) {
            std::printf("FAIL %s: exception %s\n", name, e.what());
            ++failures;
        }
        std::printf("%s %s\n", failures == before ? "PASS" : "FAIL", name);
    }
    return failures;
}
