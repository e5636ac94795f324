// sgml_cpp_more.cpp — the rest of the reference's C++ surface:
// stencil.hpp's pointwise utilities, problems.hpp's builders and curve
// functions, io.hpp.  See include/sgml/{stencil,problems,io}.hpp.
//
// * stencil.hpp: single-node host utilities with the reference's semantics
//   (stencil.cpp:13-154).  No solve path calls them: the passes of a solve
//   evaluate the same operator inside the sm_100a kernels.
// * problems.hpp: the dense fields are built on the device by the C-ABI
//   builders (csrc/builders.cpp, bit-identical to the reference's builders)
//   and copied into host Fields; the exact-solution closures are host
//   lambdas, as in the reference.
// * io.hpp: VTK writers stream through sgml_write_vtk_host (all host threads,
//   byte-identical to io.cpp); the readers and CSV files are small host code.
#include <algorithm>
#include <array>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <memory>
#include <numbers>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sgml/cycle.hpp"
#include "../../include/sgml/io.hpp"
#include "../../include/sgml/problems.hpp"
#include "../../include/sgml/stencil.hpp"
#include "sgml_cpp_internal.hpp"

namespace sgml {

using cabi::check;
using cabi::Dev;

// ============================================================================
// stencil.hpp
// ============================================================================

namespace {

struct OffsetTable {
    std::array<StencilOffset, 26> e{};
    std::size_t count = 0;
    explicit OffsetTable(int dim) {
        // r outermost, then q, then p: the reference's summation order
        for (int r = (dim == 3 ? -1 : 0); r <= (dim == 3 ? 1 : 0); ++r)
            for (int q = -1; q <= 1; ++q)
                for (int p = -1; p <= 1; ++p)
                    if (p || q || r) e[count++] = StencilOffset{p, q, r, 1.0 / static_cast<double>(p * p + q * q + r * r)};
    }
};

}  // namespace

std::span<const StencilOffset> stencil_offsets(int dim) {
    static const OffsetTable t2(2), t3(3);
    const OffsetTable& t = dim == 2 ? t2 : t3;
    return std::span<const StencilOffset>(t.e.data(), t.count);
}

namespace detail {

double ghost_value(const Field& u, const BoundarySpec& bc, int i, int j, int k) {
    const int N = u.grid().N;
    int c[3] = {i, j, k};
    // the first out-of-range axis (x before y before z) is reflected; the
    // mirror and, for a Dirichlet face, the face node are read recursively
    for (int ax = 0; ax < 3; ++ax) {
        if (c[ax] >= 0 && c[ax] <= N - 1) continue;
        const int side = c[ax] < 0 ? 0 : 1;
        int m[3] = {c[0], c[1], c[2]};
        m[ax] = side == 0 ? -c[ax] : 2 * (N - 1) - c[ax];
        const double mv = ghost_value(u, bc, m[0], m[1], m[2]);
        if (bc.face(ax, side).kind == BcKind::neumann) return mv;
        int f[3] = {c[0], c[1], c[2]};
        f[ax] = side == 0 ? 0 : N - 1;
        return 2.0 * ghost_value(u, bc, f[0], f[1], f[2]) - mv;
    }
    return u.at(i, j, k);
}

double mirror_value(const Field& u, int i, int j, int k) {
    const int N = u.grid().N;
    return u.at(mirror_index(i, N), mirror_index(j, N), mirror_index(k, N));
}

}  // namespace detail

double restrict_at(const Field& f, const NodeIndex& idx, int lam, const BoundarySpec& bc) {
    const int dim = f.grid().dim;
    double acc = 0.0;
    for (int r = (dim == 3 ? -1 : 0); r <= (dim == 3 ? 1 : 0); ++r)
        for (int q = -1; q <= 1; ++q)
            for (int p = -1; p <= 1; ++p) {
                double w = restrict_axis_weight(p) * restrict_axis_weight(q);
                if (dim == 3) w = w * restrict_axis_weight(r);
                acc += w * detail::ghost_value(f, bc, idx.i + p * lam, idx.j + q * lam,
                                               dim == 3 ? idx.k + r * lam : 0);
            }
    return acc;
}

double apply_operator(const Field& u, const OperatorCoefficients& coeff, const NodeIndex& idx, int lam,
                      const BoundarySpec& bc) {
    const Grid& g = u.grid();
    const double uc = u.at(idx.i, idx.j, idx.k);
    const double sc = coeff.sigma ? coeff.sigma->at(idx.i, idx.j, idx.k) : 1.0;
    double acc = 0.0;
    for (const StencilOffset& o : stencil_offsets(g.dim)) {
        const int ni = idx.i + o.p * lam, nj = idx.j + o.q * lam, nk = idx.k + o.r * lam;
        const double sn = coeff.sigma ? detail::mirror_value(*coeff.sigma, ni, nj, nk) : 1.0;
        acc += 0.5 * (sn + sc) * (detail::ghost_value(u, bc, ni, nj, nk) - uc) * o.inv_l2;
    }
    const double s = lam * g.h;
    return acc * stencil_prefactor(g.dim) / (s * s) + coeff.a * uc;
}

double stable_step(const OperatorCoefficients& coeff, const Grid& grid, int lam, double safety) {
    if (!(safety > 0.0 && safety <= 1.0)) throw std::invalid_argument("stable_step: safety must lie in (0, 1]");
    double smax = 1.0;
    if (coeff.sigma) {
        const Field& s = *coeff.sigma;
        smax = 0.0;
        for (std::size_t p = 0; p < s.size(); ++p) smax = std::max(smax, s[p]);
        if (!(smax > 0.0)) throw std::invalid_argument("stable_step: sigma must be positive");
    }
    const double s = lam * grid.h;
    return safety * step_constant(grid.dim) * s * s / smax;
}

// ============================================================================
// problems.hpp
// ============================================================================

namespace {

constexpr double kPi = std::numbers::pi_v<double>;

std::vector<double> flat(const std::vector<Point>& pts) {
    std::vector<double> v;
    v.reserve(3 * pts.size());
    for (const Point& p : pts) v.insert(v.end(), p.begin(), p.end());
    return v;
}

std::vector<Point> unflat(const std::vector<double>& v, std::size_t count) {
    std::vector<Point> pts(count);
    for (std::size_t i = 0; i < count; ++i) pts[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    return pts;
}

// C-ABI curve producer with the count / cap protocol -> Curve
template <typename Call>
Curve curve_from(Call&& call, bool closed, bool with_payload) {
    int count = 0;
    check(call(nullptr, nullptr, 0, &count));
    std::vector<double> pts(3 * static_cast<std::size_t>(count)), pay(with_payload ? pts.size() : 0);
    check(call(pts.data(), with_payload ? pay.data() : nullptr, count, &count));
    Curve c;
    c.closed = closed;
    c.points = unflat(pts, static_cast<std::size_t>(count));
    if (with_payload) c.payload = unflat(pay, static_cast<std::size_t>(count));
    return c;
}

VectorField download3(const std::array<std::unique_ptr<Dev>, 3>& d, const Grid& g) {
    VectorField v(g);
    for (int c = 0; c < 3; ++c) d[c]->to(v.comp[c]);
    return v;
}

}  // namespace

ProblemSpec poisson2d_problem(int n) {
    ProblemSpec prob;
    prob.grid = make_grid(2, n);
    prob.f = Field(prob.grid);
    prob.bc = BoundarySpec::all_dirichlet(0.0);
    const auto P = [](double t) { return t * t - t * t * t * t; };
    prob.exact = [P](double x, double y, double) { return -P(x) * P(y); };
    Dev d(prob.grid);
    check(sgml_build_poisson2d_source(d.f));
    d.to(prob.f);
    return prob;
}

ProblemSpec poisson3d_problem(int n) {
    ProblemSpec prob;
    prob.grid = make_grid(3, n);
    prob.f = Field(prob.grid);
    prob.bc = BoundarySpec::all_dirichlet(0.0);
    prob.exact = [](double x, double y, double z) {
        return std::sin(kPi * x) * std::sin(kPi * y) * std::sin(kPi * z);
    };
    Dev d(prob.grid);
    check(sgml_build_poisson3d_source(d.f));
    d.to(prob.f);
    return prob;
}

Curve resample_curve(const Curve& curve, double h) {
    const std::vector<double> in = flat(curve.points);
    const bool pay = !curve.payload.empty();
    const int m = static_cast<int>(curve.points.size());
    return curve_from(
        [&](double* p, double* w, int cap, int* cnt) {
            return sgml_resample_curve(in.data(), m, curve.closed, pay, h, p, w, cap, cnt);
        },
        curve.closed, pay);
}

Field deposit_delta(const Curve& curve, const Grid& grid, double strength) {
    if (curve.points.size() < 2) throw std::invalid_argument("deposit_delta: need at least 2 points");
    const std::vector<double> in = flat(curve.points);
    Dev d(grid);
    check(sgml_deposit_delta(in.data(), static_cast<int>(curve.points.size()), curve.closed, strength, d.f));
    Field f(grid);
    d.to(f);
    return f;
}

VectorField deposit_delta_vector(const Curve& curve, const Grid& grid) {
    if (curve.payload.size() != curve.points.size())
        throw std::invalid_argument("deposit_delta_vector: curve carries no payload");
    const std::vector<double> in = flat(curve.points), pay = flat(curve.payload);
    std::array<std::unique_ptr<Dev>, 3> d;
    sgml_field* f3[3];
    for (int c = 0; c < 3; ++c) {
        d[c] = std::make_unique<Dev>(grid);
        f3[c] = d[c]->f;
    }
    check(sgml_deposit_delta_vector(in.data(), pay.data(), static_cast<int>(curve.points.size()), curve.closed, f3));
    return download3(d, grid);
}

DeformationSetup deformation_problem(const Curve& curve, double a, int n) {
    int dim = 2;
    for (const Point& p : curve.points)
        if (p[2] != 0.0) dim = 3;
    const Grid grid = make_grid(dim, n);
    const std::vector<double> in = flat(curve.points);
    Dev f(grid), f_raw(grid);
    double ri = 0.0;
    check(sgml_build_deformation_problem(in.data(), static_cast<int>(curve.points.size()), curve.closed,
                                         !curve.payload.empty(), f.f, f_raw.f, &ri));
    DeformationSetup setup;
    setup.problem.grid = grid;
    setup.problem.a = a;
    setup.problem.bc = BoundarySpec::all_neumann();
    setup.problem.f = Field(grid);
    f.to(setup.problem.f);
    setup.f_raw = Field(grid);
    f_raw.to(setup.f_raw);
    setup.raw_integral = ri;
    return setup;
}

TrifoilSetup trifoil_problem(int n, double r) {
    if (!(r > 0.0)) throw std::invalid_argument("trifoil_problem: r must be positive");
    const Grid grid = make_grid(3, n);
    TrifoilSetup setup;
    setup.curve = curve_from([&](double* p, double* w, int cap, int* cnt) { return sgml_trifoil_curve(r, grid.h, p, w, cap, cnt); },
                             true, true);
    setup.omega = deposit_delta_vector(setup.curve, grid);
    for (int c = 0; c < 3; ++c) {
        ProblemSpec& prob = setup.psi[c];
        prob.grid = grid;
        prob.bc = BoundarySpec::all_dirichlet(0.0);
        prob.f = setup.omega.comp[c];
        for (std::size_t p = 0; p < prob.f.size(); ++p) prob.f[p] = -prob.f[p];
    }
    return setup;
}

ProblemSpec capacitor_problem(int n, const std::string& mode) {
    if (mode != "low" && mode != "high")
        throw std::invalid_argument("capacitor_problem: mode must be \"high\" or \"low\"");
    ProblemSpec prob;
    prob.grid = make_grid(3, n);
    prob.f = Field(prob.grid);
    prob.sigma = Field(prob.grid);
    Dev s(prob.grid);
    check(sgml_build_capacitor_sigma(s.f, mode == "high" ? 1 : 0));
    s.to(prob.sigma);
    prob.bc = BoundarySpec::all_neumann();
    prob.bc.face(2, 0) = {BcKind::dirichlet, -1.0};
    prob.bc.face(2, 1) = {BcKind::dirichlet, +1.0};
    return prob;
}

// ============================================================================
// io.hpp
// ============================================================================

namespace {

void check_io(int status) {
    if (status == SGML_EIO) throw io_error(sgml_last_error());
    check(status);
}

std::ofstream open_out(const std::string& path) {
    std::ofstream out(path);
    if (!out) throw io_error("cannot open for writing: " + path);
    return out;
}

void close_out(std::ofstream& out, const std::string& path) {
    out.close();
    if (!out) throw io_error("write failed: " + path);
}

sgml_grid c_grid(const Grid& g) {
    sgml_grid c{};
    check(sgml_make_grid(g.dim, g.n, &c));
    return c;
}

}  // namespace

std::string format_double(double x) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.17g", x);
    return buf;
}

void write_field_vtk(const Field& f, const std::string& path, const std::string& name) {
    const sgml_grid g = c_grid(f.grid());
    const double* comps[1] = {f.data()};
    check_io(sgml_write_vtk_host(comps, 1, &g, path.c_str(), name.c_str()));
}

void write_vector_vtk(const VectorField& v, const std::string& path, const std::string& name) {
    const sgml_grid g = c_grid(v.grid());
    // a default-constructed third component of a 2D field is written as zeros
    const double* comps[3] = {v.comp[0].data(), v.comp[1].data(), v.comp[2].size() ? v.comp[2].data() : nullptr};
    check_io(sgml_write_vtk_host(comps, 3, &g, path.c_str(), name.c_str()));
}

Field read_field_vtk(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw io_error("cannot open: " + path);
    std::string tok;
    long long nx = 0, ny = 0, nz = 0;
    unsigned long long count = 0;
    while (in >> tok) {
        if (tok == "DIMENSIONS") {
            if (!(in >> nx >> ny >> nz)) throw io_error("bad DIMENSIONS: " + path);
        } else if (tok == "POINT_DATA") {
            if (!(in >> count)) throw io_error("bad POINT_DATA: " + path);
        } else if (tok == "LOOKUP_TABLE") {
            in >> tok;  // the table's name; the data follow
            break;
        }
    }
    if (nx < 3 || nx != ny || (nz != 1 && nz != nx)) throw io_error("unsupported grid dimensions: " + path);
    int n = 1;
    while ((1LL << n) + 1 < nx && n < 13) ++n;
    if ((1LL << n) + 1 != nx) throw io_error("dimensions are not 2^n + 1 points: " + path);
    const Grid g = make_grid(nz == 1 ? 2 : 3, n);
    if (g.total != count) throw io_error("dimensions are not 2^n + 1 points: " + path);
    Field f(g);
    for (std::size_t p = 0; p < g.total; ++p)
        if (!(in >> f[p])) throw io_error("truncated point data: " + path);
    return f;
}

void write_report_csv(const SolveReport& report, const std::string& path) {
    std::ofstream out = open_out(path);
    out << "cycle,work_units,residual,diag_residual_min,l1_error\n";
    for (const CycleRecord& row : report.rows) {
        out << row.cycle << ',' << row.work_units << ',' << format_double(row.residual) << ','
            << format_double(row.diag_min) << ',';
        if (row.l1_error) out << format_double(*row.l1_error);
        out << '\n';
    }
    close_out(out, path);
}

void write_trace_csv(const SolveReport& report, const std::string& path) {
    std::ofstream out = open_out(path);
    out << "cycle,pass,level,diag_residual\n";
    for (const DiagSample& s : report.trace)
        out << s.cycle << ',' << s.pass << ',' << s.level << ',' << format_double(s.value) << '\n';
    close_out(out, path);
}

namespace {

// one number filling the whole cell (surrounding blanks allowed)
bool parse_cell(const std::string& cell, double& out) {
    std::size_t b = 0, e = cell.size();
    while (b < e && std::isspace(static_cast<unsigned char>(cell[b]))) ++b;
    while (e > b && std::isspace(static_cast<unsigned char>(cell[e - 1]))) --e;
    if (b == e) return false;
    try {
        std::size_t used = 0;
        out = std::stod(cell.substr(b, e - b), &used);
        return used == e - b;
    } catch (const std::exception&) {
        return false;
    }
}

}  // namespace

std::vector<Point> read_points_csv(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw io_error("cannot open: " + path);
    std::vector<Point> pts;
    std::string line;
    for (std::size_t lineno = 1; std::getline(in, line); ++lineno) {
        while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
        if (line.empty()) continue;
        // cells as std::getline(row, cell, ',') yields them: a trailing comma
        // ends the row without an empty last cell
        std::vector<std::string> cells;
        std::size_t start = 0;
        for (std::size_t pos; (pos = line.find(',', start)) != std::string::npos; start = pos + 1)
            cells.push_back(line.substr(start, pos - start));
        if (start < line.size()) cells.push_back(line.substr(start));
        double v[3] = {0.0, 0.0, 0.0};
        const bool first_numeric = !cells.empty() && parse_cell(cells[0], v[0]);
        // a header is a first line whose first cell is not a number
        if (lineno == 1 && !first_numeric) continue;
        bool ok = first_numeric && cells.size() >= 2 && cells.size() <= 3;
        for (std::size_t c = 1; ok && c < cells.size(); ++c) ok = parse_cell(cells[c], v[c]);
        if (!ok) throw io_error(path + ": malformed row " + std::to_string(lineno));
        pts.push_back({v[0], v[1], v[2]});
    }
    return pts;
}

void write_points_csv(const std::vector<Point>& pts, int dim, const std::string& path) {
    std::ofstream out = open_out(path);
    out << (dim == 3 ? "x,y,z\n" : "x,y\n");
    for (const Point& p : pts) {
        out << format_double(p[0]) << ',' << format_double(p[1]);
        if (dim == 3) out << ',' << format_double(p[2]);
        out << '\n';
    }
    close_out(out, path);
}

}  // namespace sgml
