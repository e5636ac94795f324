// sgml_b200_cli.cpp — command-line driver over the B200 solve path, the
// counterpart of the reference CLI's solve-driving subcommands
// (proj/tools/sgml_main.cpp:84-94 convergence, :166-178 capacitor,
// :184-221 bench) plus `poisson3d`, the benchmark problem.
//
// plus deform (:100-125) and trifoil (:131-164).
//
// The closed-form problems are built on the host with the reference's
// expressions (problems.cpp:160-193, 500-521) and the curve problems by the
// library's builders (problems.cpp:302-325, 374-398; libm on the host, fields
// on the device), so the inputs are the reference's bits; every solve,
// every timed cycle and every post-solve field
// (gradient, curl, node motion, streamlines) runs on the device through the
// drop-in C++ API (include/sgml/*.hpp -> libsgml_b200.so).  Outputs use the
// reference's file formats (io.cpp:35-178: %.17g, report.csv, trace.csv,
// legacy ASCII VTK, points CSV, bench.csv).  Exit codes as the reference:
// 0 success, 2 reported non-convergence, 1 input errors.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <numbers>
#include <stdexcept>
#include <string>

#include <sstream>
#include <vector>

#include "sgml/cycle.hpp"
#include "sgml/grid.hpp"
#include "sgml/kernels.hpp"
#include "sgml/problems.hpp"
#include "sgml_b200.h"

namespace {

constexpr double kPi = std::numbers::pi_v<double>;

struct RunConfig {
    int n = 7;
    int n_r = 2;
    double tol = 1e-12;
    int max_cycles = 50;
    double safety = 0.9;
    std::string mode = "high";
    std::string out = ".";
    double a = 0.1;
    double r = 0.14;
    std::string curve_path;
    std::string seeds_path;
    double t = 0.0;  // 0 = per-command default
    int steps = 0;   // 0 = per-command default
};

std::string fmt(double x) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.17g", x);
    return buf;
}

std::string join(const std::string& dir, const std::string& name) {
    return (std::filesystem::path(dir) / name).string();
}

sgml::SolverConfig solver_config(const RunConfig& c) {
    sgml::SolverConfig s;
    s.n_r = c.n_r;
    s.tol = c.tol;
    s.max_cycles = c.max_cycles;
    s.safety = c.safety;
    return s;
}

// ---- problems (the reference's closed forms, host evaluation) -------------

// u = -P(x) P(y), P(t) = t^2 - t^4 (problems.cpp:160-176)
sgml::ProblemSpec poisson2d(int n) {
    sgml::ProblemSpec p;
    p.grid = sgml::make_grid(2, n);
    p.f = sgml::Field(p.grid);
    p.bc = sgml::BoundarySpec::all_dirichlet(0.0);
    auto P = [](double t) { return t * t - t * t * t * t; };
    auto Pdd = [](double t) { return 2.0 - 12.0 * t * t; };
    p.exact = [P](double x, double y, double) { return -P(x) * P(y); };
    const double h = p.grid.h;
    for (int j = 0; j < p.grid.N; ++j)
        for (int i = 0; i < p.grid.N; ++i) {
            const double x = i * h, y = j * h;
            p.f.at(i, j) = -(Pdd(x) * P(y) + P(x) * Pdd(y));
        }
    return p;
}

// u = sin(pi x) sin(pi y) sin(pi z) (problems.cpp:178-193)
sgml::ProblemSpec poisson3d(int n) {
    sgml::ProblemSpec p;
    p.grid = sgml::make_grid(3, n);
    p.f = sgml::Field(p.grid);
    p.bc = sgml::BoundarySpec::all_dirichlet(0.0);
    p.exact = [](double x, double y, double z) {
        return std::sin(kPi * x) * std::sin(kPi * y) * std::sin(kPi * z);
    };
    const double h = p.grid.h;
    for (int k = 0; k < p.grid.N; ++k)
        for (int j = 0; j < p.grid.N; ++j)
            for (int i = 0; i < p.grid.N; ++i)
                p.f.at(i, j, k) = -3.0 * kPi * kPi * p.exact(i * h, j * h, k * h);
    return p;
}

// sphere of conductivity contrast between plates at z = 0, 1 (problems.cpp:500-521)
sgml::ProblemSpec capacitor(int n, const std::string& mode) {
    double sign;
    if (mode == "low") sign = 1.0;
    else if (mode == "high") sign = -1.0;
    else throw std::invalid_argument("capacitor_problem: mode must be \"high\" or \"low\"");
    sgml::ProblemSpec p;
    p.grid = sgml::make_grid(3, n);
    p.f = sgml::Field(p.grid);
    p.sigma = sgml::Field(p.grid);
    const double h = p.grid.h;
    auto sq = [](double v) { return v * v; };
    for (int k = 0; k < p.grid.N; ++k)
        for (int j = 0; j < p.grid.N; ++j)
            for (int i = 0; i < p.grid.N; ++i) {
                const double r = std::sqrt(sq(i * h - 0.5) + sq(j * h - 0.5) + sq(k * h - 0.5));
                p.sigma.at(i, j, k) = 0.55 + sign * 0.45 * std::tanh((r - 0.2) / 0.1);
            }
    p.bc = sgml::BoundarySpec::all_neumann();
    p.bc.face(2, 0) = {sgml::BcKind::dirichlet, -1.0};
    p.bc.face(2, 1) = {sgml::BcKind::dirichlet, +1.0};
    return p;
}


// ---- curve problems: the library's device builders (csrc/builders.cpp) ----
// deformation_problem / trifoil_problem (problems.cpp:302-325, 374-398): the
// curve work runs on the host inside the library, the fields are assembled on
// the device and copied into the host Fields the drop-in API takes.

void ck(int status) {
    if (status != SGML_OK) throw std::runtime_error(sgml_last_error());
}

sgml_ctx* builder_ctx() {
    static sgml_ctx* ctx = nullptr;
    if (!ctx) {
        const char* d = std::getenv("SGML_DEVICE");
        ck(sgml_ctx_create(d ? std::atoi(d) : 0, &ctx));
    }
    return ctx;
}

// a device field of the grid, freed on scope exit
struct DevField {
    sgml_field* f = nullptr;
    explicit DevField(const sgml::Grid& g) { ck(sgml_field_create(builder_ctx(), g.dim, g.n, &f)); }
    ~DevField() { sgml_field_destroy(f); }
    DevField(const DevField&) = delete;
    DevField& operator=(const DevField&) = delete;
    sgml::Field host(const sgml::Grid& g) const {
        sgml::Field h(g);
        ck(sgml_field_download(f, h.data()));
        return h;
    }
};

struct DeformationSetup {
    sgml::ProblemSpec problem;
    sgml::Field f_raw;
    double raw_integral = 0.0;
};

DeformationSetup deformation_problem(const std::vector<sgml::Point>& curve, double a, int n) {
    int dim = 2;
    for (const sgml::Point& p : curve)
        if (p[2] != 0.0) dim = 3;
    const sgml::Grid grid = sgml::make_grid(dim, n);
    std::vector<double> pts;
    for (const sgml::Point& p : curve) pts.insert(pts.end(), p.begin(), p.end());
    DevField f(grid), raw(grid);
    DeformationSetup setup;
    ck(sgml_build_deformation_sources(pts.data(), (int)curve.size(), f.f, raw.f, &setup.raw_integral));
    setup.problem.grid = grid;
    setup.problem.a = a;
    setup.problem.bc = sgml::BoundarySpec::all_neumann();
    setup.problem.f = f.host(grid);
    setup.f_raw = raw.host(grid);
    return setup;
}

struct TrifoilSetup {
    std::array<sgml::ProblemSpec, 3> psi;
};

TrifoilSetup trifoil_problem(int n, double r) {
    const sgml::Grid grid = sgml::make_grid(3, n);
    DevField f0(grid), f1(grid), f2(grid);
    sgml_field* fs[3] = {f0.f, f1.f, f2.f};
    ck(sgml_build_trifoil_sources(fs, r));
    TrifoilSetup setup;
    const DevField* src[3] = {&f0, &f1, &f2};
    for (int c = 0; c < 3; ++c) {
        sgml::ProblemSpec& prob = setup.psi[c];
        prob.grid = grid;
        prob.bc = sgml::BoundarySpec::all_dirichlet(0.0);
        prob.f = src[c]->host(grid);
    }
    return setup;
}

// io.cpp:126-166: x,y[,z] rows, optional non-numeric header line
std::vector<sgml::Point> read_points_csv(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open: " + path);
    std::vector<sgml::Point> pts;
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
        if (line.empty()) continue;
        std::istringstream row(line);
        sgml::Point p{0.0, 0.0, 0.0};
        std::string cell;
        std::size_t col = 0;
        bool numeric = true, first_cell_numeric = true;
        while (std::getline(row, cell, ',')) {
            if (col >= 3) { numeric = false; break; }
            try {
                std::size_t used = 0;
                p[col] = std::stod(cell, &used);
                while (used < cell.size() && std::isspace(static_cast<unsigned char>(cell[used]))) ++used;
                if (used != cell.size()) numeric = false;
            } catch (const std::exception&) {
                numeric = false;
            }
            if (!numeric) {
                if (col == 0) first_cell_numeric = false;
                break;
            }
            ++col;
        }
        if (lineno == 1 && !first_cell_numeric) continue;
        if (!numeric || col < 2) throw std::runtime_error(path + ": malformed row " + std::to_string(lineno));
        pts.push_back(p);
    }
    return pts;
}

// ---- outputs (io.cpp formats) ---------------------------------------------

std::ofstream open_out(const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    return out;
}

void write_report(const sgml::SolveReport& r, const std::string& path) {
    std::ofstream out = open_out(path);
    out << "cycle,work_units,residual,diag_residual_min,l1_error\n";
    for (const auto& row : r.rows) {
        out << row.cycle << ',' << row.work_units << ',' << fmt(row.residual) << ',' << fmt(row.diag_min) << ',';
        if (row.l1_error) out << fmt(*row.l1_error);
        out << '\n';
    }
}

void write_trace(const sgml::SolveReport& r, const std::string& path) {
    std::ofstream out = open_out(path);
    out << "cycle,pass,level,diag_residual\n";
    for (const auto& s : r.trace) out << s.cycle << ',' << s.pass << ',' << s.level << ',' << fmt(s.value) << '\n';
}

void write_vtk(const sgml::Field& f, const std::string& path, const std::string& name) {
    // io.cpp:45-53, formatted on all host threads (libsgml_b200's writer)
    const sgml::Grid& g = f.grid();
    const sgml_grid cg{g.dim, g.n, g.N, 0, g.h, (uint64_t)g.total};
    const double* comps[1] = {f.data()};
    if (sgml_write_vtk_host(comps, 1, &cg, path.c_str(), name.c_str()) != SGML_OK)
        throw std::runtime_error(sgml_last_error());
}

void write_vector_vtk(const sgml::VectorField& v, const std::string& path, const std::string& name) {
    // io.cpp:55-64
    const sgml::Grid& g = v.grid();
    const sgml_grid cg{g.dim, g.n, g.N, 0, g.h, (uint64_t)g.total};
    const double* comps[3] = {v.comp[0].data(), v.comp[1].data(), v.comp[2].size() ? v.comp[2].data() : nullptr};
    if (sgml_write_vtk_host(comps, 3, &cg, path.c_str(), name.c_str()) != SGML_OK)
        throw std::runtime_error(sgml_last_error());
}

void write_points_csv(const std::vector<sgml::Point>& pts, int dim, const std::string& path) {
    std::ofstream out = open_out(path);
    out << (dim == 3 ? "x,y,z\n" : "x,y\n");
    for (const sgml::Point& p : pts) {
        out << fmt(p[0]) << ',' << fmt(p[1]);
        if (dim == 3) out << ',' << fmt(p[2]);
        out << '\n';
    }
}

void summary(const char* label, const sgml::SolveReport& rep) {
    if (rep.rows.empty()) {
        std::cout << label << ": no cycles recorded\n";
        return;
    }
    const auto& last = rep.rows.back();
    std::cout << label << ": " << (rep.converged ? "converged" : "NOT converged") << " after " << rep.rows.size()
              << " cycle(s), residual " << fmt(last.residual) << ", work units " << last.work_units;
    if (last.l1_error) std::cout << ", l1 error " << fmt(*last.l1_error);
    std::cout << '\n';
    if (rep.nan_detected) std::cout << label << ": non-finite values detected\n";
    if (rep.stagnated) std::cout << label << ": residual stagnated\n";
}

int solve_and_write(const char* label, const sgml::ProblemSpec& prob, const RunConfig& cfg, bool vtk) {
    std::filesystem::create_directories(cfg.out);
    const auto t0 = std::chrono::steady_clock::now();
    const sgml::SolveResult res = sgml::solve(prob, solver_config(cfg));
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    write_report(res.report, join(cfg.out, "report.csv"));
    write_trace(res.report, join(cfg.out, "trace.csv"));
    if (vtk) write_vtk(res.u, join(cfg.out, "u.vtk"), "u");
    summary(label, res.report);
    std::cout << label << ": solve " << fmt(secs) << " s wall (H2D, device solve, D2H)\n";
    return res.report.converged ? 0 : 2;
}

// capacitor (sgml_main.cpp:166-178): the solve plus the force field F = grad u
int cmd_capacitor(const RunConfig& cfg, bool vtk) {
    std::filesystem::create_directories(cfg.out);
    const sgml::SolveResult res = sgml::solve(capacitor(cfg.n, cfg.mode), solver_config(cfg));
    write_report(res.report, join(cfg.out, "report.csv"));
    write_trace(res.report, join(cfg.out, "trace.csv"));
    if (vtk) {
        write_vtk(res.u, join(cfg.out, "u.vtk"), "u");
        write_vector_vtk(sgml::gradient(res.u), join(cfg.out, "F.vtk"), "F");
    }
    summary("capacitor", res.report);
    return res.report.converged ? 0 : 2;
}

// deform (sgml_main.cpp:100-125): potential of a closed curve, then node motion
int cmd_deform(const RunConfig& cfg, bool vtk) {
    if (cfg.curve_path.empty()) throw std::invalid_argument("deform: --curve PATH is required");
    std::filesystem::create_directories(cfg.out);
    const DeformationSetup setup = deformation_problem(read_points_csv(cfg.curve_path), cfg.a, cfg.n);
    const sgml::SolveResult res = sgml::solve(setup.problem, solver_config(cfg));
    write_report(res.report, join(cfg.out, "report.csv"));
    write_trace(res.report, join(cfg.out, "trace.csv"));
    if (vtk) write_vtk(res.u, join(cfg.out, "u.vtk"), "u");
    const double horizon = cfg.t > 0.0 ? cfg.t : 1.0;
    const int steps = cfg.steps > 0 ? cfg.steps : 50;
    const std::vector<sgml::Point> nodes = sgml::move_nodes(res.u, setup.f_raw, setup.raw_integral, horizon, steps);
    write_points_csv(nodes, setup.problem.grid.dim, join(cfg.out, "nodes.csv"));
    summary("deform", res.report);
    return res.report.converged ? 0 : 2;
}

// trifoil (sgml_main.cpp:131-164): three potential solves, v = curl psi, streamlines
int cmd_trifoil(const RunConfig& cfg, bool vtk) {
    std::filesystem::create_directories(cfg.out);
    const TrifoilSetup setup = trifoil_problem(cfg.n, cfg.r);
    sgml::VectorField psi(setup.psi[0].grid);
    bool converged = true;
    const char* report_names[3] = {"report.csv", "report_psi_y.csv", "report_psi_z.csv"};
    const char* trace_names[3] = {"trace.csv", "trace_psi_y.csv", "trace_psi_z.csv"};
    const char* labels[3] = {"psi_x", "psi_y", "psi_z"};
    for (int c = 0; c < 3; ++c) {
        const sgml::SolveResult res = sgml::solve(setup.psi[c], solver_config(cfg));
        write_report(res.report, join(cfg.out, report_names[c]));
        write_trace(res.report, join(cfg.out, trace_names[c]));
        summary(labels[c], res.report);
        converged = converged && res.report.converged;
        psi.comp[c] = res.u;
    }
    const sgml::VectorField v = sgml::curl(psi);
    if (vtk) {
        write_vector_vtk(psi, join(cfg.out, "psi.vtk"), "psi");
        write_vector_vtk(v, join(cfg.out, "v.vtk"), "velocity");
    }
    std::vector<sgml::Point> seeds;
    if (!cfg.seeds_path.empty()) seeds = read_points_csv(cfg.seeds_path);
    else seeds = {{0.5, 0.5, 0.5}, {0.35, 0.5, 0.5}};
    const double step = cfg.t > 0.0 ? cfg.t : 0.01;
    const int max_steps = cfg.steps > 0 ? cfg.steps : 2000;
    for (std::size_t s = 0; s < seeds.size(); ++s) {
        const sgml::Streamline line = sgml::integrate_streamline(v, seeds[s], step, max_steps);
        write_points_csv(line.points, 3, join(cfg.out, "streamline_" + std::to_string(s) + ".csv"));
    }
    return converged ? 0 : 2;
}

// single-cycle sweep over n_lo..n (sgml_main.cpp:184-221): one cycle per
// size on the device, timed on the host around the call
int cmd_bench(const RunConfig& cfg) {
    std::filesystem::create_directories(cfg.out);
    const int n_hi = cfg.n, n_lo = std::max(2, n_hi - 4);
    std::FILE* out = std::fopen(join(cfg.out, "bench.csv").c_str(), "w");
    if (!out) throw std::runtime_error("cannot open bench.csv for writing");
    std::fputs("n,nodes,work_units_per_cycle,seconds_per_cycle,node_updates_per_second\n", out);
    for (int n = n_lo; n <= n_hi; ++n) {
        const sgml::ProblemSpec prob = poisson2d(n);
        const sgml::CycleSchedule schedule = sgml::build_schedule(n, cfg.n_r);
        const std::uint64_t units = sgml::schedule_work_units(schedule);
        sgml::SolveState state(prob.grid);
        sgml::SolveReport scratch;
        std::uint64_t work = 0;
        // one untimed cycle builds the device engine of this shape
        sgml::single_cycle(state, prob.f, {}, prob.a, prob.bc, false, schedule, cfg.safety, 0, 1.0, scratch, work);
        scratch = sgml::SolveReport();
        work = 0;
        const auto t0 = std::chrono::steady_clock::now();
        sgml::single_cycle(state, prob.f, {}, prob.a, prob.bc, false, schedule, cfg.safety, 0, 1.0, scratch, work);
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (work != units) throw std::logic_error("bench: pass counter disagrees with the schedule");
        const double updates = (double)units * (double)prob.grid.total;
        std::fprintf(out, "%d,%zu,%llu,%s,%s\n", n, (size_t)prob.grid.total, (unsigned long long)units,
                     fmt(secs).c_str(), fmt(secs > 0.0 ? updates / secs : 0.0).c_str());
        std::cout << "bench n=" << n << ": " << units << " units, " << fmt(secs) << " s/cycle\n";
    }
    std::fclose(out);
    return 0;
}

void usage() {
    std::cerr << "usage: sgml_b200 {convergence|poisson3d|capacitor|deform|trifoil|bench} [--n N] [--nr R]\n"
                 "       [--tol T] [--max-cycles C] [--safety S] [--out DIR] [--mode high|low] [--no-vtk]\n"
                 "       deform: --curve PATH [--a A] [--t T] [--steps S]; trifoil: [--r R] [--seeds PATH]\n"
                 "       [--t STEP] [--steps S]\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 1;
    }
    const std::string cmd = argv[1];
    RunConfig cfg;
    bool vtk = true;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) throw std::invalid_argument("missing value for " + a);
                return argv[++i];
            };
            if (a == "--n") cfg.n = std::stoi(val());
            else if (a == "--nr") cfg.n_r = std::stoi(val());
            else if (a == "--tol") cfg.tol = std::stod(val());
            else if (a == "--max-cycles") cfg.max_cycles = std::stoi(val());
            else if (a == "--safety") cfg.safety = std::stod(val());
            else if (a == "--out") cfg.out = val();
            else if (a == "--mode") cfg.mode = val();
            else if (a == "--threads") (void)val();  // (OpenMP knob of the reference CLI)
            else if (a == "--no-vtk") vtk = false;
            else if (a == "--a") cfg.a = std::stod(val());
            else if (a == "--r") cfg.r = std::stod(val());
            else if (a == "--curve") cfg.curve_path = val();
            else if (a == "--seeds") cfg.seeds_path = val();
            else if (a == "--t") cfg.t = std::stod(val());
            else if (a == "--steps") cfg.steps = std::stoi(val());
            else throw std::invalid_argument("unknown option " + a);
        }
        if (cfg.n_r < 1 || !(cfg.tol > 0.0) || cfg.max_cycles < 1)
            throw std::invalid_argument("--nr, --tol and --max-cycles must be positive");
        if (cmd == "convergence") return solve_and_write("convergence", poisson2d(cfg.n), cfg, vtk);
        if (cmd == "poisson3d") return solve_and_write("poisson3d", poisson3d(cfg.n), cfg, vtk);
        if (cmd == "capacitor") return cmd_capacitor(cfg, vtk);
        if (cmd == "deform") return cmd_deform(cfg, vtk);
        if (cmd == "trifoil") return cmd_trifoil(cfg, vtk);
        if (cmd == "bench") return cmd_bench(cfg);
        usage();
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
