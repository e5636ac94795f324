// sgml_b200_cli.cpp — command-line driver over the B200 solve path, the
// counterpart of the reference CLI's solve-driving subcommands
// (proj/tools/sgml_main.cpp:84-94 convergence, :166-178 capacitor,
// :184-221 bench) plus `poisson3d`, the benchmark problem.
//
// The problems are built on the host with the reference's closed forms
// (problems.cpp:160-193, 500-521) so the inputs are the reference's bits;
// every solve and every timed cycle runs on the device through the drop-in
// C++ API (include/sgml/*.hpp -> libsgml_b200.so).  Outputs use the
// reference's file formats (io.cpp:35-120: %.17g, report.csv, trace.csv,
// legacy ASCII VTK, bench.csv).  Exit codes as the reference: 0 success,
// 2 reported non-convergence, 1 input errors.
//
// Not here (off the solve path): deform (curve deposition,
// node motion) and trifoil (vortex-filament sources, curl, streamlines),
// and the gradient output F.vtk of capacitor.
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

#include "sgml/cycle.hpp"
#include "sgml/grid.hpp"

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
    std::ofstream out = open_out(path);
    const sgml::Grid& g = f.grid();
    out << "# vtk DataFile Version 3.0\n" << name << "\nASCII\nDATASET STRUCTURED_POINTS\n"
        << "DIMENSIONS " << g.N << ' ' << g.N << ' ' << (g.dim == 3 ? g.N : 1) << '\n'
        << "ORIGIN 0 0 0\n"
        << "SPACING " << fmt(g.h) << ' ' << fmt(g.h) << ' ' << (g.dim == 3 ? fmt(g.h) : std::string("1")) << '\n'
        << "POINT_DATA " << g.total << '\n'
        << "SCALARS " << name << " double 1\nLOOKUP_TABLE default\n";
    for (std::size_t p = 0; p < f.size(); ++p) out << fmt(f[p]) << '\n';
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
    std::cerr << "usage: sgml_b200 {convergence|poisson3d|capacitor|bench} [--n N] [--nr R] [--tol T]\n"
                 "       [--max-cycles C] [--safety S] [--out DIR] [--mode high|low] [--no-vtk]\n";
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
            else throw std::invalid_argument("unknown option " + a);
        }
        if (cfg.n_r < 1 || !(cfg.tol > 0.0) || cfg.max_cycles < 1)
            throw std::invalid_argument("--nr, --tol and --max-cycles must be positive");
        if (cmd == "convergence") return solve_and_write("convergence", poisson2d(cfg.n), cfg, vtk);
        if (cmd == "poisson3d") return solve_and_write("poisson3d", poisson3d(cfg.n), cfg, vtk);
        if (cmd == "capacitor") return solve_and_write("capacitor", capacitor(cfg.n, cfg.mode), cfg, vtk);
        if (cmd == "bench") return cmd_bench(cfg);
        usage();
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
