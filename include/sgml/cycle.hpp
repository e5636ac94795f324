// sgml/cycle.hpp — schedule, configuration, report types and the solve driver,
// drop-in for the reference header (proj/core/include/sgml/cycle.hpp).
//
// solve() runs the whole residual-recurrence solve on the B200 (level-compact
// engine); the report (rows, trace, flags, normalization,
// node_updates) is identical to the reference's for the same inputs.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <vector>

#include "sgml/grid.hpp"
#include "sgml/kernels.hpp"

namespace sgml {

struct ScheduleStep {
    enum class Kind : std::uint8_t { restrict_source, relax };
    Kind kind = Kind::relax;
    int level = 0;
    int count = 1;
};

struct CycleSchedule {
    int n = 0;
    int n_r = 1;
    std::vector<ScheduleStep> steps;
};

CycleSchedule build_schedule(int n, int n_r);
std::uint64_t closed_form_work_units(int n, int n_r);
std::uint64_t schedule_work_units(const CycleSchedule& schedule);

struct SolverConfig {
    int n_r = 2;
    double tol = 1e-12;
    int max_cycles = 50;
    double safety = 0.9;
};

struct DiagSample {
    int cycle = 0;
    int pass = 0;
    int level = 0;
    double value = 0.0;
};

struct CycleRecord {
    int cycle = 0;
    std::uint64_t work_units = 0;
    double residual = 0.0;
    double diag_min = 0.0;
    std::optional<double> l1_error;
};

struct SolveReport {
    std::vector<CycleRecord> rows;
    std::vector<DiagSample> trace;
    bool converged = false;
    bool nan_detected = false;
    bool stagnated = false;
    double normalization = 0.0;
    std::uint64_t node_updates = 0;
};

using ExactSolution = std::function<double(double x, double y, double z)>;

struct ProblemSpec {
    Grid grid;
    Field sigma;  // empty: sigma == 1
    double a = 0.0;
    Field f;
    BoundarySpec bc;
    ExactSolution exact;  // optional: enables the l1_error column
    const Field* sigma_or_null() const { return sigma.size() ? &sigma : nullptr; }
};

struct SolveResult {
    Field u;
    SolveReport report;
};

// One cycle from the zero state (state.u receives the correction).
void single_cycle(SolveState& state, const Field& source, const std::vector<Field>& sigma_levels, double a,
                  const BoundarySpec& bc, bool homogeneous, const CycleSchedule& schedule, double safety,
                  int cycle_index, double normalization, SolveReport& report, std::uint64_t& work_units);

SolveResult solve(const ProblemSpec& problem, const SolverConfig& config);
void pure_neumann_pin(Field& u);
std::vector<Field> restrict_sigma_levels(const Field& sigma, int n);

// (l1_error, the l1_error column's quadrature, is declared in sgml/problems.hpp
// as in the reference.)

}  // namespace sgml
