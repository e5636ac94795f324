// sgml/problems.hpp — drop-in for the reference header
// (proj/core/include/sgml/problems.hpp): the experiment builders (manufactured
// Poisson problems, curve resampling and delta deposition, grid deformation,
// the trifoil vortex, the heterogeneous capacitor) and the post-solve
// operators (difference fields, deformation velocity, node motion, RK4
// streamlines).
//
// Dense fields are assembled and every per-node operator runs on the B200
// (csrc/fields.cu, csrc/builders.cpp) through the C-ABI on the calling
// thread's default device context; host Fields are copied in and out around
// the kernels.  The libm calls (sin, tanh) run on the host over their few
// distinct arguments and the curve work (a few thousand samples) stays on
// the host, so every builder returns the reference's bits.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "sgml/cycle.hpp"
#include "sgml/grid.hpp"

namespace sgml {

using Point = std::array<double, 3>;  // z = 0 in 2D

// Ordered polyline in the unit domain; payload: empty or one vector per point.
struct Curve {
    std::vector<Point> points;
    std::vector<Point> payload;
    bool closed = false;
};

struct VectorField {
    std::array<Field, 3> comp;  // comp[2] unused in 2D
    int dim = 2;

    VectorField() = default;
    explicit VectorField(const Grid& g) : comp{Field(g), Field(g), Field(g)}, dim(g.dim) {}
    const Grid& grid() const { return comp[0].grid(); }
};

// ---- manufactured Poisson problems (problems.cpp:160-193) -------------------

// 2D, u = -x^2 y^2 (1 - x^2)(1 - y^2), f = laplacian(u), Dirichlet 0.
ProblemSpec poisson2d_problem(int n);
// 3D, u = sin(pi x) sin(pi y) sin(pi z), f = -3 pi^2 u, Dirichlet 0.
ProblemSpec poisson3d_problem(int n);

// Relative L1 error by trapezoid quadrature (serial Kahan, problems.cpp:195-215);
// std::invalid_argument without an exact solution or for an all-zero one.
double l1_error(const Field& v_h, const ExactSolution& exact);

// ---- curves and singular sources (problems.cpp:217-300) ---------------------

// Uniform arc-length resampling (intervals = round(length / h) >= 1, first
// point kept, closed curves wrap); a payload becomes the unit tangents.
// std::invalid_argument for < 2 points, h <= 0, zero length, degenerate tangents.
Curve resample_curve(const Curve& curve, double h);

// Hat-weight delta deposition of strength * (arc element) per sample, scaled
// by 1 / h^dim; std::invalid_argument for a sample outside the unit domain.
Field deposit_delta(const Curve& curve, const Grid& grid, double strength);

// payload[i] * (arc element) per sample into the 3 components.
VectorField deposit_delta_vector(const Curve& curve, const Grid& grid);

// ---- grid deformation (problems.cpp:302-372) --------------------------------

struct DeformationSetup {
    ProblemSpec problem;  // all-Neumann, sigma = 1, f = f_raw - mean(f_raw)
    Field f_raw;
    double raw_integral = 0.0;  // trapezoid integral of f_raw
};

DeformationSetup deformation_problem(const Curve& curve, double a, int n);

// v = -grad(u) / (t f_raw + raw_integral); std::invalid_argument on a zero denominator
VectorField deformation_velocity(const Field& u, const Field& f_raw, double raw_integral, double t);

// forward-Euler node motion from tau = 0 to t in `steps` increments; one position per node
std::vector<Point> move_nodes(const Field& u, const Field& f_raw, double raw_integral, double t, int steps);

// ---- knotted vortex flow (problems.cpp:374-455) -----------------------------

struct TrifoilSetup {
    std::array<ProblemSpec, 3> psi;  // laplacian(psi_c) = -omega_c, Dirichlet 0
    Curve curve;                     // resampled, unit-tangent payload
    VectorField omega;               // unit-circulation tangential vorticity
};

// std::invalid_argument for r <= 0 or a curve leaving the unit cube (3r >= 1/2)
TrifoilSetup trifoil_problem(int n, double r);

VectorField curl(const VectorField& psi);  // 3D only
VectorField gradient(const Field& u);
Field divergence(const VectorField& v);
Point sample_vector(const VectorField& v, const Point& p);

enum class StreamlineStop { max_steps, left_domain, stagnation };

struct Streamline {
    std::vector<Point> points;
    StreamlineStop stop = StreamlineStop::max_steps;
};

Streamline integrate_streamline(const VectorField& v, const Point& seed, double step, int max_steps);

// ---- heterogeneous capacitor (problems.cpp:500-521) -------------------------

// sigma = 0.55 +- 0.45 tanh((r - 0.2) / 0.1) ("low": +, "high": -), f = 0,
// z faces Dirichlet -1 / +1, lateral faces Neumann.
ProblemSpec capacitor_problem(int n, const std::string& mode);

}  // namespace sgml
