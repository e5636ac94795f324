// sgml/problems.hpp — the post-solve operators of the reference's experiments
// (proj/core/include/sgml/problems.hpp:21-39, 100-148), drop-in: difference
// fields, deformation velocity, node motion and RK4 streamlines.  Each call
// runs the sm_100a kernels of csrc/fields.cu through the C-ABI on the
// calling thread's default device context; host fields are copied in and
// out around the kernels.  Results are the reference's bits (up to the sign
// of exact zeros).  The problem builders (sources, curves, deposition) are
// not part of this header: their libm calls (sin, tanh) cannot reproduce the
// host library's bits on the device.
#pragma once

#include <array>
#include <vector>

#include "sgml/grid.hpp"

namespace sgml {

using Point = std::array<double, 3>;  // z = 0 in 2D

struct VectorField {
    std::array<Field, 3> comp;  // comp[2] unused in 2D
    int dim = 2;

    VectorField() = default;
    explicit VectorField(const Grid& g) : comp{Field(g), Field(g), Field(g)}, dim(g.dim) {}
    const Grid& grid() const { return comp[0].grid(); }
};

// v = -grad(u) / (t * f_raw + raw_integral); std::invalid_argument on a zero denominator
VectorField deformation_velocity(const Field& u, const Field& f_raw, double raw_integral, double t);

// forward-Euler node motion from tau = 0 to t in `steps` increments; one position per node
std::vector<Point> move_nodes(const Field& u, const Field& f_raw, double raw_integral, double t, int steps);

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

}  // namespace sgml
