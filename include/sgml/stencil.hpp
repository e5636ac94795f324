// sgml/stencil.hpp — pointwise constants of the radial operator, drop-in for
// the reference header (proj/core/include/sgml/stencil.hpp).  The operator
// itself runs on the B200 inside the kernels; the host keeps the constants
// and the coefficient bundle that the kernel-level API takes.
#pragma once

#include <algorithm>
#include <cmath>

#include "sgml/grid.hpp"

namespace sgml {

// 1/2 in 2D (8 offsets), 3/13 in 3D (26 offsets): quadratics are exact.
constexpr double stencil_prefactor(int dim) { return dim == 2 ? 0.5 : 3.0 / 13.0; }
// Explicit pseudo-time bound dtau <= K_dim (lam h)^2 / sigma_bar_max.
constexpr double step_constant(int dim) { return dim == 2 ? 1.0 / 3.0 : 13.0 / 44.0; }
// Linear hat max(0, 1 - |x|).
inline double hat(double x) { return std::max(0.0, 1.0 - std::abs(x)); }
// Restriction weight along one axis: 1/2 centre, 1/4 neighbours.
inline double restrict_axis_weight(int o) { return o == 0 ? 0.5 : 0.25; }

struct OperatorCoefficients {
    const Field* sigma = nullptr;  // nullptr: sigma == 1
    double a = 0.0;
};

}  // namespace sgml
