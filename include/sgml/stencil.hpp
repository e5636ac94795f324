// sgml/stencil.hpp — drop-in for the reference header
// (proj/core/include/sgml/stencil.hpp): the radial operator's offset table
// and constants, ghost-aware reads and the pointwise operations.
//
// The solve path never calls the pointwise functions: every pass of a solve
// runs the same arithmetic inside the sm_100a kernels (csrc/relax_tiled.cu,
// csrc/kernels.cu).  They are the reference's host utilities for single
// nodes (operator identities, ghost rules, stability bound), kept with the
// reference's semantics for callers and tests; the definitions are in
// libsgml_b200.so (csrc/sgml_cpp_more.cpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <span>

#include "sgml/grid.hpp"

namespace sgml {

// One nonzero neighbour offset of {-1, 0, 1}^dim with 1 / (p^2 + q^2 + r^2).
struct StencilOffset {
    int p = 0, q = 0, r = 0;
    double inv_l2 = 0.0;
};

// The 8 (2D) or 26 (3D) offsets in the order r = -1..1, q = -1..1, p = -1..1
// (stencil.cpp:13-25): the order every relaxation sums its terms in.
std::span<const StencilOffset> stencil_offsets(int dim);

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
    double a = 0.0;                // Helmholtz constant
};

namespace detail {

// u at signed coordinates that may lie outside the grid, resolved one axis
// at a time (x, then y, then z): Neumann faces mirror evenly, Dirichlet faces
// reflect oddly about the stored face value (2 u(face) - u(mirror)).
double ghost_value(const Field& u, const BoundarySpec& bc, int i, int j, int k);

// Even-mirror read whatever the faces are (the coefficient sigma).
double mirror_value(const Field& u, int i, int j, int k);

}  // namespace detail

// Weighted 9 / 27-point average of f around idx at spacing lam h (axis
// weights 1/2 centre, 1/4 neighbours), out-of-range neighbours per bc.
double restrict_at(const Field& f, const NodeIndex& idx, int lam, const BoundarySpec& bc);

// The radial div(sigma grad u) + a u at idx, spacing lam h; sigma face-averaged
// with even-mirrored neighbours (1 when coeff.sigma is null).
double apply_operator(const Field& u, const OperatorCoefficients& coeff, const NodeIndex& idx, int lam,
                      const BoundarySpec& bc);

// safety K_dim (lam h)^2 / max sigma; std::invalid_argument unless
// 0 < safety <= 1 and sigma > 0.
double stable_step(const OperatorCoefficients& coeff, const Grid& grid, int lam, double safety);

}  // namespace sgml
