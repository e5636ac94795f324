// sgml/kernels.hpp — the full-grid passes of the solve path, drop-in for the
// reference header (proj/core/include/sgml/kernels.hpp).  Each call runs the
// corresponding sm_100a kernel through the C-ABI (include/sgml_b200.h) on the
// calling thread's default device context; host Fields are copied in and out
// around the kernel.  Results are bit-identical to the reference CPU path
// (up to the sign of exact zeros).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <utility>

#include "sgml/grid.hpp"
#include "sgml/stencil.hpp"

namespace sgml {

// A kernel met a non-finite value or a non-positive pseudo-time step.
struct kernel_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Double-buffered pass state (reference kernels.hpp:49-72).
struct SolveState {
    Field u;
    Field u_prev;
    Field du;
    Field du_prev;
    int level = 0;

    explicit SolveState(const Grid& g) : u(g), u_prev(g), du(g), du_prev(g) {}
    void swap_buffers() {
        std::swap(u, u_prev);
        std::swap(du, du_prev);
    }
    void reset_level(int v) {
        level = v;
        du.fill(0.0);
        du_prev.fill(0.0);
    }
};

// v averaging passes with stride 1, 2, ..., 2^(v-1); v = 0 copies.  Adds v to *work.
Field restriction(const Field& f, int v, const BoundarySpec& bc, std::uint64_t* work = nullptr);
void restriction_into(const Field& f, int v, const BoundarySpec& bc, Field& out, Field& scratch,
                      std::uint64_t* work = nullptr);

// One relaxation-interpolation pass at state.level; returns the unnormalised
// diagnostic max.  Throws kernel_error on non-finite output or safety <= 0.
double relaxation_interpolation(SolveState& state, const Field& g, const Field* sigma_level, double a,
                                double safety, const BoundarySpec& bc, bool homogeneous,
                                std::uint64_t* work = nullptr);

Field residual(const Field& u, const Field& f, const OperatorCoefficients& coeff, const BoundarySpec& bc);
void residual_update(Field& r, const Field& e, const OperatorCoefficients& coeff, const BoundarySpec& bc);
void zero_mean_projection(Field& f);
double trapezoid_mean(const Field& f);
void apply_boundary(Field& u, const BoundarySpec& bc, bool homogeneous);
double max_abs(const Field& f);

}  // namespace sgml
