// fields.cu — the post-solve operators of the reference's experiments
// (problems.cpp:74-97, 327-455): second-order difference fields (axis
// derivative, gradient, curl, divergence), the deformation velocity, node
// motion by forward Euler on multilinear samples, and RK4 streamlines.
//
// These consume the DENSE x-fastest fields of the public API (Field layout,
// grid.hpp:78-119).  Every expression keeps the reference's operation order
// and the build has no multiply-add contraction (--fmad=false), so results
// are the reference's bits (sqrt and division are IEEE correctly rounded on
// both sides; floor and clamp are exact).
//
// The difference kernels are streaming passes (HBM-bound): one thread per
// node, (32 x 4) blocks over (x, y), one plane per blockIdx.z, the +-1 / +-2
// neighbour reads served by L1 / L2.  The fused curl reads each potential
// component once and writes the three velocity components (48 B per node).
// move_nodes runs one thread per node through all Euler steps (gathers from
// L2-resident neighbourhoods); streamlines run one thread per seed.
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"

namespace sgmlb {

namespace {

// problems.cpp:74-97 (axis_derivative), for the node at coordinate c along
// an axis of stride s
__device__ __forceinline__ double daxis(const double* __restrict__ u, size_t p, ptrdiff_t s, int c, int N,
                                        double inv2h) {
    double v;
    if (c == 0)
        v = (-3.0 * u[p] + 4.0 * u[p + s] - u[p + 2 * s]) * inv2h;
    else if (c == N - 1)
        v = (3.0 * u[p] - 4.0 * u[p - s] + u[p - 2 * s]) * inv2h;
    else
        v = (u[p + s] - u[p - s]) * inv2h;
    return v;
}

struct Node {
    int i, j, k;
    size_t p;
    bool ok;
};

template <int DIM>
__device__ __forceinline__ Node node_here(int N) {
    Node n;
    n.i = blockIdx.x * 32 + threadIdx.x;
    n.j = blockIdx.y * 4 + threadIdx.y;
    n.k = DIM == 3 ? (int)blockIdx.z : 0;
    n.ok = n.i < N && n.j < N;
    n.p = (size_t)n.i + (size_t)N * ((size_t)n.j + (size_t)N * (size_t)n.k);
    return n;
}

__device__ __forceinline__ ptrdiff_t stride_of(int axis, int N) {
    return axis == 0 ? 1 : (axis == 1 ? (ptrdiff_t)N : (ptrdiff_t)N * N);
}

template <int DIM>
__global__ void __launch_bounds__(128) k_axis_derivative(const double* __restrict__ u, double* __restrict__ d,
                                                         int N, int axis, double inv2h) {
    const Node n = node_here<DIM>(N);
    if (!n.ok) return;
    const int c = axis == 0 ? n.i : (axis == 1 ? n.j : n.k);
    d[n.p] = daxis(u, n.p, stride_of(axis, N), c, N, inv2h);
}

// gradient (problems.cpp:391-396) with deformation_velocity's scaling
// (problems.cpp:327-341) when f_raw is given: comp = -comp / (t f_raw + I);
// a zero denominator raises flag[0]
template <int DIM>
__global__ void __launch_bounds__(128) k_gradient(const double* __restrict__ u, double* __restrict__ g0,
                                                  double* __restrict__ g1, double* __restrict__ g2, int N,
                                                  double inv2h, const double* __restrict__ f_raw, double raw_integral,
                                                  double t, int* flag) {
    const Node n = node_here<DIM>(N);
    if (!n.ok) return;
    double g[3];
    g[0] = daxis(u, n.p, 1, n.i, N, inv2h);
    g[1] = daxis(u, n.p, N, n.j, N, inv2h);
    if (DIM == 3) g[2] = daxis(u, n.p, (ptrdiff_t)N * N, n.k, N, inv2h);
    if (f_raw) {
        const double den = t * f_raw[n.p] + raw_integral;
        if (den == 0.0) atomicOr(flag, 1);
#pragma unroll
        for (int c = 0; c < DIM; ++c) g[c] = -g[c] / den;
    }
    g0[n.p] = g[0];
    g1[n.p] = g[1];
    if (DIM == 3) g2[n.p] = g[2];
}

// curl (problems.cpp:376-389): v = (dzy - dyz, dxz - dzx, dyx - dxy) with
// dab = d psi_a / d b
__global__ void __launch_bounds__(128) k_curl(const double* __restrict__ px, const double* __restrict__ py,
                                              const double* __restrict__ pz, double* __restrict__ vx,
                                              double* __restrict__ vy, double* __restrict__ vz, int N, double inv2h) {
    const Node n = node_here<3>(N);
    if (!n.ok) return;
    const ptrdiff_t sy = N, sz = (ptrdiff_t)N * N;
    const double dzy = daxis(pz, n.p, sy, n.j, N, inv2h);
    const double dyz = daxis(py, n.p, sz, n.k, N, inv2h);
    const double dxz = daxis(px, n.p, sz, n.k, N, inv2h);
    const double dzx = daxis(pz, n.p, 1, n.i, N, inv2h);
    const double dyx = daxis(py, n.p, 1, n.i, N, inv2h);
    const double dxy = daxis(px, n.p, sy, n.j, N, inv2h);
    vx[n.p] = dzy - dyz;
    vy[n.p] = dxz - dzx;
    vz[n.p] = dyx - dxy;
}

// divergence (problems.cpp:398-405): d = ((0 + d0) + d1) + d2
template <int DIM>
__global__ void __launch_bounds__(128) k_divergence(const double* __restrict__ v0, const double* __restrict__ v1,
                                                    const double* __restrict__ v2, double* __restrict__ d, int N,
                                                    double inv2h) {
    const Node n = node_here<DIM>(N);
    if (!n.ok) return;
    double acc = 0.0;
    acc = acc + daxis(v0, n.p, 1, n.i, N, inv2h);
    acc = acc + daxis(v1, n.p, N, n.j, N, inv2h);
    if (DIM == 3) acc = acc + daxis(v2, n.p, (ptrdiff_t)N * N, n.k, N, inv2h);
    d[n.p] = acc;
}

// std::clamp(v, lo, hi) for doubles: v < lo ? lo : (hi < v ? hi : v)
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// sample_scalar (problems.cpp:40-67): multilinear sample at a clamped point
template <int DIM>
__device__ double sample_scalar(const double* __restrict__ f, int N, double h, const double* x) {
    int idx[3] = {0, 0, 0};
    double frac[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const double xs = clampd(x[c], 0.0, 1.0) / h;
        int i0 = (int)floor(xs);
        i0 = i0 < 0 ? 0 : (N - 2 < i0 ? N - 2 : i0);
        idx[c] = i0;
        frac[c] = xs - i0;
    }
    const double wx[2] = {1.0 - frac[0], frac[0]};
    const double wy[2] = {1.0 - frac[1], frac[1]};
    double acc = 0.0;
    if (DIM == 2) {
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int a = 0; a < 2; ++a)
                acc += wx[a] * wy[b] * f[(size_t)(idx[0] + a) + (size_t)N * (size_t)(idx[1] + b)];
    } else {
        const double wz[2] = {1.0 - frac[2], frac[2]};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int a = 0; a < 2; ++a)
                    acc += wx[a] * wy[b] * wz[c] *
                           f[(size_t)(idx[0] + a) +
                             (size_t)N * ((size_t)(idx[1] + b) + (size_t)N * (size_t)(idx[2] + c))];
    }
    return acc;
}

// move_nodes (problems.cpp:343-372): one thread per node, all Euler steps;
// the components update in order (c = 1 samples at the moved x[0])
template <int DIM>
__global__ void __launch_bounds__(128) k_move_nodes(const double* __restrict__ g0, const double* __restrict__ g1,
                                                    const double* __restrict__ g2, const double* __restrict__ f_raw,
                                                    double raw_integral, int N, double h, double t, int steps,
                                                    double* __restrict__ px, double* __restrict__ py,
                                                    double* __restrict__ pz) {
    const Node n = node_here<DIM>(N);
    if (!n.ok) return;
    double x[3] = {n.i * h, n.j * h, DIM == 3 ? n.k * h : 0.0};
    const double* gc[3] = {g0, g1, g2};
    const double dt = t / steps;
    for (int s = 0; s < steps; ++s) {
        const double tau = s * dt;
        const double den = tau * sample_scalar<DIM>(f_raw, N, h, x) + raw_integral;
        if (den == 0.0) continue;  // stationary where the density is singular
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            const double gv = sample_scalar<DIM>(gc[c], N, h, x);
            x[c] = clampd(x[c] - dt * gv / den, 0.0, 1.0);
        }
    }
    px[n.p] = x[0];
    py[n.p] = x[1];
    if (pz) pz[n.p] = x[2];
}

// problems.cpp:26-28, 140-146
__device__ __forceinline__ double norm3(const double* a) {
    return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
}
template <int DIM>
__device__ __forceinline__ bool inside_unit(const double* p) {
#pragma unroll
    for (int c = 0; c < DIM; ++c)
        if (!(p[c] >= 0.0 && p[c] <= 1.0)) return false;
    return true;
}
template <int DIM>
__device__ __forceinline__ void sample_vector(const double* const* v, int N, double h, const double* p, double* out) {
    out[0] = out[1] = out[2] = 0.0;
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = sample_scalar<DIM>(v[c], N, h, p);
}

// integrate_streamline (problems.cpp:415-455): one thread per seed; points
// [seed][step][3], count and stop (0 max_steps, 1 left_domain, 2 stagnation)
template <int DIM>
__global__ void k_streamlines(const double* __restrict__ v0, const double* __restrict__ v1,
                              const double* __restrict__ v2, int N, double h, const double* __restrict__ seeds,
                              int nseeds, double step, int max_steps, double* __restrict__ pts, int* counts,
                              int* stops) {
    const int sd = blockIdx.x * blockDim.x + threadIdx.x;
    if (sd >= nseeds) return;
    const double* v[3] = {v0, v1, v2};
    double* out = pts + (size_t)sd * (size_t)(max_steps + 1) * 3;
    double p[3] = {seeds[3 * sd], seeds[3 * sd + 1], seeds[3 * sd + 2]};
    int cnt = 0;
    auto push = [&](const double* q) {
        out[3 * cnt] = q[0];
        out[3 * cnt + 1] = q[1];
        out[3 * cnt + 2] = q[2];
        ++cnt;
    };
    push(p);
    int stop = 0;
    if (!inside_unit<DIM>(p)) {
        stop = 1;
    } else {
        for (int s = 0; s < max_steps; ++s) {
            double k1[3], k2[3], k3[3], k4[3], q[3];
            sample_vector<DIM>(v, N, h, p, k1);
            if (norm3(k1) < 1e-12) {
                stop = 2;
                break;
            }
            const double hs = 0.5 * step;
            for (int c = 0; c < 3; ++c) q[c] = p[c] + hs * k1[c];
            if (!inside_unit<DIM>(q)) { stop = 1; break; }
            sample_vector<DIM>(v, N, h, q, k2);
            for (int c = 0; c < 3; ++c) q[c] = p[c] + hs * k2[c];
            if (!inside_unit<DIM>(q)) { stop = 1; break; }
            sample_vector<DIM>(v, N, h, q, k3);
            for (int c = 0; c < 3; ++c) q[c] = p[c] + step * k3[c];
            if (!inside_unit<DIM>(q)) { stop = 1; break; }
            sample_vector<DIM>(v, N, h, q, k4);
            double nx[3] = {p[0], p[1], p[2]};
            for (int c = 0; c < 3; ++c) nx[c] += step / 6.0 * (k1[c] + 2.0 * k2[c] + 2.0 * k3[c] + k4[c]);
            if (!inside_unit<DIM>(nx)) { stop = 1; break; }
            p[0] = nx[0];
            p[1] = nx[1];
            p[2] = nx[2];
            push(p);
        }
    }
    counts[sd] = cnt;
    stops[sd] = stop;
}

// sample_vector at host-given points (problems.cpp:407-413)
template <int DIM>
__global__ void k_sample_points(const double* __restrict__ v0, const double* __restrict__ v1,
                                const double* __restrict__ v2, int nv, int N, double h,
                                const double* __restrict__ pts, int count, double* __restrict__ out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const double* v[3] = {v0, v1, v2};
    double o[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < nv; ++c) o[c] = sample_scalar<DIM>(v[c], N, h, pts + 3 * q);
    out[3 * q] = o[0];
    out[3 * q + 1] = o[1];
    out[3 * q + 2] = o[2];
}

dim3 node_grid(int dim, int N) { return dim3((N + 31) / 32, (N + 3) / 4, dim == 3 ? N : 1); }

}  // namespace

void launch_axis_derivative(int dim, const double* u, double* d, int N, int axis, double inv2h, cudaStream_t s) {
    if (dim == 2) k_axis_derivative<2><<<node_grid(2, N), dim3(32, 4), 0, s>>>(u, d, N, axis, inv2h);
    else k_axis_derivative<3><<<node_grid(3, N), dim3(32, 4), 0, s>>>(u, d, N, axis, inv2h);
}

void launch_gradient(int dim, const double* u, double* const* g, int N, double inv2h, const double* f_raw,
                     double raw_integral, double t, int* flag, cudaStream_t s) {
    if (dim == 2)
        k_gradient<2><<<node_grid(2, N), dim3(32, 4), 0, s>>>(u, g[0], g[1], nullptr, N, inv2h, f_raw,
                                                               raw_integral, t, flag);
    else
        k_gradient<3><<<node_grid(3, N), dim3(32, 4), 0, s>>>(u, g[0], g[1], g[2], N, inv2h, f_raw, raw_integral,
                                                               t, flag);
}

void launch_curl(const double* const* psi, double* const* v, int N, double inv2h, cudaStream_t s) {
    k_curl<<<node_grid(3, N), dim3(32, 4), 0, s>>>(psi[0], psi[1], psi[2], v[0], v[1], v[2], N, inv2h);
}

void launch_divergence(int dim, const double* const* v, double* d, int N, double inv2h, cudaStream_t s) {
    if (dim == 2) k_divergence<2><<<node_grid(2, N), dim3(32, 4), 0, s>>>(v[0], v[1], nullptr, d, N, inv2h);
    else k_divergence<3><<<node_grid(3, N), dim3(32, 4), 0, s>>>(v[0], v[1], v[2], d, N, inv2h);
}

void launch_move_nodes(int dim, const double* const* g, const double* f_raw, double raw_integral, int N, double h,
                       double t, int steps, double* const* pos, cudaStream_t s) {
    if (dim == 2)
        k_move_nodes<2><<<node_grid(2, N), dim3(32, 4), 0, s>>>(g[0], g[1], nullptr, f_raw, raw_integral, N, h, t,
                                                                 steps, pos[0], pos[1], pos[2]);
    else
        k_move_nodes<3><<<node_grid(3, N), dim3(32, 4), 0, s>>>(g[0], g[1], g[2], f_raw, raw_integral, N, h, t,
                                                                 steps, pos[0], pos[1], pos[2]);
}

void launch_streamlines(int dim, const double* const* v, int N, double h, const double* seeds, int nseeds,
                        double step, int max_steps, double* pts, int* counts, int* stops, cudaStream_t s) {
    const int nb = (nseeds + 63) / 64;
    if (dim == 2)
        k_streamlines<2><<<nb, 64, 0, s>>>(v[0], v[1], nullptr, N, h, seeds, nseeds, step, max_steps, pts, counts,
                                           stops);
    else
        k_streamlines<3><<<nb, 64, 0, s>>>(v[0], v[1], v[2], N, h, seeds, nseeds, step, max_steps, pts, counts,
                                           stops);
}

void launch_sample_points(int dim, const double* const* v, int nv, int N, double h, const double* pts, int count,
                          double* out, cudaStream_t s) {
    const int nb = (count + 127) / 128;
    if (dim == 2)
        k_sample_points<2><<<nb, 128, 0, s>>>(v[0], nv > 1 ? v[1] : nullptr, nullptr, nv, N, h, pts, count, out);
    else
        k_sample_points<3><<<nb, 128, 0, s>>>(v[0], nv > 1 ? v[1] : nullptr, nv > 2 ? v[2] : nullptr, nv, N, h,
                                              pts, count, out);
}

}  // namespace sgmlb

// ---------------------------------------------------------------------------
// Problem builders on the device.  The reference's
// closed forms call libm (sin, tanh) per node, which a device cannot
// reproduce bit for bit; but their arguments take few distinct values: sin
// depends on one coordinate (N values per axis), the capacitor's tanh on
// r^2 = m h^2 with the integer m = di^2 + dj^2 + dk^2 (every step of
// sq(i h - 0.5) + ... is exact for dyadic h).  The host evaluates those
// values with the host libm (the reference's bits), the device assembles
// the field with the reference's arithmetic order.
// ---------------------------------------------------------------------------

namespace sgmlb {
namespace {

// problems.cpp:178-193: f = (-3 pi pi) ((s_i s_j) s_k), s_t = sin(pi t h)
__global__ void __launch_bounds__(128) k_fill_poisson3d(double* __restrict__ f, int N,
                                                        const double* __restrict__ s, double scale) {
    const Node n = node_here<3>(N);
    if (!n.ok) return;
    f[n.p] = scale * ((s[n.i] * s[n.j]) * s[n.k]);
}

// C1 config (oracle og_fill_sinsin2d): f = ((-2 pi pi) s_i) s_j
__global__ void __launch_bounds__(128) k_fill_sinsin2d(double* __restrict__ f, int N,
                                                       const double* __restrict__ s, double scale) {
    const Node n = node_here<2>(N);
    if (!n.ok) return;
    f[n.p] = (scale * s[n.i]) * s[n.j];
}

// problems.cpp:160-176: f = -(P''(x) P(y) + P(x) P''(y)), P(t) = t^2 - t^4
__global__ void __launch_bounds__(128) k_fill_poisson2d(double* __restrict__ f, int N, double h) {
    const Node n = node_here<2>(N);
    if (!n.ok) return;
    const double x = n.i * h, y = n.j * h;
    const double px = x * x - x * x * x * x, py = y * y - y * y * y * y;
    const double dx = 2.0 - 12.0 * x * x, dy = 2.0 - 12.0 * y * y;
    f[n.p] = -(dx * py + px * dy);
}

// problems.cpp:509-515: sigma = table[m], m = di^2 + dj^2 + dk^2, d = i - (N-1)/2
__global__ void __launch_bounds__(128) k_fill_radial(double* __restrict__ f, int N,
                                                     const double* __restrict__ table) {
    const Node n = node_here<3>(N);
    if (!n.ok) return;
    const int c = (N - 1) / 2;
    const int di = n.i - c, dj = n.j - c, dk = n.k - c;
    f[n.p] = table[di * di + dj * dj + dk * dk];
}

// sparse contributions (unique nodes) into a zeroed field
__global__ void k_scatter_pairs(double* __restrict__ f, const unsigned long long* __restrict__ idx,
                                const double* __restrict__ val, int count) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < count) f[idx[q]] = val[q];
}

}  // namespace

void launch_fill_poisson3d(double* f, int N, const double* s, double scale, cudaStream_t st) {
    k_fill_poisson3d<<<node_grid(3, N), dim3(32, 4), 0, st>>>(f, N, s, scale);
}
void launch_fill_sinsin2d(double* f, int N, const double* s, double scale, cudaStream_t st) {
    k_fill_sinsin2d<<<node_grid(2, N), dim3(32, 4), 0, st>>>(f, N, s, scale);
}
void launch_fill_poisson2d(double* f, int N, double h, cudaStream_t st) {
    k_fill_poisson2d<<<node_grid(2, N), dim3(32, 4), 0, st>>>(f, N, h);
}
void launch_fill_radial(double* f, int N, const double* table, cudaStream_t st) {
    k_fill_radial<<<node_grid(3, N), dim3(32, 4), 0, st>>>(f, N, table);
}
void launch_scatter_pairs(double* f, const unsigned long long* idx, const double* val, int count, cudaStream_t st) {
    if (count > 0) k_scatter_pairs<<<(count + 255) / 256, 256, 0, st>>>(f, idx, val, count);
}

}  // namespace sgmlb
