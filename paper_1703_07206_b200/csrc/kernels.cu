// kernels.cu — sm_100a fp64 kernels of the SGML solve path.
//
// Literal kernels (full-grid, one node per thread) reproduce the
// reference's passes node for node and back the kernel-level C-ABI
// (restriction_into, relaxation_interpolation, residual_update).  The
// level-compact kernels (pyramid, compact relax, materialize) back the
// solve engine (engine.cu): every array they touch holds only level-v
// subset nodes, so coarse levels read and write dense, coalesced rows.
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"

namespace sgmlb {

namespace {

constexpr int BX = 32, BY = 4;

inline dim3 grid_for(int dim, int N) {
    return dim3((N + BX - 1) / BX, (N + BY - 1) / BY, dim == 3 ? N : 1);
}

// restrict weights {1/4, 1/2, 1/4} (kernels.cpp:22); products are exact.
__device__ __forceinline__ double axw(int o) { return o == 0 ? 0.5 : 0.25; }

// kernels.cpp:39-80 / stencil.cpp:98-119 at node (i,j,k) of an N-array,
// neighbours at +-lam.  Same products and order on both paths.
template <int DIM>
__device__ __forceinline__ double restrict_point(const double* __restrict__ in, int N, int lam,
                                                 int i, int j, int k, const BcDev& bc) {
    const bool fast = i >= lam && i <= N - 1 - lam && j >= lam && j <= N - 1 - lam &&
                      (DIM == 2 || (k >= lam && k <= N - 1 - lam));
    double acc = 0.0;
    if (fast) {
        const size_t pos = lin3(N, i, j, k);
        const ptrdiff_t sy = (ptrdiff_t)N * lam, sz = (ptrdiff_t)N * N * lam;
#pragma unroll
        for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
            for (int q = -1; q <= 1; ++q)
#pragma unroll
                for (int p = -1; p <= 1; ++p) {
                    const double w = DIM == 3 ? (axw(p) * axw(q)) * axw(r) : axw(p) * axw(q);
                    acc = acc + w * in[pos + r * sz + q * sy + p * lam];
                }
    } else {
#pragma unroll
        for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
            for (int q = -1; q <= 1; ++q)
#pragma unroll
                for (int p = -1; p <= 1; ++p) {
                    const double w = DIM == 3 ? (axw(p) * axw(q)) * axw(r) : axw(p) * axw(q);
                    acc = acc + w * ghost(in, N, bc, i + p * lam, j + q * lam, k + r * lam);
                }
    }
    return acc;
}

template <int DIM>
__global__ void __launch_bounds__(BX* BY) k_restrict_pass(const double* __restrict__ in,
                                                          double* __restrict__ out, int N, int lam,
                                                          BcDev bc) {
    const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y, k = blockIdx.z;
    if (i >= N || j >= N) return;
    out[lin3(N, i, j, k)] = restrict_point<DIM>(in, N, lam, i, j, k, bc);
}

// kernels.cpp:140-174 on a full-grid du_prev (corners at i0, i0 + lam);
// zero-weight corners are skipped, so the reference's out-of-row reads on
// non-Dirichlet high faces never happen here.
template <int DIM>
__device__ __forceinline__ double interp_full(const double* __restrict__ dup, int N, int lam,
                                              int i, int j, int k) {
    const int m = lam - 1;
    const double inv_lam = 1.0 / (double)lam;
    const int i0 = i & ~m, j0 = j & ~m, k0 = k & ~m;
    const double fx = (double)(i - i0) * inv_lam;
    const double fy = (double)(j - j0) * inv_lam;
    const double wx[2] = {1.0 - fx, fx};
    const double wy[2] = {1.0 - fy, fy};
    double acc = 0.0;
    if (DIM == 2) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                if (wy[q] == 0.0 || wx[p] == 0.0) continue;
                acc = acc + ((wy[q] * wx[p]) * dup[lin3(N, i0 + p * lam, j0 + q * lam, 0)]);
            }
    } else {
        const double fz = (double)(k - k0) * inv_lam;
        const double wz[2] = {1.0 - fz, fz};
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    if (wz[r] == 0.0 || wy[q] == 0.0 || wx[p] == 0.0) continue;
                    acc = acc + (((wz[r] * wy[q]) * wx[p]) *
                                 dup[lin3(N, i0 + p * lam, j0 + q * lam, k0 + r * lam)]);
                }
    }
    return acc;
}

template <int DIM, bool SIG>
__global__ void __launch_bounds__(BX* BY)
    k_relax_literal(double* __restrict__ u, double* __restrict__ du, const double* __restrict__ up,
                    const double* __restrict__ dup, const double* __restrict__ g,
                    const double* __restrict__ sig, int N, int level, RelaxConst rc, BcDev bc,
                    unsigned long long* diag_slot, int* flag, int pass_slot) {
    const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y, k = blockIdx.z;
    const int lam = 1 << level, mask = lam - 1;
    double diag = 0.0;
    int bad = 0;
    if (i < N && j < N) {
        const size_t pos = lin3(N, i, j, k);
        const bool on_face = i == 0 || i == N - 1 || j == 0 || j == N - 1 ||
                             (DIM == 3 && (k == 0 || k == N - 1));
        double value, duv;
        if (on_face && on_dirichlet<DIM>(bc, N, i, j, k)) {
            value = rc.homogeneous ? 0.0 : dirichlet_value<DIM>(bc, N, i, j, k);
            duv = value - up[pos];
        } else if (((i | j | k) & mask) == 0) {
            value = relax_at<DIM, SIG>(up, sig, g, N, lam, i, j, k, pos, rc, bc, diag);
            duv = value - up[pos];
        } else {
            value = up[pos] + interp_full<DIM>(dup, N, lam, i, j, k);
            duv = 0.0;
        }
        bad = !isfinite(value);
        u[pos] = value;
        du[pos] = duv;
    }
    block_max_commit(diag, diag_slot);
    block_bad_commit(bad, flag, pass_slot);
}

template <int DIM, bool SIG>
__global__ void __launch_bounds__(BX* BY)
    k_residual(double* __restrict__ r, const double* __restrict__ e, double* __restrict__ utot,
               const double* __restrict__ sig, int N, double inv_h2, double pref, double a,
               int has_a, BcDev bc, unsigned long long* rmax_slot, int compact) {
    const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y, k = blockIdx.z;
    double mx = 0.0;
    if (i < N && j < N) {
        const size_t pos = lin3(N, i, j, k);
        const double ec = e[pos];
        if (utot) utot[pos] = utot[pos] + ec;
        const double sc = SIG ? sig[pos] : 1.0;
        const bool fast = i >= 1 && i <= N - 2 && j >= 1 && j <= N - 2 &&
                          (DIM == 2 || (k >= 1 && k <= N - 2));
        double acc = 0.0;
        if (fast) {
            const ptrdiff_t sy = N, sz = (ptrdiff_t)N * N;
#pragma unroll
            for (int rr = (DIM == 3 ? -1 : 0); rr <= (DIM == 3 ? 1 : 0); ++rr)
#pragma unroll
                for (int q = -1; q <= 1; ++q)
#pragma unroll
                    for (int p = -1; p <= 1; ++p) {
                        if (p == 0 && q == 0 && rr == 0) continue;
                        if (stencil_skip(compact, p * p + q * q + rr * rr)) continue;
                        const ptrdiff_t d = rr * sz + q * sy + p;
                        const double sbar = SIG ? 0.5 * (sig[pos + d] + sc) : 1.0;
                        acc = stencil_term<SIG>(acc, sbar, e[pos + d], ec, p * p + q * q + rr * rr);
                    }
        } else {
#pragma unroll
            for (int rr = (DIM == 3 ? -1 : 0); rr <= (DIM == 3 ? 1 : 0); ++rr)
#pragma unroll
                for (int q = -1; q <= 1; ++q)
#pragma unroll
                    for (int p = -1; p <= 1; ++p) {
                        if (p == 0 && q == 0 && rr == 0) continue;
                        if (stencil_skip(compact, p * p + q * q + rr * rr)) continue;
                        const int ni = i + p, nj = j + q, nk = k + rr;
                        const double sbar = SIG ? 0.5 * (mirror(sig, N, ni, nj, nk) + sc) : 1.0;
                        acc = stencil_term<SIG>(acc, sbar, ghost(e, N, bc, ni, nj, nk), ec,
                                                p * p + q * q + rr * rr);
                    }
        }
        const double opv = (acc * pref) * inv_h2;
        double rn = r[pos] - (has_a ? opv + a * ec : opv);
        const bool on_face = i == 0 || i == N - 1 || j == 0 || j == N - 1 ||
                             (DIM == 3 && (k == 0 || k == N - 1));
        if (on_face && on_dirichlet<DIM>(bc, N, i, j, k)) rn = 0.0;
        r[pos] = rn;
        mx = fabs(rn);
    }
    if (rmax_slot) block_max_commit(mx, rmax_slot);
}

__global__ void k_max_abs(const double* __restrict__ f, uint64_t total, unsigned long long* slot) {
    double m = 0.0;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < total;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const double a = fabs(f[p]);
        m = m < a ? a : m;
    }
    block_max_commit(m, slot);
}

__global__ void k_fill(double* __restrict__ f, uint64_t total, double v) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < total; p += (uint64_t)gridDim.x * blockDim.x)
        f[p] = v;
}

__global__ void k_sub_scalar(double* __restrict__ f, uint64_t total, double v) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < total;
         p += (uint64_t)gridDim.x * blockDim.x)
        f[p] = f[p] - v;
}

__global__ void k_add_into(double* __restrict__ d, const double* __restrict__ s, uint64_t total) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < total;
         p += (uint64_t)gridDim.x * blockDim.x)
        d[p] = d[p] + s[p];
}

__global__ void k_check_positive(const double* __restrict__ f, uint64_t total, int* flag) {
    int bad = 0;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < total;
         p += (uint64_t)gridDim.x * blockDim.x)
        bad |= !(f[p] > 0.0);
    block_or_commit(bad, flag);
}

__global__ void k_check_finite(const double* __restrict__ f, uint64_t total, int* flag) {
    int bad = 0;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < total;
         p += (uint64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(f[p]);
    block_or_commit(bad, flag);
}

template <int DIM>
__global__ void __launch_bounds__(BX* BY)
    k_apply_boundary(double* __restrict__ u, int N, BcDev bc, int homogeneous) {
    const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y, k = blockIdx.z;
    if (i >= N || j >= N) return;
    if (on_dirichlet<DIM>(bc, N, i, j, k))
        u[lin3(N, i, j, k)] = homogeneous ? 0.0 : dirichlet_value<DIM>(bc, N, i, j, k);
}

inline int flat_blocks(uint64_t total) {
    const uint64_t b = (total + 255) / 256;
    return (int)(b < 148ull * 16 ? (b ? b : 1) : 148ull * 16);
}

}  // namespace

void launch_restrict_pass(int dim, const double* in, double* out, int N, int lam, const BcDev& bc,
                          cudaStream_t s) {
    if (dim == 2) k_restrict_pass<2><<<grid_for(2, N), dim3(BX, BY), 0, s>>>(in, out, N, lam, bc);
    else k_restrict_pass<3><<<grid_for(3, N), dim3(BX, BY), 0, s>>>(in, out, N, lam, bc);
}

void launch_relax_literal(int dim, bool sig, double* u, double* du, const double* up,
                          const double* dup, const double* g, const double* sigma, int N, int level,
                          const RelaxConst& rc, const BcDev& bc, unsigned long long* slot, int* flag, int pass_slot,
                          cudaStream_t s) {
    const dim3 gr = grid_for(dim, N), bl(BX, BY);
    if (dim == 2) {
        if (sig) k_relax_literal<2, true><<<gr, bl, 0, s>>>(u, du, up, dup, g, sigma, N, level, rc, bc, slot, flag, pass_slot);
        else k_relax_literal<2, false><<<gr, bl, 0, s>>>(u, du, up, dup, g, sigma, N, level, rc, bc, slot, flag, pass_slot);
    } else {
        if (sig) k_relax_literal<3, true><<<gr, bl, 0, s>>>(u, du, up, dup, g, sigma, N, level, rc, bc, slot, flag, pass_slot);
        else k_relax_literal<3, false><<<gr, bl, 0, s>>>(u, du, up, dup, g, sigma, N, level, rc, bc, slot, flag, pass_slot);
    }
}

void launch_residual(int dim, bool sig, double* r, const double* e, double* utot,
                     const double* sigma, int N, double inv_h2, double pref, double a,
                     const BcDev& bc, unsigned long long* rmax_slot, cudaStream_t s, int compact) {
    const dim3 gr = grid_for(dim, N), bl(BX, BY);
    const int has_a = a != 0.0;
    if (dim == 2) {
        if (sig) k_residual<2, true><<<gr, bl, 0, s>>>(r, e, utot, sigma, N, inv_h2, pref, a, has_a, bc, rmax_slot, compact);
        else k_residual<2, false><<<gr, bl, 0, s>>>(r, e, utot, sigma, N, inv_h2, pref, a, has_a, bc, rmax_slot, compact);
    } else {
        if (sig) k_residual<3, true><<<gr, bl, 0, s>>>(r, e, utot, sigma, N, inv_h2, pref, a, has_a, bc, rmax_slot, compact);
        else k_residual<3, false><<<gr, bl, 0, s>>>(r, e, utot, sigma, N, inv_h2, pref, a, has_a, bc, rmax_slot, compact);
    }
}

void launch_max_abs(const double* f, uint64_t total, unsigned long long* slot, cudaStream_t s) {
    k_max_abs<<<flat_blocks(total), 256, 0, s>>>(f, total, slot);
}

void launch_fill(double* f, uint64_t total, double v, cudaStream_t s) {
    k_fill<<<flat_blocks(total), 256, 0, s>>>(f, total, v);
}

void launch_sub_scalar(double* f, uint64_t total, double v, cudaStream_t s) {
    k_sub_scalar<<<flat_blocks(total), 256, 0, s>>>(f, total, v);
}

void launch_add_into(double* dst, const double* src, uint64_t total, cudaStream_t s) {
    k_add_into<<<flat_blocks(total), 256, 0, s>>>(dst, src, total);
}

void launch_apply_boundary(int dim, double* u, int N, const BcDev& bc, bool homogeneous,
                           cudaStream_t s) {
    if (dim == 2) k_apply_boundary<2><<<grid_for(2, N), dim3(BX, BY), 0, s>>>(u, N, bc, homogeneous);
    else k_apply_boundary<3><<<grid_for(3, N), dim3(BX, BY), 0, s>>>(u, N, bc, homogeneous);
}

void launch_check_positive(const double* f, uint64_t total, int* flag, cudaStream_t s) {
    k_check_positive<<<flat_blocks(total), 256, 0, s>>>(f, total, flag);
}

void launch_check_finite(const double* f, uint64_t total, int* flag, cudaStream_t s) {
    k_check_finite<<<flat_blocks(total), 256, 0, s>>>(f, total, flag);
}

}  // namespace sgmlb
