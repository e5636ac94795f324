// materialize.cu — lazy application of the pending interpolation increments.
//
// In the reference every pass at level v >= 1 sweeps the whole grid and
// adds u_prev + I(du_prev) at each non-subset node (kernels.cpp:140-174,
// 225-226).  The compact engine (engine.cpp) keeps those variations on the
// level-v subset (DU arrays) and applies them only when the next level's
// input is needed, in the reference's order:
//
//   value = Dirichlet face value                 (on a Dirichlet face)
//         = U_lf[x]                              (x on the finest relaxed level lf)
//         = ((base + I_l0(du0)) + I_l1(du1)) + ...   (everything else)
//
// with I_l(du)(x) = sum over corners r, q, p of ((wz*wy)*wx) * du[corner]
// (all weights exact dyadics; zero-weight corners skipped: sign of zero only).
//
// A thread owns MV = 4 consecutive x nodes.  For every level coarser than
// the first the four nodes share one cell, so the 8 corner loads serve four
// nodes; y and z are uniform across a warp, so the zero-weight corner rows
// are skipped without divergence.  Chain descriptors sit in shared memory.
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"

namespace sgmlb {

namespace {

constexpr int MV = 4;
constexpr int MBX = 32, MBY = 4;

template <int DIM>
__global__ void __launch_bounds__(MBX* MBY)
    k_materialize4(double* __restrict__ out, int Nw, int w, const double* __restrict__ base, int N,
                   int base_zero, const double* __restrict__ ufine, int Nf, int frel,
                   const ChainEntry* __restrict__ chain, int nchain, BcDev bc, int homogeneous,
                   int* flag) {
    __shared__ ChainEntry sch[kMaxChain];
    const int tid = threadIdx.x + MBX * threadIdx.y;
    for (int c = tid; c < nchain; c += MBX * MBY) sch[c] = chain[c];
    __syncthreads();

    const int X4 = (blockIdx.x * MBX + threadIdx.x) * MV;
    const int J = blockIdx.y * MBY + threadIdx.y;
    const int K = blockIdx.z;
    int bad = 0;
    if (X4 < Nw && J < Nw) {
        const int y = J << w, z = DIM == 3 ? K << w : 0;
        const int nv = min(MV, Nw - X4);
        double val[MV];
#pragma unroll
        for (int k = 0; k < MV; ++k)
            val[k] = (!base_zero && k < nv) ? __ldg(base + lin3(N, (X4 + k) << w, y, z)) : 0.0;

        for (int c = 0; c < nchain; ++c) {
            const ChainEntry ce = sch[c];
            const int l = ce.level, Nl = ce.Nl;
            const int msk = (1 << l) - 1;
            const double inv = 1.0 / (double)(1 << l);  // exact power of two
            const int iy = y & msk, iz = z & msk;
            const double fy = (double)iy * inv, fz = (double)iz * inv;
            const double wy[2] = {1.0 - fy, fy};
            const double wz[2] = {1.0 - fz, fz};
            const int nq = iy ? 2 : 1, nr = (DIM == 3 && iz) ? 2 : 1;  // warp-uniform
            const int x0 = X4 << w;
            const int X0 = x0 >> l;
            // corner columns X0, X0+1, X0+2 (the third only when the run
            // straddles two cells, i.e. l == w + 1)
            double cc[2][2][3];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (r < nr && q < nq) {
                        const double* row = ce.du + lin3(Nl, X0, (y >> l) + q, DIM == 3 ? (z >> l) + r : 0);
#pragma unroll
                        for (int p = 0; p < 3; ++p) cc[r][q][p] = X0 + p < Nl ? __ldg(row + p) : 0.0;
                    } else {
#pragma unroll
                        for (int p = 0; p < 3; ++p) cc[r][q][p] = 0.0;
                    }
                }
#pragma unroll
            for (int k = 0; k < MV; ++k) {
                const int x = (X4 + k) << w;
                const int ix = x & msk;
                const int j = (x >> l) - X0;  // 0 or 1
                const double fx = (double)ix * inv;
                const double wx0 = 1.0 - fx, wx1 = fx;
                double acc = 0.0;
#pragma unroll
                for (int r = 0; r < 2; ++r)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        if (r < nr && q < nq) {
                            const double wzy = DIM == 3 ? wz[r] * wy[q] : wy[q];
                            const double ca = j ? cc[r][q][1] : cc[r][q][0];
                            const double cb = j ? cc[r][q][2] : cc[r][q][1];
                            acc = acc + ((wzy * wx0) * ca);
                            if (ix) acc = acc + ((wzy * wx1) * cb);
                        }
                    }
                val[k] = val[k] + acc;
            }
        }
        const bool jface = J == 0 || J == Nw - 1 || (DIM == 3 && (K == 0 || K == Nw - 1));
        const int fmask = (1 << frel) - 1;
#pragma unroll
        for (int k = 0; k < MV; ++k) {
            if (k >= nv) break;
            const int I = X4 + k;
            double value = val[k];
            if ((jface || I == 0 || I == Nw - 1) && on_dirichlet<DIM>(bc, Nw, I, J, K)) {
                value = homogeneous ? 0.0 : dirichlet_value<DIM>(bc, Nw, I, J, K);
            } else if (ufine && ((I | J | K) & fmask) == 0) {
                value = __ldg(ufine + lin3(Nf, I >> frel, J >> frel, K >> frel));
            }
            bad |= (__double_as_longlong(value) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
            out[lin3(Nw, I, J, K)] = value;
        }
    }
    block_or_commit(bad, flag);
}

}  // namespace

void launch_materialize4(int dim, double* out, int Nw, int w, const double* base, int N,
                         bool base_zero, const double* ufine, int Nf, int frel,
                         const ChainEntry* chain, int nchain, const BcDev& bc, bool homogeneous,
                         int* flag, cudaStream_t s) {
    const int threads_x = (Nw + MV - 1) / MV;
    const dim3 grid((threads_x + MBX - 1) / MBX, (Nw + MBY - 1) / MBY, dim == 3 ? Nw : 1);
    if (dim == 2)
        k_materialize4<2><<<grid, dim3(MBX, MBY), 0, s>>>(out, Nw, w, base, N, base_zero, ufine, Nf, frel,
                                                          chain, nchain, bc, homogeneous, flag);
    else
        k_materialize4<3><<<grid, dim3(MBX, MBY), 0, s>>>(out, Nw, w, base, N, base_zero, ufine, Nf, frel,
                                                          chain, nchain, bc, homogeneous, flag);
}

}  // namespace sgmlb

// ---------------------------------------------------------------------------
// Restriction pyramid step: level-(m+1) compact <- the
// reference's averaging pass at stride 2^m (kernels.cpp:39-80,
// stencil.cpp:98-119) evaluated only at level-(m+1) nodes, which in the
// level-m compact index space are the even nodes with neighbours at +-1.
// Interior outputs take the branch-free path; the one-node boundary layer
// goes out of line through the reference's ghost recursion.
// ---------------------------------------------------------------------------

namespace sgmlb {

namespace {

__device__ __forceinline__ double axw2(int o) { return o == 0 ? 0.5 : 0.25; }

template <int DIM>
__device__ __noinline__ double pyramid_cold(const double* __restrict__ in, int Nin, int i, int j, int k,
                                            BcDev bc) {
    double acc = 0.0;
#pragma unroll
    for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
        for (int q = -1; q <= 1; ++q)
#pragma unroll
            for (int p = -1; p <= 1; ++p) {
                const double w = DIM == 3 ? (axw2(p) * axw2(q)) * axw2(r) : axw2(p) * axw2(q);
                acc = acc + w * ghost(in, Nin, bc, i + p, j + q, k + r);
            }
    return acc;
}

template <int DIM>
__global__ void __launch_bounds__(128) k_pyramid2(const double* __restrict__ in, int Nin,
                                                  double* __restrict__ out, int Nout, BcDev bc) {
    const int I = blockIdx.x * 32 + threadIdx.x, J = blockIdx.y * 4 + threadIdx.y, K = blockIdx.z;
    if (I >= Nout || J >= Nout) return;
    const int i = 2 * I, j = 2 * J, k = DIM == 3 ? 2 * K : 0;
    const bool inner = I >= 1 && I <= Nout - 2 && J >= 1 && J <= Nout - 2 &&
                       (DIM == 2 || (K >= 1 && K <= Nout - 2));
    double acc = 0.0;
    if (inner) {
        const double* c = in + lin3(Nin, i, j, k);
        const ptrdiff_t sy = Nin, sz = (ptrdiff_t)Nin * Nin;
#pragma unroll
        for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
            for (int q = -1; q <= 1; ++q)
#pragma unroll
                for (int p = -1; p <= 1; ++p) {
                    const double w = DIM == 3 ? (axw2(p) * axw2(q)) * axw2(r) : axw2(p) * axw2(q);
                    acc = acc + w * __ldg(c + r * sz + q * sy + p);
                }
    } else {
        acc = pyramid_cold<DIM>(in, Nin, i, j, k, bc);
    }
    out[lin3(Nout, I, J, K)] = acc;
}

}  // namespace

void launch_pyramid2(int dim, const double* in, int Nin, double* out, int Nout, const BcDev& bc,
                     cudaStream_t s) {
    const dim3 grid((Nout + 31) / 32, (Nout + 3) / 4, dim == 3 ? Nout : 1);
    if (dim == 2) k_pyramid2<2><<<grid, dim3(32, 4), 0, s>>>(in, Nin, out, Nout, bc);
    else k_pyramid2<3><<<grid, dim3(32, 4), 0, s>>>(in, Nin, out, Nout, bc);
}

}  // namespace sgmlb
