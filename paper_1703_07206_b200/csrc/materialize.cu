// materialize.cu — level-array kernels of the compact engine other than the
// relaxation pass: lazy interpolation (materialize), the restriction
// pyramid, and dense <-> ghost-extended conversions.  All level arrays use
// the ghost-extended padded layout of device.cuh (ExtLay).
//
// Lazy interpolation.  In the reference every pass at level v >= 1 sweeps
// the whole grid and adds u_prev + I(du_prev) at each non-subset node
// (kernels.cpp:140-174, 225-226).  The compact engine keeps those
// variations on the level-v subset (DU arrays) and applies them only when
// the next level's input is needed, in the reference's order:
//
//   value = Dirichlet face value                 (on a Dirichlet face)
//         = U_lf[x]                              (x on the finest relaxed level lf)
//         = ((base + I_l0(du0)) + I_l1(du1)) + ...   (everything else)
//
// with I_l(du)(x) = sum over corners r, q, p of ((wz*wy)*wx) * du[corner]
// (all weights exact dyadics; zero-weight corner rows in y / z are skipped,
// which changes at most the sign of an exact zero).
// A thread owns MV = 4 consecutive x nodes in two "spread copies" along y:
// rows S and S + H with H = (Nw - 1) / 2 (y, not z: 3D level arrays may be
// z-slabs of a multi-GPU decomposition).
// Every chain level l has cells of 2^(l-w) target nodes, which divides H, so
// the two copies see identical interpolation weights: each weight product
// is formed once and used for 2 x 4 nodes.  For every level coarser than
// the first, the four x nodes of a copy share one cell, so its 8 corner
// loads serve four nodes; y and z are uniform across a warp, so zero-weight
// corner rows are skipped without divergence.  The row S = H holds the
// last row 2H alone (its second copy is computed redundantly and dropped).
// Threads whose nodes all lie on Dirichlet faces skip the chain.  Chain
// descriptors sit in shared memory.
#include <cstdlib>

#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"
#include "level_ops.cuh"

namespace sgmlb {

namespace {


template <int DIM, int NC, bool DIAG>
__global__ void __launch_bounds__(MBX* MBY, 5)
    k_materialize4(double* __restrict__ out, ExtLay Lw, int w, const double* __restrict__ base,
                   ExtLay L0, int wb, int base_zero, const double* __restrict__ ufine, ExtLay Lf, int frel,
                   const ChainEntry* __restrict__ chain, int nchain, BcDev bc, int homogeneous,
                   int* flag, int xtail, int k0, int kz, int ke) {
    // the first kMaxChain entries sit in shared memory; a longer chain (a
    // single visit adding more than kMaxChain increments, n_r > kMaxChain + 1)
    // reads the rest from global memory
    __shared__ ChainEntry sch[kMaxChain];
    pdl_begin();
    const int tid = threadIdx.x + MBX * threadIdx.y;
    const int nsh = min(nchain, kMaxChain);
    for (int c = tid; c < nsh; c += MBX * MBY) sch[c] = chain[c];
    __syncthreads();
    // kz planes per CTA (one chain copy, fewer CTA launches: 513^3 level 0
    // 101 -> 95 ms per solve at kz = 4; prefetching the next plane's base
    // values did not pay)
    for (int bz = blockIdx.z * kz; bz < min(blockIdx.z * kz + kz, ke); ++bz)
        mat4_body<DIM, NC, DIAG, true>(out, Lw, w, base, L0, wb, base_zero, ufine, Lf, frel, chain, nchain, sch, bc,
                                       homogeneous, flag, xtail, k0, blockIdx.x, blockIdx.y, bz, threadIdx.x,
                                       threadIdx.y);
}

// Short chains (at most kShortChain entries): one node per thread along x
// (coalesced base loads and stores), every chain corner loaded up front
// (level_ops.cuh mat_node) — the 4-node, 2-copy form above shares weights and
// corners, which pays only once the chain arithmetic dominates.
constexpr int kShortChain = 2;
constexpr int kNodeX = 256;

template <int DIM>
__global__ void __launch_bounds__(kNodeX) k_mat_node(double* __restrict__ out, ExtLay Lw, int w,
                                                     const double* __restrict__ base, ExtLay L0, int wb, int base_zero,
                                                     const double* __restrict__ ufine, ExtLay Lf, int frel,
                                                     const ChainEntry* __restrict__ chain, int nchain, BcDev bc,
                                                     int homogeneous, int* flag, int k0) {
    __shared__ ChainEntry sch[kShortChain];
    pdl_begin();
    if (threadIdx.x < nchain) sch[threadIdx.x] = chain[threadIdx.x];
    __syncthreads();
    const int I = blockIdx.x * kNodeX + threadIdx.x, J = blockIdx.y, K = DIM == 3 ? k0 + (int)blockIdx.z : 0;
    int bad = 0, tiny = 0;
    if (I < Lw.N)
        mat_node<DIM, kShortChain, true>(out, Lw, w, base, L0, wb, base_zero, ufine, Lf, frel, sch, nchain, bc,
                                         homogeneous, I, J, K, bad, tiny);
    warp_or_commit(bad, flag);
    warp_or_commit(tiny, flag + 1);
}

// ---------------------------------------------------------------------------
// Restriction pyramid step: level-(m+1) <- the reference's
// averaging pass at stride 2^m (kernels.cpp:39-80, stencil.cpp:98-119)
// evaluated only at level-(m+1) nodes, which in the level-m index space are
// the even nodes with neighbours at +-1.  The input's ghost cells hold the
// even mirror, which is the reference's ghost value wherever the result is
// consumed (see device.cuh); outputs are written with their mirror ghosts.
// ---------------------------------------------------------------------------

__device__ __forceinline__ double axw2(int o) { return o == 0 ? 0.5 : 0.25; }

template <int DIM>
__global__ void __launch_bounds__(128) k_pyramid_ext(const double* __restrict__ in, ExtLay Lin,
                                                     double* __restrict__ out, ExtLay Lout, int kb) {
    pdl_begin();
    const int Nout = Lout.N;
    // output plane: local kb + blockIdx.z, global + Lout.z0; input plane 2 * global
    const int I = blockIdx.x * 32 + threadIdx.x, J = blockIdx.y * 4 + threadIdx.y;
    const int K = DIM == 3 ? kb + (int)blockIdx.z : 0;
    if (I >= Nout || J >= Nout) return;
    const int Kin = DIM == 3 ? 2 * (K + Lout.z0) - Lin.z0 : 0;
    const double* c = in + eix<DIM>(Lin, 2 * I, 2 * J, Kin);
    const ptrdiff_t sy = Lin.Px, sz = (ptrdiff_t)Lin.Px * Lin.Ne;
    double acc = 0.0;
#pragma unroll
    for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
        for (int q = -1; q <= 1; ++q)
#pragma unroll
            for (int p = -1; p <= 1; ++p) {
                const double w = DIM == 3 ? (axw2(p) * axw2(q)) * axw2(r) : axw2(p) * axw2(q);
                acc = acc + w * __ldg(c + r * sz + q * sy + p);
            }
    store_ext<DIM>(out, Lout, I, J, K, acc);
}

// dense x-fastest field (global) -> ghost-extended array (own planes + mirror ghosts)
template <int DIM>
__global__ void __launch_bounds__(128) k_scatter_ext(const double* __restrict__ dense, double* ext,
                                                     ExtLay L) {
    const int N = L.N;
    const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 4 + threadIdx.y, k = blockIdx.z;
    if (i >= N || j >= N) return;
    store_ext<DIM>(ext, L, i, j, k, dense[lin3(N, i, j, DIM == 3 ? k + L.z0 : 0)]);
}

// ghost-extended array (own planes) -> dense x-fastest field (global)
template <int DIM>
__global__ void __launch_bounds__(128) k_gather_ext(const double* __restrict__ ext, ExtLay L,
                                                    double* __restrict__ dense) {
    const int N = L.N;
    const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 4 + threadIdx.y, k = blockIdx.z;
    if (i >= N || j >= N) return;
    dense[lin3(N, i, j, DIM == 3 ? k + L.z0 : 0)] = ext[eix<DIM>(L, i, j, k)];
}

// Dirichlet-face nodes (with their mirror ghosts) <- 0 or the face value.
// One thread per (face, a, b); nodes on edges are written by several faces
// with the same value (the lowest-face-id rule of dirichlet_value).  z-slab
// arrays: the x / y faces of the own planes, the z faces where they are own.
template <int DIM>
__global__ void __launch_bounds__(128) k_dirichlet_faces(double* a, ExtLay L, BcDev bc, int zero, int mirrors) {
    pdl_begin();
    const int N = L.N;
    const int p = blockIdx.x * 32 + threadIdx.x, q = blockIdx.y * 4 + threadIdx.y, f = blockIdx.z;
    if (p >= N || (DIM == 2 && q > 0) || bc.neu[f]) return;
    const int side = (f & 1) ? N - 1 : 0;
    int i, j, kg = 0;
    if (DIM == 2) {
        if (f < 2) { i = side; j = p; }
        else { i = p; j = side; }
    } else if (f < 4) {
        if (q >= L.Nz) return;  // q: local plane
        kg = q + L.z0;
        if (f < 2) { i = side; j = p; }
        else { i = p; j = side; }
    } else {
        if (q >= N || side < L.z0 || side >= L.z0 + L.Nz) return;
        i = p; j = q; kg = side;
    }
    const double v = zero ? 0.0 : dirichlet_value<DIM>(bc, N, i, j, kg);
    const int k = DIM == 3 ? kg - L.z0 : 0;
    if (mirrors) store_ext<DIM>(a, L, i, j, k, v);
    else a[eix<DIM>(L, i, j, k)] = v;
}

// level-(shift) subsample of a level array: out (local planes [kb, kb +
// gridDim.z)) <- in at the level-0-relative positions << shift
__global__ void __launch_bounds__(128) k_sample_ext(const double* __restrict__ in, ExtLay Lin,
                                                    double* __restrict__ out, ExtLay Lout, int shift, int kb) {
    pdl_begin();
    const int I = blockIdx.x * 32 + threadIdx.x, J = blockIdx.y * 4 + threadIdx.y;
    const int K = kb + (int)blockIdx.z;
    if (I >= Lout.N || J >= Lout.N) return;
    const int kin = ((K + Lout.z0) << shift) - Lin.z0;
    store_ext<3>(out, Lout, I, J, K, __ldg(in + eix<3>(Lin, I << shift, J << shift, kin)));
}

// Per-node pseudo-time step of the sigma relaxation (kernels.cpp:132-136):
// dtau = (safety K) / (inv_s2 smax) with smax = max over the 26 (8)
// neighbours (compact stencil: the 6 (4) axis neighbours) of
// sbar = 0.5 (sigma_n + sigma_c).  It depends on sigma only,
// so it is evaluated once per solve and level; the max is order-free and
// sbar's sum commutes, so this is the relaxation pass's own value bit for bit.
template <int DIM>
__global__ void __launch_bounds__(128) k_dtau_ext(const double* __restrict__ sig, ExtLay L, double* __restrict__ dt,
                                                  RelaxConst rc) {
    const int N = L.N;
    const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 4 + threadIdx.y, k = blockIdx.z;
    if (i >= N || j >= N) return;
    const ptrdiff_t c = eix<DIM>(L, i, j, k);
    const double sc = sig[c];
    const ptrdiff_t sy = L.Px, sz = DIM == 3 ? (ptrdiff_t)L.plane : 0;
    double smax = 0.0;
#pragma unroll
    for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
        for (int q = -1; q <= 1; ++q)
#pragma unroll
            for (int p = -1; p <= 1; ++p) {
                if (r == 0 && q == 0 && p == 0) continue;
                if (stencil_skip(rc.compact, r * r + q * q + p * p)) continue;
                const double sbar = 0.5 * (sig[c + r * sz + q * sy + p] + sc);
                smax = smax < sbar ? sbar : smax;
            }
    dt[c] = (rc.safety * rc.kdim) / (rc.inv_s2 * smax);
}

inline dim3 ext_grid(int dim, const ExtLay& L) {
    return dim3((L.N + 31) / 32, (L.N + 3) / 4, dim == 3 ? L.Nz : 1);
}

}  // namespace

ExtLay make_ext(int dim, int N, int z0, int nz) {
    ExtLay L{};
    L.N = N;
    L.Ne = N + 2;
    // pitch a multiple of 4 doubles: 32-byte aligned rows (TMA needs 16)
    L.Px = (L.Ne + 3) / 4 * 4;
    L.Nz = dim == 3 ? (nz < 0 ? N : nz) : 1;
    L.z0 = dim == 3 ? z0 : 0;
    L.plane = dim == 3 ? (long long)L.Px * L.Ne : (long long)L.Px;
    return L;
}

uint64_t ext_size(int dim, const ExtLay& L) {
    return dim == 3 ? (uint64_t)L.Px * L.Ne * (L.Nz + 2) : (uint64_t)L.Px * L.Ne;
}

void materialize_grid(int dim, const ExtLay& Lw, const BcDev& bc, int& gx, int& gy, int& gz, int& xtail) {
    const int Nw = Lw.N;
    xtail = (!bc.neu[1] && (Nw - 1) % MV == 0) ? 1 : 0;
    const int threads_x = xtail ? (Nw - 1) / MV : (Nw + MV - 1) / MV, D = (Nw - 1) / 2;
    gx = (threads_x + MBX - 1) / MBX;
    gy = (D + MBY) / MBY;
    gz = dim == 3 ? Lw.Nz : 1;
}

void launch_materialize4(int dim, double* out, const ExtLay& Lw, int w, const double* base,
                         const ExtLay& L0, int wb, bool base_zero, const double* ufine, const ExtLay& Lf,
                         int frel, const ChainEntry* chain, int nchain, const BcDev& bc,
                         bool homogeneous, int* flag, bool diag, cudaStream_t s, int kb, int ke) {
    const int Nw = Lw.N;
    if (ke < 0) ke = Lw.Nz;
    if (dim == 3 && ke <= kb) return;
    static const bool no_short = std::getenv("SGML_NO_SHORT_CHAINS") != nullptr;
    // (small levels only: on 129^3 and larger the weight and corner sharing
    // of the 4-node form wins even for one entry — 513^3 materialisations
    // 92 -> 118 ms per solve with this form, 65^3 solve 5.21 -> 5.08 ms)
    const double nodes = (double)Nw * Nw * (dim == 3 ? (double)Nw : 1.0);
    if (!diag && !no_short && nchain <= kShortChain && nodes <= 300000.0) {
        const dim3 grid((Nw + kNodeX - 1) / kNodeX, Nw, dim == 3 ? ke - kb : 1);
        if (dim == 2)
            launch_pdl(k_mat_node<2>, grid, dim3(kNodeX), 0, s, out, Lw, w, base, L0, wb, base_zero ? 1 : 0, ufine, Lf,
                       frel, chain, nchain, bc, homogeneous ? 1 : 0, flag, 0);
        else
            launch_pdl(k_mat_node<3>, grid, dim3(kNodeX), 0, s, out, Lw, w, base, L0, wb, base_zero ? 1 : 0, ufine, Lf,
                       frel, chain, nchain, bc, homogeneous ? 1 : 0, flag, kb);
        return;
    }
    // two copies (y and y + (Nw-1)/2): measured faster than one (occupancy
    // does not pay for the lost weight sharing) and than four (16 nodes per
    // thread cost occupancy)
    constexpr int NC = 2;
    // Dirichlet x-high face (Nw - 1 a multiple of MV): threads cover x < Nw - 1
    // and the last group writes the face node (xtail)
    const int xtail = (!bc.neu[1] && (Nw - 1) % MV == 0) ? 1 : 0;
    const int threads_x = xtail ? (Nw - 1) / MV : (Nw + MV - 1) / MV, D = (Nw - 1) / NC;
    const int gx = (threads_x + MBX - 1) / MBX, gy = (D + MBY) / MBY, nzp = dim == 3 ? ke - kb : 1;
    // 4 planes per CTA where that still leaves ~10 CTAs per SM (large levels)
    const int kz = (long long)gx * gy * nzp >= 4LL * 148 * 5 * 2 ? 4 : 1;
    const dim3 grid(gx, gy, (nzp + kz - 1) / kz);
#define SGML_MAT(DD, CC, GG)                                                                              \
    launch_pdl(k_materialize4<DD, CC, GG>, grid, dim3(MBX, MBY), 0, s, out, Lw, w, base, L0, wb, base_zero, ufine, \
               Lf, frel, chain, nchain, bc, homogeneous, flag, xtail, dim == 3 ? kb : 0, kz, nzp)
    if (dim == 2) {
        if (diag) SGML_MAT(2, NC, true);
        else SGML_MAT(2, NC, false);
    } else {
        if (diag) SGML_MAT(3, NC, true);
        else SGML_MAT(3, NC, false);
    }
#undef SGML_MAT
}

void launch_pyramid_ext(int dim, const double* in, const ExtLay& Lin, double* out, const ExtLay& Lout,
                        cudaStream_t s, int kb, int ke) {
    if (dim == 2) {
        launch_pdl(k_pyramid_ext<2>, ext_grid(2, Lout), dim3(32, 4), 0, s, in, Lin, out, Lout, 0);
        return;
    }
    if (ke < 0) ke = Lout.Nz;
    if (ke <= kb) return;
    dim3 g = ext_grid(3, Lout);
    g.z = ke - kb;
    launch_pdl(k_pyramid_ext<3>, g, dim3(32, 4), 0, s, in, Lin, out, Lout, kb);
}

void launch_scatter_ext(int dim, const double* dense, double* ext, const ExtLay& L, cudaStream_t s) {
    if (dim == 2) k_scatter_ext<2><<<ext_grid(2, L), dim3(32, 4), 0, s>>>(dense, ext, L);
    else k_scatter_ext<3><<<ext_grid(3, L), dim3(32, 4), 0, s>>>(dense, ext, L);
}

void launch_gather_ext(int dim, const double* ext, const ExtLay& L, double* dense, cudaStream_t s) {
    if (dim == 2) k_gather_ext<2><<<ext_grid(2, L), dim3(32, 4), 0, s>>>(ext, L, dense);
    else k_gather_ext<3><<<ext_grid(3, L), dim3(32, 4), 0, s>>>(ext, L, dense);
}

void launch_dirichlet_faces(int dim, double* a, const ExtLay& L, const BcDev& bc, bool zero,
                            bool mirrors, cudaStream_t s) {
    const int N = L.N;
    if (dim == 2)
        launch_pdl(k_dirichlet_faces<2>, dim3((N + 31) / 32, 1, 4), dim3(32, 4), 0, s, a, L, bc, zero ? 1 : 0,
                   mirrors ? 1 : 0);
    else
        launch_pdl(k_dirichlet_faces<3>, dim3((N + 31) / 32, (N + 3) / 4, 6), dim3(32, 4), 0, s, a, L, bc, zero ? 1 : 0,
                   mirrors ? 1 : 0);
}

void launch_sample_ext(const double* in, const ExtLay& Lin, double* out, const ExtLay& Lout, int shift, int kb,
                       int ke, cudaStream_t s) {
    if (ke <= kb) return;
    dim3 g = ext_grid(3, Lout);
    g.z = ke - kb;
    launch_pdl(k_sample_ext, g, dim3(32, 4), 0, s, in, Lin, out, Lout, shift, kb);
}

void launch_dtau_ext(int dim, const double* sig, const ExtLay& L, double* dt, const RelaxConst& rc, cudaStream_t s) {
    if (dim == 2) k_dtau_ext<2><<<ext_grid(2, L), dim3(32, 4), 0, s>>>(sig, L, dt, rc);
    else k_dtau_ext<3><<<ext_grid(3, L), dim3(32, 4), 0, s>>>(sig, L, dt, rc);
}

}  // namespace sgmlb
