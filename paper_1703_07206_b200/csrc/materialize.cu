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
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"

namespace sgmlb {

namespace {

constexpr int MV = 4;
constexpr int MBX = 32, MBY = 4;

template <int DIM, int NC, bool DIAG>
__global__ void __launch_bounds__(MBX* MBY, 5)
    k_materialize4(double* __restrict__ out, ExtLay Lw, int w, const double* __restrict__ base,
                   ExtLay L0, int wb, int base_zero, const double* __restrict__ ufine, ExtLay Lf, int frel,
                   const ChainEntry* __restrict__ chain, int nchain, BcDev bc, int homogeneous,
                   int* flag, int xtail, int k0) {
    // the first kMaxChain entries sit in shared memory; a longer chain (a
    // single visit adding more than kMaxChain increments, n_r > kMaxChain + 1)
    // reads the rest from global memory
    __shared__ ChainEntry sch[kMaxChain];
    pdl_begin();
    const int tid = threadIdx.x + MBX * threadIdx.y;
    const int nsh = min(nchain, kMaxChain);
    for (int c = tid; c < nsh; c += MBX * MBY) sch[c] = chain[c];
    __syncthreads();

    // NC copies along y at spacing D = (Nw - 1) / NC: rows s0 + c D
    const int Nw = Lw.N, D = (Nw - 1) / NC;
    const int X4 = (blockIdx.x * MBX + threadIdx.x) * MV;
    // spread row index S (warp-uniform); 3D: local plane K (block-uniform),
    // global plane Kg (z-slab arrays start at global plane Lw.z0)
    const int S = blockIdx.y * MBY + threadIdx.y;
    const int K = DIM == 3 ? k0 + (int)blockIdx.z : 0;
    const int Kg = DIM == 3 ? K + Lw.z0 : 0;
    int bad = 0, tiny = 0;
    if (S <= D && X4 < Nw) {
        const int ncopy = S < D ? NC : 1;
        const int s0 = S < D ? S : NC * D;
        const int nv = min(MV, Nw - X4);
        // node (k, copy cp): x = X4 + k, y = s0 + cp * D
        auto node_j = [&](int cp) { return s0 + cp * D; };
        // every node of this thread on a Dirichlet face: nothing to interpolate
        const bool xdir = nv == 1 && X4 == Nw - 1 && !bc.neu[1];
        const bool rowdir = S == D && !bc.neu[3];  // the lone last row
        const bool pdir = DIM == 3 && ((Kg == 0 && !bc.neu[4]) || (Kg == Nw - 1 && !bc.neu[5]));
        const int nch = (xdir || rowdir || pdir) ? 0 : nchain;
        const int y = s0 << w, z = Kg << w;
        const int fmask = (1 << frel) - 1;
        // rows / plane of this warp clear of the y / z faces by two nodes (no
        // Dirichlet node, no mirror ghost; warp-uniform)
        const bool rows_in = (DIM == 2 || (Kg >= 2 && Kg <= Nw - 3)) && s0 >= 2 && node_j(ncopy - 1) <= Nw - 3;
        // fast path (warp-uniform): rows / plane clear of the y / z faces,
        // frel = 1; the x faces are handled inline (lanes at the row ends).
        // The level-(w+1) nodes (even x at even rows / planes; both copies
        // have the row parity of s0 when D is even) take ufine, loaded up front
        const bool inner = rows_in && frel == 1 && (!ufine || (D & 1) == 0);
        const bool rowfine = inner && ufine && ((s0 | Kg) & 1) == 0;
        double uf[NC][2];
#pragma unroll
        for (int cp = 0; cp < NC; ++cp) {
            uf[cp][0] = uf[cp][1] = 0.0;
            if (rowfine && cp < ncopy) {
                const double* pf = ufine + (int)eix<DIM>(Lf, X4 >> 1, node_j(cp) >> 1, (Kg >> 1) - Lf.z0);
                uf[cp][0] = __ldg(pf);
                uf[cp][1] = __ldg(pf + 1);
            }
        }
        // DIAG (failure re-runs): the interpolated nodes of this thread (not on
        // a Dirichlet face, not taken from ufine) and the first chain entry
        // whose partial sum turns non-finite at one of them
        unsigned interp = 0;
        int firstbad = 0x7fffffff;
        if (DIAG) {
            for (int cp = 0; cp < ncopy; ++cp)
                for (int k = 0; k < nv; ++k) {
                    const int I = X4 + k, Jn = node_j(cp);
                    const bool dir = on_dirichlet<DIM>(bc, Nw, I, Jn, Kg);
                    const bool fine = ufine && ((I | Jn | Kg) & fmask) == 0;
                    if (!dir && !fine) interp |= 1u << (cp * MV + k);
                }
        }
        double val[NC][MV];
        {
            const int bsh = w - wb;
            const double* bp = base + (int)eix<DIM>(L0, X4 << bsh, s0 << bsh, (z >> wb) - L0.z0);
            const int bcs = (D << bsh) * L0.Px;  // copy spacing in base elements
#pragma unroll
            for (int cp = 0; cp < NC; ++cp)
#pragma unroll
                for (int k = 0; k < MV; ++k)
                    val[cp][k] = (!base_zero && k < nv && cp < ncopy) ? __ldg(bp + cp * bcs + (k << bsh)) : 0.0;
        }

        for (int c = 0; c < nch; ++c) {
            const ChainEntry ce = c < kMaxChain ? sch[c] : chain[c];
            const int l = ce.level, Nl = ce.L.N;
            const int msk = (1 << l) - 1;
            const double inv = __longlong_as_double((long long)(1023 - l) << 52);  // 2^-l, exact
            const int iy = y & msk, iz = z & msk;
            const double fy = (double)iy * inv, fz = (double)iz * inv;
            const double wy[2] = {1.0 - fy, fy};
            const double wz[2] = {1.0 - fz, fz};
            const int nq = iy ? 2 : 1, nr = (DIM == 3 && iz) ? 2 : 1;  // warp-uniform
            const int X0 = (X4 << w) >> l;
            // 32-bit element offsets (level arrays hold < 2^31 doubles, see
            // sgml_solver::build): q row, r plane, copy spacing (D in level-l
            // rows; 0 when the copies are dummies)
            const int sq = ce.L.Px, sr = DIM == 3 ? (int)ce.L.plane : 0;
            const int dsp = ncopy == NC ? ((Nl - 1) / NC) * sq : 0;
            const int o00 = (int)eix<DIM>(ce.L, X0, y >> l, DIM == 3 ? (z >> l) - ce.L.z0 : 0);
            // the run of MV nodes straddles two cells only on level w + 1 (X4 is a
            // multiple of 4: nodes 0, 1 in cell X0, nodes 2, 3 in cell X0 + 1, at
            // fractions 0 and 1/2)
            const bool straddle = l == w + 1;
            double fx[MV], wx0[MV];
#pragma unroll
            for (int k = 0; k < MV; ++k) {
                const int x = (X4 + k) << w;
                fx[k] = (double)(x & msk) * inv;
                wx0[k] = 1.0 - fx[k];
            }
            double acc[NC][MV];
            // `st` is a literal at both call sites: the straddle selects vanish
            // from the common (same-cell) path
            // `sk` (rowfine warps): the level-(w+1) nodes (even k) take ufine,
            // so their chains are not evaluated
            auto accumulate = [&](bool st, bool sk) {
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    if (r >= nr) break;
                    // corner loads of this plane first (both rows, all copies),
                    // then the products in the reference's order.  Every row exists
                    // in memory (rows up to Nl are ghost cells); past the x end
                    // the DU arrays' ghost cells, never written (0)
                    double cv[2][NC][3];
#pragma unroll
                    for (int q = 0; q < 2; ++q)
#pragma unroll
                        for (int cp = 0; cp < NC; ++cp) {
                            const double* rw = ce.du + (o00 + r * sr + q * sq + cp * dsp);
                            cv[q][cp][0] = __ldg(rw);
                            cv[q][cp][1] = __ldg(rw + 1);
                            cv[q][cp][2] = st ? __ldg(rw + 2) : 0.0;
                        }
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        if (q >= nq) break;
                        const double wzy = DIM == 3 ? wz[r] * wy[q] : wy[q];
                        // reference order per node: corner p = 0 then p = 1 of this
                        // (r, q); a zero-weight p = 1 term adds +-0 (as the reference)
#pragma unroll
                        for (int k = 0; k < MV; ++k) {
                            if (sk && (k & 1) == 0) continue;
                            const double w0 = wzy * wx0[k], w1 = wzy * fx[k];
                            const int j = st ? (k >> 1) : 0;
#pragma unroll
                            for (int cp = 0; cp < NC; ++cp) {
                                const double t0 = w0 * cv[q][cp][j];
                                acc[cp][k] = (r == 0 && q == 0) ? t0 : acc[cp][k] + t0;
                                acc[cp][k] = acc[cp][k] + w1 * cv[q][cp][j + 1];
                            }
                        }
                    }
                }
            };
            if (rowfine) {
                if (straddle) accumulate(true, true);
                else accumulate(false, true);
            } else {
                if (straddle) accumulate(true, false);
                else accumulate(false, false);
            }
#pragma unroll
            for (int cp = 0; cp < NC; ++cp)
#pragma unroll
                for (int k = 0; k < MV; ++k)
                    if (!(rowfine && (k & 1) == 0)) val[cp][k] = val[cp][k] + acc[cp][k];
            if (DIAG) {
#pragma unroll
                for (int cp = 0; cp < NC; ++cp)
#pragma unroll
                    for (int k = 0; k < MV; ++k)
                        if ((interp >> (cp * MV + k)) & 1u)
                            if ((__double_as_longlong(val[cp][k]) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL)
                                firstbad = min(firstbad, ce.fslot);
            }
        }
        if (DIAG && firstbad != 0x7fffffff) {
            atomicOr(flag, 1);
            atomicMin(flag + 4, firstbad);
        }
        // final values (Dirichlet faces, ufine nodes) and the checks
        if (inner) {
            // lane holding node 0, 1, Nw - 2 or Nw - 1: x-face values and mirrors
            const bool xedge = X4 < 2 || X4 + MV > Nw - 2;
            const double vx0 = homogeneous ? 0.0 : bc.val[0], vx1 = homogeneous ? 0.0 : bc.val[1];
#pragma unroll
            for (int cp = 0; cp < NC; ++cp) {
                if (cp >= ncopy) break;
                double* po = out + (int)eix<DIM>(Lw, X4, node_j(cp), K);
                double v[MV];
#pragma unroll
                for (int k = 0; k < MV; ++k) v[k] = (rowfine && (k & 1) == 0) ? uf[cp][k >> 1] : val[cp][k];
                if (xedge) {
#pragma unroll
                    for (int k = 0; k < MV; ++k) {
                        const int I = X4 + k;
                        if (I == 0 && !bc.neu[0]) v[k] = vx0;
                        if (I == Nw - 1 && !bc.neu[1]) v[k] = vx1;
                    }
                }
#pragma unroll
                for (int k = 0; k < MV; ++k) {
                    if (k >= nv) break;
                    const unsigned hi = (unsigned)__double2hiint(v[k]) & 0x7fffffffu;
                    bad |= hi >= 0x7ff00000u;
                    const unsigned key = hi | min((unsigned)__double2loint(v[k]), 1u);
                    tiny |= key - 1u < 0x035fffffu;
                    po[k] = v[k];
                }
                if (xedge) {
#pragma unroll
                    for (int k = 0; k < MV; ++k) {
                        if (k >= nv) break;
                        const int I = X4 + k;
                        if (I == 1) po[k - 2] = v[k];       // even mirror: ghost -1
                        if (I == Nw - 2) po[k + 2] = v[k];  // ghost Nw (both when Nw == 3)
                    }
                }
                // Dirichlet x-high face: the last group also writes node Nw - 1 (the
                // grid stops at Nw - 2, so no block is spent on that column)
                if (xtail && X4 + MV == Nw - 1) po[MV] = vx1;
            }
        } else {
#pragma unroll
            for (int cp = 0; cp < NC; ++cp) {
                if (cp >= ncopy) break;
                const int Jn = node_j(cp), Kn = Kg;
                const bool jface = Jn == 0 || Jn == Nw - 1 || (DIM == 3 && (Kn == 0 || Kn == Nw - 1));
#pragma unroll
                for (int k = 0; k < MV; ++k) {
                    if (k >= nv) break;
                    const int I = X4 + k;
                    double value = val[cp][k];
                    if ((jface || I == 0 || I == Nw - 1) && on_dirichlet<DIM>(bc, Nw, I, Jn, Kn)) {
                        value = homogeneous ? 0.0 : dirichlet_value<DIM>(bc, Nw, I, Jn, Kn);
                    } else if (ufine && ((I | Jn | Kn) & fmask) == 0) {
                        value = __ldg(ufine + eix<DIM>(Lf, I >> frel, Jn >> frel, (Kn >> frel) - Lf.z0));
                    }
                    bad |= (__double_as_longlong(value) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
                    {  // nonzero |value| < 2^-969 (see launch_relax_tma)
                        const unsigned key = ((unsigned)__double2hiint(value) & 0x7fffffffu) |
                                             (__double2loint(value) != 0 ? 1u : 0u);
                        tiny |= key - 1u < 0x035fffffu;
                    }
                    store_ext<DIM>(out, Lw, I, Jn, K, value);
                }
                // Dirichlet x-high face: the last group also writes node Nw - 1 (the
                // grid stops at Nw - 2, so no block is spent on that column),
                // with its y / z mirror ghosts (rows / planes 1 and Nw - 2 next to
                // a Neumann face: the corner ghost the relaxation reads)
                if (xtail && X4 + MV == Nw - 1)
                    store_ext<DIM>(out, Lw, Nw - 1, Jn, K,
                                   homogeneous ? 0.0 : dirichlet_value<DIM>(bc, Nw, Nw - 1, Jn, Kn));
            }
        }
    }
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
    // pitch a multiple of 4 doubles: 32-byte aligned rows (TMA needs 16; the
    // materialisation's 256-bit accesses start at data nodes 4m - 1)
    L.Px = (L.Ne + 3) / 4 * 4;
    L.Nz = dim == 3 ? (nz < 0 ? N : nz) : 1;
    L.z0 = dim == 3 ? z0 : 0;
    L.plane = dim == 3 ? (long long)L.Px * L.Ne : (long long)L.Px;
    return L;
}

uint64_t ext_size(int dim, const ExtLay& L) {
    return dim == 3 ? (uint64_t)L.Px * L.Ne * (L.Nz + 2) : (uint64_t)L.Px * L.Ne;
}

void launch_materialize4(int dim, double* out, const ExtLay& Lw, int w, const double* base,
                         const ExtLay& L0, int wb, bool base_zero, const double* ufine, const ExtLay& Lf,
                         int frel, const ChainEntry* chain, int nchain, const BcDev& bc,
                         bool homogeneous, int* flag, bool diag, cudaStream_t s, int kb, int ke) {
    const int Nw = Lw.N;
    if (ke < 0) ke = Lw.Nz;
    if (dim == 3 && ke <= kb) return;
    // two copies (y and y + (Nw-1)/2): measured faster than one (occupancy
    // does not pay for the lost weight sharing) and than four (16 nodes per
    // thread cost occupancy)
    constexpr int NC = 2;
    // Dirichlet x-high face (Nw - 1 a multiple of MV): threads cover x < Nw - 1
    // and the last group writes the face node (xtail)
    const int xtail = (!bc.neu[1] && (Nw - 1) % MV == 0) ? 1 : 0;
    const int threads_x = xtail ? (Nw - 1) / MV : (Nw + MV - 1) / MV, D = (Nw - 1) / NC;
    const dim3 grid((threads_x + MBX - 1) / MBX, (D + MBY) / MBY, dim == 3 ? ke - kb : 1);
#define SGML_MAT(DD, CC, GG)                                                                              \
    launch_pdl(k_materialize4<DD, CC, GG>, grid, dim3(MBX, MBY), 0, s, out, Lw, w, base, L0, wb, base_zero, ufine, \
               Lf, frel, chain, nchain, bc, homogeneous, flag, xtail, dim == 3 ? kb : 0)
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
