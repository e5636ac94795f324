// relax_tiled.cu — the hot kernel: one relaxation pass over a level-compact
// array (every node a subset node, neighbours at +-1 index), i.e. the
// reference's relax branch (kernels.cpp:94-137) and Dirichlet branch
// (kernels.cpp:213-218) at any level v once the level is stored compactly.
//
// Layout: a CTA owns an X x Y column bundle (3D: 32 x 8 nodes, 2D: 128 x 1)
// and marches along the slowest axis (z in 3D, y in 2D) over `zb` planes,
// two planes per step.  Planes of u (tile + one-node halo), g (tile) and
// sigma stream through an NST-deep shared-memory ring filled with cp.async
// (LDGSTS), so several planes of HBM traffic are in flight per CTA without
// holding registers.  Every thread keeps a 3 x 3 x 4 register window (planes
// m-1 .. m+2) and computes nodes m and m+1: two independent accumulation
// chains per thread hide the fp64 add latency of the reference's strictly
// sequential 26-term sum, and one __syncthreads serves two planes.  The
// window rotates by unrolling the march, so no register moves are issued.
//
// Halo cells outside the domain receive the reference's ghost value for
// that coordinate (stencil.cpp:52-85 / 87-90) by a plain store when the
// plane is staged (out-of-line cold path, boundary tiles only), so the
// stencil itself is branch-free and bit-identical to both reference paths.
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"

namespace sgmlb {

namespace {

template <int DIM>
struct Tile {
    static constexpr int X = DIM == 3 ? 32 : 128;
    static constexpr int Y = DIM == 3 ? 8 : 1;
    static constexpr int HX = X + 2;
    static constexpr int HY = DIM == 3 ? Y + 2 : 1;
    static constexpr int PLANE = HX * HY;
    static constexpr int INNER = X * Y;
    static constexpr int THREADS = X * Y;
    static constexpr int LOADS = (PLANE + THREADS - 1) / THREADS;
    static constexpr int Q = DIM == 3 ? 3 : 1;  // in-plane y extent of the stencil
    static constexpr int NST = 8;                // ring depth (planes), power of two
    static constexpr int D = NST - 2;            // staging lookahead (planes)
};

__device__ __forceinline__ void cp_async8(unsigned dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// kernel modes: one relaxation pass, or the fused residual recurrence
enum { MODE_RELAX = 0, MODE_RESID = 1 };

template <int DIM, bool SIG, int MODE = MODE_RELAX>
struct __align__(16) Ring {
    double u[Tile<DIM>::NST][Tile<DIM>::PLANE];
    double g[Tile<DIM>::NST][Tile<DIM>::INNER];   // g (relax) or r (residual)
    double s[SIG ? Tile<DIM>::NST : 1][SIG ? Tile<DIM>::PLANE : 1];
    double t[MODE == MODE_RESID ? Tile<DIM>::NST : 1][MODE == MODE_RESID ? Tile<DIM>::INNER : 1];
};

// Cold path: element e of plane m lies outside the domain (or the plane is
// a ghost plane).  Writes the reference's ghost value inside the one-node
// ghost layer, 0 beyond it (partial tiles; never read by a valid node).
template <int DIM, bool SIG>
__device__ __noinline__ void stage_cold(unsigned du_s, unsigned ds_s, int e, int m, int x0, int y0,
                                        int N, const double* __restrict__ ui,
                                        const double* __restrict__ sig, BcDev bc) {
    using TL = Tile<DIM>;
    double vu, vs = 1.0;
    int i, j, k;
    if (DIM == 3) {
        i = x0 + (e % TL::HX) - 1;
        j = y0 + (e / TL::HX) - 1;
        k = m;
    } else {
        i = x0 + e - 1;
        j = m;
        k = 0;
    }
    const bool layer = i >= -1 && i <= N && j >= -1 && j <= N && (DIM == 2 || (k >= -1 && k <= N));
    vu = layer ? ghost(ui, N, bc, i, j, k) : 0.0;
    asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(du_s), "d"(vu) : "memory");
    if (SIG) {
        vs = layer ? mirror(sig, N, i, j, k) : 1.0;
        asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(ds_s), "d"(vs) : "memory");
    }
}

// Out-of-line staging of one plane for tiles touching the domain boundary
// (and the ghost planes -1 / N): in-range elements by cp.async, the rest
// through stage_cold.  Keeps the hot loop of interior tiles small.
template <int DIM, bool SIG>
__device__ __forceinline__ void stage_general(unsigned su, unsigned ss, int tid, int m, int x0, int y0,
                                           int N, const double* __restrict__ ui,
                                           const double* __restrict__ sig, BcDev bc) {
    using TL = Tile<DIM>;
    const bool plane_in = (unsigned)m < (unsigned)N;
    const ptrdiff_t NN = DIM == 3 ? (ptrdiff_t)N * N : (ptrdiff_t)N;
    for (int e = tid; e < TL::PLANE; e += TL::THREADS) {
        const int i = DIM == 3 ? x0 + (e % TL::HX) - 1 : x0 + e - 1;
        const int j = DIM == 3 ? y0 + (e / TL::HX) - 1 : 0;
        const unsigned d = (unsigned)e * 8u;
        if (plane_in && (unsigned)i < (unsigned)N && (unsigned)j < (unsigned)N) {
            const ptrdiff_t off = (ptrdiff_t)m * NN + (DIM == 3 ? i + N * j : i);
            cp_async8(su + d, ui + off);
            if (SIG) cp_async8(ss + d, sig + off);
        } else {
            stage_cold<DIM, SIG>(su + d, ss + d, e, m, x0, y0, N, ui, sig, bc);
        }
    }
}

// Dirichlet face value of node (i, j, k) (grid.cpp:53-62), out of line.
template <int DIM>
__device__ __forceinline__ double dirichlet_cold(BcDev bc, int N, int i, int j, int k, int homogeneous) {
    return homogeneous ? 0.0 : dirichlet_value<DIM>(bc, N, i, j, k);
}

template <int DIM, bool SIG>
using SWin = double[SIG ? Tile<DIM>::Q : 1][SIG ? 3 : 1];

// MODE_RELAX:  uo <- relaxed u, duo <- u - u_prev (optional), g = source,
//              diag_slot <- max |A(u)+a u - g| over relax nodes (kernels.cpp:94-137).
// MODE_RESID:  ui = e, g = uo = r (updated in place: r -= A(e) + a e, 0 on
//              Dirichlet nodes, kernels.cpp:243-297), duo = u_tot (+= e,
//              cycle.cpp:194-195, optional), diag_slot <- max|r| (kernels.cpp:407).
template <int DIM, bool SIG, bool HAS_A, int MODE>
__global__ void __launch_bounds__(Tile<DIM>::THREADS, DIM == 3 ? (SIG ? 1 : 2) : 4)
    k_relax_tiled(double* uo, double* duo, const double* __restrict__ ui,
                  const double* g, const double* __restrict__ sig, int N, int zb,
                  RelaxConst rc, BcDev bc, unsigned long long* diag_slot, int* flag) {
    using TL = Tile<DIM>;
    constexpr int Q = TL::Q, NST = TL::NST, D = TL::D, L = TL::LOADS;
    constexpr bool RESID = MODE == MODE_RESID;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Ring<DIM, SIG, MODE>& R = *reinterpret_cast<Ring<DIM, SIG, MODE>*>(smem_raw);

    const int tx = threadIdx.x, ty = DIM == 3 ? threadIdx.y : 0;
    const int tid = tx + TL::X * ty;
    const int x0 = blockIdx.x * TL::X, y0 = DIM == 3 ? blockIdx.y * TL::Y : 0;
    const int m0 = blockIdx.z * zb;
    const int mend = min(m0 + zb, N);  // exclusive
    const int xi = x0 + tx, yi = y0 + ty;
    const bool col_ok = xi < N && (DIM == 2 || yi < N);
    const ptrdiff_t NN = DIM == 3 ? (ptrdiff_t)N * N : (ptrdiff_t)N;  // plane stride
    const int own = DIM == 3 ? xi + N * yi : xi;                       // in-plane offset
    // every in-plane halo element of this tile inside the domain?
    const bool inner = x0 >= 1 && x0 + TL::X <= N - 1 &&
                       (DIM == 2 || (y0 >= 1 && y0 + TL::Y <= N - 1));

    // hoisted staging descriptors: in-plane source offset of element l
    // (-1: outside the domain in-plane -> cold path; -2: beyond PLANE)
    int soff[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        const int e = tid + l * TL::THREADS;
        const int i = DIM == 3 ? x0 + (e % TL::HX) - 1 : x0 + e - 1;
        const int j = DIM == 3 ? y0 + (e / TL::HX) - 1 : 0;
        const bool in = (unsigned)i < (unsigned)N && (unsigned)j < (unsigned)N;
        soff[l] = e >= TL::PLANE ? -2 : (in ? (DIM == 3 ? i + N * j : i) : -1);
    }
    const unsigned su0 = (unsigned)__cvta_generic_to_shared(&R.u[0][0]) + (unsigned)tid * 8u;
    const unsigned ss0 = SIG ? (unsigned)__cvta_generic_to_shared(&R.s[0][0]) + (unsigned)tid * 8u : 0u;
    const unsigned sg0 = (unsigned)__cvta_generic_to_shared(&R.g[0][0]) + (unsigned)tid * 8u;
    const unsigned st0 = (unsigned)__cvta_generic_to_shared(&R.t[0][0]) + (unsigned)tid * 8u;
    const bool with_t = RESID && duo != nullptr;

    // Dirichlet status of this column (lowest face id wins, grid.cpp:53-62):
    // x/y faces outrank the z faces, so only z is decided per plane.
    const bool dir_ij = DIM == 3 ? ((xi == 0 && !bc.neu[0]) || (xi == N - 1 && !bc.neu[1]) ||
                                    (yi == 0 && !bc.neu[2]) || (yi == N - 1 && !bc.neu[3]))
                                 : ((xi == 0 && !bc.neu[0]) || (xi == N - 1 && !bc.neu[1]));
    constexpr int fm = DIM == 3 ? 4 : 2;  // marching-axis faces (z in 3D, y in 2D)

    auto stage = [&](int m) {
        const unsigned slot = (unsigned)m & (NST - 1);
        if (m <= mend) {
            const unsigned sb = slot * (unsigned)(TL::PLANE * 8);
            if (inner && (unsigned)m < (unsigned)N) {
                const double* up = ui + (ptrdiff_t)m * NN;
                const double* sp = SIG ? sig + (ptrdiff_t)m * NN : nullptr;
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    if (L * TL::THREADS > TL::PLANE && soff[l] == -2) continue;
                    cp_async8(su0 + sb + l * TL::THREADS * 8, up + soff[l]);
                    if (SIG) cp_async8(ss0 + sb + l * TL::THREADS * 8, sp + soff[l]);
                }
            } else {
                // su0 / ss0 carry this thread's element offset; the general stager walks
                // the plane itself
                stage_general<DIM, SIG>(su0 + sb - (unsigned)tid * 8u, ss0 + sb - (unsigned)tid * 8u, tid, m,
                                        x0, y0, N, ui, sig, bc);
            }
            if (m >= m0 && m < mend && col_ok) {
                cp_async8(sg0 + slot * (unsigned)(TL::INNER * 8), g + (ptrdiff_t)m * NN + own);
                if (RESID && with_t)
                    cp_async8(st0 + slot * (unsigned)(TL::INNER * 8), duo + (ptrdiff_t)m * NN + own);
            }
        }
        cp_async_commit();
    };

    const int rbase = tx + TL::HX * ty;  // window origin in the plane
    auto read_plane = [&](int m, double (&P)[Q][3], SWin<DIM, SIG>& Ps) {
        const int slot = m & (NST - 1);
        // compiler fence: keep the refill after the previous phase's reads
        asm volatile("" ::: "memory");
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                P[q][p] = R.u[slot][rbase + p + TL::HX * q];
                if constexpr (SIG) Ps[q][p] = R.s[slot][rbase + p + TL::HX * q];
            }
    };

    double dmax = 0.0;
    int bad = 0;

    // acc += the terms of one plane (stencil offset r) for one node
    auto plane_terms = [&](double& acc, double& smax, const double (&P)[Q][3],
                           const SWin<DIM, SIG>& Ps, double uc, double sc, int dr) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                const int dq = DIM == 3 ? q - 1 : 0, dp = p - 1;
                if (dr == 0 && dq == 0 && dp == 0) continue;
                double sbar = 1.0;
                if constexpr (SIG) {
                    sbar = 0.5 * (Ps[q][p] + sc);
                    smax = smax < sbar ? sbar : smax;
                }
                acc = stencil_term<SIG>(acc, sbar, P[q][p], uc, dr * dr + dq * dq + dp * dp);
            }
    };

    // finish one node: op, diag, Euler step, Dirichlet override, store
    auto finish = [&](int m, double acc, double smax, double uc, double gc, double tc) {
        const ptrdiff_t pos = (ptrdiff_t)m * NN + own;
        const bool dir = dir_ij || (m == 0 && !bc.neu[fm]) || (m == N - 1 && !bc.neu[fm + 1]);
        const double op = (acc * rc.pref) * rc.inv_s2;
        if constexpr (RESID) {
            // r -= ((acc*pref)*inv_h2 + a*e); r = 0 on Dirichlet nodes
            double rn = gc - (HAS_A ? op + rc.a * uc : op);
            if (dir) rn = 0.0;
            const double ar = fabs(rn);
            dmax = dmax < ar ? ar : dmax;
            uo[pos] = rn;
            if (with_t) duo[pos] = tc + uc;
            return;
        }
        const double omg = op - gc;
        const double diag = HAS_A ? fabs((op + rc.a * uc) - gc) : fabs(omg);
        double value;
        if constexpr (SIG) {
            const double dtau = (rc.safety * rc.kdim) / (rc.inv_s2 * smax);
            if (!(dtau > 0.0)) {
                value = __longlong_as_double(0x7ff8000000000000LL);
            } else {
                const double num = uc + dtau * omg;
                value = HAS_A ? num / (1.0 - dtau * rc.a) : num;
            }
        } else {
            const double num = uc + rc.dtau1 * omg;
            value = HAS_A ? num / rc.denom1 : num;
        }
        if (dir) {
            value = dirichlet_cold<DIM>(bc, N, xi, DIM == 3 ? yi : m, DIM == 3 ? m : 0, rc.homogeneous);
        } else {
            dmax = dmax < diag ? diag : dmax;
        }
        bad |= (__double_as_longlong(value) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
        uo[pos] = value;
        if (duo) duo[pos] = value - uc;
    };

    double X[Q][3], Y[Q][3], Z[Q][3];  // window planes, rotating roles
    SWin<DIM, SIG> Xs, Ys, Zs;

    // one march step over planes m, m+1.  On entry P0 = plane m-1, P1 = m;
    // P2 receives m+1 now and P0 receives m+2 once node m's r = -1 terms
    // and node m+1's r = -1 terms are summed.
    auto step = [&](int m, double (&P0)[Q][3], double (&P1)[Q][3], double (&P2)[Q][3],
                    SWin<DIM, SIG>& S0, SWin<DIM, SIG>& S1, SWin<DIM, SIG>& S2) {
        cp_async_wait<D - 3>();  // planes up to m+2 (and g of m, m+1) have landed
        __syncthreads();
        read_plane(m + 1, P2, S2);
        const double g0 = col_ok ? R.g[m & (NST - 1)][tid] : 0.0;
        const double g1 = col_ok ? R.g[(m + 1) & (NST - 1)][tid] : 0.0;
        double t0 = 0.0, t1 = 0.0;
        if constexpr (RESID) {
            if (col_ok && with_t) {
                t0 = R.t[m & (NST - 1)][tid];
                t1 = R.t[(m + 1) & (NST - 1)][tid];
            }
        }
        // planes m+D, m+D+1 into the slots of planes m-2, m-1 (read two steps ago)
        stage(m + D);
        stage(m + D + 1);
        const bool two = m + 1 < mend;
        const double uc0 = P1[Q / 2][1], uc1 = P2[Q / 2][1];
        double sc0 = 1.0, sc1 = 1.0;
        if constexpr (SIG) {
            sc0 = S1[Q / 2][1];
            sc1 = S2[Q / 2][1];
        }
        double acc0 = 0.0, acc1 = 0.0, smax0 = 0.0, smax1 = 0.0;
        plane_terms(acc0, smax0, P0, S0, uc0, sc0, -1);
        plane_terms(acc1, smax1, P1, S1, uc1, sc1, -1);
        read_plane(m + 2, P0, S0);  // plane m-1 is dead: refill with m+2
        plane_terms(acc0, smax0, P1, S1, uc0, sc0, 0);
        plane_terms(acc1, smax1, P2, S2, uc1, sc1, 0);
        plane_terms(acc0, smax0, P2, S2, uc0, sc0, 1);
        plane_terms(acc1, smax1, P0, S0, uc1, sc1, 1);
        if (col_ok) {
            finish(m, acc0, smax0, uc0, g0, t0);
            if (two) finish(m + 1, acc1, smax1, uc1, g1, t1);
        }
    };

    if (m0 < N) {
        // prologue: planes m0-1 .. m0+D-1 in flight, one group each
#pragma unroll
        for (int s = 0; s < D + 1; ++s) stage(m0 - 1 + s);
        cp_async_wait<D - 1>();  // planes m0-1, m0 landed
        __syncthreads();
        read_plane(m0 - 1, X, Xs);
        read_plane(m0, Y, Ys);
        // window roles rotate (X,Y,Z) -> (Z,X,-) every step; the loop is not
        // unrolled (register moves instead) so its body stays I-cache resident
#pragma unroll 1
        for (int m = m0; m < mend; m += 2) {
            step(m, X, Y, Z, Xs, Ys, Zs);
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
                for (int p = 0; p < 3; ++p) {
                    Y[q][p] = X[q][p];
                    X[q][p] = Z[q][p];
                    if constexpr (SIG) {
                        Ys[q][p] = Xs[q][p];
                        Xs[q][p] = Zs[q][p];
                    }
                }
        }
        cp_async_wait<0>();
    }
    if (RESID) {
        if (diag_slot) block_max_commit(dmax, diag_slot);
    } else {
        block_max_commit(dmax, diag_slot);
        block_or_commit(bad, flag);
    }
}

template <int DIM, bool SIG, bool HAS_A, int MODE>
void launch_t(dim3 grid, dim3 block, cudaStream_t s, double* uo, double* duo, const double* ui,
              const double* g, const double* sigma, int Nc, int zb, const RelaxConst& rc,
              const BcDev& bc, unsigned long long* slot, int* flag) {
    const int bytes = (int)sizeof(Ring<DIM, SIG, MODE>);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_relax_tiled<DIM, SIG, HAS_A, MODE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        configured = true;
    }
    k_relax_tiled<DIM, SIG, HAS_A, MODE><<<grid, block, bytes, s>>>(uo, duo, ui, g, sigma, Nc, zb, rc, bc,
                                                                    slot, flag);
}

template <int DIM, int MODE>
void launch_dim(dim3 grid, dim3 block, bool sig, cudaStream_t s, double* uo, double* duo,
                const double* ui, const double* g, const double* sigma, int Nc, int zb,
                const RelaxConst& rc, const BcDev& bc, unsigned long long* slot, int* flag) {
    if (sig) {
        if (rc.has_a) launch_t<DIM, true, true, MODE>(grid, block, s, uo, duo, ui, g, sigma, Nc, zb, rc, bc, slot, flag);
        else launch_t<DIM, true, false, MODE>(grid, block, s, uo, duo, ui, g, sigma, Nc, zb, rc, bc, slot, flag);
    } else {
        if (rc.has_a) launch_t<DIM, false, true, MODE>(grid, block, s, uo, duo, ui, g, sigma, Nc, zb, rc, bc, slot, flag);
        else launch_t<DIM, false, false, MODE>(grid, block, s, uo, duo, ui, g, sigma, Nc, zb, rc, bc, slot, flag);
    }
}

template <int MODE>
void launch_mode(int dim, bool sig, double* uo, double* duo, const double* ui, const double* g,
                 const double* sigma, int Nc, const RelaxConst& rc, const BcDev& bc,
                 unsigned long long* slot, int* flag, cudaStream_t s);

}  // namespace

int relax_tiled_zb(int dim, int N) {
    if (dim == 2) return N >= 1024 ? 64 : 32;
    return N >= 256 ? 32 : 16;
}

namespace {
template <int MODE>
void launch_mode(int dim, bool sig, double* uo, double* duo, const double* ui, const double* g,
                 const double* sigma, int Nc, const RelaxConst& rc, const BcDev& bc,
                 unsigned long long* slot, int* flag, cudaStream_t s) {
    const int zb = relax_tiled_zb(dim, Nc);
    if (dim == 3) {
        using TL = Tile<3>;
        const dim3 grid((Nc + TL::X - 1) / TL::X, (Nc + TL::Y - 1) / TL::Y, (Nc + zb - 1) / zb);
        launch_dim<3, MODE>(grid, dim3(TL::X, TL::Y), sig, s, uo, duo, ui, g, sigma, Nc, zb, rc, bc, slot, flag);
    } else {
        using TL = Tile<2>;
        const dim3 grid((Nc + TL::X - 1) / TL::X, 1, (Nc + zb - 1) / zb);
        launch_dim<2, MODE>(grid, dim3(TL::X, 1), sig, s, uo, duo, ui, g, sigma, Nc, zb, rc, bc, slot, flag);
    }
}
}  // namespace

void launch_relax_tiled(int dim, bool sig, double* uo, double* duo, const double* ui,
                        const double* g, const double* sigma, int Nc, const RelaxConst& rc,
                        const BcDev& bc, unsigned long long* slot, int* flag, cudaStream_t s) {
    launch_mode<MODE_RELAX>(dim, sig, uo, duo, ui, g, sigma, Nc, rc, bc, slot, flag, s);
}

void launch_residual_tiled(int dim, bool sig, double* r, const double* e, double* utot,
                           const double* sigma, int N, const RelaxConst& rc, const BcDev& bc,
                           unsigned long long* rmax_slot, cudaStream_t s) {
    launch_mode<MODE_RESID>(dim, sig, r, utot, e, r, sigma, N, rc, bc, rmax_slot, nullptr, s);
}

}  // namespace sgmlb
