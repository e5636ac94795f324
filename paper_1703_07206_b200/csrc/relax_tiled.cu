// relax_tiled.cu — the hot kernel: one relaxation pass over a level array of
// the compact engine (every node a subset node, neighbours at +-1 index),
// i.e. the reference's relax branch (kernels.cpp:94-137) and Dirichlet
// branch (kernels.cpp:213-218) at any level v; and, in MODE_RESID, the fused
// residual recurrence at level 0 (kernels.cpp:243-297 + cycle.cpp:194-198).
//
// Storage: ghost-extended padded arrays (device.cuh, ExtLay), so the tile
// halo never needs boundary code.  A CTA owns an X x Y column bundle (3D:
// 32 x 8 nodes, 2D: 128 x 1) and marches along the slowest axis over `zb`
// planes, two planes per step.  Thread 0 streams planes of u (tile + halo),
// g (tile + x halo) and sigma into an NST-deep shared-memory ring with TMA
// (cp.async.bulk.tensor), one full/empty mbarrier pair per slot: consumers
// wait on `full`, each warp releases a slot on `empty` once it has read it,
// and the producer refills a slot only after all warps released it (no
// __syncthreads in the march; warps drift freely within the ring).
// Every thread keeps a 3 x 3 x 3 register window (planes m-1 .. m+1) and
// computes nodes m and m+1: the plane m-1 registers are refilled with m+2
// as soon as node m's r = -1 terms and node m+1's r = -1 terms are summed,
// giving two independent accumulation chains per thread in the reference's
// strict 26-term order.
#include <cuda.h>
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"

namespace sgmlb {

namespace {

// kernel modes: one relaxation pass, or the fused residual recurrence
enum { MODE_RELAX = 0, MODE_RESID = 1 };

template <int DIM>
struct Tile {
    static constexpr int X = DIM == 3 ? 32 : 128;
    static constexpr int Y = DIM == 3 ? 8 : 1;
    static constexpr int HX = X + 2;
    static constexpr int HY = DIM == 3 ? Y + 2 : 1;
    static constexpr int PLANE = HX * HY;
    static constexpr int INNER = X * Y;
    // g / u_tot box: the tile rows plus the x halo, so that the box starts on
    // an even (16-byte aligned) cell as TMA requires in the innermost dim
    static constexpr int GBOX = HX * Y;
    static constexpr int THREADS = X * Y;
    static constexpr int NWARPS = THREADS / 32;
    static constexpr int Q = DIM == 3 ? 3 : 1;               // in-plane y extent of the stencil
    static constexpr int NST = 8;                            // ring depth (planes), power of two
    static constexpr int PLANE_AL = (PLANE + 15) / 16 * 16;  // slots 128-byte aligned
    static constexpr int GBOX_AL = (GBOX + 15) / 16 * 16;
};

template <int DIM, bool SIG, int MODE>
struct __align__(128) TRing {
    double u[Tile<DIM>::NST][Tile<DIM>::PLANE_AL];
    double g[Tile<DIM>::NST][Tile<DIM>::GBOX_AL];
    double s[SIG ? Tile<DIM>::NST : 1][SIG ? Tile<DIM>::PLANE_AL : 16];
    double t[MODE == MODE_RESID ? Tile<DIM>::NST : 1][MODE == MODE_RESID ? Tile<DIM>::GBOX_AL : 16];
    unsigned long long full[Tile<DIM>::NST];
    unsigned long long empty[Tile<DIM>::NST];
};

template <int DIM, bool SIG>
using SWin = double[SIG ? Tile<DIM>::Q : 1][SIG ? 3 : 1];

// MODE_RELAX:  uo <- relaxed u (with mirror ghosts), duo <- u - u_prev (optional),
//              tm_g = source g, diag_slot <- max |A(u)+a u - g| over relax nodes.
// MODE_RESID:  tm_u = e, tm_g = r, uo = r (updated in place: r -= A(e) + a e,
//              0 on Dirichlet nodes), tm_t / duo = u_tot (+= e, optional),
//              diag_slot <- max|r| (kernels.cpp:407-415).
template <int DIM, bool SIG, bool HAS_A, int MODE>
__global__ void __launch_bounds__(Tile<DIM>::THREADS, DIM == 3 ? (SIG ? 1 : 2) : 4)
    k_relax_tma(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_g,
                const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_t,
                double* uo, double* duo, ExtLay L, int zb, RelaxConst rc, BcDev bc,
                unsigned long long* diag_slot, int* flag) {
    using TL = Tile<DIM>;
    constexpr int Q = TL::Q, NST = TL::NST;
    constexpr bool RESID = MODE == MODE_RESID;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TRing<DIM, SIG, MODE>& R = *reinterpret_cast<TRing<DIM, SIG, MODE>*>(smem_raw);

    const int tx = threadIdx.x, ty = DIM == 3 ? threadIdx.y : 0;
    const int tid = tx + TL::X * ty;
    const int lane = tid & 31;
    const int N = L.N;
    const int x0 = blockIdx.x * TL::X, y0 = DIM == 3 ? blockIdx.y * TL::Y : 0;
    const int m0 = blockIdx.z * zb;
    const int mend = min(m0 + zb, N);  // exclusive
    const int xi = x0 + tx, yi = y0 + ty;
    const bool col_ok = xi < N && (DIM == 2 || yi < N);
    const bool with_t = RESID && duo != nullptr;

    // Dirichlet status of this column (lowest face id wins, grid.cpp:53-62):
    // x/y faces outrank the z faces, so only z is decided per plane.
    const bool dir_ij = DIM == 3 ? ((xi == 0 && !bc.neu[0]) || (xi == N - 1 && !bc.neu[1]) ||
                                    (yi == 0 && !bc.neu[2]) || (yi == N - 1 && !bc.neu[3]))
                                 : ((xi == 0 && !bc.neu[0]) || (xi == N - 1 && !bc.neu[1]));
    constexpr int fm = DIM == 3 ? 4 : 2;  // marching-axis faces (z in 3D, y in 2D)

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&R.full[s], 1);
            mbar_init(&R.empty[s], TL::NWARPS);
        }
        mbar_fence_init();
    }
    __syncthreads();

    constexpr unsigned BU = TL::PLANE * 8, BG = TL::GBOX * 8;
    // producer (thread 0): plane m -> slot; waits for the slot's previous use
    auto issue = [&](int m) {
        const int p = m - (m0 - 1);
        const int s = p & (NST - 1), k = p / NST;
        if (k > 0) mbar_wait(&R.empty[s], (k - 1) & 1);
        const bool comp = m >= m0 && m < mend;
        const unsigned bytes = BU + (SIG ? BU : 0u) + (comp ? BG + (with_t ? BG : 0u) : 0u);
        mbar_expect_tx(&R.full[s], bytes);
        if (DIM == 3) {
            tma_load_3d(R.u[s], &tm_u, x0, y0, m + 1, &R.full[s]);
            if (SIG) tma_load_3d(R.s[s], &tm_s, x0, y0, m + 1, &R.full[s]);
            if (comp) {
                tma_load_3d(R.g[s], &tm_g, x0, y0 + 1, m + 1, &R.full[s]);
                if (with_t) tma_load_3d(R.t[s], &tm_t, x0, y0 + 1, m + 1, &R.full[s]);
            }
        } else {
            tma_load_2d(R.u[s], &tm_u, x0, m + 1, &R.full[s]);
            if (SIG) tma_load_2d(R.s[s], &tm_s, x0, m + 1, &R.full[s]);
            if (comp) {
                tma_load_2d(R.g[s], &tm_g, x0, m + 1, &R.full[s]);
                if (with_t) tma_load_2d(R.t[s], &tm_t, x0, m + 1, &R.full[s]);
            }
        }
    };
    auto slot_of = [&](int m) { return (m - (m0 - 1)) & (NST - 1); };
    auto wait_plane = [&](int m) {
        const int p = m - (m0 - 1);
        mbar_wait(&R.full[p & (NST - 1)], (p / NST) & 1);
    };
    auto release = [&](int m) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&R.empty[slot_of(m)]);
    };

    const int rbase = tx + TL::HX * ty;  // window origin in the plane
    auto read_plane = [&](int m, double (&P)[Q][3], SWin<DIM, SIG>& Ps) {
        const int slot = slot_of(m);
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

    // finish one node: op, diag / residual, Euler step, Dirichlet override, store
    auto finish = [&](int m, double acc, double smax, double uc, double gc, double tc) {
        const int i = xi, j = DIM == 3 ? yi : m, k = DIM == 3 ? m : 0;
        const bool dir = dir_ij || (m == 0 && !bc.neu[fm]) || (m == N - 1 && !bc.neu[fm + 1]);
        const double op = (acc * rc.pref) * rc.inv_s2;
        if constexpr (RESID) {
            double rn = gc - (HAS_A ? op + rc.a * uc : op);
            if (dir) rn = 0.0;
            const double ar = fabs(rn);
            dmax = dmax < ar ? ar : dmax;
            store_ext<DIM>(uo, L, i, j, k, rn);
            if (with_t) duo[eix<DIM>(L, i, j, k)] = tc + uc;
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
            value = rc.homogeneous ? 0.0 : dirichlet_value<DIM>(bc, N, i, j, k);
        } else {
            dmax = dmax < diag ? diag : dmax;
        }
        bad |= (__double_as_longlong(value) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
        store_ext<DIM>(uo, L, i, j, k, value);
        if (duo) duo[eix<DIM>(L, i, j, k)] = value - uc;
    };

    double X[Q][3], Y[Q][3], Z[Q][3];  // window planes, rotating roles
    SWin<DIM, SIG> Xs, Ys, Zs;

    if (m0 < N) {
        int next = m0 - 1;  // next plane the producer issues
        if (tid == 0)
            for (; next <= mend && next <= m0 + NST - 2; ++next) issue(next);
        wait_plane(m0 - 1);
        read_plane(m0 - 1, X, Xs);
        wait_plane(m0);
        read_plane(m0, Y, Ys);
        release(m0 - 1);

#pragma unroll 1
        for (int m = m0; m < mend; m += 2) {
            const bool two = m + 1 < mend;
            wait_plane(m + 1);
            read_plane(m + 1, Z, Zs);
            double g0 = 0.0, g1 = 0.0, t0 = 0.0, t1 = 0.0;
            if (col_ok) {
                const int gi = tx + 1 + TL::HX * ty;  // this node in the g / u_tot box
                g0 = R.g[slot_of(m)][gi];
                if (two) g1 = R.g[slot_of(m + 1)][gi];
                if (with_t) {
                    t0 = R.t[slot_of(m)][gi];
                    if (two) t1 = R.t[slot_of(m + 1)][gi];
                }
            }
            const double uc0 = Y[Q / 2][1], uc1 = Z[Q / 2][1];
            double sc0 = 1.0, sc1 = 1.0;
            if constexpr (SIG) {
                sc0 = Ys[Q / 2][1];
                sc1 = Zs[Q / 2][1];
            }
            double acc0 = 0.0, acc1 = 0.0, smax0 = 0.0, smax1 = 0.0;
            plane_terms(acc0, smax0, X, Xs, uc0, sc0, -1);
            plane_terms(acc1, smax1, Y, Ys, uc1, sc1, -1);
            if (two) {  // plane m-1 is dead: refill with m+2
                wait_plane(m + 2);
                read_plane(m + 2, X, Xs);
            }
            plane_terms(acc0, smax0, Y, Ys, uc0, sc0, 0);
            plane_terms(acc1, smax1, Z, Zs, uc1, sc1, 0);
            plane_terms(acc0, smax0, Z, Zs, uc0, sc0, 1);
            plane_terms(acc1, smax1, X, Xs, uc1, sc1, 1);
            if (col_ok) {
                finish(m, acc0, smax0, uc0, g0, t0);
                if (two) finish(m + 1, acc1, smax1, uc1, g1, t1);
            }
            release(m);
            release(m + 1);
            if (tid == 0)
                for (; next <= mend && next <= m + NST - 1; ++next) issue(next);
            // window roles rotate (X, Y, Z) -> (Z, X, -): next P0 = m+1, P1 = m+2
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
    }
    if (RESID) {
        if (diag_slot) block_max_commit(dmax, diag_slot);
    } else {
        block_max_commit(dmax, diag_slot);
        block_or_commit(bad, flag);
    }
}

template <int DIM, bool SIG, bool HAS_A, int MODE>
void launch_t(dim3 grid, dim3 block, cudaStream_t s, const TmaSet& tm, double* uo, double* duo,
              const ExtLay& L, int zb, const RelaxConst& rc, const BcDev& bc,
              unsigned long long* slot, int* flag) {
    const int bytes = (int)sizeof(TRing<DIM, SIG, MODE>);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_relax_tma<DIM, SIG, HAS_A, MODE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        configured = true;
    }
    k_relax_tma<DIM, SIG, HAS_A, MODE><<<grid, block, bytes, s>>>(tm.u, tm.g, tm.s, tm.t, uo, duo, L, zb,
                                                                  rc, bc, slot, flag);
}

template <int DIM, int MODE>
void launch_dim(dim3 grid, dim3 block, bool sig, cudaStream_t s, const TmaSet& tm, double* uo,
                double* duo, const ExtLay& L, int zb, const RelaxConst& rc, const BcDev& bc,
                unsigned long long* slot, int* flag) {
    if (sig) {
        if (rc.has_a) launch_t<DIM, true, true, MODE>(grid, block, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
        else launch_t<DIM, true, false, MODE>(grid, block, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
    } else {
        if (rc.has_a) launch_t<DIM, false, true, MODE>(grid, block, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
        else launch_t<DIM, false, false, MODE>(grid, block, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
    }
}

template <int MODE>
void launch_mode(int dim, bool sig, const TmaSet& tm, double* uo, double* duo, const ExtLay& L,
                 const RelaxConst& rc, const BcDev& bc, unsigned long long* slot, int* flag,
                 cudaStream_t s) {
    const int Nc = L.N;
    const int zb = relax_tiled_zb(dim, Nc);
    if (dim == 3) {
        using TL = Tile<3>;
        const dim3 grid((Nc + TL::X - 1) / TL::X, (Nc + TL::Y - 1) / TL::Y, (Nc + zb - 1) / zb);
        launch_dim<3, MODE>(grid, dim3(TL::X, TL::Y), sig, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
    } else {
        using TL = Tile<2>;
        const dim3 grid((Nc + TL::X - 1) / TL::X, 1, (Nc + zb - 1) / zb);
        launch_dim<2, MODE>(grid, dim3(TL::X, 1), sig, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
    }
}

}  // namespace

int relax_tiled_zb(int dim, int N) {
    if (dim == 2) return N >= 1024 ? 64 : 32;
    return N >= 256 ? 32 : 16;
}

void tile_boxes(int dim, unsigned* box_u, unsigned* box_g) {
    if (dim == 3) {
        box_u[0] = Tile<3>::HX; box_u[1] = Tile<3>::HY; box_u[2] = 1;
        box_g[0] = Tile<3>::HX; box_g[1] = Tile<3>::Y;  box_g[2] = 1;
    } else {
        box_u[0] = Tile<2>::HX; box_u[1] = 1; box_u[2] = 1;
        box_g[0] = Tile<2>::HX; box_g[1] = 1; box_g[2] = 1;
    }
}

void launch_relax_tma(int dim, bool sig, const TmaSet& tm, double* uo, double* duo,
                      const ExtLay& L, const RelaxConst& rc, const BcDev& bc,
                      unsigned long long* slot, int* flag, cudaStream_t s) {
    launch_mode<MODE_RELAX>(dim, sig, tm, uo, duo, L, rc, bc, slot, flag, s);
}

void launch_residual_tma(int dim, bool sig, const TmaSet& tm, double* r, double* utot,
                         const ExtLay& L, const RelaxConst& rc, const BcDev& bc,
                         unsigned long long* rmax_slot, cudaStream_t s) {
    launch_mode<MODE_RESID>(dim, sig, tm, r, utot, L, rc, bc, rmax_slot, nullptr, s);
}

}  // namespace sgmlb
