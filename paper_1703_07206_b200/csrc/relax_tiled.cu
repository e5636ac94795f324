// relax_tiled.cu — the hot kernel: one relaxation pass over a level array of
// the compact engine (every node a subset node, neighbours at +-1 index),
// i.e. the reference's relax branch (kernels.cpp:94-137) and Dirichlet
// branch (kernels.cpp:213-218) at any level v; and, in MODE_RESID, the fused
// residual recurrence at level 0 (kernels.cpp:243-297 + cycle.cpp:194-198).
//
// Storage: ghost-extended padded arrays (device.cuh, ExtLay), so the tile
// halo never needs boundary code.  A CTA owns an X x ROWS column bundle (3D:
// 32 x 16 nodes, 2D: 128 x 1) and marches along the slowest axis over `zb`
// planes, one plane per step.  Thread 0 streams planes of u (tile + halo),
// g (tile rows + x halo: TMA boxes must start 16-byte aligned) and sigma
// into an NST-deep shared-memory ring with TMA (cp.async.bulk.tensor), one
// full/empty mbarrier pair per slot: consumers wait on `full`, each warp
// releases a slot on `empty` once it has read it, and the producer refills a
// slot only after all warps released it (no __syncthreads in the march).
//
// In 3D every thread computes RT = 2 adjacent rows (y, y+1) of the plane: it
// keeps a (RT+2) x 3 register window of each of planes m-1, m, m+1 (12
// values per plane, so 6 shared loads per node) and the two nodes'
// accumulation chains interleave term by term in the reference's strict
// 26-term order.  The window roles rotate with period 3, so the march is
// unrolled three steps and no register moves are issued.
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
    static constexpr int X = DIM == 3 ? 32 : 128;      // nodes per row (= threads in x)
    static constexpr int TY = DIM == 3 ? 8 : 1;        // thread rows
    static constexpr int RT = DIM == 3 ? 2 : 1;        // node rows per thread
    static constexpr int ROWS = TY * RT;               // node rows per CTA
    static constexpr int HX = X + 2;
    static constexpr int HY = DIM == 3 ? ROWS + 2 : 1;
    static constexpr int PLANE = HX * HY;              // u / sigma box (tile + halo)
    static constexpr int GBOX = HX * ROWS;             // g / u_tot box (tile rows + x halo)
    static constexpr int THREADS = X * TY;
    static constexpr int NWARPS = THREADS / 32;
    static constexpr int WR = DIM == 3 ? RT + 2 : 1;   // window rows per plane
    static constexpr int NST = 8;                      // ring depth (planes), power of two
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

template <int DIM>
using Win = double[Tile<DIM>::WR][3];
template <int DIM, bool SIG>
using SWin = double[SIG ? Tile<DIM>::WR : 1][SIG ? 3 : 1];

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
    constexpr int NST = TL::NST, RT = TL::RT, WR = TL::WR;
    constexpr bool RESID = MODE == MODE_RESID;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TRing<DIM, SIG, MODE>& R = *reinterpret_cast<TRing<DIM, SIG, MODE>*>(smem_raw);

    const int tx = threadIdx.x, ty = DIM == 3 ? threadIdx.y : 0;
    const int tid = tx + TL::X * ty;
    const int lane = tid & 31;
    const int N = L.N;
    const int x0 = blockIdx.x * TL::X, y0 = DIM == 3 ? blockIdx.y * TL::ROWS : 0;
    const int m0 = blockIdx.z * zb;
    const int mend = min(m0 + zb, N);  // exclusive
    const int xi = x0 + tx;
    const int yb = y0 + ty * RT;       // first node row of this thread (3D)
    const bool with_t = RESID && duo != nullptr;
    bool ok[RT];
#pragma unroll
    for (int a = 0; a < RT; ++a) ok[a] = xi < N && (DIM == 2 || yb + a < N);

    constexpr int fm = DIM == 3 ? 4 : 2;  // marching-axis faces (z in 3D, y in 2D)
    // can any node of this CTA lie on a Dirichlet face?  (block-uniform)
    const bool edge_tile = x0 == 0 || x0 + TL::X >= N - 1 ||
                           (DIM == 3 && (y0 == 0 || y0 + TL::ROWS >= N - 1));
    const bool maybe_dir =
        (edge_tile && (!bc.neu[0] || !bc.neu[1] || (DIM == 3 && (!bc.neu[2] || !bc.neu[3])))) ||
        (m0 == 0 && !bc.neu[fm]) || (mend == N && !bc.neu[fm + 1]);

    // per-row constants: output offset at plane 0, Dirichlet status of the
    // column (x/y faces outrank the marching-axis faces, grid.cpp:53-62) and
    // whether the node has mirror ghost cells in x/y
    ptrdiff_t obase[RT];
    bool dir_row[RT], mir_row[RT];
    double val_row[RT];
#pragma unroll
    for (int a = 0; a < RT; ++a) {
        const int j = DIM == 3 ? yb + a : 0;
        obase[a] = eix<DIM>(L, xi, j, -1);  // + (m + 1) * plane
        if (DIM == 2) obase[a] = (ptrdiff_t)(xi + 1);
        dir_row[a] = (xi == 0 && !bc.neu[0]) || (xi == N - 1 && !bc.neu[1]) ||
                     (DIM == 3 && ((j == 0 && !bc.neu[2]) || (j == N - 1 && !bc.neu[3])));
        val_row[a] = rc.homogeneous ? 0.0 : dirichlet_value<DIM>(bc, N, xi, j, 0);
        mir_row[a] = xi == 1 || xi == N - 2 || (DIM == 3 && (j == 1 || j == N - 2));
    }
    const bool dir_lo = !bc.neu[fm], dir_hi = !bc.neu[fm + 1];
    const double val_lo = rc.homogeneous ? 0.0 : bc.val[fm];
    const double val_hi = rc.homogeneous ? 0.0 : bc.val[fm + 1];

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

    const int wbase = tx + TL::HX * (DIM == 3 ? ty * RT : 0);  // window origin in the u box
    auto read_plane = [&](int m, Win<DIM>& P, SWin<DIM, SIG>& Ps) {
        const int slot = slot_of(m);
#pragma unroll
        for (int w = 0; w < WR; ++w)
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                P[w][p] = R.u[slot][wbase + p + TL::HX * w];
                if constexpr (SIG) Ps[w][p] = R.s[slot][wbase + p + TL::HX * w];
            }
    };

    double dmax = 0.0;
    int bad = 0;

    // the RT nodes' terms of one stencil plane (offset dr), interleaved term
    // by term so the independent accumulation chains overlap
    auto plane_terms = [&](double (&acc)[RT], double (&smax)[RT], const Win<DIM>& P,
                           const SWin<DIM, SIG>& Ps, const double (&uc)[RT], const double (&sc)[RT],
                           int dr) {
#pragma unroll
        for (int q = (DIM == 3 ? -1 : 0); q <= (DIM == 3 ? 1 : 0); ++q)
#pragma unroll
            for (int p = -1; p <= 1; ++p) {
                if (dr == 0 && q == 0 && p == 0) continue;
                const int l2 = dr * dr + q * q + p * p;
#pragma unroll
                for (int a = 0; a < RT; ++a) {
                    const int w = DIM == 3 ? a + q + 1 : 0;
                    double sbar = 1.0;
                    if constexpr (SIG) {
                        sbar = 0.5 * (Ps[w][p + 1] + sc[a]);
                        smax[a] = smax[a] < sbar ? sbar : smax[a];
                    }
                    acc[a] = stencil_term<SIG>(acc[a], sbar, P[w][p + 1], uc[a], l2);
                }
            }
    };

    // finish one node: op, diag / residual, Euler step, Dirichlet override, store
    auto finish = [&](int m, int a, double acc, double smax, double uc, double gc, double tc) {
        const ptrdiff_t pos = obase[a] + (ptrdiff_t)(m + 1) * L.plane;
        bool dir = false;
        double dval = 0.0;
        if (maybe_dir) {
            dir = dir_row[a] || (m == 0 && dir_lo) || (m == N - 1 && dir_hi);
            dval = dir_row[a] ? val_row[a] : (m == 0 && dir_lo ? val_lo : val_hi);
        }
        const double op = (acc * rc.pref) * rc.inv_s2;
        double value;
        if constexpr (RESID) {
            value = gc - (HAS_A ? op + rc.a * uc : op);
            if (dir) value = 0.0;
            const double ar = fabs(value);
            dmax = dmax < ar ? ar : dmax;
            if (with_t) duo[pos] = tc + uc;
        } else {
            const double omg = op - gc;
            const double diag = HAS_A ? fabs((op + rc.a * uc) - gc) : fabs(omg);
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
                value = dval;
            } else {
                dmax = dmax < diag ? diag : dmax;
            }
            bad |= (__double_as_longlong(value) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
            if (duo) duo[pos] = value - uc;
        }
        uo[pos] = value;
        if (mir_row[a] || m == 1 || m == N - 2)
            store_mirrors<DIM>(uo, L, xi, DIM == 3 ? yb + a : m, DIM == 3 ? m : 0, value);
    };

    Win<DIM> X, Y, Z;  // window planes, rotating roles
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

        // one plane: P0 = m-1, P1 = m (held), P2 <- m+1
        auto step = [&](int m, Win<DIM>& P0, Win<DIM>& P1, Win<DIM>& P2, SWin<DIM, SIG>& S0,
                        SWin<DIM, SIG>& S1, SWin<DIM, SIG>& S2) {
            if (tid == 0)
                for (; next <= mend && next <= m + NST - 2; ++next) issue(next);
            wait_plane(m + 1);
            read_plane(m + 1, P2, S2);
            const int sm = slot_of(m);
            double uc[RT], sc[RT], acc[RT], smax[RT], gc[RT], tc[RT];
#pragma unroll
            for (int a = 0; a < RT; ++a) {
                const int gi = tx + 1 + TL::HX * (DIM == 3 ? ty * RT + a : 0);  // node in the g box
                gc[a] = R.g[sm][gi];
                tc[a] = with_t ? R.t[sm][gi] : 0.0;
                uc[a] = P1[DIM == 3 ? a + 1 : 0][1];
                sc[a] = 1.0;
                if constexpr (SIG) sc[a] = S1[DIM == 3 ? a + 1 : 0][1];
                acc[a] = 0.0;
                smax[a] = 0.0;
            }
            plane_terms(acc, smax, P0, S0, uc, sc, -1);
            plane_terms(acc, smax, P1, S1, uc, sc, 0);
            plane_terms(acc, smax, P2, S2, uc, sc, 1);
#pragma unroll
            for (int a = 0; a < RT; ++a)
                if (ok[a]) finish(m, a, acc[a], smax[a], uc[a], gc[a], tc[a]);
            release(m);
        };
        // roles rotate (P0, P1, P2) -> (P1, P2, P0) each plane: period 3
#pragma unroll 1
        for (int m = m0; m < mend; m += 3) {
            step(m, X, Y, Z, Xs, Ys, Zs);
            if (m + 1 >= mend) break;
            step(m + 1, Y, Z, X, Ys, Zs, Xs);
            if (m + 2 >= mend) break;
            step(m + 2, Z, X, Y, Zs, Xs, Ys);
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
        const dim3 grid((Nc + TL::X - 1) / TL::X, (Nc + TL::ROWS - 1) / TL::ROWS, (Nc + zb - 1) / zb);
        launch_dim<3, MODE>(grid, dim3(TL::X, TL::TY), sig, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
    } else {
        using TL = Tile<2>;
        const dim3 grid((Nc + TL::X - 1) / TL::X, 1, (Nc + zb - 1) / zb);
        launch_dim<2, MODE>(grid, dim3(TL::X, 1), sig, s, tm, uo, duo, L, zb, rc, bc, slot, flag);
    }
}

}  // namespace

int relax_tiled_zb(int dim, int N) {
    if (dim == 2) return N >= 1024 ? 128 : 32;
    return N >= 512 ? 64 : (N >= 128 ? 32 : 16);
}

void tile_boxes(int dim, unsigned* box_u, unsigned* box_g) {
    if (dim == 3) {
        box_u[0] = Tile<3>::HX; box_u[1] = Tile<3>::HY;   box_u[2] = 1;
        box_g[0] = Tile<3>::HX; box_g[1] = Tile<3>::ROWS; box_g[2] = 1;
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
