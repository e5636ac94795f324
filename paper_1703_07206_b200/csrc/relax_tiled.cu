// relax_tiled.cu — the hot kernel: one relaxation pass over a level array of
// the compact engine (every node a subset node, neighbours at +-1 index),
// i.e. the reference's relax branch (kernels.cpp:94-137) at any level v; and,
// in MODE_RESID, the fused residual recurrence at level 0 (kernels.cpp:243-297
// + cycle.cpp:194-198).
//
// Range.  The kernel covers the box of nodes that are NOT on a Dirichlet face
// (Neumann faces are included).  Dirichlet nodes take their face value in
// every pass (kernels.cpp:213-218); the engine keeps that value resident in
// the output buffers (engine.cpp, face states), so the kernel has no
// boundary code at all, and the tile grid loses the thin boundary tiles.
//
// Storage: ghost-extended padded arrays (device.cuh, ExtLay), so the tile
// halo never needs boundary code either.  A CTA owns an X x ROWS column
// bundle (3D: 32 x 16 nodes, 2D: 128 x 1) and marches along the slowest axis
// over `zb` planes, one plane per step.  Planes of u (tile + halo), g (tile
// rows + x halo) and sigma are streamed with TMA (cp.async.bulk.tensor) into
// an NST-deep shared-memory ring, one full/empty mbarrier pair per slot.  TMA
// boxes must start 16-byte aligned in x, so boxes start at the even cell at
// or below the halo and the window carries an offset xoff in {0, 1}.  The
// producer role rotates over the warps (warp (m - m0) % NWARPS issues plane
// m + LEAD in step m), so every warp runs the same instruction stream;
// consumers wait on `full`, each warp releases a slot on `empty`.
//
// In 3D every thread computes RT = 2 adjacent rows (y, y+1) of the plane: it
// keeps a (RT+2) x 3 register window of the two newest planes (12 values per
// plane, so 6 shared loads per node) and the two nodes' accumulation chains
// interleave term by term in the reference's strict 26-term order.  Terms
// are summed as planes arrive (see the march); the window roles alternate
// with period 2, so the march is unrolled two steps and no register moves
// are issued.
#include <algorithm>
#include <cstdlib>

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
    static constexpr int XP = DIM == 3 ? 2 : 1;        // x nodes per thread (adjacent)
    static constexpr int X = DIM == 3 ? 32 : 128;      // threads in x
    static constexpr int NX = X * XP;                  // nodes per row
    static constexpr int TY = DIM == 3 ? 8 : 1;        // thread rows
    static constexpr int RT = DIM == 3 ? 2 : 1;        // node rows per thread
    static constexpr int ROWS = TY * RT;               // node rows per CTA
    // box widths: 3D tiles start at even x (box = halo exactly); 2D tiles
    // start at lo.x and carry the alignment offset xoff in {0, 1}
    static constexpr int HXU = DIM == 3 ? NX + 2 : NX + 4;  // u / sigma box width
    static constexpr int HXG = NX + 2;                      // g / u_tot box width
    static constexpr int HY = DIM == 3 ? ROWS + 2 : 1;
    static constexpr int PLANE = HXU * HY;             // u / sigma box (tile + halo)
    static constexpr int GBOX = HXG * ROWS;            // g / u_tot box (tile rows)
    static constexpr int THREADS = X * TY;
    static constexpr int NWARPS = THREADS / 32;
    static constexpr int WR = DIM == 3 ? RT + 2 : 1;   // window rows per plane
    static constexpr int WC = XP + 2;                  // window columns per row
    static constexpr int PLANE_AL = (PLANE + 15) / 16 * 16;  // slots 128-byte aligned
    static constexpr int GBOX_AL = (GBOX + 15) / 16 * 16;
};

// ring depth (planes) and producer lead: 3D relax passes keep two CTAs per
// SM in 2 x 107 KB; the residual pass (one more stream) uses a shallower ring
template <int DIM, bool SIG, int MODE>
struct Ring {
    static constexpr int NST = DIM == 2 ? 8 : (MODE == MODE_RESID && !SIG ? 4 : 6);
    static constexpr int LEAD = NST - 3 > 1 ? NST - 3 : NST - 2;  // step q issues plane q + LEAD
};

template <int DIM, bool SIG, int MODE>
struct __align__(128) TRing {
    static constexpr int NST = Ring<DIM, SIG, MODE>::NST;
    double u[NST][Tile<DIM>::PLANE_AL];
    double g[NST][Tile<DIM>::GBOX_AL];
    double s[SIG ? NST : 1][SIG ? Tile<DIM>::PLANE_AL : 16];
    double t[(MODE == MODE_RESID || SIG) ? NST : 1][(MODE == MODE_RESID || SIG) ? Tile<DIM>::GBOX_AL : 16];
    unsigned long long full[NST];
    unsigned long long empty[NST];
};

template <int DIM>
using Win = double[Tile<DIM>::WR][Tile<DIM>::WC];
template <int DIM, bool SIG>
using SWin = double[SIG ? Tile<DIM>::WR : 1][SIG ? Tile<DIM>::WC : 1];
template <int DIM>
using NodeD = double[Tile<DIM>::RT][Tile<DIM>::XP];

// MODE_RELAX:  uo <- relaxed u (with mirror ghosts), duo <- u - u_prev (DUO),
//              tm_g = source g, diag_slot <- max |A(u)+a u - g| over the range.
// MODE_RESID:  tm_u = e, tm_g = r, uo = r (updated in place: r -= A(e) + a e),
//              tm_t / duo = u_tot (+= e, DUO), diag_slot <- max|r|
//              (kernels.cpp:407-415; r is 0 on Dirichlet faces).
// Range: data nodes [lo.x, hi.x] x [lo.y, hi.y] x [lo.z, hi.z] (2D: x, y),
// z indices local to the array (z-slabs).
// CMP: the compact 5/7-point stencil family (axis offsets only, SURVEY.md 8a
// row a23); the constants (prefactor, step) come in rc.
template <int DIM, bool SIG, bool HAS_A, int MODE, bool DUO, bool CMP>
__global__ void __launch_bounds__(Tile<DIM>::THREADS, DIM == 3 ? (SIG ? 1 : 2) : 4)
    k_relax_tma(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_g,
                const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_t,
                double* uo, double* duo, ExtLay L, int3 lo, int3 hi, int zb, RelaxConst rc,
                unsigned long long* diag_slot, int* flag, int pass_slot) {
    using TL = Tile<DIM>;
    constexpr int NST = Ring<DIM, SIG, MODE>::NST, LEAD = Ring<DIM, SIG, MODE>::LEAD;
    constexpr int RT = TL::RT, WR = TL::WR, XP = TL::XP, WC = TL::WC;
    constexpr bool RESID = MODE == MODE_RESID;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TRing<DIM, SIG, MODE>& R = *reinterpret_cast<TRing<DIM, SIG, MODE>*>(smem_raw);

    const int tx = threadIdx.x, ty = DIM == 3 ? threadIdx.y : 0;
    const int tid = tx + TL::X * ty;
    const int lane = tid & 31, warp = tid >> 5;
    const int N = L.N;
    const int x0 = (DIM == 3 ? (lo.x & ~1) : lo.x) + blockIdx.x * TL::NX;
    const int y0 = DIM == 3 ? lo.y + blockIdx.y * TL::ROWS : 0;
    const int zlo = DIM == 3 ? lo.z : lo.y, zhi = DIM == 3 ? hi.z : hi.y;  // marching axis
    const int m0 = zlo + blockIdx.z * zb;
    const int mend = min(m0 + zb, zhi + 1);  // exclusive
    const int xb = x0 & ~1;                   // box start cell (ext index of data x0 - 1 is x0)
    const int xoff = x0 - xb;                 // 0 in 3D
    const int xi = x0 + tx * XP;              // first node column of this thread
    const int yb = y0 + ty * RT;              // first node row of this thread (3D)
    // node (a, b) in range / with mirror ghost cells in x, y: bit a * XP + b
    unsigned okm = 0, mirm = 0;
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < XP; ++b) {
            const int i = xi + b, j = yb + a;
            if (i >= lo.x && i <= hi.x && (DIM == 2 || j <= hi.y)) okm |= 1u << (a * XP + b);
            if (DIM == 3 && (j == 1 || j == N - 2)) mirm |= 1u << (a * XP + b);  // (x mirrors inline)
        }
    constexpr unsigned ALL = (1u << (RT * XP)) - 1;

    // output offset of node (0, 0) at plane m = -1 (advanced one plane per step)
    ptrdiff_t opos = DIM == 3 ? eix<DIM>(L, xi, yb, -1) : (ptrdiff_t)(xi + 1);
    const ptrdiff_t ostep = DIM == 3 ? (ptrdiff_t)L.plane : (ptrdiff_t)L.Px;

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&R.full[s], 1);
            mbar_init(&R.empty[s], TL::NWARPS);
        }
        mbar_fence_init();
    }
    pdl_begin();  // the predecessor's outputs are complete from here on
    // guarded residual (pass_slot < 0): a failed cycle (flag[0], written only
    // by the cycle's passes, never by this kernel) leaves r and u_tot as they
    // are, so the host checks the failure after the recurrence
    if (RESID && pass_slot < 0 && *(const volatile int*)flag) return;
    __syncthreads();

    const unsigned a_full = smem_u32(&R.full[0]), a_empty = smem_u32(&R.empty[0]);
    const unsigned a_u = smem_u32(&R.u[0][0]), a_g = smem_u32(&R.g[0][0]);
    const unsigned a_s = smem_u32(&R.s[0][0]), a_t = smem_u32(&R.t[0][0]);
    constexpr unsigned BU = TL::PLANE * 8, BG = TL::GBOX * 8;
    // producer (one lane): plane m -> slot; waits for the slot's previous use
    auto issue = [&](int m) {
        const unsigned p = (unsigned)(m - m0 + 1);
        const unsigned s = p % NST, k = p / NST;
        if (k > 0) mbar_wait_u32(a_empty + 8 * s, (k - 1) & 1);
        const bool comp = m >= m0 && m < mend;
        // t box: u_tot (residual) or the per-node pseudo-time step (sigma relax)
        constexpr bool TBOX = (DUO && RESID) || (SIG && !RESID);
        const unsigned bytes = BU + (SIG ? BU : 0u) + (comp ? BG + (TBOX ? BG : 0u) : 0u);
        const unsigned bar = a_full + 8 * s;
        mbar_expect_tx_u32(bar, bytes);
        if (DIM == 3) {
            tma_load_3d_u32(a_u + s * (TL::PLANE_AL * 8), &tm_u, xb, y0, m + 1, bar);
            if (SIG) tma_load_3d_u32(a_s + s * (TL::PLANE_AL * 8), &tm_s, xb, y0, m + 1, bar);
            if (comp) {
                tma_load_3d_u32(a_g + s * (TL::GBOX_AL * 8), &tm_g, xb, y0 + 1, m + 1, bar);
                if (TBOX) tma_load_3d_u32(a_t + s * (TL::GBOX_AL * 8), &tm_t, xb, y0 + 1, m + 1, bar);
            }
        } else {
            tma_load_2d_u32(a_u + s * (TL::PLANE_AL * 8), &tm_u, xb, m + 1, bar);
            if (SIG) tma_load_2d_u32(a_s + s * (TL::PLANE_AL * 8), &tm_s, xb, m + 1, bar);
            if (comp) {
                tma_load_2d_u32(a_g + s * (TL::GBOX_AL * 8), &tm_g, xb, m + 1, bar);
                if (TBOX) tma_load_2d_u32(a_t + s * (TL::GBOX_AL * 8), &tm_t, xb, m + 1, bar);
            }
        }
    };
    auto release = [&](unsigned slot) {
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(a_empty + 8 * slot);
    };

    const int wbase = tx * XP + xoff + TL::HXU * (DIM == 3 ? ty * RT : 0);  // window origin in the u box
    const int gbase = tx * XP + 1 + xoff + TL::HXG * (DIM == 3 ? ty * RT : 0);
    auto read_plane = [&](unsigned slot, Win<DIM>& P, SWin<DIM, SIG>& Ps) {
#pragma unroll
        for (int w = 0; w < WR; ++w) {
            const double* row = &R.u[slot][wbase + TL::HXU * w];
            if constexpr (XP == 2) {
                // 16-byte aligned pairs: box columns 2 tx .. 2 tx + 3
                const double2 lo2 = *reinterpret_cast<const double2*>(row);
                const double2 hi2 = *reinterpret_cast<const double2*>(row + 2);
                P[w][0] = lo2.x; P[w][1] = lo2.y; P[w][2] = hi2.x; P[w][3] = hi2.y;
            } else {
#pragma unroll
                for (int c = 0; c < WC; ++c) P[w][c] = row[c];
            }
            if constexpr (SIG) {
                const double* srow = &R.s[slot][wbase + TL::HXU * w];
#pragma unroll
                for (int c = 0; c < WC; ++c) Ps[w][c] = srow[c];
            }
        }
    };

    double dmax = 0.0;
    // exponent fields of the produced values: max (== 0x7ff: non-finite) and
    // min (< 54: |value| < 2^-969 or zero; zeros make the flag conservative,
    // which only costs the fused edge terms)
    unsigned emax = 0, emin = 0x7ff00000u;

    // Pair sharing.  A term's difference between two nodes of this thread is
    // the negative of the partner's (IEEE subtraction and the products by
    // 0.5 / fl(1/3) / sbar are sign-symmetric; sbar's sum commutes), so each
    // such pair is evaluated once: PV for the pairs (plane q-1 node, plane q
    // node) shared by the dr = +1 terms of the finishing nodes and the dr = -1
    // terms of the starting ones, IP for the pairs inside plane q (dr = 0
    // terms).  Values are the term t, or the difference d where the edge term
    // is fused (fm).  Only the sign of an exact zero can differ from the
    // reference's own evaluation.
    using PairT = double[RT][XP][3][3];
    auto inside = [](int a, int b) { return a >= 0 && a < RT && b >= 0 && b < XP; };
    // term value from a difference (and sbar) for squared offset l2; keep_d:
    // an edge term the consumer fuses (fma(d, 0.5, acc)) stays the difference
    auto term_of = [&](double d, double sbar, int l2, bool keep_d) {
        double t = d;
        if (SIG) t = sbar * t;
        if (l2 == 2 && !keep_d) t = t * 0.5;
        else if (l2 == 3) t = t * kInv3;
        return t;
    };
    // the thread's RT x XP nodes' terms of one stencil plane (offset dr),
    // interleaved term by term so the independent accumulation chains
    // overlap; the first term starts the chain (0 + t differs from t only in
    // the sign of zero).  mode 1: dr = +1 of the finishing nodes (PV), mode 2:
    // dr = -1 of the starting nodes (-PV), mode 3: dr = 0 (IP), 0: no pairs.
    auto plane_terms = [&](NodeD<DIM>& acc, NodeD<DIM>& smax, const Win<DIM>& P, const SWin<DIM, SIG>& Ps,
                           const NodeD<DIM>& uc, const NodeD<DIM>& sc, int dr, bool fm, int mode,
                           const PairT& PV, const PairT& PS, const PairT& IP, const PairT& IS) {
#pragma unroll
        for (int q = (DIM == 3 ? -1 : 0); q <= (DIM == 3 ? 1 : 0); ++q)
#pragma unroll
            for (int p = -1; p <= 1; ++p) {
                if (dr == 0 && q == 0 && p == 0) continue;
                const int l2 = dr * dr + q * q + p * p;
                if (CMP && l2 != 1) continue;
                const bool first = dr == -1 && (CMP ? (q == 0 && p == 0) : (q == (DIM == 3 ? -1 : 0) && p == -1));
                const bool fuse = !SIG && fm && l2 == 2 && !first;
#pragma unroll
                for (int a = 0; a < RT; ++a)
#pragma unroll
                    for (int b = 0; b < XP; ++b) {
                        const int aq = DIM == 3 ? a + q : a, bp = b + p;  // partner inside the thread?
                        // (across the planes only the straight pairs: the others would
                        // stay live through the whole step)
                        const bool pair = mode != 0 && inside(aq, bp) && (mode == 3 || (q == 0 && p == 0));
                        double v, sbar = 1.0;  // v: the term, or the difference when fused
                        if (pair && mode == 1) {
                            v = PV[a][b][q + 1][p + 1];
                            if (SIG) sbar = PS[a][b][q + 1][p + 1];
                        } else if (pair && mode == 2) {
                            v = -PV[aq][bp][1 - q][p < 0 ? 2 : (p > 0 ? 0 : 1)];
                            if (SIG) sbar = PS[aq][bp][1 - q][p < 0 ? 2 : (p > 0 ? 0 : 1)];
                        } else if (pair && mode == 3) {
                            const bool canon = q > 0 || (q == 0 && p > 0);
                            v = canon ? IP[a][b][q + 1][p + 1] : -IP[aq][bp][1 - q][1 - p];
                            if (SIG) sbar = canon ? IS[a][b][q + 1][p + 1] : IS[aq][bp][1 - q][1 - p];
                        } else {
                            const int w = DIM == 3 ? a + q + 1 : 0, c = b + p + 1;
                            if (SIG) sbar = 0.5 * (Ps[w][c] + sc[a][b]);
                            v = term_of(P[w][c] - uc[a][b], sbar, l2, fuse);
                        }
                        if (fuse) {
                            // edge: (d * 0.5) is exact for these inputs, so the fused
                            // multiply-add rounds once exactly like acc + (d * 0.5)
                            acc[a][b] = fma(v, 0.5, acc[a][b]);
                        } else {
                            acc[a][b] = first ? v : acc[a][b] + v;
                        }
                    }
            }
    };
    // PV / PS from the windows A (plane q-1) and B (plane q)
    auto pairs_between = [&](const Win<DIM>& A, const Win<DIM>& B, const SWin<DIM, SIG>& As,
                             const SWin<DIM, SIG>& Bs, bool fm, PairT& PV, PairT& PS) {
#pragma unroll
        for (int a = 0; a < RT; ++a)
#pragma unroll
            for (int b = 0; b < XP; ++b)
#pragma unroll
                for (int q = (DIM == 3 ? -1 : 0); q <= (DIM == 3 ? 1 : 0); ++q)
#pragma unroll
                    for (int p = -1; p <= 1; ++p) {
                        const int aq = DIM == 3 ? a + q : a, bp = b + p;
                        if (!inside(aq, bp) || q != 0 || p != 0) continue;
                        const int wa = DIM == 3 ? a + 1 : 0, wb = DIM == 3 ? aq + 1 : 0;
                        const double d = B[wb][bp + 1] - A[wa][b + 1];
                        double sb = 1.0;
                        if (SIG) sb = 0.5 * (Bs[wb][bp + 1] + As[wa][b + 1]);
                        const int l2 = 1 + q * q + p * p;
                        PV[a][b][q + 1][p + 1] = term_of(d, sb, l2, !SIG && fm);  // (pairs never start a chain)
                        if (SIG) PS[a][b][q + 1][p + 1] = sb;
                    }
    };
    // IP / IS inside plane B (canonical direction only)
    auto pairs_within = [&](const Win<DIM>& B, const SWin<DIM, SIG>& Bs, bool fm, PairT& IP, PairT& IS) {
#pragma unroll
        for (int a = 0; a < RT; ++a)
#pragma unroll
            for (int b = 0; b < XP; ++b)
#pragma unroll
                for (int q = 0; q <= (DIM == 3 ? 1 : 0); ++q)
#pragma unroll
                    for (int p = -1; p <= 1; ++p) {
                        if (!(q > 0 || (q == 0 && p > 0))) continue;
                        if (CMP && q * q + p * p != 1) continue;
                        const int aq = DIM == 3 ? a + q : a, bp = b + p;
                        if (!inside(aq, bp)) continue;
                        const int wc = DIM == 3 ? a + 1 : 0, wn = DIM == 3 ? aq + 1 : 0;
                        const double d = B[wn][bp + 1] - B[wc][b + 1];
                        double sb = 1.0;
                        if (SIG) sb = 0.5 * (Bs[wn][bp + 1] + Bs[wc][b + 1]);
                        const int l2 = q * q + p * p;
                        IP[a][b][q + 1][p + 1] = term_of(d, sb, l2, !SIG && fm);
                        if (SIG) IS[a][b][q + 1][p + 1] = sb;
                    }
    };

    // finish one node: op, diag / residual, Euler step, store
    auto finish = [&](int m, int a, int b, double acc, double smax, double uc, double gc, double tc) {
        const ptrdiff_t pos = opos + (DIM == 3 ? a * (ptrdiff_t)L.Px : 0) + b;
        // inv_s2 = 1 / (2^v h)^2 is a power of two (h = 2^-n), so op = (acc
        // pref) inv_s2 is an exact scaling and op - g == fma(acc pref, inv_s2,
        // -g) bit for bit (one multiply saved where op is not needed itself)
        const double ap = acc * rc.pref;
        const double op = ap * rc.inv_s2;
        double value;
        if constexpr (RESID) {
            value = HAS_A ? gc - (op + rc.a * uc) : fma(-ap, rc.inv_s2, gc);
            const double ar = fabs(value);
            dmax = dmax < ar ? ar : dmax;
            if (DUO) duo[pos] = tc + uc;
        } else {
            const double omg = fma(ap, rc.inv_s2, -gc);
            const double diag = HAS_A ? fabs((op + rc.a * uc) - gc) : fabs(omg);
            if constexpr (SIG) {
                // per-node step precomputed from sigma (k_dtau_ext: the same
                // expression on max sbar, which depends on sigma only)
                const double dtau = tc;
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
            dmax = dmax < diag ? diag : dmax;
            const unsigned e = (unsigned)__double2hiint(value) & 0x7ff00000u;
            emax = max(emax, e);
            emin = min(emin, e);
            if (DUO) duo[pos] = value - uc;
        }
        uo[pos] = value;
        // x mirror ghost (same row)
        const int i = xi + b;
        if (i == 1) uo[pos - 2] = value;
        if (i == N - 2) uo[pos + 2] = value;  // (both when N == 3)
        return value;
    };

    // Streaming march: the reference sums a node's terms plane by plane
    // (dr = -1, 0, +1), so when plane q arrives the nodes of plane q get
    // their dr = -1 and dr = 0 terms and the nodes of plane q-1 their dr = +1
    // terms.  Only two window planes are live.  The ring position of plane
    // q (slot, phase) is carried from step to step.
    Win<DIM> X, Y;  // planes q-1 / q, alternating roles
    SWin<DIM, SIG> Xs, Ys;
    NodeD<DIM> acc, smax;  // partial chains of the nodes of the newest plane

    if (m0 < mend) {
        if (tid == 0)
            for (int q = m0 - 1; q <= mend && q <= m0 + LEAD; ++q) issue(q);
        mbar_wait_u32(a_full, 0);  // plane m0 - 1: slot 0, phase 0
        read_plane(0, X, Xs);
        release(0);
        opos += (ptrdiff_t)m0 * ostep;  // plane m0 - 1
        unsigned sq = 1, ph = 0;         // ring slot / phase of plane q = m0
        int pcount = warp;               // steps until this warp issues (rotating producer)

        // plane q arrives in B (A holds plane q - 1, in ring slot sp)
        auto step = [&](int q, Win<DIM>& A, Win<DIM>& B, SWin<DIM, SIG>& As, SWin<DIM, SIG>& Bs,
                        bool fm) {
            // rotating producer: warp (q - m0) % NWARPS issues plane q + LEAD (the
            // prologue issued up to m0 + LEAD); its slot held plane q + LEAD - NST,
            // released in step q + LEAD - NST + 1
            if (pcount == 0) {
                if (lane == 0 && q > m0 && q + LEAD <= mend) issue(q + LEAD);
                pcount = TL::NWARPS;
            }
            --pcount;
            const unsigned sp = sq == 0 ? NST - 1 : sq - 1;
            mbar_wait_u32(a_full + 8 * sq, ph);
            read_plane(sq, B, Bs);
            PairT PV, PS, IP, IS;
            pairs_between(A, B, As, Bs, fm, PV, PS);
            if (q > m0) {  // nodes of plane q - 1: dr = +1 terms, then the update
                const int m = q - 1;
                opos += ostep;
                NodeD<DIM> uc, sc, gc, tc;
#pragma unroll
                for (int a = 0; a < RT; ++a)
#pragma unroll
                    for (int b = 0; b < XP; ++b) {
                        const int gi = gbase + TL::HXG * a + b;  // node in the g box
                        gc[a][b] = R.g[sp][gi];
                        tc[a][b] = ((DUO && RESID) || (SIG && !RESID)) ? R.t[sp][gi] : 0.0;
                        uc[a][b] = A[DIM == 3 ? a + 1 : 0][b + 1];
                        sc[a][b] = 1.0;
                        if constexpr (SIG) sc[a][b] = As[DIM == 3 ? a + 1 : 0][b + 1];
                    }
                plane_terms(acc, smax, B, Bs, uc, sc, 1, fm, 1, PV, PS, IP, IS);
                const int mg = DIM == 3 ? m + L.z0 : m;  // global plane
                const unsigned mm = (mg == 1 || mg == N - 2) ? ALL : mirm;
                NodeD<DIM> val;
                if (okm == ALL) {  // (block-uniform except at the range edges)
#pragma unroll
                    for (int a = 0; a < RT; ++a)
#pragma unroll
                        for (int b = 0; b < XP; ++b)
                            val[a][b] = finish(m, a, b, acc[a][b], smax[a][b], uc[a][b], gc[a][b], tc[a][b]);
                } else {
#pragma unroll
                    for (int a = 0; a < RT; ++a)
#pragma unroll
                        for (int b = 0; b < XP; ++b)
                            val[a][b] = (okm >> (a * XP + b)) & 1u
                                            ? finish(m, a, b, acc[a][b], smax[a][b], uc[a][b], gc[a][b], tc[a][b])
                                            : 0.0;
                }
                if (mm & okm) {  // rare: nodes next to a face write their mirror ghosts
#pragma unroll
                    for (int a = 0; a < RT; ++a)
#pragma unroll
                        for (int b = 0; b < XP; ++b)
                            if ((mm & okm) >> (a * XP + b) & 1u)
                                store_mirrors<DIM>(uo, L, xi + b, DIM == 3 ? yb + a : m, DIM == 3 ? m : 0,
                                                   val[a][b]);
                }
                release(sp);
            }
            if (q < mend) {  // nodes of plane q: dr = -1 and dr = 0 terms
                NodeD<DIM> uc, sc;
#pragma unroll
                for (int a = 0; a < RT; ++a)
#pragma unroll
                    for (int b = 0; b < XP; ++b) {
                        uc[a][b] = B[DIM == 3 ? a + 1 : 0][b + 1];
                        sc[a][b] = 1.0;
                        if constexpr (SIG) sc[a][b] = Bs[DIM == 3 ? a + 1 : 0][b + 1];
                    }
                plane_terms(acc, smax, A, As, uc, sc, -1, fm, 2, PV, PS, IP, IS);
                pairs_within(B, Bs, fm, IP, IS);
                plane_terms(acc, smax, B, Bs, uc, sc, 0, fm, 3, PV, PS, IP, IS);
            }
            if (++sq == NST) {
                sq = 0;
                ph ^= 1;
            }
        };
        // roles alternate each plane: period 2.  `fm` is a literal at both
        // call sites (two specialised marches)
        auto march = [&](bool fm) {
#pragma unroll 1
            for (int q = m0; q <= mend; q += 2) {
                step(q, X, Y, Xs, Ys, fm);
                if (q + 1 > mend) break;
                step(q + 1, Y, X, Ys, Xs, fm);
            }
        };
        // edge terms fused when no input value is tiny (flag[1], set by the
        // producers of this cycle's level arrays): then every difference d of
        // two inputs is 0 or >= 2^-1021 in magnitude and d * 0.5 is exact
        // (flag[2], flag[3]: the neighbour ranks' flag[1], received with the halos)
        const volatile int* fv = flag;
        if (!SIG && (fv[1] | fv[2] | fv[3]) == 0) march(true);
        else march(false);
    }
    block_max_commit(dmax, diag_slot);
    if (!RESID) {
        warp_bad_commit(emax == 0x7ff00000u, flag, pass_slot);
        warp_or_commit(emin < 0x03600000u, flag + 1);
    }
}

template <int DIM, bool SIG, bool HAS_A, int MODE, bool DUO, bool CMP>
void launch_k(dim3 grid, dim3 block, cudaStream_t s, const TmaSet& tm, double* uo, double* duo,
              const ExtLay& L, int3 lo, int3 hi, int zb, const RelaxConst& rc,
              unsigned long long* slot, int* flag, int pass_slot) {
    const int bytes = (int)sizeof(TRing<DIM, SIG, MODE>);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_relax_tma<DIM, SIG, HAS_A, MODE, DUO, CMP>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        configured = true;
    }
    launch_pdl(k_relax_tma<DIM, SIG, HAS_A, MODE, DUO, CMP>, grid, block, bytes, s, tm.u, tm.g, tm.s, tm.t, uo, duo, L,
               lo, hi, zb, rc, slot, flag, pass_slot);
}

template <int DIM, bool SIG, bool HAS_A, int MODE, bool DUO>
void launch_t(dim3 grid, dim3 block, cudaStream_t s, const TmaSet& tm, double* uo, double* duo,
              const ExtLay& L, int3 lo, int3 hi, int zb, const RelaxConst& rc,
              unsigned long long* slot, int* flag, int pass_slot) {
    if (rc.compact)
        launch_k<DIM, SIG, HAS_A, MODE, DUO, true>(grid, block, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag,
                                                   pass_slot);
    else
        launch_k<DIM, SIG, HAS_A, MODE, DUO, false>(grid, block, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag,
                                                    pass_slot);
}

template <int DIM, int MODE, bool DUO>
void launch_duo(dim3 grid, dim3 block, bool sig, cudaStream_t s, const TmaSet& tm, double* uo,
                double* duo, const ExtLay& L, int3 lo, int3 hi, int zb, const RelaxConst& rc,
                unsigned long long* slot, int* flag, int pass_slot) {
    if (sig) {
        if (rc.has_a) launch_t<DIM, true, true, MODE, DUO>(grid, block, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
        else launch_t<DIM, true, false, MODE, DUO>(grid, block, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
    } else {
        if (rc.has_a) launch_t<DIM, false, true, MODE, DUO>(grid, block, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
        else launch_t<DIM, false, false, MODE, DUO>(grid, block, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
    }
}

template <int MODE>
void launch_mode(int dim, bool sig, const TmaSet& tm, double* uo, double* duo, const ExtLay& L,
                 const NodeRange& rg, const RelaxConst& rc, unsigned long long* slot, int* flag,
                 int pass_slot, cudaStream_t s) {
    const int3 lo = make_int3(rg.lo[0], rg.lo[1], rg.lo[2]);
    const int3 hi = make_int3(rg.hi[0], rg.hi[1], rg.hi[2]);
    const int nx = rg.hi[0] - rg.lo[0] + 1, ny = rg.hi[1] - rg.lo[1] + 1, nz = rg.hi[2] - rg.lo[2] + 1;
    if (nx <= 0 || ny <= 0 || (dim == 3 && nz <= 0)) return;  // nothing off the Dirichlet faces
    // 3D tiles start at the even column at or below lo.x (16-byte TMA boxes
    // with the halo exactly); 2D tiles start at lo.x
    const int nxt = dim == 3 ? rg.hi[0] - (rg.lo[0] & ~1) + 1 : nx;
    const int tilesx = dim == 3 ? (nxt + Tile<3>::NX - 1) / Tile<3>::NX : (nxt + Tile<2>::NX - 1) / Tile<2>::NX;
    const int cols = dim == 3 ? tilesx * ((ny + Tile<3>::ROWS - 1) / Tile<3>::ROWS) : tilesx;
    const int zb = relax_tiled_zb(dim, cols, dim == 3 ? nz : ny, dim == 3 ? (sig ? 1 : 2) : 4);
    dim3 grid, block;
    if (dim == 3) {
        using TL = Tile<3>;
        grid = dim3(tilesx, (ny + TL::ROWS - 1) / TL::ROWS, (nz + zb - 1) / zb);
        block = dim3(TL::X, TL::TY);
    } else {
        using TL = Tile<2>;
        grid = dim3(tilesx, 1, (ny + zb - 1) / zb);
        block = dim3(TL::X, 1);
    }
    if (dim == 3) {
        if (duo) launch_duo<3, MODE, true>(grid, block, sig, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
        else launch_duo<3, MODE, false>(grid, block, sig, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
    } else {
        if (duo) launch_duo<2, MODE, true>(grid, block, sig, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
        else launch_duo<2, MODE, false>(grid, block, sig, s, tm, uo, duo, L, lo, hi, zb, rc, slot, flag, pass_slot);
    }
}


// ---------------------------------------------------------------------------
// Small level arrays: all c passes of one level visit in one CTA (the levels
// whose arrays hold a few thousand nodes are launch-latency bound as one
// kernel per pass).  Same arithmetic as the reference's relax branch
// (kernels.cpp:94-137) on the ghost-extended array (mirror ghosts in memory),
// with the edge terms unfused (identical bits whenever the fused form is
// exact).  The visit runs out of shared memory: the input array, the first
// output array (its Dirichlet faces are resident, engine face states) and
// the source are staged whole (<= 3 x 58 KB); pass p reads one staged array
// and writes the other (with its mirror ghosts), so only the first touch of
// each array waits for L2; every pass output and du also go to global memory
// as before.  Passes are separated by barriers.
// ---------------------------------------------------------------------------
template <int DIM, bool SIG, bool HAS_A>
__global__ void __launch_bounds__(kSmallThreads) k_relax_small(SmallPasses sp, ExtLay L, int3 lo, int3 hi,
                                                               RelaxConst rc, int* flag, int next) {
    pdl_begin();
    extern __shared__ __align__(16) double sm[];
    double* X = sm;             // pass input of even passes (the visit's input array)
    double* Y = sm + next;      // first output array
    double* G = sm + 2 * next;  // source
    for (int e = threadIdx.x; e < next; e += blockDim.x) {
        X[e] = sp.in[0][e];
        Y[e] = sp.out[0][e];
        G[e] = sp.g[e];
    }
    __syncthreads();
    const int nx = hi.x - lo.x + 1, ny = hi.y - lo.y + 1, nz = DIM == 3 ? hi.z - lo.z + 1 : 1;
    const int total = nx * ny * nz;
    const ptrdiff_t sy = L.Px, sz = DIM == 3 ? (ptrdiff_t)L.plane : 0;
    for (int p = 0; p < sp.count; ++p) {
        const double* __restrict__ u = (p & 1) ? Y : X;
        double* __restrict__ so = (p & 1) ? X : Y;
        double* __restrict__ o = sp.out[p];
        double* __restrict__ du = sp.du[p];
        double dmax = 0.0;
        int bad = 0, tiny = 0;
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
            const int i = lo.x + e % nx, j = lo.y + (e / nx) % ny, k = DIM == 3 ? lo.z + e / (nx * ny) : 0;
            const ptrdiff_t pos = eix<DIM>(L, i, j, k);
            const double uc = u[pos];
            const double sc = SIG ? sp.sig[pos] : 1.0;
            double acc = 0.0;
#pragma unroll
            for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
                for (int q = -1; q <= 1; ++q)
#pragma unroll
                    for (int pp = -1; pp <= 1; ++pp) {
                        if (r == 0 && q == 0 && pp == 0) continue;
                        const int l2 = r * r + q * q + pp * pp;
                        if (stencil_skip(rc.compact, l2)) continue;
                        const ptrdiff_t d = r * sz + q * sy + pp;
                        const double sbar = SIG ? 0.5 * (sp.sig[pos + d] + sc) : 1.0;
                        acc = acc + stencil_t<SIG>(sbar, u[pos + d], uc, l2);
                    }
            const double op = (acc * rc.pref) * rc.inv_s2;
            const double gc = G[pos];
            const double diag = HAS_A ? fabs((op + rc.a * uc) - gc) : fabs(op - gc);
            double value;
            if (SIG) {
                const double dtau = sp.dt[pos];
                if (!(dtau > 0.0)) value = __longlong_as_double(0x7ff8000000000000LL);
                else {
                    const double num = uc + dtau * (op - gc);
                    value = HAS_A ? num / (1.0 - dtau * rc.a) : num;
                }
            } else {
                const double num = uc + rc.dtau1 * (op - gc);
                value = HAS_A ? num / rc.denom1 : num;
            }
            dmax = dmax < diag ? diag : dmax;
            const unsigned ex = (unsigned)__double2hiint(value) & 0x7ff00000u;
            bad |= ex == 0x7ff00000u;
            tiny |= ex < 0x03600000u;
            store_ext<DIM>(so, L, i, j, k, value);
            store_ext<DIM>(o, L, i, j, k, value);
            if (du) du[pos] = value - uc;
        }
        block_max_commit(dmax, sp.slot[p]);
        block_bad_commit(bad, flag, sp.pass_slot[p]);
        block_or_commit(tiny, flag + 1);
        __syncthreads();  // pass p's outputs (and the reduction scratch) before pass p + 1
    }
}
}  // namespace

bool pdl_enabled() {
    static const bool on = std::getenv("SGML_NO_PDL") == nullptr;
    return on;
}

// planes per CTA: long marches amortise the 2-plane prologue, short ones
// give small levels enough CTAs (2D: about two waves of 148 SMs x 4 CTAs;
// 3D: about four waves of 148 x per_sm — 257^3 passes then march 12 planes,
// ~1 ms per 513^3 solve faster than 24; the sigma kernel, one CTA per SM,
// keeps 24 there)
int relax_tiled_zb(int dim, int cols, int nz, int per_sm) {
    const int target = (dim == 3 ? 4 : 2) * 148 * per_sm;
    // 3D: 24 planes per CTA (513^3 level-0 pass measured over 8..64: 16-24
    // best, 0.69 ms; 64: 0.72-0.75 ms — shorter marches spread the ring
    // fills of the two co-resident CTAs better and shrink the tail wave)
    int zb = dim == 3 ? 24 : 128;
    while (zb > 4 && (long long)cols * ((nz + zb - 1) / zb) < target) zb = std::max(4, zb / 2);
    return zb;
}

void tile_boxes(int dim, unsigned* box_u, unsigned* box_g) {
    if (dim == 3) {
        box_u[0] = Tile<3>::HXU; box_u[1] = Tile<3>::HY;   box_u[2] = 1;
        box_g[0] = Tile<3>::HXG; box_g[1] = Tile<3>::ROWS; box_g[2] = 1;
    } else {
        box_u[0] = Tile<2>::HXU; box_u[1] = 1; box_u[2] = 1;
        box_g[0] = Tile<2>::HXG; box_g[1] = 1; box_g[2] = 1;
    }
}

void launch_relax_tma(int dim, bool sig, const TmaSet& tm, double* uo, double* duo,
                      const ExtLay& L, const NodeRange& rg, const RelaxConst& rc,
                      unsigned long long* slot, int* flag, int pass_slot, cudaStream_t s) {
    launch_mode<MODE_RELAX>(dim, sig, tm, uo, duo, L, rg, rc, slot, flag, pass_slot, s);
}

void launch_relax_small(int dim, bool sig, const SmallPasses& sp, const ExtLay& L, const NodeRange& rg,
                        const RelaxConst& rc, int* flag, cudaStream_t s) {
    const int3 lo = make_int3(rg.lo[0], rg.lo[1], rg.lo[2]);
    const int3 hi = make_int3(rg.hi[0], rg.hi[1], rg.hi[2]);
    const int next = (int)ext_size(dim, L);  // doubles per staged array
    const size_t bytes = 3 * (size_t)next * sizeof(double);
#define SGML_SMALL(DD, SS, AA)                                                                                   \
    do {                                                                                                        \
        static bool configured = false;                                                                         \
        if (!configured) {                                                                                      \
            cudaFuncSetAttribute(k_relax_small<DD, SS, AA>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallSmem); \
            configured = true;                                                                                  \
        }                                                                                                       \
        launch_pdl(k_relax_small<DD, SS, AA>, dim3(1), dim3(kSmallThreads), bytes, s, sp, L, lo, hi, rc, flag, next); \
    } while (0)
    if (dim == 2) {
        if (sig) { if (rc.has_a) SGML_SMALL(2, true, true); else SGML_SMALL(2, true, false); }
        else { if (rc.has_a) SGML_SMALL(2, false, true); else SGML_SMALL(2, false, false); }
    } else {
        if (sig) { if (rc.has_a) SGML_SMALL(3, true, true); else SGML_SMALL(3, true, false); }
        else { if (rc.has_a) SGML_SMALL(3, false, true); else SGML_SMALL(3, false, false); }
    }
#undef SGML_SMALL
}

void launch_residual_tma(int dim, bool sig, const TmaSet& tm, double* r, double* utot,
                         const ExtLay& L, const NodeRange& rg, const RelaxConst& rc,
                         unsigned long long* rmax_slot, int* flag, bool guarded, cudaStream_t s) {
    launch_mode<MODE_RESID>(dim, sig, tm, r, utot, L, rg, rc, rmax_slot, flag, guarded ? -1 : 0, s);
}

}  // namespace sgmlb
