// level_ops.cuh — bodies of the compact engine's level-array operations that
// run both as their own kernels (materialize.cu) and inside the small-level
// interpreter (interp.cu).  Per-node arithmetic and term order exactly as
// documented in materialize.cu.
#pragma once

#include "device.cuh"
#include "internal.hpp"

namespace sgmlb {

// materialisation blocks: MBX x MBY threads, MV consecutive x nodes per thread
constexpr int MV = 4;
constexpr int MBX = 32, MBY = 4;

// read-only load: non-coherent path when allowed
template <bool NCLD>
__device__ __forceinline__ double ldx(const double* p) {
    if constexpr (NCLD) return __ldg(p);
    else return *p;
}

// The materialisation of one (virtual) block: the body of k_materialize4,
// also run by the small-level interpreter (interp.cu) with virtual block
// indices.  sch: the first kMaxChain chain entries in shared memory.  NCLD:
// read-only data may go through the non-coherent path (false when an earlier
// operation of the same kernel wrote it).
template <int DIM, int NC, bool DIAG, bool NCLD>
__device__ __forceinline__ void mat4_body(double* __restrict__ out, ExtLay Lw, int w,
                                          const double* __restrict__ base, ExtLay L0, int wb, int base_zero,
                                          const double* __restrict__ ufine, ExtLay Lf, int frel,
                                          const ChainEntry* __restrict__ chain, int nchain, const ChainEntry* sch,
                                          BcDev bc, int homogeneous, int* flag, int xtail, int k0, int bx,
                                          int by, int bz, int tx, int ty) {

    // NC copies along y at spacing D = (Nw - 1) / NC: rows s0 + c D
    const int Nw = Lw.N, D = (Nw - 1) / NC;
    const int X4 = (bx * MBX + tx) * MV;
    // spread row index S (warp-uniform); 3D: local plane K (block-uniform),
    // global plane Kg (z-slab arrays start at global plane Lw.z0)
    const int S = by * MBY + ty;
    const int K = DIM == 3 ? k0 + bz : 0;
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
                uf[cp][0] = ldx<NCLD>(pf);
                uf[cp][1] = ldx<NCLD>(pf + 1);
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
                    val[cp][k] = (!base_zero && k < nv && cp < ncopy) ? ldx<NCLD>(bp + cp * bcs + (k << bsh)) : 0.0;
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
                            cv[q][cp][0] = ldx<NCLD>(rw);
                            cv[q][cp][1] = ldx<NCLD>(rw + 1);
                            cv[q][cp][2] = st ? ldx<NCLD>(rw + 2) : 0.0;
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
                        value = ldx<NCLD>(ufine + eix<DIM>(Lf, I >> frel, Jn >> frel, (Kn >> frel) - Lf.z0));
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
// One node of a materialisation (k_materialize4's arithmetic for a single
// node): the Dirichlet value, the level-(w + frel) value, or
// ((base + I_l0(du0)) + I_l1(du1)) + ... with I_l = sum over r, q, p of
// ((wz * wy) * wx) * du (zero-weight rows in y / z skipped, the p = 1 corner
// always added).  Every corner of every entry (at most MC) is loaded before
// any arithmetic.  Node (I, J, K), K local; stores with the mirror ghosts and
// folds the non-finite / tiny checks into bad / tiny.
template <int DIM>
struct NodeChain {
    static constexpr int max = DIM == 3 ? 3 : 6;  // (all corners in registers)
};

template <int DIM, int MC, bool NCLD>
__device__ __forceinline__ void mat_node(double* __restrict__ out, const ExtLay& Lw, int w,
                                         const double* __restrict__ base, const ExtLay& L0, int wb, int base_zero,
                                         const double* __restrict__ ufine, const ExtLay& Lf, int frel,
                                         const ChainEntry* ch, int nchain, const BcDev& bc, int homogeneous, int I,
                                         int J, int K, int& bad, int& tiny) {
    constexpr int NCV = DIM == 3 ? 8 : 4;  // corner values per entry: [r][q][p]
    const int Nw = Lw.N, Kg = DIM == 3 ? K + Lw.z0 : 0;
    const int bsh = w - wb, fmask = (1 << frel) - 1;
    double value;
    if (on_dirichlet<DIM>(bc, Nw, I, J, Kg)) {
        value = homogeneous ? 0.0 : dirichlet_value<DIM>(bc, Nw, I, J, Kg);
    } else if (ufine && ((I | J | Kg) & fmask) == 0) {
        value = ldx<NCLD>(ufine + eix<DIM>(Lf, I >> frel, J >> frel, (Kg >> frel) - Lf.z0));
    } else {
        const int x = I << w, y = J << w, z = Kg << w;
        double val = base_zero ? 0.0 : ldx<NCLD>(base + eix<DIM>(L0, I << bsh, J << bsh, (z >> wb) - L0.z0));
        double cv[MC][NCV];
#pragma unroll
        for (int c = 0; c < MC; ++c) {
            const bool in = c < nchain;
            const ChainEntry& ce = ch[in ? c : 0];
            const int l = ce.level, msk = (1 << l) - 1;
            const int nq = (y & msk) ? 2 : 1, nr = (DIM == 3 && (z & msk)) ? 2 : 1;
            const int sq = ce.L.Px, sr = DIM == 3 ? (int)ce.L.plane : 0;
            const double* o = ce.du + eix<DIM>(ce.L, x >> l, y >> l, DIM == 3 ? (z >> l) - ce.L.z0 : 0);
#pragma unroll
            for (int r = 0; r < (DIM == 3 ? 2 : 1); ++r)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const bool live = in && r < nr && q < nq;
                    cv[c][(r * 2 + q) * 2] = live ? ldx<NCLD>(o + r * sr + q * sq) : 0.0;
                    cv[c][(r * 2 + q) * 2 + 1] = live ? ldx<NCLD>(o + r * sr + q * sq + 1) : 0.0;
                }
        }
#pragma unroll
        for (int c = 0; c < MC; ++c) {
            if (c >= nchain) continue;
            const ChainEntry& ce = ch[c];
            const int l = ce.level, msk = (1 << l) - 1;
            const double inv = __longlong_as_double((long long)(1023 - l) << 52);  // 2^-l, exact
            const int iy = y & msk, iz = z & msk;
            const double fy = (double)iy * inv, fz = (double)iz * inv;
            const double wy[2] = {1.0 - fy, fy};
            const double wz[2] = {1.0 - fz, fz};
            const int nq = iy ? 2 : 1, nr = (DIM == 3 && iz) ? 2 : 1;
            const double fx = (double)(x & msk) * inv, wx0 = 1.0 - fx;
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < (DIM == 3 ? 2 : 1); ++r) {
                if (r >= nr) continue;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (q >= nq) continue;
                    const double wzy = DIM == 3 ? wz[r] * wy[q] : wy[q];
                    const double w0 = wzy * wx0, w1 = wzy * fx;
                    const double t0 = w0 * cv[c][(r * 2 + q) * 2];
                    acc = (r == 0 && q == 0) ? t0 : acc + t0;
                    acc = acc + w1 * cv[c][(r * 2 + q) * 2 + 1];
                }
            }
            val = val + acc;
        }
        value = val;
    }
    bad |= (__double_as_longlong(value) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
    {  // nonzero |value| < 2^-969 (see launch_relax_tma)
        const unsigned key = ((unsigned)__double2hiint(value) & 0x7fffffffu) | (__double2loint(value) != 0 ? 1u : 0u);
        tiny |= key - 1u < 0x035fffffu;
    }
    store_ext<DIM>(out, Lw, I, J, K, value);
}

}  // namespace sgmlb
