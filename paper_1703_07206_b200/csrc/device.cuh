// device.cuh — pointwise fp64 math of the SGML path, shared by all kernels.
//
// Operation order follows the reference exactly:
//   acc = acc + ((sbar * (u_nb - u_c)) * inv_l2)  over offsets r, q, p
//   op  = (acc * pref) * inv_s2
// The whole library is compiled with --fmad=false, so no multiply-add is
// ever contracted.  Bit-safe shortcuts used here (each exact in IEEE):
//   x * 1.0 == x (sigma == 1, inv_l2 == 1), x / 1.0 == x (a == 0),
//   and zero-weight interpolation corners are skipped (sign of zero only).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sgmlb {

// Boundary description in kernel-parameter form (grid.hpp:125-157).
struct BcDev {
    int neu[6];      // 1 = Neumann, 0 = Dirichlet
    double val[6];   // Dirichlet values
};

// 1 / 3 rounded once, as stencil.cpp:21 computes 1.0 / l2 for l2 = 3.
constexpr double kInv3 = 1.0 / 3.0;

__device__ __forceinline__ size_t lin3(int N, int i, int j, int k) {
    return (size_t)i + (size_t)N * ((size_t)j + (size_t)N * (size_t)k);
}

// grid.cpp:44-51 (node already known to lie on some face or not)
template <int DIM>
__device__ __forceinline__ bool on_dirichlet(const BcDev& bc, int N, int i, int j, int k) {
    if ((i == 0 && !bc.neu[0]) || (i == N - 1 && !bc.neu[1])) return true;
    if ((j == 0 && !bc.neu[2]) || (j == N - 1 && !bc.neu[3])) return true;
    if (DIM == 3 && ((k == 0 && !bc.neu[4]) || (k == N - 1 && !bc.neu[5]))) return true;
    return false;
}

// grid.cpp:53-62: lowest Dirichlet face id wins
template <int DIM>
__device__ __forceinline__ double dirichlet_value(const BcDev& bc, int N, int i, int j, int k) {
    if (i == 0 && !bc.neu[0]) return bc.val[0];
    if (i == N - 1 && !bc.neu[1]) return bc.val[1];
    if (j == 0 && !bc.neu[2]) return bc.val[2];
    if (j == N - 1 && !bc.neu[3]) return bc.val[3];
    if (DIM == 3) {
        if (k == 0 && !bc.neu[4]) return bc.val[4];
        if (k == N - 1 && !bc.neu[5]) return bc.val[5];
    }
    return 0.0;
}

// stencil.cpp:52-85, unrolled by axis: x resolves first, then y, then z.
// Odd reflection evaluates 2*u(face) - u(mirror).
__device__ __forceinline__ double ghost_z(const double* __restrict__ u, int N, const BcDev& bc,
                                          int i, int j, int k) {
    if (k < 0) {
        const double m = u[lin3(N, i, j, -k)];
        return bc.neu[4] ? m : 2.0 * u[lin3(N, i, j, 0)] - m;
    }
    if (k > N - 1) {
        const double m = u[lin3(N, i, j, 2 * (N - 1) - k)];
        return bc.neu[5] ? m : 2.0 * u[lin3(N, i, j, N - 1)] - m;
    }
    return u[lin3(N, i, j, k)];
}

__device__ __forceinline__ double ghost_y(const double* __restrict__ u, int N, const BcDev& bc,
                                          int i, int j, int k) {
    if (j < 0) {
        const double m = ghost_z(u, N, bc, i, -j, k);
        return bc.neu[2] ? m : 2.0 * ghost_z(u, N, bc, i, 0, k) - m;
    }
    if (j > N - 1) {
        const double m = ghost_z(u, N, bc, i, 2 * (N - 1) - j, k);
        return bc.neu[3] ? m : 2.0 * ghost_z(u, N, bc, i, N - 1, k) - m;
    }
    return ghost_z(u, N, bc, i, j, k);
}

__device__ __forceinline__ double ghost(const double* __restrict__ u, int N, const BcDev& bc,
                                        int i, int j, int k) {
    if (i < 0) {
        const double m = ghost_y(u, N, bc, -i, j, k);
        return bc.neu[0] ? m : 2.0 * ghost_y(u, N, bc, 0, j, k) - m;
    }
    if (i > N - 1) {
        const double m = ghost_y(u, N, bc, 2 * (N - 1) - i, j, k);
        return bc.neu[1] ? m : 2.0 * ghost_y(u, N, bc, N - 1, j, k) - m;
    }
    return ghost_y(u, N, bc, i, j, k);
}

// grid.hpp:63-69 and stencil.cpp:87-90: sigma is always even-mirrored.
__device__ __forceinline__ int mirror_index(int i, int N) {
    return i < 0 ? -i : (i > N - 1 ? 2 * (N - 1) - i : i);
}
__device__ __forceinline__ double mirror(const double* __restrict__ u, int N, int i, int j, int k) {
    return u[lin3(N, mirror_index(i, N), mirror_index(j, N), mirror_index(k, N))];
}

// acc + ((sbar*(un-uc)) * inv_l2) with the exact shortcuts for sbar == 1 and
// inv_l2 == 1 (l2 = 1: face neighbours).
template <bool SIG>
__device__ __forceinline__ double stencil_t(double sbar, double un, double uc, int l2) {
    double t = un - uc;
    if (SIG) t = sbar * t;
    if (l2 == 2) t = t * 0.5;
    else if (l2 == 3) t = t * kInv3;
    return t;
}

template <bool SIG>
__device__ __forceinline__ double stencil_term(double acc, double sbar, double un, double uc, int l2) {
    double t = un - uc;
    if (SIG) t = sbar * t;
    if (l2 == 2) t = t * 0.5;
    else if (l2 == 3) t = t * kInv3;
    return acc + t;
}

// Per-pass constants of relax_pass (kernels.cpp:182-188) plus the host-side
// precomputed step for sigma == 1 (smax == 1 exactly, so
// dtau = (safety*kdim)/(inv_s2*1.0), identical to the per-node formula).
struct RelaxConst {
    double inv_s2;
    double pref;
    double kdim;
    double a;
    double safety;
    double dtau1;      // used when sigma == 1
    double denom1;     // 1.0 - dtau1*a (sigma == 1)
    int homogeneous;
    int has_a;
    int compact;       // stencil family: 0 radial (the reference's), 1 compact 5/7-point
};

// compact 5/7-point family: only the axis offsets
__device__ __forceinline__ bool stencil_skip(int compact, int l2) { return compact && l2 != 1; }

// kernels.cpp:94-137 at a subset node whose stencil neighbours sit at
// +-lam in the index space of `up` (lam = 2^v for full-grid fields, 1 for
// level-compact fields).  Returns the new value; diag through the reference.
template <int DIM, bool SIG>
__device__ __forceinline__ double relax_at(const double* __restrict__ up,
                                           const double* __restrict__ sig,
                                           const double* __restrict__ g, int N, int lam, int i,
                                           int j, int k, size_t pos, const RelaxConst& rc,
                                           const BcDev& bc, double& diag) {
    const double uc = up[pos];
    const double sc = SIG ? sig[pos] : 1.0;
    const bool fast = i >= lam && i <= N - 1 - lam && j >= lam && j <= N - 1 - lam &&
                      (DIM == 2 || (k >= lam && k <= N - 1 - lam));
    double acc = 0.0, smax = 0.0;
    if (fast) {
        const ptrdiff_t sy = (ptrdiff_t)N * lam, sz = (ptrdiff_t)N * N * lam;
#pragma unroll
        for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
            for (int q = -1; q <= 1; ++q)
#pragma unroll
                for (int p = -1; p <= 1; ++p) {
                    if (p == 0 && q == 0 && r == 0) continue;
                    if (stencil_skip(rc.compact, p * p + q * q + r * r)) continue;
                    const ptrdiff_t d = r * sz + q * sy + p * lam;
                    double sbar = 1.0;
                    if (SIG) {
                        sbar = 0.5 * (sig[pos + d] + sc);
                        smax = smax < sbar ? sbar : smax;
                    }
                    acc = stencil_term<SIG>(acc, sbar, up[pos + d], uc, p * p + q * q + r * r);
                }
    } else {
#pragma unroll
        for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
            for (int q = -1; q <= 1; ++q)
#pragma unroll
                for (int p = -1; p <= 1; ++p) {
                    if (p == 0 && q == 0 && r == 0) continue;
                    if (stencil_skip(rc.compact, p * p + q * q + r * r)) continue;
                    const int ni = i + p * lam, nj = j + q * lam, nk = k + r * lam;
                    double sbar = 1.0;
                    if (SIG) {
                        sbar = 0.5 * (mirror(sig, N, ni, nj, nk) + sc);
                        smax = smax < sbar ? sbar : smax;
                    }
                    acc = stencil_term<SIG>(acc, sbar, ghost(up, N, bc, ni, nj, nk), uc,
                                            p * p + q * q + r * r);
                }
    }
    const double op = (acc * rc.pref) * rc.inv_s2;
    const double gc = g[pos];
    if (rc.has_a) {
        diag = fabs((op + rc.a * uc) - gc);
    } else {
        diag = fabs(op - gc);
    }
    if (SIG) {
        const double dtau = (rc.safety * rc.kdim) / (rc.inv_s2 * smax);
        if (!(dtau > 0.0)) return __longlong_as_double(0x7ff8000000000000LL);
        const double num = uc + dtau * (op - gc);
        return rc.has_a ? num / (1.0 - dtau * rc.a) : num;
    } else {
        const double num = uc + rc.dtau1 * (op - gc);
        return rc.has_a ? num / rc.denom1 : num;
    }
}

// Interpolated increment of a level-l variation at full-grid node (x,y,z)
// (kernels.cpp:140-174).  `du` is the level-l compact array with Nl nodes
// per axis.  Weights are exact dyadics; zero-weight corners are skipped.
template <int DIM>
__device__ __forceinline__ double interp_compact(const double* __restrict__ du, int Nl, int l,
                                                 int x, int y, int z) {
    const int m = (1 << l) - 1;
    const double inv_lam = 1.0 / (double)(1 << l);
    const int x0 = x & ~m, y0 = y & ~m, z0 = z & ~m;
    const double fx = (double)(x - x0) * inv_lam;
    const double fy = (double)(y - y0) * inv_lam;
    const double wx[2] = {1.0 - fx, fx};
    const double wy[2] = {1.0 - fy, fy};
    const int X0 = x0 >> l, Y0 = y0 >> l, Z0 = z0 >> l;
    double acc = 0.0;
    if (DIM == 2) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                if (wy[q] == 0.0 || wx[p] == 0.0) continue;
                acc = acc + ((wy[q] * wx[p]) * du[(size_t)(X0 + p) + (size_t)Nl * (Y0 + q)]);
            }
    } else {
        const double fz = (double)(z - z0) * inv_lam;
        const double wz[2] = {1.0 - fz, fz};
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    if (wz[r] == 0.0 || wy[q] == 0.0 || wx[p] == 0.0) continue;
                    acc = acc + (((wz[r] * wy[q]) * wx[p]) * du[lin3(Nl, X0 + p, Y0 + q, Z0 + r)]);
                }
    }
    return acc;
}

// Non-negative double max via the ordered uint64 bit pattern.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
    if (v > 0.0) atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

// Block-wide max of a non-negative value, one atomic per block.
__device__ __forceinline__ void block_max_commit(double v, unsigned long long* slot) {
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = v < w ? w : v;
    }
    __shared__ double red[32];
    const int nthreads = blockDim.x * blockDim.y * blockDim.z;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (nthreads + 31) / 32 ? red[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(0xffffffffu, v, o);
            v = v < w ? w : v;
        }
        if (lane == 0) atomic_max_nonneg(slot, v);
    }
}

// warp-level variant: no block barrier (finished warps leave immediately)
__device__ __forceinline__ void warp_or_commit(int bad, int* flag) {
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// a failing pass: flag[0] <- 1 and flag[4] <- min(flag[4], slot) (the first
// failing pass of the cycle in the reference's order, for the partial trace)
__device__ __forceinline__ void warp_bad_commit(int bad, int* flag, int slot) {
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
        atomicOr(flag, 1);
        atomicMin(flag + 4, slot);
    }
}

__device__ __forceinline__ void block_or_commit(int bad, int* flag) {
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0) atomicOr(flag, 1);
    }
}

__device__ __forceinline__ void block_bad_commit(int bad, int* flag, int slot) {
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0) {
            atomicOr(flag, 1);
            atomicMin(flag + 4, slot);
        }
    }
}

}  // namespace sgmlb

// ---------------------------------------------------------------------------
// Ghost-extended, padded level arrays (compact engine storage)
//
// A level array with N data nodes per axis is stored with one ghost layer on
// every side (Ne = N + 2 cells per axis) and an even row pitch Px >= Ne, so
// that every row starts 16-byte aligned and TMA can stream tiles.  Data node
// (i, j, k), i in [0, N), sits at cell (i+1, j+1, k+1).  Ghost cells hold
// the even mirror of the data (u(-1) = u(1), u(N) = u(N-2), per axis); every
// kernel that writes a node at data index 1 or N-2 also writes its mirror
// cells.  The even mirror is the reference's ghost value across Neumann
// faces (stencil.cpp:52-85) and for sigma (stencil.cpp:87-90); across a
// Dirichlet face the reference's odd ghost is only ever read by nodes on
// that face, which take their Dirichlet value instead, so those cells never
// influence a result.
// ---------------------------------------------------------------------------
namespace sgmlb {

struct ExtLay {
    int N;            // data nodes per axis (global)
    int Ne;           // N + 2
    int Px;           // row pitch in doubles (even)
    int Nz;           // 3D: data planes held (N, or a z-slab's own planes)
    int z0;           // 3D: global index of local data plane 0 (0 unless a z-slab)
    int pad_;
    long long plane;  // stride of the slowest axis: Px * Ne (3D) or Px (2D)
};
// Indices passed to eix are LOCAL in z (global - z0).  A z-slab holds planes
// z0 - 1 .. z0 + Nz (halo planes from the neighbour ranks, or the mirror
// ghost planes at the global faces).

template <int DIM>
__device__ __forceinline__ ptrdiff_t eix(const ExtLay& L, int i, int j, int k) {
    return DIM == 3 ? (ptrdiff_t)(i + 1) + (ptrdiff_t)L.Px * ((j + 1) + (ptrdiff_t)L.Ne * (k + 1))
                    : (ptrdiff_t)(i + 1) + (ptrdiff_t)L.Px * (j + 1);
}

// write the even-mirror ghost cells of data node (i, j, k) (rare path; k
// local: the z mirrors exist at the global faces only)
template <int DIM>
__device__ __noinline__ void store_mirrors(double* a, ExtLay L, int i, int j, int k, double v) {
    const int N = L.N;
    k += DIM == 3 ? L.z0 : 0;  // global
    int ci[3], cj[3], ck[3];
    int ni = 1, nj = 1, nk = 1;
    ci[0] = i;
    cj[0] = j;
    ck[0] = k;
    if (i == 1) ci[ni++] = -1;
    if (i == N - 2) ci[ni++] = N;
    if (j == 1) cj[nj++] = -1;
    if (j == N - 2) cj[nj++] = N;
    if (DIM == 3) {
        if (k == 1) ck[nk++] = -1;
        if (k == N - 2) ck[nk++] = N;
    }
    for (int ia = 0; ia < ni; ++ia)
        for (int ib = 0; ib < nj; ++ib)
            for (int ic = 0; ic < nk; ++ic)
                if (ia | ib | ic) a[eix<DIM>(L, ci[ia], cj[ib], DIM == 3 ? ck[ic] - L.z0 : 0)] = v;
}

// store with the mirror ghosts: the x mirror (same row) inline, y / z
// mirrors (rows / planes 1 and N-2, usually warp-uniform) out of line
template <int DIM>
__device__ __forceinline__ void store_ext(double* a, const ExtLay& L, int i, int j, int k, double v) {
    double* p = a + eix<DIM>(L, i, j, k);
    *p = v;
    const int N = L.N, kg = DIM == 3 ? k + L.z0 : 0;
    if (i == 1) p[-2] = v;
    if (i == N - 2) p[2] = v;  // (both when N == 3)
    if (j == 1 || j == N - 2 || (DIM == 3 && (kg == 1 || kg == N - 2))) store_mirrors<DIM>(a, L, i, j, k, v);
}

// ---- programmatic dependent launch (PDL) -----------------------------------
// The engine launches its cycle kernels with programmatic stream
// serialization (internal.hpp launch_pdl): a kernel may then begin while its
// predecessor in the stream is still running and must wait for it (grid
// completion + memory flush) before touching any data.  Grids of at most
// kPdlEarly CTAs also let THEIR successor begin at once (its CTAs park in
// pdl_wait), so chains of small launches -- the coarse levels -- overlap
// their launch latency; large grids trigger implicitly at completion so
// parked successors never take SM slots from their waves.  Both are no-ops
// for a plain launch.
constexpr unsigned kPdlEarly = 296;
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (gridDim.x * gridDim.y * gridDim.z <= kPdlEarly) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// ---- mbarrier / TMA (sm_90+; used on sm_100a) ------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// shared-window (u32) address variants for hot loops: no generic->shared
// conversion per use
__device__ __forceinline__ void mbar_expect_tx_u32(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// try_wait with a suspend-time hint: the thread sleeps in the instruction
// until the phase completes (or the hint expires) instead of spinning
__device__ __forceinline__ void mbar_wait_u32(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Ampere-style asynchronous 8-byte copy global -> shared (LDGSTS), grouped
// with commit / wait_group
__device__ __forceinline__ void cp_async8(unsigned dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// 1D bulk copy global -> shared (16-byte aligned ends, bytes a multiple of 16),
// completion counted on the mbarrier's transaction bytes
__device__ __forceinline__ void bulk_load_u32(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_u32(unsigned dst, const void* map, int c0, int c1, int c2,
                                                unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_u32(unsigned dst, const void* map, int c0, int c1, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace sgmlb
