// internal.hpp — launchers shared by the engine and the C-ABI layer.
#pragma once

#include <cstdint>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

#include "device.cuh"

namespace sgmlb {

// Kernel launch with programmatic stream serialization (PDL, device.cuh
// pdl_begin); SGML_NO_PDL=1 launches plainly (A/B switch, same results).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// Literal (reference-shaped, dense x-fastest) kernels: kernels.cu.  They back
// the kernel-level C-ABI and the literal engine.
// ---------------------------------------------------------------------------

// kernels.cpp:28-81 — one literal full-grid averaging pass at stride lam.
void launch_restrict_pass(int dim, const double* in, double* out, int N, int lam, const BcDev& bc,
                          cudaStream_t s);
// kernels.cpp:176-237 — literal full-grid relaxation-interpolation pass.
void launch_relax_literal(int dim, bool sig, double* u, double* du, const double* up,
                          const double* dup, const double* g, const double* sigma, int N, int level,
                          const RelaxConst& rc, const BcDev& bc, unsigned long long* diag_slot,
                          int* flag, int pass_slot, cudaStream_t s);
// kernels.cpp:243-297 (+ cycle.cpp:194-198 fused): r -= A(e) + a e,
// r = 0 on Dirichlet faces, u_tot += e (if non-null), max|r| (if non-null).
void launch_residual(int dim, bool sig, double* r, const double* e, double* utot,
                     const double* sigma, int N, double inv_h2, double pref, double a,
                     const BcDev& bc, unsigned long long* rmax_slot, cudaStream_t s, int compact = 0);
void launch_max_abs(const double* f, uint64_t total, unsigned long long* slot, cudaStream_t s);
void launch_fill(double* f, uint64_t total, double v, cudaStream_t s);
void launch_sub_scalar(double* f, uint64_t total, double v, cudaStream_t s);
void launch_add_into(double* dst, const double* src, uint64_t total, cudaStream_t s);
void launch_apply_boundary(int dim, double* u, int N, const BcDev& bc, bool homogeneous,
                           cudaStream_t s);
void launch_check_positive(const double* f, uint64_t total, int* flag, cudaStream_t s);
void launch_check_finite(const double* f, uint64_t total, int* flag, cudaStream_t s);

// ---------------------------------------------------------------------------
// Compact engine (ghost-extended padded level arrays, device.cuh ExtLay)
// ---------------------------------------------------------------------------

// nz < 0: the whole level (Nz = N, z0 = 0); otherwise a z-slab of planes
// [z0, z0 + nz) with halo planes
ExtLay make_ext(int dim, int N, int z0 = 0, int nz = -1);
uint64_t ext_size(int dim, const ExtLay& L);  // doubles to allocate

// One pending interpolation increment: a level-`level` compact variation.
struct ChainEntry {
    const double* du;
    ExtLay L;
    int level;
    int fslot;  // cycle slot of the reference pass that adds this increment
};
// Most increments one materialisation keeps in shared memory; the engine
// folds pending increments into a full-grid base before a chain outgrows it
// (only reached for large n_r).  A single visit may still add more (n_r >
// kMaxChain + 1): the kernel then reads the entries past kMaxChain from
// global memory.
constexpr int kMaxChain = 96;

// TMA descriptors of one relaxation / residual launch (relax_tiled.cu):
// u = input window array (box tile + halo), g = source / r (box tile),
// s = sigma (box tile + halo), t = u_tot (box tile).
struct TmaSet {
    CUtensorMap u, g, s, t;
};
// TMA box shapes of the relaxation tiles: u/sigma box (tile + halo) and
// g/r/u_tot box (tile), {x, y, plane}.
void tile_boxes(int dim, unsigned* box_u, unsigned* box_g);
int relax_tiled_zb(int dim, int cols, int nz, int per_sm);

// Box of data nodes a relaxation / residual launch covers: every node not on
// a Dirichlet face (those keep their face value, resident in the buffers).
struct NodeRange {
    int lo[3], hi[3];
};
// All c passes of one visit of a small level array in one CTA (engine:
// levels of at most kSmallNodes relaxed nodes, single GPU, faces settled).
constexpr int kSmallThreads = 512;
constexpr int kSmallNodes = 6144;
constexpr int kSmallMaxPasses = 16;
// the one-CTA visit stages three whole level arrays in shared memory; the
// largest small array is 3D N = 17 (20 x 19 x 19 doubles) or 2D N = 65 (68 x 67)
constexpr int kSmallMaxExt = 20 * 19 * 19;
constexpr int kSmallSmem = 3 * kSmallMaxExt * 8;
struct SmallPasses {
    const double* in[kSmallMaxPasses];
    double* out[kSmallMaxPasses];
    double* du[kSmallMaxPasses];
    unsigned long long* slot[kSmallMaxPasses];
    int pass_slot[kSmallMaxPasses];
    int count;
    const double* g;
    const double* sig;  // level sigma (with ghosts), SIG only
    const double* dt;   // per-node pseudo-time step, SIG only
};
void launch_relax_small(int dim, bool sig, const SmallPasses& sp, const ExtLay& L, const NodeRange& rg,
                        const RelaxConst& rc, int* flag, cudaStream_t s);
// One relaxation pass over a level array (every node a subset node):
// uo (with mirror ghosts), duo = uo - ui (nullable, DU arrays), diag max
// into diag_slot.  flag[0] <- 1 on a non-finite output, flag[1] <- 1 on a
// nonzero output below 2^-969 in magnitude; flag[1] == 0 on entry lets the
// pass fuse its edge terms (exact for such inputs).
void launch_relax_tma(int dim, bool sig, const TmaSet& tm, double* uo, double* duo,
                      const ExtLay& L, const NodeRange& rg, const RelaxConst& rc,
                      unsigned long long* diag_slot, int* flag, int pass_slot, cudaStream_t s);
// Residual recurrence at level 0 over the range: r -= A(e) + a e (tm.u = e,
// tm.g = r, r written with mirror ghosts), u_tot += e (tm.t / utot,
// nullable), max|r| into rmax_slot; reads flag[1] as the relaxation pass.
// rc = relax_const(level 0).  guarded: nothing happens when flag[0] (a failed
// cycle) is set.
void launch_residual_tma(int dim, bool sig, const TmaSet& tm, double* r, double* utot,
                         const ExtLay& L, const NodeRange& rg, const RelaxConst& rc,
                         unsigned long long* rmax_slot, int* flag, bool guarded, cudaStream_t s);
// Dirichlet-face nodes of an extended level array <- 0 (zero) or their face
// value (the reference's lowest-face-id rule), with their mirror ghost cells
// unless `mirrors` is false (DU arrays keep all-zero ghosts).
void launch_dirichlet_faces(int dim, double* a, const ExtLay& L, const BcDev& bc, bool zero,
                            bool mirrors, cudaStream_t s);
// Materialise the level-w input of the next relax step from the tooth's
// state: Dirichlet value, the finest relaxed level lf = w + frel (ufine) at
// its subset nodes, or base + the pending increments chain[0..nchain).
// base holds the level-wb subset (0: the level-0 array; a multi-GPU solve
// passes the replicated level-vrep sample for replicated targets).
// diag: also report the first chain entry whose partial sum turns non-finite
// at an interpolated node (flag[4] <- min entry fslot; failure re-runs only)
void launch_materialize4(int dim, double* out, const ExtLay& Lw, int w, const double* base,
                         const ExtLay& L0, int wb, bool base_zero, const double* ufine, const ExtLay& Lf,
                         int frel, const ChainEntry* chain, int nchain, const BcDev& bc,
                         bool homogeneous, int* flag, bool diag, cudaStream_t s, int kb = 0, int ke = -1);
// ---- small-level interpreter (interp.cu) -------------------------------------
// The operations of a cycle on small level arrays (coarse levels of large
// grids; whole cycles of small ones) recorded by the engine and executed
// in order by ONE launch of a thread-block cluster, with a cluster barrier
// between operations, instead of one kernel each.  Same per-node arithmetic
// as the kernels they replace.
enum KOpKind : int { KOP_MEMSET = 0, KOP_FACES = 1, KOP_PYRAMID = 2, KOP_MATERIALIZE = 3, KOP_RELAX = 4 };
struct KOpMemset {
    double* p;
    long long count;
};
struct KOpFaces {  // k_dirichlet_faces
    double* a;
    ExtLay L;
    int zero, mirrors;
};
struct KOpPyramid {  // k_pyramid_ext: level m -> m + 1
    const double* in;
    double* out;
    ExtLay Lin, Lout;
};
struct KOpMaterialize {  // k_materialize4 (no diagnostic mode)
    double* out;
    const double* base;
    const double* ufine;
    const ChainEntry* chain;
    ExtLay Lw, L0, Lf;
    int w, wb, base_zero, frel, nchain, xtail, gx, gy, gz;
};
struct KOpRelax {  // one relaxation pass over a level array (k_relax_small's per-node arithmetic)
    const double* in;
    double* out;
    double* du;
    const double* g;
    const double* sig;
    const double* dt;
    unsigned long long* slot;
    ExtLay L;
    int lo[3], hi[3];
    int pass_slot;
};
struct KOp {
    int kind;
    int level;
    int solo;  // run by the batch's first CTA alone (small arrays, see interp.cu)
    union {
        KOpMemset ms;
        KOpFaces fc;
        KOpPyramid py;
        KOpMaterialize mt;
        KOpRelax rx;
    };
};
// one launch: the operations share the cycle's boundary set, relaxation
// constants per level and flags; kernel parameters are limited to 32 KB
constexpr int kMaxKOps = 160;
struct KOpBatch {
    BcDev bc;
    int* flag;
    int homogeneous;
    int count;
    int sig;
    // the solver's whole pending-increment table when it has at most
    // kMaxChain entries (copied to shared memory once per batch), else null
    const ChainEntry* chains;
    int nchains;
    RelaxConst rc[14];  // per level
    KOp op[kMaxKOps];
};
static_assert(sizeof(KOpBatch) <= 32000, "KOpBatch travels as kernel parameters (32 KB)");
static_assert(sizeof(KOp) % 8 == 0 && alignof(KOp) >= 8, "KOp is staged in 8-byte words");
// level arrays of at most this many nodes are interpreted (2D: at most
// kClusterNodes2D)
constexpr int kClusterNodes = 5000;
constexpr int kClusterNodes2D = 129 * 129;
// interpreted 2D operations on level arrays of at most this many nodes run
// on one CTA of the cluster (<= 17^2: at most one node per thread; C1 129^2
// 4.13 -> 3.99 ms per solve; 3D levels <= 5^3 gained nothing, <= 9^3 and 2D
// <= 33^2 lost — several nodes per thread, each round an L2 round trip)
constexpr int kSoloNodes = 512;
// cluster of CTAs that runs a batch (16 where the device allows it, else 8)
int interp_cluster_size();
// the launch geometry launch_materialize4 uses for a whole level array
// (virtual grid of the interpreter's materialisation)
void materialize_grid(int dim, const ExtLay& Lw, const BcDev& bc, int& gx, int& gy, int& gz, int& xtail);
void launch_kop_batch(int dim, const KOpBatch& b, cudaStream_t s);

// per-node pseudo-time step of the sigma relaxation at every node of a level
// array (own planes), from the level's sigma (with ghosts / halos)
void launch_dtau_ext(int dim, const double* sig, const ExtLay& L, double* dt, const RelaxConst& rc, cudaStream_t s);
// 3D: out planes [kb, ke) (local) <- in at positions << shift (level subsample)
void launch_sample_ext(const double* in, const ExtLay& Lin, double* out, const ExtLay& Lout, int shift, int kb,
                       int ke, cudaStream_t s);
// Restriction pyramid step level m -> m+1, output planes
// [kb, ke) (local; ke < 0: all planes of Lout).
void launch_pyramid_ext(int dim, const double* in, const ExtLay& Lin, double* out, const ExtLay& Lout,
                        cudaStream_t s, int kb = 0, int ke = -1);
void launch_scatter_ext(int dim, const double* dense, double* ext, const ExtLay& L, cudaStream_t s);
void launch_gather_ext(int dim, const double* ext, const ExtLay& L, double* dense, cudaStream_t s);

// ---- post-solve fields (fields.cu; dense x-fastest layout) ----------------
// axis_derivative (problems.cpp:74-97)
void launch_axis_derivative(int dim, const double* u, double* d, int N, int axis, double inv2h, cudaStream_t s);
// gradient (problems.cpp:391-396); with f_raw, deformation_velocity's
// -g / (t f_raw + raw_integral) (problems.cpp:327-341), flag[0] on a zero denominator
void launch_gradient(int dim, const double* u, double* const* g, int N, double inv2h, const double* f_raw,
                     double raw_integral, double t, int* flag, cudaStream_t s);
void launch_curl(const double* const* psi, double* const* v, int N, double inv2h, cudaStream_t s);
void launch_divergence(int dim, const double* const* v, double* d, int N, double inv2h, cudaStream_t s);
// move_nodes (problems.cpp:343-372) from the gradient fields g
void launch_move_nodes(int dim, const double* const* g, const double* f_raw, double raw_integral, int N, double h,
                       double t, int steps, double* const* pos, cudaStream_t s);
// integrate_streamline (problems.cpp:415-455), one thread per seed
void launch_streamlines(int dim, const double* const* v, int N, double h, const double* seeds, int nseeds,
                        double step, int max_steps, double* pts, int* counts, int* stops, cudaStream_t s);
// sample_vector (problems.cpp:407-413) at device points (3 doubles each)
void launch_sample_points(int dim, const double* const* v, int nv, int N, double h, const double* pts, int count,
                          double* out, cudaStream_t s);

// ---- problem builders (fields.cu; host-evaluated libm tables) -------------
void launch_fill_poisson3d(double* f, int N, const double* s, double scale, cudaStream_t st);
void launch_fill_sinsin2d(double* f, int N, const double* s, double scale, cudaStream_t st);
void launch_fill_poisson2d(double* f, int N, double h, cudaStream_t st);
void launch_fill_radial(double* f, int N, const double* table, cudaStream_t st);
void launch_scatter_pairs(double* f, const unsigned long long* idx, const double* val, int count, cudaStream_t st);

}  // namespace sgmlb
