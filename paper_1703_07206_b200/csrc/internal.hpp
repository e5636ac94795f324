// internal.hpp — launchers shared by the engine and the C-ABI layer.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace sgmlb {

// One pending interpolation increment: a level-`level` compact variation.
struct ChainEntry {
    const double* du;
    int level;
    int Nl;
};

// Ordered list of pending interpolation increments (level, compact du).
// Applied left to right: u <- ((u + I_l0(du0)) + I_l1(du1)) + ...
constexpr int kMaxChain = 96;
struct Chain {
    int count;
    int level[kMaxChain];
    int Nl[kMaxChain];
    const double* du[kMaxChain];
};

// Production pyramid step (materialize.cu): same contract as launch_pyramid_step.
void launch_pyramid2(int dim, const double* in, int Nin, double* out, int Nout, const BcDev& bc,
                     cudaStream_t s);
// kernels.cpp:28-81 — one literal full-grid averaging pass at stride lam.
void launch_restrict_pass(int dim, const double* in, double* out, int N, int lam, const BcDev& bc,
                          cudaStream_t s);
// One restriction-pyramid step: level-(m+1) compact <- level-m compact
// (bitwise equal to restriction(f, m+1) on the subset).
void launch_pyramid_step(int dim, const double* in, int Nin, double* out, int Nout,
                         const BcDev& bc, cudaStream_t s);
// kernels.cpp:176-237 — literal full-grid relaxation-interpolation pass.
void launch_relax_literal(int dim, bool sig, double* u, double* du, const double* up,
                          const double* dup, const double* g, const double* sigma, int N, int level,
                          const RelaxConst& rc, const BcDev& bc, unsigned long long* diag_slot,
                          int* flag, cudaStream_t s);
// Relaxation of every node of a level-compact array (all nodes are subset
// nodes there); du_out may be null.
void launch_relax_compact(int dim, bool sig, double* uo, double* duo, const double* ui,
                          const double* g, const double* sigma, int Nc, const RelaxConst& rc,
                          const BcDev& bc, unsigned long long* diag_slot, int* flag,
                          cudaStream_t s);
// The production relaxation pass (relax_tiled.cu): same contract as
// launch_relax_compact, z-marching shared-memory tiles.
void launch_relax_tiled(int dim, bool sig, double* uo, double* duo, const double* ui,
                        const double* g, const double* sigma, int Nc, const RelaxConst& rc,
                        const BcDev& bc, unsigned long long* diag_slot, int* flag, cudaStream_t s);
// The production residual recurrence on the same tiles: r -= A(e) + a e,
// r = 0 on Dirichlet nodes, u_tot += e (utot may be null), max|r| (slot may
// be null); rc = relax_const(level 0).
void launch_residual_tiled(int dim, bool sig, double* r, const double* e, double* utot,
                           const double* sigma, int N, const RelaxConst& rc, const BcDev& bc,
                           unsigned long long* rmax_slot, cudaStream_t s);
// Materialise the level-w compact input of the next relax step from the
// tooth's state: Dirichlet value, the finest relaxed level lf = w + frel
// (ufine, Nf nodes per axis) at its subset nodes, or base + pending
// increments elsewhere.
void launch_materialize(int dim, double* out, int Nw, int w, const double* base, int N,
                        bool base_zero, const double* ufine, int Nf, int frel, const Chain& chain,
                        const BcDev& bc, bool homogeneous, int* flag, cudaStream_t s);
// Production materialisation (materialize.cu): same contract, chain read
// from a device array of `nchain` entries, 4 x-nodes per thread.
void launch_materialize4(int dim, double* out, int Nw, int w, const double* base, int N,
                         bool base_zero, const double* ufine, int Nf, int frel,
                         const ChainEntry* chain, int nchain, const BcDev& bc, bool homogeneous,
                         int* flag, cudaStream_t s);
// kernels.cpp:243-297 (+ cycle.cpp:194-198 fused): r -= A(e) + a e,
// r = 0 on Dirichlet faces, u_tot += e (if non-null), max|r| (if non-null).
void launch_residual(int dim, bool sig, double* r, const double* e, double* utot,
                     const double* sigma, int N, double inv_h2, double pref, double a,
                     const BcDev& bc, unsigned long long* rmax_slot, cudaStream_t s);
void launch_max_abs(const double* f, uint64_t total, unsigned long long* slot, cudaStream_t s);
void launch_sub_scalar(double* f, uint64_t total, double v, cudaStream_t s);
void launch_add_into(double* dst, const double* src, uint64_t total, cudaStream_t s);
void launch_apply_boundary(int dim, double* u, int N, const BcDev& bc, bool homogeneous,
                           cudaStream_t s);
void launch_check_positive(const double* f, uint64_t total, int* flag, cudaStream_t s);
void launch_check_finite(const double* f, uint64_t total, int* flag, cudaStream_t s);

}  // namespace sgmlb
