// interp.cu — the small-level interpreter: one thread-block cluster runs a
// batch of recorded level-array operations (internal.hpp KOp) in order, with
// a cluster barrier (release / acquire) between operations.
//
// Why: on a small level array an operation is a few microseconds of work and
// its kernel is launch- and latency-bound (a C1 129^2 cycle is 70 such
// kernels).  A cluster of 16 CTAs x 512 threads keeps the arrays hot in L2
// and replaces each launch by a hardware barrier.  Measured (B200): an
// interpreted operation costs ~2 us (L2 round trips + the barrier), so the
// engine interprets the levels of <= kClusterNodes nodes (3D <= 17^3, 2D <=
// 65^2), where that beats a kernel; larger levels run faster as full-GPU
// kernels than on the 16 SMs of one cluster (C1 129^2: 4.35 -> 4.11 ms,
// 3D 65^3: 6.39 -> 5.72 ms per solve; SGML_KOP_NODES for A/B).
//
// Per-node arithmetic is exactly that of the kernels the operations replace:
// relaxation passes follow k_relax_small (the reference's relax branch,
// kernels.cpp:94-137, edge terms unfused), materialisations follow
// k_materialize4 (one node per thread with every chain corner loaded up
// front, op_mat_node; longer chains run its body, level_ops.cuh), pyramid
// steps and Dirichlet faces
// follow k_pyramid_ext and k_dirichlet_faces.  Data written by an earlier
// operation of the batch is read with coherent loads (never .nc).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.hpp"
#include "level_ops.cuh"

namespace cg = cooperative_groups;

namespace sgmlb {

namespace {

constexpr int kIThreads = 512;  // threads per CTA (4 virtual 128-thread blocks)

__device__ __forceinline__ double axw(int o) { return o == 0 ? 0.5 : 0.25; }

template <int DIM>
__device__ void op_faces(const KOpFaces& o, const BcDev& bc, int gtid, int gthreads) {
    const ExtLay& L = o.L;
    const int N = L.N;
    const int per_face = N * (DIM == 3 ? N : 1);
    for (int e = gtid; e < per_face * 2 * DIM; e += gthreads) {
        const int f = (int)(e / per_face);
        const int r = e - f * per_face;
        const int p = (int)(r % N), q = (int)(r / N);
        if (bc.neu[f]) continue;
        const int side = (f & 1) ? N - 1 : 0;
        int i, j, kg = 0;
        if (DIM == 2) {
            if (f < 2) { i = side; j = p; }
            else { i = p; j = side; }
        } else if (f < 4) {
            if (q >= L.Nz) continue;
            kg = q + L.z0;
            if (f < 2) { i = side; j = p; }
            else { i = p; j = side; }
        } else {
            if (side < L.z0 || side >= L.z0 + L.Nz) continue;
            i = p; j = q; kg = side;
        }
        const double v = o.zero ? 0.0 : dirichlet_value<DIM>(bc, N, i, j, kg);
        const int k = DIM == 3 ? kg - L.z0 : 0;
        if (o.mirrors) store_ext<DIM>(o.a, L, i, j, k, v);
        else o.a[eix<DIM>(L, i, j, k)] = v;
    }
}

template <int DIM>
__device__ void op_pyramid(const KOpPyramid& o, int gtid, int gthreads) {
    const ExtLay &Lin = o.Lin, &Lout = o.Lout;
    const int Nout = Lout.N;
    const int total = Nout * Nout * (DIM == 3 ? Lout.Nz : 1);
    const ptrdiff_t sy = Lin.Px, sz = (ptrdiff_t)Lin.Px * Lin.Ne;
    for (int e = gtid; e < total; e += gthreads) {
        const int I = e % Nout, J = (e / Nout) % Nout, K = DIM == 3 ? e / (Nout * Nout) : 0;
        const int Kin = DIM == 3 ? 2 * (K + Lout.z0) - Lin.z0 : 0;
        const double* c = o.in + eix<DIM>(Lin, 2 * I, 2 * J, Kin);
        double acc = 0.0;
#pragma unroll
        for (int r = (DIM == 3 ? -1 : 0); r <= (DIM == 3 ? 1 : 0); ++r)
#pragma unroll
            for (int q = -1; q <= 1; ++q)
#pragma unroll
                for (int p = -1; p <= 1; ++p) {
                    const double w = DIM == 3 ? (axw(p) * axw(q)) * axw(r) : axw(p) * axw(q);
                    acc = acc + w * c[r * sz + q * sy + p];
                }
        store_ext<DIM>(o.out, Lout, I, J, K, acc);
    }
}

// one relaxation pass (k_relax_small's per-node arithmetic); diag max and
// the flags through the CTA, then atomics
template <int DIM, bool SIG, bool HAS_A>
__device__ void op_relax(const KOpRelax& o, const RelaxConst& rc, int* flag, int gtid, int gthreads) {
    const ExtLay& L = o.L;
    const int nx = o.hi[0] - o.lo[0] + 1, ny = o.hi[1] - o.lo[1] + 1, nz = DIM == 3 ? o.hi[2] - o.lo[2] + 1 : 1;
    const int total = (nx > 0 && ny > 0 && nz > 0) ? nx * ny * nz : 0;
    const ptrdiff_t sy = L.Px, sz = DIM == 3 ? (ptrdiff_t)L.plane : 0;
    const double* __restrict__ u = o.in;
    double dmax = 0.0;
    int bad = 0, tiny = 0;
    for (int e = gtid; e < total; e += gthreads) {
        const int i = o.lo[0] + e % nx, j = o.lo[1] + (e / nx) % ny;
        const int k = DIM == 3 ? o.lo[2] + e / (nx * ny) : 0;
        const ptrdiff_t pos = eix<DIM>(L, i, j, k);
        const double uc = u[pos];
        const double sc = SIG ? o.sig[pos] : 1.0;
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
                    const double sbar = SIG ? 0.5 * (o.sig[pos + d] + sc) : 1.0;
                    acc = acc + stencil_t<SIG>(sbar, u[pos + d], uc, l2);
                }
        const double op = (acc * rc.pref) * rc.inv_s2;
        const double gc = o.g[pos];
        const double diag = HAS_A ? fabs((op + rc.a * uc) - gc) : fabs(op - gc);
        double value;
        if (SIG) {
            const double dtau = o.dt[pos];
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
        store_ext<DIM>(o.out, L, i, j, k, value);
        if (o.du) o.du[pos] = value - uc;
    }
    // (the flags are rare: warp-level atomics, no block barrier)
    warp_bad_commit(bad, flag, o.pass_slot);
    warp_or_commit(tiny, flag + 1);
    block_max_commit(dmax, o.slot);
}

// (release / acquire at cluster scope orders the operations' global-memory
// writes for every CTA of the cluster; an added __threadfence cost ~3 % of
// C1's solve time)
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// A materialisation one node per thread (the interpreter's form: the
// operation is latency-bound, so every corner of every chain entry is loaded
// before any arithmetic — one L2 round trip for the whole chain instead of
// one per entry; mat_node, level_ops.cuh).  Chains of at most
// NodeChain::max entries.
template <int DIM>
__device__ void op_mat_node(const KOpMaterialize& m, const ChainEntry* ch, const KOpBatch& b, int gtid,
                            int gthreads) {
    const ExtLay& Lw = m.Lw;
    const int Nw = Lw.N, nz = DIM == 3 ? Lw.Nz : 1;
    const int total = Nw * Nw * nz;
    int bad = 0, tiny = 0;
    for (int e = gtid; e < total; e += gthreads)
        mat_node<DIM, NodeChain<DIM>::max, false>(m.out, Lw, m.w, m.base, m.L0, m.wb, m.base_zero, m.ufine, m.Lf,
                                                  m.frel, ch, m.nchain, b.bc, b.homogeneous, e % Nw, (e / Nw) % Nw,
                                                  DIM == 3 ? e / (Nw * Nw) : 0, bad, tiny);
    warp_or_commit(bad, b.flag);
    warp_or_commit(tiny, b.flag + 1);
}

// one recorded operation, by the threads gtid < gthreads (materialisations:
// virtual 128-thread blocks vb0, vb0 + vstride, ...)
template <int DIM>
__device__ __forceinline__ void run_op(const KOpBatch& b, const KOp& op, ChainEntry* sch, int gtid, int gthreads,
                                       int vb0, int vstride, int vtx, int vty) {
    switch (op.kind) {
        case KOP_MEMSET:
            for (int e = gtid; e < (int)op.ms.count; e += gthreads) op.ms.p[e] = 0.0;
            break;
        case KOP_FACES:
            op_faces<DIM>(op.fc, b.bc, gtid, gthreads);
            break;
        case KOP_PYRAMID:
            op_pyramid<DIM>(op.py, gtid, gthreads);
            break;
        case KOP_MATERIALIZE: {
            const KOpMaterialize& m = op.mt;
            // the batch's copy of the whole increment table, or this chain's
            const ChainEntry* ch = m.nchain > 0 && b.chains ? sch + (m.chain - b.chains) : sch;
            if (!b.chains) {
                const int nsh = min(m.nchain, kMaxChain);
                for (int c = threadIdx.x; c < nsh; c += kIThreads) sch[c] = m.chain[c];
                __syncthreads();
                ch = sch;
            }
            if (m.nchain <= NodeChain<DIM>::max) {
                op_mat_node<DIM>(m, ch, b, gtid, gthreads);
                if (!b.chains) __syncthreads();
                break;
            }
            const int nvb = m.gx * m.gy * m.gz;
            for (int vb = vb0; vb < nvb; vb += vstride) {
                const int bx = vb % m.gx, by = (vb / m.gx) % m.gy, bz = vb / (m.gx * m.gy);
                mat4_body<DIM, 2, false, false>(m.out, m.Lw, m.w, m.base, m.L0, m.wb, m.base_zero, m.ufine, m.Lf,
                                                m.frel, m.chain, m.nchain, ch, b.bc, b.homogeneous, b.flag,
                                                m.xtail, 0, bx, by, bz, vtx, vty);
            }
            if (!b.chains) __syncthreads();  // sch is reused by the next materialisation
            break;
        }
        case KOP_RELAX: {
            const RelaxConst& rc = b.rc[op.level];
            if (b.sig) {
                if (rc.has_a) op_relax<DIM, true, true>(op.rx, rc, b.flag, gtid, gthreads);
                else op_relax<DIM, true, false>(op.rx, rc, b.flag, gtid, gthreads);
            } else {
                if (rc.has_a) op_relax<DIM, false, true>(op.rx, rc, b.flag, gtid, gthreads);
                else op_relax<DIM, false, false>(op.rx, rc, b.flag, gtid, gthreads);
            }
            break;
        }
        default:
            break;
    }
}

template <int DIM>
__global__ void __launch_bounds__(kIThreads, 1) k_kop_batch(const __grid_constant__ KOpBatch b) {
    __shared__ ChainEntry sch[kMaxChain];
    // the recorded operations, staged once in shared memory: an operation's
    // fields then cost a shared-memory read instead of a constant-cache miss
    // (one L2 round trip) when the interpreter reaches it
    __shared__ KOp sop[kMaxKOps];
    {
        const unsigned long long* src = reinterpret_cast<const unsigned long long*>(b.op);
        unsigned long long* dst = reinterpret_cast<unsigned long long*>(sop);
        const int words = b.count * (int)(sizeof(KOp) / sizeof(unsigned long long));
        for (int t = threadIdx.x; t < words; t += kIThreads) dst[t] = src[t];
    }
    pdl_begin();
    if (b.chains)  // (static per solver: one copy serves every materialisation)
        for (int c = threadIdx.x; c < b.nchains; c += kIThreads) sch[c] = b.chains[c];
    __syncthreads();
    // (interpreted level arrays hold far fewer than 2^31 elements)
    const int crank = (int)cg::this_cluster().block_rank();
    const int csize = (int)cg::this_cluster().num_blocks();
    constexpr int VB = kIThreads / (MBX * MBY);  // virtual 128-thread blocks per CTA
    const int sub = threadIdx.x / (MBX * MBY);
    const int vtx = threadIdx.x % MBX, vty = (threadIdx.x / MBX) % MBY;
    for (int i = 0; i < b.count; ++i) {
        const KOp& op = sop[i];
        // Solo operations (arrays of <= kSoloNodes nodes) run on CTA 0 alone,
        // consecutive ones separated by __syncthreads (CTA-scope ordering of
        // its global-memory accesses) instead of a cluster barrier each; a
        // cluster barrier closes the run.  Saves the barrier and the wait for
        // L2 store acknowledgements per operation where the work is a few
        // hundred nodes.
        const bool solo = op.solo != 0;
        if (!solo) run_op<DIM>(b, op, sch, crank * kIThreads + threadIdx.x, csize * kIThreads, crank * VB + sub,
                               csize * VB, vtx, vty);
        else if (crank == 0) run_op<DIM>(b, op, sch, threadIdx.x, kIThreads, sub, VB, vtx, vty);
        if (solo && i + 1 < b.count && sop[i + 1].solo) {
            if (crank == 0) __syncthreads();
        } else {
            cluster_barrier();
        }
    }
}

int g_cluster = 0;

}  // namespace

int interp_cluster_size() {
    if (g_cluster) return g_cluster;
    int best = 8;
    if (cudaFuncSetAttribute(k_kop_batch<3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        cudaFuncSetAttribute(k_kop_batch<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(kIThreads);
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 16;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_kop_batch<3>, &cfg) == cudaSuccess && n > 0) best = 16;
    }
    (void)cudaGetLastError();
    g_cluster = best;
    return best;
}

void launch_kop_batch(int dim, const KOpBatch& b, cudaStream_t s) {
    const int cs = interp_cluster_size();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kIThreads);
    cfg.stream = s;
    cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = a;
    cfg.numAttrs = 2;
    if (dim == 2) cudaLaunchKernelEx(&cfg, k_kop_batch<2>, b);
    else cudaLaunchKernelEx(&cfg, k_kop_batch<3>, b);
}

}  // namespace sgmlb
