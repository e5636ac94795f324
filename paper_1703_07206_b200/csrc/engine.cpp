// engine.cpp — host orchestration of the SGML schedule on one B200.
//
// Two engines run the reference's cycle (cycle.cpp:76-111):
//
//  * literal: the reference's full-grid passes one for one (restriction
//    recomputed per Restrict(v) step, every relax pass over all N^d nodes).
//    Kept as the parity/measurement baseline.
//
//  * compact (default): the same arithmetic on level-compact arrays.
//    - Restriction: one pyramid per cycle, P_{m+1} = pass_m(P_m) on
//      level-(m+1) nodes only (bit-identical on the subset,
//      which is all relax reads, F3).
//    - Relax at level v >= 1 touches only the S_v subset nodes (compact U_v).
//      Non-subset nodes of the reference receive u_prev + I(du_prev) each
//      pass; with du reset at every level change the first of those adds
//      I(0) and the others add I(du_k) of the previous passes.  Those
//      increments are kept compact (DU_v) and applied lazily, in the
//      reference's order, when the next level's input is materialised
//      (base + I_v1(du) + ... + I_{w+1}(du)), so coarse levels never sweep
//      the full grid.  Dirichlet nodes always hold their face value after
//      the first pass of a cycle.
//    - Level-0 passes are full-grid relaxations (every node is a subset
//      node at level 0); du at level 0 is never read, so it is not written.
//   Everything a reference caller observes (state.u, the diagnostic trace,
//   the work counter, the residual history) is bit-identical, up to the
//   sign of exact zeros (I(0) is not added).
#include "engine.hpp"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>

namespace sgmlb {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }

void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(SGML_ECUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what);
}

BcDev to_dev(const sgml_bc& bc) {
    BcDev d{};
    for (int f = 0; f < 6; ++f) {
        d.neu[f] = bc.kind[f] == 1;
        d.val[f] = bc.value[f];
    }
    return d;
}

bool any_dirichlet(const sgml_bc& bc, int dim) {
    for (int f = 0; f < 2 * dim; ++f)
        if (bc.kind[f] != 1) return true;
    return false;
}

// grid.cpp:10-23
sgml_grid make_grid_or_throw(int dim, int n) {
    if (dim != 2 && dim != 3) fail(SGML_EINVAL, "make_grid: dim must be 2 or 3");
    if (n < 1 || n > 13) fail(SGML_EINVAL, "make_grid: n must lie in [1, 13]");
    sgml_grid g{};
    g.dim = dim;
    g.n = n;
    g.N = (1 << n) + 1;
    g.h = 1.0 / (g.N - 1);
    g.total = 1;
    for (int d = 0; d < dim; ++d) g.total *= (uint64_t)g.N;
    return g;
}

// cycle.cpp:21-24
int relax_count(int n, int n_r, int v1) {
    const long long doubling = 1LL << (n - v1);
    return (int)std::min<long long>(n_r, doubling);
}

int slab_vrep(int n, int nranks, int replicate_n) {
    if (nranks <= 1) return 0;
    const int t0 = (1 << n) / nranks, rn = replicate_n > 0 ? replicate_n : SGML_REPLICATE_N;
    int v = 0;
    // replicated coarse levels cost a redundant pass on every rank; slab
    // levels cost a halo exchange (latency) per producer
    while ((t0 >> v) >= 2 && (1 << (n - v)) + 1 > rn) ++v;
    return v;
}

// kernels.cpp:182-188 and the sigma == 1 step (see RelaxConst)
RelaxConst relax_const(int dim, int level, double h, double a, double safety, bool homogeneous, int compact) {
    RelaxConst rc{};
    const int lam = 1 << level;
    const double s = lam * h;
    rc.inv_s2 = 1.0 / (s * s);
    // stencil.hpp:49,52 for the radial form; the compact 5/7-point form
    // has prefactor 1 and the Gershgorin step K = 1/(2d)
    rc.pref = compact ? 1.0 : (dim == 2 ? 0.5 : 3.0 / 13.0);
    rc.kdim = compact ? (dim == 2 ? 1.0 / 4.0 : 1.0 / 6.0) : (dim == 2 ? 1.0 / 3.0 : 13.0 / 44.0);
    rc.compact = compact ? 1 : 0;
    rc.a = a;
    rc.safety = safety;
    const double smax = 1.0;
    rc.dtau1 = safety * rc.kdim / (rc.inv_s2 * smax);
    rc.denom1 = 1.0 - rc.dtau1 * a;
    rc.homogeneous = homogeneous ? 1 : 0;
    rc.has_a = a != 0.0;
    return rc;
}

double* dalloc(size_t count) {
    void* p = nullptr;
    SGML_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double)));
    return (double*)p;
}

void dfree(double* p) {
    if (p) cudaFree(p);
}

// kernels.cpp:367-386: serial Kahan sum in linear order, on a host copy.
double trapezoid_mean_host(sgml_ctx* ctx, const sgml_grid& g, const double* dfield) {
    const size_t bytes = g.total * sizeof(double);
    if (ctx->h_stage_bytes < bytes) {
        if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
        ctx->h_stage = nullptr;
        SGML_CUDA(cudaMallocHost((void**)&ctx->h_stage, bytes));
        ctx->h_stage_bytes = bytes;
    }
    // the copy streams in chunks; the (inherently serial) sum runs behind it
    constexpr size_t kChunk = size_t(1) << 18;  // doubles (2 MB)
    const size_t nchunks = (g.total + kChunk - 1) / kChunk;
    while (ctx->h_stage_events.size() < std::min<size_t>(nchunks, 64)) {
        cudaEvent_t e;
        SGML_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->h_stage_events.push_back(e);
    }
    const size_t nev = ctx->h_stage_events.size();
    const size_t per = (nchunks + nev - 1) / nev * kChunk;  // elements per event
    for (size_t c0 = 0, q = 0; c0 < g.total; c0 += per, ++q) {
        const size_t cnt = std::min(per, (size_t)g.total - c0);
        SGML_CUDA(cudaMemcpyAsync(ctx->h_stage + c0, dfield + c0, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                  ctx->stream));
        SGML_CUDA(cudaEventRecord(ctx->h_stage_events[q], ctx->stream));
    }
    size_t ready = 0, next = 0;
    const double* f = ctx->h_stage;
    const int N = g.N;
    double sum = 0.0, comp = 0.0;
    size_t pos = 0;
    const int KMAX = g.dim == 3 ? N : 1;
    for (int k = 0; k < KMAX; ++k) {
        const double wk = (g.dim == 3 && (k == 0 || k == N - 1)) ? 0.5 : 1.0;
        for (int j = 0; j < N; ++j) {
            while (ready < pos + (size_t)N) {  // this row has arrived
                SGML_CUDA(cudaEventSynchronize(ctx->h_stage_events[next++]));
                ready = std::min((size_t)g.total, ready + per);
            }
            const bool jf = j == 0 || j == N - 1;
            for (int i = 0; i < N; ++i, ++pos) {
                double w = 1.0;
                if (i == 0 || i == N - 1) w *= 0.5;
                if (jf) w *= 0.5;
                if (wk != 1.0) w *= 0.5;
                const double y = w * f[pos] - comp;
                const double t = sum + y;
                comp = (t - sum) - y;
                sum = t;
            }
        }
    }
    double wsum = 1.0;
    for (int d = 0; d < g.dim; ++d) wsum *= (double)(N - 1);
    return sum / wsum;
}

}  // namespace sgmlb

using namespace sgmlb;

// ---------------------------------------------------------------------------
// TMA descriptors
// ---------------------------------------------------------------------------

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        SGML_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) fail(SGML_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

CUtensorMap make_map(int dim, const double* p, const ExtLay& L, const unsigned* box) {
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)L.Ne, (cuuint64_t)L.Ne, (cuuint64_t)(L.Nz + 2)};
    cuuint64_t strides[2] = {(cuuint64_t)L.Px * 8, (cuuint64_t)L.Px * L.Ne * 8};
    cuuint32_t bx[3] = {box[0], box[1], box[2]};
    cuuint32_t es[3] = {1, 1, 1};
    const CUresult rc = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, dim, const_cast<double*>(p), dims,
                                    strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) fail(SGML_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)rc) + ")");
    return m;
}

}  // namespace

void sgml_solver::add_maps(const double* p, const ExtLay& L, bool want_u, bool want_g) {
    unsigned bu[3], bg[3];
    tile_boxes(g.dim, bu, bg);
    if (want_u) map_u.emplace_back(p, make_map(g.dim, p, L, bu));
    if (want_g) map_g.emplace_back(p, make_map(g.dim, p, L, bg));
}

const CUtensorMap& sgml_solver::umap(const double* p) const {
    for (const auto& e : map_u)
        if (e.first == p) return e.second;
    fail(SGML_ELOGIC, "internal: no TMA descriptor for buffer");
}
const CUtensorMap& sgml_solver::gmap(const double* p) const {
    for (const auto& e : map_g)
        if (e.first == p) return e.second;
    fail(SGML_ELOGIC, "internal: no TMA descriptor for buffer");
}

// ---------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------

double* sgml_solver::alloc(size_t count) {
    double* p = dalloc(count);
    bytes += std::max<size_t>(count, 1) * sizeof(double);
    SGML_CUDA(cudaMemsetAsync(p, 0, std::max<size_t>(count, 1) * sizeof(double), ctx->stream));
    return p;
}

sgml_solver::~sgml_solver() {
    if (ctx) cudaSetDevice(ctx->device);
    dfree(r); dfree(utot); dfree(A); dfree(B); dfree(fin); dfree(dense);
    dfree(fin2); dfree(uout[0]); dfree(uout[1]);
    for (size_t m = 1; m < P.size(); ++m) dfree(P[m]);
    for (double* s : S) dfree(s);
    for (double* d : DT) dfree(d);
    for (size_t v = 1; v < U.size(); ++v) { dfree(U[v][0]); dfree(U[v][1]); }
    for (auto& lst : DU) for (double* d : lst) dfree(d);
    dfree(Lg); dfree(Lscr); dfree(Lu); dfree(Lup); dfree(Ldu); dfree(Ldup);
    for (double* s : Lsig) dfree(s);
    for (cudaEvent_t e : evpool) cudaEventDestroy(e);
    if (hx_stream) {
        cudaStreamSynchronize(hx_stream);
        cudaStreamDestroy(hx_stream);
        cudaEventDestroy(hx_ready);
        cudaEventDestroy(hx_done);
    }
    for (CycleGraph& G : graphs) {
        if (G.exec) cudaGraphExecDestroy(G.exec);
        for (cudaEvent_t e : G.events) cudaEventDestroy(e);
    }
    if (tev0) cudaEventDestroy(tev0);
    if (tev1) cudaEventDestroy(tev1);
    if (d_chain) cudaFree(d_chain);
    dfree(BS);
    if (d_cycle) cudaFree(d_cycle);
    if (d_flag) cudaFree(d_flag);
    if (h_cycle) cudaFreeHost(h_cycle);
    if (h_flag) cudaFreeHost(h_flag);
}


void sgml_solver::check_launch(int cls) {
    static const char* names[] = {"relax0", "relax_coarse", "materialize", "pyramid", "residual",
                                  "literal", "other", "?"};
    const cudaError_t e1 = cudaGetLastError();
    const cudaError_t e2 = cudaStreamSynchronize(ctx->stream);
    const cudaError_t e = e1 != cudaSuccess ? e1 : e2;
    if (e != cudaSuccess)
        fail(SGML_ECUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in kernel class " +
                             names[cls & 7] + " (launch #" + std::to_string(launches) + ")");
}

cudaEvent_t sgml_solver::next_event() {
    if (capturing) {  // events recorded inside a graph belong to it
        cudaEvent_t e;
        SGML_CUDA(cudaEventCreate(&e));
        capturing->events.push_back(e);
        return e;
    }
    if (evused == evpool.size()) {
        cudaEvent_t e;
        SGML_CUDA(cudaEventCreate(&e));
        evpool.push_back(e);
    }
    return evpool[evused++];
}

void sgml_solver::harvest_spans() {
    for (const Span& sp : spans) {
        float ms = 0.f;
        const cudaError_t e = cudaEventElapsedTime(&ms, sp.a, sp.b);
        if (e == cudaSuccess) {
            cls_ms[sp.cls] += ms;
            cls_n[sp.cls] += 1;
        } else {
            static int reported = 0;
            if (!reported++) std::fprintf(stderr, "sgml: span timing unavailable (%s)\n", cudaGetErrorString(e));
            (void)cudaGetLastError();  // (not sticky: clear it)
        }
    }
    spans.clear();
    evused = 0;
}

void sgml_solver::build(sgml_ctx* c, int dim, int n, const sgml_bc& bcin, double a_,
                        const double* sigma_dev, const sgml_solver_cfg& cfg_,
                        const sgml_solver_opts& opts_) {
    ctx = c;
    g = make_grid_or_throw(dim, n);
    if (!(cfg_.tol > 0.0)) fail(SGML_EINVAL, "solve: tol must be positive");
    if (cfg_.n_r < 1) fail(SGML_EINVAL, "solve: n_r must be >= 1");
    if (opts_.stencil != SGML_STENCIL_RADIAL && opts_.stencil != SGML_STENCIL_COMPACT)
        fail(SGML_EINVAL, "solver: unknown stencil family");
    bc_host = bcin;
    bc = to_dev(bcin);
    all_neumann = !any_dirichlet(bcin, dim);
    a = a_;
    has_sigma = sigma_dev != nullptr;
    cfg = cfg_;
    opts = opts_;
    if (std::getenv("SGML_NO_SMALL_LEVELS")) opts.small_levels = -1;  // (INTEGRATION.md switch)
    SGML_CUDA(cudaSetDevice(ctx->device));

    // schedule (cycle.cpp:28-45) flattened to relax passes
    int pass_idx = 0;
    for (int v1 = n - 1; v1 >= 0; --v1) {
        const int cnt = relax_count(n, cfg.n_r, v1);
        for (int v = v1; v >= 0; --v) {
            pass_idx += v;  // Restrict(v) costs v passes
            for (int k = 0; k < cnt; ++k) { pass_level.push_back(v); pass_index.push_back(pass_idx++); }
        }
    }
    const int tail = relax_count(n, cfg.n_r, 0 /* 2^n cap */);
    for (int k = 0; k < tail; ++k) { pass_level.push_back(0); pass_index.push_back(pass_idx++); }
    units_per_cycle = (uint64_t)pass_idx;
    n_slots = (int)pass_level.size();

    SGML_CUDA(cudaMalloc((void**)&d_cycle, (n_slots + 4) * sizeof(unsigned long long)));
    SGML_CUDA(cudaMalloc((void**)&d_flag, 8 * sizeof(int)));
    SGML_CUDA(cudaMallocHost((void**)&h_cycle, (n_slots + 4) * sizeof(unsigned long long)));
    SGML_CUDA(cudaMallocHost((void**)&h_flag, 8 * sizeof(int)));

    const uint64_t T = g.total;
    Nl.resize(n);
    for (int v = 0; v < n; ++v) Nl[v] = (1 << (n - v)) + 1;

    // multi-GPU clique of the context: z-slab plan
    tp = ctx->tp.get();
    nrk = tp ? tp->size : 1;
    rank = tp ? tp->rank : 0;
    if (nrk > 1) {
        if (dim != 3) fail(SGML_EINVAL, "solve: multi-GPU solves are 3D");
        if (!compact()) fail(SGML_EINVAL, "solve: multi-GPU solves use the compact engine");
        if (nrk & (nrk - 1)) fail(SGML_EINVAL, "solve: the number of ranks must be a power of two");
        if (nrk > (1 << (n - 1))) fail(SGML_EINVAL, "solve: too many ranks for this grid (>= 2 planes each)");
        T0 = (1 << n) / nrk;  // level-0 planes per rank (the last rank also owns plane N-1)
        vrep = slab_vrep(n, nrk, opts.replicate_n);  // levels v < vrep are z-slabs
        // the transfer stream of the overlapped halo exchanges (created here,
        // not inside a graph capture)
        SGML_CUDA(cudaStreamCreateWithFlags(&hx_stream, cudaStreamNonBlocking));
        SGML_CUDA(cudaEventCreateWithFlags(&hx_ready, cudaEventDisableTiming));
        SGML_CUDA(cudaEventCreateWithFlags(&hx_done, cudaEventDisableTiming));
    }

    if (compact()) {
        Lv.resize(n);
        for (int v = 0; v < n; ++v) {
            if (dist(v)) {
                int kb, cnt;
                own_planes(v, rank, kb, cnt);
                Lv[v] = make_ext(dim, Nl[v], kb, cnt);
            } else {
                Lv[v] = make_ext(dim, Nl[v]);
            }
        }
        // the small-level interpreter's levels: arrays of at most kClusterNodes
        // nodes (3D <= 17^3, 2D <= 65^2; measured: with larger levels the 16
        // SMs of one cluster run them slower than full-GPU kernels do).
        // SGML_KOP_NODES overrides the bound (A/B and the parity suite).
        // 2D levels of <= 129^2 nodes are interpreted too (C1 129^2: the whole
        // cycle but the residual in one batch per tooth, 3.99 -> 3.85 ms per
        // solve; 257^2: 3.89 -> 3.82 ms with its 129^2 level 1 interpreted).
        kop_ok.assign(n, 0);
        const char* kn = std::getenv("SGML_KOP_NODES");
        const double kop_max = kn ? std::atof(kn) : (double)kClusterNodes;
        for (int v = 0; v < n; ++v) {
            double nodes = 1.0;
            for (int d = 0; d < dim; ++d) nodes *= Nl[v];
            kop_ok[v] = nodes <= kop_max || (!kn && dim == 2 && nodes <= kClusterNodes2D) ? 1 : 0;
        }
        // nodes off the Dirichlet faces, per level (local z indices); face values
        rng.assign(n, NodeRange{});
        for (int v = 0; v < n; ++v)
            for (int ax = 0; ax < 3; ++ax) {
                const bool live = ax < dim;
                rng[v].lo[ax] = live && bc_host.kind[2 * ax] == 0 ? 1 : 0;
                rng[v].hi[ax] = !live ? 0 : (bc_host.kind[2 * ax + 1] == 0 ? Nl[v] - 2 : Nl[v] - 1);
                if (live && ax == 2 && dist(v)) {
                    const ExtLay& L = Lv[v];
                    rng[v].lo[2] = (bc_host.kind[4] == 0 && L.z0 == 0) ? 1 : 0;
                    rng[v].hi[2] = (bc_host.kind[5] == 0 && L.z0 + L.Nz == Nl[v]) ? L.Nz - 2 : L.Nz - 1;
                }
            }
        for (int f = 0; f < 2 * dim; ++f)
            if (bc_host.kind[f] == 0) {
                bval_zero = bval_zero && bc_host.value[f] == 0.0;
                bval_finite = bval_finite && std::isfinite(bc_host.value[f]);
                const double av = std::fabs(bc_host.value[f]);
                bval_tiny = bval_tiny || (av != 0.0 && av < 0x1p-969);
            }
        const uint64_t E0 = ext_size(dim, Lv[0]);
        // the interpolation kernels index level arrays with 32-bit offsets
        if (E0 >= (1ULL << 31)) fail(SGML_EINVAL, "solve: grid too large for the compact engine (n <= 10 in 3D)");
        r = alloc(E0);
        utot = alloc(E0);
        A = alloc(E0);
        B = alloc(E0);
        dense = alloc(T);
        if (nrk > 1 && vrep < n) BS = alloc(ext_size(dim, Lv[vrep]));
        P.assign(n, nullptr);
        for (int m = 1; m < n; ++m) P[m] = alloc(ext_size(dim, Lv[m]));
        U.assign(n, {nullptr, nullptr});
        DU.assign(n, {});
        for (int v = 1; v < n; ++v) {
            const uint64_t Ev = ext_size(dim, Lv[v]);
            U[v][0] = alloc(Ev);
            U[v][1] = alloc(Ev);
            const int cmax = relax_count(n, cfg.n_r, v);
            for (int k = 0; k + 1 < cmax; ++k) DU[v].push_back(alloc(Ev));
        }
        // tooth v1's increments in application order: levels v1..1, passes 1..c-1;
        // fslot = the pass that applies the increment (pass k + 2 of level v in
        // tooth v1, numbered like pass_level: teeth n-1..0, levels v1..0)
        std::vector<ChainEntry> entries;
        tooth_off.assign(n, 0);
        std::vector<int> tooth_slot(n, 0);
        for (int v1 = n - 1, sl = 0; v1 >= 0; --v1) {
            tooth_slot[v1] = sl;
            sl += (v1 + 1) * relax_count(n, cfg.n_r, v1);
        }
        for (int v1 = 0; v1 < n; ++v1) {
            tooth_off[v1] = (int)entries.size();
            const int cc = relax_count(n, cfg.n_r, v1);
            for (int v = v1; v >= 1; --v) {
                const int first_slot = tooth_slot[v1] + (v1 - v) * cc;
                for (int k = 0; k + 1 < cc; ++k)
                    entries.push_back(ChainEntry{DU[v][k], Lv[v], v, first_slot + k + 1});
            }
        }
        for (int v = 1; v < n; ++v)
            for (double* d : DU[v]) du_bufs.push_back(d);
        h_chain = entries;
        if (!entries.empty()) {
            SGML_CUDA(cudaMalloc((void**)&d_chain, entries.size() * sizeof(ChainEntry)));
            SGML_CUDA(cudaMemcpy(d_chain, entries.data(), entries.size() * sizeof(ChainEntry),
                                 cudaMemcpyHostToDevice));
        }
        if (has_sigma) {
            S.assign(n, nullptr);
            DT.assign(n, nullptr);
            for (int m = 0; m < n; ++m) {
                S[m] = alloc(ext_size(dim, Lv[m]));
                DT[m] = alloc(ext_size(dim, Lv[m]));
            }
        }
        // TMA descriptors: window arrays (relax inputs, sigma) and tile arrays
        // (sources, residual, u_tot)
        add_maps(A, Lv[0], true, false);
        add_maps(B, Lv[0], true, false);
        add_maps(r, Lv[0], false, true);
        add_maps(utot, Lv[0], false, true);
        for (int v = 1; v < n; ++v) {
            add_maps(U[v][0], Lv[v], true, false);
            add_maps(U[v][1], Lv[v], true, false);
            add_maps(P[v], Lv[v], false, true);
        }
        if (has_sigma)
            for (int v = 0; v < n; ++v) {
                add_maps(S[v], Lv[v], true, false);
                add_maps(DT[v], Lv[v], false, true);
            }
    } else {
        r = alloc(T);
        utot = alloc(T);
        ensure_literal();
        if (has_sigma) {
            Lsig.assign(n, nullptr);
            for (int v = 0; v < n; ++v) Lsig[v] = alloc(T);
        }
    }
    if (compact()) {
        // alloc() zeroes: every level buffer starts with zero faces
        fstate[r] = FS_ZERO;
        fstate[utot] = FS_ZERO;
        fstate[A] = FS_ZERO;
        fstate[B] = FS_ZERO;
        for (int v = 1; v < n; ++v) {
            fstate[U[v][0]] = FS_ZERO;
            fstate[U[v][1]] = FS_ZERO;
            for (double* d : DU[v]) fstate[d] = FS_ZERO;
        }
    }
    if (has_sigma) load_sigma(sigma_dev);
    SGML_CUDA(cudaGetLastError());
    SGML_CUDA(cudaStreamSynchronize(ctx->stream));
}

int sgml_solver::faces_of(const double* p) const {
    const auto it = fstate.find(p);
    return it == fstate.end() ? FS_OTHER : it->second;
}

void sgml_solver::set_faces(double* p, int level, int st) {
    if (all_neumann || faces_of(p) == st) return;
    if (st == FS_OTHER) fail(SGML_ELOGIC, "set_faces: no target content");
    // DU arrays: data nodes only (their ghost cells stay 0, the past-the-end
    // corner reads of the interpolation)
    const bool mirrors = std::find(du_bufs.begin(), du_bufs.end(), p) == du_bufs.end();
    if (kop_level(level)) {
        KOp op{};
        op.kind = KOP_FACES;
        op.level = level;
        op.fc = KOpFaces{p, Lv[level], st == FS_ZERO ? 1 : 0, mirrors ? 1 : 0};
        record(op);
    } else {
        launch(SGML_CLASS_OTHER, [&] {
            launch_dirichlet_faces(g.dim, p, Lv[level], bc, st == FS_ZERO, mirrors, ctx->stream);
        });
    }
    fstate[p] = st;
}

// ---------------------------------------------------------------------------
// z-slab decomposition helpers
// ---------------------------------------------------------------------------

// rank p's planes of level v: T0 >> v each, the last rank also the plane N-1
// (levels >= vrep hold one plane per rank in this sizing)
void sgml_solver::own_planes(int v, int p, int& kb, int& cnt) const {
    const int t = std::max(1, T0 >> v);
    kb = p * t;
    cnt = t + (p == nrk - 1 ? 1 : 0);
}

void sgml_solver::halo(double* a, int v) {
    if (!dist(v)) return;
    tp->halo(a, Lv[v].plane, Lv[v].Nz, d_flag, ctx->stream);
}

// relaxation passes of z-slab levels overlap their halo exchange with the
// interior planes (SGML_NO_HALO_OVERLAP=1: exchange after the whole pass)
bool sgml_solver::overlap_halos(int v) {
    static const bool off = std::getenv("SGML_NO_HALO_OVERLAP") != nullptr;
    return !off && dist(v) && hx_stream && rng[v].hi[2] - rng[v].lo[2] >= 2;
}

// a replicated level array whose planes were produced rank by rank (own
// planes, own_planes sizing) -> every rank holds all of them.  The z ghost
// planes are the even mirrors of planes 1 and N-2 (whichever rank wrote
// them), so every rank rebuilds them from its gathered copy.
void sgml_solver::gather_level(double* a, int v) {
    if (nrk == 1) return;
    const long long pl = Lv[v].plane;
    std::vector<long long> off(nrk), cnt(nrk);
    for (int p = 0; p < nrk; ++p) {
        int kb, c;
        own_planes(v, p, kb, c);
        off[p] = (kb + 1) * pl;
        cnt[p] = (long long)c * pl;
    }
    tp->allgather(a, off, cnt, ctx->stream);
    const int N = Nl[v];
    const size_t bytes = (size_t)pl * sizeof(double);
    SGML_CUDA(cudaMemcpyAsync(a, a + 2 * pl, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    SGML_CUDA(cudaMemcpyAsync(a + (N + 1) * pl, a + (N - 1) * pl, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
}

// base (level 0, z-slab) sampled on level vrep, replicated on every rank
void sgml_solver::refresh_bs(const double* base) {
    int kb, cnt;
    own_planes(vrep, rank, kb, cnt);
    launch(SGML_CLASS_OTHER, [&] { launch_sample_ext(base, Lv[0], BS, Lv[vrep], vrep, kb, kb + cnt, ctx->stream); });
    gather_level(BS, vrep);
    bs_valid = true;
}

// one restriction-pyramid step level m -> m+1 (also for sigma)
void sgml_solver::pyramid_step(const double* in, int m, double* out) {
    const int dim = g.dim;
    const cudaStream_t s = ctx->stream;
    if (dist(m + 1)) {
        launch(SGML_CLASS_PYRAMID, [&] { launch_pyramid_ext(dim, in, Lv[m], out, Lv[m + 1], s); });
        halo(out, m + 1);
    } else if (dist(m)) {
        // first replicated level: own planes from the slab, then all-gather
        int kb, cnt;
        own_planes(m + 1, rank, kb, cnt);
        launch(SGML_CLASS_PYRAMID, [&] { launch_pyramid_ext(dim, in, Lv[m], out, Lv[m + 1], s, kb, kb + cnt); });
        gather_level(out, m + 1);
    } else if (kop_level(m + 1)) {
        KOp op{};
        op.kind = KOP_PYRAMID;
        op.level = m + 1;
        op.py = KOpPyramid{in, out, Lv[m], Lv[m + 1]};
        record(op);
    } else {
        launch(SGML_CLASS_PYRAMID, [&] { launch_pyramid_ext(dim, in, Lv[m], out, Lv[m + 1], s); });
    }
}

// the recorded small-level operations as one cluster launch per batch
void sgml_solver::flush_kops() {
    if (kops.empty()) return;
    std::vector<KOp> ops;
    ops.swap(kops);
    if (!kop_batch) kop_batch = std::make_unique<KOpBatch>();  // (~29 KB: passed by value as kernel parameters)
    KOpBatch& b = *kop_batch;
    b.bc = bc;
    b.flag = d_flag;
    b.homogeneous = cyc_homog ? 1 : 0;
    b.sig = has_sigma ? 1 : 0;
    b.chains = d_chain && h_chain.size() <= (size_t)kMaxChain ? d_chain : nullptr;
    b.nchains = b.chains ? (int)h_chain.size() : 0;
    for (int v = 0; v < g.n && v < 14; ++v) b.rc[v] = relax_const(g.dim, v, g.h, a, cfg.safety, cyc_homog, opts.stencil);
    static const bool no_solo = std::getenv("SGML_NO_SOLO_OPS") != nullptr;
    for (KOp& op : ops) {
        double nodes = 1.0;
        for (int d = 0; d < g.dim; ++d) nodes *= Nl[op.level];
        op.solo = !no_solo && g.dim == 2 && nodes <= kSoloNodes ? 1 : 0;
    }
    for (size_t i0 = 0; i0 < ops.size(); i0 += kMaxKOps) {
        b.count = (int)std::min<size_t>(kMaxKOps, ops.size() - i0);
        std::copy(ops.begin() + (long)i0, ops.begin() + (long)i0 + b.count, b.op);
        launch(SGML_CLASS_RELAX_COARSE, [&] { launch_kop_batch(g.dim, b, ctx->stream); });
    }
}

// cycle.cpp:117-133: sigma restricted per level with even (all-Neumann)
// ghosts; every level must stay positive.  The compact engine keeps level v
// only on its subset nodes (pyramid); positivity is checked on
// the full level-0 field, every coarser value being a positive average.
void sgml_solver::load_sigma(const double* sigma_dense) {
    const int dim = g.dim, n = g.n;
    const uint64_t T = g.total;
    const cudaStream_t s = ctx->stream;
    SGML_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
    if (compact()) {
        launch(SGML_CLASS_OTHER, [&] { launch_check_positive(sigma_dense, T, d_flag, s); });
        launch(SGML_CLASS_OTHER, [&] { launch_scatter_ext(dim, sigma_dense, S[0], Lv[0], s); });
        halo(S[0], 0);
        for (int m = 1; m < n; ++m) pyramid_step(S[m - 1], m - 1, S[m]);
        // per-node pseudo-time steps of the sigma relaxation, per level
        for (int m = 0; m < n; ++m) {
            const RelaxConst rcm = relax_const(dim, m, g.h, a, cfg.safety, false, opts.stencil);
            launch(SGML_CLASS_OTHER, [&] { launch_dtau_ext(dim, S[m], Lv[m], DT[m], rcm, s); });
        }
    } else {
        sgml_bc even{};
        for (int f = 0; f < 6; ++f) even.kind[f] = 1;
        const BcDev ev = to_dev(even);
        for (int v = 0; v < n; ++v) {
            // restriction_into(sigma, v, even): v literal passes ending in Lsig[v]
            if (v == 0) {
                if (sigma_dense != Lsig[0])
                    SGML_CUDA(cudaMemcpyAsync(Lsig[0], sigma_dense, T * sizeof(double), cudaMemcpyDeviceToDevice, s));
            } else {
                const double* src = Lsig[0];
                double* dst = (v % 2 == 1) ? Lsig[v] : Lscr;
                for (int m = 0; m < v; ++m) {
                    launch(SGML_CLASS_LITERAL, [&] { launch_restrict_pass(dim, src, dst, g.N, 1 << m, ev, s); });
                    src = dst;
                    dst = (dst == Lsig[v]) ? Lscr : Lsig[v];
                }
            }
            launch(SGML_CLASS_OTHER, [&] { launch_check_positive(Lsig[v], T, d_flag, s); });
        }
    }
    SGML_CUDA(cudaMemcpyAsync(h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    SGML_CUDA(cudaStreamSynchronize(s));
    SGML_CUDA(cudaGetLastError());
    if (h_flag[0]) fail(SGML_EINVAL, "restrict_sigma_levels: coefficient must stay positive");
}

void sgml_solver::ensure_literal() {
    if (Lg) return;
    const uint64_t T = g.total;
    Lg = alloc(T); Lscr = alloc(T); Lu = alloc(T); Lup = alloc(T); Ldu = alloc(T); Ldup = alloc(T);
}

// ---------------------------------------------------------------------------
// layout-dependent helpers
// ---------------------------------------------------------------------------

void sgml_solver::load_source(const double* f) {
    const cudaStream_t s = ctx->stream;
    if (compact()) {
        launch(SGML_CLASS_OTHER, [&] { launch_scatter_ext(g.dim, f, r, Lv[0], s); });
        halo(r, 0);
        fstate[r] = FS_OTHER;
    }
    else
        SGML_CUDA(cudaMemcpyAsync(r, f, g.total * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

const double* sgml_solver::dense_view(const double* field) {
    if (!compact()) return field;
    launch(SGML_CLASS_OTHER, [&] { launch_gather_ext(g.dim, field, Lv[0], dense, ctx->stream); });
    if (dist(0)) {  // every rank's planes of the dense field
        const long long pl = (long long)g.N * g.N;
        std::vector<long long> off(nrk), cnt(nrk);
        for (int p = 0; p < nrk; ++p) {
            int kb, c;
            own_planes(0, p, kb, c);
            off[p] = kb * pl;
            cnt[p] = c * pl;
        }
        tp->allgather(dense, off, cnt, ctx->stream);
    }
    return dense;
}

// kernels.cpp:388-395 on r (serial Kahan mean on the host, then subtract;
// the subtraction also covers r's mirror ghosts, which stay consistent)
void sgml_solver::zero_mean_r() {
    const double mean = trapezoid_mean_host(ctx, g, dense_view(r));
    const uint64_t count = compact() ? ext_size(g.dim, Lv[0]) : g.total;
    launch(SGML_CLASS_OTHER, [&] { launch_sub_scalar(r, count, mean, ctx->stream); });
}

double sgml_solver::max_abs_r(const double* f_dense) {
    const cudaStream_t s = ctx->stream;
    unsigned long long* d_rmax = d_cycle + n_slots;
    const double* src = all_neumann ? dense_view(r) : (compact() ? f_dense : r);
    SGML_CUDA(cudaMemsetAsync(d_rmax, 0, sizeof(unsigned long long), s));
    launch(SGML_CLASS_OTHER, [&] { launch_max_abs(src, g.total, d_rmax, s); });
    SGML_CUDA(cudaMemcpyAsync(h_cycle + n_slots, d_rmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SGML_CUDA(cudaStreamSynchronize(s));
    double norm;
    std::memcpy(&norm, &h_cycle[n_slots], sizeof(double));
    return norm;
}

// u_tot += e; r -= A(e) + a e; r = 0 on Dirichlet; max|r| into d_cycle[n_slots]
// The recurrence can run before the host has seen the cycle's kernel-error
// flag (one host synchronisation per cycle instead of two) when it changes
// nothing but r, u_tot and the max|r| slot — the faces it would set are in
// place (every homogeneous cycle of a problem with Dirichlet faces) — and the
// kernel itself skips the update on a failed cycle (guarded).
bool sgml_solver::residual_guardable(const double* e) const {
    static const bool off = std::getenv("SGML_NO_GUARDED_RESIDUAL") != nullptr;
    return !off && compact() && !all_neumann && faces_of(r) == FS_ZERO && faces_of(e) == FS_ZERO;
}

void sgml_solver::residual(const double* e, bool guarded) {
    const int dim = g.dim;
    const cudaStream_t s = ctx->stream;
    unsigned long long* d_rmax = d_cycle + n_slots;
    const RelaxConst rc0 = relax_const(dim, 0, g.h, a, cfg.safety, false, opts.stencil);
    if (compact()) {
        // faces: r = 0 on Dirichlet nodes (kernels.cpp:351-358), u_tot += e
        // there (e holds 0 or the face value)
        set_faces(r, 0, FS_ZERO);
        const int es = faces_of(e);
        if (es == FS_BVAL) {
            if (faces_of(utot) != FS_ZERO) fail(SGML_ELOGIC, "residual: u_tot faces out of step");
            set_faces(utot, 0, FS_BVAL);
        } else if (es != FS_ZERO) {
            fail(SGML_ELOGIC, "residual: e faces unknown");
        }
        TmaSet tm;
        tm.u = umap(e);
        tm.g = gmap(r);
        tm.s = has_sigma ? umap(S[0]) : tm.u;
        tm.t = gmap(utot);
        launch(SGML_CLASS_RESIDUAL, [&] {
            launch_residual_tma(dim, has_sigma, tm, r, utot, Lv[0], rng[0], rc0, d_rmax, d_flag, guarded, s);
        });
        halo(r, 0);  // the next cycle's pyramid reads r across the slab faces
    } else {
        const double inv_h2 = 1.0 / (g.h * g.h);
        const double pref = relax_const(dim, 0, g.h, a, cfg.safety, true, opts.stencil).pref;
        launch(SGML_CLASS_RESIDUAL, [&] {
            launch_residual(dim, has_sigma, r, e, utot, has_sigma ? Lsig[0] : nullptr, g.N, inv_h2, pref, a, bc,
                            d_rmax, s, opts.stencil);
        });
    }
}

// ---------------------------------------------------------------------------
// one cycle
// ---------------------------------------------------------------------------

const double* sgml_solver::cycle(bool homogeneous) {
    return compact() ? cycle_compact(homogeneous) : cycle_literal(homogeneous);
}

void sgml_solver::cycle_dense(const double* src_dense, double* out_dense, bool homogeneous) {
    if (nrk > 1) fail(SGML_EINVAL, "single_cycle: single-GPU only");
    load_source(src_dense);
    const double* e = cycle(homogeneous);
    if (compact()) {
        launch(SGML_CLASS_OTHER, [&] { launch_gather_ext(g.dim, e, Lv[0], out_dense, ctx->stream); });
    } else {
        SGML_CUDA(cudaMemcpyAsync(out_dense, e, g.total * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    }
}

// A level visit qualifies for the one-CTA path when the level array is small,
// single-GPU (or replicated), and no pass needs its Dirichlet faces rewritten
// (set_faces would be a no-op for every output and du buffer).
bool sgml_solver::small_visit(int v, const double* in, int c, const double* p0, const double* p1,
                              bool homogeneous) const {
    if (opts.small_levels < 0 || dist(v) || c > kSmallMaxPasses || !compact()) return false;
    long long nodes = 1;
    for (int ax = 0; ax < g.dim; ++ax) nodes *= (long long)(rng[v].hi[ax] - rng[v].lo[ax] + 1);
    if (nodes <= 0 || nodes > kSmallNodes) return false;
    if (ext_size(g.dim, Lv[v]) > (uint64_t)kSmallMaxExt) return false;  // (staged whole in shared memory)
    if (all_neumann) return true;
    const int want = face_want(homogeneous);
    const double* cur = in;
    for (int p = 1; p <= c; ++p) {
        const double* out = cur == p0 ? p1 : p0;
        const int ins = faces_of(cur);
        if (faces_of(out) != want) return false;
        if (v > 0 && p < c) {
            const int need = ins == want ? FS_ZERO : (ins == FS_ZERO && want == FS_BVAL ? FS_BVAL : -1);
            if (need < 0 || faces_of(DU[v][p - 1]) != need) return false;
        }
        cur = out;
    }
    return true;
}

// Single-GPU solves replay each cycle from a CUDA graph; z-slab solves too
// when the transport's exchanges are stream-ordered (NCCL: the halo
// send/recv and the plane broadcasts become graph nodes between the kernels).
bool sgml_solver::use_graphs() const {
    static const int off = std::getenv("SGML_NO_GRAPHS") ? 1 : 0;
    const bool clique_ok = nrk == 1 || (tp && tp->graph_capturable() && !slab_graphs_off);
    return compact() && clique_ok && !off && opts.use_graph >= 0 && debug_sync <= 0 && !diag_mode;
}

const double* sgml_solver::cycle_graph(bool homogeneous) {
    CycleGraph& G = graphs[homogeneous ? 1 : 0];
    const cudaStream_t s = ctx->stream;
    if (G.exec && fstate == G.pre) {
        SGML_CUDA(cudaGraphLaunch(G.exec, s));
        fstate = G.post;
        launches += G.nlaunch;
        spans.insert(spans.end(), G.spans.begin(), G.spans.end());
        return G.out;
    }
    if (G.exec) {
        SGML_CUDA(cudaGraphExecDestroy(G.exec));
        G.exec = nullptr;
        for (cudaEvent_t e : G.events) cudaEventDestroy(e);
        G.events.clear();
    }
    G.pre = fstate;
    const uint64_t l0 = launches;
    const size_t s0 = spans.size();
    cudaGraph_t graph = nullptr;
    SGML_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    capturing = &G;
    const double* e = nullptr;
    try {
        e = cycle_compact(homogeneous);
    } catch (...) {
        capturing = nullptr;
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    capturing = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (ce == cudaSuccess) {
        ce = cudaGraphInstantiate(&G.exec, graph, 0);
        cudaGraphDestroy(graph);
    }
    if (nrk > 1) {
        // a z-slab clique captures together: every rank must replay (or none),
        // or the ranks' exchanges would not pair up
        h_flag[6] = ce != cudaSuccess ? 1 : 0;
        (void)cudaGetLastError();
        SGML_CUDA(cudaMemcpyAsync(d_flag + 6, h_flag + 6, sizeof(int), cudaMemcpyHostToDevice, s));
        tp->allreduce_max_i32(d_flag + 6, 1, s);
        SGML_CUDA(cudaMemcpyAsync(h_flag + 6, d_flag + 6, sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        if (h_flag[6]) {
            if (G.exec) cudaGraphExecDestroy(G.exec);
            G.exec = nullptr;
            slab_graphs_off = true;  // this solver runs its cycles eagerly from now on
            fstate = G.pre;
            spans.resize(s0);
            launches = l0;
            return cycle_compact(homogeneous);
        }
    }
    SGML_CUDA(ce);
    G.post = fstate;
    G.out = e;
    G.nlaunch = launches - l0;
    G.spans.assign(spans.begin() + (long)s0, spans.end());
    SGML_CUDA(cudaGraphLaunch(G.exec, s));
    return e;
}

const double* sgml_solver::cycle_compact(bool homogeneous) {
    const int dim = g.dim, n = g.n;
    const cudaStream_t s = ctx->stream;
    const uint64_t E0 = ext_size(dim, Lv[0]);
    unsigned long long* diag = d_cycle;
    int* flag = d_flag;
    // operations on small level arrays are recorded and run as cluster batches
    // (interp.cu; single GPU, outside failure re-runs)
    static const bool no_kops = std::getenv("SGML_NO_CLUSTER_LEVELS") != nullptr;
    flush_kops();
    kops_cycle = !no_kops && opts.cluster_levels >= 0 && nrk == 1 && !diag_mode;
    cyc_homog = homogeneous;

    // a non-finite Dirichlet value makes the first pass throw
    // (kernels.cpp:228, 343-346); the kernels never write face nodes
    if (!homogeneous && !bval_finite) SGML_CUDA(cudaMemsetAsync(flag, 1, 1, s));
    // flag[1]: some level array of this cycle holds a nonzero value below
    // 2^-969 (relax passes then keep the unfused edge terms); every level
    // array of a cycle is produced within it, Dirichlet values included
    // flag[2], flag[3]: the neighbours' flag[1] (multi-GPU, sent with the halos)
    SGML_CUDA(cudaMemsetAsync(flag + 1, 0, 3 * sizeof(int), s));
    if (!homogeneous && bval_tiny) SGML_CUDA(cudaMemsetAsync(flag + 1, 1, 1, s));
    // restriction pyramid of the cycle's source (once per cycle, F4)
    for (int m = 0; m + 1 < n; ++m) pyramid_step(m == 0 ? r : P[m], m, P[m + 1]);
    auto gsrc = [&](int v) { return v == 0 ? (const double*)r : (const double*)P[v]; };

    int slot = 0;
    bool first = true;          // no pass has run in this cycle yet
    double* base = A;           // full-grid state after the last level-0 visit
    double* other = B;
    bool base_zero = true;      // state.u entered the cycle zeroed

    // a materialisation into a z-slab level array and its halo exchange: the
    // two own boundary planes first, their exchange overlapping the rest
    auto mat_halo = [&](double* dst, int w, auto&& mat) {
        if (dim == 3 && overlap_halos(w) && Lv[w].Nz >= 3) {
            const int nz = Lv[w].Nz;
            mat(0, 1);
            mat(nz - 1, nz);
            SGML_CUDA(cudaEventRecord(hx_ready, s));
            SGML_CUDA(cudaStreamWaitEvent(hx_stream, hx_ready, 0));
            tp->halo(dst, Lv[w].plane, nz, d_flag, hx_stream);
            SGML_CUDA(cudaEventRecord(hx_done, hx_stream));
            mat(1, nz - 1);
            SGML_CUDA(cudaStreamWaitEvent(s, hx_done, 0));
        } else {
            mat(0, -1);
            halo(dst, w);
        }
    };
    // a materialisation into level w: recorded for small levels, else launched
    // (z-slab levels with their halo exchange)
    auto materialize = [&](double* dst, int w, const double* bp, const ExtLay& bl, int wb, const double* uf,
                           const ExtLay& Lf, int frel, const ChainEntry* ch, int count) {
        if (kop_level(w)) {
            KOp op{};
            op.kind = KOP_MATERIALIZE;
            op.level = w;
            KOpMaterialize& m = op.mt;
            m.out = dst;
            m.base = bp;
            m.ufine = uf;
            m.chain = ch;
            m.Lw = Lv[w];
            m.L0 = bl;
            m.Lf = Lf;
            m.w = w;
            m.wb = wb;
            m.base_zero = base_zero ? 1 : 0;
            m.frel = frel;
            m.nchain = count;
            materialize_grid(dim, Lv[w], bc, m.gx, m.gy, m.gz, m.xtail);
            record(op);
            return;
        }
        mat_halo(dst, w, [&](int kb, int ke) {
            launch(SGML_CLASS_MATERIALIZE, [&] {
                launch_materialize4(dim, dst, Lv[w], w, bp, bl, wb, base_zero, uf, Lf, frel, ch, count, bc,
                                    homogeneous, flag, diag_mode, s, kb, ke);
            });
        });
    };
    auto relax_level = [&](int v, double* in, int c, double* p0, double* p1) -> double* {
        const RelaxConst rc = relax_const(dim, v, g.h, a, cfg.safety, homogeneous, opts.stencil);
        double* cur = in;
        if (kop_level(v)) {  // recorded passes (small-level interpreter)
            for (int p = 1; p <= c; ++p) {
                double* out = cur == p0 ? p1 : p0;
                double* duo = (v > 0 && p < c) ? DU[v][p - 1] : nullptr;
                const int want = face_want(homogeneous), ins = faces_of(cur);
                set_faces(out, v, want);
                if (duo) {
                    if (ins == want) set_faces(duo, v, FS_ZERO);
                    else if (ins == FS_ZERO && want == FS_BVAL) set_faces(duo, v, FS_BVAL);
                    else fail(SGML_ELOGIC, "relax: input faces out of step");
                }
                KOp op{};
                op.kind = KOP_RELAX;
                op.level = v;
                KOpRelax& x = op.rx;
                x.in = cur;
                x.out = out;
                x.du = duo;
                x.g = gsrc(v);
                x.sig = has_sigma ? S[v] : nullptr;
                x.dt = has_sigma ? DT[v] : nullptr;
                x.slot = diag + slot;
                x.L = Lv[v];
                for (int d = 0; d < 3; ++d) {
                    x.lo[d] = rng[v].lo[d];
                    x.hi[d] = rng[v].hi[d];
                }
                x.pass_slot = slot;
                record(op);
                ++slot;
                cur = out;
                first = false;
            }
            return cur;
        }
        // small level array, faces already what every pass needs: all c
        // passes in one CTA (one launch instead of c)
        if (small_visit(v, in, c, p0, p1, homogeneous)) {
            SmallPasses sp{};
            sp.count = c;
            sp.g = gsrc(v);
            sp.sig = has_sigma ? S[v] : nullptr;
            sp.dt = has_sigma ? DT[v] : nullptr;
            for (int p = 1; p <= c; ++p) {
                double* out = cur == p0 ? p1 : p0;
                sp.in[p - 1] = cur;
                sp.out[p - 1] = out;
                sp.du[p - 1] = (v > 0 && p < c) ? DU[v][p - 1] : nullptr;
                sp.slot[p - 1] = diag + slot + (p - 1);
                sp.pass_slot[p - 1] = slot + (p - 1);
                cur = out;
            }
            launch(v == 0 ? SGML_CLASS_RELAX0 : SGML_CLASS_RELAX_COARSE, [&] {
                launch_relax_small(dim, has_sigma, sp, Lv[v], rng[v], rc, flag, s);
            });
            slot += c;
            first = false;
            return cur;
        }
        for (int p = 1; p <= c; ++p) {
            double* out = cur == p0 ? p1 : p0;
            double* duo = (v > 0 && p < c) ? DU[v][p - 1] : nullptr;
            // Dirichlet faces: out holds the face value of this cycle, du =
            // face value - input face value (0, or the value on a zeroed input)
            const int want = face_want(homogeneous), ins = faces_of(cur);
            set_faces(out, v, want);
            if (duo) {
                if (ins == want) set_faces(duo, v, FS_ZERO);
                else if (ins == FS_ZERO && want == FS_BVAL) set_faces(duo, v, FS_BVAL);
                else fail(SGML_ELOGIC, "relax: input faces out of step");
            }
            TmaSet tm;
            tm.u = umap(cur);
            tm.g = gmap(gsrc(v));
            tm.s = has_sigma ? umap(S[v]) : tm.u;
            tm.t = has_sigma ? gmap(DT[v]) : tm.g;
            auto relax_range = [&](const NodeRange& rg) {
                launch(v == 0 ? SGML_CLASS_RELAX0 : SGML_CLASS_RELAX_COARSE, [&] {
                    launch_relax_tma(dim, has_sigma, tm, out, duo, Lv[v], rg, rc, diag + slot, flag, slot, s);
                });
            };
            if (overlap_halos(v)) {
                // z-slab level: the two planes the neighbours need first, their
                // halo exchange on the transfer stream while the interior planes
                // are relaxed (all three launches share the pass's diag slot)
                NodeRange b0 = rng[v], b1 = rng[v], mid = rng[v];
                b0.hi[2] = b0.lo[2];
                b1.lo[2] = b1.hi[2];
                mid.lo[2] += 1;
                mid.hi[2] -= 1;
                relax_range(b0);
                relax_range(b1);
                SGML_CUDA(cudaEventRecord(hx_ready, s));
                SGML_CUDA(cudaStreamWaitEvent(hx_stream, hx_ready, 0));
                tp->halo(out, Lv[v].plane, Lv[v].Nz, d_flag, hx_stream);
                if (duo) tp->halo(duo, Lv[v].plane, Lv[v].Nz, d_flag, hx_stream);
                SGML_CUDA(cudaEventRecord(hx_done, hx_stream));
                relax_range(mid);
                SGML_CUDA(cudaStreamWaitEvent(s, hx_done, 0));
            } else {
                relax_range(rng[v]);
                halo(out, v);  // z-slab levels: the next consumer reads across the slab faces
                if (duo) halo(duo, v);
            }
            ++slot;
            cur = out;
            first = false;
        }
        return cur;
    };
    // replicated targets read the base from its replicated level-vrep sample
    bs_valid = false;
    auto base_src = [&](int w, const double*& bp, ExtLay& bl, int& wb) {
        bp = base;
        bl = Lv[0];
        wb = 0;
        if (nrk > 1 && !dist(w) && !base_zero) {
            if (!bs_valid) refresh_bs(base);
            bp = BS;
            bl = Lv[vrep];
            wb = vrep;
        }
    };

    for (int v1 = n - 1; v1 >= 0; --v1) {
        const int c = relax_count(n, cfg.n_r, v1);
        // pending increments of this tooth: d_chain[tooth_off[v1] + start, + count)
        int start = 0, count = 0;
        auto chain_at = [&]() { return d_chain ? d_chain + tooth_off[v1] + start : nullptr; };
        const double* ufinal = nullptr;  // last pass output of level v+1
        for (int v = v1; v >= 1; --v) {
            double* in = U[v][0];
            if (first) {
                if (kop_level(v)) {
                    KOp op{};
                    op.kind = KOP_MEMSET;
                    op.level = v;
                    op.ms = KOpMemset{in, (long long)ext_size(dim, Lv[v])};
                    record(op);
                } else {
                    flush_kops();
                    SGML_CUDA(cudaMemsetAsync(in, 0, ext_size(dim, Lv[v]) * sizeof(double), s));
                }
                fstate[in] = FS_ZERO;
            } else {
                if (count > 0 && count + (c - 1) > kMaxChain) {
                    // fold the pending increments into a full-grid base
                    const ChainEntry* ch = chain_at();
                    materialize(other, 0, base, Lv[0], 0, ufinal, Lv[v + 1], v + 1, ch, count);
                    fstate[other] = face_want(homogeneous);
                    bs_valid = false;
                    std::swap(base, other);
                    base_zero = false;
                    start += count;
                    count = 0;
                    ufinal = nullptr;  // already folded into base
                }
                const ChainEntry* ch = chain_at();
                const ExtLay Lf = v + 1 < n ? Lv[v + 1] : Lv[v];
                const double* bp;
                ExtLay bl;
                int wb;
                base_src(v, bp, bl, wb);
                materialize(in, v, bp, bl, wb, ufinal, Lf, 1, ch, count);
                fstate[in] = face_want(homogeneous);
            }
            ufinal = relax_level(v, in, c, U[v][0], U[v][1]);
            count += c - 1;
        }
        // level 0 visit of this tooth
        double* in0;
        if (first) {
            if (kop_level(0)) {
                KOp op{};
                op.kind = KOP_MEMSET;
                op.level = 0;
                op.ms = KOpMemset{base, (long long)E0};
                record(op);
            } else {
                flush_kops();
                SGML_CUDA(cudaMemsetAsync(base, 0, E0 * sizeof(double), s));
            }
            fstate[base] = FS_ZERO;
            in0 = base;
        } else if (v1 >= 1) {
            const ChainEntry* ch = chain_at();
            const ExtLay Lf = n > 1 ? Lv[1] : Lv[0];
            materialize(other, 0, base, Lv[0], 0, ufinal, Lf, 1, ch, count);
            fstate[other] = face_want(homogeneous);
            in0 = other;
        } else {
            in0 = base;
        }
        base = relax_level(0, in0, c, A, B);
        other = base == A ? B : A;
        base_zero = false;
        bs_valid = false;
    }
    // tail Relax(0, min(n_r, 2^n))
    base = relax_level(0, base, relax_count(n, cfg.n_r, 0), A, B);
    flush_kops();
    kops_cycle = false;
    return base;
}

const double* sgml_solver::cycle_literal(bool homogeneous) {
    const int dim = g.dim, n = g.n, N = g.N;
    const cudaStream_t s = ctx->stream;
    const uint64_t T = g.total;
    const double* source = r;
    // state.u / u_prev zeroed by solve (cycle.cpp:179-180); du reset at the
    // first relax step
    SGML_CUDA(cudaMemsetAsync(Lu, 0, T * sizeof(double), s));
    SGML_CUDA(cudaMemsetAsync(Lup, 0, T * sizeof(double), s));
    double *u = Lu, *up = Lup, *du = Ldu, *dup = Ldup;
    int slot = 0, current = -1;
    for (int v1 = n - 1; v1 >= -1; --v1) {
        const bool tail = v1 < 0;
        const int c = tail ? relax_count(n, cfg.n_r, 0) : relax_count(n, cfg.n_r, v1);
        for (int v = tail ? 0 : v1; v >= 0; --v) {
            if (!tail) {
                // restriction_into(source, v, bc, g, scratch) (kernels.cpp:305-325)
                if (v == 0) {
                    SGML_CUDA(cudaMemcpyAsync(Lg, source, T * sizeof(double), cudaMemcpyDeviceToDevice, s));
                } else {
                    const double* src = source;
                    double* dst = (v % 2 == 1) ? Lg : Lscr;
                    for (int m = 0; m < v; ++m) {
                        launch(SGML_CLASS_LITERAL, [&] { launch_restrict_pass(dim, src, dst, N, 1 << m, bc, s); });
                        src = dst;
                        dst = (dst == Lg) ? Lscr : Lg;
                    }
                }
            }
            if (v != current) {  // SolveState::reset_level
                SGML_CUDA(cudaMemsetAsync(du, 0, T * sizeof(double), s));
                SGML_CUDA(cudaMemsetAsync(dup, 0, T * sizeof(double), s));
                current = v;
            }
            const RelaxConst rc = relax_const(dim, v, g.h, a, cfg.safety, homogeneous, opts.stencil);
            for (int p = 0; p < c; ++p) {
                std::swap(u, up);
                std::swap(du, dup);
                launch(SGML_CLASS_LITERAL, [&] {
                    launch_relax_literal(dim, has_sigma, u, du, up, dup, Lg, has_sigma ? Lsig[v] : nullptr,
                                         N, v, rc, bc, d_cycle + slot, d_flag, slot, s);
                });
                ++slot;
            }
            if (tail) break;
        }
    }
    Lu = u; Lup = up; Ldu = du; Ldup = dup;
    return Lu;
}

// cycle.cpp:244-245 (pure_neumann_pin) and the dense result
void sgml_solver::pin_and_emit(double* u_out) {
    const cudaStream_t s = ctx->stream;
    const uint64_t T = g.total;
    double* res = compact() ? dense : utot;
    if (compact()) dense_view(utot);  // (every rank's planes in a multi-GPU solve)
    if (all_neumann && a == 0.0) {
        const double mean = trapezoid_mean_host(ctx, g, res);
        launch(SGML_CLASS_OTHER, [&] { launch_sub_scalar(res, T, mean, s); });
    }
    if (u_out && u_out != res)
        SGML_CUDA(cudaMemcpyAsync(u_out, res, T * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

// flag[0] (some pass failed) and flag[4] (the first failing pass, atomicMin)
void sgml_solver::reset_fail_flags() {
    SGML_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), ctx->stream));
    SGML_CUDA(cudaMemsetAsync(d_flag + 4, 0x7f, sizeof(int), ctx->stream));
}

// After a failed cycle: the first pass of the cycle the reference would throw
// at (kernels.cpp:343-346), with the cycle's per-pass diag maxima in h_cycle.
// The literal engine checks every node in every pass.  The compact engine's
// relaxation kernels report their own pass, but the interpolated nodes exist
// only as lazy chains: the cycle is re-run (same inputs: r is untouched until
// the recurrence) with the materialisations checking every partial sum of
// their chains, each chain entry carrying the pass that applies it.
int sgml_solver::first_failing_pass(bool homogeneous) {
    const cudaStream_t s = ctx->stream;
    if (compact()) {
        SGML_CUDA(cudaMemsetAsync(d_cycle, 0, (n_slots + 1) * sizeof(unsigned long long), s));
        reset_fail_flags();
        diag_mode = true;
        try {
            cycle(homogeneous);
        } catch (...) {
            diag_mode = false;
            throw;
        }
        diag_mode = false;
    }
    SGML_CUDA(cudaMemcpyAsync(h_flag, d_flag, 8 * sizeof(int), cudaMemcpyDeviceToHost, s));
    SGML_CUDA(cudaStreamSynchronize(s));
    int first = h_flag[4];  // 0x7f7f7f7f: flagged outside any pass (the first pass)
    if (first == 0x7f7f7f7f) first = 0;
    if (nrk > 1) {
        // min over the ranks as a max of the complement
        h_flag[5] = 0x7f7f7f7f - first;
        SGML_CUDA(cudaMemcpyAsync(d_flag + 5, h_flag + 5, sizeof(int), cudaMemcpyHostToDevice, s));
        tp->allreduce_max_i32(d_flag + 5, 1, s);
        tp->allreduce_max_u64(d_cycle, n_slots + 1, s);
        SGML_CUDA(cudaMemcpyAsync(h_flag + 5, d_flag + 5, sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    SGML_CUDA(cudaMemcpyAsync(h_cycle, d_cycle, (n_slots + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              s));
    SGML_CUDA(cudaStreamSynchronize(s));
    if (nrk > 1) first = 0x7f7f7f7f - h_flag[5];
    return first;
}

// ---------------------------------------------------------------------------
// solve (cycle.cpp:140-247)
// ---------------------------------------------------------------------------

void sgml_solver::run(const double* f, double* u_out, sgml_report* rep) {
    SGML_CUDA(cudaSetDevice(ctx->device));
    const cudaStream_t s = ctx->stream;
    const uint64_t T = g.total;
    launches = 0;
    for (int k = 0; k < 8; ++k) { cls_ms[k] = 0.0; cls_n[k] = 0; }
    spans.clear();
    evused = 0;
    if (!tev0) {
        SGML_CUDA(cudaEventCreate(&tev0));
        SGML_CUDA(cudaEventCreate(&tev1));
    }
    SGML_CUDA(cudaEventRecord(tev0, s));

    // input validation (cycle.cpp:150-152)
    SGML_CUDA(cudaMemsetAsync(d_flag, 0, 8 * sizeof(int), s));
    launch(SGML_CLASS_OTHER, [&] { launch_check_finite(f, T, d_flag, s); });
    SGML_CUDA(cudaMemcpyAsync(h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    SGML_CUDA(cudaStreamSynchronize(s));
    if (h_flag[0]) fail(SGML_EINVAL, "solve: source contains non-finite values");

    rep->n_rows = 0;
    rep->n_trace = 0;
    rep->converged = rep->nan_detected = rep->stagnated = 0;
    rep->normalization = 0.0;
    rep->node_updates = 0;

    load_source(f);
    SGML_CUDA(cudaMemsetAsync(utot, 0, (compact() ? ext_size(g.dim, Lv[0]) : T) * sizeof(double), s));
    if (compact()) fstate[utot] = FS_ZERO;  // (a reused engine's u_tot held last solve's faces)
    if (all_neumann) zero_mean_r();
    double norm = max_abs_r(f);  // D = max|f|; 0 falls back to the cycle-0 residual
    bool norm_pending = norm == 0.0;

    uint64_t work = 0;
    double prev_res = std::numeric_limits<double>::infinity();
    int non_decreasing = 0;
    const bool badstep = !(cfg.safety > 0.0);

    for (int cyc = 0; cyc < cfg.max_cycles; ++cyc) {
        const bool homogeneous = cyc > 0;
        if (all_neumann && cyc > 0) zero_mean_r();
        if (badstep) {  // kernels.cpp:197,343: the first pass throws
            rep->nan_detected = 1;
            rep->converged = 0;
            break;
        }
        SGML_CUDA(cudaMemsetAsync(d_cycle, 0, (n_slots + 1) * sizeof(unsigned long long), s));
        reset_fail_flags();
        const double* e = use_graphs() ? cycle_graph(homogeneous) : cycle(homogeneous);
        // kernel_error check before the recurrence touches u_tot and r (or,
        // guarded, the recurrence skips itself on a failed cycle)
        if (nrk > 1) tp->allreduce_max_i32(d_flag, 1, s);
        static const bool dbg_flags = std::getenv("SGML_DEBUG_FLAGS") != nullptr;
        // the reference throws at the first failing pass: the trace keeps the
        // samples of the passes before it, the cycle gets no row
        // (cycle.cpp:98-107, 182-190)
        auto failed = [&] {
            if (dbg_flags) std::fprintf(stderr, "sgml: cycle %d flags %d %d %d %d\n", cyc, h_flag[0], h_flag[1], h_flag[2], h_flag[3]);
            if (!h_flag[0]) return false;
            const int fail_slot = first_failing_pass(homogeneous);
            const double inv_norm = !norm_pending && norm > 0.0 ? 1.0 / norm : 1.0;
            for (int p = 0; p < fail_slot && p < n_slots; ++p) {
                double d;
                std::memcpy(&d, &h_cycle[p], sizeof(double));
                if (rep->n_trace < rep->trace_cap)
                    rep->trace[rep->n_trace] = sgml_diag_sample{cyc, pass_index[p], pass_level[p], 0, d * inv_norm};
                rep->n_trace++;
            }
            rep->nan_detected = 1;
            rep->converged = 0;
            return true;
        };
        const bool guarded = residual_guardable(e);
        if (!guarded) {
            SGML_CUDA(cudaMemcpyAsync(h_flag, d_flag, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
            SGML_CUDA(cudaStreamSynchronize(s));
            if (failed()) break;
        }
        residual(e, guarded);
        SGML_CUDA(cudaGetLastError());
        // per-pass diag maxima and max|r| over the ranks (max is order-free:
        // bit-identical to the single-GPU values)
        if (nrk > 1) tp->allreduce_max_u64(d_cycle, n_slots + 1, s);
        if (guarded) SGML_CUDA(cudaMemcpyAsync(h_flag, d_flag, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaMemcpyAsync(h_cycle, d_cycle, (n_slots + 1) * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        if (guarded && failed()) break;
        if (opts.timing) harvest_spans();

        const double inv_norm = !norm_pending && norm > 0.0 ? 1.0 / norm : 1.0;
        const int64_t trace_mark = rep->n_trace;
        for (int p = 0; p < n_slots; ++p) {
            double d;
            std::memcpy(&d, &h_cycle[p], sizeof(double));
            if (rep->n_trace < rep->trace_cap)
                rep->trace[rep->n_trace] = sgml_diag_sample{cyc, pass_index[p], pass_level[p], 0, d * inv_norm};
            rep->n_trace++;
        }
        work += units_per_cycle;
        rep->node_updates += units_per_cycle * T;

        double r_max;
        std::memcpy(&r_max, &h_cycle[n_slots], sizeof(double));
        if (norm_pending) {
            norm = r_max;
            norm_pending = false;
            if (norm == 0.0) {
                if (rep->n_rows < rep->rows_cap)
                    rep->rows[rep->n_rows] = sgml_cycle_record{cyc, 0, work, 0.0, 0.0, 0.0};
                rep->n_rows++;
                rep->converged = 1;
                break;
            }
            for (int64_t t = trace_mark; t < rep->n_trace && t < rep->trace_cap; ++t)
                rep->trace[t].value /= norm;
        }
        const double res = r_max / norm;
        double diag_min = std::numeric_limits<double>::infinity();
        for (int64_t t = trace_mark; t < rep->n_trace && t < rep->trace_cap; ++t)
            diag_min = std::min(diag_min, rep->trace[t].value);
        sgml_cycle_record row{cyc, 0, work, res, diag_min, 0.0};
        if (rep->hook) {
            sgml_field view;
            view.ctx = ctx;
            view.grid = g;
            view.d = const_cast<double*>(dense_view(utot));
            SGML_CUDA(cudaStreamSynchronize(s));
            double l1 = 0.0;
            if (rep->hook(rep->hook_user, cyc, &view, &l1)) {
                row.has_l1 = 1;
                row.l1_error = l1;
            }
        }
        if (rep->n_rows < rep->rows_cap) rep->rows[rep->n_rows] = row;
        rep->n_rows++;

        if (!std::isfinite(res)) { rep->nan_detected = 1; break; }
        if (res <= cfg.tol) { rep->converged = 1; break; }
        if (res >= prev_res) {
            if (++non_decreasing >= 3) { rep->stagnated = 1; break; }
        } else {
            non_decreasing = 0;
        }
        prev_res = res;
    }
    rep->normalization = norm_pending ? 0.0 : norm;
    pin_and_emit(u_out);
    SGML_CUDA(cudaEventRecord(tev1, s));
    SGML_CUDA(cudaEventSynchronize(tev1));
    float ms = 0.f;
    SGML_CUDA(cudaEventElapsedTime(&ms, tev0, tev1));
    if (opts.timing) harvest_spans();
    rep->device_ms = ms;
    rep->kernel_launches = launches;
    for (int k = 0; k < 8; ++k) {
        rep->class_ms[k] = cls_ms[k];
        rep->class_launches[k] = cls_n[k];
    }
    evused = 0;
    SGML_CUDA(cudaGetLastError());
}
