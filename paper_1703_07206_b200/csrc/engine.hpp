// engine.hpp — host side of the B200 SGML engine (C++, behind the C-ABI).
#pragma once

#include <array>
#include <memory>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <new>
#include <stdexcept>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sgml_b200.h"
#include "device.cuh"
#include "internal.hpp"
#include "transport.hpp"

namespace sgmlb {
struct HostStager;
}

// ---- opaque C-ABI objects ----------------------------------------------
struct sgml_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    unsigned long long* d_slots = nullptr;  // generic reduction slots
    int* d_flags = nullptr;
    unsigned long long* h_slots = nullptr;  // pinned mirrors
    int* h_flags = nullptr;
    double* h_stage = nullptr;              // pinned staging for host reductions
    size_t h_stage_bytes = 0;
    std::vector<cudaEvent_t> h_stage_events;  // chunk arrival of the staging copy
    // sgml_solve's engine cache (one problem shape), see capi.cpp
    struct sgml_solver* cached = nullptr;
    std::string cached_key;
    // serialises every entry point that uses the context's stream scratch
    // (d_slots / d_flags / h_slots / h_flags / h_stage) or its solver cache;
    // recursive: a guarded entry point may call another one
    std::recursive_mutex mu;
    // multi-GPU clique this context belongs to (z-slab solves); null: single GPU
    std::unique_ptr<sgmlb::Transport> tp;
    // pinned ring + memcpy workers for pageable host transfers (hoststage.cpp)
    sgmlb::HostStager* stager = nullptr;
};

struct sgml_field {
    sgml_ctx* ctx = nullptr;
    sgml_grid grid{};
    double* d = nullptr;
};

namespace sgmlb {

// error plumbing ----------------------------------------------------------
struct Error {
    int code;
    std::string msg;
};
void set_error(const std::string& msg);

// C-ABI wrapper body: run fn, translate exceptions into sgml_status codes
// (the message goes to sgml_last_error)
template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return SGML_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return SGML_ECUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SGML_ELOGIC;
    }
}
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define SGML_CUDA(call) ::sgmlb::cuda_check((call), #call)

BcDev to_dev(const sgml_bc& bc);
bool any_dirichlet(const sgml_bc& bc, int dim);
sgml_grid make_grid_or_throw(int dim, int n);
int relax_count(int n, int n_r, int v1);
// first replicated level of a z-slab solve on nranks ranks:
// levels v < vrep are z-slabs while a rank holds >= 2 planes of them and their
// arrays have more than replicate_n (0: SGML_REPLICATE_N) nodes per axis
int slab_vrep(int n, int nranks, int replicate_n);
RelaxConst relax_const(int dim, int level, double h, double a, double safety, bool homogeneous,
                       int compact = 0);
double* dalloc(size_t count);
void dfree(double* p);

// host <-> device copies at pinned speed for pageable host buffers
// (hoststage.cpp); call with the context lock held.  copy_h2d returns once
// the source is consumed, copy_d2h once the destination holds the data.
void copy_h2d(sgml_ctx* ctx, void* dst, const void* src, size_t bytes);
void copy_d2h(sgml_ctx* ctx, void* dst, const void* src, size_t bytes);
void destroy_stager(HostStager* st);

// serial Kahan trapezoid mean over a host copy (kernels.cpp:367-386)
double trapezoid_mean_host(sgml_ctx* ctx, const sgml_grid& g, const double* dfield);

}  // namespace sgmlb

// ---- the engine ---------------------------------------------------------
struct sgml_solver {
    sgml_ctx* ctx = nullptr;
    sgml_grid g{};
    sgml_bc bc_host{};
    sgmlb::BcDev bc{};
    bool all_neumann = false;
    double a = 0.0;
    bool has_sigma = false;
    sgml_solver_cfg cfg{};
    sgml_solver_opts opts{};
    uint64_t units_per_cycle = 0;
    int n_slots = 0;
    bool compact() const { return opts.engine == 0; }

    // schedule flattened: for every relax pass, its (level, pass_index)
    std::vector<int> pass_level, pass_index;

    // Full-grid buffers.  Compact engine: ghost-extended layout Lv[0]
    // (utot: extended without ghosts); literal engine: dense x-fastest.
    double* r = nullptr;
    double* utot = nullptr;
    double* A = nullptr;
    double* B = nullptr;
    double* fin = nullptr;     // dense staging for host-buffer solves (sgml_solve)
    double* fin2 = nullptr;    // second source / two result buffers (sgml_solve_many pipeline)
    double* uout[2] = {nullptr, nullptr};
    double* dense = nullptr;   // dense scratch / result (compact engine)
    // level arrays of the compact engine (index = level), extended layout
    std::vector<int> Nl;
    std::vector<sgmlb::ExtLay> Lv;
    std::vector<double*> P;                   // P[m], m >= 1 (P[0] is r)
    std::vector<double*> S;                   // S[m] sigma pyramid, S[0] full sigma
    std::vector<double*> DT;                  // DT[m] per-node pseudo-time step (sigma relax)
    std::vector<std::array<double*, 2>> U;    // U[v][0..1], v >= 1
    std::vector<std::vector<double*>> DU;     // DU[v][k]
    sgmlb::ChainEntry* d_chain = nullptr;     // per-tooth pending-increment lists
    std::vector<sgmlb::ChainEntry> h_chain;   // (host copy)
    std::vector<int> tooth_off;               // offset of tooth v1's list in d_chain
    std::vector<const double*> du_bufs;       // DU arrays (faces without mirror ghosts)
    // TMA descriptors per buffer: window box (tile + halo) and tile box
    std::vector<std::pair<const double*, CUtensorMap>> map_u, map_g;
    const CUtensorMap& umap(const double* p) const;
    const CUtensorMap& gmap(const double* p) const;
    void add_maps(const double* p, const sgmlb::ExtLay& L, bool want_u, bool want_g);
    // literal-engine buffers
    double *Lg = nullptr, *Lscr = nullptr, *Lu = nullptr, *Lup = nullptr, *Ldu = nullptr,
           *Ldup = nullptr;
    std::vector<double*> Lsig;                // full sigma levels
    // per-cycle device scratch: [0..n_slots) diag, n_slots = rmax
    unsigned long long* d_cycle = nullptr;
    // flag[0] failed pass, [1] tiny level value, [2..3] neighbours' [1],
    // [4] first failing pass (min), [5] scratch
    int* d_flag = nullptr;
    bool diag_mode = false;  // materialisations attribute non-finite values to passes
    unsigned long long* h_cycle = nullptr;
    int* h_flag = nullptr;
    uint64_t bytes = 0;
    uint64_t launches = 0;
    // per-class device timing (opts.timing): event pairs harvested per cycle
    struct Span {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<cudaEvent_t> evpool;
    size_t evused = 0;
    std::vector<Span> spans;
    cudaEvent_t tev0 = nullptr, tev1 = nullptr;  // whole-solve timing
    double cls_ms[8] = {0};
    uint64_t cls_n[8] = {0};

    ~sgml_solver();
    void build(sgml_ctx* c, int dim, int n, const sgml_bc& bcin, double a_, const double* sigma_dev,
               const sgml_solver_cfg& cfg_, const sgml_solver_opts& opts_);
    // (re)load the coefficient from a DENSE device field: sigma pyramid /
    // literal sigma levels, positivity check (cycle.cpp:117-133)
    void load_sigma(const double* sigma_dense);
    // dense device buffer an uploaded coefficient can be staged in
    double* sigma_stage() { return compact() ? dense : Lsig[0]; }
    // timed launch: records an event pair around fn when opts.timing
    int debug_sync = -1;  // SGML_DEBUG_SYNC=1: synchronize + check after every launch
    void check_launch(int cls);
    template <typename F>
    void launch(int cls, F&& fn) {
        flush_kops();  // recorded small-level operations run before anything launched after them
        ++launches;
        if (debug_sync < 0) debug_sync = std::getenv("SGML_DEBUG_SYNC") ? 1 : 0;
        if (debug_sync) {
            fn();
            check_launch(cls);
            return;
        }
        if (!opts.timing || (opts.timing_classes && !((opts.timing_classes >> cls) & 1))) {
            fn();
            return;
        }
        Span sp{cls, next_event(), next_event()};
        // (inside a stream capture an external record makes a real record node)
        const unsigned fl = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
        cudaEventRecordWithFlags(sp.a, ctx->stream, fl);
        fn();
        cudaEventRecordWithFlags(sp.b, ctx->stream, fl);
        spans.push_back(sp);
    }
    // One cycle as a CUDA graph (single-GPU compact engine): the ~145
    // launches of a cycle replay from the device's queue instead of the
    // host's, so the coarse levels do not pay host launch latency.  A graph
    // is valid for the face-state map it was captured from (the host-side
    // bookkeeping of cycle_compact); a mismatch recaptures.
    struct CycleGraph {
        cudaGraphExec_t exec = nullptr;
        std::unordered_map<const double*, int> pre, post;
        const double* out = nullptr;
        uint64_t nlaunch = 0;
        std::vector<Span> spans;          // timing spans (graph-owned events)
        std::vector<cudaEvent_t> events;
    };
    CycleGraph graphs[2];                 // by homogeneous
    CycleGraph* capturing = nullptr;
    bool slab_graphs_off = false;         // a z-slab capture failed on some rank: eager cycles
    bool use_graphs() const;
    bool small_visit(int v, const double* in, int c, const double* p0, const double* p1, bool homogeneous) const;
    // small-level interpreter (interp.cu): operations on level arrays of at
    // most kClusterNodes nodes are recorded during a cycle and run by one cluster
    // launch per batch (single GPU, compact engine, outside failure re-runs)
    std::vector<sgmlb::KOp> kops;
    bool kops_cycle = false;   // this cycle records small-level operations
    bool cyc_homog = false;    // the cycle's homogeneous flag (relaxation constants of a batch)
    bool kop_level(int v) const { return kops_cycle && v < (int)kop_ok.size() && kop_ok[v]; }
    std::vector<char> kop_ok;  // level v's array is small enough
    std::unique_ptr<sgmlb::KOpBatch> kop_batch;
    void flush_kops();
    void record(const sgmlb::KOp& op) { kops.push_back(op); }
    const double* cycle_graph(bool homogeneous);
    cudaEvent_t next_event();
    void harvest_spans();  // call after a stream synchronize
    // cycle.cpp:140-247 on a DENSE device source; the dense result goes to
    // u_out_dev (or the internal dense buffer, see result())
    void run(const double* f_dev, double* u_out_dev, sgml_report* rep);
    const double* result() const { return compact() ? dense : utot; }
    // one cycle on the engine's own source buffer r; returns state.u in the
    // engine layout
    const double* cycle(bool homogeneous);
    const double* cycle_compact(bool homogeneous);
    const double* cycle_literal(bool homogeneous);
    // one cycle from a dense source into a dense state.u (sgml_single_cycle)
    void cycle_dense(const double* src_dense, double* out_dense, bool homogeneous);
    void load_source(const double* f_dense);            // r <- f
    void zero_mean_r();                                  // zero_mean_projection(r)
    double max_abs_r(const double* f_dense);             // max |r| (data nodes)
    void residual(const double* e, bool guarded = false);  // fused recurrence step
    bool residual_guardable(const double* e) const;
    void reset_fail_flags();
    int first_failing_pass(bool homogeneous);            // after a failed cycle
    const double* dense_view(const double* engine_field);  // dense device view
    void pin_and_emit(double* u_out_dev);                // pure_neumann_pin + result
    void ensure_literal();
    double* alloc(size_t count);

    // z-slab decomposition (3D compact engine on a clique of nrk ranks,
    // SURVEY.md §8e).  Level v < vrep is a z-slab per rank (own planes plus
    // one halo plane each side, exchanged after every producer); levels
    // v >= vrep are replicated (computed redundantly by every rank from
    // replicated inputs).  nrk = 1: nothing is distributed.
    sgmlb::Transport* tp = nullptr;
    int nrk = 1, rank = 0, vrep = 0, T0 = 0;
    bool dist(int v) const { return nrk > 1 && v < vrep; }
    double* BS = nullptr;      // base sampled on level vrep (replicated), for replicated targets
    bool bs_valid = false;
    void halo(double* a, int v);
    bool overlap_halos(int v);
    cudaStream_t hx_stream = nullptr;  // halo transfers overlapped with interior planes
    cudaEvent_t hx_ready = nullptr, hx_done = nullptr;                          // after a producer at a z-slab level
    void gather_level(double* a, int v);                  // replicated level: own planes -> all
    void own_planes(int v, int p, int& kb, int& cnt) const;  // rank p's planes of level v
    void refresh_bs(const double* base);
    void pyramid_step(const double* in, int m, double* out);

    // Dirichlet-face bookkeeping of the compact engine.  Relaxation and
    // residual kernels cover only the nodes off the Dirichlet faces
    // (rng[v]); the face nodes of every buffer keep a known content, tracked
    // here, and are rewritten only when a consumer needs another one.
    enum { FS_ZERO = 0, FS_BVAL = 1, FS_OTHER = 2 };
    std::vector<sgmlb::NodeRange> rng;
    bool bval_zero = true;     // every Dirichlet face value is 0
    bool bval_finite = true;
    bool bval_tiny = false;    // a Dirichlet value in (0, 2^-969)
    std::unordered_map<const double*, int> fstate;
    int face_want(bool homogeneous) const { return (homogeneous || bval_zero) ? FS_ZERO : FS_BVAL; }
    int faces_of(const double* p) const;
    void set_faces(double* p, int level, int st);
};
