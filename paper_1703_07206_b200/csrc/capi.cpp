// capi.cpp — extern "C" boundary (include/sgml_b200.h).
//
// Translates C++ exceptions into sgml_status codes, owns contexts and
// device fields, and implements the kernel-level entry points of
// kernels.hpp on top of the literal sm_100a kernels.
#include <cmath>
#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

#include "engine.hpp"

namespace sgmlb {
const char* last_error_cstr();
}

using namespace sgmlb;

namespace {

void require(bool ok, int code, const char* msg) {
    if (!ok) fail(code, msg);
}

void same_grid(const sgml_field* a, const sgml_field* b, const char* what) {
    require(a && b, SGML_EINVAL, what);
    require(a->grid.dim == b->grid.dim && a->grid.n == b->grid.n, SGML_EINVAL, what);
}

void activate(sgml_ctx* ctx) { SGML_CUDA(cudaSetDevice(ctx->device)); }

// entry points that use the context's reduction slots, flags or pinned
// staging hold its lock for the whole call (the reference's functions are
// reentrant; concurrent callers of one context must not share that scratch)
using CtxLock = std::lock_guard<std::recursive_mutex>;

double slot_to_double(unsigned long long bits) {
    double d;
    std::memcpy(&d, &bits, sizeof d);
    return d;
}


// RAII device scratch (post-solve temporaries)
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { SGML_CUDA(cudaMalloc(&p, bytes ? bytes : 1)); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    double* d() const { return static_cast<double*>(p); }
    int* i() const { return static_cast<int*>(p); }
};

double inv2h_of(const sgml_grid& g) { return 1.0 / (2.0 * g.h); }  // problems.cpp:80

}  // namespace

extern "C" {

const char* sgml_last_error(void) { return last_error_cstr(); }

const char* sgml_version(void) { return "sgml-b200 0.1 (sm_100a, fp64, no-FMA parity build)"; }

int sgml_device_count(int* count) {
    return guarded([&] {
        int c = 0;
        const cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *count = c;
    });
}

int sgml_ctx_create(int device, sgml_ctx** out) {
    return guarded([&] {
        require(out != nullptr, SGML_EINVAL, "ctx_create: null out");
        int count = 0;
        SGML_CUDA(cudaGetDeviceCount(&count));
        require(device >= 0 && device < count, SGML_EINVAL, "ctx_create: no such CUDA device");
        auto ctx = std::make_unique<sgml_ctx>();
        ctx->device = device;
        SGML_CUDA(cudaSetDevice(device));
        SGML_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        SGML_CUDA(cudaMalloc((void**)&ctx->d_slots, 64 * sizeof(unsigned long long)));
        SGML_CUDA(cudaMalloc((void**)&ctx->d_flags, 16 * sizeof(int)));
        SGML_CUDA(cudaMallocHost((void**)&ctx->h_slots, 64 * sizeof(unsigned long long)));
        SGML_CUDA(cudaMallocHost((void**)&ctx->h_flags, 16 * sizeof(int)));
        *out = ctx.release();
    });
}

struct sgml_group {
    std::shared_ptr<sgmlb::LocalGroup> g;
};

int sgml_nccl_unique_id(unsigned char id[128]) {
    return guarded([&] {
        require(id != nullptr, SGML_EINVAL, "nccl_unique_id: null id");
        sgmlb::nccl_unique_id(id);
    });
}

int sgml_ctx_join_nccl(sgml_ctx* ctx, int nranks, int rank, const unsigned char id[128]) {
    return guarded([&] {
        require(ctx && id, SGML_EINVAL, "ctx_join_nccl: null argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, SGML_EINVAL, "ctx_join_nccl: bad rank");
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        SGML_CUDA(cudaSetDevice(ctx->device));
        delete ctx->cached;
        ctx->cached = nullptr;
        ctx->cached_key.clear();
        ctx->tp = sgmlb::make_nccl_transport(nranks, rank, id);
    });
}

int sgml_local_group_create(int nranks, sgml_group** out) {
    return guarded([&] {
        require(out != nullptr && nranks >= 1, SGML_EINVAL, "local_group_create: bad arguments");
        auto g = std::make_unique<sgml_group>();
        g->g = std::make_shared<sgmlb::LocalGroup>(nranks);
        *out = g.release();
    });
}

int sgml_local_group_destroy(sgml_group* g) {
    return guarded([&] { delete g; });
}

int sgml_ctx_join_local(sgml_ctx* ctx, sgml_group* g, int rank) {
    return guarded([&] {
        require(ctx && g, SGML_EINVAL, "ctx_join_local: null argument");
        require(rank >= 0 && rank < g->g->size, SGML_EINVAL, "ctx_join_local: bad rank");
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        delete ctx->cached;
        ctx->cached = nullptr;
        ctx->cached_key.clear();
        ctx->tp.reset(new sgmlb::LocalTransport(g->g, rank));
    });
}

int sgml_ctx_clique(sgml_ctx* ctx, int* nranks, int* rank) {
    return guarded([&] {
        require(ctx && nranks && rank, SGML_EINVAL, "ctx_clique: null argument");
        *nranks = ctx->tp ? ctx->tp->size : 1;
        *rank = ctx->tp ? ctx->tp->rank : 0;
    });
}

int sgml_slab_plan(int n, int nranks, int rank, int* vrep, int* z0, int* nz) {
    return sgml_slab_plan_ex(n, nranks, rank, 0, vrep, z0, nz);
}

int sgml_slab_plan_ex(int n, int nranks, int rank, int replicate_n, int* vrep, int* z0, int* nz) {
    return guarded([&] {
        require(vrep && z0 && nz, SGML_EINVAL, "slab_plan: null argument");
        require(n >= 1 && n <= 13, SGML_EINVAL, "slab_plan: n must lie in [1, 13]");
        require(nranks >= 1 && (nranks & (nranks - 1)) == 0, SGML_EINVAL,
                "slab_plan: the number of ranks must be a power of two");
        require(nranks <= (1 << (n - 1)) || nranks == 1, SGML_EINVAL,
                "slab_plan: too many ranks for this grid (>= 2 planes each)");
        require(rank >= 0 && rank < nranks, SGML_EINVAL, "slab_plan: bad rank");
        const int t0 = (1 << n) / nranks;
        *vrep = slab_vrep(n, nranks, replicate_n);
        *z0 = rank * t0;
        *nz = t0 + (rank == nranks - 1 ? 1 : 0);
    });
}

int sgml_ctx_destroy(sgml_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaFree(ctx->d_slots);
        cudaFree(ctx->d_flags);
        cudaFreeHost(ctx->h_slots);
        cudaFreeHost(ctx->h_flags);
        if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
        for (cudaEvent_t e : ctx->h_stage_events) cudaEventDestroy(e);
        destroy_stager(ctx->stager);
        delete ctx->cached;
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int sgml_ctx_synchronize(sgml_ctx* ctx) {
    return guarded([&] {
        activate(ctx);
        SGML_CUDA(cudaStreamSynchronize(ctx->stream));
        SGML_CUDA(cudaGetLastError());
    });
}

void* sgml_ctx_stream(sgml_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

// ---- grid / schedule -----------------------------------------------------

int sgml_make_grid(int dim, int n, sgml_grid* out) {
    return guarded([&] { *out = make_grid_or_throw(dim, n); });
}

int sgml_build_schedule(int n, int n_r, int* kinds, int* levels, int* counts, int cap, int* count) {
    return guarded([&] {
        require(n >= 1, SGML_EINVAL, "build_schedule: n must be >= 1");
        require(n_r >= 1, SGML_EINVAL, "build_schedule: n_r must be >= 1");
        int c = 0;
        auto push = [&](int k, int l, int cnt) {
            if (c < cap) { kinds[c] = k; levels[c] = l; counts[c] = cnt; }
            ++c;
        };
        for (int v1 = n - 1; v1 >= 0; --v1) {
            const int cnt = relax_count(n, n_r, v1);
            for (int v = v1; v >= 0; --v) {
                push(0, v, 1);
                push(1, v, cnt);
            }
        }
        const long long tail_cap = n < 62 ? (1LL << n) : (1LL << 62);
        push(1, 0, (int)std::min<long long>(n_r, tail_cap));
        *count = c;
    });
}

uint64_t sgml_closed_form_work_units(int n, int n_r) {
    if (n < 1 || n_r < 1) return 0;
    uint64_t total = 0;
    for (int v1 = 0; v1 <= n - 1; ++v1) {
        total += (uint64_t)v1 * (v1 + 1) / 2;
        total += (uint64_t)(v1 + 1) * relax_count(n, n_r, v1);
    }
    const long long tail_cap = n < 62 ? (1LL << n) : (1LL << 62);
    total += (uint64_t)std::min<long long>(n_r, tail_cap);
    return total;
}

// ---- fields ----------------------------------------------------------------

int sgml_field_create(sgml_ctx* ctx, int dim, int n, sgml_field** out) {
    return guarded([&] {
        require(ctx && out, SGML_EINVAL, "field_create: null argument");
        auto f = std::make_unique<sgml_field>();
        f->ctx = ctx;
        f->grid = make_grid_or_throw(dim, n);
        activate(ctx);
        f->d = dalloc(f->grid.total);
        SGML_CUDA(cudaMemsetAsync(f->d, 0, f->grid.total * sizeof(double), ctx->stream));
        SGML_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = f.release();
    });
}

int sgml_field_destroy(sgml_field* f) {
    return guarded([&] {
        if (!f) return;
        cudaSetDevice(f->ctx->device);
        cudaStreamSynchronize(f->ctx->stream);
        dfree(f->d);
        delete f;
    });
}

int sgml_field_upload(sgml_field* f, const double* host) {
    return guarded([&] {
        require(f && host, SGML_EINVAL, "field_upload: null argument");
        activate(f->ctx);
        CtxLock lk(f->ctx->mu);
        copy_h2d(f->ctx, f->d, host, f->grid.total * sizeof(double));
        SGML_CUDA(cudaStreamSynchronize(f->ctx->stream));
    });
}

int sgml_field_download(const sgml_field* f, double* host) {
    return guarded([&] {
        require(f && host, SGML_EINVAL, "field_download: null argument");
        activate(f->ctx);
        CtxLock lk(f->ctx->mu);
        copy_d2h(f->ctx, host, f->d, f->grid.total * sizeof(double));
    });
}

int sgml_field_copy(sgml_field* dst, const sgml_field* src) {
    return guarded([&] {
        same_grid(dst, src, "field_copy: grid mismatch");
        activate(dst->ctx);
        SGML_CUDA(cudaMemcpyAsync(dst->d, src->d, dst->grid.total * sizeof(double),
                                  cudaMemcpyDeviceToDevice, dst->ctx->stream));
        SGML_CUDA(cudaStreamSynchronize(dst->ctx->stream));
    });
}

int sgml_field_fill(sgml_field* f, double value) {
    return guarded([&] {
        require(f != nullptr, SGML_EINVAL, "field_fill: null field");
        activate(f->ctx);
        launch_fill(f->d, f->grid.total, value, f->ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(f->ctx->stream));
    });
}

int sgml_field_grid(const sgml_field* f, sgml_grid* out) {
    return guarded([&] {
        require(f && out, SGML_EINVAL, "field_grid: null argument");
        *out = f->grid;
    });
}

void* sgml_field_device_ptr(sgml_field* f) { return f ? (void*)f->d : nullptr; }

// ---- kernels -------------------------------------------------------------

int sgml_restriction_into(const sgml_field* f, int v, const sgml_bc* bc, sgml_field* out,
                          sgml_field* scratch, uint64_t* work) {
    return guarded([&] {
        same_grid(f, out, "restriction_into: grid mismatch");
        same_grid(f, scratch, "restriction_into: grid mismatch");
        require(bc != nullptr, SGML_EINVAL, "restriction_into: null bc");
        require(out != scratch, SGML_EINVAL, "restriction_into: out and scratch must differ");
        require(v >= 0 && v <= f->grid.n, SGML_EINVAL, "restriction_into: level out of range");
        sgml_ctx* ctx = f->ctx;
        activate(ctx);
        const sgml_grid& g = f->grid;
        const cudaStream_t s = ctx->stream;
        if (v == 0) {
            SGML_CUDA(cudaMemcpyAsync(out->d, f->d, g.total * sizeof(double), cudaMemcpyDeviceToDevice, s));
        } else {
            const BcDev b = to_dev(*bc);
            const double* src = f->d;
            double* dst = (v % 2 == 1) ? out->d : scratch->d;
            for (int m = 0; m < v; ++m) {
                launch_restrict_pass(g.dim, src, dst, g.N, 1 << m, b, s);
                src = dst;
                dst = (dst == out->d) ? scratch->d : out->d;
            }
            if (work) *work += (uint64_t)v;
        }
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(s));
    });
}

int sgml_relaxation_interpolation(sgml_field* u, const sgml_field* u_prev, sgml_field* du,
                                  const sgml_field* du_prev, int level, const sgml_field* g,
                                  const sgml_field* sigma, double a, double safety,
                                  const sgml_bc* bc, int homogeneous, double* diag_out,
                                  uint64_t* work) {
    return guarded([&] {
        same_grid(u, u_prev, "relaxation_interpolation: grid mismatch");
        same_grid(u, du, "relaxation_interpolation: grid mismatch");
        same_grid(u, du_prev, "relaxation_interpolation: grid mismatch");
        same_grid(u, g, "relaxation_interpolation: grid mismatch");
        if (sigma) same_grid(u, sigma, "relaxation_interpolation: grid mismatch");
        require(bc != nullptr, SGML_EINVAL, "relaxation_interpolation: null bc");
        require(level >= 0 && level <= u->grid.n, SGML_EINVAL, "relaxation_interpolation: bad level");
        sgml_ctx* ctx = u->ctx;
        activate(ctx);
        CtxLock lk(ctx->mu);
        const cudaStream_t s = ctx->stream;
        const sgml_grid& gr = u->grid;
        SGML_CUDA(cudaMemsetAsync(ctx->d_slots, 0, sizeof(unsigned long long), s));
        SGML_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), s));
        const RelaxConst rc = relax_const(gr.dim, level, gr.h, a, safety, homogeneous != 0);
        launch_relax_literal(gr.dim, sigma != nullptr, u->d, du->d, u_prev->d, du_prev->d, g->d,
                             sigma ? sigma->d : nullptr, gr.N, level, rc, to_dev(*bc), ctx->d_slots,
                             ctx->d_flags, 0, s);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaMemcpyAsync(ctx->h_slots, ctx->d_slots, sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        if (diag_out) *diag_out = slot_to_double(ctx->h_slots[0]);
        // kernels.cpp:343-346: badstep is checked first, then non-finite
        if (!(safety > 0.0)) fail(SGML_EBADSTEP, "relaxation_interpolation: non-positive pseudo-time step");
        if (ctx->h_flags[0]) fail(SGML_ENONFINITE, "relaxation_interpolation: non-finite value produced");
        if (work) *work += 1;
    });
}

int sgml_residual_update(sgml_field* r, const sgml_field* e, const sgml_field* sigma, double a,
                         const sgml_bc* bc) {
    return guarded([&] {
        same_grid(r, e, "residual_update: grid mismatch");
        if (sigma) same_grid(r, sigma, "residual_update: grid mismatch");
        require(bc != nullptr, SGML_EINVAL, "residual_update: null bc");
        sgml_ctx* ctx = r->ctx;
        activate(ctx);
        const sgml_grid& g = r->grid;
        launch_residual(g.dim, sigma != nullptr, r->d, e->d, nullptr, sigma ? sigma->d : nullptr, g.N,
                        1.0 / (g.h * g.h), g.dim == 2 ? 0.5 : 3.0 / 13.0, a, to_dev(*bc), nullptr, ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int sgml_max_abs(const sgml_field* f, double* out) {
    return guarded([&] {
        require(f && out, SGML_EINVAL, "max_abs: null argument");
        sgml_ctx* ctx = f->ctx;
        activate(ctx);
        CtxLock lk(ctx->mu);
        const cudaStream_t s = ctx->stream;
        SGML_CUDA(cudaMemsetAsync(ctx->d_slots, 0, sizeof(unsigned long long), s));
        launch_max_abs(f->d, f->grid.total, ctx->d_slots, s);
        SGML_CUDA(cudaMemcpyAsync(ctx->h_slots, ctx->d_slots, sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        *out = slot_to_double(ctx->h_slots[0]);
    });
}

int sgml_trapezoid_mean(const sgml_field* f, double* out) {
    return guarded([&] {
        require(f && out, SGML_EINVAL, "trapezoid_mean: null argument");
        activate(f->ctx);
        CtxLock lk(f->ctx->mu);
        *out = trapezoid_mean_host(f->ctx, f->grid, f->d);
    });
}

int sgml_zero_mean_projection(sgml_field* f) {
    return guarded([&] {
        require(f != nullptr, SGML_EINVAL, "zero_mean_projection: null field");
        activate(f->ctx);
        CtxLock lk(f->ctx->mu);
        const double mean = trapezoid_mean_host(f->ctx, f->grid, f->d);
        launch_sub_scalar(f->d, f->grid.total, mean, f->ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(f->ctx->stream));
    });
}

int sgml_pure_neumann_pin(sgml_field* u) { return sgml_zero_mean_projection(u); }

int sgml_apply_boundary(sgml_field* u, const sgml_bc* bc, int homogeneous) {
    return guarded([&] {
        require(u && bc, SGML_EINVAL, "apply_boundary: null argument");
        activate(u->ctx);
        launch_apply_boundary(u->grid.dim, u->d, u->grid.N, to_dev(*bc), homogeneous != 0, u->ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(u->ctx->stream));
    });
}

int sgml_restrict_sigma_levels(const sgml_field* sigma, sgml_field* const* levels) {
    return guarded([&] {
        require(sigma && levels, SGML_EINVAL, "restrict_sigma_levels: null argument");
        const sgml_grid& g = sigma->grid;
        for (int v = 0; v < g.n; ++v) same_grid(sigma, levels[v], "restrict_sigma_levels: grid mismatch");
        sgml_ctx* ctx = sigma->ctx;
        activate(ctx);
        CtxLock lk(ctx->mu);
        const cudaStream_t s = ctx->stream;
        sgml_bc even{};
        for (int f = 0; f < 6; ++f) even.kind[f] = 1;
        const BcDev ev = to_dev(even);
        double* scr = dalloc(g.total);
        SGML_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), s));
        for (int v = 0; v < g.n; ++v) {
            double* out = levels[v]->d;
            if (v == 0) {
                SGML_CUDA(cudaMemcpyAsync(out, sigma->d, g.total * sizeof(double), cudaMemcpyDeviceToDevice, s));
            } else {
                const double* src = sigma->d;
                double* dst = (v % 2 == 1) ? out : scr;
                for (int m = 0; m < v; ++m) {
                    launch_restrict_pass(g.dim, src, dst, g.N, 1 << m, ev, s);
                    src = dst;
                    dst = (dst == out) ? scr : out;
                }
            }
            launch_check_positive(out, g.total, ctx->d_flags, s);
        }
        SGML_CUDA(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        dfree(scr);
        if (ctx->h_flags[0]) fail(SGML_EINVAL, "restrict_sigma_levels: coefficient must stay positive");
    });
}

// ---- driver ----------------------------------------------------------------

int sgml_single_cycle(sgml_ctx* ctx, sgml_field* state_u, const sgml_field* source,
                      sgml_field* const* sigma_levels, double a, const sgml_bc* bc, int homogeneous,
                      int n_r, double safety, int cycle_index, double normalization,
                      const sgml_solver_opts* opts, sgml_report* rep, uint64_t* work) {
    return guarded([&] {
        require(ctx && state_u && source && bc && rep && work, SGML_EINVAL, "single_cycle: null argument");
        same_grid(state_u, source, "single_cycle: grid mismatch");
        require(n_r >= 1, SGML_EINVAL, "build_schedule: n_r must be >= 1");
        const sgml_grid& g = source->grid;
        activate(ctx);
        CtxLock lk(ctx->mu);
        sgml_solver_opts o{};
        if (opts) o = *opts;
        sgml_solver_cfg cfg{n_r, 1, 1.0, safety};
        sgml_solver sv;
        // literal engine when full sigma levels are supplied; the compact
        // engine rebuilds its own sigma pyramid from level 0 (identical bits)
        sv.build(ctx, g.dim, g.n, *bc, a, sigma_levels ? sigma_levels[0]->d : nullptr, cfg, o);
        const cudaStream_t s = ctx->stream;
        if (!(safety > 0.0)) {
            // the first Restrict(n-1) step completes before the first pass throws
            *work += (uint64_t)(g.n - 1);
            fail(SGML_EBADSTEP, "relaxation_interpolation: non-positive pseudo-time step");
        }
        SGML_CUDA(cudaMemsetAsync(sv.d_cycle, 0, (sv.n_slots + 1) * sizeof(unsigned long long), s));
        sv.reset_fail_flags();
        sv.cycle_dense(source->d, state_u->d, homogeneous != 0);
        SGML_CUDA(cudaMemcpyAsync(sv.h_cycle, sv.d_cycle, sv.n_slots * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaMemcpyAsync(sv.h_flag, sv.d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        SGML_CUDA(cudaGetLastError());
        // a failing pass throws after the samples and work units of the steps
        // before it (cycle.cpp:88-107): pass_index[p] counts the units before pass p
        int passes = sv.n_slots;
        if (sv.h_flag[0]) passes = std::min(sv.first_failing_pass(homogeneous != 0), sv.n_slots);
        const double inv_norm = normalization > 0.0 ? 1.0 / normalization : 1.0;
        for (int p = 0; p < passes; ++p) {
            if (rep->n_trace < rep->trace_cap)
                rep->trace[rep->n_trace] = sgml_diag_sample{cycle_index, sv.pass_index[p], sv.pass_level[p], 0,
                                                            slot_to_double(sv.h_cycle[p]) * inv_norm};
            rep->n_trace++;
        }
        if (sv.h_flag[0]) {
            *work += passes < sv.n_slots ? (uint64_t)sv.pass_index[passes] : sv.units_per_cycle;
            fail(SGML_ENONFINITE, "relaxation_interpolation: non-finite value produced");
        }
        *work += sv.units_per_cycle;
    });
}

int sgml_single_cycle_state(sgml_ctx* ctx, sgml_field* u, sgml_field* u_prev, sgml_field* du,
                            sgml_field* du_prev, int* level, const sgml_field* source,
                            sgml_field* const* sigma_levels, double a, const sgml_bc* bc, int homogeneous,
                            const int* step_kinds, const int* step_levels, const int* step_counts, int nsteps,
                            double safety, int cycle_index, double normalization, sgml_report* rep,
                            uint64_t* work) {
    return guarded([&] {
        require(ctx && u && u_prev && du && du_prev && level && source && bc && rep && work, SGML_EINVAL,
                "single_cycle: null argument");
        require(nsteps >= 0 && (nsteps == 0 || (step_kinds && step_levels && step_counts)), SGML_EINVAL,
                "single_cycle: bad schedule");
        const sgml_field* others[4] = {u_prev, du, du_prev, source};
        for (const sgml_field* f : others) same_grid(u, f, "single_cycle: grid mismatch");
        const sgml_grid& g = u->grid;
        for (int i = 0; i < nsteps; ++i)
            require(step_levels[i] >= 0 && step_levels[i] <= g.n && step_counts[i] >= 0, SGML_EINVAL,
                    "single_cycle: bad schedule step");
        activate(ctx);
        CtxLock lk(ctx->mu);
        const cudaStream_t s = ctx->stream;
        const BcDev b = to_dev(*bc);
        // cycle.cpp:83-84: g and scratch start zeroed every cycle
        DevBuf gbuf(g.total * sizeof(double)), sbuf(g.total * sizeof(double));
        double* gd = gbuf.d();
        double* sd = sbuf.d();
        SGML_CUDA(cudaMemsetAsync(gd, 0, g.total * sizeof(double), s));
        SGML_CUDA(cudaMemsetAsync(sd, 0, g.total * sizeof(double), s));
        int pass_index = 0, current = -1;
        const double inv_norm = normalization > 0.0 ? 1.0 / normalization : 1.0;
        for (int i = 0; i < nsteps; ++i) {
            const int v = step_levels[i];
            if (step_kinds[i] == 0) {
                // restriction_into(source, v, bc, g, scratch, &work) (kernels.cpp:305-325)
                if (v == 0) {
                    SGML_CUDA(cudaMemcpyAsync(gd, source->d, g.total * sizeof(double), cudaMemcpyDeviceToDevice, s));
                } else {
                    const double* src = source->d;
                    double* dst = (v % 2 == 1) ? gd : sd;
                    for (int m = 0; m < v; ++m) {
                        launch_restrict_pass(g.dim, src, dst, g.N, 1 << m, b, s);
                        src = dst;
                        dst = (dst == gd) ? sd : gd;
                    }
                    *work += (uint64_t)v;
                    pass_index += v;
                }
                continue;
            }
            if (v != current) {  // SolveState::reset_level
                SGML_CUDA(cudaMemsetAsync(du->d, 0, g.total * sizeof(double), s));
                SGML_CUDA(cudaMemsetAsync(du_prev->d, 0, g.total * sizeof(double), s));
                *level = v;
                current = v;
            }
            const sgml_field* sig = sigma_levels ? sigma_levels[v] : nullptr;
            if (sig) same_grid(u, sig, "single_cycle: sigma level grid mismatch");
            const RelaxConst rc = relax_const(g.dim, v, g.h, a, safety, homogeneous != 0);
            for (int c = 0; c < step_counts[i]; ++c) {
                std::swap(u->d, u_prev->d);  // SolveState::swap_buffers
                std::swap(du->d, du_prev->d);
                SGML_CUDA(cudaMemsetAsync(ctx->d_slots, 0, sizeof(unsigned long long), s));
                SGML_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), s));
                launch_relax_literal(g.dim, sig != nullptr, u->d, du->d, u_prev->d, du_prev->d, gd,
                                     sig ? sig->d : nullptr, g.N, v, rc, b, ctx->d_slots, ctx->d_flags, 0, s);
                SGML_CUDA(cudaGetLastError());
                SGML_CUDA(cudaMemcpyAsync(ctx->h_slots, ctx->d_slots, sizeof(unsigned long long),
                                          cudaMemcpyDeviceToHost, s));
                SGML_CUDA(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s));
                SGML_CUDA(cudaStreamSynchronize(s));
                // kernels.cpp:343-346: the pass throws before its work unit and sample
                if (!(safety > 0.0)) fail(SGML_EBADSTEP, "relaxation_interpolation: non-positive pseudo-time step");
                if (ctx->h_flags[0]) fail(SGML_ENONFINITE, "relaxation_interpolation: non-finite value produced");
                *work += 1;
                if (rep->n_trace < rep->trace_cap)
                    rep->trace[rep->n_trace] =
                        sgml_diag_sample{cycle_index, pass_index, v, 0, slot_to_double(ctx->h_slots[0]) * inv_norm};
                rep->n_trace++;
                ++pass_index;
            }
        }
        SGML_CUDA(cudaStreamSynchronize(s));
    });
}

int sgml_solver_create(sgml_ctx* ctx, int dim, int n, const sgml_bc* bc, double a,
                       const sgml_field* sigma, const sgml_solver_cfg* cfg,
                       const sgml_solver_opts* opts, sgml_solver** out) {
    return guarded([&] {
        require(ctx && bc && cfg && out, SGML_EINVAL, "solver_create: null argument");
        if (sigma) require(sigma->grid.dim == dim && sigma->grid.n == n, SGML_EINVAL, "solve: sigma grid mismatch");
        sgml_solver_opts o{};
        if (opts) o = *opts;
        CtxLock lk(ctx->mu);
        auto sv = std::make_unique<sgml_solver>();
        sv->build(ctx, dim, n, *bc, a, sigma ? sigma->d : nullptr, *cfg, o);
        *out = sv.release();
    });
}

int sgml_solver_destroy(sgml_solver* s) {
    return guarded([&] { delete s; });
}

int sgml_solver_run(sgml_solver* s, const sgml_field* f, sgml_field* u_out, sgml_report* rep) {
    return guarded([&] {
        require(s && f && rep, SGML_EINVAL, "solver_run: null argument");
        require(f->grid.dim == s->g.dim && f->grid.n == s->g.n, SGML_EINVAL, "solve: source grid mismatch");
        if (u_out) require(u_out->grid.dim == s->g.dim && u_out->grid.n == s->g.n, SGML_EINVAL,
                           "solve: output grid mismatch");
        CtxLock lk(s->ctx->mu);
        s->run(f->d, u_out ? u_out->d : nullptr, rep);
    });
}

int sgml_solver_footprint(const sgml_solver* s, uint64_t* bytes) {
    return guarded([&] {
        require(s && bytes, SGML_EINVAL, "solver_footprint: null argument");
        *bytes = s->bytes;
    });
}

}  // extern "C"

namespace {

// sgml_solve's engine cache: one engine per context for the last problem
// shape (grid, bc, a, cfg, opts, sigma present); sigma is (re)loaded when given.
// Call with ctx->mu held.
sgml_solver* cached_solver(sgml_ctx* ctx, int dim, int n, const sgml_bc* bc, const double* sigma_host, double a,
                           const sgml_solver_cfg* cfg, const sgml_solver_opts& o) {
    const sgml_grid g = make_grid_or_throw(dim, n);
    std::string key(reinterpret_cast<const char*>(&g), sizeof g);
    key.append(reinterpret_cast<const char*>(bc), sizeof *bc);
    key.append(reinterpret_cast<const char*>(&a), sizeof a);
    key.append(reinterpret_cast<const char*>(cfg), sizeof *cfg);
    key.append(reinterpret_cast<const char*>(&o), sizeof o);
    key.push_back(sigma_host ? 's' : '-');
    const size_t bytes = g.total * sizeof(double);
    if (!ctx->cached || ctx->cached_key != key) {
        delete ctx->cached;
        ctx->cached = nullptr;
        ctx->cached_key.clear();
        double* sig = nullptr;
        struct Guard {
            double* p = nullptr;
            ~Guard() { dfree(p); }
        } sg;
        if (sigma_host) {
            sg.p = sig = dalloc(g.total);
            copy_h2d(ctx, sig, sigma_host, bytes);
        }
        auto sv = std::make_unique<sgml_solver>();
        sv->build(ctx, dim, n, *bc, a, sig, *cfg, o);
        sv->fin = sv->alloc(g.total);
        ctx->cached = sv.release();
        ctx->cached_key = key;
    } else if (sigma_host) {
        sgml_solver* sv = ctx->cached;
        copy_h2d(ctx, sv->sigma_stage(), sigma_host, bytes);
        sv->load_sigma(sv->sigma_stage());
    }
    return ctx->cached;
}

void check_solve_args(const sgml_solver_cfg* cfg) {
    // cycle.cpp:142-152 validation order: tol, n_r (finite source: in run)
    require(cfg->tol > 0.0, SGML_EINVAL, "solve: tol must be positive");
    require(cfg->n_r >= 1, SGML_EINVAL, "solve: n_r must be >= 1");
}

}  // namespace

extern "C" {

int sgml_solve(sgml_ctx* ctx, int dim, int n, const sgml_bc* bc, const double* f_host,
               const double* sigma_host, double a, const sgml_solver_cfg* cfg,
               const sgml_solver_opts* opts, double* u_host_out, sgml_report* rep) {
    return guarded([&] {
        require(ctx && bc && f_host && cfg && rep, SGML_EINVAL, "solve: null argument");
        const sgml_grid g = make_grid_or_throw(dim, n);
        activate(ctx);
        check_solve_args(cfg);
        sgml_solver_opts o{};
        if (opts) o = *opts;
        std::lock_guard<std::recursive_mutex> lock(ctx->mu);
        sgml_solver* sv = cached_solver(ctx, dim, n, bc, sigma_host, a, cfg, o);
        const size_t bytes = g.total * sizeof(double);
        copy_h2d(ctx, sv->fin, f_host, bytes);  // (pageable sources at pinned speed)
        sv->run(sv->fin, nullptr, rep);
        if (u_host_out) copy_d2h(ctx, u_host_out, sv->result(), bytes);
        SGML_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int sgml_solve_many(sgml_ctx* ctx, int dim, int n, const sgml_bc* bc, int count, const double* const* f_hosts,
                    const double* sigma_host, double a, const sgml_solver_cfg* cfg,
                    const sgml_solver_opts* opts, double* const* u_hosts, sgml_report* reps) {
    return guarded([&] {
        require(ctx && bc && f_hosts && cfg && reps && count >= 0, SGML_EINVAL, "solve: null argument");
        const sgml_grid g = make_grid_or_throw(dim, n);
        activate(ctx);
        const cudaStream_t s = ctx->stream;
        check_solve_args(cfg);
        sgml_solver_opts o{};
        if (opts) o = *opts;
        std::lock_guard<std::recursive_mutex> lock(ctx->mu);
        sgml_solver* sv = cached_solver(ctx, dim, n, bc, sigma_host, a, cfg, o);
        if (count == 0) return;
        const size_t bytes = g.total * sizeof(double);
        // double-buffered staging: the copy stream moves solve k+1's source in
        // and solve k-1's solution out while solve k runs
        if (!sv->fin2) sv->fin2 = sv->alloc(g.total);
        for (int b = 0; b < 2; ++b)
            if (!sv->uout[b]) sv->uout[b] = sv->alloc(g.total);
        cudaStream_t cs = nullptr;
        cudaEvent_t in_ready[2] = {nullptr, nullptr}, out_ready[2] = {nullptr, nullptr}, out_done[2] = {nullptr, nullptr};
        struct Cleanup {
            cudaStream_t* cs;
            cudaEvent_t* ev[3];
            ~Cleanup() {
                if (*cs) {
                    cudaStreamSynchronize(*cs);
                    cudaStreamDestroy(*cs);
                }
                for (auto* e : ev)
                    for (int b = 0; b < 2; ++b)
                        if (e[b]) cudaEventDestroy(e[b]);
            }
        } cleanup{&cs, {in_ready, out_ready, out_done}};
        SGML_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            SGML_CUDA(cudaEventCreateWithFlags(&in_ready[b], cudaEventDisableTiming));
            SGML_CUDA(cudaEventCreateWithFlags(&out_ready[b], cudaEventDisableTiming));
            SGML_CUDA(cudaEventCreateWithFlags(&out_done[b], cudaEventDisableTiming));
        }
        double* fin[2] = {sv->fin, sv->fin2};
        auto stage_in = [&](int k) {
            SGML_CUDA(cudaMemcpyAsync(fin[k & 1], f_hosts[k], bytes, cudaMemcpyHostToDevice, cs));
            SGML_CUDA(cudaEventRecord(in_ready[k & 1], cs));
        };
        stage_in(0);
        for (int k = 0; k < count; ++k) {
            const int b = k & 1;
            // (solve k-1 finished reading fin[b ^ 1] before run returned)
            if (k + 1 < count) stage_in(k + 1);
            SGML_CUDA(cudaStreamWaitEvent(s, in_ready[b], 0));
            if (k >= 2) SGML_CUDA(cudaStreamWaitEvent(s, out_done[b], 0));  // uout[b] drained
            sv->run(fin[b], sv->uout[b], &reps[k]);
            SGML_CUDA(cudaEventRecord(out_ready[b], s));
            if (u_hosts && u_hosts[k]) {
                SGML_CUDA(cudaStreamWaitEvent(cs, out_ready[b], 0));
                SGML_CUDA(cudaMemcpyAsync(u_hosts[k], sv->uout[b], bytes, cudaMemcpyDeviceToHost, cs));
            }
            SGML_CUDA(cudaEventRecord(out_done[b], cs));
        }
        SGML_CUDA(cudaStreamSynchronize(cs));
        SGML_CUDA(cudaStreamSynchronize(s));
    });
}

int sgml_host_alloc(uint64_t bytes, void** out) {
    return guarded([&] {
        require(out != nullptr, SGML_EINVAL, "host_alloc: null out");
        SGML_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
    });
}

int sgml_host_free(void* p) {
    return guarded([&] {
        if (p) SGML_CUDA(cudaFreeHost(p));
    });
}

// ---- post-solve fields (problems.hpp:100-148) --------------------------------

int sgml_axis_derivative(const sgml_field* u, int axis, sgml_field* out) {
    return guarded([&] {
        same_grid(u, out, "axis_derivative: grid mismatch");
        require(axis >= 0 && axis < u->grid.dim, SGML_EINVAL, "axis_derivative: axis out of range");
        activate(u->ctx);
        const sgml_grid& g = u->grid;
        launch_axis_derivative(g.dim, u->d, out->d, g.N, axis, inv2h_of(g), u->ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(u->ctx->stream));
    });
}

int sgml_gradient(const sgml_field* u, sgml_field* const* out) {
    return guarded([&] {
        require(u && out, SGML_EINVAL, "gradient: null argument");
        const sgml_grid& g = u->grid;
        double* o[3] = {nullptr, nullptr, nullptr};
        for (int c = 0; c < g.dim; ++c) {
            same_grid(u, out[c], "gradient: grid mismatch");
            o[c] = out[c]->d;
        }
        activate(u->ctx);
        launch_gradient(g.dim, u->d, o, g.N, inv2h_of(g), nullptr, 0.0, 0.0, nullptr, u->ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(u->ctx->stream));
    });
}

int sgml_curl(const sgml_field* const* psi, sgml_field* const* out) {
    return guarded([&] {
        require(psi && out && psi[0], SGML_EINVAL, "curl: null argument");
        const sgml_grid& g = psi[0]->grid;
        require(g.dim == 3, SGML_EINVAL, "curl: defined for 3D fields");
        const double* p[3];
        double* o[3];
        for (int c = 0; c < 3; ++c) {
            same_grid(psi[0], psi[c], "curl: grid mismatch");
            same_grid(psi[0], out[c], "curl: grid mismatch");
            p[c] = psi[c]->d;
            o[c] = out[c]->d;
        }
        activate(psi[0]->ctx);
        launch_curl(p, o, g.N, inv2h_of(g), psi[0]->ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(psi[0]->ctx->stream));
    });
}

int sgml_divergence(const sgml_field* const* v, sgml_field* out) {
    return guarded([&] {
        require(v && out && v[0], SGML_EINVAL, "divergence: null argument");
        const sgml_grid& g = out->grid;
        const double* p[3] = {nullptr, nullptr, nullptr};
        for (int c = 0; c < g.dim; ++c) {
            same_grid(out, v[c], "divergence: grid mismatch");
            p[c] = v[c]->d;
        }
        activate(out->ctx);
        launch_divergence(g.dim, p, out->d, g.N, inv2h_of(g), out->ctx->stream);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(out->ctx->stream));
    });
}

int sgml_deformation_velocity(const sgml_field* u, const sgml_field* f_raw, double raw_integral, double t,
                              sgml_field* const* out) {
    return guarded([&] {
        require(u && f_raw && out, SGML_EINVAL, "deformation_velocity: null argument");
        same_grid(u, f_raw, "deformation_velocity: grid mismatch");
        const sgml_grid& g = u->grid;
        double* o[3] = {nullptr, nullptr, nullptr};
        for (int c = 0; c < g.dim; ++c) {
            same_grid(u, out[c], "deformation_velocity: grid mismatch");
            o[c] = out[c]->d;
        }
        sgml_ctx* ctx = u->ctx;
        activate(ctx);
        CtxLock lk(ctx->mu);
        const cudaStream_t s = ctx->stream;
        SGML_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), s));
        launch_gradient(g.dim, u->d, o, g.N, inv2h_of(g), f_raw->d, raw_integral, t, ctx->d_flags, s);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
        if (ctx->h_flags[0]) fail(SGML_EINVAL, "deformation_velocity: zero denominator");
    });
}

int sgml_move_nodes(const sgml_field* u, const sgml_field* f_raw, double raw_integral, double t, int steps,
                    sgml_field* const* pos) {
    return guarded([&] {
        require(u && f_raw && pos, SGML_EINVAL, "move_nodes: null argument");
        if (steps < 1) fail(SGML_EINVAL, "move_nodes: steps must be >= 1");
        same_grid(u, f_raw, "move_nodes: grid mismatch");
        const sgml_grid& g = u->grid;
        double* o[3] = {nullptr, nullptr, nullptr};
        for (int c = 0; c < 3; ++c) {
            if (c >= g.dim && !pos[c]) continue;
            same_grid(u, pos[c], "move_nodes: grid mismatch");
            o[c] = pos[c]->d;
        }
        sgml_ctx* ctx = u->ctx;
        activate(ctx);
        const cudaStream_t s = ctx->stream;
        // grad(u) on the full grid first (problems.cpp:347)
        DevBuf gb((size_t)g.dim * g.total * sizeof(double));
        double* gr[3] = {gb.d(), gb.d() + g.total, g.dim == 3 ? gb.d() + 2 * g.total : nullptr};
        launch_gradient(g.dim, u->d, gr, g.N, inv2h_of(g), nullptr, 0.0, 0.0, nullptr, s);
        if (g.dim == 2 && o[2]) SGML_CUDA(cudaMemsetAsync(o[2], 0, g.total * sizeof(double), s));
        launch_move_nodes(g.dim, gr, f_raw->d, raw_integral, g.N, g.h, t, steps, o, s);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaStreamSynchronize(s));
    });
}

int sgml_sample_vector(const sgml_field* const* v, int nv, const double* points, int count, double* out) {
    return guarded([&] {
        require(v && v[0] && points && out && count >= 0, SGML_EINVAL, "sample_vector: bad argument");
        require(nv >= 1 && nv <= 3, SGML_EINVAL, "sample_vector: 1..3 components");
        const sgml_grid& g = v[0]->grid;
        const double* p[3] = {nullptr, nullptr, nullptr};
        for (int c = 0; c < nv; ++c) {
            same_grid(v[0], v[c], "sample_vector: grid mismatch");
            p[c] = v[c]->d;
        }
        if (count == 0) return;
        sgml_ctx* ctx = v[0]->ctx;
        activate(ctx);
        const cudaStream_t s = ctx->stream;
        DevBuf pin((size_t)count * 3 * sizeof(double)), po((size_t)count * 3 * sizeof(double));
        SGML_CUDA(cudaMemcpyAsync(pin.p, points, (size_t)count * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        launch_sample_points(g.dim, p, nv, g.N, g.h, pin.d(), count, po.d(), s);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaMemcpyAsync(out, po.p, (size_t)count * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
    });
}

int sgml_integrate_streamlines(const sgml_field* const* v, const double* seeds, int nseeds, double step,
                               int max_steps, double* points, int* counts, int* stops) {
    return guarded([&] {
        require(v && v[0] && seeds && points && counts && stops, SGML_EINVAL, "integrate_streamline: null argument");
        if (!(step > 0.0)) fail(SGML_EINVAL, "integrate_streamline: step must be positive");
        require(nseeds >= 0 && max_steps >= 0, SGML_EINVAL, "integrate_streamline: bad sizes");
        const sgml_grid& g = v[0]->grid;
        const double* p[3] = {nullptr, nullptr, nullptr};
        for (int c = 0; c < g.dim; ++c) {
            same_grid(v[0], v[c], "integrate_streamline: grid mismatch");
            p[c] = v[c]->d;
        }
        if (nseeds == 0) return;
        sgml_ctx* ctx = v[0]->ctx;
        activate(ctx);
        const cudaStream_t s = ctx->stream;
        const size_t npts = (size_t)nseeds * (size_t)(max_steps + 1) * 3;
        DevBuf sd((size_t)nseeds * 3 * sizeof(double)), pts(npts * sizeof(double)),
            ci((size_t)nseeds * sizeof(int)), si((size_t)nseeds * sizeof(int));
        SGML_CUDA(cudaMemcpyAsync(sd.p, seeds, (size_t)nseeds * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        launch_streamlines(g.dim, p, g.N, g.h, sd.d(), nseeds, step, max_steps, pts.d(), ci.i(), si.i(), s);
        SGML_CUDA(cudaGetLastError());
        SGML_CUDA(cudaMemcpyAsync(points, pts.p, npts * sizeof(double), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaMemcpyAsync(counts, ci.p, (size_t)nseeds * sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaMemcpyAsync(stops, si.p, (size_t)nseeds * sizeof(int), cudaMemcpyDeviceToHost, s));
        SGML_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
