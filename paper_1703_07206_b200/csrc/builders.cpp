// builders.cpp — the reference's problem builders with the fields assembled
// on the device (problems.cpp:100-325, 374-398,
// 500-521).
//
// What stays on the host is exactly what must: the libm calls (sin, cos,
// tanh), whose bits a device implementation cannot reproduce, evaluated on
// their few distinct arguments (one coordinate for the manufactured sines,
// the integer m = |x - c|^2 / h^2 for the capacitor's tanh), and the curve
// work (a few thousand samples: resampling, arc elements, hat weights, the
// per-node sums in the reference's sample order).  The dense fields are
// never built on the host: the device fills them from the tables, or
// scatters the sparse deposits into a zeroed field.
#include <algorithm>
#include <array>
#include <cmath>
#include <stdexcept>
#include <unordered_map>
#include <vector>

#include "engine.hpp"

using namespace sgmlb;

namespace {

constexpr double kPi = 0x1.921fb54442d18p+1;  // std::numbers::pi_v<double>
using Point = std::array<double, 3>;

void need(bool ok, const char* msg) {
    if (!ok) fail(SGML_EINVAL, msg);
}

// device copy of a small host table, freed on scope exit
struct DevTable {
    void* p = nullptr;
    DevTable(const void* host, size_t bytes, cudaStream_t s) {
        SGML_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
        SGML_CUDA(cudaMemcpyAsync(p, host, bytes, cudaMemcpyHostToDevice, s));
    }
    ~DevTable() {
        if (p) cudaFree(p);
    }
    DevTable(const DevTable&) = delete;
    DevTable& operator=(const DevTable&) = delete;
};

void finish(sgml_ctx* ctx) {
    SGML_CUDA(cudaGetLastError());
    SGML_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ---- curves (problems.cpp:20-28, 100-140, 217-300) --------------------------

Point sub(const Point& a, const Point& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
Point add_scaled(const Point& a, double s, const Point& b) { return {a[0] + s * b[0], a[1] + s * b[1], a[2] + s * b[2]}; }
double norm(const Point& a) { return std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

struct Curve {
    std::vector<Point> points, payload;
    bool closed = false;
};

Curve resample_curve(const Curve& curve, double h) {
    const std::size_t m_in = curve.points.size();
    need(m_in >= 2, "resample_curve: need at least 2 points");
    need(h > 0.0, "resample_curve: spacing must be positive");
    const std::size_t segs = curve.closed ? m_in : m_in - 1;
    std::vector<double> cum(segs + 1, 0.0);
    for (std::size_t s = 0; s < segs; ++s)
        cum[s + 1] = cum[s] + norm(sub(curve.points[(s + 1) % m_in], curve.points[s]));
    const double length = cum[segs];
    need(length > 0.0, "resample_curve: curve has zero length");
    const std::size_t m = static_cast<std::size_t>(std::max<long long>(1, std::llround(length / h)));
    const double ds = length / static_cast<double>(m);
    const std::size_t count = curve.closed ? m : m + 1;
    Curve out;
    out.closed = curve.closed;
    std::size_t seg = 0;
    for (std::size_t i = 0; i < count; ++i) {
        const double s = std::min(static_cast<double>(i) * ds, length);
        while (seg + 1 < segs && cum[seg + 1] < s) ++seg;
        const double seg_len = cum[seg + 1] - cum[seg];
        const double t = seg_len > 0.0 ? (s - cum[seg]) / seg_len : 0.0;
        const Point& a = curve.points[seg % m_in];
        const Point& b = curve.points[(seg + 1) % m_in];
        out.points.push_back(add_scaled(a, t, sub(b, a)));
    }
    if (!curve.payload.empty()) {
        const std::size_t mo = out.points.size();
        out.payload.resize(mo);
        for (std::size_t i = 0; i < mo; ++i) {
            Point d;
            if (curve.closed) d = sub(out.points[(i + 1) % mo], out.points[(i + mo - 1) % mo]);
            else if (i == 0) d = sub(out.points[1], out.points[0]);
            else if (i == mo - 1) d = sub(out.points[mo - 1], out.points[mo - 2]);
            else d = sub(out.points[i + 1], out.points[i - 1]);
            const double len = norm(d);
            need(len > 0.0, "resample_curve: degenerate tangent");
            out.payload[i] = {d[0] / len, d[1] / len, d[2] / len};
        }
    }
    return out;
}

std::vector<double> arc_elements(const Curve& curve) {
    const std::size_t m = curve.points.size();
    std::vector<double> ds(m, 0.0);
    const std::size_t segs = curve.closed ? m : m - 1;
    for (std::size_t s = 0; s < segs; ++s) {
        const double len = norm(sub(curve.points[(s + 1) % m], curve.points[s]));
        ds[s] += 0.5 * len;
        ds[(s + 1) % m] += 0.5 * len;
    }
    return ds;
}

// sparse field: per-node sums in first-touch order (each node's terms are
// added in the reference's sample order, starting from 0.0 like the dense field)
struct Sparse {
    std::unordered_map<unsigned long long, std::size_t> at;
    std::vector<unsigned long long> idx;
    std::vector<double> val;
    double& operator[](unsigned long long p) {
        auto it = at.find(p);
        if (it == at.end()) {
            it = at.emplace(p, idx.size()).first;
            idx.push_back(p);
            val.push_back(0.0);
        }
        return val[it->second];
    }
};

template <typename Deposit>
void scatter_mass(const Point& p, const sgml_grid& g, Deposit&& into) {
    int idx[3] = {0, 0, 0};
    double frac[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < g.dim; ++c) {
        const double x = p[c];
        need(x >= 0.0 && x <= 1.0, "deposit_delta: curve sample outside the unit domain");
        int i0 = static_cast<int>(std::floor(x / g.h));
        i0 = std::clamp(i0, 0, g.N - 2);
        idx[c] = i0;
        frac[c] = x / g.h - i0;
    }
    const double inv_hd = g.dim == 2 ? 1.0 / (g.h * g.h) : 1.0 / (g.h * g.h * g.h);
    const double wx[2] = {1.0 - frac[0], frac[0]};
    const double wy[2] = {1.0 - frac[1], frac[1]};
    const unsigned long long N = (unsigned long long)g.N;
    auto lin = [&](int a, int b, int c) { return (unsigned long long)a + N * ((unsigned long long)b + N * (unsigned long long)c); };
    if (g.dim == 2) {
        for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) into(lin(idx[0] + a, idx[1] + b, 0), wx[a] * wy[b] * inv_hd);
    } else {
        const double wz[2] = {1.0 - frac[2], frac[2]};
        for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    into(lin(idx[0] + a, idx[1] + b, idx[2] + c), wx[a] * wy[b] * wz[c] * inv_hd);
    }
}

bool inside_unit(const Point& p, int dim) {
    for (int c = 0; c < dim; ++c)
        if (!(p[c] >= 0.0 && p[c] <= 1.0)) return false;
    return true;
}

// zero-fill (or fill with `z`) a device field and scatter a sparse field into it
void upload_sparse(sgml_field* f, const Sparse& sp, double z, bool negate) {
    sgml_ctx* ctx = f->ctx;
    const cudaStream_t s = ctx->stream;
    launch_fill(f->d, f->grid.total, z, s);
    std::vector<double> v = sp.val;
    if (negate)
        for (double& x : v) x = -x;
    if (sp.idx.empty()) return;
    DevTable di(sp.idx.data(), sp.idx.size() * sizeof(unsigned long long), s);
    DevTable dv(v.data(), v.size() * sizeof(double), s);
    launch_scatter_pairs(f->d, static_cast<const unsigned long long*>(di.p), static_cast<const double*>(dv.p),
                         (int)sp.idx.size(), s);
    finish(ctx);
}

Curve curve_of(const double* pts, const double* payload, int npts, bool closed) {
    Curve c;
    c.closed = closed;
    for (int q = 0; q < npts; ++q) {
        c.points.push_back({pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]});
        if (payload) c.payload.push_back({payload[3 * q], payload[3 * q + 1], payload[3 * q + 2]});
    }
    return c;
}

void emit_curve(const Curve& c, double* pts, double* payload, int cap, int* count) {
    const std::size_t m = c.points.size();
    need(m <= 0x7fffffff, "resample_curve: too many samples");
    *count = (int)m;
    for (std::size_t i = 0; i < m && (long long)i < cap; ++i)
        for (int k = 0; k < 3; ++k) {
            if (pts) pts[3 * i + k] = c.points[i][k];
            if (payload && !c.payload.empty()) payload[3 * i + k] = c.payload[i][k];
        }
}

// problems.cpp:282-291: strength * ds per sample, summed per node in sample order
Sparse deposit_scalar(const Curve& curve, const sgml_grid& g, double strength) {
    need(curve.points.size() >= 2, "deposit_delta: need at least 2 points");
    const std::vector<double> ds = arc_elements(curve);
    Sparse out;
    for (std::size_t i = 0; i < curve.points.size(); ++i) {
        const double mass = strength * ds[i];
        scatter_mass(curve.points[i], g, [&](unsigned long long p, double w) { out[p] += mass * w; });
    }
    return out;
}

// problems.cpp:293-302: payload_c * ds * w into the three components
void deposit_vector(const Curve& curve, const sgml_grid& g, Sparse* w3) {
    need(curve.payload.size() == curve.points.size(), "deposit_delta_vector: curve carries no payload");
    const std::vector<double> ds = arc_elements(curve);
    for (std::size_t i = 0; i < curve.points.size(); ++i) {
        const Point& pay = curve.payload[i];
        scatter_mass(curve.points[i], g, [&](unsigned long long p, double w) {
            for (int comp = 0; comp < 3; ++comp) w3[comp][p] += pay[comp] * ds[i] * w;
        });
    }
}

// problems.cpp:374-398: the overhand knot, 512 samples, resampled at h with unit tangents
Curve trifoil_curve(double r, double h) {
    need(r > 0.0, "trifoil_problem: r must be positive");
    Curve raw;
    raw.closed = true;
    const int samples = 512;
    raw.payload.resize(samples);
    for (int s = 0; s < samples; ++s) {
        const double t = 2.0 * kPi * s / samples;
        raw.points.push_back({0.5 + r * (std::sin(t) + 2.0 * std::sin(2.0 * t)),
                              0.5 + r * (std::cos(t) - 2.0 * std::cos(2.0 * t)), 0.5 - r * std::sin(3.0 * t)});
    }
    for (const Point& p : raw.points)
        need(inside_unit(p, 3), "trifoil_problem: curve leaves the unit domain (max extent 3r)");
    return resample_curve(raw, h);
}

}  // namespace

extern "C" {

int sgml_build_poisson2d_source(sgml_field* f) {
    return guarded([&] {
        need(f && f->grid.dim == 2, "poisson2d_problem: a 2D field is required");
        SGML_CUDA(cudaSetDevice(f->ctx->device));
        launch_fill_poisson2d(f->d, f->grid.N, f->grid.h, f->ctx->stream);
        finish(f->ctx);
    });
}

int sgml_build_poisson3d_source(sgml_field* f) {
    return guarded([&] {
        need(f && f->grid.dim == 3, "poisson3d_problem: a 3D field is required");
        SGML_CUDA(cudaSetDevice(f->ctx->device));
        const int N = f->grid.N;
        std::vector<double> s(N);
        for (int i = 0; i < N; ++i) s[i] = std::sin(kPi * (i * f->grid.h));  // exact(x) factors
        DevTable t(s.data(), N * sizeof(double), f->ctx->stream);
        launch_fill_poisson3d(f->d, N, static_cast<const double*>(t.p), -3.0 * kPi * kPi, f->ctx->stream);
        finish(f->ctx);
    });
}

int sgml_build_sinsin2d_source(sgml_field* f) {
    return guarded([&] {
        need(f && f->grid.dim == 2, "sinsin2d: a 2D field is required");
        SGML_CUDA(cudaSetDevice(f->ctx->device));
        const int N = f->grid.N;
        std::vector<double> s(N);
        for (int i = 0; i < N; ++i) s[i] = std::sin(kPi * (i * f->grid.h));
        DevTable t(s.data(), N * sizeof(double), f->ctx->stream);
        launch_fill_sinsin2d(f->d, N, static_cast<const double*>(t.p), -2.0 * kPi * kPi, f->ctx->stream);
        finish(f->ctx);
    });
}

int sgml_build_capacitor_sigma(sgml_field* sigma, int high) {
    return guarded([&] {
        need(sigma && sigma->grid.dim == 3, "capacitor_problem: a 3D field is required");
        SGML_CUDA(cudaSetDevice(sigma->ctx->device));
        const sgml_grid& g = sigma->grid;
        const double sign = high ? -1.0 : 1.0;
        // r = sqrt(sq(i h - 0.5) + sq(j h - 0.5) + sq(k h - 0.5)): every step is
        // exact for h = 2^-n, so r depends on m = di^2 + dj^2 + dk^2 only
        const long long c = (g.N - 1) / 2, mmax = 3 * c * c;
        std::vector<double> table((size_t)mmax + 1);
        for (long long m = 0; m <= mmax; ++m) {
            const double r = std::sqrt((double)m * g.h * g.h);
            table[(size_t)m] = 0.55 + sign * 0.45 * std::tanh((r - 0.2) / 0.1);
        }
        DevTable t(table.data(), table.size() * sizeof(double), sigma->ctx->stream);
        launch_fill_radial(sigma->d, g.N, static_cast<const double*>(t.p), sigma->ctx->stream);
        finish(sigma->ctx);
    });
}

int sgml_build_trifoil_sources(sgml_field* const* f3, double r) {
    return guarded([&] {
        need(f3 && f3[0] && f3[1] && f3[2], "trifoil_problem: three source fields are required");
        const sgml_grid g = f3[0]->grid;
        need(g.dim == 3, "trifoil_problem: 3D fields are required");
        for (int c = 1; c < 3; ++c)
            need(f3[c]->grid.dim == 3 && f3[c]->grid.n == g.n, "trifoil_problem: grid mismatch");
        SGML_CUDA(cudaSetDevice(f3[0]->ctx->device));
        const Curve curve = trifoil_curve(r, g.h);
        Sparse omega[3];
        deposit_vector(curve, g, omega);
        // psi_c's source is -omega_c over the whole field (-0.0 away from the curve)
        for (int comp = 0; comp < 3; ++comp) upload_sparse(f3[comp], omega[comp], -0.0, true);
        finish(f3[0]->ctx);
    });
}

int sgml_build_deformation_problem(const double* points, int npts, int closed, int with_payload, sgml_field* f,
                                   sgml_field* f_raw, double* raw_integral) {
    return guarded([&] {
        need(points && npts >= 0 && f && f_raw && raw_integral, "deformation_problem: bad arguments");
        Curve curve = curve_of(points, nullptr, npts, closed);
        if (with_payload) curve.payload.assign(curve.points.size(), Point{0.0, 0.0, 0.0});
        int dim = 2;
        for (const Point& p : curve.points)
            if (p[2] != 0.0) dim = 3;
        const sgml_grid g = f->grid;
        need(g.dim == dim && f_raw->grid.dim == dim && f_raw->grid.n == g.n,
             "deformation_problem: field grids must match the curve's dimension");
        sgml_ctx* ctx = f->ctx;
        SGML_CUDA(cudaSetDevice(ctx->device));
        const Curve rs = resample_curve(curve, g.h);
        upload_sparse(f_raw, deposit_scalar(rs, g, 1.0), 0.0, false);  // strength 1 (problems.cpp:309)
        // raw_integral = trapezoid_mean(f_raw); f = f_raw projected to zero mean
        *raw_integral = trapezoid_mean_host(ctx, g, f_raw->d);
        SGML_CUDA(cudaMemcpyAsync(f->d, f_raw->d, g.total * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        const double mean = trapezoid_mean_host(ctx, g, f->d);
        launch_sub_scalar(f->d, g.total, mean, ctx->stream);
        finish(ctx);
    });
}

int sgml_build_deformation_sources(const double* points, int npts, sgml_field* f, sgml_field* f_raw,
                                   double* raw_integral) {
    return sgml_build_deformation_problem(points, npts, 1, 0, f, f_raw, raw_integral);
}

int sgml_resample_curve(const double* points, int npts, int closed, int with_payload, double h, double* out_points,
                        double* out_payload, int cap, int* count) {
    return guarded([&] {
        need(points && npts >= 0 && count && cap >= 0, "resample_curve: bad arguments");
        Curve c = curve_of(points, nullptr, npts, closed);
        if (with_payload) c.payload.assign(c.points.size(), Point{0.0, 0.0, 0.0});
        emit_curve(resample_curve(c, h), out_points, with_payload ? out_payload : nullptr, cap, count);
    });
}

int sgml_deposit_delta(const double* points, int npts, int closed, double strength, sgml_field* f) {
    return guarded([&] {
        need(points && f, "deposit_delta: bad arguments");
        need(npts >= 2, "deposit_delta: need at least 2 points");
        SGML_CUDA(cudaSetDevice(f->ctx->device));
        upload_sparse(f, deposit_scalar(curve_of(points, nullptr, npts, closed), f->grid, strength), 0.0, false);
        finish(f->ctx);
    });
}

int sgml_deposit_delta_vector(const double* points, const double* payload, int npts, int closed,
                              sgml_field* const* f3) {
    return guarded([&] {
        need(points && f3 && f3[0] && f3[1] && f3[2], "deposit_delta_vector: bad arguments");
        need(payload != nullptr, "deposit_delta_vector: curve carries no payload");
        const sgml_grid g = f3[0]->grid;
        for (int c = 1; c < 3; ++c)
            need(f3[c]->grid.dim == g.dim && f3[c]->grid.n == g.n, "deposit_delta_vector: grid mismatch");
        SGML_CUDA(cudaSetDevice(f3[0]->ctx->device));
        Sparse w[3];
        deposit_vector(curve_of(points, payload, npts, closed), g, w);
        for (int comp = 0; comp < 3; ++comp) upload_sparse(f3[comp], w[comp], 0.0, false);
        finish(f3[0]->ctx);
    });
}

int sgml_trifoil_curve(double r, double h, double* out_points, double* out_payload, int cap, int* count) {
    return guarded([&] {
        need(count && cap >= 0, "trifoil_problem: bad arguments");
        emit_curve(trifoil_curve(r, h), out_points, out_payload, cap, count);
    });
}

}  // extern "C"
