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
        need(r > 0.0, "trifoil_problem: r must be positive");
        SGML_CUDA(cudaSetDevice(f3[0]->ctx->device));
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
        const Curve curve = resample_curve(raw, g.h);
        const std::vector<double> ds = arc_elements(curve);
        Sparse omega[3];
        for (std::size_t i = 0; i < curve.points.size(); ++i) {
            const Point& pay = curve.payload[i];
            scatter_mass(curve.points[i], g, [&](unsigned long long p, double w) {
                for (int comp = 0; comp < 3; ++comp) omega[comp][p] += pay[comp] * ds[i] * w;
            });
        }
        // psi_c's source is -omega_c over the whole field (-0.0 away from the curve)
        for (int comp = 0; comp < 3; ++comp) upload_sparse(f3[comp], omega[comp], -0.0, true);
        finish(f3[0]->ctx);
    });
}

int sgml_build_deformation_sources(const double* points, int npts, sgml_field* f, sgml_field* f_raw,
                                   double* raw_integral) {
    return guarded([&] {
        need(points && npts >= 2 && f && f_raw && raw_integral, "deformation_problem: bad arguments");
        Curve curve;
        curve.closed = true;
        int dim = 2;
        for (int q = 0; q < npts; ++q) {
            curve.points.push_back({points[3 * q], points[3 * q + 1], points[3 * q + 2]});
            if (points[3 * q + 2] != 0.0) dim = 3;
        }
        const sgml_grid g = f->grid;
        need(g.dim == dim && f_raw->grid.dim == dim && f_raw->grid.n == g.n,
             "deformation_problem: field grids must match the curve's dimension");
        sgml_ctx* ctx = f->ctx;
        SGML_CUDA(cudaSetDevice(ctx->device));
        const Curve rs = resample_curve(curve, g.h);
        const std::vector<double> ds = arc_elements(rs);
        Sparse raw;
        for (std::size_t i = 0; i < rs.points.size(); ++i) {
            const double mass = 1.0 * ds[i];  // strength 1 (problems.cpp:309)
            scatter_mass(rs.points[i], g, [&](unsigned long long p, double w) { raw[p] += mass * w; });
        }
        upload_sparse(f_raw, raw, 0.0, false);
        // raw_integral = trapezoid_mean(f_raw); f = f_raw projected to zero mean
        *raw_integral = trapezoid_mean_host(ctx, g, f_raw->d);
        SGML_CUDA(cudaMemcpyAsync(f->d, f_raw->d, g.total * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        const double mean = trapezoid_mean_host(ctx, g, f->d);
        launch_sub_scalar(f->d, g.total, mean, ctx->stream);
        finish(ctx);
    });
}

}  // extern "C"
