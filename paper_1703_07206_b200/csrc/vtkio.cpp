// vtkio.cpp — the reference's legacy ASCII VTK writers (io.cpp:14-64) for
// device fields, streamed.  u.vtk at 1025^3 is ~20 GB
// of "%.17g" text; the reference formats it with one snprintf per value on
// one thread.  Here the field leaves the device in chunks through two pinned
// buffers (the copy of chunk q+1 overlaps the formatting of chunk q), each
// chunk is formatted by all host threads into per-thread text blocks with
// std::to_chars (general, precision 17: the same characters as "%.17g"),
// and the blocks are written in order.  The bytes equal the reference's
// writer output (tests/test_gpu_fields.py compares them).
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

using namespace sgmlb;

namespace {

// io.cpp:35-39 format_double: "%.17g"
inline char* fmt17(char* p, double x) {
    return std::to_chars(p, p + 32, x, std::chars_format::general, 17).ptr;
}

std::string fmt_str(double x) {
    char b[32];
    return std::string(b, fmt17(b, x));
}

// io.cpp:21-31
std::string vtk_header(const sgml_grid& g, const std::string& name) {
    std::string h = "# vtk DataFile Version 3.0\n" + name + "\nASCII\nDATASET STRUCTURED_POINTS\n";
    h += "DIMENSIONS " + std::to_string(g.N) + ' ' + std::to_string(g.N) + ' ' +
         std::to_string(g.dim == 3 ? g.N : 1) + '\n';
    h += "ORIGIN 0 0 0\n";
    h += "SPACING " + fmt_str(g.h) + ' ' + fmt_str(g.h) + ' ' + (g.dim == 3 ? fmt_str(g.h) : std::string("1")) +
         '\n';
    h += "POINT_DATA " + std::to_string(g.total) + '\n';
    return h;
}

struct File {
    std::FILE* f = nullptr;
    std::string path;
    explicit File(const std::string& p) : path(p) {
        f = std::fopen(p.c_str(), "wb");
        if (!f) fail(SGML_EIO, "cannot open for writing: " + p);
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void put(const char* s, size_t n) {
        if (n && std::fwrite(s, 1, n, f) != n) fail(SGML_EIO, "write failed: " + path);
    }
    void close() {
        if (std::fclose(f) != 0) {
            f = nullptr;
            fail(SGML_EIO, "write failed: " + path);
        }
        f = nullptr;
    }
};

// format rows of host arrays in parallel blocks, written in order
void format_block(const double* const* src, int ncomp, uint64_t lo, uint64_t hi, std::string& out) {
    out.resize((size_t)(hi - lo) * (size_t)ncomp * 26);
    char* p = out.data();
    for (uint64_t i = lo; i < hi; ++i)
        for (int c = 0; c < ncomp; ++c) {
            p = fmt17(p, src[c] ? src[c][i] : 0.0);
            *p++ = c + 1 < ncomp ? ' ' : '\n';
        }
    out.resize((size_t)(p - out.data()));
}

void format_rows(const double* const* comp, int ncomp, uint64_t total, File& out) {
    const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    constexpr uint64_t kChunk = uint64_t(1) << 22;
    std::vector<std::string> text(nth);
    for (uint64_t c0 = 0; c0 < total; c0 += kChunk) {
        const uint64_t cnt = std::min(kChunk, total - c0);
        const double* src[3] = {nullptr, nullptr, nullptr};
        for (int c = 0; c < ncomp; ++c) src[c] = comp[c] ? comp[c] + c0 : nullptr;
        auto work = [&](unsigned t) { format_block(src, ncomp, cnt * t / nth, cnt * (t + 1) / nth, text[t]); };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nth; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
        for (unsigned t = 0; t < nth; ++t) out.put(text[t].data(), text[t].size());
    }
}

// Stream ncomp device arrays (comp[c] == nullptr: zeros) as text rows of
// ncomp values ("a\n" or "a b c\n"); ctx == nullptr: the arrays are host
// memory (no copies).
void stream_rows(sgml_ctx* ctx, const double* const* comp, int ncomp, uint64_t total, File& out) {
    if (!ctx) {
        format_rows(comp, ncomp, total, out);
        return;
    }
    const cudaStream_t s = ctx->stream;
    constexpr uint64_t kChunk = uint64_t(1) << 22;  // nodes per chunk
    const uint64_t per = std::min<uint64_t>(kChunk, std::max<uint64_t>(total, 1));
    double* pin[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    struct Cleanup {
        double** pin;
        cudaEvent_t* ev;
        ~Cleanup() {
            for (int b = 0; b < 2; ++b) {
                if (pin[b]) cudaFreeHost(pin[b]);
                if (ev[b]) cudaEventDestroy(ev[b]);
            }
        }
    } cleanup{pin, ev};
    for (int b = 0; b < 2; ++b) {
        SGML_CUDA(cudaMallocHost((void**)&pin[b], per * ncomp * sizeof(double)));
        SGML_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    auto issue = [&](uint64_t c0, int b) {
        const uint64_t cnt = std::min(per, total - c0);
        for (int c = 0; c < ncomp; ++c) {
            if (comp[c])
                SGML_CUDA(cudaMemcpyAsync(pin[b] + c * per, comp[c] + c0, cnt * sizeof(double),
                                          cudaMemcpyDeviceToHost, s));
            else
                std::fill(pin[b] + c * per, pin[b] + c * per + cnt, 0.0);
        }
        SGML_CUDA(cudaEventRecord(ev[b], s));
    };
    const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::string> text(nth);
    if (total) issue(0, 0);
    for (uint64_t c0 = 0, q = 0; c0 < total; c0 += per, ++q) {
        const int b = (int)(q & 1);
        const uint64_t cnt = std::min(per, total - c0);
        SGML_CUDA(cudaEventSynchronize(ev[b]));
        if (c0 + per < total) issue(c0 + per, b ^ 1);
        const double* src = pin[b];
        auto work = [&](unsigned t) {
            const uint64_t lo = cnt * t / nth, hi = cnt * (t + 1) / nth;
            std::string& out = text[t];
            out.resize((hi - lo) * (size_t)ncomp * 26);
            char* p = out.data();
            for (uint64_t i = lo; i < hi; ++i)
                for (int c = 0; c < ncomp; ++c) {
                    p = fmt17(p, src[c * per + i]);
                    *p++ = c + 1 < ncomp ? ' ' : '\n';
                }
            out.resize((size_t)(p - out.data()));
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nth; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
        for (unsigned t = 0; t < nth; ++t) out.put(text[t].data(), text[t].size());
    }
}

}  // namespace

extern "C" {

// io.cpp:45-53 write_field_vtk
int sgml_write_field_vtk(const sgml_field* f, const char* path, const char* name) {
    return guarded([&] {
        if (!f || !path || !name) fail(SGML_EINVAL, "write_field_vtk: null argument");
        SGML_CUDA(cudaSetDevice(f->ctx->device));
        SGML_CUDA(cudaStreamSynchronize(f->ctx->stream));
        File out(path);
        const std::string head =
            vtk_header(f->grid, name) + "SCALARS " + name + " double 1\nLOOKUP_TABLE default\n";
        out.put(head.data(), head.size());
        const double* comp[1] = {f->d};
        stream_rows(f->ctx, comp, 1, f->grid.total, out);
        out.close();
    });
}

// io.cpp:55-64 write_vector_vtk: three values per node (v[2] may be null: zeros)
int sgml_write_vector_vtk(const sgml_field* const* v, const char* path, const char* name) {
    return guarded([&] {
        if (!v || !v[0] || !v[1] || !path || !name) fail(SGML_EINVAL, "write_vector_vtk: null argument");
        SGML_CUDA(cudaSetDevice(v[0]->ctx->device));
        SGML_CUDA(cudaStreamSynchronize(v[0]->ctx->stream));
        File out(path);
        const std::string head = vtk_header(v[0]->grid, name) + "VECTORS " + name + " double\n";
        out.put(head.data(), head.size());
        const double* comp[3] = {v[0]->d, v[1]->d, v[2] ? v[2]->d : nullptr};
        stream_rows(v[0]->ctx, comp, 3, v[0]->grid.total, out);
        out.close();
    });
}

// the same writers for host arrays (the command-line driver's fields)
int sgml_write_vtk_host(const double* const* comps, int ncomp, const sgml_grid* g, const char* path,
                        const char* name) {
    return guarded([&] {
        if (!comps || !comps[0] || !g || !path || !name || (ncomp != 1 && ncomp != 3))
            fail(SGML_EINVAL, "write_vtk_host: bad argument");
        File out(path);
        std::string head = vtk_header(*g, name);
        head += ncomp == 1 ? std::string("SCALARS ") + name + " double 1\nLOOKUP_TABLE default\n"
                           : std::string("VECTORS ") + name + " double\n";
        out.put(head.data(), head.size());
        stream_rows(nullptr, comps, ncomp, g->total, out);
        out.close();
    });
}

}  // extern "C"
