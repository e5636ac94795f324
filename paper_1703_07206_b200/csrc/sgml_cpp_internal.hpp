// sgml_cpp_internal.hpp — helpers shared by the C++ mirror of the reference
// API (sgml_cpp.cpp, sgml_cpp_more.cpp): status -> reference exception,
// the process-wide device context, host <-> device field copies.
#pragma once

#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/sgml/grid.hpp"
#include "../../include/sgml/kernels.hpp"
#include "../../include/sgml_b200.h"

namespace sgml {
namespace cabi {

inline void check(int status) {
    if (status == SGML_OK) return;
    const std::string msg = sgml_last_error();
    switch (status) {
        case SGML_EINVAL: throw std::invalid_argument(msg);
        case SGML_EBADSTEP:
        case SGML_ENONFINITE: throw kernel_error(msg);
        case SGML_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

// One context per process on SGML_DEVICE (default 0), created on first use.
inline sgml_ctx* context() {
    static std::once_flag once;
    static sgml_ctx* ctx = nullptr;
    std::call_once(once, [] {
        const char* d = std::getenv("SGML_DEVICE");
        check(sgml_ctx_create(d ? std::atoi(d) : 0, &ctx));
    });
    return ctx;
}

inline sgml_bc to_c(const BoundarySpec& bc) {
    sgml_bc b{};
    for (int f = 0; f < 6; ++f) {
        b.kind[f] = bc.faces[f].kind == BcKind::neumann ? 1 : 0;
        b.value[f] = bc.faces[f].value;
    }
    return b;
}

// device copy of a host field for the duration of one call
struct Dev {
    sgml_field* f = nullptr;
    explicit Dev(const Grid& g) { check(sgml_field_create(context(), g.dim, g.n, &f)); }
    Dev(const Field& h) : Dev(h.grid()) { check(sgml_field_upload(f, h.data())); }
    ~Dev() { sgml_field_destroy(f); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    void to(Field& h) const { check(sgml_field_download(f, h.data())); }
};

}  // namespace cabi
}  // namespace sgml
