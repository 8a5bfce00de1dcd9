// Shared host-side helpers: thread-local error text and status plumbing.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/seqcfr_b200.h"

namespace scfr {

// Carries a SCFR_E* code through C++ code; converted at the C-ABI edge.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Error(code, buf);
}

// Runs `body` and maps exceptions onto the ABI's int status.
template <class F>
int guarded(F&& body) {
    try {
        body();
        return SCFR_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return SCFR_ENOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SCFR_EINVAL;
    }
}

}  // namespace scfr
