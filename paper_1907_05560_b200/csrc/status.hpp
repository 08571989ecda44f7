// Error plumbing for the C-ABI: C++ exceptions stay inside the library and
// become an OscStatus + thread-local message (osc_last_error).
#pragma once

#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "oscflat_b200.h"

namespace oscb200 {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OSC_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return OSC_ERR_CUDA;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return OSC_ERR_CUDA;
    }
}

}  // namespace oscb200
