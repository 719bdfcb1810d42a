// Error convention of the C ABI: every entry point runs its
// body under guard(), which maps a thrown Failure to its status code and
// keeps the message for saap_last_error() (thread-local).
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "common.cuh"

namespace saap_b200 {

inline thread_local std::string g_err;

struct Failure {
    int code;
    std::string msg;
};

template <typename F>
int guard(F&& f) {
    try {
        f();
        return SAAP_OK;
    } catch (const Failure& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SAAP_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SAAP_ERR_CUDA;
    }
}

[[noreturn]] inline void invalid(const std::string& m) { throw Failure{SAAP_ERR_INVALID_ARGUMENT, m}; }
[[noreturn]] inline void unsupported(const std::string& m) { throw Failure{SAAP_ERR_UNSUPPORTED, m}; }

inline void need(const void* p, const char* what) {
    if (!p) invalid(std::string(what) + ": null argument");
}

struct DeviceGuard {
    explicit DeviceGuard(const saap_ctx* c) {
        if (!c) invalid("null context");
        SAAP_CUDA(cudaSetDevice(c->device));
    }
};

}  // namespace saap_b200
