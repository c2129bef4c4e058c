// host_common.hpp — host-side error plumbing shared by the engine and the ABI.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "clo.h"

namespace clo {

// Exception carrying a clo_status; the ABI layer maps it to the return code
// (the reference's exception taxonomy, errors.hpp:10-41).
struct Error : std::runtime_error {
    clo_status status;
    Error(clo_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(clo_status s, const std::string& msg) { throw Error(s, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(CLO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CLO_CUDA(call) ::clo::cuda_check((call), #call)

void set_last_error(const std::string& msg);

template <class F>
clo_status guarded(F&& f) {
    try {
        f();
        return CLO_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return CLO_ERR_INTERNAL;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CLO_ERR_INTERNAL;
    }
}

// Device buffer owned by the engine.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void alloc(size_t n, bool zero = true) {
        reset();
        if (n == 0) return;
        CLO_CUDA(cudaMalloc(&p, n));
        bytes = n;
        if (zero) CLO_CUDA(cudaMemset(p, 0, n));
    }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// Host-side restatements that the engine needs (pure functions).
void sign_hash_projection(int hash_bits, int d, uint64_t seed, double* out);  // [bits][d]
uint64_t mix_seed3(uint64_t base, uint64_t a, uint64_t b);

}  // namespace clo
