// common.cuh -- shared helpers for libgcharm (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>

#include "../../include/gcharm.h"

namespace gc {

// thread-local last error message (gc_last_error)
void set_error(const std::string &msg);

struct Error {
    gc_status code;
    std::string msg;
};

#define GC_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t _e = (call);                                                               \
        if (_e != cudaSuccess)                                                                 \
            throw ::gc::Error{GC_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)};  \
    } while (0)

#define GC_REQUIRE(cond, code, msg)                                                            \
    do {                                                                                       \
        if (!(cond)) throw ::gc::Error{(code), (msg)};                                         \
    } while (0)

// Wrap a C-ABI body: exceptions -> status codes.
template <class F>
gc_status guard(F &&f)
{
    try {
        f();
        return GC_OK;
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc &) {
        set_error("host allocation failed");
        return GC_E_NOMEM;
    } catch (const std::exception &e) {
        set_error(e.what());
        return GC_E_VALUE;
    }
}

// Simple owning device buffer.
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    size_t cap = 0;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    ~DBuf() { release(); }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = cap = 0;
    }
    // grow-only: keeps the allocation when it is large enough
    void resize(size_t count)
    {
        if (count > cap) {
            release();
            size_t c = count ? count : 1;
            GC_CUDA(cudaMalloc(&p, c * sizeof(T)));
            cap = c;
        }
        n = count;
    }
    // grow-only, keeping the first n elements (device-side copy on the stream)
    void grow(size_t count, cudaStream_t s)
    {
        if (count > cap) {
            T *q = nullptr;
            const size_t c = std::max(count, cap + cap / 2);
            GC_CUDA(cudaMalloc(&q, c * sizeof(T)));
            if (p && n) GC_CUDA(cudaMemcpyAsync(q, p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
            GC_CUDA(cudaStreamSynchronize(s));
            if (p) cudaFree(p);
            p = q;
            cap = c;
        }
        n = count;
    }
    void upload(const T *h, size_t count, cudaStream_t s)
    {
        resize(count);
        if (count) GC_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void download(T *h, size_t count, cudaStream_t s, size_t offset = 0) const
    {
        if (count) GC_CUDA(cudaMemcpyAsync(h, p + offset, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    void zero(cudaStream_t s)
    {
        if (n) GC_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

}  // namespace gc

struct gc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaDeviceProp prop{};
    gc::DBuf<unsigned char> scratch;  // cub temp storage
};

namespace gc {
inline void check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error{GC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }
}  // namespace gc
