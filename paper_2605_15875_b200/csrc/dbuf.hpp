// Minimal owning device/pinned buffers and CUDA error plumbing for the host
// side of dabd_gpu. Errors become dabd_gpu::Error (mapped to
// DABD_GPU_ERR_RUNTIME by the C ABI, like proj/src/capi.cpp:20-34).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace dabd_gpu {

struct Error : std::runtime_error {
    explicit Error(const std::string& w) : std::runtime_error(w) {}
};

// A device-side error code (common.cuh DevError) raised by a kernel.
struct DeviceError : Error {
    int code;
    DeviceError(const std::string& w, int c) : Error(w), code(c) {}
};

struct InvalidArg : std::runtime_error {
    explicit InvalidArg(const std::string& w) : std::runtime_error(w) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CUDA_CHECK(x) ::dabd_gpu::cuda_check((x), #x)

template <typename T>
class DBuf {
  public:
    DBuf() = default;
    explicit DBuf(size_t n) { resize(n); }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), cap_(o.cap_) {
        o.p_ = nullptr;
        o.n_ = o.cap_ = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            cap_ = o.cap_;
            o.p_ = nullptr;
            o.n_ = o.cap_ = 0;
        }
        return *this;
    }
    // Grows capacity geometrically; contents are not preserved.
    void resize(size_t n) {
        if (n > cap_) {
            release();
            size_t c = cap_ == 0 ? n : std::max(n, cap_ + cap_ / 2);
            if (c == 0) c = 1;
            CUDA_CHECK(cudaMalloc(&p_, c * sizeof(T)));
            cap_ = c;
        }
        n_ = n;
    }
    void upload(const T* h, size_t n, cudaStream_t s) {
        resize(n);
        if (n) CUDA_CHECK(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
    void download(T* h, size_t n, cudaStream_t s) const {
        if (n) CUDA_CHECK(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    std::vector<T> to_host(cudaStream_t s) const {
        std::vector<T> h(n_);
        download(h.data(), n_, s);
        CUDA_CHECK(cudaStreamSynchronize(s));
        return h;
    }
    void zero(cudaStream_t s) {
        if (n_) CUDA_CHECK(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t capacity() const { return cap_; }

  private:
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        cap_ = 0;
        n_ = 0;
    }
    T* p_ = nullptr;
    size_t n_ = 0, cap_ = 0;
};

template <typename T>
class PinnedBuf {
  public:
    PinnedBuf() = default;
    ~PinnedBuf() {
        if (p_) cudaFreeHost(p_);
    }
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    void resize(size_t n) {
        if (n > cap_) {
            if (p_) cudaFreeHost(p_);
            CUDA_CHECK(cudaMallocHost(&p_, n * sizeof(T)));
            cap_ = n;
        }
    }
    T* get() const { return p_; }
    T& operator[](size_t i) { return p_[i]; }

  private:
    T* p_ = nullptr;
    size_t cap_ = 0;
};

inline int grid_for(long long n, int block, int max_blocks = 148 * 16) {
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return static_cast<int>(g);
}

} // namespace dabd_gpu
