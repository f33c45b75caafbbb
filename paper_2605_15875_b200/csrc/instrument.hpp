// Launch accounting and opt-in per-kernel CUDA-event timing (bench.py uses
// them for `gpu_launches` and the roofline of the dominant kernel).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <string>
#include <vector>

namespace dabd_gpu {

// Number of dabd_gpu __global__ launches (CUB library kernels excluded).
inline std::atomic<long long>& launch_counter() {
    static std::atomic<long long> c{0};
    return c;
}
inline void count_launch(long long n = 1) { launch_counter() += n; }

// Records an event pair around each launch of one named kernel on its stream.
class KernelTimer {
  public:
    static KernelTimer& get() {
        static KernelTimer t;
        return t;
    }
    void enable(const std::string& name) {
        name_ = name;
        flush();
        total_ms_ = 0.0;
        count_ = 0;
        bytes_ = 0.0;
    }
    bool active(const char* name) const { return !suspended_ && !name_.empty() && name_ == name; }
    // No event pairs while a stream is being captured into a graph.
    void suspend(bool on) { suspended_ = on; }
    void begin(cudaStream_t s) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        pending_.push_back({a, b});
    }
    void end(cudaStream_t s) { cudaEventRecord(pending_.back().b, s); }
    // Algorithmic bytes of the launch just recorded (SURVEY.md 8(d) model).
    void add_bytes(double b) { bytes_ += b; }
    double bytes() const { return bytes_; }
    // Resolves recorded pairs (call after the stream is synchronised).
    void flush() {
        for (auto& p : pending_) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
                total_ms_ += ms;
                ++count_;
            }
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        pending_.clear();
    }
    double total_ms() {
        flush();
        return total_ms_;
    }
    long long count() {
        flush();
        return count_;
    }

  private:
    struct Pair {
        cudaEvent_t a, b;
    };
    std::string name_;
    bool suspended_ = false;
    std::vector<Pair> pending_;
    double total_ms_ = 0.0;
    long long count_ = 0;
    double bytes_ = 0.0;
};

} // namespace dabd_gpu

// Launch helper: counts the launch and, when this kernel is the timed one,
// brackets it with CUDA events on `stream`.
#define DABD_LAUNCH(name, stream, ...)                                                     \
    do {                                                                                   \
        const bool _t = ::dabd_gpu::KernelTimer::get().active(name);                       \
        if (_t) ::dabd_gpu::KernelTimer::get().begin(stream);                              \
        __VA_ARGS__;                                                                       \
        if (_t) ::dabd_gpu::KernelTimer::get().end(stream);                                \
        ::dabd_gpu::count_launch();                                                        \
        CUDA_CHECK(cudaGetLastError());                                                    \
    } while (0)
