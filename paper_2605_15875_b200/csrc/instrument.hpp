// Launch accounting and opt-in per-kernel CUDA-event timing (bench.py uses
// them for `gpu_launches`, the roofline of the dominant kernel and the
// per-kernel breakdown written to profiles/).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <map>
#include <string>
#include <vector>

namespace dabd_gpu {

// Number of dabd_gpu __global__ launches (CUB library kernels excluded).
inline std::atomic<long long>& launch_counter() {
    static std::atomic<long long> c{0};
    return c;
}
inline void count_launch(long long n = 1) { launch_counter() += n; }

// Records an event pair around each launch of one named kernel (or of every
// kernel with name "*") on its stream. Disabled while a graph is captured.
class KernelTimer {
  public:
    static KernelTimer& get() {
        static KernelTimer t;
        return t;
    }
    void enable(const std::string& name) {
        flush();
        name_ = name;
        stats_.clear();
        bytes_ = 0.0;
    }
    bool active(const char* name) const {
        return !suspended_ && !name_.empty() && (name_ == "*" || name_ == name);
    }
    void suspend(bool on) { suspended_ = on; }
    void begin(const char* name, cudaStream_t s) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        pending_.push_back({a, b, name});
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
                Stat& st = stats_[p.name];
                st.ms += ms;
                ++st.count;
            }
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        pending_.clear();
    }
    double total_ms() {
        flush();
        double t = 0.0;
        for (auto& kv : stats_) t += kv.second.ms;
        return t;
    }
    long long count() {
        flush();
        long long c = 0;
        for (auto& kv : stats_) c += kv.second.count;
        return c;
    }
    // "name count total_ms;..." for every timed kernel.
    std::string report() {
        flush();
        std::string out;
        for (auto& kv : stats_)
            out += kv.first + " " + std::to_string(kv.second.count) + " " +
                   std::to_string(kv.second.ms) + ";";
        return out;
    }

  private:
    struct Pair {
        cudaEvent_t a, b;
        std::string name;
    };
    struct Stat {
        double ms = 0.0;
        long long count = 0;
    };
    std::string name_;
    bool suspended_ = false;
    std::vector<Pair> pending_;
    std::map<std::string, Stat> stats_;
    double bytes_ = 0.0;
};

// NVTX range over a host scope (header-only NVTX v3: a no-op unless a tool
// such as ncu --nvtx or Nsight Systems is attached). The frame phases carry
// the names of the reference's timers: frame, solve (runtime.cpp:466-468),
// coll (consensus + merge gate, 399-402), sync (fan-in / commit, 586-601).
class NvtxRange {
  public:
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

} // namespace dabd_gpu

// Launch helper: counts the launch and, when this kernel is timed, brackets
// it with CUDA events on `stream`.
#define DABD_LAUNCH(name, stream, ...)                                                     \
    do {                                                                                   \
        const bool _t = ::dabd_gpu::KernelTimer::get().active(name);                       \
        if (_t) ::dabd_gpu::KernelTimer::get().begin(name, stream);                        \
        __VA_ARGS__;                                                                       \
        if (_t) ::dabd_gpu::KernelTimer::get().end(stream);                                \
        ::dabd_gpu::count_launch();                                                        \
        CUDA_CHECK(cudaGetLastError());                                                    \
    } while (0)
