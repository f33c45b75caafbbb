// Host-side ADMM controller rules shared by the multi-partition frame and the
// C ABI (dabd_gpu_check_stopping / dabd_gpu_timestep_apply), so the
// reference's known answers pin the code the engine runs.
#pragma once

#include "dbuf.hpp"

#include <algorithm>
#include <vector>

namespace dabd_gpu {

// consensus.cpp:54-64: end iff dq, r and s, each over h * l, are strictly
// below theta and every merge gate passed (toi exactly 1.0).
inline bool check_stopping(double dq, double r, double s, const double* tois, int n_tois, double h,
                           double l, double theta) {
    const double nrm = h * l;
    bool end = dq / nrm < theta && r / nrm < theta && s / nrm < theta;
    for (int i = 0; i < n_tois; ++i)
        if (tois[i] != 1.0) end = false;
    return end;
}
inline bool check_stopping(double dq, double r, double s, const std::vector<double>& tois, double h,
                           double l, double theta) {
    return check_stopping(dq, r, s, tois.data(), static_cast<int>(tois.size()), h, l, theta);
}

// consensus.hpp:60-87: h halves on a failed frame (at most max_halvings
// times in a row), doubles back towards h0 on each commit.
class TimestepController {
  public:
    TimestepController() = default;
    TimestepController(double h0, int max_halvings) : h0_(h0), h_(h0), max_halvings_(max_halvings) {}
    double h() const { return h_; }
    int halvings() const { return halvings_; }
    bool can_halve() const { return halvings_ < max_halvings_; }
    double on_frame_failed() {
        if (!can_halve()) throw Error("adaptive_timestep: frame failed after max halvings");
        h_ /= 2.0;
        ++halvings_;
        return h_;
    }
    void on_frame_committed() {
        h_ = std::min(h0_, 2.0 * h_);
        halvings_ = 0;
    }

  private:
    double h0_ = 0.0, h_ = 0.0;
    int halvings_ = 0, max_halvings_ = 4;
};

} // namespace dabd_gpu
