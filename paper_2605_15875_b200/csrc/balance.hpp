// PD load balancer of the interface planes (proj/include/dabd/balance.hpp:9-56,
// proj/src/balance.cpp:8-83): host control logic, fed once per committed
// frame with per-partition compute costs (runtime.cpp:537-552, 674-675).
#pragma once

#include <vector>

#include "scene.hpp"

namespace dabd_gpu {

// T = (eta - 1)/(eta + 1), eta = tau_i / tau_j (balance.cpp:8-13).
double imbalance_metric(double tau_i, double tau_j);
// kp t + kd (t - t_prev), clamped to +-dp_max when dp_max > 0 (balance.cpp:15-19).
double pd_update(double t, double t_prev, double kp, double kd, double dp_max);
// p' = p + dp n (balance.cpp:21-25).
PlaneH shift_boundary(const PlaneH& plane, double dp);
// mean / max of the times (balance.cpp:27-36).
double balance_factor(const std::vector<double>& times);

class Balancer {
  public:
    Balancer() = default;
    Balancer(int num_workers, const BalanceOpts& opts)
        : opts_(opts), smoothed_(num_workers, 0.0), t_prev_(num_workers > 1 ? num_workers - 1 : 0, 0.0) {}
    // balance.cpp:38-81: EMA of the times, one PD step per interface, the
    // shift kept w clear of the neighbouring planes. Returns the shifts.
    std::vector<double> update(const std::vector<double>& compute_times, std::vector<PlaneH>& planes,
                               double w);
    const std::vector<double>& smoothed_times() const { return smoothed_; }

  private:
    BalanceOpts opts_;
    std::vector<double> smoothed_;
    std::vector<double> t_prev_;
    bool primed_ = false;
};

} // namespace dabd_gpu
