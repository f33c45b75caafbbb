// Whole-scene penetration audit (audit.cu): intersection_test
// (proj/src/geometry.cpp:389-454) and the minimum point-edge distance
// (proj/tests/support/oracles.cpp:153-173) over a body subset on the device.
#pragma once

#include "geometry.cuh"

#include <vector>

namespace dabd_gpu {

struct AuditResult {
    int violations = 0;        // body pairs that interpenetrate (intersection_test == any)
    int pairs_tested = 0;      // body pairs whose cutoff-inflated boxes overlap
    double min_distance = 1.7976931348623157e308; // exact when below the cutoff
};

class Auditor {
  public:
    // q_dev: device [nb][6]; subset: ascending body ids. cutoff > 0 also
    // computes the minimum distance over pairs (a != b, not both static)
    // whose boxes inflated by the cutoff overlap.
    AuditResult run(const SceneView& sc, const double* q_dev, const std::vector<int>& subset,
                    double cutoff, cudaStream_t s);

  private:
    DBuf<int> sub_, idx_, order_, cnt_, flags_;
    DBuf<Box> box_, boxc_;
    DBuf<unsigned long long> key_, key2_;
    DBuf<int2> pairs_;
    DBuf<double> dmin_;
    DBuf<unsigned char> temp_;
    PinnedBuf<int> pin_;
    PinnedBuf<double> pind_;
    int cap_ = 0;
};

} // namespace dabd_gpu
