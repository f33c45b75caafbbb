// Device-resident scene (SoA, FP64) and the views the kernels take.
//
// HBM layout:
//   rest[nv]   double2  centroid-centred rest vertex, bodies contiguous, loop order
//   vstart[nb+1] int    body -> vertex range;  vnext[nv] int  edge e -> 2nd endpoint
//   mblk[nb][6] double  density*(area,sx,sy,sxx,sxy,syy) (the two identical 3x3 mass blocks)
//   minv[nb][3] double  first column of the 3x3 block inverse (q_tilde)
//   mass, rest_area, arap_scale [nb] double;  is_static [nb] int
// Configurations are AoS double[n][6] (the reference's Configs layout,
// 48 B per body) so one body is three 16-byte loads.
#pragma once

#include "dbuf.hpp"
#include "scene.hpp"

namespace dabd_gpu {

struct SceneView {
    int nb = 0, nv = 0;
    const double2* rest = nullptr;
    const int* vstart = nullptr;
    const int* vnext = nullptr;
    const int* is_static = nullptr;
    const double* mass = nullptr;
    const double* mblk = nullptr;
    const double* minv = nullptr;
    const double* rest_area = nullptr;
    const double* arap_scale = nullptr;
};

class DeviceScene {
  public:
    void upload(const HostScene& h, cudaStream_t s) {
        nb = h.nb;
        nv = h.nv;
        max_verts = h.max_verts_per_body;
        rest.upload(reinterpret_cast<const double2*>(h.rest.data()), h.nv, s);
        vstart.upload(h.vstart, s);
        vnext.upload(h.vnext, s);
        is_static.upload(h.is_static, s);
        mass.upload(h.mass, s);
        mblk.upload(h.mblk, s);
        minv.upload(h.minv, s);
        rest_area.upload(h.rest_area, s);
        arap_scale.upload(h.arap_scale, s);
    }
    SceneView view() const {
        SceneView v;
        v.nb = nb;
        v.nv = nv;
        v.rest = rest.get();
        v.vstart = vstart.get();
        v.vnext = vnext.get();
        v.is_static = is_static.get();
        v.mass = mass.get();
        v.mblk = mblk.get();
        v.minv = minv.get();
        v.rest_area = rest_area.get();
        v.arap_scale = arap_scale.get();
        return v;
    }
    int nb = 0, nv = 0, max_verts = 0;

  private:
    DBuf<double2> rest;
    DBuf<int> vstart, vnext, is_static;
    DBuf<double> mass, mblk, minv, rest_area, arap_scale;
};

// A set of body *instances* (a body replicated on a partition), sorted by
// (partition, body). q0/q1 are per-instance configurations: replicas of a
// shared body carry different states on different partitions.
struct InstView {
    int n = 0;
    const int* body = nullptr;
    const int* part = nullptr;
    const double* q0 = nullptr;
    const double* q1 = nullptr; // == q0 for a static (non-swept) query
    // optional per-instance skin (skin-list build): body boxes grow by
    // skin[i], point-edge tests by skin[P] + skin[E] on top of the margin
    const double* skin = nullptr;
};

// Sorted candidate keys: a | b | v | e with the bit widths below.
struct KeyFmt {
    int ibits = 1, vbits = 1;
    __host__ __device__ unsigned long long pack(int a, int b, int v, int e) const {
        return (static_cast<unsigned long long>(a) << (ibits + 2 * vbits)) |
               (static_cast<unsigned long long>(b) << (2 * vbits)) |
               (static_cast<unsigned long long>(v) << vbits) | static_cast<unsigned long long>(e);
    }
    __host__ __device__ void unpack(unsigned long long k, int& a, int& b, int& v, int& e) const {
        const unsigned long long vm = (1ull << vbits) - 1ull, im = (1ull << ibits) - 1ull;
        e = static_cast<int>(k & vm);
        v = static_cast<int>((k >> vbits) & vm);
        b = static_cast<int>((k >> (2 * vbits)) & im);
        a = static_cast<int>((k >> (ibits + 2 * vbits)) & im);
    }
    int total_bits() const { return 2 * ibits + 2 * vbits; }
};

inline int bits_for(long long n) {
    int b = 1;
    while ((1ll << b) < n) ++b;
    return b;
}

} // namespace dabd_gpu
