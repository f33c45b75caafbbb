// Collision detection on sm_100a: per-instance AABBs, a spatial-hash broad
// phase producing the reference's exact candidate set in its sorted order,
// narrow phase, CCD and the partition holder masks.
//
// Replaces proj/src/geometry.cpp:99-341 and partition.cpp:36-67. The
// candidate predicate is the reference's exactly:
// body boxes inflated by `margin` on both sides overlap (<=), then the point
// box (start U end when swept, never inflated) overlaps the margin-inflated
// edge box. Instead of the CPU's sort-and-sweep the body pairs come from a
// uniform hash grid (cell = max dynamic box extent, 3x3 query), statics are
// tested against every dynamic instance, and the candidate keys
// a|b|v|e are radix-sorted, which reproduces ContactPair::operator< order.
#pragma once

#include "common.cuh"
#include "device_scene.hpp"

namespace dabd_gpu {

// ---------------------------------------------------------------------------
// Bit-exact CCD (geometry.cpp:232-307)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void quadratic_roots01(double c2, double c1, double c0, double* r,
                                                  int& n) {
    const double scale = fmax(fabs(c2), fmax(fabs(c1), fabs(c0)));
    if (scale == 0.0) return;
    const double eps = xmul(1e-14, scale);
    if (fabs(c2) <= eps) {
        if (fabs(c1) <= eps) return;
        const double t = xdiv(-c0, c1);
        if (t >= 0.0 && t <= 1.0) r[n++] = t;
        return;
    }
    const double disc = xsub(xmul(c1, c1), xmul(xmul(4.0, c2), c0));
    if (disc < 0.0) return;
    const double sq = xsqrt(disc);
    const double q = xmul(-0.5, xadd(c1, copysign(sq, c1 == 0.0 ? 1.0 : c1)));
    const double t0 = xdiv(q, c2);
    if (t0 >= 0.0 && t0 <= 1.0) r[n++] = t0;
    if (q != 0.0) {
        const double t1 = xdiv(c0, q);
        if (t1 >= 0.0 && t1 <= 1.0) r[n++] = t1;
    }
}

__device__ __forceinline__ double pair_impact_time(V2 p0, V2 p1, V2 a0, V2 a1, V2 b0, V2 b1) {
    const V2 vp = vsub(p1, p0), va = vsub(a1, a0), vb = vsub(b1, b0);
    const V2 w0 = vsub(p0, a0), vw = vsub(vp, va);
    const V2 e0 = vsub(b0, a0), ve = vsub(vb, va);
    const double c0 = vcross(e0, w0);
    const double c1 = xadd(vcross(e0, vw), vcross(ve, w0));
    const double c2 = vcross(ve, vw);
    const double scale = fmax(fabs(c0), fmax(fabs(c1), fabs(c2)));
    double roots[4];
    int n = 0;
    if (scale > 0.0 && fabs(c2) <= xmul(1e-14, scale) && fabs(c1) <= xmul(1e-14, scale) &&
        fabs(c0) <= xmul(1e-14, scale)) {
        const V2 w1 = vsub(p0, b0), vw1 = vsub(vp, vb);
        quadratic_roots01(vdot(vw, ve), xadd(vdot(w0, ve), vdot(vw, e0)), vdot(w0, e0), roots, n);
        quadratic_roots01(vdot(vw1, ve), xadd(vdot(w1, ve), vdot(vw1, e0)), vdot(w1, e0), roots,
                          n);
    } else if (scale == 0.0) {
        return 2.0;
    } else {
        quadratic_roots01(c2, c1, c0, roots, n);
    }
    for (int i = 1; i < n; ++i) // ascending (std::sort in the reference)
        for (int j = i; j > 0 && roots[j] < roots[j - 1]; --j) {
            const double t = roots[j];
            roots[j] = roots[j - 1];
            roots[j - 1] = t;
        }
    for (int i = 0; i < n; ++i) {
        const double t = roots[i];
        const V2 pt = vadd(p0, vscale(t, vp)), at = vadd(a0, vscale(t, va)),
                 bt = vadd(b0, vscale(t, vb));
        const V2 et = vsub(bt, at);
        const double len2 = vsqn(et);
        bool inside;
        if (len2 <= 0.0) {
            inside = vsqn(vsub(pt, at)) <= 0.0;
        } else {
            const double s = xdiv(vdot(vsub(pt, at), et), len2);
            inside = s >= -1e-9 && s <= 1.0 + 1e-9;
        }
        if (inside) return t;
    }
    return 2.0;
}

// ---------------------------------------------------------------------------
// Candidate predicate pieces
// ---------------------------------------------------------------------------
__device__ __forceinline__ V2 rest_of(const SceneView& sc, int v) {
    const double2 r = sc.rest[v];
    return {r.x, r.y};
}

// Inflated edge box (geometry.cpp:124-138), edge given by its flat index.
__device__ __forceinline__ Box edge_box(const SceneView& sc, const double* qa, const double* qb,
                                        bool swept, int eflat, double margin) {
    const V2 r0 = rest_of(sc, eflat), r1 = rest_of(sc, sc.vnext[eflat]);
    const V2 x0 = world_point(qa, r0), x1 = world_point(qa, r1);
    Box b{vmin(x0, x1), vmax(x0, x1)};
    if (swept) {
        const V2 y0 = world_point(qb, r0), y1 = world_point(qb, r1);
        b = merge(b, Box{vmin(y0, y1), vmax(y0, y1)});
    }
    return inflate(b, margin);
}

__device__ __forceinline__ Box point_box(const SceneView& sc, const double* qa, const double* qb,
                                         bool swept, int vflat) {
    const V2 r = rest_of(sc, vflat);
    const V2 x = world_point(qa, r);
    Box b{x, x};
    if (swept) {
        const V2 y = world_point(qb, r);
        b = merge(b, Box{y, y});
    }
    return b;
}

// Whole pipeline object (geometry.cu).
class Detector {
  public:
    Detector();
    ~Detector();
    // Sorted candidate superset over instance configurations [q0, q1]
    // (swept when q1 != q0) for the given margin. `stat` lists static
    // instance indices (ascending). Returns the candidate count.
    int build(const SceneView& sc, const InstView& iv, const int* stat, int n_stat, bool swept,
              double margin, int max_verts, cudaStream_t s);
    // Graph-safe variant: fixed capacity, no host reads. Keys past the count
    // are ~0ull (sorted to the end); overflow raises kErrCapacity in `err`.
    void prepare(int n_inst, int max_verts, int cap);
    // prepare() only when the capacity, table size or key format must change
    // (what build() checks before each attempt).
    void ensure(int n_inst, int max_verts, int cap);
    // `dmargin` (device, optional) overrides `margin` at run time, so a
    // captured graph can rebuild with a margin computed on the device.
    void enqueue(const SceneView& sc, const InstView& iv, const int* stat, int n_stat, bool swept,
                 double margin, int* err, cudaStream_t s, const double* dmargin = nullptr);
    const int* d_count() const { return counter_.get(); }
    int cap() const { return cap_; }
    const unsigned long long* keys() const { return keys_sorted_.get(); }
    const Box* boxes() const { return box_.get(); }
    KeyFmt fmt() const { return fmt_; }
    int count() const { return count_; }

  private:
    DBuf<Box> box_;
    DBuf<double> cell_;
    DBuf<int> hcount_, hstart_, hfill_, hitems_, hkey_;
    DBuf<unsigned long long> keys_, keys_sorted_;
    DBuf<int> counter_; // [0] count, [1] overflow-needed
    DBuf<unsigned char> temp_;
    PinnedBuf<int> pin_;
    KeyFmt fmt_;
    int count_ = 0;
    int cap_ = 0;
    int n_cap_ = 0; // instances the per-instance buffers (boxes, hash items) hold
    unsigned tsize_ = 0;
    size_t temp_bytes_ = 0;
};

void launch_narrow_bodies(const SceneView& sc, const double* q, const int* cand, int n,
                          double d_hat, double* d, int* flag, int* err, cudaStream_t s);

// Per-instance boxes (body_aabb, optionally swept, inflated by margin).
void launch_inst_boxes(const SceneView& sc, const InstView& iv, bool swept, double margin, Box* box,
                       double* cell_max, cudaStream_t s, const double* dmargin = nullptr);

} // namespace dabd_gpu
