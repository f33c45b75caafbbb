// Device-side helpers shared by every dabd_gpu kernel (sm_100a).
//
// Bit-exact paths (world points, AABBs, point-edge distance value, CCD,
// holder masks) must round like the reference's unfused x86-64 SSE2 code
// (SURVEY.md Appendix A, H1). They use the *_rn intrinsics below, which
// nvcc never contracts into FMA; tolerance-level paths (energies, Hessians,
// PCG) use plain arithmetic and may contract.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dabd_gpu {

constexpr int kWarp = 32;
constexpr int kSMs = 148;

// ---------------------------------------------------------------- exact ops
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double xsqrt(double a) { return __dsqrt_rn(a); }

struct V2 {
    double x, y;
};
__device__ __forceinline__ V2 vsub(V2 a, V2 b) { return {xsub(a.x, b.x), xsub(a.y, b.y)}; }
__device__ __forceinline__ V2 vadd(V2 a, V2 b) { return {xadd(a.x, b.x), xadd(a.y, b.y)}; }
__device__ __forceinline__ V2 vscale(double s, V2 a) { return {xmul(s, a.x), xmul(s, a.y)}; }
// a.x*b.x + a.y*b.y, two roundings then one add (Eigen 2-vector redux).
__device__ __forceinline__ double vdot(V2 a, V2 b) { return xadd(xmul(a.x, b.x), xmul(a.y, b.y)); }
__device__ __forceinline__ double vsqn(V2 a) { return xadd(xmul(a.x, a.x), xmul(a.y, a.y)); }
__device__ __forceinline__ double vcross(V2 a, V2 b) { return xsub(xmul(a.x, b.y), xmul(a.y, b.x)); }
__device__ __forceinline__ V2 vmin(V2 a, V2 b) { return {fmin(a.x, b.x), fmin(a.y, b.y)}; }
__device__ __forceinline__ V2 vmax(V2 a, V2 b) { return {fmax(a.x, b.x), fmax(a.y, b.y)}; }

// x = A*xbar + p with A = [[q2,q3],[q4,q5]] (types.hpp:28-30), unfused.
__device__ __forceinline__ V2 world_point(const double* q, V2 xb) {
    return {xadd(xadd(xmul(q[2], xb.x), xmul(q[3], xb.y)), q[0]),
            xadd(xadd(xmul(q[4], xb.x), xmul(q[5], xb.y)), q[1])};
}

struct Box {
    V2 lo, hi;
};
__device__ __forceinline__ bool overlaps(const Box& a, const Box& b) { // body.hpp:74-77
    return a.lo.x <= b.hi.x && b.lo.x <= a.hi.x && a.lo.y <= b.hi.y && b.lo.y <= a.hi.y;
}
__device__ __forceinline__ Box inflate(Box b, double r) { // body.hpp:78-80
    return {{xsub(b.lo.x, r), xsub(b.lo.y, r)}, {xadd(b.hi.x, r), xadd(b.hi.y, r)}};
}
__device__ __forceinline__ Box merge(Box a, Box b) { return {vmin(a.lo, b.lo), vmax(a.hi, b.hi)}; }

// point_edge_distance value (geometry.cpp:34-56), bit-exact. Returns -1 for a
// degenerate edge (reference throws).
__device__ __forceinline__ double pe_distance(V2 p, V2 e0, V2 e1) {
    const V2 e = vsub(e1, e0);
    const double len2 = vsqn(e);
    if (len2 <= 0.0) return -1.0;
    const double t = xdiv(vdot(vsub(p, e0), e), len2);
    if (t <= 0.0) return xsqrt(vsqn(vsub(p, e0)));
    if (t >= 1.0) return xsqrt(vsqn(vsub(p, e1)));
    const V2 w = vsub(p, e0);
    const double c = vcross(e, w);
    const double s = c >= 0.0 ? 1.0 : -1.0;
    return xdiv(xmul(s, c), xsqrt(len2));
}

// Ordered-bits helpers for exact atomic max/min on non-negative doubles.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}
__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
    atomicMin(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

// Device error codes (mapped to dabd_gpu status RUNTIME with a message).
enum DevError : int {
    kErrNone = 0,
    kErrStraddle = 1,       // partition.cpp:55-56
    kErrTouching = 2,       // geometry.cpp:328-329
    kErrBarrierDomain = 3,  // energy.cpp:51
    kErrDegenerateEdge = 4, // geometry.cpp:39
    kErrCapacity = 5,       // candidate/neighbour buffer overflow (host regrows)
    kErrNoHolder = 6,       // objective.cpp:275-276
    kErrFactor = 7,         // newton.cpp:26-27 analogue: non-SPD block
    kErrLineSearch = 8,     // newton.cpp:60-62
    kErrReplica = 9,        // runtime.cpp:384-385 replica rho mismatch
    kErrSettle = 10,        // sim.cpp:239 Newton stepping failed to settle
    kErrEll = 11,           // a BSR row couples more bodies than the ELL width (host regrows)
};

__device__ __forceinline__ void raise(int* err, int code) { atomicCAS(err, 0, code); }

} // namespace dabd_gpu
