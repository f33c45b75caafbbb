// Whole-scene penetration audit on the device:
//   intersection_test  (proj/src/geometry.cpp:389-454, used by sim.cpp:390-391)
//   min_pair_distance  (proj/tests/support/oracles.cpp:153-173)
//
// The reference is O(n^2) over body pairs with an AABB reject. Here:
//   1. k_audit_boxes   body AABBs from the world vertices (body.cpp:136-161,
//                      unfused FP64 like the predicates), inflated by the
//                      distance cutoff, and a sortable key of lo.x;
//   2. CUB radix sort of the keys (stable: ties stay in body order);
//   3. k_audit_sweep   one warp per body in sorted order walks the following
//                      bodies 32 at a time until lo.x passes its hi.x (the
//                      reference's sort-and-sweep break, geometry.cpp:171-176)
//                      and emits every overlapping pair;
//   4. k_audit_pairs   one thread per pair: the reference's exact predicate
//                      (vertex / loop-centroid strictly inside, proper segment
//                      crossings; only for pairs whose uninflated boxes
//                      overlap) and the minimum point-edge distance both ways.
// Decisions are per pair, so the OR over pairs is order-independent and the
// result is bit-exact against the reference; the distance minimum is exact
// whenever it is below the cutoff (the inflated boxes of any pair closer
// than that overlap).
#include "audit.hpp"

#include "instrument.hpp"

#include <cub/device/device_radix_sort.cuh>

#include <cfloat>

namespace dabd_gpu {

namespace {

constexpr int kAB = 256;

// lo.x as an unsigned key whose order is the double order (NaN-free input).
__device__ __forceinline__ unsigned long long order_key(double x) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_audit_boxes(SceneView sc, const double* q, const int* sub, int n, double cutoff,
                              Box* box, Box* boxc, unsigned long long* key, int* idx) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int b = sub[i];
        const double* qb = q + 6 * b;
        Box bx{{DBL_MAX, DBL_MAX}, {-DBL_MAX, -DBL_MAX}};
        for (int v = sc.vstart[b]; v < sc.vstart[b + 1]; ++v) {
            const V2 x = world_point(qb, rest_of(sc, v));
            bx.lo = vmin(bx.lo, x);
            bx.hi = vmax(bx.hi, x);
        }
        box[i] = bx;
        const Box bi = cutoff > 0.0 ? inflate(bx, cutoff) : bx;
        boxc[i] = bi;
        key[i] = order_key(bi.lo.x);
        idx[i] = i;
    }
}

// One warp per sorted position; pairs (i, j) with i < j in subset order.
__global__ void k_audit_sweep(const Box* boxc, const int* order, int n, int2* pairs, int cap,
                              int* count) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int s = gw; s < n; s += nw) {
        const int i = order[s];
        const Box bi = boxc[i];
        for (int base = s + 1; base < n; base += 32) {
            const int t = base + lane;
            bool hit = false, stop = t >= n;
            int j = -1;
            if (!stop) {
                j = order[t];
                const Box bj = boxc[j];
                if (bj.lo.x > bi.hi.x) stop = true; // sorted by lo.x: nothing further overlaps
                else hit = overlaps(bi, bj);
            }
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            if (hm) {
                int slot = 0;
                if (lane == 0) slot = atomicAdd(count, __popc(hm));
                slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(hm & ((1u << lane) - 1u));
                if (hit && slot < cap) pairs[slot] = make_int2(min(i, j), max(i, j));
            }
            if (__ballot_sync(0xffffffffu, stop)) break; // every lane past the break sees lo.x > hi.x too
        }
    }
}

// geometry.cpp:346-367
__device__ bool strictly_inside_loop(V2 p, const SceneView& sc, const double* q, int s) {
    bool inside = false;
    int v = s;
    do {
        const int w = sc.vnext[v];
        const V2 a = world_point(q, rest_of(sc, v)), b = world_point(q, rest_of(sc, w));
        const V2 e = vsub(b, a);
        const double len2 = vsqn(e);
        if (len2 > 0.0) {
            const double t = xdiv(vdot(vsub(p, a), e), len2);
            const double tc = fmin(fmax(t, 0.0), 1.0);
            if (vsqn(vsub(p, vadd(a, vscale(tc, e)))) == 0.0) return false;
        }
        if ((a.y > p.y) != (b.y > p.y)) {
            const double xint = xadd(a.x, xmul(xdiv(xsub(p.y, a.y), xsub(b.y, a.y)), xsub(b.x, a.x)));
            if (xint > p.x) inside = !inside;
        }
        v = w;
    } while (v != s);
    return inside;
}

// first vertex of every loop of body b: v is a loop start iff it is the
// body's first vertex or the previous vertex closes its own loop
__device__ __forceinline__ bool loop_start(const SceneView& sc, int b, int v) {
    return v == sc.vstart[b] || sc.vnext[v - 1] != v;
}

__device__ bool inside_body(V2 p, const SceneView& sc, const double* q, int b) {
    for (int v = sc.vstart[b]; v < sc.vstart[b + 1]; ++v)
        if (loop_start(sc, b, v) && strictly_inside_loop(p, sc, q, v)) return true;
    return false;
}

// geometry.cpp:409-421 (loop centroid; first vertex for a zero-area loop)
__device__ V2 loop_centroid(const SceneView& sc, const double* q, int s) {
    double area = 0.0;
    V2 c{0.0, 0.0};
    int v = s;
    do {
        const int w = sc.vnext[v];
        const V2 a = world_point(q, rest_of(sc, v)), b = world_point(q, rest_of(sc, w));
        const double cr = xsub(xmul(a.x, b.y), xmul(b.x, a.y));
        area = xadd(area, xdiv(cr, 2.0));
        const double k = xdiv(cr, 6.0);
        c = vadd(c, vscale(k, vadd(a, b)));
        v = w;
    } while (v != s);
    if (area != 0.0) return {xdiv(c.x, area), xdiv(c.y, area)};
    return world_point(q, rest_of(sc, s));
}

// geometry.cpp:369-380
__device__ __forceinline__ bool proper_cross(V2 a, V2 b, V2 c, V2 d) {
    const double o1 = vcross(vsub(b, a), vsub(c, a)), o2 = vcross(vsub(b, a), vsub(d, a));
    const double o3 = vcross(vsub(d, c), vsub(a, c)), o4 = vcross(vsub(d, c), vsub(b, c));
    return ((o1 > 0.0 && o2 < 0.0) || (o1 < 0.0 && o2 > 0.0)) &&
           ((o3 > 0.0 && o4 < 0.0) || (o3 < 0.0 && o4 > 0.0));
}

// every vertex and loop centroid of body x strictly inside body y
__device__ bool any_inside(const SceneView& sc, const double* qx, int x, const double* qy, int y) {
    for (int v = sc.vstart[x]; v < sc.vstart[x + 1]; ++v) {
        if (inside_body(world_point(qx, rest_of(sc, v)), sc, qy, y)) return true;
        const int w = sc.vnext[v];
        if (w <= v) { // v closes its loop (loop starts at w): centroid after the vertices
            if (inside_body(loop_centroid(sc, qx, w), sc, qy, y)) return true;
        }
    }
    return false;
}

__global__ void k_audit_pairs(SceneView sc, const double* q, const int* sub, const Box* box,
                              const int2* pairs, const int* count, int cap, int want_dist,
                              int* n_viol, int* flags, double* dmin) {
    const int n = min(*count, cap);
    double best = DBL_MAX;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int2 pr = pairs[t];
        const int bi = sub[pr.x], bj = sub[pr.y];
        const double* qi = q + 6 * bi;
        const double* qj = q + 6 * bj;
        int bad = 0;
        if (overlaps(box[pr.x], box[pr.y])) {
            bad = any_inside(sc, qi, bi, qj, bj) || any_inside(sc, qj, bj, qi, bi);
            for (int a = sc.vstart[bi]; !bad && a < sc.vstart[bi + 1]; ++a) {
                const V2 a0 = world_point(qi, rest_of(sc, a)), a1 = world_point(qi, rest_of(sc, sc.vnext[a]));
                for (int b = sc.vstart[bj]; b < sc.vstart[bj + 1]; ++b) {
                    const V2 b0 = world_point(qj, rest_of(sc, b)),
                             b1 = world_point(qj, rest_of(sc, sc.vnext[b]));
                    if (proper_cross(a0, a1, b0, b1)) {
                        bad = 1;
                        break;
                    }
                }
            }
        }
        flags[t] = bad;
        if (bad) atomicAdd(n_viol, 1);
        if (want_dist && !(sc.is_static[bi] && sc.is_static[bj])) {
            for (int dir = 0; dir < 2; ++dir) {
                const int ba = dir ? bj : bi, bb = dir ? bi : bj;
                const double* qa = dir ? qj : qi;
                const double* qb = dir ? qi : qj;
                for (int v = sc.vstart[ba]; v < sc.vstart[ba + 1]; ++v) {
                    const V2 p = world_point(qa, rest_of(sc, v));
                    for (int e = sc.vstart[bb]; e < sc.vstart[bb + 1]; ++e) {
                        const V2 e0 = world_point(qb, rest_of(sc, e)),
                                 e1 = world_point(qb, rest_of(sc, sc.vnext[e]));
                        best = fmin(best, pe_distance(p, e0, e1));
                    }
                }
            }
        }
    }
    if (want_dist) {
        for (int off = 16; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, off));
        if ((threadIdx.x & 31) == 0 && best < DBL_MAX) atomic_min_nonneg(dmin, best);
    }
}

} // namespace

AuditResult Auditor::run(const SceneView& sc, const double* q_dev, const std::vector<int>& subset,
                         double cutoff, cudaStream_t s) {
    AuditResult res;
    const int n = static_cast<int>(subset.size());
    if (n < 2) return res;
    sub_.upload(subset, s);
    box_.resize(n);
    boxc_.resize(n);
    key_.resize(n);
    key2_.resize(n);
    idx_.resize(n);
    order_.resize(n);
    cnt_.resize(3);
    pin_.resize(4);
    pind_.resize(1);
    const int g = std::min(4096, (n + kAB - 1) / kAB);
    DABD_LAUNCH("k_audit_boxes", s,
                (k_audit_boxes<<<g, kAB, 0, s>>>(sc, q_dev, sub_.get(), n, cutoff, box_.get(),
                                                 boxc_.get(), key_.get(), idx_.get())));
    size_t tb = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key_.get(), key2_.get(), idx_.get(),
                                               order_.get(), n, 0, 64, s));
    temp_.resize(tb);
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp_.get(), tb, key_.get(), key2_.get(), idx_.get(),
                                               order_.get(), n, 0, 64, s));
    if (cap_ == 0) cap_ = 16 * n + 1024;
    for (int attempt = 0; attempt < 2; ++attempt) {
        pairs_.resize(cap_);
        flags_.resize(cap_);
        cnt_.zero(s);
        const int gs = std::min(148 * 16, (n * 32 + kAB - 1) / kAB);
        DABD_LAUNCH("k_audit_sweep", s,
                    (k_audit_sweep<<<gs, kAB, 0, s>>>(boxc_.get(), order_.get(), n, pairs_.get(), cap_,
                                                      cnt_.get())));
        CUDA_CHECK(cudaMemcpyAsync(pin_.get(), cnt_.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (pin_[0] <= cap_) break;
        cap_ = pin_[0] + pin_[0] / 4 + 1024; // overflow: exact count known, re-sweep once
    }
    const int np = std::min(pin_[0], cap_);
    res.pairs_tested = np;
    dmin_.resize(1);
    const double init = DBL_MAX;
    dmin_.upload(&init, 1, s);
    if (np > 0) {
        const int gp = std::min(4096, (np + kAB - 1) / kAB);
        DABD_LAUNCH("k_audit_pairs", s,
                    (k_audit_pairs<<<gp, kAB, 0, s>>>(sc, q_dev, sub_.get(), box_.get(), pairs_.get(),
                                                      cnt_.get(), cap_, cutoff > 0.0 ? 1 : 0,
                                                      cnt_.get() + 1, flags_.get(), dmin_.get())));
    }
    CUDA_CHECK(cudaMemcpyAsync(pin_.get() + 1, cnt_.get() + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(pind_.get(), dmin_.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    CUDA_CHECK(cudaGetLastError());
    res.violations = pin_[1];
    res.min_distance = pind_[0];
    return res;
}

} // namespace dabd_gpu
