// 3D broad phase: candidate point-triangle and
// edge-edge pairs between 12-DoF affine bodies, following the reference's 2D
// broad_phase / broad_phase_swept (proj/src/geometry.cpp:106-208) in 3D:
//   body boxes over the world vertices (swept: merged with q_end), inflated by
//   the margin; bodies sorted by (lo.x, id) and swept with the same break rule
//   (lo_j.x > hi_i.x), full 3D overlap test;
//   per overlapping body pair, both orders: point box (merged, not inflated)
//   against the inflated triangle box -> (PT, a, b, vertex, triangle);
//   once per pair (a = lower id): edge box of a against the inflated edge box
//   of b -> (EE, a, b, edge a, edge b);
//   output sorted lexicographically by (kind, a, b, primitive a, primitive b).
// World points round like the reference's unfused arithmetic (x = (A00 xb +
// A01 yb) + A02 zb + p, two roundings per product and sum), so boxes, and
// therefore the candidate lists, are bit-exact against the CPU restatement.
#include "broad3d.hpp"

#include "common.cuh"
#include "dbuf.hpp"
#include "instrument.hpp"

#include <cub/cub.cuh>

#include <cfloat>

namespace dabd_gpu {

namespace {

struct Box3 {
    double lo[3], hi[3];
};

__device__ __forceinline__ void world_x(const double* q, const double* xb, double (&x)[3]) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
        x[r] = xadd(xadd(xadd(xmul(q[3 + 3 * r], xb[0]), xmul(q[4 + 3 * r], xb[1])), xmul(q[5 + 3 * r], xb[2])), q[r]);
}

__device__ __forceinline__ void grow(Box3& b, const double (&x)[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        b.lo[c] = fmin(b.lo[c], x[c]);
        b.hi[c] = fmax(b.hi[c], x[c]);
    }
}

__device__ __forceinline__ Box3 empty_box() {
    return Box3{{DBL_MAX, DBL_MAX, DBL_MAX}, {-DBL_MAX, -DBL_MAX, -DBL_MAX}};
}

__device__ __forceinline__ Box3 inflate3(Box3 b, double m) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        b.lo[c] = xsub(b.lo[c], m);
        b.hi[c] = xadd(b.hi[c], m);
    }
    return b;
}

__device__ __forceinline__ bool overlap3(const Box3& a, const Box3& b) {
    return a.lo[0] <= b.hi[0] && b.lo[0] <= a.hi[0] && a.lo[1] <= b.hi[1] && b.lo[1] <= a.hi[1] &&
           a.lo[2] <= b.hi[2] && b.lo[2] <= a.hi[2];
}

// box of local vertices vs[0..k) of body b at q (and q_end)
__device__ __forceinline__ Box3 prim_box(const Broad3dView& v, int b, const int* vs, int k) {
    Box3 bx = empty_box();
    for (int i = 0; i < k; ++i) {
        const double* xb = v.verts + 3 * static_cast<size_t>(v.vstart[b] + vs[i]);
        double x[3];
        world_x(v.q + 12 * b, xb, x);
        grow(bx, x);
        if (v.q_end) {
            world_x(v.q_end + 12 * b, xb, x);
            grow(bx, x);
        }
    }
    return bx;
}

__global__ void k_body_boxes3(Broad3dView v, Box3* box, double* keyx, int* idx) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= v.n) return;
    Box3 bx = empty_box();
    for (int i = v.vstart[b]; i < v.vstart[b + 1]; ++i) {
        double x[3];
        world_x(v.q + 12 * b, v.verts + 3 * static_cast<size_t>(i), x);
        grow(bx, x);
        if (v.q_end) {
            world_x(v.q_end + 12 * b, v.verts + 3 * static_cast<size_t>(i), x);
            grow(bx, x);
        }
    }
    bx = inflate3(bx, v.margin);
    box[b] = bx;
    keyx[b] = bx.lo[0] + 0.0; // -0.0 -> +0.0: equal keys, ties by id (stable sort)
    idx[b] = b;
}

__global__ void k_sweep3(int n, const Box3* box, const double* keyx_sorted, const int* idx_sorted,
                         int2* pairs, int cap, int* count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = idx_sorted[i];
    const Box3 ba = box[a];
    for (int j = i + 1; j < n; ++j) {
        if (keyx_sorted[j] > ba.hi[0]) break;
        const int b = idx_sorted[j];
        if (!overlap3(ba, box[b])) continue;
        const int k = atomicAdd(count, 1);
        if (k < cap) pairs[k] = make_int2(min(a, b), max(a, b));
    }
}

__device__ __forceinline__ void emit(unsigned long long key, unsigned long long* keys, int cap, int* count) {
    const int k = atomicAdd(count, 1);
    if (k < cap) keys[k] = key;
}

// one block per body pair (a < b)
__global__ void k_prims3(Broad3dView v, const int2* pairs, const int* n_pairs, int cap_pairs,
                         Key3Fmt f, unsigned long long* keys, int cap, int* count) {
    const int np = min(*n_pairs, cap_pairs);
    for (int pi = blockIdx.x; pi < np; pi += gridDim.x) {
        const int2 pr = pairs[pi];
        for (int dir = 0; dir < 2; ++dir) { // PT, both orders (geometry.cpp:198-199)
            const int pa = dir == 0 ? pr.x : pr.y, tb = dir == 0 ? pr.y : pr.x;
            const int nv = v.vstart[pa + 1] - v.vstart[pa], nt = v.tstart[tb + 1] - v.tstart[tb];
            for (int w = threadIdx.x; w < nv * nt; w += blockDim.x) {
                const int vi = w / nt, ti = w - vi * nt;
                const int vv[1] = {vi};
                const int* t = v.tris + 3 * static_cast<size_t>(v.tstart[tb] + ti);
                const int tv[3] = {t[0], t[1], t[2]};
                if (overlap3(prim_box(v, pa, vv, 1), inflate3(prim_box(v, tb, tv, 3), v.margin)))
                    emit(f.pack(0, pa, tb, vi, ti), keys, cap, count);
            }
        }
        const int a = pr.x, b = pr.y; // EE once, a = lower id
        const int na = v.estart[a + 1] - v.estart[a], nb = v.estart[b + 1] - v.estart[b];
        for (int w = threadIdx.x; w < na * nb; w += blockDim.x) {
            const int ea = w / nb, eb = w - ea * nb;
            const int* e0 = v.edges + 2 * static_cast<size_t>(v.estart[a] + ea);
            const int* e1 = v.edges + 2 * static_cast<size_t>(v.estart[b] + eb);
            const int av[2] = {e0[0], e0[1]}, bv[2] = {e1[0], e1[1]};
            if (overlap3(prim_box(v, a, av, 2), inflate3(prim_box(v, b, bv, 2), v.margin)))
                emit(f.pack(1, a, b, ea, eb), keys, cap, count);
        }
    }
}

} // namespace

int broad_phase3d_device(const Broad3dView& v, Key3Fmt f, DBuf<unsigned long long>& sorted, cudaStream_t s) {
    if (v.n < 2) return 0;
    DBuf<Box3> box;
    DBuf<double> kx, kx2;
    DBuf<int> idx, idx2, cnt;
    box.resize(v.n);
    kx.resize(v.n);
    kx2.resize(v.n);
    idx.resize(v.n);
    idx2.resize(v.n);
    cnt.resize(2);
    DABD_LAUNCH("k_body_boxes3", s, k_body_boxes3<<<(v.n + 127) / 128, 128, 0, s>>>(v, box.get(), kx.get(), idx.get()));
    size_t tb = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kx.get(), kx2.get(), idx.get(), idx2.get(), v.n, 0, 64, s));
    DBuf<unsigned char> tmp;
    tmp.resize(std::max<size_t>(tb, 1));
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kx.get(), kx2.get(), idx.get(), idx2.get(), v.n, 0, 64, s));
    // body pairs, then primitive pairs; regrow on overflow (counts are exact)
    int cap_pairs = 16 * v.n, cap = 1 << 16;
    PinnedBuf<int> pin;
    pin.resize(2);
    for (int attempt = 0; attempt < 3; ++attempt) {
        DBuf<int2> pairs;
        pairs.resize(cap_pairs);
        cnt.zero(s);
        DABD_LAUNCH("k_sweep3", s, k_sweep3<<<(v.n + 127) / 128, 128, 0, s>>>(v.n, box.get(), kx2.get(), idx2.get(),
                                                                               pairs.get(), cap_pairs, cnt.get()));
        CUDA_CHECK(cudaMemcpyAsync(pin.get(), cnt.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (pin[0] > cap_pairs) {
            cap_pairs = pin[0];
            continue;
        }
        const int n_pairs = pin[0];
        if (n_pairs == 0) return 0;
        for (int a2 = 0; a2 < 3; ++a2) {
            DBuf<unsigned long long> keys;
            keys.resize(cap);
            sorted.resize(cap);
            CUDA_CHECK(cudaMemsetAsync(cnt.get() + 1, 0, sizeof(int), s));
            DABD_LAUNCH("k_prims3", s, k_prims3<<<std::min(n_pairs, 148 * 8), 128, 0, s>>>(
                                           v, pairs.get(), cnt.get(), cap_pairs, f, keys.get(), cap, cnt.get() + 1));
            CUDA_CHECK(cudaMemcpyAsync(pin.get() + 1, cnt.get() + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
            CUDA_CHECK(cudaStreamSynchronize(s));
            const int nk = pin[1];
            if (nk > cap) {
                cap = nk;
                continue;
            }
            if (nk > 0) {
                size_t sb = 0;
                CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, sb, keys.get(), sorted.get(), nk, 0, f.total_bits(), s));
                tmp.resize(std::max(sb, tmp.size()));
                CUDA_CHECK(cub::DeviceRadixSort::SortKeys(tmp.get(), sb, keys.get(), sorted.get(), nk, 0, f.total_bits(), s));
            }
            return nk;
        }
        throw Error("broad phase 3d: candidate buffer growth failed");
    }
    throw Error("broad phase 3d: body-pair buffer growth failed");
}

std::vector<unsigned long long> broad_phase3d(const Broad3dView& v, Key3Fmt f, cudaStream_t s) {
    DBuf<unsigned long long> sorted;
    const int nk = broad_phase3d_device(v, f, sorted, s);
    std::vector<unsigned long long> out(nk);
    if (nk > 0) {
        CUDA_CHECK(cudaMemcpyAsync(out.data(), sorted.get(), nk * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
    }
    return out;
}

} // namespace dabd_gpu
