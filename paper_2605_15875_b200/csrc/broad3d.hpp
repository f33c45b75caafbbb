// 3D broad phase (broad3d.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace dabd_gpu {

// Device pointers. Body b owns rest vertices [vstart[b], vstart[b+1]) of
// verts [nv][3], triangles [tstart[b], tstart[b+1]) of tris [nt][3] and
// edges [estart[b], estart[b+1]) of edges [ne][2] (local vertex indices).
struct Broad3dView {
    int n;
    const double* q;     // [n][12]
    const double* q_end; // [n][12] or nullptr (static broad phase)
    const int* vstart;
    const double* verts;
    const int* tstart;
    const int* tris;
    const int* estart;
    const int* edges;
    double margin;
};

// Candidate key: kind (1 bit) | a | b (bb bits each) | prim a | prim b (pb bits each).
struct Key3Fmt {
    int bb = 1, pb = 1;
    __host__ __device__ int total_bits() const { return 1 + 2 * bb + 2 * pb; }
    __host__ __device__ unsigned long long pack(int kind, int a, int b, int pa, int pbi) const {
        unsigned long long k = static_cast<unsigned long long>(kind);
        k = (k << bb) | static_cast<unsigned long long>(a);
        k = (k << bb) | static_cast<unsigned long long>(b);
        k = (k << pb) | static_cast<unsigned long long>(pa);
        k = (k << pb) | static_cast<unsigned long long>(pbi);
        return k;
    }
    void unpack(unsigned long long k, int& kind, int& a, int& b, int& pa, int& pbi) const {
        const unsigned long long mp = (1ull << pb) - 1ull, mb = (1ull << bb) - 1ull;
        pbi = static_cast<int>(k & mp);
        k >>= pb;
        pa = static_cast<int>(k & mp);
        k >>= pb;
        b = static_cast<int>(k & mb);
        k >>= bb;
        a = static_cast<int>(k & mb);
        k >>= bb;
        kind = static_cast<int>(k);
    }
};

// Sorted candidate keys (host vector); the sort order is the lexicographic
// (kind, a, b, prim a, prim b) order.
std::vector<unsigned long long> broad_phase3d(const Broad3dView& v, Key3Fmt f, cudaStream_t s);
// The same, device-resident: the sorted keys stay in `sorted`; returns their count.
template <typename T>
class DBuf;
int broad_phase3d_device(const Broad3dView& v, Key3Fmt f, DBuf<unsigned long long>& sorted, cudaStream_t s);

} // namespace dabd_gpu
