// Microbenchmark: cost of one cluster-wide reduction round as used by the
// cluster PCG (per-warp DSMEM push + barrier.cluster + table fold), vs a bare
// barrier and vs __syncthreads, for cluster sizes 2..16 at 512 threads/CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cluster_probe tools/cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;
constexpr int kT = 512, kW = kT / 32;

__device__ __forceinline__ double warp_sum(double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}
__device__ __forceinline__ void cbar() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cbar_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
}

__global__ void k_probe(int mode, int iters, int csize, double* out, long long* cycles) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double tab[16 * kW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = cl.block_rank();
    double acc = threadIdx.x * 1e-3;
    cbar();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
            cbar();
        } else if (mode == 1) {
            __syncthreads();
        } else if (mode == 2) { // push + barrier + fold (the PCG reduction)
            const double w = warp_sum(acc);
            if (lane < csize) cl.map_shared_rank(tab, lane)[rank * kW + warp] = w;
            cbar();
            double v = 0.0;
            for (int i = lane; i < csize * kW; i += 32) v += tab[i];
            acc += 1e-9 * warp_sum(v);
        } else if (mode == 3) {
            cbar_relaxed();
        } else if (mode == 4) { // push + barrier only
            if (lane < csize) cl.map_shared_rank(tab, lane)[rank * kW + warp] = acc;
            cbar();
        } else if (mode == 5) { // warp_sum only
            acc += 1e-9 * warp_sum(acc);
        } else if (mode == 6) { // CTA pre-reduce, one push per CTA, barrier, fold 16
            __shared__ double red[kW];
            __shared__ double tab2[2][16];
            double w = warp_sum(acc);
            if (lane == 0) red[warp] = w;
            __syncthreads();
            if (warp == 0) {
                double v = lane < kW ? red[lane] : 0.0;
                v = warp_sum(v);
                if (lane < csize) cl.map_shared_rank(&tab2[it & 1][0], lane)[rank] = v;
            }
            cbar();
            double v = lane < csize ? tab2[it & 1][lane] : 0.0;
            acc += 1e-9 * warp_sum(v);
        } else if (mode == 7) { // 3 interleaved warp sums
            double a = acc, b = acc * 2, c = acc * 3;
            for (int off = 16; off > 0; off >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, off);
                b += __shfl_xor_sync(0xffffffffu, b, off);
                c += __shfl_xor_sync(0xffffffffu, c, off);
            }
            acc += 1e-9 * (a + b + c);
        } else if (mode == 8) { // per-warp push, parity tables, relaxed-arrive barrier
            const double w = warp_sum(acc);
            if (lane < csize) cl.map_shared_rank(tab, lane)[rank * kW + warp] = w;
            asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
            double v = 0.0;
            for (int i = lane; i < csize * kW; i += 32) v += tab[i];
            acc += 1e-9 * warp_sum(v);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const char* names[] = {"barrier.cluster (release/acquire)", "__syncthreads", "push+barrier+fold",
                           "barrier.cluster relaxed", "push+barrier", "warp_sum",
                           "CTA-reduce+push1+barrier+fold", "3 interleaved warp_sum", "per-warp (dup of 2)"};
    for (int csize : {1, 2, 4, 8, 16}) {
        for (int mode = 0; mode < 9; ++mode) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(csize);
            cfg.blockDim = dim3(kT);
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = csize;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            const int iters = 2000;
            cudaLaunchKernelEx(&cfg, k_probe, mode, iters, csize, out, cyc);
            long long c = 0;
            cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            cudaError_t e = cudaGetLastError();
            printf("csize %2d %-36s %8.1f cycles/iter %s\n", csize, names[mode], double(c) / iters,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
