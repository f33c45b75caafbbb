// Microbenchmark: one cluster-wide exchange round of 3 doubles per CTA (the
// cluster PCG's per-iteration partials), 16 CTAs x 512 threads, cycles per
// round for several send mechanisms:
//   0 scalar warp: CTA tree, lanes < csize st.async (2 x v2.f64) to every peer,
//     mbarrier complete_tx wait, fold (the round-1 kernel)
//   1 warp k -> peer k st.async
//   2 scalar warp: plain remote stores + remote mbarrier arrive (release.cluster)
//   3 local store + barrier.cluster + 16-lane DSMEM pull + fold
//   4 warp k -> peer k: plain remote stores + remote arrive
//   5 scalar warp, one 32-lane st.async (lane k: (t0, t1) to k, lane 16 + k: (t2, 0))
//   6 local only: the same trees, __syncthreads and hand-off, no remote traffic
//   7 as 6 without the FP64 division
//   8 as 0 without the FP64 division
//   9 as 5, every warp folds (no hand-off)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/exchange_probe tools/exchange_probe.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa(unsigned a, int r) {
    unsigned o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void cbar() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void st_async2(unsigned dst, double a, double b, unsigned bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
                 "d"(a), "d"(b), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(bar),
                 "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned bar, unsigned parity) {
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(bar),
                 "r"(parity)
                 : "memory");
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

template <int kT>
__global__ void __launch_bounds__(kT) k_probe(int mode, int iters, double* out, long long* cycles) {
    constexpr int kW = kT / 32;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ __align__(16) double tab[2][16][4];
    __shared__ double red[kW][3];
    __shared__ double scal[3];
    __shared__ __align__(8) unsigned long long bar[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cl.block_rank());
    const int csize = static_cast<int>(cl.num_blocks());
    const bool remote_arrive = mode == 2 || mode == 4;
    if (threadIdx.x == 0) {
        // complete_tx modes: 1 local arrival + bytes; remote-arrive modes: csize arrivals
        const unsigned cnt = remote_arrive ? csize : 1;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(cnt));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[1])), "r"(cnt));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 2 * 16 * 4; i += kT) (&tab[0][0][0])[i] = 0.0;
    __syncthreads();
    cbar();
    double acc = 1e-3 * threadIdx.x + rank;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const unsigned b = smem_u32(&bar[par]);
        double l0 = warp_sum(acc), l1 = warp_sum(acc * 0.5), l2 = warp_sum(acc * 0.25);
        if (lane == 0) {
            red[warp][0] = l0;
            red[warp][1] = l1;
            red[warp][2] = l2;
        }
        const bool remote = mode != 6 && mode != 7;
        if (!remote_arrive && mode != 3 && remote && threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(32u * csize) : "memory");
        __syncthreads();
        const bool sender = (mode == 1 || mode == 4) ? warp < csize : warp == kW - 1;
        if (sender) {
            double t0s = lane < kW ? red[lane][0] : 0.0, t1 = lane < kW ? red[lane][1] : 0.0,
                   t2 = lane < kW ? red[lane][2] : 0.0;
            t0s = warp_sum(t0s);
            t1 = warp_sum(t1);
            t2 = warp_sum(t2);
            const int peer = (mode == 1 || mode == 4) ? warp : lane;
            const bool go = (mode == 1 || mode == 4) ? lane == 0 : lane < csize;
            if (mode == 5 || mode == 9) {
                const int pr = lane & 15;
                if (pr < csize) {
                    const unsigned dst = mapa(smem_u32(&tab[par][rank][0]), pr) + (lane >> 4) * 16u;
                    st_async2(dst, lane < 16 ? t0s : t2, lane < 16 ? t1 : 0.0, mapa(b, pr));
                }
            } else if (mode == 6 || mode == 7) {
                if (lane < csize) tab[par][lane][0] = t0s + t1 + t2;
            } else if (go) {
                const unsigned dst = mapa(smem_u32(&tab[par][rank][0]), peer);
                if (mode == 0 || mode == 1 || mode == 8) {
                    st_async2(dst, t0s, t1, mapa(b, peer));
                    st_async2(dst + 16, t2, 0.0, mapa(b, peer));
                } else if (mode == 2 || mode == 4) {
                    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(dst), "d"(t0s), "d"(t1) : "memory");
                    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst + 16), "d"(t2) : "memory");
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(b, peer))
                                 : "memory");
                }
            }
            if (mode == 3 && lane == 0) {
                tab[par][rank][0] = t0s;
                tab[par][rank][1] = t1;
                tab[par][rank][2] = t2;
            }
        }
        // ... local work would go here ...
        if (mode == 3) {
            cbar();
        } else if (!remote) {
            __syncwarp();
        } else if (remote_arrive) {
            mbar_wait_cluster(b, (it >> 1) & 1);
        } else {
            mbar_wait(b, (it >> 1) & 1);
        }
        if (warp == kW - 1 || mode == 9) {
            double g = 0.0, d = 0.0, r = 0.0;
            if (lane < csize) {
                const double* src = mode == 3 ? cl.map_shared_rank(&tab[par][lane][0], lane) : &tab[par][lane][0];
                g = src[0];
                d = src[1];
                r = src[2];
            }
            g = warp_sum(g);
            d = warp_sum(d);
            r = warp_sum(r);
            const double alpha = (mode == 7 || mode == 8) ? g * (d + 1.0 + r * r) : g / (d + 1.0 + r * r);
            if (mode == 9) {
                acc += 1e-12 * alpha;
            } else {
                if (lane == 0) scal[0] = alpha;
                asm volatile("bar.arrive 1, %0;" ::"r"(kT) : "memory");
            }
        } else {
            asm volatile("bar.sync 1, %0;" ::"r"(kT) : "memory");
        }
        if (mode != 9) acc += 1e-12 * scal[0];
        if (mode == 3) __syncthreads(); // scal reuse
    }
    const long long t1c = clock64();
    cbar();
    if (threadIdx.x == 0) {
        cycles[blockIdx.x] = t1c - t0;
        out[blockIdx.x] = acc;
    }
}

template <int kT>
void run_all(double* out, long long* cyc);

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&cyc, 64 * sizeof(long long));
    run_all<512>(out, cyc);
    run_all<256>(out, cyc);
    run_all<128>(out, cyc);
    return 0;
}

template <int kT>
void run_all(double* out, long long* cyc) {
    cudaFuncSetAttribute(k_probe<kT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int iters = 2000;
    for (int cs : {16, 8}) {
        for (int mode = 0; mode <= 9; ++mode) {
            if ((mode == 1 || mode == 4) && kT / 32 < cs) continue; // warp k -> peer k needs csize warps
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(kT);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k_probe<kT>, mode, iters, out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[64];
            cudaMemcpy(h, cyc, cs * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < cs; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("{\"threads\": %d, \"csize\": %d, \"mode\": %d, \"cycles_per_round\": %.1f, \"err\": \"%s\"}\n", kT, cs, mode,
                   double(mx) / iters, cudaGetErrorString(e));
        }
    }
}
