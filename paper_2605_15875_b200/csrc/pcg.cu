// Block-Jacobi PCG for every partition of the batch in ONE persistent
// cooperative kernel (replaces SimplicialLDLT, proj/src/newton.cpp:25-28).
//
// Each block owns a contiguous chunk of BSR rows (rows are sorted by
// partition). Per iteration:
//   phase A: beta from the previous r.z sums; p_new = z + beta p_old;
//            Ap = (D + eps I) p_new + sum_k B_k (z_c + beta p_old_c); block partial p.Ap
//   grid.sync()
//   phase B: alpha = r.z / p.Ap; x += alpha p; r -= alpha Ap; z = Dinv r;
//            block partials r.z, r.r
//   grid.sync()
// Every block re-derives the per-partition scalars from the block partials
// with the same fixed-order warp reduction, so all blocks agree bitwise and
// the convergence decision (||r|| <= tol ||b||) needs no host round trip.
#include "kernels.hpp"

#include "instrument.hpp"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace dabd_gpu {

namespace {

constexpr int kT = 256;
constexpr int kWarps = kT / 32;

__device__ __forceinline__ void ld6(const double* s, double (&d)[6]) {
    const double2* p = reinterpret_cast<const double2*>(s);
    const double2 a = p[0], b = p[1], c = p[2];
    d[0] = a.x;
    d[1] = a.y;
    d[2] = b.x;
    d[3] = b.y;
    d[4] = c.x;
    d[5] = c.y;
}

__device__ __forceinline__ void st6(double* s, const double (&d)[6]) {
    double2* p = reinterpret_cast<double2*>(s);
    p[0] = make_double2(d[0], d[1]);
    p[1] = make_double2(d[2], d[3]);
    p[2] = make_double2(d[4], d[5]);
}

__device__ __forceinline__ void mv36(const double* m, const double (&x)[6], double (&y)[6]) {
#pragma unroll
    for (int a = 0; a < 6; ++a) {
        const double2* row = reinterpret_cast<const double2*>(m + 6 * a);
        const double2 r0 = row[0], r1 = row[1], r2 = row[2];
        y[a] = r0.x * x[0] + r0.y * x[1] + r1.x * x[2] + r1.y * x[3] + r2.x * x[4] + r2.y * x[5];
    }
}

struct PcgArgs {
    double* pa;      // [2][n_rows][6] ping-pong search directions
    double* part;    // [3][G][P] block partials: pAp, rz, rr
    double* rowval;  // [n_rows] per-row scratch
    double tol;
    int max_iters;
};

// Block-local, partition-segmented sum of rowval over this block's chunk,
// written to out[blockIdx.x * P + p] (fixed order -> deterministic).
__device__ void block_partials(const SolverView& sv, const double* rowval, int r0, int r1,
                               double* out, double* sh) {
    const int P = sv.n_parts;
    for (int p = 0; p < P; ++p) {
        const int s0 = max(r0, sv.part_row_off[p]), s1 = min(r1, sv.part_row_off[p + 1]);
        if (s0 >= s1) { // uniform across the block
            if (threadIdx.x == 0) out[blockIdx.x * P + p] = 0.0;
            continue;
        }
        double acc = 0.0;
        for (int r = s0 + threadIdx.x; r < s1; r += kT) acc += rowval[r];
        sh[threadIdx.x] = acc;
        __syncthreads();
#pragma unroll
        for (int w = kT / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[blockIdx.x * P + p] = sh[0];
        __syncthreads();
    }
}

// sums[p] = sum_g part[g*P + p], identical in every block.
__device__ void grid_sums(const double* part, int G, int P, double* sums) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int p = warp; p < P; p += kWarps) {
        double v = 0.0;
        for (int g = lane; g < G; g += 32) v += __ldcg(part + g * P + p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) sums[p] = v;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kT) k_pcg(SolverView sv, PcgArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[kT];
    __shared__ double s_rz[kMaxParts], s_rr[kMaxParts], s_pap[kMaxParts], s_beta[kMaxParts],
        s_alpha[kMaxParts], s_bn[kMaxParts];
    __shared__ int s_done[kMaxParts], s_it[kMaxParts], s_all;
    const int G = gridDim.x, P = sv.n_parts, R = sv.n_rows;
    const int chunk = (R + G - 1) / G;
    const int r0 = min(R, blockIdx.x * chunk), r1 = min(R, r0 + chunk);
    double* pap_part = a.part;
    double* rz_part = a.part + G * P;
    double* rr_part = a.part + 2 * G * P;
    double* pbuf[2] = {a.pa, a.pa + 6 * static_cast<size_t>(R)};

    // ---- init: r = -grad, x = 0, z = Dinv r, p_old = 0
    for (int r = r0 + threadIdx.x; r < r1; r += kT) {
        const int p = sv.rpart[r] - sv.part_base;
        const bool act = sv.ps[p].active != 0;
        double g[6], z[6];
        ld6(sv.rgrad + 6 * r, g);
#pragma unroll
        for (int k = 0; k < 6; ++k) g[k] = act ? -g[k] : 0.0;
        mv36(sv.rdinv + 36 * r, g, z);
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            if (!act) z[k] = 0.0;
            s1 += g[k] * z[k];
            s2 += g[k] * g[k];
        }
        const double zero[6] = {0, 0, 0, 0, 0, 0};
        st6(sv.r + 6 * r, g);
        st6(sv.z + 6 * r, z);
        st6(sv.x + 6 * r, zero);
        st6(pbuf[0] + 6 * r, zero);
        a.rowval[r] = s1;
        sv.ap[6 * r] = s2; // scratch for r.r
    }
    __syncthreads();
    block_partials(sv, a.rowval, r0, r1, rz_part, sh);
    for (int r = r0 + threadIdx.x; r < r1; r += kT) a.rowval[r] = sv.ap[6 * r];
    __syncthreads();
    block_partials(sv, a.rowval, r0, r1, rr_part, sh);
    grid.sync();
    grid_sums(rz_part, G, P, s_rz);
    grid_sums(rr_part, G, P, s_bn);
    if (threadIdx.x < P) {
        const int p = threadIdx.x;
        s_done[p] = (!sv.ps[p].active || s_bn[p] == 0.0) ? 1 : 0;
        s_it[p] = 0;
        s_beta[p] = 0.0;
    }
    __syncthreads();

    int cur = 0;
    for (int it = 0; it < a.max_iters; ++it) {
        if (threadIdx.x == 0) {
            int all = 1;
            for (int p = 0; p < P; ++p) all &= s_done[p];
            s_all = all;
        }
        __syncthreads();
        if (s_all) break; // uniform across blocks (identical scalars)
        const double* pold = pbuf[cur];
        double* pnew = pbuf[cur ^ 1];
        // ---- phase A
        for (int r = r0 + threadIdx.x; r < r1; r += kT) {
            const int p = sv.rpart[r] - sv.part_base;
            if (s_done[p]) {
                a.rowval[r] = 0.0;
                continue;
            }
            const double beta = s_beta[p];
            double pr[6], zr[6], y[6];
            ld6(pold + 6 * r, pr);
            ld6(sv.z + 6 * r, zr);
#pragma unroll
            for (int k = 0; k < 6; ++k) pr[k] = zr[k] + beta * pr[k];
            st6(pnew + 6 * r, pr);
            mv36(sv.rdiag + 36 * r, pr, y);
            const double eps = sv.ps[p].eps;
#pragma unroll
            for (int k = 0; k < 6; ++k) y[k] += eps * pr[k];
            const int nb = sv.ell_cnt[r];
            for (int t = 0; t < nb; ++t) {
                const int c = sv.ell_col[r * kEll + t];
                double pc[6], zc[6], yc[6];
                ld6(pold + 6 * c, pc);
                ld6(sv.z + 6 * c, zc);
#pragma unroll
                for (int k = 0; k < 6; ++k) pc[k] = zc[k] + beta * pc[k];
                mv36(sv.ell_blk + (static_cast<size_t>(r) * kEll + t) * 36, pc, yc);
#pragma unroll
                for (int k = 0; k < 6; ++k) y[k] += yc[k];
            }
            st6(sv.ap + 6 * r, y);
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s += pr[k] * y[k];
            a.rowval[r] = s;
        }
        __syncthreads();
        block_partials(sv, a.rowval, r0, r1, pap_part, sh);
        grid.sync();
        grid_sums(pap_part, G, P, s_pap);
        if (threadIdx.x < P) {
            const int p = threadIdx.x;
            if (!s_done[p] && !(s_pap[p] > 0.0)) s_done[p] = 1; // breakdown
            s_alpha[p] = s_done[p] ? 0.0 : s_rz[p] / s_pap[p];
        }
        __syncthreads();
        // ---- phase B
        for (int r = r0 + threadIdx.x; r < r1; r += kT) {
            const int p = sv.rpart[r] - sv.part_base;
            if (s_done[p]) {
                a.rowval[r] = 0.0;
                sv.ap[6 * r + 1] = 0.0;
                continue;
            }
            const double alpha = s_alpha[p];
            double x[6], rv[6], pv[6], av[6], z[6];
            ld6(sv.x + 6 * r, x);
            ld6(sv.r + 6 * r, rv);
            ld6(pnew + 6 * r, pv);
            ld6(sv.ap + 6 * r, av);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                x[k] += alpha * pv[k];
                rv[k] -= alpha * av[k];
            }
            mv36(sv.rdinv + 36 * r, rv, z);
            double s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                s1 += rv[k] * z[k];
                s2 += rv[k] * rv[k];
            }
            st6(sv.x + 6 * r, x);
            st6(sv.r + 6 * r, rv);
            st6(sv.z + 6 * r, z);
            a.rowval[r] = s1;
            sv.ap[6 * r + 1] = s2; // Ap is dead after this row's update
        }
        __syncthreads();
        block_partials(sv, a.rowval, r0, r1, rz_part, sh);
        for (int r = r0 + threadIdx.x; r < r1; r += kT) a.rowval[r] = sv.ap[6 * r + 1];
        __syncthreads();
        block_partials(sv, a.rowval, r0, r1, rr_part, sh);
        grid.sync();
        grid_sums(rz_part, G, P, sh); // sh[p] = rz_new
        grid_sums(rr_part, G, P, s_rr);
        if (threadIdx.x < P) {
            const int p = threadIdx.x;
            if (!s_done[p]) {
                const double rz_new = sh[p];
                s_beta[p] = s_rz[p] != 0.0 ? rz_new / s_rz[p] : 0.0;
                s_rz[p] = rz_new;
                ++s_it[p];
                if (s_rr[p] <= a.tol * a.tol * s_bn[p] || s_it[p] >= a.max_iters) s_done[p] = 1;
            }
        }
        __syncthreads();
        cur ^= 1;
    }
    if (blockIdx.x == 0 && threadIdx.x < P) {
        sv.ps[threadIdx.x].pcg_iters = s_it[threadIdx.x];
        sv.ps[threadIdx.x].pcg_done = 1;
        sv.ps[threadIdx.x].rr = s_rr[threadIdx.x];
        sv.ps[threadIdx.x].bnorm2 = s_bn[threadIdx.x];
    }
}

} // namespace

int pcg_grid_size(int n_rows) {
    static int max_blocks = 0;
    if (max_blocks == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg, kT, 0);
        max_blocks = std::max(1, sms * std::max(per_sm, 1));
    }
    // ~2 rows per thread keeps each block's chunk busy; never exceed residency.
    const int want = (n_rows + 2 * kT - 1) / (2 * kT);
    return std::max(1, std::min(want, max_blocks));
}

void launch_pcg_persistent(const SolverView& sv, double* pbuf, double* partials, double* rowval,
                           double tol, int max_iters, cudaStream_t s) {
    if (sv.n_rows == 0) return;
    const int G = pcg_grid_size(sv.n_rows);
    PcgArgs a{pbuf, partials, rowval, tol, max_iters};
    // cudaLaunchKernelEx with the cooperative attribute is stream-capturable,
    // so the persistent solver becomes one node of the frame graph.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DABD_LAUNCH("k_pcg", s, CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_pcg, sv, a)));
}

} // namespace dabd_gpu
