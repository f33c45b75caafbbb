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

// ---------------------------------------------------------------------------
// Cluster-resident PCG: one thread-block cluster (up to 16 SMs) per
// partition. Every CTA stages its chunk of the partition's BSR rows (diagonal
// + eps I and coupling blocks, the DSMEM address of every block's column,
// block-Jacobi inverses) and all PCG vectors in shared memory; neighbours'
// z / p come from the owning CTA's shared memory through DSMEM and the dot
// products meet through DSMEM + cluster barriers. Nothing but the final dq
// leaves the SMs. Rows that do not fit the shared-memory budget read their
// blocks from global memory (L2).
//
// Lane layout: a warp owns 5 rows, lane = 6 * slot + comp computes component
// `comp` of row `slot` (lanes 30, 31 idle), so a 6x6 block costs one row of
// 6 FMAs per lane and no cross-lane reduction. Per iteration:
//   A: Ap_i = sum_j M_ij (z_j + beta p_j)   (p_new recomputed by the reader),
//      p_new = z + beta p_old, partial p.Ap       -> push, cluster barrier
//   B: x += alpha p, r -= alpha Ap, z = Dinv r, partials r.z, r.r
//                                                -> push, cluster barrier
// ---------------------------------------------------------------------------
constexpr int kCT = 512;
constexpr int kCW = kCT / 32;
constexpr int kRowsPerWarp = 5;
constexpr int kCSmemBytes = 200 * 1024;

// Every warp pushes its partials into slot [rank][warp] of every peer's
// table (fire-and-forget DSMEM stores), so after one cluster barrier each
// thread folds the whole table locally in a fixed order -- same bits in every
// thread of every CTA, and no CTA-level barrier on the reduction path.
struct ClusterScalars {
    double pap[16 * kCW];
    double2 rzr[16 * kCW]; // (r.z, r.r)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Fold of the first n entries of a [rank][warp] table (n = csize * kCW).
__device__ __forceinline__ double fold_table(const double* t, int n) {
    const int lane = threadIdx.x & 31;
    double v = 0.0;
    for (int i = lane; i < n; i += 32) v += t[i];
    return warp_sum(v);
}

__device__ __forceinline__ double2 fold_table2(const double2* t, int n) {
    const int lane = threadIdx.x & 31;
    double x = 0.0, y = 0.0;
    for (int i = lane; i < n; i += 32) {
        x += t[i].x;
        y += t[i].y;
    }
    return make_double2(warp_sum(x), warp_sum(y));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// One 6x6 block-row product term: y += M_row . (z + beta p), M/z/p 16B aligned.
__device__ __forceinline__ void blk_row(const double* M, const double* zc, const double* pc,
                                        double beta, double& y) {
    const double2* M2 = reinterpret_cast<const double2*>(M);
    const double2* z2 = reinterpret_cast<const double2*>(zc);
    const double2* p2 = reinterpret_cast<const double2*>(pc);
    const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2];
    const double2 z0 = z2[0], z1 = z2[1], z2v = z2[2];
    const double2 q0 = p2[0], q1 = p2[1], q2 = p2[2];
    y += m0.x * (z0.x + beta * q0.x);
    y += m0.y * (z0.y + beta * q0.y);
    y += m1.x * (z1.x + beta * q1.x);
    y += m1.y * (z1.y + beta * q1.y);
    y += m2.x * (z2v.x + beta * q2.x);
    y += m2.y * (z2v.y + beta * q2.y);
}

__global__ void __launch_bounds__(kCT) k_pcg_cluster(SolverView sv, PcgArgs a, int csize, int cmax_rows) {
    cg::cluster_group cl = cg::this_cluster();
    unsigned long long t_start = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ ClusterScalars sc;
    __shared__ __align__(8) unsigned long long mbar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = lane / 6, comp = lane - 6 * slot;
    const int rank = static_cast<int>(cl.block_rank());
    const int p = blockIdx.x / csize;
    const int R0 = sv.part_row_off[p], R1 = sv.part_row_off[p + 1];
    // CTAs per partition from the partition's own row count (launch csize is
    // the batch maximum): the reduction trees, hence the bits, do not depend
    // on which other partitions share the launch or the GPU. Surplus CTAs
    // get no rows and push exact zeros.
    int cs_p = 1;
    while (cs_p < csize && cs_p * 32 < R1 - R0) cs_p *= 2;
    const int chunk = max(1, (R1 - R0 + cs_p - 1) / cs_p);
    const int r0 = min(R1, R0 + rank * chunk), r1 = min(R1, r0 + chunk);
    const int nr = r1 - r0;
    const PartState& st = sv.ps[p];
    const bool act = st.active != 0 && R1 > R0;
    const double eps = st.eps;
    const int ntab = csize * kCW;
    // shared-memory carve-up (cmax_rows = chunk upper bound used at launch)
    double* vx = reinterpret_cast<double*>(smem);
    double* vr = vx + 6 * cmax_rows;
    double* vz = vr + 6 * cmax_rows;
    double* vap = vz + 6 * cmax_rows;
    double* vp0 = vap + 6 * cmax_rows;
    double* vp1 = vp0 + 6 * cmax_rows;
    double* dinv = vp1 + 6 * cmax_rows;
    int* bstart = reinterpret_cast<int*>(dinv + 36 * cmax_rows); // [cmax_rows + 1]
    const size_t used = (72ull * cmax_rows) * 8 + 4ull * (cmax_rows + 2);
    const int cap_blocks = static_cast<int>((kCSmemBytes - used - 16) / (36 * 8 + 8)) & ~1; // blk 16B-aligned
    const double** bptr = reinterpret_cast<const double**>(
        (reinterpret_cast<uintptr_t>(bstart + cmax_rows + 1) + 15) & ~uintptr_t(15));
    double* blk = reinterpret_cast<double*>(bptr + cap_blocks);
    const ptrdiff_t off_p0 = vp0 - vz, off_p1 = vp1 - vz;

    // ---- stage rows with TMA bulk copies: per row the diagonal block and the
    // contiguous run of coupling blocks, plus the chunk's Dinv in one copy.
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    for (int lr = threadIdx.x; lr < nr; lr += kCT) bstart[lr + 1] = sv.ell_cnt[r0 + lr] + 1;
    __syncthreads();
    if (warp == 0) { // warp-wide inclusive scan in chunks of 32 rows
        int carry = 0;
        for (int b = 0; b < nr; b += 32) {
            int v = b + lane < nr ? bstart[b + lane + 1] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += u;
            }
            if (b + lane < nr) bstart[b + lane + 1] = v + carry;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) bstart[0] = 0;
        __syncwarp();
        // bytes this CTA will receive, then the copies (lanes over rows)
        unsigned bytes = 0;
        for (int lr = lane; lr < nr; lr += 32) {
            const int b0 = bstart[lr], nb = bstart[lr + 1] - b0;
            const int ncp = min(nb, cap_blocks - b0);
            if (ncp > 0) bytes += 288u * ncp;
        }
        for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        if (nr > 0) bytes += 288u * nr; // Dinv
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)),
                         "r"(bytes)
                         : "memory");
        __syncwarp();
        const unsigned bar = smem_u32(&mbar);
        for (int lr = lane; lr < nr; lr += 32) {
            const int r = r0 + lr;
            const int b0 = bstart[lr], nb = bstart[lr + 1] - b0;
            const int ncp = min(nb, cap_blocks - b0);
            if (ncp <= 0) continue;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(blk + 36 * b0)), "l"(sv.rdiag + 36 * r), "r"(288u), "r"(bar)
                         : "memory");
            if (ncp > 1)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(blk + 36 * (b0 + 1))),
                             "l"(sv.ell_blk + static_cast<size_t>(r) * kEll * 36),
                             "r"(288u * (ncp - 1)), "r"(bar)
                             : "memory");
        }
        if (lane == 0 && nr > 0)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(dinv)), "l"(sv.rdinv + 36 * r0), "r"(288u * nr), "r"(bar)
                         : "memory");
    }
    __syncthreads();
    // DSMEM address of every staged block's column (lanes over a row's blocks)
    for (int lr = warp; lr < nr; lr += kCW) {
        const int r = r0 + lr;
        const int b0 = bstart[lr], nb = bstart[lr + 1] - b0;
        for (int t = lane; t < nb && b0 + t < cap_blocks; t += 32) {
            const int col = t == 0 ? r : sv.ell_col[r * kEll + t - 1];
            const int crank = (col - R0) / chunk, cl_row = (col - R0) - crank * chunk;
            bptr[b0 + t] = cl.map_shared_rank(vz, crank) + 6 * cl_row;
        }
    }
    {
        const unsigned bar = smem_u32(&mbar);
        asm volatile("{\n.reg .pred P;\nWAIT%=:\n"
                     "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n"
                     "@!P bra WAIT%=;\n}" ::"r"(bar)
                     : "memory");
    }
    for (int i = threadIdx.x; i < 6 * nr; i += kCT) { // (D + eps I)
        const int lr = i / 6, k = i - 6 * lr;
        const int b0 = bstart[lr];
        if (b0 < cap_blocks) blk[36 * b0 + 7 * k] += eps;
    }
    __syncthreads();

    const int row_step = kCW * kRowsPerWarp;
    // ---- init: r = -grad, x = 0, z = Dinv r, p_old = 0
    double s_rz = 0.0, s_rr = 0.0;
    for (int base = warp * kRowsPerWarp; base < nr; base += row_step) {
        const int lr = base + slot;
        const bool on = lane < 30 && lr < nr;
        const double g = on && act ? -sv.rgrad[6 * (r0 + lr) + comp] : 0.0;
        double z = 0.0;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const double gc = __shfl_sync(0xffffffffu, g, (6 * slot + c) & 31);
            if (on) z += dinv[36 * lr + 6 * comp + c] * gc;
        }
        if (on) {
            const int i = 6 * lr + comp;
            vr[i] = g;
            vz[i] = z;
            vx[i] = 0.0;
            vp0[i] = 0.0;
            s_rz += g * z;
            s_rr += g * g;
        }
    }
    {
        const double2 w = make_double2(warp_sum(s_rz), warp_sum(s_rr));
        if (lane < csize) cl.map_shared_rank(&sc, lane)->rzr[rank * kCW + warp] = w;
    }
    cluster_barrier();
    const double2 bb = fold_table2(sc.rzr, ntab);
    double rz = bb.x;
    const double bnorm2 = bb.y;
    bool done = !act || bnorm2 == 0.0;
    double beta = 0.0;
    int it = 0, cur = 0;
    while (!done) {
        double* pold = cur ? vp1 : vp0;
        double* pnew = cur ? vp0 : vp1;
        const ptrdiff_t poff = cur ? off_p1 : off_p0;
        // ---- phase A: Ap over (z + beta p_old) of the columns; p_new; p.Ap
        double pap = 0.0;
        for (int base = warp * kRowsPerWarp; base < nr; base += row_step) {
            const int lr = base + slot;
            if (lane < 30 && lr < nr) {
                const int b0 = bstart[lr], b1 = bstart[lr + 1];
                double y = 0.0;
                if (b1 <= cap_blocks) { // all blocks staged: two at a time, loads first
                    int s = b0;
                    for (; s + 1 < b1; s += 2) {
                        const double* za = bptr[s];
                        const double* zb = bptr[s + 1];
                        double ya = 0.0, yb = 0.0;
                        blk_row(blk + 36 * s + 6 * comp, za, za + poff, beta, ya);
                        blk_row(blk + 36 * (s + 1) + 6 * comp, zb, zb + poff, beta, yb);
                        y += ya;
                        y += yb;
                    }
                    if (s < b1) {
                        const double* za = bptr[s];
                        double ya = 0.0;
                        blk_row(blk + 36 * s + 6 * comp, za, za + poff, beta, ya);
                        y += ya;
                    }
                } else {
                    for (int s = b0; s < b1; ++s) {
                        double ya = 0.0;
                        if (s < cap_blocks) {
                            blk_row(blk + 36 * s + 6 * comp, bptr[s], bptr[s] + poff, beta, ya);
                        } else { // spilled block: global memory, eps added here
                            const int r = r0 + lr, t = s - b0;
                            const int col = t == 0 ? r : sv.ell_col[r * kEll + t - 1];
                            const double* M = (t == 0 ? sv.rdiag + 36 * r
                                                      : sv.ell_blk + (static_cast<size_t>(r) * kEll + t - 1) * 36) + 6 * comp;
                            const int crank = (col - R0) / chunk, cl_row = (col - R0) - crank * chunk;
                            const double* zc = cl.map_shared_rank(vz, crank) + 6 * cl_row;
                            blk_row(M, zc, zc + poff, beta, ya);
                            if (t == 0) ya += eps * (zc[comp] + beta * zc[poff + comp]);
                        }
                        y += ya;
                    }
                }
                const int i = 6 * lr + comp;
                const double pr = vz[i] + beta * pold[i];
                pnew[i] = pr;
                vap[i] = y;
                pap += pr * y;
            }
        }
        {
            const double w = warp_sum(pap);
            if (lane < csize) cl.map_shared_rank(&sc, lane)->pap[rank * kCW + warp] = w;
        }
        cluster_barrier();
        const double pap_all = fold_table(sc.pap, ntab);
        if (!(pap_all > 0.0)) break; // exact solution or breakdown (uniform)
        const double alpha = rz / pap_all;
        // ---- phase B: x += alpha p ; r -= alpha Ap ; z = Dinv r
        double l_rz = 0.0, l_rr = 0.0;
        for (int base = warp * kRowsPerWarp; base < nr; base += row_step) {
            const int lr = base + slot;
            const bool on = lane < 30 && lr < nr;
            const int i = 6 * lr + comp;
            double rv = 0.0;
            if (on) {
                vx[i] += alpha * pnew[i];
                rv = vr[i] - alpha * vap[i];
                vr[i] = rv;
            }
            double z = 0.0;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                const double rc = __shfl_sync(0xffffffffu, rv, (6 * slot + c) & 31);
                if (on) z += dinv[36 * lr + 6 * comp + c] * rc;
            }
            if (on) {
                vz[i] = z;
                l_rz += rv * z;
                l_rr += rv * rv;
            }
        }
        {
            const double2 w = make_double2(warp_sum(l_rz), warp_sum(l_rr));
            if (lane < csize) cl.map_shared_rank(&sc, lane)->rzr[rank * kCW + warp] = w;
        }
        cluster_barrier();
        const double2 v = fold_table2(sc.rzr, ntab);
        const double rz_new = v.x, rr = v.y;
        beta = rz != 0.0 ? rz_new / rz : 0.0;
        rz = rz_new;
        ++it;
        if (rr <= a.tol * a.tol * bnorm2 || it >= a.max_iters) done = true;
        cur ^= 1;
        // Two barriers per iteration suffice: the one above orders our z /
        // p_new writes before the peers' next phase A, the one in phase A
        // orders their reads of our z before our next phase-B writes.
    }
    for (int base = warp * kRowsPerWarp; base < nr; base += row_step) {
        const int lr = base + slot;
        if (lane < 30 && lr < nr) sv.x[6 * (r0 + lr) + comp] = vx[6 * lr + comp];
    }
    if (rank == 0 && threadIdx.x == 0) {
        sv.ps[p].pcg_iters = it;
        sv.ps[p].pcg_done = 1;
    }
    cluster_barrier(); // no CTA leaves while a peer may still read its shared memory
    if (sv.perf && threadIdx.x == 0) {
        if (rank == 0) { // algorithmic bytes of this partition's solve
            int nblk = 0;
            for (int r = R0; r < R1; ++r) nblk += sv.ell_cnt[r] + 1;
            atomicAdd(&sv.perf->bytes, static_cast<double>(it) * (288.0 * nblk + 504.0 * (R1 - R0)));
            atomicAdd(&sv.perf->iters, static_cast<unsigned long long>(it));
        }
        if (blockIdx.x == 0) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            atomicAdd(&sv.perf->ns, t1 - t_start);
            atomicAdd(&sv.perf->launches, 1ull);
        }
    }
}

} // namespace

int pcg_cluster_size() {
    static int c = 0;
    if (c == 0) {
        cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kCSmemBytes);
        c = 16;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(kCT);
        cfg.dynamicSmemBytes = kCSmemBytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 16;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_pcg_cluster, &cfg) != cudaSuccess || n < 1) c = 8;
        cudaGetLastError();
    }
    return c;
}

void launch_pcg_cluster(const SolverView& sv, int max_rows_per_part, double* pbuf, double tol,
                        int max_iters, cudaStream_t s) {
    if (sv.n_rows == 0) return;
    const int cmax = pcg_cluster_size();
    int csize = 1;
    while (csize < cmax && csize * 32 < max_rows_per_part) csize *= 2; // >= ~32 rows per CTA
    // largest per-partition chunk under the per-partition rule of k_pcg_cluster
    const int cmax_rows = std::max(std::min(max_rows_per_part, 32), (max_rows_per_part + csize - 1) / csize);
    PcgArgs a{pbuf, nullptr, nullptr, tol, max_iters};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize * sv.n_parts);
    cfg.blockDim = dim3(kCT);
    cfg.dynamicSmemBytes = kCSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DABD_LAUNCH("k_pcg", s,
                CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_pcg_cluster, sv, a, csize, cmax_rows)));
}

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
