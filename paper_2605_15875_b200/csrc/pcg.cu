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
constexpr int kCSmemBytes = 220 * 1024;

// Per-iteration partials (r.u, w.u, r.r) of every CTA, pushed into slot
// [parity][rank] of every peer (fire-and-forget DSMEM stores); after the
// cluster barrier every thread folds the csize entries in rank order, so all
// threads of all CTAs hold the same bits. Parity double-buffering lets a fast
// CTA push iteration k+1 while a slow peer still folds iteration k.
struct ClusterScalars {
    double3 tab[2][16];
    double3 red[kCW];
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
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// CTA-wide sums of three values, pushed to every peer's tab[par][rank].
// Ends with the values visible only after the next cluster barrier.
__device__ __forceinline__ void cta_push3(cg::cluster_group& cl, ClusterScalars& sc, int par,
                                          int rank, int csize, double a, double b, double c) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
        c += __shfl_xor_sync(0xffffffffu, c, off);
    }
    if (lane == 0) sc.red[warp] = make_double3(a, b, c);
    __syncthreads();
    if (warp == 0 && lane < csize) {
        double3 t = make_double3(0.0, 0.0, 0.0);
#pragma unroll
        for (int w = 0; w < kCW; ++w) { // fixed order
            t.x += sc.red[w].x;
            t.y += sc.red[w].y;
            t.z += sc.red[w].z;
        }
        cl.map_shared_rank(&sc, lane)->tab[par][rank] = t;
    }
}

__device__ __forceinline__ double3 fold3(const ClusterScalars& sc, int par, int csize) {
    double3 t = make_double3(0.0, 0.0, 0.0);
    for (int k = 0; k < csize; ++k) { // rank order; surplus CTAs pushed zeros
        const double3 v = sc.tab[par][k];
        t.x += v.x;
        t.y += v.y;
        t.z += v.z;
    }
    return t;
}

// Pipelined block-Jacobi PCG (Ghysels & Vanroose 2014, preconditioned
// variant): the three dot products of an iteration travel in ONE cluster
// reduction whose barrier also publishes m = Dinv w to the peers, and the
// barrier latency is hidden behind the local-column half of n = A m:
//   local:  m = Dinv w; partials (r.u, w.u, r.r)  -> push, arrive
//           n_loc = sum_{j in CTA} A_ij m_j
//   wait:   fold; beta, alpha; n += sum_{j in peers} A_ij m_j (DSMEM)
//   update: z = n + b z, q = m + b q, s = w + b s, p = u + b p,
//           x += a p, r -= a s, u -= a q, w -= a z
// Lane layout: a warp owns 5 rows, lane = 6 * slot + comp (lanes 30, 31
// idle), so a 6x6 block costs one row of 6 FMAs per lane.
__global__ void __launch_bounds__(kCT) k_pcg_cluster(SolverView sv, PcgArgs a, int csize, int cmax_rows) {
    cg::cluster_group cl = cg::this_cluster();
    unsigned long long t_start = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ ClusterScalars sc;
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ int n_remote;
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
    // shared-memory carve-up (cmax_rows = chunk upper bound used at launch)
    const int V = 6 * cmax_rows;
    double* vx = reinterpret_cast<double*>(smem);
    double* vr = vx + V;
    double* vu = vr + V;
    double* vw = vu + V;
    double* vz = vw + V;
    double* vq = vz + V;
    double* vs = vq + V;
    double* vp = vs + V;
    double* vm0 = vp + V; // m ping-pong: the vector the peers read
    double* vm1 = vm0 + V;
    double* dinv = vm1 + V;
    int* bstart = reinterpret_cast<int*>(dinv + 36 * cmax_rows); // [cmax_rows + 1]
    // per staged block: the block (288 B), its column code (4 B) and, for a
    // column in a peer CTA, the DSMEM address of that row's m0 entry (8 B)
    const size_t used = (96ull * cmax_rows) * 8 + 4ull * (cmax_rows + 2) + 16;
    const int cap_blocks = static_cast<int>((kCSmemBytes - used - 32) / (288 + 4 + 8)) & ~1;
    double* blk = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(bstart + cmax_rows + 1) + 15) & ~uintptr_t(15));
    const double** rptr = reinterpret_cast<const double**>(blk + 36 * cap_blocks);
    int* bcode = reinterpret_cast<int*>(rptr + cap_blocks);
    const ptrdiff_t m_off = vm1 - vm0;

    // ---- stage rows with TMA bulk copies: per row the diagonal block and the
    // contiguous run of coupling blocks, plus the chunk's Dinv in one copy.
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        n_remote = 0;
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
    // column code of every staged block: >= 0 a row of this CTA, < 0 the
    // remote slot -1 - j (DSMEM address of the peer row's m0 entry)
    for (int lr = warp; lr < nr; lr += kCW) {
        const int r = r0 + lr;
        const int b0 = bstart[lr], nb = bstart[lr + 1] - b0;
        for (int t = lane; t < nb && b0 + t < cap_blocks; t += 32) {
            const int col = t == 0 ? r : sv.ell_col[r * kEll + t - 1];
            const int crank = (col - R0) / chunk, cl_row = (col - R0) - crank * chunk;
            if (crank == rank) {
                bcode[b0 + t] = cl_row;
            } else {
                const int j = atomicAdd(&n_remote, 1);
                rptr[j] = cl.map_shared_rank(vm0, crank) + 6 * cl_row;
                bcode[b0 + t] = -1 - j;
            }
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
    // y = (A v)_row comp over the blocks of one class: local columns (v in
    // this CTA at vloc) or remote columns (peer m buffer `moff` from m0) and
    // spilled blocks (global memory, after the barrier only).
    auto spmv_local = [&](int lr, const double* vloc) -> double {
        const int b0 = bstart[lr], bs = min(bstart[lr + 1], cap_blocks);
        double y = 0.0;
        for (int s = b0; s < bs; ++s) {
            const int code = bcode[s];
            if (code < 0) continue;
            const double2* M2 = reinterpret_cast<const double2*>(blk + 36 * s + 6 * comp);
            const double2* v2 = reinterpret_cast<const double2*>(vloc + 6 * code);
            const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2];
            const double2 w0 = v2[0], w1 = v2[1], w2 = v2[2];
            double ya = m0.x * w0.x;
            ya += m0.y * w0.y;
            ya += m1.x * w1.x;
            ya += m1.y * w1.y;
            ya += m2.x * w2.x;
            ya += m2.y * w2.y;
            y += ya;
        }
        return y;
    };
    auto spmv_remote = [&](int lr, ptrdiff_t moff, double y) -> double {
        const int b0 = bstart[lr], b1 = bstart[lr + 1], bs = min(b1, cap_blocks);
        for (int s = b0; s < bs; ++s) {
            const int code = bcode[s];
            if (code >= 0) continue;
            const double2* M2 = reinterpret_cast<const double2*>(blk + 36 * s + 6 * comp);
            const double2* v2 = reinterpret_cast<const double2*>(rptr[-1 - code] + moff);
            const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2];
            const double2 w0 = v2[0], w1 = v2[1], w2 = v2[2];
            double ya = m0.x * w0.x;
            ya += m0.y * w0.y;
            ya += m1.x * w1.x;
            ya += m1.y * w1.y;
            ya += m2.x * w2.x;
            ya += m2.y * w2.y;
            y += ya;
        }
        for (int s = bs; s < b1; ++s) { // spilled block: global memory + DSMEM
            const int r = r0 + lr, t = s - b0;
            const int col = t == 0 ? r : sv.ell_col[r * kEll + t - 1];
            const double* M = (t == 0 ? sv.rdiag + 36 * r
                                      : sv.ell_blk + (static_cast<size_t>(r) * kEll + t - 1) * 36) + 6 * comp;
            const int crank = (col - R0) / chunk, cl_row = (col - R0) - crank * chunk;
            const double* v = cl.map_shared_rank(vm0, crank) + moff + 6 * cl_row;
            double ya = 0.0;
            for (int c = 0; c < 6; ++c) ya += M[c] * v[c];
            if (t == 0) ya += eps * v[comp];
            y += ya;
        }
        return y;
    };

    // ---- init: r = b = -grad, x = 0, u = Dinv r (published in m1), w = A u
    for (int base = warp * kRowsPerWarp; base < nr; base += row_step) {
        const int lr = base + slot;
        const bool on = lane < 30 && lr < nr;
        const double g = on && act ? -sv.rgrad[6 * (r0 + lr) + comp] : 0.0;
        double u = 0.0;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const double gc = __shfl_sync(0xffffffffu, g, (6 * slot + c) & 31);
            if (on) u += dinv[36 * lr + 6 * comp + c] * gc;
        }
        if (on) {
            const int i = 6 * lr + comp;
            vr[i] = g;
            vu[i] = u;
            vm1[i] = u;
            vx[i] = 0.0;
            vz[i] = 0.0;
            vq[i] = 0.0;
            vs[i] = 0.0;
            vp[i] = 0.0;
        }
    }
    cluster_barrier();
    for (int base = warp * kRowsPerWarp; base < nr; base += row_step) {
        const int lr = base + slot;
        if (lane < 30 && lr < nr) vw[6 * lr + comp] = spmv_remote(lr, m_off, spmv_local(lr, vm1));
    }
    __syncthreads();

    bool done = !act;
    double gamma_old = 0.0, alpha_old = 0.0, bnorm2 = 0.0;
    int it = 0;
    while (!done) {
        const int par = it & 1;
        double* mcur = par ? vm1 : vm0;
        const ptrdiff_t moff = par ? m_off : 0;
        // ---- local: m = Dinv w; partials (r.u, w.u, r.r)
        double l_g = 0.0, l_d = 0.0, l_r = 0.0;
        for (int base = warp * kRowsPerWarp; base < nr; base += row_step) {
            const int lr = base + slot;
            const bool on = lane < 30 && lr < nr;
            const int i = 6 * lr + comp;
            const double wv = on ? vw[i] : 0.0;
            double m = 0.0;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                const double wc = __shfl_sync(0xffffffffu, wv, (6 * slot + c) & 31);
                if (on) m += dinv[36 * lr + 6 * comp + c] * wc;
            }
            if (on) {
                mcur[i] = m;
                const double rv = vr[i], uv = vu[i];
                l_g += rv * uv;
                l_d += wv * uv;
                l_r += rv * rv;
            }
        }
        cta_push3(cl, sc, par, rank, csize, l_g, l_d, l_r); // includes __syncthreads
        cluster_arrive();
        // local-column half of n = A m while the barrier completes
        // (the first two row groups of the warp; more only when nr > 160)
        double nloc0 = 0.0, nloc1 = 0.0;
        {
            const int lr0 = warp * kRowsPerWarp + slot, lr1 = lr0 + row_step;
            if (lane < 30 && lr0 < nr) nloc0 = spmv_local(lr0, mcur);
            if (lane < 30 && lr1 < nr) nloc1 = spmv_local(lr1, mcur);
        }
        cluster_wait();
        const double3 f = fold3(sc, par, csize);
        const double gamma = f.x, delta = f.y, rr = f.z;
        if (it == 0) bnorm2 = rr;
        if (bnorm2 == 0.0 || rr <= a.tol * a.tol * bnorm2 || it >= a.max_iters) break;
        double alpha, beta;
        if (it == 0) {
            beta = 0.0;
            alpha = gamma / delta;
        } else {
            beta = gamma / gamma_old;
            alpha = gamma / (delta - beta * gamma / alpha_old);
        }
        if (!(alpha > 0.0) || !isfinite(alpha)) break; // breakdown (uniform)
        // ---- remote half of n, then the recurrences
        {
            int k = 0;
            for (int base = warp * kRowsPerWarp; base < nr; base += row_step, ++k) {
                const int lr = base + slot;
                if (lane < 30 && lr < nr) {
                    const double n0 = k == 0 ? nloc0 : k == 1 ? nloc1 : spmv_local(lr, mcur);
                    const double n = spmv_remote(lr, moff, n0);
                    const int i = 6 * lr + comp;
                    const double z = n + beta * vz[i];
                    const double q = mcur[i] + beta * vq[i];
                    const double s = vw[i] + beta * vs[i];
                    const double pv = vu[i] + beta * vp[i];
                    vz[i] = z;
                    vq[i] = q;
                    vs[i] = s;
                    vp[i] = pv;
                    vx[i] += alpha * pv;
                    vr[i] -= alpha * s;
                    vu[i] -= alpha * q;
                    vw[i] -= alpha * z;
                }
            }
        }
        gamma_old = gamma;
        alpha_old = alpha;
        ++it;
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
