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

#include <algorithm>
#include <cstdlib>

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

// Sums of four values over a warp with 6 double shuffles instead of 20:
// after the first two levels different lane groups reduce different values.
// sum(a) in lanes 0-7, sum(b) in 8-15, sum(c) in 16-23, sum(d) in 24-31
// (fixed pattern, so every warp and CTA rounds identically).
__device__ __forceinline__ double warp_sum4(double a, double b, double c, double d, int lane) {
    const bool lo = lane < 16, q = (lane & 8) != 0;
    const double r1 = __shfl_xor_sync(0xffffffffu, lo ? c : a, 16);
    const double r2 = __shfl_xor_sync(0xffffffffu, lo ? d : b, 16);
    if (lo) {
        a += r1;
        b += r2;
    } else {
        c += r1;
        d += r2;
    }
    const double r3 = __shfl_xor_sync(0xffffffffu, lo ? (q ? a : b) : (q ? c : d), 8);
    double v = (lo ? (q ? b : a) : (q ? d : c)) + r3;
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v;
}

struct PcgArgs {
    double* pa;      // [2][n_rows][6] ping-pong search directions
    double* part;    // [3][G][P] block partials: pAp, rz, rr
    double* rowval;  // [n_rows] per-row scratch
    double tol;
    int max_iters;
    // fused Newton head (cluster kernel): the kernel also sums the row traces,
    // sets eps (newton.cpp:20-24, kOpEps), factors the block-Jacobi
    // preconditioner, and after the solve computes ||dq||_inf and takes the
    // convergence decision of newton.cpp:30-36 (kOpNewtonCheck) for every
    // partition, steering the graph's IF node: 5 launches fewer per iteration.
    int fused;
    const double* row_trace; // [n_rows] trace of each assembled diagonal block
    FrameCtrl* ctrl;
    CondHandles hd;
    unsigned* ticket;        // last-cluster detection, reset by the last one
    // warm start (cluster kernel): 1 = x0 the A-norm-optimal multiple of the
    // previous solve's solution (sv.x); 2 = x0 the Galerkin solution over the
    // previous two solutions (sv.x and pa, which the kernel rotates); 0 = off
    int warm;
    int min_rows; // rows per CTA the cluster size aims for (>= min_rows per CTA)
    int spread;   // 1: every warp sends to one peer (partials + halo); 0: the scalar warp sends to
                  // all (two remote stores per peer), 2: the same in one 32-lane store
    int fold_all; // 1: every warp folds the cluster partials itself, 0: the scalar warp folds
    int remote_first; // 1: remote-column SpMV before the scalar hand-off
    int fast_rcp;     // 1: alpha from a MUFU reciprocal + 2 Newton steps, 0: IEEE division
    int close_loop;   // folded Newton tail (PcgFuse::close_loop)
    // inexact Newton (fused cluster kernel, 0: off): stop at the relative
    // residual eta_loose while rms(x) > eta_factor x the Newton tolerance
    double eta_loose;
    double eta_factor;
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
                const int c = sv.ell_col[r * sv.ell_w + t];
                double pc[6], zc[6], yc[6];
                ld6(pold + 6 * c, pc);
                ld6(sv.z + 6 * c, zc);
#pragma unroll
                for (int k = 0; k < 6; ++k) pc[k] = zc[k] + beta * pc[k];
                mv36(sv.ell_blk + (static_cast<size_t>(r) * sv.ell_w + t) * 36, pc, yc);
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
        sv.ps[threadIdx.x].pcg_total += s_it[threadIdx.x];
        sv.ps[threadIdx.x].pcg_done = 1;
        sv.ps[threadIdx.x].rr = s_rr[threadIdx.x];
        sv.ps[threadIdx.x].bnorm2 = s_bn[threadIdx.x];
    }
}

// ---------------------------------------------------------------------------
// Grid-wide pipelined block-Jacobi PCG for partitions too large for one
// cluster (> 4096 rows: undivided C3, C5 partitions). Ghysels & Vanroose's
// pipelined recurrences as in k_pcg_cluster, so ONE grid-wide exchange per
// iteration: every block folds its warps' partials per partition, writes
// them to a parity-double-buffered table, and after the grid barrier every
// block folds the table in the same fixed order (same scalars everywhere).
// One block of 512 threads per SM; lane = 6 * slot + comp, a warp owns row
// groups of 5 rows of one partition (groups aligned to partitions), strided
// over all warps of the grid. Vectors live in global memory (L2-resident,
// read with ld.global.cg across blocks), m = Dinv w double-buffered.
constexpr int kGT = 512, kGW = kGT / 32;

struct GridVecs {
    double *x, *r, *u, *w, *z, *q, *s, *p, *m0, *m1; // [6 R] each
};

__global__ void __launch_bounds__(kGT) k_pcg_grid(SolverView sv, PcgArgs a, GridVecs v) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int s_goff[kMaxParts + 1];
    __shared__ double s_acc[kGW][kMaxParts][4];
    __shared__ double s_beta[kMaxParts], s_alpha[kMaxParts], s_igo[kMaxParts], s_iao[kMaxParts], s_bn[kMaxParts];
    __shared__ int s_done[kMaxParts], s_it[kMaxParts], s_all;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = lane / 6, comp = lane - 6 * slot;
    const int P = sv.n_parts, G = gridDim.x;
    const int gw = blockIdx.x * kGW + warp, NW = G * kGW;
    if (threadIdx.x == 0) {
        int g = 0;
        for (int p = 0; p < P; ++p) {
            s_goff[p] = g;
            g += (sv.part_row_off[p + 1] - sv.part_row_off[p] + 4) / 5;
        }
        s_goff[P] = g;
    }
    if (threadIdx.x < P) {
        const int p = threadIdx.x;
        s_done[p] = sv.ps[p].active ? 0 : 1;
        s_it[p] = 0;
        s_igo[p] = s_iao[p] = 0.0;
    }
    __syncthreads();
    const int n_groups = s_goff[P];
    // row of this lane in group rg (-1: past the partition's end / idle lane)
    auto row_of = [&](int rg, int& part) {
        int p = 0;
        while (rg >= s_goff[p + 1]) ++p;
        part = p;
        const int row = sv.part_row_off[p] + 5 * (rg - s_goff[p]) + slot;
        return (lane < 30 && row < sv.part_row_off[p + 1]) ? row : -1;
    };
    auto spmv = [&](int row, int p, const double* vec) -> double {
        // (D + eps I) v_row + sum_t B_t v_col, row `comp` of every block
        const double2* d2 = reinterpret_cast<const double2*>(sv.rdiag + 36 * static_cast<size_t>(row) + 6 * comp);
        const double2* o2 = reinterpret_cast<const double2*>(vec + 6 * static_cast<size_t>(row));
        double2 m0 = d2[0], m1 = d2[1], m2 = d2[2];
        double2 w0 = __ldcg(o2), w1 = __ldcg(o2 + 1), w2 = __ldcg(o2 + 2);
        double y = m0.x * w0.x + m0.y * w0.y + m1.x * w1.x + m1.y * w1.y + m2.x * w2.x + m2.y * w2.y;
        y += sv.ps[p].eps * __ldcg(vec + 6 * static_cast<size_t>(row) + comp);
        const int nb = sv.ell_cnt[row];
        for (int t = 0; t < nb; ++t) {
            const int c = sv.ell_col[static_cast<size_t>(row) * sv.ell_w + t];
            const double2* b2 = reinterpret_cast<const double2*>(
                sv.ell_blk + (static_cast<size_t>(row) * sv.ell_w + t) * 36 + 6 * comp);
            const double2* c2 = reinterpret_cast<const double2*>(vec + 6 * static_cast<size_t>(c));
            m0 = b2[0], m1 = b2[1], m2 = b2[2];
            w0 = __ldcg(c2), w1 = __ldcg(c2 + 1), w2 = __ldcg(c2 + 2);
            y += m0.x * w0.x + m0.y * w0.y + m1.x * w1.x + m1.y * w1.y + m2.x * w2.x + m2.y * w2.y;
        }
        return y;
    };
    // Dinv (6x6 row `comp`) times the 6 lane values of this slot
    auto dinv_apply = [&](int row, double val) -> double {
        double vc[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) vc[c] = __shfl_sync(0xffffffffu, val, (6 * slot + c) & 31);
        if (row < 0) return 0.0;
        const double2* d2 = reinterpret_cast<const double2*>(sv.rdinv + 36 * static_cast<size_t>(row) + 6 * comp);
        const double2 d0 = d2[0], d1 = d2[1], dd = d2[2];
        return d0.x * vc[0] + d0.y * vc[1] + d1.x * vc[2] + d1.y * vc[3] + dd.x * vc[4] + dd.y * vc[5];
    };
    // per-warp partials per partition in s_acc (fixed order), then the block
    // fold into the parity table part[par][block][P][4]
    auto zero_acc = [&] {
        for (int i = threadIdx.x; i < kGW * kMaxParts * 4; i += kGT) (&s_acc[0][0][0])[i] = 0.0;
        __syncthreads();
    };
    auto flush = [&](int p, double l0, double l1, double l2, double l3) {
        const double v = warp_sum4(l0, l1, l2, l3, lane);
        if ((lane & 7) == 0) s_acc[warp][p][lane >> 3] += v;
    };
    auto block_fold = [&](int par) {
        __syncthreads();
        double* out = a.part + static_cast<size_t>(par) * G * P * 4 + static_cast<size_t>(blockIdx.x) * P * 4;
        for (int i = threadIdx.x; i < P * 4; i += kGT) {
            const int p = i >> 2, k = i & 3;
            double t = 0.0;
            for (int w = 0; w < kGW; ++w) t += s_acc[w][p][k];
            out[i] = t;
        }
    };

    // ---- warm start (a.warm): x0 = c x_prev, the A-optimal multiple of the
    // previous solve's solution (sv.x, carried across instance sets), with
    // ||b||^2 from the same reduction for the stopping test
    __shared__ double s_c[kMaxParts];
    if (a.warm) {
        zero_acc();
        for (int rg = gw; rg < n_groups; rg += NW) {
            int p;
            const int row = row_of(rg, p);
            const bool on = row >= 0 && !s_done[p];
            const size_t e = 6 * static_cast<size_t>(row) + comp;
            double l0 = 0.0, l1 = 0.0, l2 = 0.0;
            if (on) {
                const double ap = spmv(row, p, sv.x);
                const double pv = sv.x[e], bv = -sv.rgrad[e];
                v.z[e] = ap; // A x_prev, consumed below
                l0 = pv * bv;
                l1 = pv * ap;
                l2 = bv * bv;
            }
            flush(p, l0, l1, l2, 0.0);
        }
        block_fold(1);
        grid.sync();
        if (warp < P) {
            const int p = warp;
            const double* tb = a.part + static_cast<size_t>(G) * P * 4;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int b = lane; b < G; b += 32) {
                const double2* q2 = reinterpret_cast<const double2*>(tb + (static_cast<size_t>(b) * P + p) * 4);
                const double2 ab = __ldcg(q2), cd = __ldcg(q2 + 1);
                t0 += ab.x;
                t1 += ab.y;
                t2 += cd.x;
            }
            const double fv = warp_sum4(t0, t1, t2, 0.0, lane);
            const double pb = __shfl_sync(0xffffffffu, fv, 0), pap = __shfl_sync(0xffffffffu, fv, 8),
                         bb = __shfl_sync(0xffffffffu, fv, 16);
            if (lane == 0) {
                double c = pap > 0.0 ? pb / pap : 0.0;
                if (!isfinite(c)) c = 0.0;
                s_c[p] = c;
                s_bn[p] = bb;
            }
        }
        __syncthreads();
    }
    // ---- init: r = b - A x0, u = Dinv r; then w = A u, m = Dinv w
    for (int rg = gw; rg < n_groups; rg += NW) {
        int p;
        const int row = row_of(rg, p);
        const bool on = row >= 0 && !s_done[p];
        const size_t e = 6 * static_cast<size_t>(row) + comp;
        const double c = a.warm ? s_c[p] : 0.0;
        double rv = on ? -sv.rgrad[e] : 0.0, xv = 0.0;
        if (on && c != 0.0) { // (c == 0: A x_prev / x_prev never touch x, r)
            xv = c * sv.x[e];
            rv -= c * __ldcg(v.z + e);
        }
        const double uv = dinv_apply(on ? row : -1, rv);
        if (row >= 0) {
            v.r[e] = rv;
            v.u[e] = uv;
            v.x[e] = xv;
        }
    }
    grid.sync(); // (v.z is reset only after every block consumed A x_prev)
    for (int rg = gw; rg < n_groups; rg += NW) {
        int p;
        const int row = row_of(rg, p);
        if (row < 0) continue;
        const size_t e = 6 * static_cast<size_t>(row) + comp;
        v.z[e] = v.q[e] = v.s[e] = v.p[e] = 0.0;
    }
    zero_acc();
    for (int rg = gw; rg < n_groups; rg += NW) {
        int p;
        const int row = row_of(rg, p);
        const bool on = row >= 0 && !s_done[p];
        const size_t e = 6 * static_cast<size_t>(row) + comp;
        const double wv = on ? spmv(row, p, v.u) : 0.0;
        const double mv = dinv_apply(on ? row : -1, wv);
        double l0 = 0.0, l1 = 0.0, l2 = 0.0;
        if (on) {
            const double rv = __ldcg(v.r + e), uv = __ldcg(v.u + e);
            v.w[e] = wv;
            v.m0[e] = mv;
            l0 = rv * uv;
            l1 = wv * uv;
            l2 = rv * rv;
        }
        flush(p, l0, l1, l2, 0.0); // x = 0
    }
    block_fold(0);
    grid.sync();

    for (int it = 0;; ++it) {
        const int par = it & 1;
        const double* mcur = par ? v.m1 : v.m0;
        double* mnext = par ? v.m0 : v.m1;
        // every block folds the table in the same order -> identical scalars
        if (warp < P) {
            const int p = warp;
            const double* tb = a.part + static_cast<size_t>(par) * G * P * 4;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
            for (int b = lane; b < G; b += 32) {
                const double2* q2 = reinterpret_cast<const double2*>(tb + (static_cast<size_t>(b) * P + p) * 4);
                const double2 ab = __ldcg(q2), cd = __ldcg(q2 + 1);
                t0 += ab.x;
                t1 += ab.y;
                t2 += cd.x;
                t3 += cd.y;
            }
            const double fv = warp_sum4(t0, t1, t2, t3, lane);
            const double gamma = __shfl_sync(0xffffffffu, fv, 0), delta = __shfl_sync(0xffffffffu, fv, 8),
                         rr = __shfl_sync(0xffffffffu, fv, 16), xx = __shfl_sync(0xffffffffu, fv, 24);
            if (lane == 0 && !s_done[p]) {
                if (it == 0 && !a.warm) s_bn[p] = rr;
                const double bn = s_bn[p];
                // inexact Newton as in k_pcg_cluster: loose only while rms(x) > eta_factor tol
                const double xcut = a.eta_factor * sv.ps[p].tol;
                const bool loose = a.eta_loose > a.tol && rr <= a.eta_loose * a.eta_loose * bn &&
                                   xx > static_cast<double>(sv.ps[p].ndof) * xcut * xcut;
                bool stop = bn == 0.0 || rr <= a.tol * a.tol * bn || it >= a.max_iters || loose;
                const double beta = gamma * s_igo[p];
                const double alpha = gamma / (delta - beta * gamma * s_iao[p]);
                stop = stop || !(alpha > 0.0) || !isfinite(alpha);
                s_beta[p] = beta;
                s_alpha[p] = alpha;
                s_igo[p] = 1.0 / gamma;
                s_iao[p] = 1.0 / alpha;
                if (stop) {
                    s_done[p] = 1;
                    s_it[p] = it;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int all = 1;
            for (int p = 0; p < P; ++p) all &= s_done[p];
            s_all = all;
        }
        zero_acc(); // (its __syncthreads also publishes s_all)
        if (s_all) break; // uniform across blocks
        for (int rg = gw; rg < n_groups; rg += NW) {
            int p;
            const int row = row_of(rg, p);
            if (s_done[p]) continue; // uniform per group: the whole warp skips
            const bool on = row >= 0;
            const size_t e = 6 * static_cast<size_t>(row) + comp;
            const double beta = s_beta[p], alpha = s_alpha[p];
            double wv = 0.0, l0 = 0.0, l1 = 0.0, l2 = 0.0, l3 = 0.0;
            if (on) {
                const double n = spmv(row, p, mcur);
                const double mv = __ldcg(mcur + e);
                const double zv = n + beta * __ldcg(v.z + e);
                const double qv = mv + beta * __ldcg(v.q + e);
                const double sv_ = __ldcg(v.w + e) + beta * __ldcg(v.s + e);
                const double pv = __ldcg(v.u + e) + beta * __ldcg(v.p + e);
                const double xv = __ldcg(v.x + e) + alpha * pv;
                const double rv = __ldcg(v.r + e) - alpha * sv_;
                const double uv = __ldcg(v.u + e) - alpha * qv;
                wv = __ldcg(v.w + e) - alpha * zv;
                v.z[e] = zv;
                v.q[e] = qv;
                v.s[e] = sv_;
                v.p[e] = pv;
                v.x[e] = xv;
                v.r[e] = rv;
                v.u[e] = uv;
                v.w[e] = wv;
                l0 = rv * uv;
                l1 = wv * uv;
                l2 = rv * rv;
                l3 = xv * xv;
            }
            const double mn = dinv_apply(on ? row : -1, wv);
            if (on) mnext[e] = mn;
            flush(p, l0, l1, l2, l3);
        }
        block_fold(par ^ 1);
        grid.sync();
    }
    // solution to sv.x (the Newton direction)
    for (int rg = gw; rg < n_groups; rg += NW) {
        int p;
        const int row = row_of(rg, p);
        if (row < 0) continue;
        const size_t e = 6 * static_cast<size_t>(row) + comp;
        sv.x[e] = sv.ps[p].active ? __ldcg(v.x + e) : 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x < P) {
        const int p = threadIdx.x;
        sv.ps[p].pcg_iters = s_it[p];
        sv.ps[p].pcg_total += s_it[p];
        sv.ps[p].pcg_done = 1;
        sv.ps[p].bnorm2 = s_bn[p];
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
constexpr int kSW = kCW - 1; // scalar warp: partial push, fold, CG scalars
constexpr int kCSmemBytes = 220 * 1024;

// Per-iteration partials (r.u, w.u, r.r) of every CTA land in slot
// [parity][rank] of every peer; every thread folds the csize entries in rank
// order, so all threads of all CTAs hold the same bits. Parity
// double-buffering lets a fast CTA send iteration k+1 while a slow peer still
// reads iteration k.
struct ClusterScalars {
    double tab[2][16][4]; // (r.u, w.u, r.r, pad): 32 B slots for v2 stores
    double red[kCW][4];
    double scal[3];       // (beta, alpha, stop) of the iteration, from the scalar warp
    unsigned long long bar[2]; // per-parity mbarriers (st.async complete_tx)
    unsigned long long stage_bar;
    int n_remote, fallback, nobulk, push_ok;
    int wsum[kCW];
    int rlo[16], rcnt[16], rbase[16]; // rows this CTA needs from each peer (bulk mode)
    int2 req[16];                     // per consumer: (first local row, count) it needs from us
    int reqbase[16];                  // ... and where they land in its halo
    double dqm[16];                   // fused: every CTA's max |dq|, by rank (rank 0 only)
    double wsp[6];                    // warm start: this CTA's (p1.b, p2.b, p1.Ap1, p1.Ap2, p2.Ap2, b.b)
    double wred[kCW][6];
};


__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// 1/x from the MUFU approximation and two Newton steps (a few ulp; the CG
// scalars need not be correctly rounded, only identical in every CTA)
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
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

// shared::cluster address of `local_addr` (a shared::cta address) in CTA `rank`
__device__ __forceinline__ unsigned mapa(unsigned local_addr, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}

// 16-byte remote store that completes `bytes` on the destination's mbarrier.
__device__ __forceinline__ void st_async2(unsigned dst, double a, double b, unsigned bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(dst), "d"(a), "d"(b), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile("{\n.reg .pred P;\nWAIT%=:\n"
                 "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                 "@!P bra WAIT%=;\n}" ::"r"(bar), "r"(parity)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

// Pipelined block-Jacobi PCG (Ghysels & Vanroose 2014, preconditioned
// variant) on one thread-block cluster per partition, every vector and the
// partition's BSR rows resident in shared memory:
//   local:  m = Dinv w; partials (r.u, w.u, r.r) -> CTA sum -> st.async to
//           every peer; the m rows a peer's blocks need -> st.async into the
//           peer's halo slots (push, one-way latency, no cluster barrier)
//           n_loc = sum_{j in CTA} A_ij m_j while the messages fly
//   wait:   this CTA's mbarrier (partials + halo bytes); fold; beta, alpha;
//           n += sum_{j remote} A_ij halo_j
//   update: z = n + b z, q = m + b q, s = w + b s, p = u + b p,
//           x += a p, r -= a s, u -= a q, w -= a z
// Lane layout: a warp owns 5 rows, lane = 6 * slot + comp (lanes 30, 31
// idle), so a 6x6 block costs one row of 6 FMAs per lane.
// A cluster whose rows overflow the shared-memory budget (spilled blocks or
// send lists) takes the barrier-synchronised path that reads peers' m
// through DSMEM and spilled blocks from global memory.
// PH: per-phase clock64 accounting (DABD_GPU_PCG_PHASES); a separate
// instantiation because the clock reads cost ~10% even when predicated off.
template <int G, bool PH>
__global__ void __launch_bounds__(kCT) k_pcg_cluster(SolverView sv, PcgArgs a, int csize, int cmax_rows) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned long long c_start = PH ? clock64() : 0ull;
    unsigned long long cs[8] = {}, ci[4] = {};
    unsigned long long t_start = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(16) ClusterScalars sc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = lane / 6, comp = lane - 6 * slot;
    const int rank = static_cast<int>(cl.block_rank());
    const int p = blockIdx.x / csize;
    const int R0 = sv.part_row_off[p], R1 = sv.part_row_off[p + 1];
    // CTAs per partition from the partition's own row count (launch csize is
    // the batch maximum): the reduction trees, hence the bits, do not depend
    // on which other partitions share the launch or the GPU. Surplus CTAs
    // get no rows and send exact zeros.
    int cs_p = 1;
    while (cs_p < csize && cs_p * a.min_rows < R1 - R0) cs_p *= 2;
    const int chunk = max(1, (R1 - R0 + cs_p - 1) / cs_p);
    const int r0 = min(R1, R0 + rank * chunk), r1 = min(R1, r0 + chunk);
    const int nr = r1 - r0;
    const PartState& st = sv.ps[p];
    const bool act = st.active != 0 && R1 > R0;
    double eps = st.eps;
    // the warm start's previous solutions, loaded now so their L2 latency
    // hides behind the staging and the exchange plan
    double wp1[G], wp2[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int lrw = warp * kRowsPerWarp + slot + g * kCW * kRowsPerWarp;
        const bool onw = lane < 30 && lrw < nr;
        const size_t e = 6 * static_cast<size_t>(r0 + lrw) + comp;
        wp1[g] = a.warm && onw && act ? sv.x[e] : 0.0;
        wp2[g] = a.warm > 1 && onw && act ? a.pa[e] : 0.0;
    }
    // inexact Newton (a.eta_loose > 0): the solve may stop at the relative
    // residual eta_loose instead of tol, but only while the iterate's
    // ||x||_2^2 (a fourth sum next to the CG dots, same shuffles) exceeds
    // ndof (eta_factor tol)^2, i.e. rms(x) > eta_factor x the Newton
    // tolerance, so ||x||_inf does too: a direction that can decide
    // convergence (newton.cpp:30-36) is always solved to tol, one that can
    // end the line search (56-62) only after the step halved below 1/factor
    const bool inexact = a.fused && a.eta_loose > a.tol;
    const double xcut2 = static_cast<double>(st.ndof) * (a.eta_factor * st.tol) * (a.eta_factor * st.tol);
    // shared-memory carve-up (cmax_rows = chunk upper bound used at launch)
    const int V = 6 * cmax_rows;
    double* vm0 = reinterpret_cast<double*>(smem); // m = Dinv w, double-buffered by parity
    double* vm1 = vm0 + V;
    double* dinv = vm1 + V;
    int* bstart = reinterpret_cast<int*>(dinv + 36 * cmax_rows); // [cmax_rows + 1]
    // per staged block: the block (288 B), its column code and column (8 B);
    // per remote block additionally two parity halo rows (96 B) and the DSMEM
    // address of the peer row (8 B)
    const size_t used = (48ull * cmax_rows) * 8 + 4ull * (cmax_rows + 2) + 64;
    const int cap_blocks = static_cast<int>((kCSmemBytes - used) / (288 + 4 + 4 + 96 + 8)) & ~1;
    double* blk = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(bstart + cmax_rows + 1) + 15) & ~uintptr_t(15));
    double* halo = blk + 36 * cap_blocks; // [2][cap_blocks][6]
    const double** rptr = reinterpret_cast<const double**>(halo + 12 * cap_blocks);
    int* bcode = reinterpret_cast<int*>(rptr + cap_blocks);
    int* bcol = bcode + cap_blocks; // column (partition row) of every staged block
    const ptrdiff_t m_off = vm1 - vm0;

    // ---- stage the rows: per row the diagonal block and the contiguous run
    // of coupling blocks (cooperative 16-byte copies), the chunk's Dinv with
    // one bulk copy when it is not factored here.
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sc.stage_bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sc.bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sc.bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sc.n_remote = 0;
        sc.fallback = 0;
        sc.nobulk = 0;
    }
    for (int i = threadIdx.x; i < 2 * 16 * 4; i += kCT) (&sc.tab[0][0][0])[i] = 0.0;
    if (threadIdx.x < 16) sc.req[threadIdx.x] = make_int2(0, 0);
    if constexpr (PH) cs[5] = clock64(); // launch parameters and partition bounds read
    for (int lr = threadIdx.x; lr < nr; lr += kCT) bstart[lr + 1] = sv.ell_cnt[r0 + lr] + 1;
    __syncthreads();
    if constexpr (PH) cs[6] = clock64(); // block counts staged
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
        // the blocks are copied by all threads below (one small TMA copy costs
        // ~70 cycles to issue); only the chunk's Dinv (one contiguous run) is a
        // bulk copy, and the fused kernel factors Dinv itself
        unsigned bytes = 0;
        if (nr > 0 && !a.fused) bytes += 288u * nr;
        if (lane == 0) mbar_expect(smem_u32(&sc.stage_bar), bytes);
        __syncwarp();
        const unsigned bar = smem_u32(&sc.stage_bar);
        if (lane == 0 && nr > 0 && !a.fused)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(dinv)), "l"(sv.rdinv + 36 * r0), "r"(288u * nr), "r"(bar)
                         : "memory");
    }
    __syncthreads(); // bstart complete
    // stage the rows' blocks (diagonal + coupling run): warp per row, one
    // 16-byte cp.async per lane and chunk, all in flight at once (waited for
    // before the plan barrier); the blocks' columns with batched loads
    for (int lr = warp; lr < nr; lr += kCW) {
        const int r = r0 + lr;
        const int b0 = bstart[lr], nb = bstart[lr + 1] - b0;
        const int ncp = min(nb, cap_blocks - b0);
        const double2* d0 = reinterpret_cast<const double2*>(sv.rdiag + 36 * r);
        const double2* o0 = reinterpret_cast<const double2*>(sv.ell_blk + static_cast<size_t>(r) * sv.ell_w * 36);
        const unsigned dst = smem_u32(blk + 36 * b0);
        for (int c = lane; c < 18 * ncp; c += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * c),
                         "l"(c < 18 ? d0 + c : o0 + (c - 18))
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int lr0 = warp; lr0 < nr; lr0 += 4 * kCW) {
        int cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int lr = lr0 + u * kCW;
            cv[u] = -1;
            if (lr < nr && lane < min(bstart[lr + 1] - bstart[lr], cap_blocks - bstart[lr]))
                cv[u] = lane == 0 ? r0 + lr : sv.ell_col[(r0 + lr) * sv.ell_w + lane - 1];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (cv[u] >= 0) bcol[bstart[lr0 + u * kCW] + lane] = cv[u];
    }
    if (sv.ell_w >= 32) // rows wider than a warp (grown ELL): the remaining columns
        for (int lr = warp; lr < nr; lr += kCW) {
            const int nb = min(bstart[lr + 1] - bstart[lr], cap_blocks - bstart[lr]);
            for (int t = 32 + lane; t < nb; t += 32) bcol[bstart[lr] + t] = sv.ell_col[(r0 + lr) * sv.ell_w + t - 1];
        }
    if constexpr (PH) cs[7] = clock64(); // staging issued
    // fused head, part 1 (overlaps the block copies): kOpEps with the trace
    // summed redundantly by every CTA of the partition in one fixed order
    // (same bits everywhere, no exchange), then the block-Jacobi factor.
    double trace_p = 0.0;
    if (a.fused && act) {
        double t = 0.0;
        for (int i = threadIdx.x; i < R1 - R0; i += kCT) t += a.row_trace[R0 + i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) sc.red[warp][0] = t;
        __syncthreads();
        for (int w = 0; w < kCW; ++w) trace_p += sc.red[w][0];
        eps = 1e-8 * trace_p / st.ndof;
    }
    if (a.fused && act) { // block-Jacobi factor: Dinv = (D + eps I)^{-1} by Cholesky (k_precond)
        for (int lr = threadIdx.x; lr < nr; lr += kCT) {
            const double* d = sv.rdiag + 36 * (r0 + lr); // L2: the staged copy may still be in flight
            const double ex = eps;
            // one reciprocal square root per pivot, no divisions on the chain
            double L[6][6], rd[6];
            bool ok = true;
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                double s = d[6 * j + j] + ex;
#pragma unroll
                for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
                if (!(s > 0.0)) ok = false;
                rd[j] = rsqrt(fmax(s, 1e-300));
#pragma unroll
                for (int i = j + 1; i < 6; ++i) {
                    double t = d[6 * i + j];
#pragma unroll
                    for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
                    L[i][j] = t * rd[j];
                }
            }
            if (!ok) atomicCAS(sv.err, 0, kErrFactor);
            double Li[6][6];
#pragma unroll
            for (int c = 0; c < 6; ++c)
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
                    for (int k = 0; k < i; ++k)
                        if (k >= c) s -= L[i][k] * Li[k][c];
                    Li[i][c] = (i < c) ? 0.0 : s * rd[i];
                }
            double* o = dinv + 36 * lr;
#pragma unroll
            for (int r = 0; r < 6; ++r)
#pragma unroll
                for (int c = r; c < 6; ++c) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 6; ++k)
                        if (k >= r && k >= c) s += Li[k][r] * Li[k][c];
                    o[6 * r + c] = s;
                    o[6 * c + r] = s;
                }
        }
        __syncthreads();
    }

    // every CTA's counters and barriers are initialised before any peer
    // appends to its send list
    cluster_barrier();
    if constexpr (PH) cs[0] = clock64();
    // column code of every staged block: >= 0 a row of this CTA, < 0 the
    // remote slot -1 - j. Remote columns are deduplicated: one halo slot per
    // distinct remote row, slots numbered in partition-row order (a CTA-wide
    // scan over marks kept in the halo buffer, which peers only write after
    // the setup barrier), and the owning peer gets one send entry per slot.
    {
        const int R = R1 - R0;
        int* mark = reinterpret_cast<int*>(halo);
        if (4ll * R > 96ll * cap_blocks) { // marks do not fit: barrier path (never for <= 4096 rows)
            if (threadIdx.x == 0) atomicOr(&sc.fallback, 1);
        } else {
            for (int i = threadIdx.x; i < R; i += kCT) mark[i] = 0;
            __syncthreads();
            for (int lr = warp; lr < nr; lr += kCW) {
                const int r = r0 + lr;
                const int b0 = bstart[lr], nb = bstart[lr + 1] - b0;
                if (b0 + nb > cap_blocks && lane == 0) atomicOr(&sc.fallback, 1); // spilled blocks
                for (int t = lane; t < nb && b0 + t < cap_blocks; t += 32) {
                    const int col = bcol[b0 + t];
                    const int crank = (col - R0) / chunk;
                    if (crank == rank) bcode[b0 + t] = (col - R0) - crank * chunk;
                    else mark[col - R0] = 1;
                }
            }
            __syncthreads();
            // exclusive scan of the marks: thread t owns [t * per, (t + 1) * per)
            const int per = (R + kCT - 1) / kCT;
            const int i0 = min(R, threadIdx.x * per), i1 = min(R, i0 + per);
            int cnt = 0;
            for (int i = i0; i < i1; ++i) cnt += mark[i];
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            if (lane == 31) sc.wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                const int v = lane < kCW ? sc.wsum[lane] : 0;
                int w = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, w, o);
                    if (lane >= o) w += u;
                }
                if (lane < kCW) sc.wsum[lane] = w - v;
                if (lane == kCW - 1) sc.n_remote = w;
            }
            __syncthreads();
            int j = sc.wsum[warp] + incl - cnt;
            for (int i = i0; i < i1; ++i) {
                if (!mark[i]) {
                    mark[i] = -1;
                    continue;
                }
                const int crank = i / chunk, cl_row = i - crank * chunk;
                mark[i] = j;
                rptr[j] = cl.map_shared_rank(vm0, crank) + 6 * cl_row;
                ++j;
            }
            __syncthreads();
            // bulk mode: per peer the contiguous range of its rows we need;
            // the peer copies that range into our halo with one bulk DSMEM
            // copy per iteration instead of one 16-byte st.async per value pair
            if (warp < csize) {
                int lo = 0x7fffffff, hi = -1;
                for (int i = warp * chunk + lane; i < min(R, (warp + 1) * chunk); i += 32)
                    if (mark[i] >= 0) {
                        lo = min(lo, i);
                        hi = max(hi, i);
                    }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
                }
                if (lane == 0) {
                    sc.rlo[warp] = lo;
                    sc.rcnt[warp] = hi >= lo ? hi - lo + 1 : 0;
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int h = 0;
                for (int k = 0; k < csize; ++k) {
                    sc.rbase[k] = h;
                    h += sc.rcnt[k];
                }
                if (h > cap_blocks) atomicOr(&cl.map_shared_rank(&sc, 0)->nobulk, 1);
            }
            __syncthreads();
            if (threadIdx.x < csize && sc.rcnt[threadIdx.x] > 0) {
                const int k = threadIdx.x;
                ClusterScalars* peer = cl.map_shared_rank(&sc, k);
                peer->req[rank] = make_int2(sc.rlo[k] - k * chunk, sc.rcnt[k]);
                peer->reqbase[rank] = sc.rbase[k];
            }
        }
    }
    if constexpr (PH) cs[1] = clock64();
    mbar_wait(smem_u32(&sc.stage_bar), 0);
    asm volatile("cp.async.wait_all;" ::: "memory"); // this thread's block copies
    if constexpr (PH) cs[2] = clock64();
    __syncthreads();
    // any overflow in the cluster selects the barrier path everywhere
    if (threadIdx.x == 0 && sc.fallback) atomicOr(&cl.map_shared_rank(&sc, 0)->fallback, 1);
    if (a.warm) { // the warm start's p1 (vm1) and p2 (vm0): published by the barrier below
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int lrw = warp * kRowsPerWarp + slot + g * kCW * kRowsPerWarp;
            if (lane < 30 && lrw < nr) {
                vm1[6 * lrw + comp] = wp1[g];
                vm0[6 * lrw + comp] = wp2[g];
                if (a.warm > 1) a.pa[6 * static_cast<size_t>(r0 + lrw) + comp] = wp1[g]; // the next solve's p2
            }
        }
    }
    cluster_barrier(); // send lists, requests, trace partials, fallback flags (and p1 / p2) complete
    if constexpr (PH) cs[3] = clock64();
    if (a.fused && act && rank == 0 && threadIdx.x == 0) { // kOpEps (newton.cpp:20-24)
        sv.ps[p].trace = trace_p;
        sv.ps[p].eps = eps;
        ++sv.ps[p].iterations;
    }
    for (int i = threadIdx.x; i < 6 * nr; i += kCT) { // (D + eps I)
        const int lr = i / 6, k = i - 6 * lr;
        const int b0 = bstart[lr];
        if (b0 < cap_blocks) blk[36 * b0 + 7 * k] += eps;
    }
    __syncthreads();
    // push: every peer range arrives by bulk copy (st.async partials); the
    // barrier path (DSMEM pulls through rptr) when blocks spill or the halo
    // ranges do not fit
    // (one DSMEM read per CTA, broadcast through shared memory)
    if (threadIdx.x == 0) {
        const ClusterScalars* r0s = cl.map_shared_rank(&sc, 0);
        sc.push_ok = r0s->fallback == 0 && r0s->nobulk == 0;
    }
    __syncthreads();
    const bool push = sc.push_ok != 0;
    if constexpr (PH) cs[4] = clock64();
    const bool bulk = push;
    {
        const int* mark = reinterpret_cast<const int*>(halo); // peers write halo only after the next barrier
        for (int lr = warp; lr < nr; lr += kCW) {
            const int r = r0 + lr;
            const int b0 = bstart[lr], nb = bstart[lr + 1] - b0;
            for (int t = lane; t < nb && b0 + t < cap_blocks; t += 32) {
                const int col = bcol[b0 + t];
                const int k = (col - R0) / chunk;
                if (k == rank) continue;
                const int j = bulk ? sc.rbase[k] + (col - R0) - sc.rlo[k] : mark[col - R0];
                bcode[b0 + t] = -1 - j;
                if (bulk) rptr[j] = cl.map_shared_rank(vm0, k) + 6 * ((col - R0) - k * chunk);
            }
        }
    }
    __syncthreads();
    const int n_remote = sc.n_remote;

    const int row_step = kCW * kRowsPerWarp;
    // (A v) row comp over the staged blocks with local columns
    // skip_diag: the row's diagonal block is left out; the caller adds
    // (D + eps I) v_i itself where it is known without a product (v = Dinv w
    // gives exactly w for the operator whose diagonal block is Dinv^-1)
    auto spmv_local = [&](int lr, const double* vloc, bool skip_diag = false) -> double {
        const int b0 = bstart[lr], bs = max(b0, min(bstart[lr + 1], cap_blocks));
        double y0 = 0.0, y1 = 0.0;
        int s = skip_diag && b0 < bs ? b0 + 1 : b0;
        for (; s + 1 < bs; s += 2) {
            const int c0 = bcode[s], c1 = bcode[s + 1];
            if (c0 >= 0) {
                const double2* M2 = reinterpret_cast<const double2*>(blk + 36 * s + 6 * comp);
                const double2* v2 = reinterpret_cast<const double2*>(vloc + 6 * c0);
                const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2], w0 = v2[0], w1 = v2[1], w2 = v2[2];
                y0 += m0.x * w0.x + m0.y * w0.y + m1.x * w1.x + m1.y * w1.y + m2.x * w2.x + m2.y * w2.y;
            }
            if (c1 >= 0) {
                const double2* M2 = reinterpret_cast<const double2*>(blk + 36 * (s + 1) + 6 * comp);
                const double2* v2 = reinterpret_cast<const double2*>(vloc + 6 * c1);
                const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2], w0 = v2[0], w1 = v2[1], w2 = v2[2];
                y1 += m0.x * w0.x + m0.y * w0.y + m1.x * w1.x + m1.y * w1.y + m2.x * w2.x + m2.y * w2.y;
            }
        }
        if (s < bs && bcode[s] >= 0) {
            const double2* M2 = reinterpret_cast<const double2*>(blk + 36 * s + 6 * comp);
            const double2* v2 = reinterpret_cast<const double2*>(vloc + 6 * bcode[s]);
            const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2], w0 = v2[0], w1 = v2[1], w2 = v2[2];
            y0 += m0.x * w0.x + m0.y * w0.y + m1.x * w1.x + m1.y * w1.y + m2.x * w2.x + m2.y * w2.y;
        }
        return y0 + y1;
    };
    // staged blocks with remote columns: values from `hv` (halo rows, push
    // path) or through DSMEM from the peer's m buffer at `moff` (fallback),
    // then spilled blocks (global memory + DSMEM, fallback only)
    auto spmv_remote = [&](int lr, const double* hv, ptrdiff_t moff, double y, bool skip_diag = false) -> double {
        // staged blocks [b0, bs), spilled [bs, b1); a row may lie wholly past
        // the budget (bs = b0)
        const int b0 = bstart[lr], b1 = bstart[lr + 1], bs = max(b0, min(b1, cap_blocks));
        for (int s = b0; s < bs; ++s) {
            const int code = bcode[s];
            if (code >= 0) continue;
            const double2* M2 = reinterpret_cast<const double2*>(blk + 36 * s + 6 * comp);
            const double2* v2 = reinterpret_cast<const double2*>(
                hv ? hv + 6 * (-1 - code) : rptr[-1 - code] + moff);
            const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2], w0 = v2[0], w1 = v2[1], w2 = v2[2];
            y += m0.x * w0.x + m0.y * w0.y + m1.x * w1.x + m1.y * w1.y + m2.x * w2.x + m2.y * w2.y;
        }
        for (int s = bs; s < b1; ++s) { // spilled block
            const int r = r0 + lr, t = s - b0;
            if (t == 0 && skip_diag) continue;
            const int col = t == 0 ? r : sv.ell_col[r * sv.ell_w + t - 1];
            const double* M = (t == 0 ? sv.rdiag + 36 * r
                                      : sv.ell_blk + (static_cast<size_t>(r) * sv.ell_w + t - 1) * 36) + 6 * comp;
            const int crank = (col - R0) / chunk, cl_row = (col - R0) - crank * chunk;
            const double* v = cl.map_shared_rank(vm0, crank) + moff + 6 * cl_row;
            double ya = 0.0;
            for (int c = 0; c < 6; ++c) ya += M[c] * v[c];
            if (t == 0) ya += eps * v[comp];
            y += ya;
        }
        return y;
    };

    // (A v1, A v0) rows in one pass over the staged blocks (warm start): the
    // matrix is read once and the two vectors' DSMEM loads overlap; v1 = vm1
    // (peers' copies at moff = m_off), v0 = vm0 (moff = 0). Same per-block
    // summation order as spmv_local / spmv_remote, so each result equals the
    // single-vector SpMV.
    auto spmv_pair = [&](int lr, double& y1, double& y0) {
        const int b0 = bstart[lr], b1 = bstart[lr + 1], bs = max(b0, min(b1, cap_blocks));
        double l1a = 0.0, l1b = 0.0, l0a = 0.0, l0b = 0.0;
        int s = b0;
        auto dot6 = [&](int blkidx, const double* v) {
            const double2* M2 = reinterpret_cast<const double2*>(blk + 36 * blkidx + 6 * comp);
            const double2* v2 = reinterpret_cast<const double2*>(v);
            const double2 m0 = M2[0], m1 = M2[1], m2 = M2[2], w0 = v2[0], w1 = v2[1], w2 = v2[2];
            return m0.x * w0.x + m0.y * w0.y + m1.x * w1.x + m1.y * w1.y + m2.x * w2.x + m2.y * w2.y;
        };
        for (; s + 1 < bs; s += 2) {
            const int c0 = bcode[s], c1 = bcode[s + 1];
            if (c0 >= 0) {
                l1a += dot6(s, vm1 + 6 * c0);
                l0a += dot6(s, vm0 + 6 * c0);
            }
            if (c1 >= 0) {
                l1b += dot6(s + 1, vm1 + 6 * c1);
                l0b += dot6(s + 1, vm0 + 6 * c1);
            }
        }
        if (s < bs && bcode[s] >= 0) {
            l1a += dot6(s, vm1 + 6 * bcode[s]);
            l0a += dot6(s, vm0 + 6 * bcode[s]);
        }
        y1 = l1a + l1b;
        y0 = l0a + l0b;
        for (int t = b0; t < bs; ++t) {
            const int code = bcode[t];
            if (code >= 0) continue;
            const double* base = rptr[-1 - code];
            const double d1 = dot6(t, base + m_off), d0 = dot6(t, base);
            y1 += d1;
            y0 += d0;
        }
        if (bs < b1) { // spilled blocks: the single-vector path
            y1 = spmv_remote(lr, nullptr, m_off, spmv_local(lr, vm1));
            y0 = spmv_remote(lr, nullptr, 0, spmv_local(lr, vm0));
        }
    };

    // ---- init: r = b = -grad, x = 0, u = Dinv r (read by the peers from m1), w = A u.
    // Every lane keeps its (row, component) entries of all PCG vectors in
    // registers (row group g of the warp: local row warp * 5 + slot + g * 80);
    // only m = Dinv w lives in shared memory, double-buffered by parity
    // (vm0 / vm1), because the SpMV of other lanes and CTAs reads it.
    double x[G], r[G], u[G], w[G], z[G], qv[G], sv_[G], pv[G], mr[G];
    bool on[G];
    int lrg[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        lrg[g] = warp * kRowsPerWarp + slot + g * row_step;
        on[g] = lane < 30 && lrg[g] < nr;
        r[g] = on[g] && act ? -sv.rgrad[6 * (r0 + lrg[g]) + comp] : 0.0;
        x[g] = z[g] = qv[g] = sv_[g] = pv[g] = 0.0;
    }
    double bnorm2_ws = -1.0; // ||b||^2 when the warm start computed it
    if constexpr (PH) ci[0] = clock64();
    if (a.warm) {
        // x0 in span{p1, p2}, the previous two solves' solutions (sv.x and
        // a.pa), by the Galerkin condition: [p_i . A p_j] c = [p_i . b] (2x2,
        // one-vector fallback when nearly dependent). Two SpMVs through DSMEM
        // (p1 from vm1, p2 from vm0) and one cluster reduction, rank order.
        double p1[G], p2[G], ap1[G], ap2[G];
#pragma unroll
        for (int g = 0; g < G; ++g) { // in vm1 / vm0 since the plan barrier
            p1[g] = wp1[g];
            p2[g] = wp2[g];
        }
        double l[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int g = 0; g < G; ++g) {
            ap1[g] = ap2[g] = 0.0;
            if (on[g]) spmv_pair(lrg[g], ap1[g], ap2[g]); // ap2 = A p2 (p2 = 0 when warm == 1)
            l[0] += p1[g] * r[g];
            l[1] += p2[g] * r[g];
            l[2] += p1[g] * ap1[g];
            l[3] += p1[g] * ap2[g];
            l[4] += p2[g] * ap2[g];
            l[5] += r[g] * r[g];
        }
        {
            const double va = warp_sum4(l[0], l[1], l[2], l[3], lane), vb = warp_sum4(l[4], l[5], 0.0, 0.0, lane);
            if ((lane & 7) == 0) sc.wred[warp][lane >> 3] = va;
            if ((lane & 7) == 0 && lane < 16) sc.wred[warp][4 + (lane >> 3)] = vb;
        }
        __syncthreads();
        if (threadIdx.x < 6) {
            double t = 0.0;
            for (int k = 0; k < kCW; ++k) t += sc.wred[k][threadIdx.x];
            sc.wsp[threadIdx.x] = t;
        }
        cluster_barrier(); // wsp of every CTA ready; every peer done reading vm0 / vm1
        // one warp per CTA folds the csize CTA records: lane k loads CTA k's
        // record (6 x csize DSMEM loads per CTA, not per thread), a fixed
        // shuffle tree sums them, and lane 0 solves the 2x2 system
        if (warp == 0) { // lane k loads CTA k's record; fixed shuffle tree
            double tt[6];
#pragma unroll
            for (int m = 0; m < 6; ++m) tt[m] = lane < csize ? cl.map_shared_rank(&sc, lane)->wsp[m] : 0.0;
            {
                const double va = warp_sum4(tt[0], tt[1], tt[2], tt[3], lane), vb = warp_sum4(tt[4], tt[5], 0.0, 0.0, lane);
#pragma unroll
                for (int m = 0; m < 4; ++m) tt[m] = __shfl_sync(0xffffffffu, va, 8 * m);
                tt[4] = __shfl_sync(0xffffffffu, vb, 0);
                tt[5] = __shfl_sync(0xffffffffu, vb, 8);
            }
            const double b1 = tt[0], b2 = tt[1], a11 = tt[2], a12 = tt[3], a22 = tt[4];
            double c1 = 0.0, c2 = 0.0;
            const double det = a11 * a22 - a12 * a12;
            bool two = false; // 2x2 Galerkin solution usable
            if (a.warm > 1 && a11 > 0.0 && a22 > 0.0 && det > 1e-8 * a11 * a22) {
                c1 = (b1 * a22 - b2 * a12) / det;
                c2 = (b2 * a11 - b1 * a12) / det;
                two = isfinite(c1) && isfinite(c2);
            }
            if (!two) { // one-vector fallback; a non-finite p2 never enters it
                c2 = 0.0;
                c1 = a11 > 0.0 ? b1 / a11 : 0.0;
                if (!isfinite(c1)) c1 = 0.0;
            }
            if (lane == 0) {
                sc.scal[0] = c1;
                sc.scal[1] = c2;
                sc.scal[2] = tt[5];
            }
        }
        __syncthreads();
        const double c1 = sc.scal[0], c2 = sc.scal[1];
        bnorm2_ws = sc.scal[2];
        if (c2 != 0.0) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                x[g] = c1 * p1[g] + c2 * p2[g];
                r[g] -= c1 * ap1[g] + c2 * ap2[g];
            }
        } else if (c1 != 0.0) { // p2 / A p2 untouched: 0 * NaN never reaches x or r
#pragma unroll
            for (int g = 0; g < G; ++g) {
                x[g] = c1 * p1[g];
                r[g] -= c1 * ap1[g];
            }
        }
        // (no trailing barrier: wsp is never rewritten in this launch, and the
        // barrier above already ordered every peer's reads of vm0 / vm1)
    }
    if constexpr (PH) ci[1] = clock64();
#pragma unroll
    for (int g = 0; g < G; ++g) {
        double uu = 0.0;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const double rc = __shfl_sync(0xffffffffu, r[g], (6 * slot + c) & 31);
            if (on[g]) uu += dinv[36 * lrg[g] + 6 * comp + c] * rc;
        }
        u[g] = uu;
        if (on[g]) vm1[6 * lrg[g] + comp] = uu;
    }
    cluster_barrier();
    if constexpr (PH) ci[2] = clock64();
    // w = A u with u = Dinv r: the diagonal block contributes r itself
#pragma unroll
    for (int g = 0; g < G; ++g)
        w[g] = on[g] ? spmv_remote(lrg[g], nullptr, m_off, r[g] + spmv_local(lrg[g], vm1, true), true) : 0.0;
    // m = Dinv w for iteration 0 (into vm0) and the partials (r.u, w.u, r.r)
    double l_g = 0.0, l_d = 0.0, l_r = 0.0, l_x = 0.0; // l_x: x.x (inexact Newton)
    auto make_m = [&](double* mdst) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            double wc[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) wc[c] = __shfl_sync(0xffffffffu, w[g], (6 * slot + c) & 31);
            double m = 0.0;
            if (on[g]) {
                const double2* d2 = reinterpret_cast<const double2*>(dinv + 36 * lrg[g] + 6 * comp);
                const double2 d0 = d2[0], d1 = d2[1], dd = d2[2];
                m = d0.x * wc[0] + d0.y * wc[1] + d1.x * wc[2] + d1.y * wc[3] + dd.x * wc[4] + dd.y * wc[5];
                mdst[6 * lrg[g] + comp] = m;
                l_g += r[g] * u[g];
                l_d += w[g] * u[g];
                l_r += r[g] * r[g];
                l_x += x[g] * x[g];
            }
            mr[g] = m;
        }
    };
    make_m(vm0);
    if (bulk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // m feeds the bulk copies
    // the fallback path's peers may still read our vm1 (init SpMV) until
    // this barrier; the push path only writes vm1 after a full exchange
    if (!push) cluster_barrier();

    bool done = !act;
    double inv_gamma_old = 0.0, inv_alpha_old = 0.0, bnorm2 = 0.0;
    int it = 0;
    const int ph_at = sv.pcg_phases - 1; // 256 * CTA + 16 * warp of the timed thread
    const bool timed = PH && sv.perf != nullptr && static_cast<int>(blockIdx.x) == (ph_at >> 8) &&
                       static_cast<int>(threadIdx.x) == 32 * ((ph_at >> 4) & 15);
    unsigned long long ph[10] = {}, tc = PH ? clock64() : 0ull;
    if constexpr (PH) ph[8] = tc - c_start;
    auto mark = [&](int k) {
        if constexpr (PH) {
            if (!timed) return;
            const unsigned long long t = clock64();
            ph[k] += t - tc;
            tc = t;
        }
    };
    int n_halo = n_remote;
    if (bulk) {
        n_halo = 0;
        for (int k = 0; k < csize; ++k) n_halo += sc.rcnt[k];
    }
    const unsigned expect = static_cast<unsigned>(32 * csize + 48 * n_halo);
    while (!done) {
        mark(7);
        const int par = it & 1;
        double* mcur = par ? vm1 : vm0;
        double* mnext = par ? vm0 : vm1;
        const ptrdiff_t moff = par ? m_off : 0;
        const unsigned bar = smem_u32(&sc.bar[par]);
        if (push && threadIdx.x == 0) mbar_expect(bar, expect);
        // ---- partials of this CTA: warp trees, then one fixed 32-lane tree
        {
            const double v = warp_sum4(l_g, l_d, l_r, l_x, lane);
            if ((lane & 7) == 0) sc.red[warp][lane >> 3] = v;
        }
        mark(0);
        __syncthreads(); // red[] and this CTA's m (mcur) complete
        mark(1);
        if (a.spread == 1) {
            // every warp folds the CTA's partials (same fixed tree in every
            // warp) and warp k sends them, plus the halo rows consumer k
            // needs, to peer k: one remote store pair and one bulk copy per
            // warp instead of csize of each serialised in one warp
            const double tv = warp_sum4(lane < kCW ? sc.red[lane][0] : 0.0, lane < kCW ? sc.red[lane][1] : 0.0,
                                        lane < kCW ? sc.red[lane][2] : 0.0, lane < kCW ? sc.red[lane][3] : 0.0,
                                        lane);
            const double t0 = __shfl_sync(0xffffffffu, tv, 0), t1 = __shfl_sync(0xffffffffu, tv, 8),
                         t2 = __shfl_sync(0xffffffffu, tv, 16), t3 = __shfl_sync(0xffffffffu, tv, 24);
            if (warp < csize) {
                if (lane == 0) {
                    if (push) {
                        const unsigned dst = mapa(smem_u32(&sc.tab[par][rank][0]), warp);
                        const unsigned pbar = mapa(bar, warp);
                        st_async2(dst, t0, t1, pbar);
                        st_async2(dst + 16, t2, t3, pbar);
                    } else {
                        double* d = &cl.map_shared_rank(&sc, warp)->tab[par][rank][0];
                        d[0] = t0;
                        d[1] = t1;
                        d[2] = t2;
                    d[3] = t3;
                        d[3] = t3;
                    }
                } else if (lane == 1 && bulk) {
                    const int2 rq = sc.req[warp];
                    if (rq.y > 0) {
                        const unsigned dst = mapa(smem_u32(halo + 6 * (par * cap_blocks + sc.reqbase[warp])), warp);
                        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                     ::"r"(dst), "r"(smem_u32(mcur + 6 * rq.x)), "r"(48u * rq.y),
                                     "r"(mapa(bar, warp))
                                     : "memory");
                    }
                }
            }
            if (!bulk) cluster_arrive();
        } else {
            if (warp == kSW) { // the scalar warp: CTA tree and push to every peer
                const double tv = warp_sum4(lane < kCW ? sc.red[lane][0] : 0.0, lane < kCW ? sc.red[lane][1] : 0.0,
                                            lane < kCW ? sc.red[lane][2] : 0.0, lane < kCW ? sc.red[lane][3] : 0.0,
                                            lane);
                const double t0 = __shfl_sync(0xffffffffu, tv, 0), t1 = __shfl_sync(0xffffffffu, tv, 8),
                             t2 = __shfl_sync(0xffffffffu, tv, 16), t3 = __shfl_sync(0xffffffffu, tv, 24);
                if (push && a.spread == 2) {
                    // one remote-store instruction: lane k < 16 sends (r.u, w.u)
                    // to peer k, lane 16 + k sends (r.r, 0)
                    const int peer = lane & 15;
                    if (peer < csize) {
                        const unsigned dst = mapa(smem_u32(&sc.tab[par][rank][0]), peer) + (lane >> 4) * 16u;
                        st_async2(dst, lane < 16 ? t0 : t2, lane < 16 ? t1 : t3, mapa(bar, peer));
                    }
                } else if (lane < csize) {
                    if (push) {
                        const unsigned dst = mapa(smem_u32(&sc.tab[par][rank][0]), lane);
                        const unsigned pbar = mapa(bar, lane);
                        st_async2(dst, t0, t1, pbar);
                        st_async2(dst + 16, t2, t3, pbar);
                    } else {
                        double* d = &cl.map_shared_rank(&sc, lane)->tab[par][rank][0];
                        d[0] = t0;
                        d[1] = t1;
                        d[2] = t2;
                    d[3] = t3;
                        d[3] = t3;
                    }
                }
            }
            if (bulk) { // per consumer one bulk DSMEM copy of the row range it needs
                if (warp == 1 && lane < csize) {
                    const int2 rq = sc.req[lane];
                    if (rq.y > 0) {
                        const unsigned dst = mapa(smem_u32(halo + 6 * (par * cap_blocks + sc.reqbase[lane])), lane);
                        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                     ::"r"(dst), "r"(smem_u32(mcur + 6 * rq.x)), "r"(48u * rq.y),
                                     "r"(mapa(bar, lane))
                                     : "memory");
                    }
                }
            } else {
                cluster_arrive();
            }
        }
        mark(2);
        // local-column half of n = A m while the messages fly
        double nloc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) nloc[g] = on[g] ? w[g] + spmv_local(lrg[g], mcur, true) : 0.0; // m = Dinv w
        mark(3);
        if (push)
            mbar_wait(bar, (it >> 1) & 1);
        else
            cluster_wait();
        mark(4);
        // the scalar warp folds the csize CTA partials (fixed 32-lane tree)
        // and derives the CG scalars while the other warps compute the
        // remote half of n; they meet at named barrier 1
        const double* hv = push ? halo + 6 * par * cap_blocks : nullptr;
        double beta = 0.0, alpha = 0.0;
        bool stop = false;
        const bool folder = a.fold_all || warp == kSW; // fold_all: every warp, no hand-off
        if (folder) {
            double2 gd = make_double2(0.0, 0.0), rx = make_double2(0.0, 0.0);
            if (lane < 16) {
                gd = *reinterpret_cast<const double2*>(&sc.tab[par][lane][0]);
                rx = *reinterpret_cast<const double2*>(&sc.tab[par][lane][2]);
            }
            const double fv = warp_sum4(gd.x, gd.y, rx.x, rx.y, lane);
            const double gamma = __shfl_sync(0xffffffffu, fv, 0), delta = __shfl_sync(0xffffffffu, fv, 8),
                         rr = __shfl_sync(0xffffffffu, fv, 16), xx = __shfl_sync(0xffffffffu, fv, 24);
            if (it == 0) bnorm2 = bnorm2_ws >= 0.0 ? bnorm2_ws : rr;
            stop = bnorm2 == 0.0 || rr <= a.tol * a.tol * bnorm2 || it >= a.max_iters ||
                   (inexact && rr <= a.eta_loose * a.eta_loose * bnorm2 && xx > xcut2);
            // beta = gamma / gamma_old, alpha = gamma / (delta - beta gamma / alpha_old),
            // with the previous iteration's reciprocals: one division on the
            // critical path
            beta = gamma * inv_gamma_old;
            alpha = a.fast_rcp ? gamma * fast_rcp(delta - beta * gamma * inv_alpha_old)
                               : gamma / (delta - beta * gamma * inv_alpha_old);
            stop = stop || !(alpha > 0.0) || !isfinite(alpha); // breakdown
            if (!a.fold_all) {
                if (lane == 0) {
                    sc.scal[0] = beta;
                    sc.scal[1] = alpha;
                    sc.scal[2] = stop ? 1.0 : 0.0;
                }
                asm volatile("bar.arrive 1, %0;" ::"r"(kCT) : "memory");
            }
            inv_gamma_old = fast_rcp(gamma); // off the critical path: next iteration
            inv_alpha_old = fast_rcp(alpha);
        }
        // remote_first: the other warps take the remote half of n while the
        // scalar warp folds (it needs no scalar); else they keep the shared-
        // memory pipe idle for the scalar warp's shuffle tree and take it after
        double nrem[G];
        const bool early = a.remote_first && !folder;
        if (early) {
#pragma unroll
            for (int g = 0; g < G; ++g) nrem[g] = on[g] ? spmv_remote(lrg[g], hv, moff, nloc[g], true) : 0.0;
        }
        if (!folder) {
            asm volatile("bar.sync 1, %0;" ::"r"(kCT) : "memory");
            beta = sc.scal[0];
            alpha = sc.scal[1];
            stop = sc.scal[2] != 0.0;
        }
        if (stop) break; // uniform across the CTA and the cluster
        if (!early) {
#pragma unroll
            for (int g = 0; g < G; ++g) nrem[g] = on[g] ? spmv_remote(lrg[g], hv, moff, nloc[g], true) : 0.0;
        }
        mark(5);
        // ---- the recurrences, then m = Dinv w and the partials of the next
        // iteration (register-resident)
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (!on[g]) continue;
            const double n = nrem[g];
            z[g] = n + beta * z[g];
            qv[g] = mr[g] + beta * qv[g];
            sv_[g] = w[g] + beta * sv_[g];
            pv[g] = u[g] + beta * pv[g];
            x[g] += alpha * pv[g];
            r[g] -= alpha * sv_[g];
            u[g] -= alpha * qv[g];
            w[g] -= alpha * z[g];
        }
        l_g = l_d = l_r = l_x = 0.0;
        make_m(mnext);
        if (bulk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mark(6);
        ++it;
    }
    const unsigned long long c_loop_end = PH ? clock64() : 0ull;
#pragma unroll
    for (int g = 0; g < G; ++g)
        if (on[g]) sv.x[6 * (r0 + lrg[g]) + comp] = x[g];
    if (rank == 0 && threadIdx.x == 0) {
        sv.ps[p].pcg_iters = it;
        sv.ps[p].pcg_total += it;
        sv.ps[p].pcg_done = 1;
    }
    if (a.fused) { // ||dq||_inf of this CTA's rows -> rank 0's dqm[rank]
        double m = 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g)
            if (on[g]) m = fmax(m, fabs(x[g]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (lane == 0) sc.red[warp][0] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            double mm = 0.0;
            for (int w = 0; w < kCW; ++w) mm = fmax(mm, sc.red[w][0]);
            cl.map_shared_rank(&sc, 0)->dqm[rank] = mm;
        }
    }
    cluster_barrier(); // no CTA leaves while a peer may still touch its shared memory
    if (a.fused && rank == 0 && threadIdx.x == 0) {
        if (act) {
            double mm = 0.0;
            for (int k = 0; k < csize; ++k) mm = fmax(mm, sc.dqm[k]);
            sv.ps[p].dq_inf = mm;
        }
        // the last partition's cluster takes kOpNewtonCheck for all of them
        __threadfence();
        if (atomicAdd(a.ticket, 1u) == static_cast<unsigned>(sv.n_parts - 1)) {
            *a.ticket = 0u;
            __threadfence();
            // every partition's fields read from L2 (ld.global.cg, after the
            // fence that follows the ticket) in one batch per partition, not
            // as a chain of volatile loads and read-modify-writes
            PartState* ps = sv.ps;
            int any_act = 0, any_srch = 0, tot = 0;
            for (int q = 0; q < sv.n_parts; ++q) {
                const int itq = __ldcg(&ps[q].pcg_iters), actq = __ldcg(&ps[q].active),
                          srchq = __ldcg(&ps[q].searching);
                const double dqq = __ldcg(&ps[q].dq_inf), tolq = __ldcg(&ps[q].tol);
                tot += itq;
                bool still = actq != 0;
                if (still && dqq < tolq) {
                    ps[q].final_update = dqq;
                    ps[q].converged = 1;
                    ps[q].active = 0;
                    still = false;
                }
                any_act |= still;
                any_srch |= srchq != 0;
            }
            if (a.ctrl) {
                a.ctrl->pcg_total += tot;
                a.ctrl->any_active = any_act;
                a.ctrl->any_searching = any_srch;
            }
            if (a.hd.graph) {
                if (a.hd.has_step)
                    cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(a.hd.step), any_act ? 1u : 0u);
                if (a.close_loop && !any_act) // the folded tail never runs: close the Newton loop here
                    cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(a.hd.newton), 0u);
            }
        }
    }
    if constexpr (PH) {
        if (timed) {
            ph[7] = it;
            ph[9] = clock64() - c_loop_end;
            for (int k = 0; k < 10; ++k) atomicAdd(&sv.perf->phase[k], ph[k]);
            // setup sub-phases: start -> params -> counts -> staging issued ->
            // first cluster barrier -> exchange plan -> rest of the setup
            const unsigned long long pts[6] = {cs[5], cs[6], cs[7], cs[0], cs[3], c_start + ph[8]};
            unsigned long long prev = c_start;
            for (int k = 0; k < 6; ++k) {
                atomicAdd(&sv.perf->phase[10 + k], pts[k] - prev);
                prev = pts[k];
            }
            // init sub-phases: [cs[3], ci0) eps + send plan, [ci0, ci1) warm
            // start, [ci1, ci2) u + barrier, [ci2, loop) initial SpMV + m
            const unsigned long long qi[5] = {cs[3], ci[0], ci[1], ci[2], c_start + ph[8]};
            for (int k = 0; k < 4; ++k) atomicAdd(&sv.perf->phase[16 + k], qi[k + 1] - qi[k]);
        }
    }
    if (sv.perf && it > 0) {
        // algorithmic bytes of this partition's solve: every CTA counts the
        // blocks of its own rows (one row per thread, warp sums; integer-valued
        // doubles, so the atomic order does not matter) instead of one thread
        // walking all the partition's rows after the solve
        const int r = r0 + static_cast<int>(threadIdx.x);
        const int nb = r < r1 ? sv.ell_cnt[r] + 1 : 0;
        const int nw = __reduce_add_sync(0xffffffffu, nb);
        const int rw = __reduce_add_sync(0xffffffffu, r < r1 ? 1 : 0);
        if ((threadIdx.x & 31) == 0 && rw > 0)
            atomicAdd(&sv.perf->bytes, static_cast<double>(it) * (288.0 * nw + 504.0 * rw));
        for (int rr = r + kCT; rr < r1; rr += kCT) // chunks wider than the CTA (not on the fused path)
            atomicAdd(&sv.perf->bytes, static_cast<double>(it) * (288.0 * (sv.ell_cnt[rr] + 1) + 504.0));
    }
    if (sv.perf && threadIdx.x == 0) {
        if (rank == 0) atomicAdd(&sv.perf->iters, static_cast<unsigned long long>(it));
        if (blockIdx.x == 0) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            atomicAdd(&sv.perf->ns, t1 - t_start);
            atomicAdd(&sv.perf->launches, 1ull);
        }
    }
}

} // namespace

// Ticket of the fused kernel's last-cluster decision; launches on one device
// are stream ordered.
__device__ unsigned g_pcg_ticket = 0;

static unsigned* pcg_ticket() { // resolved once per device, outside any graph capture
    static void* cache[64] = {};
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    if (!cache[dev & 63]) CUDA_CHECK(cudaGetSymbolAddress(&cache[dev & 63], g_pcg_ticket));
    return static_cast<unsigned*>(cache[dev & 63]);
}

template <int G>
static void cluster_attrs() {
    cudaFuncSetAttribute(k_pcg_cluster<G, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_pcg_cluster<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmemBytes);
    cudaFuncSetAttribute(k_pcg_cluster<G, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_pcg_cluster<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmemBytes);
}

int pcg_cluster_size() {
    static int c = 0;
    if (c == 0) {
        (void)pcg_ticket();
        cluster_attrs<1>();
        cluster_attrs<2>();
        cluster_attrs<4>();
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
        if (cudaOccupancyMaxActiveClusters(&n, k_pcg_cluster<4, false>, &cfg) != cudaSuccess || n < 1) c = 8;
        cudaGetLastError();
    }
    return c;
}

void launch_pcg_cluster(const SolverView& sv, int max_rows_per_part, double* pbuf, double tol,
                        int max_iters, cudaStream_t s, const PcgFuse* fuse) {
    if (sv.n_rows == 0) return;
    const int cmax = pcg_cluster_size();
    static const int min_rows = [] {
        const char* e = std::getenv("DABD_GPU_PCG_MIN_ROWS");
        return e ? std::max(8, std::atoi(e)) : 32;
    }();
    // >= ~min_rows rows per CTA; at least 2 CTAs: st.async / bulk DSMEM
    // copies need a cluster of two or more (a surplus CTA gets no rows)
    int csize = 2;
    while (csize < cmax && csize * min_rows < max_rows_per_part) csize *= 2;
    // largest per-partition chunk under the per-partition rule of k_pcg_cluster
    const int cmax_rows = std::max(std::min(max_rows_per_part, min_rows), (max_rows_per_part + csize - 1) / csize);
    // register-resident row groups per warp (kCW warps x kRowsPerWarp rows each)
    const int groups = (cmax_rows + kCW * kRowsPerWarp - 1) / (kCW * kRowsPerWarp);
    if (groups > 4) throw Error("pcg: cluster chunk exceeds 4 row groups per warp");
    PcgArgs a{pbuf, nullptr, nullptr, tol, max_iters, 0, nullptr, nullptr, CondHandles{}, nullptr, 0};
    static const int warm = [] {
        const char* e = std::getenv("DABD_GPU_PCG_WARM");
        return e ? std::atoi(e) : 2;
    }();
    a.warm = warm;
    a.min_rows = min_rows;
    static const int spread = [] {
        const char* e = std::getenv("DABD_GPU_PCG_SPREAD");
        return e ? std::atoi(e) : 0;
    }();
    a.spread = spread;
    static const int fold_all = [] {
        const char* e = std::getenv("DABD_GPU_PCG_FOLD_ALL");
        return e ? std::atoi(e) : 0;
    }();
    a.fold_all = fold_all;
    static const int remote_first = [] {
        const char* e = std::getenv("DABD_GPU_PCG_REMOTE_FIRST");
        return e ? std::atoi(e) : 0;
    }();
    a.remote_first = remote_first;
    static const int frcp = [] {
        const char* e = std::getenv("DABD_GPU_PCG_FAST_RCP");
        return e ? std::atoi(e) : 0;
    }();
    a.fast_rcp = frcp;
    a.eta_loose = 0.0;
    a.eta_factor = 0.0;
    if (fuse) {
        a.fused = 1;
        a.row_trace = fuse->row_trace;
        a.ctrl = fuse->ctrl;
        a.hd = fuse->hd;
        a.ticket = pcg_ticket();
        a.eta_loose = fuse->eta_loose;
        a.eta_factor = fuse->eta_factor;
        a.close_loop = fuse->close_loop ? 1 : 0;
    }
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
    const bool ph = sv.pcg_phases != 0;
    auto go = [&](auto kern) { DABD_LAUNCH("k_pcg", s, CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, sv, a, csize, cmax_rows))); };
    if (groups <= 1) ph ? go(k_pcg_cluster<1, true>) : go(k_pcg_cluster<1, false>);
    else if (groups == 2) ph ? go(k_pcg_cluster<2, true>) : go(k_pcg_cluster<2, false>);
    else ph ? go(k_pcg_cluster<4, true>) : go(k_pcg_cluster<4, false>);
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

int pcg_grid_blocks() {
    static int g = 0;
    if (g == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_grid, kGT, 0);
        g = std::max(1, sms * std::min(std::max(per_sm, 1), 1));
    }
    return g;
}

void launch_pcg_grid(const SolverView& sv, double* vecs, double* partials, double tol, int max_iters,
                     cudaStream_t s, double eta_loose, double eta_factor) {
    if (sv.n_rows == 0) return;
    if (sv.n_parts > kGW) throw Error("pcg: grid kernel folds at most 16 partitions per launch");
    const size_t n = 6 * static_cast<size_t>(sv.n_rows);
    GridVecs v{vecs, vecs + n, vecs + 2 * n, vecs + 3 * n, vecs + 4 * n, vecs + 5 * n, vecs + 6 * n,
               vecs + 7 * n, vecs + 8 * n, vecs + 9 * n};
    PcgArgs a{nullptr, partials, nullptr, tol, max_iters};
    a.eta_loose = eta_loose;
    a.eta_factor = eta_factor;
    static const int warm = [] {
        const char* e = std::getenv("DABD_GPU_PCG_WARM");
        return e ? std::min(std::atoi(e), 1) : 1;
    }();
    a.warm = warm;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pcg_grid_blocks());
    cfg.blockDim = dim3(kGT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DABD_LAUNCH("k_pcg_grid", s, CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_pcg_grid, sv, a, v)));
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
