// Kernels of the batched local solve: energies + PSD projection, active-set
// filtering, deterministic BSR assembly, block-Jacobi PCG, line-search
// trial states, CCD and segment reductions. Orchestrated by engine.cu.
#include "geometry.cuh"
#include "energy.cuh"
#include "kernels.hpp"
#include "scalar_ops.cuh"

#include <cub/cub.cuh>

#include <cfloat>

#include "instrument.hpp"

namespace dabd_gpu {

namespace {

constexpr int kB = 128;
constexpr int kCH = 1024; // segment-sum chunk (k_segsum)
constexpr int kECH = kB;  // k_energy chunk: one entry per thread (latency-bound entries)

__device__ __forceinline__ void load6(const double* src, double (&d)[6]) {
    const double2* s = reinterpret_cast<const double2*>(src);
    const double2 a = s[0], b = s[1], c = s[2];
    d[0] = a.x;
    d[1] = a.y;
    d[2] = b.x;
    d[3] = b.y;
    d[4] = c.x;
    d[5] = c.y;
}

__device__ __forceinline__ void store6(double* dst, const double (&d)[6]) {
    double2* s = reinterpret_cast<double2*>(dst);
    s[0] = make_double2(d[0], d[1]);
    s[1] = make_double2(d[2], d[3]);
    s[2] = make_double2(d[4], d[5]);
}

__device__ __forceinline__ bool part_flag(const SolverView& sv, int p, int which) {
    const PartState& s = sv.ps[p];
    return which == 0 ? s.active != 0 : (which == 1 ? s.searching != 0 : true);
}

// ---------------------------------------------------------------------------
// Body terms: value (+ gradient + PSD-clamped 6x6 block) per dynamic row
// (objective.cpp:117-141, 143-167).
// ---------------------------------------------------------------------------
// iter_begin: block 0 also takes kOpIterBegin (resets of the per-iteration
// partition counters, before any later kernel of the iteration reads them).
__global__ void k_body_terms(SolverView sv, const double* qsrc, int with_derivs, int which,
                             int* reset_counter, FrameCtrl* iter_begin) {
    if (reset_counter && blockIdx.x == 0 && threadIdx.x == 0) *reset_counter = 0;
    if (iter_begin && blockIdx.x == 0) {
        for (int p = threadIdx.x; p < sv.n_parts; p += blockDim.x) {
            PartState& st = sv.ps[p];
            st.dq_inf = 0.0;
            st.toi_earliest = 2.0;
            st.n_candidates = 0;
            st.n_active_contacts = 0;
        }
        if (threadIdx.x == 0) ++iter_begin->exec_newton;
    }
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < sv.n_rows; r += gridDim.x * blockDim.x) {
        const int p = sv.rpart[r] - sv.part_base;
        if (!part_flag(sv, p, which)) continue;
        const int i = sv.rinst[r];
        const int b = sv.ibody[i];
        double q[6], qt[6];
        load6(qsrc + 6 * i, q);
        load6(sv.iqt + 6 * i, qt);
        const double* k = sv.sc.mblk + 6 * b;
        double diff[6], md[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) diff[j] = q[j] - qt[j];
        // M diff with the two 3x3 blocks on (0,2,3) and (1,4,5)
        md[0] = k[0] * diff[0] + k[1] * diff[2] + k[2] * diff[3];
        md[2] = k[1] * diff[0] + k[3] * diff[2] + k[4] * diff[3];
        md[3] = k[2] * diff[0] + k[4] * diff[2] + k[5] * diff[3];
        md[1] = k[0] * diff[1] + k[1] * diff[4] + k[2] * diff[5];
        md[4] = k[1] * diff[1] + k[3] * diff[4] + k[4] * diff[5];
        md[5] = k[2] * diff[1] + k[4] * diff[4] + k[5] * diff[5];
        double ein = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) ein += diff[j] * md[j];
        ein *= 0.5;
        const double h2 = sv.h * sv.h;
        const double ik = sv.iinvk[i];
        const double w = (sv.kappa_arap * sv.sc.arap_scale[b]) * sv.sc.rest_area[b];
        double g[6] = {0, 0, 0, 0, 0, 0};
        double H[6][6];
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int c = 0; c < 6; ++c) H[a][c] = 0.0;
        const double ear = arap_terms(q, w, h2, g, H, with_derivs != 0);
        double value = ik * (ein + h2 * ear);
        double dz[6];
        const bool anc = sv.ianc[i] != 0;
        double rho = 0.0;
        if (anc) {
            rho = sv.irho[i];
            double s2 = 0.0;
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                dz[j] = (q[j] - sv.iz[6 * i + j]) + sv.iu[6 * i + j];
                s2 += dz[j] * dz[j];
            }
            value += 0.5 * rho * s2;
        }
        sv.rval[r] = value;
        if (!with_derivs) continue;
        double m[6][6];
        mass_full(k, m);
#pragma unroll
        for (int a = 0; a < 6; ++a) {
            g[a] = ik * (md[a] + g[a]);
#pragma unroll
            for (int c = 0; c < 6; ++c) H[a][c] = ik * (m[a][c] + H[a][c]);
        }
        if (anc) {
#pragma unroll
            for (int a = 0; a < 6; ++a) {
                g[a] += rho * dz[a];
                H[a][a] += rho;
            }
        }
        if (sv.project) clamp_body_block(H);
        store6(sv.rgrad + 6 * r, g);
        double* dst = sv.rdiag + 36 * r;
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int c = 0; c < 6; ++c) dst[6 * a + c] = H[a][c];
    }
}

// Value-only body term of row r (instance i) at q: the arithmetic of
// k_body_terms without derivatives, so values (and their sums) agree bitwise.
__device__ __forceinline__ double body_value(const SolverView& sv, int i, const double (&q)[6]) {
    const int b = sv.ibody[i];
    double qt[6];
    load6(sv.iqt + 6 * i, qt);
    const double* k = sv.sc.mblk + 6 * b;
    double diff[6], md[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) diff[j] = q[j] - qt[j];
    md[0] = k[0] * diff[0] + k[1] * diff[2] + k[2] * diff[3];
    md[2] = k[1] * diff[0] + k[3] * diff[2] + k[4] * diff[3];
    md[3] = k[2] * diff[0] + k[4] * diff[2] + k[5] * diff[3];
    md[1] = k[0] * diff[1] + k[1] * diff[4] + k[2] * diff[5];
    md[4] = k[1] * diff[1] + k[3] * diff[4] + k[4] * diff[5];
    md[5] = k[2] * diff[1] + k[4] * diff[4] + k[5] * diff[5];
    double ein = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j) ein += diff[j] * md[j];
    ein *= 0.5;
    const double h2 = sv.h * sv.h;
    const double ik = sv.iinvk[i];
    const double w = (sv.kappa_arap * sv.sc.arap_scale[b]) * sv.sc.rest_area[b];
    double g[6] = {0, 0, 0, 0, 0, 0};
    double H[6][6];
    const double ear = arap_terms(q, w, h2, g, H, false);
    double value = ik * (ein + h2 * ear);
    if (sv.ianc[i] != 0) {
        const double rho = sv.irho[i];
        double s2 = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const double dz = (q[j] - sv.iz[6 * i + j]) + sv.iu[6 * i + j];
            s2 += dz * dz;
        }
        value += 0.5 * rho * s2;
    }
    return value;
}

// ---------------------------------------------------------------------------
// Candidate filter at a configuration: exact static broad-phase predicate
// (margin d_hat) & not static-static & d < d_hat (objective.cpp:91-106).
// mode 0: flag active contacts (derivatives); mode 1: weighted barrier value.
// ---------------------------------------------------------------------------
// pair.kappa_c of objective.cpp:84-105: contact_weight = 1 / popcount(common
// holders), kappa_c = 1 / contact_weight (1 in a single domain). The value
// weighs the barrier by h^2 * (1 / kappa_c) (objective.cpp:135-137), the
// derivatives by h^2 / kappa_c (objective.cpp:187): both restated exactly.
__device__ __forceinline__ double kappa_c_of(const SolverView& sv, int ba, int bb) {
    if (sv.single_domain) return 1.0 / 1.0;
    const int kc = __popc(sv.bmask[ba] & sv.bmask[bb]);
    if (kc == 0) {
        raise(sv.err, kErrNoHolder);
        return 1.0;
    }
    return 1.0 / (1.0 / kc);
}

__global__ void k_filter(SolverView sv, const unsigned long long* keys, int n, const int* dn,
                         KeyFmt fmt, const Box* box, const double* qsrc, int mode, int which,
                         unsigned char* flag, double* val) {
    const int nn = dn ? min(*dn, n) : n;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        if (t >= nn) { // padding past the device-side count
            if (flag) flag[t] = 0;
            if (val) val[t] = 0.0;
            continue;
        }
        int a, b, v, e;
        fmt.unpack(keys[t], a, b, v, e);
        const int p = sv.ipart[a] - sv.part_base;
        bool act = false;
        double value = 0.0;
        if (part_flag(sv, p, which)) {
            const int ba = sv.ibody[a], bb = sv.ibody[b];
            const bool ss = sv.sc.is_static[ba] && sv.sc.is_static[bb];
            if (!ss && overlaps(box[a], box[b])) {
                const double* qa = qsrc + 6 * a;
                const double* qb = qsrc + 6 * b;
                const int vf = sv.sc.vstart[ba] + v, ef = sv.sc.vstart[bb] + e;
                const Box pb = point_box(sv.sc, qa, qa, false, vf);
                const Box eb = edge_box(sv.sc, qb, qb, false, ef, sv.d_hat);
                if (overlaps(pb, eb)) {
                    if (mode == 0) atomicAdd(&sv.ps[p].n_candidates, 1);
                    const V2 P = world_point(qa, rest_of(sv.sc, vf));
                    const V2 E0 = world_point(qb, rest_of(sv.sc, ef));
                    const V2 E1 = world_point(qb, rest_of(sv.sc, sv.sc.vnext[ef]));
                    const double d = pe_distance(P, E0, E1);
                    if (d < sv.d_hat) {
                        if (d <= 0.0) raise(sv.err, d < 0.0 && d == -1.0 ? kErrDegenerateEdge : kErrBarrierDomain);
                        act = true;
                        if (mode == 1 && d > 0.0) {
                            const double kinv = 1.0 / kappa_c_of(sv, ba, bb); // w of objective.cpp:135
                            const Barrier br = barrier(d, sv.d_hat, sv.kappa_bar);
                            value = (sv.h * sv.h * kinv) * br.b;
                        }
                    }
                }
            }
        }
        if (flag) flag[t] = act ? 1 : 0;
        if (val) val[t] = value;
    }
}

// ---------------------------------------------------------------------------
// World-space contact Hessian C (6x6 over (p, e0, e1), symmetric) -> the
// three DoF-space 6x6 blocks the row assembly sums. x = A xbar + p gives
// d(world)/d(q) = J(xbar) with J = [[1, 0, x, y, 0, 0], [0, 1, 0, 0, x, y]]:
//   TL = J(rp)^T C_pp J(rp), BR = sum_kl J(rk)^T C_kl J(rl),
//   TR = sum_l J(rp)^T C_pl J(rl)  (BL = TR^T).
// DoF alpha -> (world component, coefficient index into (1, x, y)).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int dof_comp(int alpha) { return (alpha == 1 || alpha >= 4) ? 1 : 0; }
__host__ __device__ constexpr int dof_idx(int alpha) { return alpha <= 1 ? 0 : (alpha == 2 || alpha == 4 ? 1 : 2); }

__device__ __forceinline__ double dof_coef(V2 x, int idx) { return idx == 0 ? 1.0 : (idx == 1 ? x.x : x.y); }

__device__ __forceinline__ void store_dof_blocks(double* dst, const double (&C)[6][6], V2 rp, V2 r0,
                                                 V2 r1) {
    const V2 pt[3] = {rp, r0, r1};
#pragma unroll
    for (int a = 0; a < 6; ++a) {
        const int ca = dof_comp(a), ia = dof_idx(a);
        double tl[6], br[6], tr[6];
#pragma unroll
        for (int b = 0; b < 6; ++b) {
            const int cb = dof_comp(b), ib = dof_idx(b);
            // same term order as a (ra outer, rb inner) double loop
            tl[b] = 0.0 + C[ca][cb] * (dof_coef(pt[0], ia) * dof_coef(pt[0], ib));
            double v = 0.0;
#pragma unroll
            for (int ra = 1; ra <= 2; ++ra)
#pragma unroll
                for (int rb = 1; rb <= 2; ++rb)
                    v += C[2 * ra + ca][2 * rb + cb] * (dof_coef(pt[ra], ia) * dof_coef(pt[rb], ib));
            br[b] = v;
            double w = 0.0;
#pragma unroll
            for (int rb = 1; rb <= 2; ++rb) w += C[ca][2 * rb + cb] * (dof_coef(pt[0], ia) * dof_coef(pt[rb], ib));
            tr[b] = w;
        }
        double2* d2 = reinterpret_cast<double2*>(dst + 6 * a);
#pragma unroll
        for (int b = 0; b < 6; b += 2) {
            d2[b / 2] = make_double2(tl[b], tl[b + 1]);
            d2[18 + b / 2] = make_double2(br[b], br[b + 1]);
            d2[36 + b / 2] = make_double2(tr[b], tr[b + 1]);
        }
    }
}

// ---------------------------------------------------------------------------
// Contact terms with the rank-6 PSD projection (energy.cpp:63-94,
// objective.cpp:184-207).
// ---------------------------------------------------------------------------
// Terms of active list entry c (energy.cpp:63-94 + the rank-6 projection).
__device__ __forceinline__ void contact_terms_one(const SolverView& sv, const ContactView& cv, int c) {
    int a, b, v, e;
    cv.fmt.unpack(cv.key[c], a, b, v, e);
    const int ba = sv.ibody[a], bb = sv.ibody[b];
    const int vf = sv.sc.vstart[ba] + v, ef = sv.sc.vstart[bb] + e, ef1 = sv.sc.vnext[ef];
    const V2 rp = rest_of(sv.sc, vf), r0 = rest_of(sv.sc, ef), r1 = rest_of(sv.sc, ef1);
    const double* qa = sv.iq + 6 * a;
    const double* qb = sv.iq + 6 * b;
    const V2 P = world_point(qa, rp), E0 = world_point(qb, r0), E1 = world_point(qb, r1);
    double g[6], A[6][6];
    const double d = pe_distance_full(P, E0, E1, g, A);
    if (!(d > 0.0)) {
        raise(sv.err, kErrBarrierDomain);
        return;
    }
    const Barrier br = barrier(d, sv.d_hat, sv.kappa_bar);
    const double w = (sv.h * sv.h) / kappa_c_of(sv, ba, bb); // h^2 / kappa_c (objective.cpp:187)
    cv.cval[c] = w * br.b;
    // weighted gradient w * b' * t^T g
    const double s = w * br.db;
    double* cg = cv.cgrad + 12 * c;
    cg[0] = s * g[0];
    cg[1] = s * g[1];
    cg[2] = s * (g[0] * rp.x);
    cg[3] = s * (g[0] * rp.y);
    cg[4] = s * (g[1] * rp.x);
    cg[5] = s * (g[1] * rp.y);
    cg[6] = s * (g[2] + g[4]);
    cg[7] = s * (g[3] + g[5]);
    cg[8] = s * (g[2] * r0.x + g[4] * r1.x);
    cg[9] = s * (g[2] * r0.y + g[4] * r1.y);
    cg[10] = s * (g[3] * r0.x + g[5] * r1.x);
    cg[11] = s * (g[3] * r0.y + g[5] * r1.y);
    // A = w (b'' g g^T + b' H_d)
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) A[i][j] = w * (br.ddb * (g[i] * g[j]) + br.db * A[i][j]);
    if (!sv.project) {
        store_dof_blocks(cv.cblk + 108 * static_cast<size_t>(c), A, rp, r0, r1);
        return;
    }
    // G = t t^T = L L^T in closed form: L = Lp (x) I2 with the 3x3 lower
    // Lp = [[sp, 0, 0], [0, l00, 0], [0, l10, l11]] over the points
    // (p, e0, e1), and B = L^T A L. A annihilates the two rigid
    // translations T = 1 (x) e_c (d is translation invariant), so B
    // annihilates L^{-1} T = u (x) e_c with u = Lp^{-1} 1: the projection
    // lives on the 4-dim complement Q = W (x) I2, W = an orthonormal basis
    // of u-perp (Householder). With Kp = Lp W and Pp = Lp^{-T} W:
    //   B4 = (Kp (x) I2)^T A (Kp (x) I2),  C = (Pp (x) I2) clamp(B4) (Pp (x) I2)^T
    // = L^{-T} clamp(B) L^{-1}: a 4x4 Jacobi instead of 6x6.
    const double sp = sqrt(1.0 + rp.x * rp.x + rp.y * rp.y);
    const double g00 = 1.0 + r0.x * r0.x + r0.y * r0.y;
    const double g01 = 1.0 + r0.x * r1.x + r0.y * r1.y;
    const double g11 = 1.0 + r1.x * r1.x + r1.y * r1.y;
    const double l00 = sqrt(g00), l10 = g01 / l00, l11 = sqrt(fmax(g11 - l10 * l10, 1e-300));
    const double ip = 1.0 / sp, i0 = 1.0 / l00, i1 = 1.0 / l11, m10 = -l10 / (l00 * l11);
    double W[3][2];
    {
        double u[3] = {ip, i0, m10 + i1};
        const double un = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
#pragma unroll
        for (int k = 0; k < 3; ++k) u[k] /= un;
        // Householder H = I - 2 v v^T / v^T v, v = u + sign(u0) e0: H u = -sign(u0) e0,
        // so columns 1 and 2 of H span u-perp (orthonormal)
        const double sg = u[0] >= 0.0 ? 1.0 : -1.0;
        const double v[3] = {u[0] + sg, u[1], u[2]};
        const double f = 2.0 / (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int j = 0; j < 2; ++j) W[k][j] = (k == j + 1 ? 1.0 : 0.0) - f * v[k] * v[j + 1];
    }
    double Kp[3][2], Pp[3][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        Kp[0][j] = sp * W[0][j];
        Kp[1][j] = l00 * W[1][j];
        Kp[2][j] = l10 * W[1][j] + l11 * W[2][j];
        Pp[0][j] = ip * W[0][j];
        Pp[1][j] = i0 * W[1][j] + m10 * W[2][j];
        Pp[2][j] = i1 * W[2][j];
    }
    // AK = A (Kp (x) I2): column (b, d) -> 2b + d
    double AK[6][4];
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int d = 0; d < 2; ++d)
                AK[r][2 * b + d] = A[r][d] * Kp[0][b] + A[r][2 + d] * Kp[1][b] + A[r][4 + d] * Kp[2][b];
    double B4[4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
            for (int col = 0; col < 4; ++col)
                B4[2 * a + c2][col] = Kp[0][a] * AK[c2][col] + Kp[1][a] * AK[2 + c2][col] +
                                      Kp[2][a] * AK[4 + c2][col];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i + 1; j < 4; ++j) {
            const double m = 0.5 * (B4[i][j] + B4[j][i]);
            B4[i][j] = m;
            B4[j][i] = m;
        }
    clamp_psd<4>(B4);
    // C = (Pp (x) I2) B4+ (Pp (x) I2)^T
    double PE[6][4]; // (Pp (x) I2) B4+
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
            for (int col = 0; col < 4; ++col)
                PE[2 * i + c2][col] = Pp[i][0] * B4[c2][col] + Pp[i][1] * B4[2 + c2][col];
    double Cf[6][6];
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int d = 0; d < 2; ++d) {
                if (2 * j + d < r) continue;
                const double val = PE[r][d] * Pp[j][0] + PE[r][2 + d] * Pp[j][1];
                Cf[r][2 * j + d] = val;
                Cf[2 * j + d][r] = val;
            }
    store_dof_blocks(cv.cblk + 108 * static_cast<size_t>(c), Cf, rp, r0, r1);
}

__global__ void __launch_bounds__(kB)
    k_contact_terms(SolverView sv, ContactView cv) {
    const int nc = min(cv.ls->n_act, cv.n);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x)
        contact_terms_one(sv, cv, cv.act[k]);
}

// ---------------------------------------------------------------------------
// Fused objective value (objective.cpp:117-141) for the Newton start and
// every line-search trial, replacing inst_boxes + body_terms + segsum +
// filter + segsum (+ make_trial, scalar(Accept)):
//   q of instance i: iq (qmode 0), the trial iq + alpha dq of partitions
//   still searching (qmode 1, k_make_trial's unfused arithmetic);
//   blocks [0, ncr): kCH-row chunks of body values, blocks [ncr, ncr + nck):
//   kCH-entry chunks of the candidate list with the filter's exact value
//   predicate (body boxes recomputed from the vertices, margin d_hat).
// Chunks of kECH entries (one per thread: every entry is a long dependent
// load chain, so parallelism wins) sum per partition with a fixed tree, and
// the last block folds rows then candidates into dst in block order: the same
// bits for the Newton start and every trial (deterministic, graph == eager).
// accept: the last block then takes kOpAccept (scalar_block).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void eval_q(const SolverView& sv, int i, int qmode, double (&q)[6]) {
    load6(sv.iq + 6 * i, q);
    if (qmode == 0) return;
    const int r = sv.irow[i];
    const int p = sv.ipart[i] - sv.part_base;
    const PartState& st = sv.ps[p];
    if (r >= 0 && (qmode == 1 ? st.searching != 0 : st.accepted != 0)) {
        const double alpha = st.alpha;
        double dq[6];
        load6(sv.x + 6 * r, dq);
#pragma unroll
        for (int k = 0; k < 6; ++k) q[k] = xadd(q[k], xmul(alpha, dq[k]));
    }
}

// filter value of candidate t (k_filter, mode 1)
__device__ __forceinline__ double cand_value(const SolverView& sv, unsigned long long key, KeyFmt fmt,
                                             int qmode, int which) {
    int a, b, v, e;
    fmt.unpack(key, a, b, v, e);
    const int ba = sv.ibody[a], bb = sv.ibody[b]; // beside the partition index, not after its flag
    const int p = sv.ipart[a] - sv.part_base;
    if (!part_flag(sv, p, which)) return 0.0;
    if (sv.sc.is_static[ba] && sv.sc.is_static[bb]) return 0.0;
    double qa[6], qb[6];
    eval_q(sv, a, qmode, qa);
    eval_q(sv, b, qmode, qb);
    // (the body-box test of the broad phase is implied by the point / edge box
    // test below, see k_contact_select, and is not repeated)
    const int vf = sv.sc.vstart[ba] + v, ef = sv.sc.vstart[bb] + e;
    const Box pb = point_box(sv.sc, qa, qa, false, vf);
    const Box eb = edge_box(sv.sc, qb, qb, false, ef, sv.d_hat);
    if (!overlaps(pb, eb)) return 0.0;
    const V2 P = world_point(qa, rest_of(sv.sc, vf));
    const V2 E0 = world_point(qb, rest_of(sv.sc, ef));
    const V2 E1 = world_point(qb, rest_of(sv.sc, sv.sc.vnext[ef]));
    const double d = pe_distance(P, E0, E1);
    if (!(d < sv.d_hat)) return 0.0;
    if (d <= 0.0) {
        raise(sv.err, d < 0.0 && d == -1.0 ? kErrDegenerateEdge : kErrBarrierDomain);
        return 0.0;
    }
    const double kinv = 1.0 / kappa_c_of(sv, ba, bb); // w of objective.cpp:135
    const Barrier br = barrier(d, sv.d_hat, sv.kappa_bar);
    return (sv.h * sv.h * kinv) * br.b;
}

struct EnergyArgs {
    const unsigned long long* keys;
    int cap;         // list capacity (entries past *dn are padding, value 0)
    const int* dn;
    KeyFmt fmt;
    int qmode, which;
    int ncr;         // row chunks (the remaining blocks are candidate chunks)
    double* partial; // [gridDim][P]
    unsigned* ticket;
    double* dst;     // PartState field of partition 0
    int stride;      // PartState stride in doubles
    int accept;      // run kOpAccept in the last block
    FrameCtrl* ctrl;
    CondHandles hd;
    int apply;       // accept: the last block also applies iq += alpha dq (k_accept_trial's work)
    int tail;        // captured fused Newton body: when no partition searches any more, the last
    int max_iters;   // block also takes kOpNewtonTail (the loop bound, the Newton WHILE
    int* iter_reset; // condition, the next iteration's resets): one node fewer per iteration
};

__device__ __forceinline__ void accept_trial_range(const SolverView& sv, int i0, int step) {
    for (int i = i0; i < sv.n_inst; i += step) {
        const int p = sv.ipart[i] - sv.part_base;
        if (!sv.ps[p].accepted || sv.irow[i] < 0) continue;
        double q[6];
        eval_q(sv, i, 2, q);
        store6(sv.iq + 6 * i, q);
    }
}

// accept_trial_range run by the last block alone: the partitions' accept
// decisions staged in shared memory (alpha, or -1 when rejected), then
// kApplyU instances per thread in flight (index loads, then state loads,
// then stores), so the L2 round trips of a thread's instances overlap
// instead of chaining through the stores (~8 x 3 dependent trips per thread
// on pile-1k otherwise). Same predicate and arithmetic as eval_q(qmode 2).
constexpr int kApplyU = 2;
__device__ __forceinline__ void accept_trial_block(const SolverView& sv, double* s_alpha) {
    const int P = sv.n_parts;
    for (int p = threadIdx.x; p < P; p += blockDim.x)
        s_alpha[p] = sv.ps[p].accepted ? sv.ps[p].alpha : -1.0;
    __syncthreads();
    for (int base = threadIdx.x; base < sv.n_inst; base += kApplyU * blockDim.x) {
        int row[kApplyU];
        double alpha[kApplyU];
#pragma unroll
        for (int u = 0; u < kApplyU; ++u) {
            const int i = base + u * blockDim.x;
            row[u] = -1;
            alpha[u] = 0.0;
            if (i < sv.n_inst) {
                const int r = sv.irow[i];
                const double a = s_alpha[sv.ipart[i] - sv.part_base];
                if (a >= 0.0 && r >= 0) {
                    row[u] = r;
                    alpha[u] = a;
                }
            }
        }
        double q[kApplyU][6], dq[kApplyU][6];
#pragma unroll
        for (int u = 0; u < kApplyU; ++u) {
            if (row[u] < 0) continue;
            load6(sv.iq + 6 * (base + u * blockDim.x), q[u]);
            load6(sv.x + 6 * row[u], dq[u]);
        }
#pragma unroll
        for (int u = 0; u < kApplyU; ++u) {
            if (row[u] < 0) continue;
#pragma unroll
            for (int k = 0; k < 6; ++k) q[u][k] = xadd(q[u][k], xmul(alpha[u], dq[u][k]));
            store6(sv.iq + 6 * (base + u * blockDim.x), q[u]);
        }
    }
}

// sum_{k in [k0, k1), k = k0 + lane mod 32} part[k * P + p] in ascending k
// (the order of the plain strided loop, so the same bits), loads issued
// eight at a time ahead of the dependent adds.
__device__ __forceinline__ double fold_partials(const double* part, int P, int p, int k0, int k1, int lane) {
    double s = 0.0;
    for (int k = k0 + lane; k < k1; k += 8 * 32) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int kk = k + 32 * u;
            v[u] = kk < k1 ? __ldcg(part + static_cast<size_t>(kk) * P + p) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k + 32 * u < k1) s += v[u];
    }
    return s;
}

__global__ void __launch_bounds__(kB) k_energy(SolverView sv, EnergyArgs ea) {
    __shared__ double sh[kB];
    __shared__ bool last;
    const int P = sv.n_parts;
    const bool rows = static_cast<int>(blockIdx.x) < ea.ncr;
    const int c = rows ? blockIdx.x : blockIdx.x - ea.ncr;
    const int n = rows ? sv.n_rows : ea.cap;
    const int nn = rows ? n : min(*ea.dn, n);
    const int s0 = c * kECH, s1 = min(n, s0 + kECH);
    auto pof = [&](int t) -> int {
        if (rows) return sv.rpart[t] - sv.part_base;
        if (t >= nn) return P - 1; // padding belongs to the last partition (KeyPart)
        int a, b, v, e;
        ea.fmt.unpack(ea.keys[t], a, b, v, e);
        return sv.ipart[a] - sv.part_base;
    };
    const int plo = s0 < s1 ? pof(s0) : 0;
    const int phi = s0 < s1 ? pof(s1 - 1) : -1;
    double* part = ea.partial + static_cast<size_t>(blockIdx.x) * P;
    for (int p = threadIdx.x; p < P; p += kB)
        if (p < plo || p > phi) part[p] = 0.0;
    for (int p = plo; p <= phi; ++p) {
        double acc = 0.0;
        for (int t = s0 + threadIdx.x; t < s1; t += kB) {
            if (plo != phi && pof(t) != p) continue;
            double v = 0.0;
            if (rows) {
                if (part_flag(sv, p, ea.which)) {
                    const int i = sv.rinst[t];
                    double q[6];
                    eval_q(sv, i, ea.qmode, q);
                    v = body_value(sv, i, q);
                }
            } else if (t < nn) {
                v = cand_value(sv, ea.keys[t], ea.fmt, ea.qmode, ea.which);
            }
            acc += v;
        }
        sh[threadIdx.x] = acc;
        __syncthreads();
        for (int w = kB / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) part[p] = sh[0];
        __syncthreads();
    }
    __threadfence();
    if (threadIdx.x == 0) last = atomicAdd(ea.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int p = warp; p < P; p += kB / 32) {
        double sr = fold_partials(ea.partial, P, p, 0, ea.ncr, lane);
        double sk = fold_partials(ea.partial, P, p, ea.ncr, static_cast<int>(gridDim.x), lane);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            sr += __shfl_xor_sync(0xffffffffu, sr, off);
            sk += __shfl_xor_sync(0xffffffffu, sk, off);
        }
        if (lane == 0) {
            double d = sr;
            d += sk;
            ea.dst[p * ea.stride] = d;
        }
    }
    if (threadIdx.x == 0) *ea.ticket = 0u;
    if (!ea.accept) return;
    __syncthreads();
    scalar_block(sv.ps, P, kOpAccept, ea.ctrl, ea.hd, 0.0, 0, sv.err);
    if (ea.apply) {
        __syncthreads(); // the accept decisions of this block are visible to it
        accept_trial_block(sv, sh);
    }
    if (!ea.tail) return;
    __syncthreads();
    const bool srch = threadIdx.x < P && sv.ps[threadIdx.x].searching != 0;
    if (__syncthreads_or(srch)) return; // the line search goes on: the tail comes later
    scalar_block(sv.ps, P, kOpNewtonTail, ea.ctrl, ea.hd, 0.0, ea.max_iters, sv.err, ea.iter_reset);
}

// iq += alpha dq for the instances of partitions whose trial was accepted
// (k_make_trial + k_accept_copy: the same unfused arithmetic as the trial).
__global__ void k_accept_trial(SolverView sv) {
    accept_trial_range(sv, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------------------
// Segment offsets of sorted keys: off[i] = first index whose instance >= i.
// ---------------------------------------------------------------------------
__global__ void k_seg_offsets(const unsigned long long* keys, int n, const int* dn, KeyFmt fmt,
                              int n_inst, int* off, int which_field, const int* perm) {
    const int nn = dn ? min(*dn, n) : n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n_inst; i += gridDim.x * blockDim.x) {
        int lo = 0, hi = nn;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            int a, b, v, e;
            fmt.unpack(keys[perm ? perm[mid] : mid], a, b, v, e);
            const int key = which_field == 0 ? a : b;
            if (key < i) lo = mid + 1;
            else hi = mid;
        }
        off[i] = lo;
    }
}

__global__ void k_make_bkeys(const unsigned long long* keys, int n, const int* dn, KeyFmt fmt,
                             unsigned long long* bkeys, int* idx) {
    const int nn = dn ? min(*dn, n) : n;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        if (t < nn) {
            int a, b, v, e;
            fmt.unpack(keys[t], a, b, v, e);
            bkeys[t] = fmt.pack(b, a, v, e);
        } else {
            bkeys[t] = ~0ull; // padding sorts last
        }
        idx[t] = t;
    }
}

// ---------------------------------------------------------------------------
// Active-set selection over the skin list at the current iterate: the exact
// static broad-phase predicate (margin d_hat) & not static-static & d < d_hat
// (objective.cpp:91-106). Writes flag[t] for every list entry, appends the
// active positions to cv.act (warp-aggregated; the order of `act` only
// decides which thread evaluates which contact, never a result) and counts
// candidates / active contacts per partition.
// ---------------------------------------------------------------------------
// box == nullptr: body boxes recomputed on the fly (no k_inst_boxes launch);
// terms: also evaluate the contact terms of every active entry in place (no
// separate k_contact_terms launch over the compacted list).
__global__ void __launch_bounds__(kB) k_contact_select(SolverView sv, ContactView cv, const Box* box, int terms) {
    const int nn = cv.dn ? min(*cv.dn, cv.n) : cv.n;
    const int lane = threadIdx.x & 31;
    const int span = (nn + 31) & ~31; // whole warps stay in the loop (ballots)
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < span; t += gridDim.x * blockDim.x) {
        bool cand = false, act = false;
        int p = -1;
        if (t < nn) {
            int a, b, v, e;
            cv.fmt.unpack(cv.key[t], a, b, v, e);
            // the instances' bodies load beside the partition index instead of
            // after the partition's flag (two L2 trips off every thread's chain)
            const int ba = sv.ibody[a], bb = sv.ibody[b];
            p = sv.ipart[a] - sv.part_base;
            if (sv.ps[p].active) {
                const bool ss = sv.sc.is_static[ba] && sv.sc.is_static[bb];
                const double* qa = sv.iq + 6 * a;
                const double* qb = sv.iq + 6 * b;
                // box == nullptr: no body-box test. It is implied by the point /
                // edge box test: pb = {P} lies in a's d_hat-inflated body box and
                // eb in b's (the same world points, the min / max over a superset
                // of vertices, and the inflation rounds monotonically), so pb and
                // eb overlapping makes the body boxes overlap; dropping it only
                // removes the two 4-vertex box chains from every thread.
                if (!ss && (!box || overlaps(box[a], box[b]))) {
                    const int vf = sv.sc.vstart[ba] + v, ef = sv.sc.vstart[bb] + e;
                    const Box pb = point_box(sv.sc, qa, qa, false, vf);
                    const Box eb = edge_box(sv.sc, qb, qb, false, ef, sv.d_hat);
                    if (overlaps(pb, eb)) {
                        cand = true;
                        const V2 P = world_point(qa, rest_of(sv.sc, vf));
                        const V2 E0 = world_point(qb, rest_of(sv.sc, ef));
                        const V2 E1 = world_point(qb, rest_of(sv.sc, sv.sc.vnext[ef]));
                        const double d = pe_distance(P, E0, E1);
                        if (d < sv.d_hat) {
                            if (d <= 0.0) raise(sv.err, d == -1.0 ? kErrDegenerateEdge : kErrBarrierDomain);
                            act = true;
                        }
                    }
                }
            }
            cv.flag[t] = act ? 1 : 0;
            if (!act) cv.cval[t] = 0.0;
            else if (terms) contact_terms_one(sv, cv, t);
        }
        const unsigned ab = __ballot_sync(0xffffffffu, act);
        const unsigned cb = __ballot_sync(0xffffffffu, cand);
        int base = 0;
        if (lane == 0 && ab) base = atomicAdd(&cv.ls->n_act, __popc(ab));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (act) cv.act[base + __popc(ab & ((1u << lane) - 1u))] = t;
        // per-partition counts: one atomic per warp when the partition is warp-uniform
        const int p0 = __shfl_sync(0xffffffffu, p, 0);
        const bool uniform = __all_sync(0xffffffffu, p == p0 || p < 0);
        if (uniform) {
            if (lane == 0 && p0 >= 0) {
                if (cb) atomicAdd(&sv.ps[p0].n_candidates, __popc(cb));
                if (ab) atomicAdd(&sv.ps[p0].n_active_contacts, __popc(ab));
            }
        } else {
            if (cand) atomicAdd(&sv.ps[p].n_candidates, 1);
            if (act) atomicAdd(&sv.ps[p].n_active_contacts, 1);
        }
    }
}

// ---------------------------------------------------------------------------
// Deterministic BSR assembly (ELL storage, sv.ell_w off-diagonal blocks / row):
// one warp per row, lane l owns entries l and l + 32 of each 6x6 block and
// sums the contacts' precomputed DoF-space blocks (store_dof_blocks) in list
// order: TL where the row's body is the point body, BR where it is the edge
// body; off-diagonal blocks TR / BL = TR^T grouped by partner instance.
// ---------------------------------------------------------------------------
// One row whose a- and b-segments have at most 32 entries each: every lane
// loads one entry's flag, partner and partner row up front, so the block
// sums walk ballot masks with independent loads (unrolled by 4) instead of a
// chain of dependent flag/key/perm loads per entry. Same entries, same order
// of additions as the general loop below (bitwise identical results).
__device__ __forceinline__ void add_blocks(const ContactView& cv, unsigned m, int cidx, int off,
                                           int k0, int k1, bool has1, double& x0, double& x1,
                                           int gofs, int lane, double* g) {
    while (m) {
        int c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = m ? __ffs(m) - 1 : -1;
            if (m) m &= m - 1;
            c[u] = __shfl_sync(0xffffffffu, cidx, j < 0 ? 0 : j);
            if (j < 0) c[u] = -1;
        }
        double v0[4], v1[4], vg[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            v0[u] = v1[u] = vg[u] = 0.0;
            if (c[u] >= 0) {
                const double* bk = cv.cblk + 108 * static_cast<size_t>(c[u]) + off;
                v0[u] = bk[k0];
                if (has1) v1[u] = bk[k1];
                if (g && lane < 6) vg[u] = cv.cgrad[12 * c[u] + gofs + lane];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (c[u] < 0) continue;
            x0 += v0[u];
            if (has1) x1 += v1[u];
            if (g && lane < 6) *g += vg[u];
        }
    }
}

__device__ __forceinline__ void assemble_row_fast(const SolverView& sv, const ContactView& cv, int r,
                                                  int a0, int a1, int b0, int b1, int lane, int e0,
                                                  int e1, int t0, int t1, bool has1, double d0,
                                                  double d1, double g, double* row_trace) {
    int ca = -1, pa = 0x7fffffff, ra = -1;
    bool fa = false;
    if (a0 + lane < a1) {
        ca = a0 + lane;
        fa = cv.flag[ca] != 0;
        if (fa) {
            int x, y, v, e;
            cv.fmt.unpack(cv.key[ca], x, y, v, e);
            pa = y;
            ra = sv.irow[y];
        }
    }
    int cb = -1, pb = 0x7fffffff, rb = -1;
    bool fb = false;
    if (b0 + lane < b1) {
        cb = cv.perm_b[b0 + lane];
        fb = cv.flag[cb] != 0;
        if (fb) {
            int x, y, v, e;
            cv.fmt.unpack(cv.key[cb], x, y, v, e);
            pb = x;
            rb = sv.irow[x];
        }
    }
    unsigned ma = __ballot_sync(0xffffffffu, fa), mb = __ballot_sync(0xffffffffu, fb);
    add_blocks(cv, ma, ca, 0, e0, e1, has1, d0, d1, 0, lane, &g);  // TL, gradient 0..5
    add_blocks(cv, mb, cb, 36, e0, e1, has1, d0, d1, 6, lane, &g); // BR, gradient 6..11
    if (lane < 6) sv.rgrad[6 * r + lane] = g;
    sv.rdiag[36 * r + e0] = d0;
    if (has1) sv.rdiag[36 * r + e1] = d1;
    double tr = (e0 % 7 == 0) ? d0 : 0.0;
    if (lane == 3) tr += d1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, off);
    if (lane == 0) row_trace[r] = tr;
    // off-diagonal blocks by ascending partner: the partner's run in the
    // a-segment (TR) then in the b-segment (BL = TR^T)
    int nblk = 0;
    while (ma | mb) {
        const int ja = ma ? __ffs(ma) - 1 : 0, jb = mb ? __ffs(mb) - 1 : 0;
        const int qa = ma ? __shfl_sync(0xffffffffu, pa, ja) : 0x7fffffff;
        const int qb = mb ? __shfl_sync(0xffffffffu, pb, jb) : 0x7fffffff;
        const int partner = min(qa, qb);
        const int prow = qa == partner ? __shfl_sync(0xffffffffu, ra, ja) : __shfl_sync(0xffffffffu, rb, jb);
        const unsigned runa = __ballot_sync(0xffffffffu, ((ma >> lane) & 1u) && pa == partner);
        const unsigned runb = __ballot_sync(0xffffffffu, ((mb >> lane) & 1u) && pb == partner);
        ma &= ~runa;
        mb &= ~runb;
        if (prow < 0) continue; // static partner: no block
        double o0 = 0.0, o1 = 0.0;
        add_blocks(cv, runa, ca, 72, e0, e1, has1, o0, o1, 0, lane, nullptr);
        add_blocks(cv, runb, cb, 72, t0, t1, has1, o0, o1, 0, lane, nullptr);
        if (nblk >= sv.ell_w) {
            if (lane == 0) raise(sv.err, kErrEll);
            break;
        }
        if (lane == 0) sv.ell_col[r * sv.ell_w + nblk] = prow;
        double* odst = sv.ell_blk + (static_cast<size_t>(r) * sv.ell_w + nblk) * 36;
        odst[e0] = o0;
        if (has1) odst[e1] = o1;
        ++nblk;
    }
    if (lane == 0) sv.ell_cnt[r] = nblk;
}

__global__ void __launch_bounds__(128) k_assemble(SolverView sv, ContactView cv, double* row_trace) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    // the two entries of this lane
    const int e0 = lane, e1 = lane + 32;
    const bool has1 = e1 < 36;
    // the transposed entries (BL = TR^T)
    const int t0 = 6 * (e0 % 6) + e0 / 6, t1 = has1 ? 6 * (e1 % 6) + e1 / 6 : 0;
    for (int r = gw; r < sv.n_rows; r += nw) {
        // the row's instance, segment bounds and body terms load beside the
        // partition flag, not after it (the flag only decides whether to store)
        const int i = sv.rinst[r];
        const int p = sv.rpart[r] - sv.part_base;
        const int a0 = cv.aoff[i], a1 = cv.aoff[i + 1];
        const int b0 = cv.boff[i], b1 = cv.boff[i + 1];
        double d0 = sv.rdiag[36 * r + e0];
        double d1 = has1 ? sv.rdiag[36 * r + e1] : 0.0;
        double g = lane < 6 ? sv.rgrad[6 * r + lane] : 0.0;
        if (!sv.ps[p].active) continue;
        if (a1 - a0 <= 32 && b1 - b0 <= 32) { // the usual row: warp-parallel metadata
            assemble_row_fast(sv, cv, r, a0, a1, b0, b1, lane, e0, e1, t0, t1, has1, d0, d1, g, row_trace);
            continue;
        }
        for (int c = a0; c < a1; ++c) { // point body: TL, gradient 0..5
            if (!cv.flag[c]) continue;
            const double* bk = cv.cblk + 108 * static_cast<size_t>(c);
            d0 += bk[e0];
            if (has1) d1 += bk[e1];
            if (lane < 6) g += cv.cgrad[12 * c + lane];
        }
        for (int t = b0; t < b1; ++t) { // edge body: BR, gradient 6..11
            const int c = cv.perm_b[t];
            if (!cv.flag[c]) continue;
            const double* bk = cv.cblk + 108 * static_cast<size_t>(c) + 36;
            d0 += bk[e0];
            if (has1) d1 += bk[e1];
            if (lane < 6) g += cv.cgrad[12 * c + 6 + lane];
        }
        if (lane < 6) sv.rgrad[6 * r + lane] = g;
        sv.rdiag[36 * r + e0] = d0;
        if (has1) sv.rdiag[36 * r + e1] = d1;
        // trace: diagonal entries 0, 7, 14, 21, 28 (lanes) and 35 (lane 3, second entry)
        double tr = (e0 % 7 == 0) ? d0 : 0.0;
        if (lane == 3) tr += d1;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, off);
        if (lane == 0) row_trace[r] = tr;
        // off-diagonal blocks: merge the a-segment (sorted by b) and the
        // b-segment (sorted by a) by partner instance, active contacts only
        int ia = a0, ib = b0, nblk = 0;
        while (true) {
            while (ia < a1 && !cv.flag[ia]) ++ia;
            while (ib < b1 && !cv.flag[cv.perm_b[ib]]) ++ib;
            if (ia >= a1 && ib >= b1) break;
            int ca, cb, vv, ee;
            int pa = 0x7fffffff, pb = 0x7fffffff;
            if (ia < a1) {
                cv.fmt.unpack(cv.key[ia], ca, cb, vv, ee);
                pa = cb;
            }
            if (ib < b1) {
                cv.fmt.unpack(cv.key[cv.perm_b[ib]], ca, cb, vv, ee);
                pb = ca;
            }
            const int partner = min(pa, pb);
            const int prow = sv.irow[partner];
            double o0 = 0.0, o1 = 0.0;
            for (; ia < a1; ++ia) { // TR: rows = point body (this), cols = edge body
                cv.fmt.unpack(cv.key[ia], ca, cb, vv, ee);
                if (cb != partner) break;
                if (!cv.flag[ia] || prow < 0) continue;
                const double* bk = cv.cblk + 108 * static_cast<size_t>(ia) + 72;
                o0 += bk[e0];
                if (has1) o1 += bk[e1];
            }
            for (; ib < b1; ++ib) { // BL = TR^T: rows = edge body (this), cols = point body
                const int c = cv.perm_b[ib];
                cv.fmt.unpack(cv.key[c], ca, cb, vv, ee);
                if (ca != partner) break;
                if (!cv.flag[c] || prow < 0) continue;
                const double* bk = cv.cblk + 108 * static_cast<size_t>(c) + 72;
                o0 += bk[t0];
                if (has1) o1 += bk[t1];
            }
            if (prow < 0) continue;
            if (nblk >= sv.ell_w) {
                if (lane == 0) raise(sv.err, kErrEll);
                break;
            }
            if (lane == 0) sv.ell_col[r * sv.ell_w + nblk] = prow;
            double* odst = sv.ell_blk + (static_cast<size_t>(r) * sv.ell_w + nblk) * 36;
            odst[e0] = o0;
            if (has1) odst[e1] = o1;
            ++nblk;
        }
        if (lane == 0) sv.ell_cnt[r] = nblk;
    }
}

// ---------------------------------------------------------------------------
// Skin-list validity (see ListState): every dynamic vertex of q and q1 within
// 0.99 s_i of its qref position. Every thread also proposes the skin of a
// rebuild at qref = q: s_i = max(s_min, grow * (largest move of one of the
// instance's vertices from q to q1 or to q_tilde)), so a rebuilt list covers
// q1 and the predicted motion of the frame. The last block decides, sets the
// rebuild flag and steers the conditional IF node of the rebuild.
// ---------------------------------------------------------------------------
// Skin-list test of instance i (see k_list_check): true if a vertex of q0
// or q1 left 0.99 of its skin around qref; proposes the rebuild skin.
__device__ __forceinline__ bool list_check_one(const SceneView& sc, int b, int i, const double* q0,
                                               const double* q1, const double* qref, const double* qt,
                                               const double* skin, double* skin_next, double s_min,
                                               double grow) {
    if (sc.is_static[b]) {
        skin_next[i] = 0.0;
        return false;
    }
    const double* qr = qref + 6 * i;
    const double* qs = qt ? qt + 6 * i : q0;
    double dref = 0.0, dstep = 0.0;
    for (int v = sc.vstart[b]; v < sc.vstart[b + 1]; ++v) {
        const V2 r = rest_of(sc, v);
        const V2 x0 = world_point(q0, r), x1 = world_point(q1, r), xr = world_point(qr, r),
                 xs = world_point(qs, r);
        dref = fmax(dref, fmax(fmax(fabs(x0.x - xr.x), fabs(x0.y - xr.y)),
                               fmax(fabs(x1.x - xr.x), fabs(x1.y - xr.y))));
        dstep = fmax(dstep, fmax(fmax(fabs(x1.x - x0.x), fabs(x1.y - x0.y)),
                                 fmax(fabs(xs.x - x0.x), fabs(xs.y - x0.y))));
    }
    skin_next[i] = fmax(s_min, grow * dstep);
    return !(dref <= 0.99 * skin[i]); // NaN-safe
}

// Block-wide vote + last-block decision of the list test (steers the IF node
// of the conditional rebuild). All threads of every block call it.
__device__ __forceinline__ void list_check_finish(bool bad, ListState* ls, unsigned long long cond,
                                                  int graph) {
    __shared__ bool last;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&ls->invalid_acc, 1);
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&ls->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    const bool rebuild = !ls->valid || __ldcg(&ls->invalid_acc) != 0;
    if (rebuild) ++ls->n_rebuilds;
    ls->valid = 1;
    ls->rebuild = rebuild ? 1 : 0;
    ls->invalid_acc = 0;
    ls->ticket = 0u;
    if (graph) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(cond), rebuild ? 1u : 0u);
}

__global__ void k_list_check(SceneView sc, InstView iv, const double* qref, const double* qt,
                             const double* skin, double* skin_next, double s_min, double grow,
                             ListState* ls, unsigned long long cond, int graph) {
    bool bad = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < iv.n; i += gridDim.x * blockDim.x)
        bad |= list_check_one(sc, iv.body[i], i, iv.q0 + 6 * i, iv.q1 + 6 * i, qref, qt, skin,
                              skin_next, s_min, grow);
    list_check_finish(bad, ls, cond, graph);
}

// CCD preparation of a Newton iteration (newton.cpp:38-42) in one launch:
// q1 = q + dq for the active partitions (k_make_trial, alpha 1, unfused),
// the skin-list test over [q, q1] (k_list_check) and the margin-0 swept
// instance boxes for the CCD filter (k_inst_boxes).
__global__ void k_ccd_prep(SolverView sv, const double* qref, const double* skin, double* skin_next,
                           double s_min, double grow, ListState* ls, unsigned long long cond,
                           int graph, Box* box) {
    bool bad = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < sv.n_inst; i += gridDim.x * blockDim.x) {
        const int p = sv.ipart[i] - sv.part_base;
        const int r = sv.irow[i];
        double q0[6], q1[6];
        load6(sv.iq + 6 * i, q0);
#pragma unroll
        for (int k = 0; k < 6; ++k) q1[k] = q0[k];
        if (r >= 0 && sv.ps[p].active) {
            double dq[6];
            load6(sv.x + 6 * r, dq);
#pragma unroll
            for (int k = 0; k < 6; ++k) q1[k] = xadd(q0[k], xmul(1.0, dq[k]));
        }
        store6(sv.iq_try + 6 * i, q1);
        const int b = sv.ibody[i];
        bad |= list_check_one(sv.sc, b, i, q0, q1, qref, sv.iqt, skin, skin_next, s_min, grow);
        if (!box) continue; // k_ccd without body boxes (see there)
        Box bx{{DBL_MAX, DBL_MAX}, {-DBL_MAX, -DBL_MAX}};
        for (int v = sv.sc.vstart[b]; v < sv.sc.vstart[b + 1]; ++v) {
            const V2 rr = rest_of(sv.sc, v);
            const V2 x = world_point(q0, rr), y = world_point(q1, rr);
            bx.lo = vmin(bx.lo, vmin(x, y));
            bx.hi = vmax(bx.hi, vmax(x, y));
        }
        box[i] = inflate(bx, 0.0);
    }
    list_check_finish(bad, ls, cond, graph);
}

// First node of a rebuild: qref = q, skin = the proposal of the check.
__global__ void k_list_commit(int n, const double* iq, double* qref, const double* skin_next,
                              double* skin) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 6 * n; i += gridDim.x * blockDim.x) {
        qref[i] = iq[i];
        if (i < n) skin[i] = skin_next[i];
    }
}

// Block-Jacobi preconditioner: inverse of (D + eps I) through its Cholesky.
__global__ void k_precond(SolverView sv) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < sv.n_rows; r += gridDim.x * blockDim.x) {
        const int p = sv.rpart[r] - sv.part_base;
        if (!sv.ps[p].active) continue;
        const double eps = sv.ps[p].eps;
        double L[6][6];
        const double* d = sv.rdiag + 36 * r;
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            double s = d[6 * j + j] + eps;
#pragma unroll
            for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
            if (!(s > 0.0)) ok = false;
            const double dj = sqrt(fmax(s, 1e-300));
            L[j][j] = dj;
#pragma unroll
            for (int i = j + 1; i < 6; ++i) {
                double t = d[6 * i + j];
#pragma unroll
                for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
                L[i][j] = t / dj;
            }
#pragma unroll
            for (int i = 0; i < j; ++i) L[i][j] = 0.0;
        }
        if (!ok) raise(sv.err, kErrFactor);
        // inverse of L (lower), then Dinv = Linv^T Linv
        double Li[6][6];
#pragma unroll
        for (int c = 0; c < 6; ++c)
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
                for (int k = 0; k < i; ++k) s -= L[i][k] * Li[k][c];
                Li[i][c] = (i < c) ? 0.0 : s / L[i][i];
            }
        double* o = sv.rdinv + 36 * r;
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < 6; ++k) s += Li[k][a] * Li[k][c];
                o[6 * a + c] = s;
            }
    }
}

// ---------------------------------------------------------------------------
// Two-level deterministic segment sums. Chunk c covers [c*CH, (c+1)*CH).
// ---------------------------------------------------------------------------

// One launch: every block writes its chunk's per-partition partials, the
// last block to finish (threadfence + ticket) folds them in chunk order with
// a fixed warp butterfly, so the result is bitwise reproducible.
template <typename PartOf>
__global__ void k_segsum(const double* v, int n, int P, int part_base, PartOf pof,
                         double* partial, unsigned* ticket, double* dst, int stride,
                         int accumulate) {
    __shared__ double sh[kB];
    __shared__ bool last;
    const int c = blockIdx.x;
    const int s0 = c * kCH, s1 = min(n, s0 + kCH);
    // partitions present in this chunk: [pof(s0), pof(s1-1)]
    const int plo = s0 < s1 ? pof(s0) - part_base : 0;
    const int phi = s0 < s1 ? pof(s1 - 1) - part_base : -1;
    for (int p = threadIdx.x; p < P; p += kB)
        if (p < plo || p > phi) partial[static_cast<size_t>(c) * P + p] = 0.0;
    for (int p = plo; p <= phi; ++p) {
        double acc = 0.0;
        for (int t = s0 + threadIdx.x; t < s1; t += kB)
            if (plo == phi || pof(t) - part_base == p) acc += v[t];
        sh[threadIdx.x] = acc;
        __syncthreads();
        for (int w = kB / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[static_cast<size_t>(c) * P + p] = sh[0];
        __syncthreads();
    }
    __threadfence();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int p = warp; p < P; p += kB / 32) {
        double s = 0.0;
        for (int k = lane; k < static_cast<int>(gridDim.x); k += 32)
            s += __ldcg(partial + static_cast<size_t>(k) * P + p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) {
            if (accumulate) dst[p * stride] += s;
            else dst[p * stride] = s;
        }
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

struct RowPart {
    const int* rpart;
    __device__ int operator()(int t) const { return rpart[t]; }
};
struct KeyPart {
    const unsigned long long* keys;
    KeyFmt fmt;
    const int* ipart;
    const int* dn;   // device count (padding past it belongs to the last partition)
    int last_part;
    __device__ int operator()(int t) const {
        if (dn && t >= *dn) return last_part;
        int a, b, v, e;
        fmt.unpack(keys[t], a, b, v, e);
        return ipart[a];
    }
};

// ---------------------------------------------------------------------------
// Line search helpers
// ---------------------------------------------------------------------------
// q_try = q + alpha * dq (objective.cpp:215-221), unfused like the reference.
__global__ void k_make_trial(SolverView sv, int use_alpha_field, double fixed_alpha, int which) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < sv.n_inst; i += gridDim.x * blockDim.x) {
        const int p = sv.ipart[i] - sv.part_base;
        const int r = sv.irow[i];
        double q[6];
        load6(sv.iq + 6 * i, q);
        if (r >= 0 && part_flag(sv, p, which)) {
            const double alpha = use_alpha_field ? sv.ps[p].alpha : fixed_alpha;
            double dq[6];
            load6(sv.x + 6 * r, dq);
#pragma unroll
            for (int k = 0; k < 6; ++k) q[k] = xadd(q[k], xmul(alpha, dq[k]));
        }
        store6(sv.iq_try + 6 * i, q);
    }
}

// toi_earliest of every partition back to "no impact" (kOpIterBegin's reset)
// before k_ccd re-runs over a rebuilt candidate list; the discarded first
// k_ccd's kOpAlphaMax is taken out of the step-body execution count.
__global__ void k_toi_reset(PartState* ps, int P, FrameCtrl* ctrl) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) ps[p].toi_earliest = 2.0;
    if (ctrl && threadIdx.x == 0) --ctrl->exec_step;
}

__global__ void k_dq_inf(SolverView sv) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < sv.n_rows; r += gridDim.x * blockDim.x) {
        const int p = sv.rpart[r] - sv.part_base;
        if (!sv.ps[p].active) continue;
        double m = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k) m = fmax(m, fabs(sv.x[6 * r + k]));
        atomic_max_nonneg(&sv.ps[p].dq_inf, m);
    }
}

// CCD over the candidate superset with the exact swept margin-0 predicate
// (geometry.cpp:311-341). box0: per-instance swept boxes with margin 0.
// fin != nullptr: the last block then takes kOpAlphaMax (scalar_block).
struct CcdFinish {
    FrameCtrl* ctrl;
    CondHandles hd;
    unsigned* ticket;
};

// The CCD end point of instance i, q0 + 1.0 dq for a row of an active
// partition (else q0): k_ccd_prep's arithmetic, so k_ccd can form it itself
// (q1 == nullptr) and run beside k_ccd_prep instead of after it.
__device__ __forceinline__ void ccd_end_point(const SolverView& sv, int i, const double (&q0)[6],
                                              double (&q1)[6]) {
    const int r = sv.irow[i];
    const int p = sv.ipart[i] - sv.part_base;
#pragma unroll
    for (int k = 0; k < 6; ++k) q1[k] = q0[k];
    if (r >= 0 && sv.ps[p].active) {
        double dq[6];
        load6(sv.x + 6 * r, dq);
#pragma unroll
        for (int k = 0; k < 6; ++k) q1[k] = xadd(q1[k], xmul(1.0, dq[k]));
    }
}

__global__ void k_ccd(SolverView sv, const unsigned long long* keys, int n, const int* dn,
                      KeyFmt fmt, const Box* box0, const double* q0, const double* q1, int which,
                      double* earliest_override, CcdFinish fin) {
    __shared__ bool last;
    const int nn = dn ? min(*dn, n) : n;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nn; t += gridDim.x * blockDim.x) {
        int a, b, v, e;
        fmt.unpack(keys[t], a, b, v, e);
        // bodies load beside the partition index, not after its flag.
        // box0 == nullptr: no swept body-box test. It is implied by the swept
        // point / edge box test below (the same world points at q0 and q1, the
        // min / max over a superset of the body's vertices, margin 0), so it
        // only filters early; k_ccd_prep then writes no boxes.
        const int ba = sv.ibody[a], bb = sv.ibody[b];
        const int p = sv.ipart[a] - sv.part_base;
        if (!part_flag(sv, p, which)) continue;
        if (box0 && !overlaps(box0[a], box0[b])) continue;
        const int vf = sv.sc.vstart[ba] + v, ef = sv.sc.vstart[bb] + e;
        // both configurations in registers; the end points formed here when
        // q1 == nullptr
        double qa0[6], qa1[6], qb0[6], qb1[6];
        load6(q0 + 6 * a, qa0);
        load6(q0 + 6 * b, qb0);
        if (q1) {
            load6(q1 + 6 * a, qa1);
            load6(q1 + 6 * b, qb1);
        } else {
            ccd_end_point(sv, a, qa0, qa1);
            ccd_end_point(sv, b, qb0, qb1);
        }
        const Box pb = point_box(sv.sc, qa0, qa1, true, vf);
        const Box eb = edge_box(sv.sc, qb0, qb1, true, ef, 0.0);
        if (!overlaps(pb, eb)) continue;
        const V2 rp = rest_of(sv.sc, vf), r0 = rest_of(sv.sc, ef),
                 r1 = rest_of(sv.sc, sv.sc.vnext[ef]);
        const V2 P0 = world_point(qa0, rp), P1 = world_point(qa1, rp);
        const V2 A0 = world_point(qb0, r0), A1 = world_point(qb1, r0);
        const V2 B0 = world_point(qb0, r1), B1 = world_point(qb1, r1);
        const double d0 = pe_distance(P0, A0, B0);
        if (d0 <= 0.0) {
            raise(sv.err, d0 == -1.0 ? kErrDegenerateEdge : kErrTouching);
            continue;
        }
        const double toi = pair_impact_time(P0, P1, A0, A1, B0, B1);
        if (toi <= 1.0)
            atomic_min_nonneg(earliest_override ? &earliest_override[p] : &sv.ps[p].toi_earliest, toi);
    }
    if (!fin.ticket) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(fin.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x == 0) *fin.ticket = 0u;
    scalar_block(sv.ps, sv.n_parts, kOpAlphaMax, fin.ctrl, fin.hd, 0.0, 0, sv.err);
}

} // namespace

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
void launch_body_terms(const SolverView& sv, const double* q, bool derivs, int which,
                       cudaStream_t s, int* reset_counter, FrameCtrl* iter_begin) {
    if (sv.n_rows == 0) {
        if (reset_counter) CUDA_CHECK(cudaMemsetAsync(reset_counter, 0, sizeof(int), s));
        return;
    }
    DABD_LAUNCH("k_body_terms", s, k_body_terms<<<grid_for(sv.n_rows, 64), 64, 0, s>>>(sv, q, derivs ? 1 : 0, which,
                                                                                      reset_counter, iter_begin));
}

void launch_filter(const SolverView& sv, const unsigned long long* keys, int n, const int* dn,
                   KeyFmt fmt, const Box* box, const double* q, int mode, int which,
                   unsigned char* flag, double* val, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_filter", s,
                k_filter<<<grid_for(n, kB), kB, 0, s>>>(sv, keys, n, dn, fmt, box, q, mode, which,
                                                        flag, val));
}

void launch_contact_terms(const SolverView& sv, const ContactView& cv, cudaStream_t s) {
    if (cv.n == 0) return;
    // 32-thread blocks spread the few thousand active contacts over every SM
    DABD_LAUNCH("k_contact_terms", s, k_contact_terms<<<grid_for(cv.n, 32, 148 * 8), 32, 0, s>>>(sv, cv));
}

void launch_seg_offsets(const unsigned long long* keys, int n, const int* dn, KeyFmt fmt,
                        int n_inst, int* off, int field, const int* perm, cudaStream_t s) {
    DABD_LAUNCH("k_seg_offsets", s,
                k_seg_offsets<<<grid_for(n_inst + 1, kB), kB, 0, s>>>(keys, n, dn, fmt, n_inst, off,
                                                                      field, perm));
}

void launch_make_bkeys(const unsigned long long* keys, int n, const int* dn, KeyFmt fmt,
                       unsigned long long* bkeys, int* idx, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_make_bkeys", s,
                k_make_bkeys<<<grid_for(n, kB), kB, 0, s>>>(keys, n, dn, fmt, bkeys, idx));
}

void launch_assemble(const SolverView& sv, const ContactView& cv, double* row_trace,
                     cudaStream_t s) {
    if (sv.n_rows == 0) return;
    DABD_LAUNCH("k_assemble", s, k_assemble<<<grid_for(32ll * sv.n_rows, 128), 128, 0, s>>>(sv, cv, row_trace));
}

void launch_contact_select(const SolverView& sv, const ContactView& cv, const Box* box,
                           cudaStream_t s, bool terms) {
    if (cv.n == 0) return;
    DABD_LAUNCH("k_contact_select", s,
                k_contact_select<<<grid_for(cv.n, kB, 148 * 4), kB, 0, s>>>(sv, cv, box, terms ? 1 : 0));
}

void launch_list_check(const SceneView& sc, const InstView& iv, const double* qref,
                       const double* qt, const double* skin, double* skin_next, double s_min,
                       double grow, ListState* ls, unsigned long long cond, int graph,
                       cudaStream_t s) {
    DABD_LAUNCH("k_list_check", s,
                k_list_check<<<grid_for(std::max(iv.n, 1), kB, 148), kB, 0, s>>>(
                    sc, iv, qref, qt, skin, skin_next, s_min, grow, ls, cond, graph));
}

void launch_list_commit(int n, const double* iq, double* qref, const double* skin_next,
                        double* skin, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_list_commit", s,
                k_list_commit<<<grid_for(6ll * n, kB), kB, 0, s>>>(n, iq, qref, skin_next, skin));
}

void launch_precond(const SolverView& sv, cudaStream_t s) {
    if (sv.n_rows == 0) return;
    DABD_LAUNCH("k_precond", s, k_precond<<<grid_for(sv.n_rows, 64), 64, 0, s>>>(sv));
}

int segsum_chunks(int n) { return std::max(1, (n + kCH - 1) / kCH); }
int energy_chunks(int n) { return std::max(1, (n + kECH - 1) / kECH); }

// Ticket for the last-block fold; launches on one device are stream ordered.
__device__ unsigned g_segsum_ticket = 0;

// Shared-memory carveout of the per-iteration kernels: the same as the
// cluster PCG's (maximum shared memory), so an SM never reconfigures its
// L1/shared split between the PCG and its neighbours in the Newton loop.
void set_solver_carveout(int pct) {
    const void* fns[] = {reinterpret_cast<const void*>(k_body_terms), reinterpret_cast<const void*>(k_contact_select),
                         reinterpret_cast<const void*>(k_assemble), reinterpret_cast<const void*>(k_energy),
                         reinterpret_cast<const void*>(k_accept_trial), reinterpret_cast<const void*>(k_ccd_prep),
                         reinterpret_cast<const void*>(k_ccd), reinterpret_cast<const void*>(k_list_check),
                         reinterpret_cast<const void*>(k_list_commit), reinterpret_cast<const void*>(k_seg_offsets),
                         reinterpret_cast<const void*>(k_make_bkeys), reinterpret_cast<const void*>(k_contact_terms),
                         reinterpret_cast<const void*>(k_precond), reinterpret_cast<const void*>(k_dq_inf),
                         reinterpret_cast<const void*>(k_make_trial), reinterpret_cast<const void*>(k_filter)};
    for (const void* f : fns) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();
}

static unsigned* segsum_ticket() { // resolved once per device, outside any graph capture
    static void* cache[64] = {};
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    if (!cache[dev & 63]) CUDA_CHECK(cudaGetSymbolAddress(&cache[dev & 63], g_segsum_ticket));
    return static_cast<unsigned*>(cache[dev & 63]);
}

void launch_segsum_rows(const double* v, int n, const int* rpart, int P, int part_base,
                        double* partial, double* dst, int stride, bool accumulate, cudaStream_t s) {
    const int nc = segsum_chunks(n);
    DABD_LAUNCH("k_segsum", s,
                k_segsum<<<nc, kB, 0, s>>>(v, n, P, part_base, RowPart{rpart}, partial,
                                           segsum_ticket(), dst, stride, accumulate ? 1 : 0));
}

void launch_segsum_keys(const double* v, int n, const int* dn, const unsigned long long* keys,
                        KeyFmt fmt, const int* ipart, int P, int part_base, double* partial,
                        double* dst, int stride, bool accumulate, cudaStream_t s) {
    const int nc = segsum_chunks(n);
    DABD_LAUNCH("k_segsum", s,
                k_segsum<<<nc, kB, 0, s>>>(v, n, P, part_base,
                                           KeyPart{keys, fmt, ipart, dn, part_base + P - 1},
                                           partial, segsum_ticket(), dst, stride,
                                           accumulate ? 1 : 0));
}

void launch_energy(const SolverView& sv, const unsigned long long* keys, int cap, const int* dn,
                   KeyFmt fmt, int qmode, int which, double* partial, double* dst, int stride,
                   bool accept, FrameCtrl* ctrl, CondHandles hd, cudaStream_t s, bool apply, int tail_max_iters,
                   int* iter_reset) {
    const int ncr = energy_chunks(sv.n_rows), nck = energy_chunks(cap);
    EnergyArgs ea{keys, cap, dn, fmt, qmode, which, ncr, partial, segsum_ticket(), dst, stride,
                  accept ? 1 : 0, ctrl, hd, apply && accept ? 1 : 0, accept && tail_max_iters > 0 ? 1 : 0,
                  tail_max_iters, iter_reset};
    DABD_LAUNCH("k_energy", s, k_energy<<<ncr + nck, kB, 0, s>>>(sv, ea));
}

void launch_accept_trial(const SolverView& sv, cudaStream_t s) {
    if (sv.n_inst == 0) return;
    DABD_LAUNCH("k_accept_trial", s, k_accept_trial<<<grid_for(sv.n_inst, kB), kB, 0, s>>>(sv));
}

void launch_make_trial(const SolverView& sv, bool use_alpha, double alpha, int which,
                       cudaStream_t s) {
    if (sv.n_inst == 0) return;
    DABD_LAUNCH("k_make_trial", s, k_make_trial<<<grid_for(sv.n_inst, kB), kB, 0, s>>>(sv, use_alpha ? 1 : 0, alpha, which));
}

void launch_dq_inf(const SolverView& sv, cudaStream_t s) {
    if (sv.n_rows == 0) return;
    DABD_LAUNCH("k_dq_inf", s, k_dq_inf<<<grid_for(sv.n_rows, kB), kB, 0, s>>>(sv));
}

void launch_ccd(const SolverView& sv, const unsigned long long* keys, int n, const int* dn,
                KeyFmt fmt, const Box* box0, const double* q0, const double* q1, int which,
                double* earliest_override, cudaStream_t s, FrameCtrl* alpha_max_ctrl,
                const CondHandles* hd) {
    CcdFinish fin{nullptr, CondHandles{}, nullptr};
    if (alpha_max_ctrl) fin = CcdFinish{alpha_max_ctrl, *hd, segsum_ticket()};
    if (n == 0 && !alpha_max_ctrl) return;
    DABD_LAUNCH("k_ccd", s,
                k_ccd<<<grid_for(std::max(n, 1), kB), kB, 0, s>>>(sv, keys, n, dn, fmt, box0, q0, q1, which,
                                                                   earliest_override, fin));
}

void launch_toi_reset(PartState* ps, int P, FrameCtrl* ctrl, cudaStream_t s) {
    DABD_LAUNCH("k_toi_reset", s, k_toi_reset<<<1, 64, 0, s>>>(ps, P, ctrl));
}

void launch_ccd_prep(const SolverView& sv, const double* qref, const double* skin, double* skin_next,
                     double s_min, double grow, ListState* ls, unsigned long long cond, int graph,
                     Box* box, cudaStream_t s) {
    DABD_LAUNCH("k_ccd_prep", s,
                k_ccd_prep<<<grid_for(std::max(sv.n_inst, 1), kB, 148), kB, 0, s>>>(
                    sv, qref, skin, skin_next, s_min, grow, ls, cond, graph, box));
}

} // namespace dabd_gpu
