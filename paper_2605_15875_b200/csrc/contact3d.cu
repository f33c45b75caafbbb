// Batched 3D contact terms: per point-triangle or
// edge-edge pair of two 12-DoF affine bodies, the closest-feature type, the
// unsigned distance, the barrier value (energy.cpp:50-61 in 3D) and its
// gradient and PSD-clamped Hessian over the 24 body DoF. The projection uses
// the rank structure of the 2D kernel (solver.cu, contact_terms_one): with T
// the 12x24 map from the bodies' DoF to the four points, G = T T^T =
// (Gp (x) I3) with Gp = blockdiag over bodies of (1 + xbar_i . xbar_j), so
// clamp(T^T A T) = T^T L^-T clamp(L^T A L) L^-1 T, L = Lp (x) I3: a 12x12
// eigenproblem instead of 24x24 (energy.cuh's round-robin Jacobi). One
// thread per pair.
#include "geometry3d.cuh"

#include "contact3d.hpp"
#include "dbuf.hpp"
#include "instrument.hpp"

namespace dabd_gpu {

namespace {

__global__ void k_contact3d(Contact3dArgs ar) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ar.n) return;
    const int kind = ar.kind[k];
    const double* qa = ar.qa + 12 * static_cast<size_t>(k);
    const double* qb = ar.qb + 12 * static_cast<size_t>(k);
    V3 xb[4], x[4];
    int body[4];
    for (int i = 0; i < 4; ++i) {
        xb[i] = v3(ar.rest + 12 * static_cast<size_t>(k) + 3 * i);
        body[i] = kind == 0 ? (i == 0 ? 0 : 1) : (i < 2 ? 0 : 1);
        x[i] = world3(body[i] == 0 ? qa : qb, xb[i]);
    }
    const int type = kind == 0 ? pt_type(x[0], x[1], x[2], x[3]) : ee_type(x[0], x[1], x[2], x[3]);
    double gf[12], Hf[12][12];
    const double f = f_pair(kind, type, x, gf, Hf);
    const double d = sqrt(f);
    ar.d[k] = d;
    ar.dtype[k] = type;
    double* gout = ar.grad + 24 * static_cast<size_t>(k);
    double* hout = ar.hess ? ar.hess + 576 * static_cast<size_t>(k) : nullptr;
    for (int i = 0; i < 24; ++i) gout[i] = 0.0;
    if (hout)
        for (int i = 0; i < 576; ++i) hout[i] = 0.0;
    if (!(d < ar.d_hat)) {
        ar.value[k] = 0.0;
        return;
    }
    if (!(d > 0.0)) {
        atomicCAS(ar.err, 0, 1);
        ar.value[k] = 0.0;
        return;
    }
    const Barrier br = barrier(d, ar.d_hat, ar.kappa);
    ar.value[k] = ar.weight * br.b;
    // grad d = grad f / 2d, hess d = hess f / 2d - grad f grad f^T / 4d^3
    double gd[12];
    const double i2d = 0.5 / d;
    for (int i = 0; i < 12; ++i) gd[i] = gf[i] * i2d;
    double A[12][12];
    for (int i = 0; i < 12; ++i)
        for (int j = 0; j < 12; ++j) {
            const double hd = Hf[i][j] * i2d - gd[i] * gd[j] / d;
            A[i][j] = ar.weight * (br.ddb * (gd[i] * gd[j]) + br.db * hd);
        }
    // body-space gradient: J(xbar)^T g per point (J = [I3 | I3 (x) xbar^T])
    for (int i = 0; i < 4; ++i) {
        double* gb = gout + 12 * body[i];
        for (int r = 0; r < 3; ++r) {
            const double gi = ar.weight * br.db * gd[3 * i + r];
            gb[r] += gi;
            gb[3 + 3 * r + 0] += gi * xb[i].x;
            gb[3 + 3 * r + 1] += gi * xb[i].y;
            gb[3 + 3 * r + 2] += gi * xb[i].z;
        }
    }
    if (!hout) return;
    if (ar.project) {
        // Gp = blockdiag over bodies of (1 + xbar_i . xbar_j), Cholesky Lp,
        // Li = Lp^-1 (both lower triangular)
        double Gp[4][4], Lp[4][4], Li[4][4];
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                Gp[i][j] = body[i] == body[j] ? 1.0 + dot3(xb[i], xb[j]) : 0.0;
                Lp[i][j] = 0.0;
                Li[i][j] = 0.0;
            }
        for (int j = 0; j < 4; ++j) {
            double s = Gp[j][j];
            for (int l = 0; l < j; ++l) s -= Lp[j][l] * Lp[j][l];
            Lp[j][j] = sqrt(fmax(s, 1e-300));
            for (int i = j + 1; i < 4; ++i) {
                double t = Gp[i][j];
                for (int l = 0; l < j; ++l) t -= Lp[i][l] * Lp[j][l];
                Lp[i][j] = t / Lp[j][j];
            }
        }
        for (int j = 0; j < 4; ++j) {
            Li[j][j] = 1.0 / Lp[j][j];
            for (int i = j + 1; i < 4; ++i) {
                double t = 0.0;
                for (int l = j; l < i; ++l) t -= Lp[i][l] * Li[l][j];
                Li[i][j] = t / Lp[i][i];
            }
        }
        // B = L^T A L, L = Lp (x) I3
        double B[12][12];
        for (int i = 0; i < 4; ++i)
            for (int c = 0; c < 3; ++c)
                for (int j = 0; j < 4; ++j)
                    for (int e = 0; e < 3; ++e) {
                        double s = 0.0;
                        for (int kk = i; kk < 4; ++kk)
                            for (int l = j; l < 4; ++l) s += Lp[kk][i] * A[3 * kk + c][3 * l + e] * Lp[l][j];
                        B[3 * i + c][3 * j + e] = s;
                    }
        for (int i = 0; i < 12; ++i)
            for (int j = i + 1; j < 12; ++j) {
                const double m = 0.5 * (B[i][j] + B[j][i]);
                B[i][j] = m;
                B[j][i] = m;
            }
        clamp_psd<12>(B);
        // A <- L^-T B+ L^-1
        for (int i = 0; i < 4; ++i)
            for (int c = 0; c < 3; ++c)
                for (int j = 0; j < 4; ++j)
                    for (int e = 0; e < 3; ++e) {
                        double s = 0.0;
                        for (int kk = i; kk < 4; ++kk)
                            for (int l = j; l < 4; ++l) s += Li[kk][i] * B[3 * kk + c][3 * l + e] * Li[l][j];
                        A[3 * i + c][3 * j + e] = s;
                    }
    }
    // H = T^T A T: block (body[i], body[j]) += J_i^T A_ij J_j
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            const double xi[3] = {xb[i].x, xb[i].y, xb[i].z}, xj[3] = {xb[j].x, xb[j].y, xb[j].z};
            double* H = hout + 24 * (12 * body[i]) + 12 * body[j];
            for (int r = 0; r < 3; ++r)
                for (int s = 0; s < 3; ++s) {
                    const double m = A[3 * i + r][3 * j + s];
                    // rows: translation r, A_rc (3 + 3r + c); columns likewise with s
                    H[24 * r + s] += m;
                    for (int c = 0; c < 3; ++c) {
                        H[24 * r + 3 + 3 * s + c] += m * xj[c];
                        H[24 * (3 + 3 * r + c) + s] += m * xi[c];
                        for (int c2 = 0; c2 < 3; ++c2) H[24 * (3 + 3 * r + c) + 3 + 3 * s + c2] += m * xi[c] * xj[c2];
                    }
                }
        }
}

// Additive CCD (Li, Kaufman, Jiang 2021) of one 3D pair under linear point
// motion x_i(t) = x_i + t dx_i: conservative advancement by the distance over
// an upper bound l_p of the relative speed, first step (1 - s) d / l_p, later
// steps 0.9 d / l_p, stopping once the distance falls below s d(0). Returns
// 1.0 when the pair stays apart over [0, 1], else a time at which the pair
// still keeps a gap of at least s d(0) (s = 0.1): the 3D counterpart of the
// reference's 0.9 x earliest-root rule (geometry.cpp:232-341).
__device__ double accd_pair(int kind, V3 (&x)[4], V3 (&dx)[4]) {
    constexpr double kS = 0.1;
    V3 mean = 0.25 * (((dx[0] + dx[1]) + dx[2]) + dx[3]);
    double m0 = 0.0, m1 = 0.0;
    for (int i = 0; i < 4; ++i) {
        dx[i] = dx[i] - mean;
        const double n = sqrt(dot3(dx[i], dx[i]));
        if (kind == 0 ? i == 0 : i < 2) m0 = fmax(m0, n);
        else m1 = fmax(m1, n);
    }
    const double lp = m0 + m1;
    if (!(lp > 0.0)) return 1.0;
    auto dist = [&](const V3 (&y)[4]) {
        const int type = kind == 0 ? pt_type(y[0], y[1], y[2], y[3]) : ee_type(y[0], y[1], y[2], y[3]);
        return d_pair_value(kind, type, y);
    };
    double d = dist(x);
    if (!(d > 0.0)) return 0.0;
    const double g = kS * d;
    double t = 0.0, tl = (1.0 - kS) * d / lp;
    for (int it = 0; it < 100000; ++it) {
        for (int i = 0; i < 4; ++i) x[i] = x[i] + tl * dx[i];
        d = dist(x);
        if (t > 0.0 && d < g) break;
        t += tl;
        if (t > 1.0) return 1.0;
        tl = 0.9 * d / lp;
    }
    return t;
}

__global__ void k_ccd3d(Ccd3dArgs ar) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ar.n) return;
    const int kind = ar.kind[k];
    const size_t o = 12 * static_cast<size_t>(k);
    V3 x[4], dx[4];
    for (int i = 0; i < 4; ++i) {
        const V3 xb = v3(ar.rest + o + 3 * i);
        const bool on_a = kind == 0 ? i == 0 : i < 2;
        const V3 x0 = world3((on_a ? ar.qa0 : ar.qb0) + o, xb), x1 = world3((on_a ? ar.qa1 : ar.qb1) + o, xb);
        x[i] = x0;
        dx[i] = x1 - x0;
    }
    ar.toi[k] = accd_pair(kind, x, dx);
}

// 3D body terms (the 12-DoF counterpart of energy.cpp:7-48 / objective.cpp:
// 117-167): inertia 1/2 (q - qt)^T M (q - qt) with M = per-row 4x4 blocks
// [[m, s^T], [s, S]] over (p_r, A_r0, A_r1, A_r2) (s, S: first / second mass
// moments about the rest centroid), plus scale * w ||A^T A - I||_F^2, and the
// PSD clamp of the 12x12 Hessian. With centroid-centred rest shapes the
// translation coupling s is rounding-level: then only the 9x9 A block is
// clamped (padded to 10 for the round-robin Jacobi), else the full 12x12.
__global__ void k_body3d(Body3dArgs ar) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= ar.n) return;
    const double* q = ar.q + 12 * static_cast<size_t>(b);
    const double* qt = ar.qt + 12 * static_cast<size_t>(b);
    const double* mo = ar.moments + 10 * static_cast<size_t>(b);
    const double m = mo[0], s[3] = {mo[1], mo[2], mo[3]};
    const double S[3][3] = {{mo[4], mo[5], mo[6]}, {mo[5], mo[7], mo[8]}, {mo[6], mo[8], mo[9]}};
    double H[12][12], g[12];
    for (int i = 0; i < 12; ++i) {
        g[i] = 0.0;
        for (int j = 0; j < 12; ++j) H[i][j] = 0.0;
    }
    // mass matrix rows: translation r -> r, A_rc -> 3 + 3r + c
    for (int r = 0; r < 3; ++r) {
        H[r][r] = m;
        for (int c = 0; c < 3; ++c) {
            H[r][3 + 3 * r + c] = s[c];
            H[3 + 3 * r + c][r] = s[c];
            for (int c2 = 0; c2 < 3; ++c2) H[3 + 3 * r + c][3 + 3 * r + c2] = S[c][c2];
        }
    }
    double diff[12], md[12];
    for (int i = 0; i < 12; ++i) diff[i] = q[i] - qt[i];
    double ein = 0.0;
    for (int i = 0; i < 12; ++i) {
        double t = 0.0;
        for (int j = 0; j < 12; ++j) t += H[i][j] * diff[j];
        md[i] = t;
        ein += diff[i] * t;
    }
    ein *= 0.5;
    // ||A^T A - I||^2: grad 4 A G, hess_{(ij),(kl)} = 4 (d_ik G_lj + A_il A_kj + d_jl (A A^T)_ik)
    double A[3][3], G[3][3], AAt[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) A[i][j] = q[3 + 3 * i + j];
    double psi = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double t = 0.0, u = 0.0;
            for (int k = 0; k < 3; ++k) {
                t += A[k][i] * A[k][j];
                u += A[i][k] * A[j][k];
            }
            G[i][j] = t - (i == j ? 1.0 : 0.0);
            AAt[i][j] = u;
            psi += G[i][j] * G[i][j];
        }
    const double w = ar.scale * ar.w[b];
    ar.value[b] = ein + w * psi;
    double* gout = ar.grad + 12 * static_cast<size_t>(b);
    for (int i = 0; i < 12; ++i) g[i] = md[i];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double t = 0.0;
            for (int k = 0; k < 3; ++k) t += A[i][k] * G[k][j];
            g[3 + 3 * i + j] += 4.0 * w * t;
        }
    for (int i = 0; i < 12; ++i) gout[i] = g[i];
    if (!ar.hess) return;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l) {
                    double v = A[i][l] * A[k][j];
                    if (i == k) v += G[l][j];
                    if (j == l) v += AAt[i][k];
                    H[3 + 3 * i + j][3 + 3 * k + l] += 4.0 * w * v;
                }
    if (ar.project) {
        const double tol = 1e-13 * m;
        bool decoupled = m > 0.0;
        for (int c = 0; c < 3; ++c) decoupled = decoupled && fabs(s[c]) <= tol;
        if (decoupled) {
            double B[10][10];
            for (int i = 0; i < 10; ++i)
                for (int j = 0; j < 10; ++j) B[i][j] = i < 9 && j < 9 ? H[3 + i][3 + j] : (i == j ? 1.0 : 0.0);
            if (!is_pd<10>(B)) {
                clamp_psd<10>(B);
                for (int i = 0; i < 9; ++i)
                    for (int j = 0; j < 9; ++j) H[3 + i][3 + j] = B[i][j];
            }
        } else if (!is_pd<12>(H)) {
            clamp_psd<12>(H);
        }
    }
    double* hout = ar.hess + 144 * static_cast<size_t>(b);
    for (int i = 0; i < 12; ++i)
        for (int j = 0; j < 12; ++j) hout[12 * i + j] = H[i][j];
}

} // namespace

void launch_body3d(const Body3dArgs& a, cudaStream_t s) {
    if (a.n <= 0) return;
    DABD_LAUNCH("k_body3d", s, k_body3d<<<(a.n + 63) / 64, 64, 0, s>>>(a));
}

void launch_ccd3d(const Ccd3dArgs& a, cudaStream_t s) {
    if (a.n <= 0) return;
    DABD_LAUNCH("k_ccd3d", s, k_ccd3d<<<(a.n + 63) / 64, 64, 0, s>>>(a));
}

void launch_contact3d(const Contact3dArgs& a, cudaStream_t s) {
    if (a.n <= 0) return;
    DABD_LAUNCH("k_contact3d", s, k_contact3d<<<(a.n + 63) / 64, 64, 0, s>>>(a));
}

} // namespace dabd_gpu
