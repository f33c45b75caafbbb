// Per-body and per-contact energy terms (proj/src/energy.cpp:7-94) and the
// eigenvalue clamp of objective.cpp:12-17, as register-resident device code.
//
// The 12x12 contact block H = t^T A t (t: 6x12 constant map from the two
// bodies' DoF to the world coordinates of (p, e0, e1)) has rank <= 6, so its
// PSD projection is computed exactly through the 6x6 problem
//     G = t t^T = L L^T,  B = L^T A L,  clamp(H) = t^T (L^{-T} clamp(B) L^{-1}) t
// (SURVEY.md 2.3 K7). G is block-structured (point block g_p I2, edge block
// [[g00,g01],[g01,g11]] (x) I2), so L is closed form. Only the 6x6 C =
// L^{-T} clamp(B) L^{-1} (21 unique values) is stored per contact.
#pragma once

#include "common.cuh"

namespace dabd_gpu {

// Jacobi rotation (c, s) that (nearly) annihilates a[p][q]. With d = aqq - app
// and e = 2 apq the annihilating tangent is t = sgn(d) e / (|d| + sqrt(d^2 +
// e^2)) (t = 1 for d = 0). The angle only steers the iteration: it is taken in
// FP32 (MUFU reciprocal / square root on d, e pre-scaled by a power of two, so
// no FP64 divide or square-root chain), and the rotation built from it is
// orthogonal to FP64 rounding (c = (1 + t^2)^-1/2 by two Newton steps from an
// FP32 seed, s = t c). jacobi_rotate applies it as an exact similarity, so the
// eigenvalues keep FP64 accuracy; an angle off by ~1e-7 leaves a residual
// a[p][q] ~1e-7 of the old one, which the next sweep removes. Branch-free
// (selects only), so the N/2 angles of a round interleave.
__device__ __forceinline__ void jacobi_cs(double app, double aqq, double apq, double& c, double& s) {
    const bool on = apq != 0.0;
    const double d = aqq - app, e = 2.0 * apq;
    // 2^-k with 2^k ~ max(|d|, |e|): exponent arithmetic, no division
    const int ex = (max(__double2hiint(fabs(d)), __double2hiint(fabs(e))) >> 20) & 0x7ff;
    const double sc = __hiloint2double((2046 - min(ex, 2045)) << 20, 0);
    const float df = static_cast<float>(d * sc), ef = static_cast<float>(e * sc);
    const float r = sqrtf(fmaf(df, df, ef * ef));
    float tf = copysignf(1.0f, df) * __fdividef(ef, fabsf(df) + r);
    tf = df == 0.0f ? 1.0f : tf;
    const double t = on ? static_cast<double>(tf) : 0.0;
    const double x = fma(t, t, 1.0);
    double y = static_cast<double>(rsqrtf(static_cast<float>(x)));
    y = y * fma(-0.5 * x, y * y, 1.5);
    y = y * fma(-0.5 * x, y * y, 1.5);
    c = on ? y : 1.0;
    s = t * c;
}

// a <- J^T a J, v <- v J for the rotation J in the (p, q) plane (column p =
// (c, -s), column q = (s, c)): the 2x2 pivot block in closed form, rows and
// columns p, q of the rest rotated once and mirrored. The identity rotation
// (1, 0) is an exact no-op.
template <int N>
__device__ __forceinline__ void jacobi_rotate(double (&a)[N][N], double (&v)[N][N], int p, int q,
                                              double c, double s) {
    const double app = a[p][p], aqq = a[q][q], apq = a[p][q];
    const double cc = c * c, ss = s * s, cs2 = 2.0 * c * s;
    const double npp = (cc * app + ss * aqq) - cs2 * apq;
    const double nqq = (ss * app + cc * aqq) + cs2 * apq;
    const double npq = (c * s) * (app - aqq) + (cc - ss) * apq;
    a[p][p] = npp;
    a[q][q] = nqq;
    a[p][q] = npq;
    a[q][p] = npq;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (k == p || k == q) continue;
        const double akp = a[k][p], akq = a[k][q];
        const double np = c * akp - s * akq, nq = s * akp + c * akq;
        a[k][p] = np;
        a[p][k] = np;
        a[k][q] = nq;
        a[q][k] = nq;
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const double vkp = v[k][p], vkq = v[k][q];
        v[k][p] = c * vkp - s * vkq;
        v[k][q] = s * vkp + c * vkq;
    }
}

// Jacobi eigensolver on a symmetric NxN matrix held in registers (N even).
// On return a is diagonal (eigenvalues) and v holds the eigenvectors in its
// columns. Each sweep visits the N(N-1)/2 pairs in round-robin (circle
// method) order: N-1 rounds of N/2 disjoint pairs. The rotations of a round
// commute, so their angles all come from the round's starting matrix and the
// N/2 divide/sqrt chains run side by side (instruction-level parallelism)
// instead of back to back as in cyclic-by-row order: ~N/2 x shorter
// dependent chain per sweep, same quadratic convergence.
template <int N>
__device__ __forceinline__ void jacobi_eig(double (&a)[N][N], double (&v)[N][N]) {
    static_assert(N % 2 == 0, "round-robin ordering needs an even order");
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) v[i][j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 24; ++sweep) {
        double off = 0.0, dg = 0.0;
#pragma unroll
        for (int p = 0; p < N; ++p) {
            dg += a[p][p] * a[p][p];
#pragma unroll
            for (int q = p + 1; q < N; ++q) off += a[p][q] * a[p][q];
        }
        if (!(off > 1e-34 * (2.0 * off + dg))) break;
#pragma unroll
        for (int round = 0; round < N - 1; ++round) {
            // circle method: position 0 fixed, positions 1..N-1 hold
            // players (i - 1 - round) mod (N - 1) + 1; pair position i with N-1-i
            int pp[N / 2], qq[N / 2];
            double cc[N / 2], ss[N / 2];
#pragma unroll
            for (int i = 0; i < N / 2; ++i) {
                const int j = N - 1 - i;
                const int x = i == 0 ? 0 : ((i - 1 + (N - 1) - round) % (N - 1)) + 1;
                const int y = ((j - 1 + (N - 1) - round) % (N - 1)) + 1;
                pp[i] = x < y ? x : y;
                qq[i] = x < y ? y : x;
                jacobi_cs(a[pp[i]][pp[i]], a[qq[i]][qq[i]], a[pp[i]][qq[i]], cc[i], ss[i]);
            }
#pragma unroll
            for (int i = 0; i < N / 2; ++i) jacobi_rotate<N>(a, v, pp[i], qq[i], cc[i], ss[i]);
        }
    }
}

// True iff the symmetric a is positive definite (every Cholesky pivot > 0):
// then clamp_psd(a) == a up to rounding and the eigensolve can be skipped.
template <int N>
__device__ __forceinline__ bool is_pd(const double (&a)[N][N]) {
    double l[N][N];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double d = a[j][j];
#pragma unroll
        for (int k = 0; k < j; ++k) d -= l[j][k] * l[j][k];
        ok = ok && d > 0.0;
        const double ljj = sqrt(fmax(d, 1e-300));
        l[j][j] = ljj;
        const double inv = 1.0 / ljj;
#pragma unroll
        for (int i = j + 1; i < N; ++i) {
            double v = a[i][j];
#pragma unroll
            for (int k = 0; k < j; ++k) v -= l[i][k] * l[j][k];
            l[i][j] = v * inv;
        }
    }
    return ok;
}

// In place: a <- V max(Lambda, 0) V^T.
template <int N>
__device__ __forceinline__ void clamp_psd(double (&a)[N][N]) {
    double v[N][N];
    jacobi_eig<N>(a, v);
    double lam[N];
#pragma unroll
    for (int i = 0; i < N; ++i) lam[i] = fmax(a[i][i], 0.0);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i; j < N; ++j) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) s += v[i][k] * lam[k] * v[j][k];
            a[i][j] = s;
            a[j][i] = s;
        }
}

// clamp_psd of a body block H = ik (M + h^2 H_arap) (+ rho I): translation x
// couples only to (A00, A01) through rho*sx, rho*sy and y only to (A10, A11)
// (mass_full), the ARAP Hessian lives on A alone. Rest shapes are centroid-
// centred (body.cpp:96-118), so those couplings are rounding-level; then the
// translation block is positive and the clamp is that of the 4x4 A block
// (4x4 Jacobi instead of 6x6), exact up to O(|coupling|) <= 1e-13 relative.
// Otherwise (or when the A block is PD, the usual exit) it is the full
// 6x6 clamp of objective.cpp:12-17.
__device__ __forceinline__ void clamp_body_block(double (&H)[6][6]) {
    const double tol = 1e-13 * fmin(H[0][0], H[1][1]);
    const bool decoupled = H[0][0] > 0.0 && H[1][1] > 0.0 && fabs(H[0][2]) <= tol &&
                           fabs(H[0][3]) <= tol && fabs(H[1][4]) <= tol && fabs(H[1][5]) <= tol;
    if (!decoupled) {
        if (!is_pd<6>(H)) clamp_psd<6>(H);
        return;
    }
    double B[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) B[i][j] = H[2 + i][2 + j];
    if (is_pd<4>(B)) return;
    clamp_psd<4>(B);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) H[2 + i][2 + j] = B[i][j];
}

// Inertia 1/2 (q-qt)^T M (q-qt) with the two identical 3x3 blocks of M
// (energy.cpp:7-15; mass layout body.cpp:84-93).
__device__ __forceinline__ void mass_full(const double* k, double (&m)[6][6]) {
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) m[i][j] = 0.0;
    const double blk[3][3] = {{k[0], k[1], k[2]}, {k[1], k[3], k[4]}, {k[2], k[4], k[5]}};
    const int gx[3] = {0, 2, 3}, gy[3] = {1, 4, 5};
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            m[gx[r]][gx[c]] = blk[r][c];
            m[gy[r]][gy[c]] = blk[r][c];
        }
}

// ARAP kappa*area*||A^T A - I||_F^2 on the linear slots (energy.cpp:17-48).
// Adds scale*value to val, scale*grad to g, scale*hess to H.
__device__ __forceinline__ double arap_terms(const double* q, double w, double scale,
                                             double (&g)[6], double (&H)[6][6], bool want_d) {
    const double a[2][2] = {{q[2], q[3]}, {q[4], q[5]}};
    double G[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) G[i][j] = (a[0][i] * a[0][j] + a[1][i] * a[1][j]) - (i == j ? 1.0 : 0.0);
    const double value = w * (G[0][0] * G[0][0] + G[1][0] * G[1][0] + G[0][1] * G[0][1] +
                              G[1][1] * G[1][1]);
    if (want_d) {
        const double w4 = 4.0 * w * scale;
        const double ag00 = a[0][0] * G[0][0] + a[0][1] * G[1][0];
        const double ag01 = a[0][0] * G[0][1] + a[0][1] * G[1][1];
        const double ag10 = a[1][0] * G[0][0] + a[1][1] * G[1][0];
        const double ag11 = a[1][0] * G[0][1] + a[1][1] * G[1][1];
        g[2] += w4 * ag00;
        g[3] += w4 * ag01;
        g[4] += w4 * ag10;
        g[5] += w4 * ag11;
        double aat[2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) aat[i][j] = a[i][0] * a[j][0] + a[i][1] * a[j][1];
        const int slot[2][2] = {{2, 3}, {4, 5}};
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int l = 0; l < 2; ++l)
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        double v = 0.0;
                        if (i == k) v += G[j][l];
                        v += a[i][l] * a[k][j];
                        if (j == l) v += aat[i][k];
                        H[slot[k][l]][slot[i][j]] += w4 * v;
                    }
    }
    return value;
}

struct Barrier {
    double b, db, ddb;
};

// energy.cpp:50-61. Caller guarantees d > 0.
__device__ __forceinline__ Barrier barrier(double d, double dh, double kappa) {
    Barrier o{0.0, 0.0, 0.0};
    if (d >= dh) return o;
    const double gap = d - dh;
    const double lg = log(d / dh);
    o.b = -kappa * gap * gap * lg;
    o.db = -kappa * (2.0 * gap * lg + gap * gap / d);
    o.ddb = -kappa * (2.0 * lg + 2.0 * gap / d + gap * (d + dh) / (d * d));
    return o;
}

// Full point-edge distance with gradient and Hessian (geometry.cpp:15-97).
// Returns d (value bit-exact with pe_distance); g/H over x = (p, e0, e1).
__device__ __forceinline__ double pe_distance_full(V2 p, V2 e0, V2 e1, double (&g)[6],
                                                   double (&H)[6][6]) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        g[i] = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) H[i][j] = 0.0;
    }
    const V2 e = vsub(e1, e0);
    const double len2 = vsqn(e);
    const double t = xdiv(vdot(vsub(p, e0), e), len2);
    if (t <= 0.0 || t >= 1.0) {
        const V2 ee = t <= 0.0 ? e0 : e1;
        const int ei = t <= 0.0 ? 2 : 4;
        const V2 u = vsub(p, ee);
        const double d = xsqrt(vsqn(u));
        if (d <= 0.0) return d;
        const double gx = u.x / d, gy = u.y / d;
        const double k[2][2] = {{(1.0 - gx * gx) / d, (0.0 - gx * gy) / d},
                                {(0.0 - gy * gx) / d, (1.0 - gy * gy) / d}};
        g[0] = gx;
        g[1] = gy;
        // branch-free placement: ei in {2, 4}
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) H[r][c] = k[r][c];
        if (ei == 2) {
            g[2] = -gx;
            g[3] = -gy;
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    H[2 + r][2 + c] = k[r][c];
                    H[r][2 + c] = -k[r][c];
                    H[2 + r][c] = -k[r][c];
                }
        } else {
            g[4] = -gx;
            g[5] = -gy;
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    H[4 + r][4 + c] = k[r][c];
                    H[r][4 + c] = -k[r][c];
                    H[4 + r][c] = -k[r][c];
                }
        }
        return d;
    }
    const V2 w = vsub(p, e0);
    const double c = vcross(e, w);
    const double len = xsqrt(len2);
    const double s = c >= 0.0 ? 1.0 : -1.0;
    const double d = xdiv(xmul(s, c), len);
    const double gc[6] = {-e.y, e.x, e.y - w.y, w.x - e.x, w.y, -w.x};
    const double gl[6] = {0.0, 0.0, -e.x / len, -e.y / len, e.x / len, e.y / len};
    const double a1 = s / len, a2 = d / len;
#pragma unroll
    for (int i = 0; i < 6; ++i) g[i] = a1 * gc[i] - a2 * gl[i];
    const double ehx = e.x / len, ehy = e.y / len;
    const double perp[2][2] = {{(1.0 - ehx * ehx) / len, (0.0 - ehx * ehy) / len},
                               {(0.0 - ehy * ehx) / len, (1.0 - ehy * ehy) / len}};
    const double b1 = s / len, b2 = s / len2, b3 = 2.0 * d / len2, b4 = d / len;
    // hc: constant coupling of cross(e1-e0, p-e0)
    const double hc[6][6] = {{0, 0, 0, 1, 0, -1}, {0, 0, -1, 0, 1, 0}, {0, -1, 0, 0, 0, 1},
                             {1, 0, 0, 0, -1, 0}, {0, 1, 0, -1, 0, 0}, {-1, 0, 1, 0, 0, 0}};
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            double hl = 0.0;
            if (i >= 2 && j >= 2) {
                const double pv = perp[(i - 2) & 1][(j - 2) & 1];
                hl = ((i - 2) >> 1) == ((j - 2) >> 1) ? pv : -pv;
            }
            H[i][j] = ((b1 * hc[i][j] - b2 * (gc[i] * gl[j] + gl[i] * gc[j])) + b3 * (gl[i] * gl[j])) -
                      b4 * hl;
        }
    return d;
}

} // namespace dabd_gpu
