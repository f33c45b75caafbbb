// 3D affine-body contact primitives ("3D ABD: 12-DoF
// bodies, point-triangle and edge-edge distance, barrier"). The reference is
// 2D (point-edge only, proj/src/geometry.cpp:15-97), so this extends its
// formulation: the same unsigned distance d, the same log barrier on d
// (energy.cpp:50-61) and the same PSD clamp of the contact Hessian
// (objective.cpp:12-17), for
//   point-triangle (PT): p of body a against triangle (t0, t1, t2) of body b,
//   edge-edge (EE):      edge (a0, a1) of body a against edge (b0, b1) of body b.
// Body DoF q = [p_x, p_y, p_z, A00, A01, A02, A10, ..., A22] (12), world
// point x = A xbar + p. Parity is unpinned (no reference); the checker is the
// independent CPU restatement in oracle/geometry3d.cpp plus finite
// differences (tests/test_gpu_contact3d.py).
//
// Distance types (closest features):
//   PT: 0..2 point-vertex t_k, 3..5 point-edge (t0t1, t1t2, t2t0), 6 point-plane;
//   EE: 0..3 vertex-vertex (a0b0, a0b1, a1b0, a1b1), 4..5 a_k against edge b,
//       6..7 b_k against edge a, 8 line-line.
// Derivatives come from f = d^2 written over 1..3 difference vectors v_m =
// sum_i R[m][i] x_i of the four contact points (R entries in {-1, 0, 1}):
//   point-point  f = |v|^2,                       v = x_i - x_j
//   point-edge   f = |r|^2 - (r.e)^2 / |e|^2,       r = p - e0, e = e1 - e0
//   plane / line f = (w.(a x b))^2 / |a x b|^2,     w, a, b (triple product)
// then d = sqrt f, grad d = grad f / 2d, hess d = hess f / 2d - grad f grad f^T / 4d^3.
#pragma once

#include "energy.cuh"

namespace dabd_gpu {

struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 v3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross3(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

// x = A xbar + p (row-major A in q[3..11]).
__device__ __forceinline__ V3 world3(const double* q, V3 xb) {
    return {q[0] + (q[3] * xb.x + q[4] * xb.y + q[5] * xb.z),
            q[1] + (q[6] * xb.x + q[7] * xb.y + q[8] * xb.z),
            q[2] + (q[9] * xb.x + q[10] * xb.y + q[11] * xb.z)};
}

// ---------------------------------------------------------------------------
// closest-feature classification
// ---------------------------------------------------------------------------
// Point-segment: parameter of the closest point, clamped to [0, 1].
__device__ __forceinline__ double seg_param(V3 p, V3 e0, V3 e1) {
    const V3 e = e1 - e0;
    const double L = dot3(e, e);
    if (!(L > 0.0)) return 0.0;
    const double t = dot3(p - e0, e) / L;
    return fmin(fmax(t, 0.0), 1.0);
}

// PT type: Voronoi regions of the triangle (vertex, edge, face) for p.
__device__ __forceinline__ int pt_type(V3 p, V3 t0, V3 t1, V3 t2) {
    const V3 ab = t1 - t0, ac = t2 - t0, ap = p - t0;
    const double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) return 0;
    const V3 bp = p - t1;
    const double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) return 1;
    const V3 cp = p - t2;
    const double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) return 2;
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return 3; // edge t0t1
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return 5; // edge t2t0
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) return 4; // edge t1t2
    return 6;
}

// EE type from the clamped closest-point parameters (s on a, t on b);
// near-parallel edges (|a x b|^2 <= 1e-20 |a|^2 |b|^2) take the endpoint cases.
__device__ __forceinline__ int ee_type(V3 a0, V3 a1, V3 b0, V3 b1) {
    const V3 u = a1 - a0, v = b1 - b0, w = a0 - b0;
    const double a = dot3(u, u), b = dot3(u, v), c = dot3(v, v), d = dot3(u, w), e = dot3(v, w);
    const double den = a * c - b * b;
    const V3 n = cross3(u, v);
    const bool parallel = !(dot3(n, n) > 1e-20 * a * c);
    double s = 0.0;
    if (!parallel) s = fmin(fmax((b * e - c * d) / den, 0.0), 1.0);
    double t = (b * s + e) / c;
    if (t < 0.0) {
        t = 0.0;
        s = fmin(fmax(-d / a, 0.0), 1.0);
    } else if (t > 1.0) {
        t = 1.0;
        s = fmin(fmax((b - d) / a, 0.0), 1.0);
    }
    const bool s_end = s == 0.0 || s == 1.0, t_end = t == 0.0 || t == 1.0;
    if (!parallel && !s_end && !t_end) return 8;
    if (s_end && t_end) return (s == 0.0 ? 0 : 2) + (t == 0.0 ? 0 : 1);
    if (s_end) return s == 0.0 ? 4 : 5; // a endpoint against edge b
    if (t_end) return t == 0.0 ? 6 : 7; // b endpoint against edge a
    // parallel with both interior (overlapping parallel edges): any endpoint
    // realises the distance; take a0 against edge b
    return 4;
}

// ---------------------------------------------------------------------------
// f = d^2 and its derivatives over the 12 point coordinates
// ---------------------------------------------------------------------------
// Scatter local derivatives over difference vectors v_m = sum_i R[m][i] x_i
// into the 12-coordinate gradient / Hessian.
template <int M>
__device__ __forceinline__ void scatter(const int (&R)[M][4], const double (&gv)[3 * M],
                                        const double (&Hv)[3 * M][3 * M], double (&g)[12],
                                        double (&H)[12][12]) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        g[i] = 0.0;
#pragma unroll
        for (int j = 0; j < 12; ++j) H[i][j] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (R[m][i] == 0) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c) g[3 * i + c] += R[m][i] * gv[3 * m + c];
        }
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
        for (int n = 0; n < M; ++n)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int rr = R[m][i] * R[n][j];
                    if (rr == 0) continue;
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int e = 0; e < 3; ++e) H[3 * i + c][3 * j + e] += rr * Hv[3 * m + c][3 * n + e];
                }
}

__device__ __forceinline__ double f_pp(const V3 (&x)[4], int i, int j, double (&g)[12], double (&H)[12][12]) {
    const V3 v = x[i] - x[j];
    int R[1][4] = {{0, 0, 0, 0}};
    R[0][i] = 1;
    R[0][j] = -1;
    double gv[3] = {2.0 * v.x, 2.0 * v.y, 2.0 * v.z};
    double Hv[3][3] = {{2, 0, 0}, {0, 2, 0}, {0, 0, 2}};
    scatter<1>(R, gv, Hv, g, H);
    return dot3(v, v);
}

// point x[ip] against the line through x[i0], x[i1]
__device__ __forceinline__ double f_pe(const V3 (&x)[4], int ip, int i0, int i1, double (&g)[12],
                                       double (&H)[12][12]) {
    const V3 r = x[ip] - x[i0], e = x[i1] - x[i0];
    const double L = dot3(e, e), s = dot3(r, e), t = s / L;
    const V3 xc = r - t * e; // r minus its projection
    int R[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    R[0][ip] = 1;
    R[0][i0] = -1;
    R[1][i1] = 1;
    R[1][i0] = -1;
    double gv[6], Hv[6][6];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        gv[c] = 2.0 * comp(xc, c);
        gv[3 + c] = -2.0 * t * comp(xc, c);
    }
    const double iL = 1.0 / L;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double ec = comp(e, c), ek = comp(e, k), rc = comp(r, c), rk = comp(r, k);
            const double dl = c == k ? 1.0 : 0.0;
            Hv[c][k] = 2.0 * dl - 2.0 * ec * ek * iL;                                   // f_rr
            Hv[c][3 + k] = -2.0 * ec * rk * iL + 4.0 * s * ec * ek * iL * iL - 2.0 * t * dl; // f_re
            Hv[3 + k][c] = Hv[c][3 + k];
            Hv[3 + c][3 + k] = -2.0 * rc * rk * iL + 4.0 * t * (rc * ek + ec * rk) * iL -
                               8.0 * t * t * ec * ek * iL + 2.0 * t * t * dl; // f_ee
        }
    scatter<2>(R, gv, Hv, g, H);
    return dot3(xc, xc);
}

// f = (w . (a x b))^2 / |a x b|^2 with w, a, b given by R (point-plane, line-line)
__device__ __forceinline__ double f_triple(const V3 (&x)[4], const int (&R)[3][4], double (&g)[12],
                                           double (&H)[12][12]) {
    V3 v[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        V3 s{0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (R[m][i] != 0) s = s + static_cast<double>(R[m][i]) * x[i];
        v[m] = s;
    }
    const V3 w = v[0], a = v[1], b = v[2];
    const V3 n = cross3(a, b);
    const double N = dot3(w, n), D = dot3(n, n);
    // grad / hess of N and D over (w, a, b) (9 coordinates)
    double gN[9], gD[9], HN[9][9], HD[9][9];
    const V3 bw = cross3(b, w), wa = cross3(w, a), bn = cross3(b, n), na = cross3(n, a);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        gN[c] = comp(n, c);
        gN[3 + c] = comp(bw, c);
        gN[6 + c] = comp(wa, c);
        gD[c] = 0.0;
        gD[3 + c] = 2.0 * comp(bn, c);
        gD[6 + c] = 2.0 * comp(na, c);
    }
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = 0; j < 9; ++j) {
            HN[i][j] = 0.0;
            HD[i][j] = 0.0;
        }
    // [y]x z = y x z; d(a x b)/da = -[b]x, d(a x b)/db = [a]x
    auto skew = [](V3 y, int i, int j) {
        // ([y]x)_{ij}
        const double m[3][3] = {{0.0, -y.z, y.y}, {y.z, 0.0, -y.x}, {-y.y, y.x, 0.0}};
        return m[i][j];
    };
    const double ab = dot3(a, b), aa = dot3(a, a), bb = dot3(b, b);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            // N: d2N/dw da = -[b]x, d2N/dw db = [a]x, d2N/da db = -[w]x
            HN[i][3 + j] = -skew(b, i, j);
            HN[3 + j][i] = HN[i][3 + j];
            HN[i][6 + j] = skew(a, i, j);
            HN[6 + j][i] = HN[i][6 + j];
            HN[3 + i][6 + j] = -skew(w, i, j);
            HN[6 + j][3 + i] = HN[3 + i][6 + j];
            const double dl = i == j ? 1.0 : 0.0;
            // D: d2D/da2 = 2(|b|^2 I - b b^T), d2D/db2 = 2(|a|^2 I - a a^T),
            //    d2D/da db = 2(a b^T - (a.b) I) - 2[n]x
            HD[3 + i][3 + j] = 2.0 * (bb * dl - comp(b, i) * comp(b, j));
            HD[6 + i][6 + j] = 2.0 * (aa * dl - comp(a, i) * comp(a, j));
            HD[3 + i][6 + j] = 2.0 * (comp(a, i) * comp(b, j) - ab * dl) - 2.0 * skew(n, i, j);
            HD[6 + j][3 + i] = HD[3 + i][6 + j];
        }
    const double iD = 1.0 / D, f = N * N * iD;
    double gv[9], Hv[9][9];
#pragma unroll
    for (int i = 0; i < 9; ++i) gv[i] = 2.0 * N * gN[i] * iD - f * gD[i] * iD;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = 0; j < 9; ++j)
            Hv[i][j] = (2.0 * gN[i] * gN[j] + 2.0 * N * HN[i][j]) * iD -
                       2.0 * N * (gN[i] * gD[j] + gD[i] * gN[j]) * iD * iD - f * HD[i][j] * iD +
                       2.0 * f * gD[i] * gD[j] * iD * iD;
    scatter<3>(R, gv, Hv, g, H);
    return f;
}

// d^2 of the classified PT / EE pair and its derivatives over the 12
// coordinates of (x0, x1, x2, x3) = (p, t0, t1, t2) or (a0, a1, b0, b1).
__device__ __forceinline__ double f_pair(int kind, int type, const V3 (&x)[4], double (&g)[12],
                                         double (&H)[12][12]) {
    if (kind == 0) { // point-triangle
        if (type <= 2) return f_pp(x, 0, 1 + type, g, H);
        if (type == 3) return f_pe(x, 0, 1, 2, g, H);
        if (type == 4) return f_pe(x, 0, 2, 3, g, H);
        if (type == 5) return f_pe(x, 0, 3, 1, g, H);
        const int R[3][4] = {{1, -1, 0, 0}, {0, -1, 1, 0}, {0, -1, 0, 1}}; // w = p - t0, a = t1 - t0, b = t2 - t0
        return f_triple(x, R, g, H);
    }
    if (type <= 3) return f_pp(x, type >> 1, 2 + (type & 1), g, H);
    if (type == 4) return f_pe(x, 0, 2, 3, g, H);
    if (type == 5) return f_pe(x, 1, 2, 3, g, H);
    if (type == 6) return f_pe(x, 2, 0, 1, g, H);
    if (type == 7) return f_pe(x, 3, 0, 1, g, H);
    const int R[3][4] = {{-1, 0, 1, 0}, {-1, 1, 0, 0}, {0, 0, -1, 1}}; // w = b0 - a0, a = a1 - a0, b = b1 - b0
    return f_triple(x, R, g, H);
}

// Unsigned distance value only (no derivatives), same formulas.
__device__ __forceinline__ double d_pair_value(int kind, int type, const V3 (&x)[4]) {
    double g[12], H[12][12];
    return sqrt(f_pair(kind, type, x, g, H));
}

} // namespace dabd_gpu
