// TEST INFRASTRUCTURE ONLY: CPU restatement of the 3D affine-body contact
// primitives of paper_2605_15875_b200/csrc/geometry3d.cuh / contact3d.cu
// (SURVEY.md 8(f) row 1). The reference is 2D, so nothing pins these values
// ("parity unpinned"); this file computes them a second, independent way:
//   * the unsigned distance as the minimum over every candidate feature pair
//     (point-plane when the projection falls inside the triangle, the three
//     point-segment distances; for edges the interior line-line distance when
//     both closest parameters are interior, the four endpoint-segment
//     distances), instead of the kernel's Voronoi-region classification;
//   * the barrier value b(d) = -kappa (d - d_hat)^2 ln(d / d_hat) of
//     proj/src/energy.cpp:50-61.
// tests/test_gpu_contact3d.py checks the kernel's distance, type and value
// against this, its gradient against central differences of this value and
// its projected Hessian against numpy's eigen-clamp of the finite-difference
// Hessian.
#include <algorithm>
#include <array>
#include <cmath>

namespace oracle3d {

using V = std::array<double, 3>;

static V sub(const V& a, const V& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
static double dot(const V& a, const V& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static V cross(const V& a, const V& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
static V axpy(double s, const V& x, const V& y) { return {y[0] + s * x[0], y[1] + s * x[1], y[2] + s * x[2]}; }

static V world(const double* q, const double* xb) {
    V x;
    for (int r = 0; r < 3; ++r) x[r] = q[r] + (q[3 + 3 * r] * xb[0] + q[4 + 3 * r] * xb[1] + q[5 + 3 * r] * xb[2]);
    return x;
}

// distance from p to segment [a, b]; *interior = closest point strictly inside
static double point_segment(const V& p, const V& a, const V& b, bool* interior) {
    const V e = sub(b, a);
    const double L = dot(e, e);
    double t = L > 0.0 ? dot(sub(p, a), e) / L : 0.0;
    *interior = t > 0.0 && t < 1.0;
    t = std::clamp(t, 0.0, 1.0);
    const V c = axpy(t, e, a);
    const V r = sub(p, c);
    return std::sqrt(dot(r, r));
}

static double point_point(const V& a, const V& b) {
    const V r = sub(a, b);
    return std::sqrt(dot(r, r));
}

// PT: types 0-2 vertex, 3-5 edge (t0t1, t1t2, t2t0), 6 face
static double pt_distance(const V& p, const V& t0, const V& t1, const V& t2, int* type) {
    double best = INFINITY;
    int bt = -1;
    auto take = [&](double d, int t) {
        if (d < best) {
            best = d;
            bt = t;
        }
    };
    const V n = cross(sub(t1, t0), sub(t2, t0));
    const double nn = dot(n, n);
    // barycentric coordinates of the projection
    const V w = sub(p, t0);
    const double s = dot(w, n) / nn;
    const V pr = axpy(-s, n, p);
    const double a0 = dot(cross(sub(t1, pr), sub(t2, pr)), n), a1 = dot(cross(sub(t2, pr), sub(t0, pr)), n),
                 a2 = dot(cross(sub(t0, pr), sub(t1, pr)), n);
    if (a0 > 0.0 && a1 > 0.0 && a2 > 0.0) take(std::fabs(s) * std::sqrt(nn), 6);
    const V tv[3] = {t0, t1, t2};
    for (int e = 0; e < 3; ++e) {
        bool inside;
        const double d = point_segment(p, tv[e], tv[(e + 1) % 3], &inside);
        if (inside) take(d, 3 + e);
    }
    for (int v = 0; v < 3; ++v) take(point_point(p, tv[v]), v);
    *type = bt;
    return best;
}

// EE: 0-3 vertex pairs (a0b0, a0b1, a1b0, a1b1), 4-5 a0/a1 vs edge b, 6-7 b0/b1 vs edge a, 8 line-line
static double ee_distance(const V& a0, const V& a1, const V& b0, const V& b1, int* type) {
    double best = INFINITY;
    int bt = -1;
    auto take = [&](double d, int t) {
        if (d < best) {
            best = d;
            bt = t;
        }
    };
    const V u = sub(a1, a0), v = sub(b1, b0), w = sub(a0, b0);
    const double a = dot(u, u), b = dot(u, v), c = dot(v, v), d = dot(u, w), e = dot(v, w);
    const double den = a * c - b * b;
    const V n = cross(u, v);
    if (dot(n, n) > 1e-20 * a * c) {
        const double s = (b * e - c * d) / den, t = (a * e - b * d) / den;
        if (s > 0.0 && s < 1.0 && t > 0.0 && t < 1.0) take(std::fabs(dot(sub(b0, a0), n)) / std::sqrt(dot(n, n)), 8);
    }
    bool in;
    double dd = point_segment(a0, b0, b1, &in);
    if (in) take(dd, 4);
    dd = point_segment(a1, b0, b1, &in);
    if (in) take(dd, 5);
    dd = point_segment(b0, a0, a1, &in);
    if (in) take(dd, 6);
    dd = point_segment(b1, a0, a1, &in);
    if (in) take(dd, 7);
    take(point_point(a0, b0), 0);
    take(point_point(a0, b1), 1);
    take(point_point(a1, b0), 2);
    take(point_point(a1, b1), 3);
    *type = bt;
    return best;
}

} // namespace oracle3d

extern "C" {

// kind 0 PT / 1 EE; qa, qb [12]; rest [4][3]. Writes d, type, value = weight * b(d).
int oracle_contact3d_value(int kind, const double* qa, const double* qb, const double* rest,
                           double d_hat, double kappa, double weight, double* d, int* type,
                           double* value) {
    using namespace oracle3d;
    V x[4];
    for (int i = 0; i < 4; ++i) {
        const bool on_a = kind == 0 ? i == 0 : i < 2;
        x[i] = world(on_a ? qa : qb, rest + 3 * i);
    }
    const double dist = kind == 0 ? pt_distance(x[0], x[1], x[2], x[3], type)
                                  : ee_distance(x[0], x[1], x[2], x[3], type);
    *d = dist;
    if (!(dist < d_hat)) {
        *value = 0.0;
        return 0;
    }
    if (!(dist > 0.0)) return 1;
    const double r = dist - d_hat; // energy.cpp:50-61
    *value = weight * (-kappa * r * r * std::log(dist / d_hat));
    return 0;
}

} // extern "C"

extern "C" {

// Additive CCD of one pair (same rule as csrc/contact3d.cu accd_pair), with
// this file's minimum-over-features distance.
double oracle_ccd3d(int kind, const double* qa0, const double* qa1, const double* qb0,
                    const double* qb1, const double* rest) {
    using namespace oracle3d;
    V x[4], dx[4];
    for (int i = 0; i < 4; ++i) {
        const bool on_a = kind == 0 ? i == 0 : i < 2;
        x[i] = world(on_a ? qa0 : qb0, rest + 3 * i);
        const V x1 = world(on_a ? qa1 : qb1, rest + 3 * i);
        dx[i] = sub(x1, x[i]);
    }
    V mean;
    for (int c = 0; c < 3; ++c) mean[c] = 0.25 * (((dx[0][c] + dx[1][c]) + dx[2][c]) + dx[3][c]);
    double m0 = 0.0, m1 = 0.0;
    for (int i = 0; i < 4; ++i) {
        dx[i] = sub(dx[i], mean);
        const double n = std::sqrt(dot(dx[i], dx[i]));
        if (kind == 0 ? i == 0 : i < 2) m0 = std::max(m0, n);
        else m1 = std::max(m1, n);
    }
    const double lp = m0 + m1;
    if (!(lp > 0.0)) return 1.0;
    auto dist = [&]() {
        int t;
        return kind == 0 ? pt_distance(x[0], x[1], x[2], x[3], &t) : ee_distance(x[0], x[1], x[2], x[3], &t);
    };
    double d = dist();
    if (!(d > 0.0)) return 0.0;
    const double g = 0.1 * d;
    double t = 0.0, tl = 0.9 * d / lp;
    for (int it = 0; it < 100000; ++it) {
        for (int i = 0; i < 4; ++i) x[i] = axpy(tl, dx[i], x[i]);
        d = dist();
        if (t > 0.0 && d < g) break;
        t += tl;
        if (t > 1.0) return 1.0;
        tl = 0.9 * d / lp;
    }
    return t;
}

} // extern "C"
