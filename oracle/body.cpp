// TEST INFRASTRUCTURE ONLY (see oracle.hpp). Restates proj/src/body.cpp and
// params.hpp validation.
#include "oracle.hpp"

#include <algorithm>
#include <limits>

namespace oracle {

void SimParams::validate() const { // params.hpp:17-22
    if (h <= 0.0) throw Error("SimParams: h must be > 0");
    if (d_hat <= 0.0) throw Error("SimParams: d_hat must be > 0");
    if (theta <= 0.0) throw Error("SimParams: theta must be > 0");
    if (scene_scale <= 0.0) throw Error("SimParams: scene_scale must be > 0");
}

void AdaptParams::validate() const { // params.hpp:34-40
    if (beta <= 0.0) throw Error("AdaptParams: beta must be > 0");
    if (tau <= 1.0) throw Error("AdaptParams: tau must be > 1");
    if (mu <= 1.0) throw Error("AdaptParams: mu must be > 1");
    if (!(sigma_min > 0.0 && sigma_min < 1.0 && sigma_max > 1.0))
        throw Error("AdaptParams: need 0 < sigma_min < 1 < sigma_max");
}

// body.cpp:10-29
PolygonMoments loop_moments(const Loop& loop) {
    PolygonMoments m;
    const int n = static_cast<int>(loop.size());
    for (int i = 0; i < n; ++i) {
        const Vec2 a = loop[i];
        const Vec2 b = loop[(i + 1) % n];
        const double cr = a.x * b.y - b.x * a.y;
        m.area += cr / 2.0;
        m.sx += (a.x + b.x) * cr / 6.0;
        m.sy += (a.y + b.y) * cr / 6.0;
        m.sxx += (a.x * a.x + a.x * b.x + b.x * b.x) * cr / 12.0;
        m.syy += (a.y * a.y + a.y * b.y + b.y * b.y) * cr / 12.0;
        m.sxy += (a.x * b.y + 2.0 * a.x * a.y + 2.0 * b.x * b.y + b.x * a.y) * cr / 24.0;
    }
    return m;
}

// body.cpp:31-43
PolygonMoments loops_moments(const std::vector<Loop>& loops) {
    PolygonMoments t;
    for (const Loop& l : loops) {
        const PolygonMoments m = loop_moments(l);
        t.area += m.area;
        t.sx += m.sx;
        t.sy += m.sy;
        t.sxx += m.sxx;
        t.sxy += m.sxy;
        t.syy += m.syy;
    }
    return t;
}

// body.cpp:49-69: flattened vertex/edge indexing in loop order.
void AffineBody::build_flat() {
    flat.clear();
    next.clear();
    for (const Loop& l : rest_loops) {
        const int base = static_cast<int>(flat.size());
        const int n = static_cast<int>(l.size());
        for (int i = 0; i < n; ++i) {
            flat.push_back(l[i]);
            next.push_back(base + (i + 1) % n);
        }
    }
}

// body.cpp:71-94
void build_mass_matrix(const std::vector<Loop>& loops, double density, double& mass,
                       Mat6& out) {
    const PolygonMoments m = loops_moments(loops);
    if (!(m.area > 0.0)) throw Error("build_mass_matrix: degenerate polygon (area <= 0)");
    mass = density * m.area;
    const double blk[3][3] = {{m.area * density, m.sx * density, m.sy * density},
                              {m.sx * density, m.sxx * density, m.sxy * density},
                              {m.sy * density, m.sxy * density, m.syy * density}};
    const int gx[3] = {0, 2, 3};
    const int gy[3] = {1, 4, 5};
    out = Mat6();
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            out(gx[r], gx[c]) = blk[r][c];
            out(gy[r], gy[c]) = blk[r][c];
        }
}

// body.cpp:96-118
AffineBody make_affine_body(int id, const std::vector<Loop>& world_loops, double density,
                            bool is_static) {
    const PolygonMoments m = loops_moments(world_loops);
    if (!(m.area > 0.0)) throw Error("make_affine_body: degenerate polygon (area <= 0)");
    const Vec2 c{m.sx / m.area, m.sy / m.area};
    AffineBody b;
    b.id = id;
    b.density = density;
    b.is_static = is_static;
    b.rest_loops = world_loops;
    for (Loop& l : b.rest_loops)
        for (Vec2& v : l) v = v - c;
    build_mass_matrix(b.rest_loops, density, b.mass, b.mass_matrix);
    b.rest_area = m.area;
    b.q = zero6();
    b.q[0] = c.x;
    b.q[1] = c.y;
    b.q[2] = 1.0;
    b.q[5] = 1.0;
    b.build_flat();
    return b;
}

// body.cpp:120-127. Eigen::LDLT<Mat6> with diagonal pivoting, restated
// (largest remaining diagonal first, left-looking update).
Vec6 predicted_position(const Vec6& q, const Vec6& q_dot, const Vec6& f, double h,
                        const Mat6& mm) {
    Mat6 a = mm;
    int tr[6];
    for (int k = 0; k < 6; ++k) {
        int big = k;
        double bv = std::abs(a(k, k));
        for (int i = k + 1; i < 6; ++i)
            if (std::abs(a(i, i)) > bv) {
                bv = std::abs(a(i, i));
                big = i;
            }
        tr[k] = big;
        if (big != k) {
            for (int c = 0; c < 6; ++c) std::swap(a(k, c), a(big, c));
            for (int r = 0; r < 6; ++r) std::swap(a(r, k), a(r, big));
        }
        double temp[6];
        for (int j = 0; j < k; ++j) temp[j] = a(j, j) * a(k, j);
        double acc = 0.0;
        for (int j = 0; j < k; ++j) acc += a(k, j) * temp[j];
        a(k, k) -= acc;
        for (int i = k + 1; i < 6; ++i) {
            double s = 0.0;
            for (int j = 0; j < k; ++j) s += a(i, j) * temp[j];
            a(i, k) -= s;
        }
        if (a(k, k) != 0.0)
            for (int i = k + 1; i < 6; ++i) a(i, k) /= a(k, k);
    }
    double dmin = a(0, 0), dmax = a(0, 0);
    for (int i = 1; i < 6; ++i) {
        dmin = std::min(dmin, a(i, i));
        dmax = std::max(dmax, a(i, i));
    }
    if (dmin <= 1e-12 * std::max(dmax, 1e-300))
        throw Error("predicted_position: singular mass matrix");
    double x[6];
    for (int i = 0; i < 6; ++i) x[i] = f[i];
    for (int k = 0; k < 6; ++k) std::swap(x[k], x[tr[k]]);
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < i; ++j) x[i] -= a(i, j) * x[j];
    for (int i = 0; i < 6; ++i) x[i] /= a(i, i);
    for (int i = 5; i >= 0; --i)
        for (int j = i + 1; j < 6; ++j) x[i] -= a(j, i) * x[j];
    for (int k = 5; k >= 0; --k) std::swap(x[k], x[tr[k]]);
    Vec6 out;
    const double h2 = h * h;
    for (int i = 0; i < 6; ++i) out[i] = (q[i] + h * q_dot[i]) + h2 * x[i];
    return out;
}

// body.cpp:129-134
Vec6 gravity_force(const AffineBody& body, Vec2 g) {
    Vec6 f = zero6();
    f[0] = body.mass * g.x;
    f[1] = body.mass * g.y;
    return f;
}

// body.cpp:136-149
Aabb body_aabb(const AffineBody& body, const Vec6& q) {
    Aabb box;
    const double big = std::numeric_limits<double>::max();
    box.lo = {big, big};
    box.hi = {-big, -big};
    for (const Vec2& v : body.flat) {
        const Vec2 x = world_point(q, v);
        box.lo = vmin(box.lo, x);
        box.hi = vmax(box.hi, x);
    }
    return box;
}

// body.cpp:151-161
double max_vertex_speed(const AffineBody& body, const Vec6& qd) {
    double best = 0.0;
    for (const Vec2& v : body.flat) {
        const Vec2 xd{qd[0] + qd[2] * v.x + qd[3] * v.y, qd[1] + qd[4] * v.x + qd[5] * v.y};
        best = std::max(best, norm(xd));
    }
    return best;
}

} // namespace oracle
