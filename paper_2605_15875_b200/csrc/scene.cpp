// Host scene construction (see scene.hpp). Compiled with -ffp-contract=off so
// the moment sums round like the reference (proj/src/body.cpp:10-29).
#include "scene.hpp"

#include "dbuf.hpp"

#include <algorithm>
#include <cmath>

namespace dabd_gpu {

void SimParams::validate() const { // params.hpp:17-22
    if (h <= 0.0) throw InvalidArg("SimParams: h must be > 0");
    if (d_hat <= 0.0) throw InvalidArg("SimParams: d_hat must be > 0");
    if (theta <= 0.0) throw InvalidArg("SimParams: theta must be > 0");
    if (scene_scale <= 0.0) throw InvalidArg("SimParams: scene_scale must be > 0");
}

void AdaptParams::validate() const { // params.hpp:34-40
    if (beta <= 0.0) throw InvalidArg("AdaptParams: beta must be > 0");
    if (tau <= 1.0) throw InvalidArg("AdaptParams: tau must be > 1");
    if (mu <= 1.0) throw InvalidArg("AdaptParams: mu must be > 1");
    if (!(sigma_min > 0.0 && sigma_min < 1.0 && sigma_max > 1.0))
        throw InvalidArg("AdaptParams: need 0 < sigma_min < 1 < sigma_max");
}

namespace {

struct Moments {
    double area = 0, sx = 0, sy = 0, sxx = 0, sxy = 0, syy = 0;
};

// Green's theorem over one positively oriented loop (body.cpp:10-29).
void add_loop(Moments& t, const double* xy, int n) {
    Moments m;
    for (int i = 0; i < n; ++i) {
        const double ax = xy[2 * i], ay = xy[2 * i + 1];
        const int j = (i + 1) % n;
        const double bx = xy[2 * j], by = xy[2 * j + 1];
        const double cr = ax * by - bx * ay;
        m.area += cr / 2.0;
        m.sx += (ax + bx) * cr / 6.0;
        m.sy += (ay + by) * cr / 6.0;
        m.sxx += (ax * ax + ax * bx + bx * bx) * cr / 12.0;
        m.syy += (ay * ay + ay * by + by * by) * cr / 12.0;
        m.sxy += (ax * by + 2.0 * ax * ay + 2.0 * bx * by + bx * ay) * cr / 24.0;
    }
    t.area += m.area;
    t.sx += m.sx;
    t.sy += m.sy;
    t.sxx += m.sxx;
    t.sxy += m.sxy;
    t.syy += m.syy;
}

} // namespace

void HostScene::full_mass_matrix(int b, double* m) const {
    const double* k = &mblk[6 * b];
    const double blk[3][3] = {{k[0], k[1], k[2]}, {k[1], k[3], k[4]}, {k[2], k[4], k[5]}};
    const int gx[3] = {0, 2, 3}, gy[3] = {1, 4, 5};
    for (int i = 0; i < 36; ++i) m[i] = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            m[gx[r] * 6 + gx[c]] = blk[r][c];
            m[gy[r] * 6 + gy[c]] = blk[r][c];
        }
}

HostScene build_scene(int nb, const int* bls, const int* lvs, const double* verts,
                      const double* density, const int* is_static, const double* arap_scale,
                      const double* qdot) {
    if (nb < 0) throw InvalidArg("scene: negative body count");
    HostScene s;
    s.nb = nb;
    s.vstart.assign(nb + 1, 0);
    s.is_static.assign(nb, 0);
    s.mass.assign(nb, 0.0);
    s.mblk.assign(6 * nb, 0.0);
    s.minv.assign(3 * nb, 0.0);
    s.rest_area.assign(nb, 0.0);
    s.arap_scale.assign(nb, 1.0);
    s.q0.assign(6 * nb, 0.0);
    s.qdot0.assign(6 * nb, 0.0);
    for (int b = 0; b < nb; ++b) {
        Moments m;
        for (int l = bls[b]; l < bls[b + 1]; ++l) {
            const int n = lvs[l + 1] - lvs[l];
            if (n < 3) throw InvalidArg("scene: loop with fewer than 3 vertices");
            add_loop(m, verts + 2 * lvs[l], n);
        }
        if (!(m.area > 0.0)) throw InvalidArg("make_affine_body: degenerate polygon (area <= 0)");
        const double cx = m.sx / m.area, cy = m.sy / m.area; // body.cpp:99-100
        s.vstart[b] = static_cast<int>(s.rest.size() / 2);
        std::vector<double> rl; // re-centred loops (body.cpp:106-108)
        for (int l = bls[b]; l < bls[b + 1]; ++l) {
            const int base = static_cast<int>(s.rest.size() / 2);
            const int n = lvs[l + 1] - lvs[l];
            for (int i = 0; i < n; ++i) {
                const double x = verts[2 * (lvs[l] + i)] - cx;
                const double y = verts[2 * (lvs[l] + i) + 1] - cy;
                s.rest.push_back(x);
                s.rest.push_back(y);
                s.vnext.push_back(base + (i + 1) % n);
                s.vbody.push_back(b);
            }
        }
        Moments rm; // mass from the re-centred loops (body.cpp:109, 71-94)
        for (int l = bls[b], v = s.vstart[b]; l < bls[b + 1]; ++l) {
            const int n = lvs[l + 1] - lvs[l];
            add_loop(rm, &s.rest[2 * v], n);
            v += n;
        }
        if (!(rm.area > 0.0)) throw InvalidArg("build_mass_matrix: degenerate polygon (area <= 0)");
        const double d = density[b];
        s.mass[b] = d * rm.area;
        double* k = &s.mblk[6 * b];
        k[0] = rm.area * d;
        k[1] = rm.sx * d;
        k[2] = rm.sy * d;
        k[3] = rm.sxx * d;
        k[4] = rm.sxy * d;
        k[5] = rm.syy * d;
        // First column of the 3x3 block inverse (cofactors), for
        // q_tilde = q + h qdot + h^2 M^{-1} f with f on the translation slots.
        const double a = k[0], bb = k[1], c = k[2], e = k[3], f = k[4], g = k[5];
        const double c00 = e * g - f * f, c10 = -(bb * g - c * f), c20 = bb * f - c * e;
        const double det = a * c00 + bb * c10 + c * c20;
        if (!(det > 0.0) || !(a > 0.0)) throw InvalidArg("predicted_position: singular mass matrix");
        s.minv[3 * b + 0] = c00 / det;
        s.minv[3 * b + 1] = c10 / det;
        s.minv[3 * b + 2] = c20 / det;
        s.rest_area[b] = m.area; // body.cpp:110 (world-loop area)
        s.is_static[b] = is_static[b] != 0;
        s.arap_scale[b] = arap_scale[b];
        double* q = &s.q0[6 * b];
        q[0] = cx;
        q[1] = cy;
        q[2] = 1.0;
        q[5] = 1.0;
        for (int i = 0; i < 6; ++i) s.qdot0[6 * b + i] = qdot[6 * b + i];
    }
    s.vstart[nb] = static_cast<int>(s.rest.size() / 2);
    s.nv = s.vstart[nb];
    for (int b = 0; b < nb; ++b)
        s.max_verts_per_body = std::max(s.max_verts_per_body, s.vstart[b + 1] - s.vstart[b]);
    if (s.max_verts_per_body > 1024) throw InvalidArg("scene: more than 1024 vertices in one body");
    return s;
}

} // namespace dabd_gpu
