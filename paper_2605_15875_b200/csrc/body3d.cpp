// Mass moments of a 3D affine body from its closed, outward-oriented
// triangle surface (the 3D counterpart of the polygon moments of
// proj/src/body.cpp:10-93): volume integrals of 1, x, x x^T by the
// divergence theorem (Eberly, "Polyhedral Mass Properties"), then re-centred
// at the centroid like make_affine_body (body.cpp:96-118).
#include "body3d.hpp"

#include "dbuf.hpp"

#include <cmath>

namespace dabd_gpu {

namespace {

void subexpr(double w0, double w1, double w2, double& f1, double& f2, double& f3, double& g0,
             double& g1, double& g2) {
    const double t0 = w0 + w1;
    f1 = t0 + w2;
    const double t1 = w0 * w0;
    const double t2 = t1 + w1 * t0;
    f2 = t2 + w2 * f1;
    f3 = w0 * t1 + w1 * t2 + w2 * f2;
    g0 = f2 + w0 * (f1 + w0);
    g1 = f2 + w1 * (f1 + w1);
    g2 = f2 + w2 * (f1 + w2);
}

} // namespace

Moments3 polyhedron_moments(int n_verts, const double* v, int n_tris, const int* tri, double density) {
    double in[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int t = 0; t < n_tris; ++t) {
        const int i0 = tri[3 * t], i1 = tri[3 * t + 1], i2 = tri[3 * t + 2];
        if (i0 < 0 || i1 < 0 || i2 < 0 || i0 >= n_verts || i1 >= n_verts || i2 >= n_verts)
            throw InvalidArg("body3d: triangle vertex index out of range");
        const double x0 = v[3 * i0], y0 = v[3 * i0 + 1], z0 = v[3 * i0 + 2];
        const double x1 = v[3 * i1], y1 = v[3 * i1 + 1], z1 = v[3 * i1 + 2];
        const double x2 = v[3 * i2], y2 = v[3 * i2 + 1], z2 = v[3 * i2 + 2];
        const double a1 = x1 - x0, b1 = y1 - y0, c1 = z1 - z0, a2 = x2 - x0, b2 = y2 - y0, c2 = z2 - z0;
        const double d0 = b1 * c2 - b2 * c1, d1 = a2 * c1 - a1 * c2, d2 = a1 * b2 - a2 * b1;
        double f1x, f2x, f3x, g0x, g1x, g2x, f1y, f2y, f3y, g0y, g1y, g2y, f1z, f2z, f3z, g0z, g1z, g2z;
        subexpr(x0, x1, x2, f1x, f2x, f3x, g0x, g1x, g2x);
        subexpr(y0, y1, y2, f1y, f2y, f3y, g0y, g1y, g2y);
        subexpr(z0, z1, z2, f1z, f2z, f3z, g0z, g1z, g2z);
        in[0] += d0 * f1x;
        in[1] += d0 * f2x;
        in[2] += d1 * f2y;
        in[3] += d2 * f2z;
        in[4] += d0 * f3x;
        in[5] += d1 * f3y;
        in[6] += d2 * f3z;
        in[7] += d0 * (y0 * g0x + y1 * g1x + y2 * g2x);
        in[8] += d1 * (z0 * g0y + z1 * g1y + z2 * g2y);
        in[9] += d2 * (x0 * g0z + x1 * g1z + x2 * g2z);
    }
    in[0] /= 6.0;
    for (int k = 1; k <= 3; ++k) in[k] /= 24.0;
    for (int k = 4; k <= 6; ++k) in[k] /= 60.0;
    for (int k = 7; k <= 9; ++k) in[k] /= 120.0;
    const double vol = in[0];
    if (!(vol > 0.0)) throw InvalidArg("body3d: volume must be > 0 (closed, outward-oriented surface)");
    Moments3 m;
    m.volume = vol;
    for (int c = 0; c < 3; ++c) m.centroid[c] = in[1 + c] / vol;
    const double* c = m.centroid;
    // S about the centroid: int x_i x_j - V c_i c_j (xx, xy, xz, yy, yz, zz)
    const double sxx = in[4] - vol * c[0] * c[0], syy = in[5] - vol * c[1] * c[1], szz = in[6] - vol * c[2] * c[2];
    const double sxy = in[7] - vol * c[0] * c[1], syz = in[8] - vol * c[1] * c[2], szx = in[9] - vol * c[2] * c[0];
    m.mom[0] = density * vol;
    m.mom[1] = m.mom[2] = m.mom[3] = 0.0;
    m.mom[4] = density * sxx;
    m.mom[5] = density * sxy;
    m.mom[6] = density * szx;
    m.mom[7] = density * syy;
    m.mom[8] = density * syz;
    m.mom[9] = density * szz;
    return m;
}

} // namespace dabd_gpu
