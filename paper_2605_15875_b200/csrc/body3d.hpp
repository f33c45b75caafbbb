// 3D affine-body mass moments (body3d.cpp).
#pragma once

namespace dabd_gpu {

struct Moments3 {
    double mom[10];     // density * (V, 0, 0, 0, S_xx, S_xy, S_xz, S_yy, S_yz, S_zz) about the centroid
    double centroid[3]; // rest centroid (the initial translation, body.cpp:96-118)
    double volume;
};

Moments3 polyhedron_moments(int n_verts, const double* verts, int n_tris, const int* tris, double density);

} // namespace dabd_gpu
