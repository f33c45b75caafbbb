// Batched 3D contact terms (contact3d.cu).
#pragma once

#include <cuda_runtime.h>

namespace dabd_gpu {

// Device pointers. kind[k]: 0 point-triangle, 1 edge-edge; qa/qb [n][12];
// rest [n][4][3] (PT: p of a, t0 t1 t2 of b; EE: a0 a1 of a, b0 b1 of b).
// Outputs: d [n], dtype [n], value [n] = weight * b(d) (0 when d >= d_hat),
// grad [n][24] (body a then b), hess [n][24][24] or nullptr.
struct Contact3dArgs {
    int n;
    const int* kind;
    const double* qa;
    const double* qb;
    const double* rest;
    double d_hat, kappa, weight;
    int project;
    double* d;
    int* dtype;
    double* value;
    double* grad;
    double* hess;
    int* err;
};

void launch_contact3d(const Contact3dArgs& a, cudaStream_t s);

// CCD of the same pairs moving linearly from (qa0, qb0) to (qa1, qb1).
struct Ccd3dArgs {
    int n;
    const int* kind;
    const double* qa0;
    const double* qa1;
    const double* qb0;
    const double* qb1;
    const double* rest;
    double* toi;
};

void launch_ccd3d(const Ccd3dArgs& a, cudaStream_t s);

// Body terms of 12-DoF bodies: moments [n][10] = (m, s_x, s_y, s_z, S_xx,
// S_xy, S_xz, S_yy, S_yz, S_zz), w [n] = kappa * volume * arap_scale, scale
// (h^2 in the objective). Outputs value [n], grad [n][12], hess [n][12][12]
// (nullable).
struct Body3dArgs {
    int n;
    const double* q;
    const double* qt;
    const double* moments;
    const double* w;
    double scale;
    int project;
    double* value;
    double* grad;
    double* hess;
};

void launch_body3d(const Body3dArgs& a, cudaStream_t s);

} // namespace dabd_gpu
