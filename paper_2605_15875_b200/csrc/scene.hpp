// Host-side scene for dabd_gpu: affine bodies built from world-space loops
// exactly as proj/src/body.cpp:10-118 does (polygon moments, centroid
// re-centring, two identical 3x3 mass blocks), flattened into the SoA layout
// the kernels read. Parameter structs keep the field order and meaning of
// proj/include/dabd/params.hpp:8-41 and scene.hpp:15-56.
#pragma once

#include <cstdint>
#include <map>
#include <utility>
#include <vector>

namespace dabd_gpu {

struct SimParams { // params.hpp:8-15
    double h = 0.01;
    double gravity[2] = {0.0, -9.81};
    double arap_stiffness = 1e6;
    double barrier_stiffness = 1e4;
    double d_hat = 0.01;
    double theta = 1e-3;
    double scene_scale = 1.0;
    void validate() const;
};

struct AdaptParams { // params.hpp:26-32
    double beta = 1.0, tau = 2.0, mu = 5.0, sigma_min = 1e-3, sigma_max = 1e3;
    bool adapt_enabled = true;
    void validate() const;
};

struct PlaneH { // partition.hpp:13-16
    double px = 0.0, py = 0.0, nx = 1.0, ny = 0.0;
};

// Balancer::Options + SceneData::balance_enabled (balance.hpp:24-29, scene.hpp:31-32).
struct BalanceOpts {
    bool enabled = false;
    double kp = 0.0, kd = 0.0, smoothing = 0.5, dp_max = 0.0;
};

struct HostScene {
    // bodies
    int nb = 0;
    int nv = 0;
    std::vector<double> rest;     // [2*nv] centroid-centred rest vertices, loop order
    std::vector<int> vstart;      // [nb+1]
    std::vector<int> vnext;       // [nv] flat index of edge e's second endpoint
    std::vector<int> vbody;       // [nv]
    std::vector<int> is_static;   // [nb]
    std::vector<double> mass;     // [nb]
    std::vector<double> mblk;     // [6*nb] density*(area, sx, sy, sxx, sxy, syy)
    std::vector<double> minv;     // [3*nb] first column of the 3x3 block inverse
    std::vector<double> rest_area;
    std::vector<double> arap_scale;
    std::vector<double> q0, qdot0; // [6*nb]
    int max_verts_per_body = 0;
    // knobs
    SimParams params;
    AdaptParams adapt;
    std::vector<PlaneH> planes;
    double w_min = 0.1;
    int admm_max_iterations = 300;
    int newton_cap = 32;
    int max_halvings = 4;
    int force_split_frames = -1;
    std::map<int, std::pair<double, double>> force_split;
    BalanceOpts balance;

    void full_mass_matrix(int b, double* m36) const; // row-major, body.cpp:84-93
};

// Builds the scene from the flattened JSON-level body specs (scene.cpp:81-98).
HostScene build_scene(int n_bodies, const int* body_loop_start, const int* loop_vert_start,
                      const double* verts, const double* density, const int* is_static,
                      const double* arap_scale, const double* qdot);

} // namespace dabd_gpu
