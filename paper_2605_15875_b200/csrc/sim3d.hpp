// 3D affine-body scene stepping: the reference's
// single-domain frame (sim.cpp:186-249 with newton.cpp:7-71) for 12-DoF
// bodies (q = [p(3), A row-major(9)], x = A xbar + p), on the 3D primitives
// of contact3d.cu / broad3d.cu: predict, then Newton on inertia +
// orthogonality + IPC barrier with a CCD-capped backtracking line search.
// The reference is 2D, so there is no reference 3D frame to be parity-checked
// against; the checks are analytic (free fall), structural (the assembled
// system against the per-term kernels, the PCG direction against a dense
// solve) and physical (penetration-free, monotone energy, rest).
#pragma once

#include "dbuf.hpp"

#include <cuda_runtime.h>

#include <vector>

namespace dabd_gpu {

struct Sim3dParams {
    double h = 1.0 / 60.0;
    double gravity[3] = {0.0, -9.81, 0.0};
    double d_hat = 1e-2;        // barrier activation distance
    double kappa = 1e3;         // barrier stiffness
    double kappa_arap = 1e4;    // orthogonality stiffness x volume (w_b)
    double theta = 1e-3;        // Newton tolerance theta h l on ||dq||_inf (newton.cpp:30-36)
    double scene_scale = 1.0;   // l
    int newton_cap = 64;
    double pcg_rel_tol = 1e-10;
    int pcg_max_iters = 4000;
};

struct Sim3dStats {
    int newton_iterations = 0, line_search_steps = 0, pcg_iterations = 0, max_candidates = 0;
    int converged = 0;
    double min_distance = 0.0; // over the frame's final candidate set (d_hat margin), 0 if none
};

class Sim3d {
  public:
    // verts [nv][3] body-local rest coordinates (about each body's centroid),
    // tris [nt][3] / edges [ne][2] with per-body starts; moments [n][10]
    // (body3d_moments), volume [n]; q0 / qd0 [n][12].
    Sim3d(int device, int n, const int* vstart, const double* verts, const int* tstart, const int* tris,
          const int* estart, const int* edges, const int* is_static, const double* moments,
          const double* volume, const double* q0, const double* qd0, const Sim3dParams& p);
    ~Sim3d();
    Sim3d(const Sim3d&) = delete;
    Sim3d& operator=(const Sim3d&) = delete;

    Sim3dStats frame();
    void state(double* q, double* qd) const;
    void set_state(const double* q, const double* qd);
    // The Newton system at the current state for the predicted q_tilde of the
    // next frame: dense H [12 R][12 R] (R dynamic bodies, PSD-projected,
    // + eps I) and gradient g [12 R], and the PCG direction dq solving H dq = -g.
    int system(double* H, double* g, double* dq);

  private:
    struct Contacts {
        int n = 0;
        DBuf<unsigned long long> keys;
        DBuf<int> kind, a, b;
        DBuf<double> qa, qb, rest, d, value, grad, hess;
        DBuf<int> dtype;
    };
    int candidates(const double* q0, const double* q1, double margin, Contacts& c);
    void contact_terms(Contacts& c, const double* q, bool hess);
    double energy(const double* q, Contacts& c, bool* bad);
    void assemble(Contacts& c);
    int solve();
    double dq_inf();

    int device_ = 0;
    cudaStream_t s_ = nullptr;
    int n_ = 0, R_ = 0;
    Sim3dParams p_;
    std::vector<int> is_static_, row_of_, body_of_row_;
    int pb_bits_ = 1, bb_bits_ = 1;
    DBuf<int> vstart_, tstart_, estart_, tris_, edges_, row_of_d_, stat_d_;
    DBuf<double> verts_, moments_, w_;
    DBuf<double> q_, qd_, qt_, qstart_, dq_, qtry_;
    DBuf<double> bval_, bgrad_, bhess_;
    // BSR system: rows = dynamic bodies; diagonal block + off-diagonal blocks
    std::vector<int> h_bptr_, h_bcol_;
    DBuf<int> bptr_, bcol_, contrib_ptr_, contrib_, gcontrib_ptr_, gcontrib_;
    DBuf<double> blk_, rhs_, x_, pcg_scratch_, red_;
    DBuf<int> cerr_; // a pair at zero distance (k_contact3d)
    PinnedBuf<double> pin_;
    PinnedBuf<int> pin_i_;
    Contacts c0_, cs_;
    int last_pcg_iters_ = 0;
};

} // namespace dabd_gpu
