// Host launch wrappers of the solver/ADMM kernels (solver.cu, admm.cu).
#pragma once

#include "geometry.cuh"
#include "solver.hpp"

namespace dabd_gpu {

// which: 0 = partitions with an active Newton, 1 = partitions in a line
// search, 2 = every partition.
void launch_body_terms(const SolverView& sv, const double* q, bool derivs, int which,
                       cudaStream_t s);
void launch_filter(const SolverView& sv, const unsigned long long* keys, int n, KeyFmt fmt,
                   const Box* box, const double* q, int mode, int which, unsigned char* flag,
                   double* val, cudaStream_t s);
void launch_contact_terms(const SolverView& sv, const ContactView& cv, cudaStream_t s);
void launch_seg_offsets(const unsigned long long* keys, int n, KeyFmt fmt, int n_inst, int* off,
                        int field, const int* perm, cudaStream_t s);
void launch_make_bkeys(const unsigned long long* keys, int n, KeyFmt fmt, unsigned long long* bkeys,
                       int* idx, cudaStream_t s);
void launch_assemble(const SolverView& sv, const ContactView& cv, double* row_trace,
                     cudaStream_t s);
void launch_precond(const SolverView& sv, cudaStream_t s);
int segsum_chunks(int n);
void launch_segsum_rows(const double* v, int n, const int* rpart, int P, int part_base,
                        double* partial, double* dst, int stride, bool accumulate, cudaStream_t s);
void launch_segsum_keys(const double* v, int n, const unsigned long long* keys, KeyFmt fmt,
                        const int* ipart, int P, int part_base, double* partial, double* dst,
                        int stride, bool accumulate, cudaStream_t s);
void launch_pcg_init(const SolverView& sv, double* rz, double* rr, cudaStream_t s);
void launch_pcg_spmv(const SolverView& sv, const double* pold, double* pnew, const double* beta,
                     double* pap_row, cudaStream_t s);
void launch_pcg_update(const SolverView& sv, const double* pnew, const double* alpha, double* rz,
                       double* rr, cudaStream_t s);
void launch_make_trial(const SolverView& sv, bool use_alpha, double alpha, int which,
                       cudaStream_t s);
void launch_dq_inf(const SolverView& sv, cudaStream_t s);
void launch_ccd(const SolverView& sv, const unsigned long long* keys, int n, KeyFmt fmt,
                const Box* box0, const double* q0, const double* q1, int which,
                double* earliest_override, cudaStream_t s);

// Persistent cooperative block-Jacobi PCG over all partitions (pcg.cu).
// pbuf: 12 * n_rows doubles; partials: 3 * pcg_grid_size(n_rows) * P doubles.
int pcg_grid_size(int n_rows);
void launch_pcg_persistent(const SolverView& sv, double* pbuf, double* partials, double* rowval,
                           double tol, int max_iters, cudaStream_t s);

// Per-partition scalar steps (solver_scalar.cu). `op` selects the update.
enum ScalarOp : int {
    kOpPcgStart = 0,  // bnorm2 = rr; pcg_done = (bnorm2 == 0); iters = 0; beta = 0
    kOpPcgAlpha = 1,  // alpha = rz / pap
    kOpPcgBeta = 2,   // beta = rz_new / rz; rz = rz_new; done if rr <= tol^2 bnorm2 or iters>=max
    kOpEps = 3,       // eps = 1e-8 * trace / ndof
    kOpAlphaMax = 4,  // alpha_max from toi_earliest; alpha = alpha_max; searching = 1
    kOpAccept = 5,    // line-search decision (newton.cpp:47-62)
    kOpNewtonCheck = 6, // dq_inf < tol -> converged without moving (newton.cpp:30-36)
    kOpIterBegin = 7    // dq_inf = 0, toi_earliest = 2, n_candidates = 0
};
void launch_scalar(PartState* ps, int P, int op, double* a, double* b, double* c, double tol,
                   int max_iters, int* err, cudaStream_t s);

} // namespace dabd_gpu
