// Per-partition scalar updates of the batched Newton/PCG (see kernels.hpp).
#include "kernels.hpp"

#include "instrument.hpp"

namespace dabd_gpu {

namespace {

__global__ void k_scalar(PartState* ps, int P, int op, double* a, double* b, double* c, double tol,
                         int max_iters, int* err) {
    const int p = threadIdx.x;
    if (p >= P) return;
    PartState& s = ps[p];
    switch (op) {
    case kOpPcgStart:
        s.bnorm2 = s.rr;
        s.pcg_done = (!s.active || s.bnorm2 == 0.0) ? 1 : 0;
        s.pcg_iters = 0;
        a[p] = 0.0;
        break;
    case kOpPcgAlpha:
        if (!s.active || s.pcg_done) {
            a[p] = 0.0;
        } else if (!(s.pap > 0.0)) {
            a[p] = 0.0; // breakdown (exactly converged or indefinite): stop
            s.pcg_done = 1;
        } else {
            a[p] = s.rz / s.pap;
        }
        break;
    case kOpPcgBeta:
        if (s.active && !s.pcg_done) {
            const double rz_new = b[p];
            a[p] = s.rz != 0.0 ? rz_new / s.rz : 0.0;
            s.rz = rz_new;
            ++s.pcg_iters;
            if (s.rr <= tol * tol * s.bnorm2 || s.pcg_iters >= max_iters) s.pcg_done = 1;
        }
        break;
    case kOpEps: // newton.cpp:20-24
        if (s.active) {
            s.eps = 1e-8 * s.trace / s.ndof;
            ++s.iterations;
        }
        break;
    case kOpAlphaMax: // geometry.cpp:333-334, newton.cpp:38-44
        if (s.active) {
            const double e = s.toi_earliest;
            s.alpha_max = e > 1.0 ? 1.0 : fmin(1.0, 0.9 * e);
            s.alpha = s.alpha_max;
            s.searching = 1;
        } else {
            s.searching = 0;
        }
        s.accepted = 0;
        break;
    case kOpAccept: // newton.cpp:47-68 (armijo_c = 0: pure decrease)
        s.accepted = 0;
        if (s.searching) {
            if (s.trial < s.energy) {
                s.energy = s.trial;
                s.accepted = 1;
                s.searching = 0;
                s.final_update = s.alpha * s.dq_inf;
                if (s.final_update < s.tol) {
                    s.converged = 1;
                    s.active = 0;
                }
            } else {
                s.alpha *= 0.5;
                ++s.ls_steps;
                if (!(s.alpha >= 1e-12)) {
                    s.searching = 0;
                    atomicCAS(err, 0, 8); // line search failed below 1e-12
                }
            }
        }
        break;
    case kOpNewtonCheck: // newton.cpp:30-36
        if (s.active && s.dq_inf < s.tol) {
            s.final_update = s.dq_inf;
            s.converged = 1;
            s.active = 0;
        }
        break;
    case kOpIterBegin:
        s.dq_inf = 0.0;
        s.toi_earliest = 2.0;
        s.n_candidates = 0;
        break;
    default:
        break;
    }
}

} // namespace

void launch_scalar(PartState* ps, int P, int op, double* a, double* b, double* c, double tol,
                   int max_iters, int* err, cudaStream_t s) {
    DABD_LAUNCH("k_scalar", s, k_scalar<<<1, 32, 0, s>>>(ps, P, op, a, b, c, tol, max_iters, err));
}

} // namespace dabd_gpu
