// Per-partition scalar control of the batched Newton solve and the N=1 ADMM
// frame controller. In graph mode these kernels also steer the conditional
// WHILE nodes (cudaGraphSetConditional), so a whole frame runs without a
// host round trip.
#include "kernels.hpp"

#include "instrument.hpp"

namespace dabd_gpu {

namespace {

__device__ __forceinline__ void set_cond(unsigned long long h, bool v, int graph) {
    if (graph) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(h), v ? 1u : 0u);
}

__global__ void k_scalar(PartState* ps, int P, int op, FrameCtrl* ctrl, CondHandles hd,
                         double tol, int max_iters, int* err) {
    const int p = threadIdx.x;
    bool act = false, srch = false;
    if (p < P) {
        PartState& s = ps[p];
        switch (op) {
        case kOpReset: {
            const int ndof = s.ndof;
            const bool stop = ctrl && ctrl->ended;
            const int ls = 0;
            s.active = (ndof > 0 && !stop) ? 1 : 0;
            s.converged = ndof > 0 ? 0 : 1;
            s.searching = 0;
            s.accepted = 0;
            s.iterations = 0;
            s.ls_steps = ls;
            s.tol = tol;
            s.final_update = 0.0;
            s.dq_inf = 0.0;
            s.toi_earliest = 2.0;
            s.alpha = 1.0;
            break;
        }
        case kOpEps: // newton.cpp:20-24
            if (s.active) {
                s.eps = 1e-8 * s.trace / s.ndof;
                ++s.iterations;
            }
            break;
        case kOpIterBegin:
            s.dq_inf = 0.0;
            s.toi_earliest = 2.0;
            s.n_candidates = 0;
            s.n_active_contacts = 0;
            break;
        case kOpNewtonCheck: // newton.cpp:30-36
            if (ctrl) atomicAdd(&ctrl->pcg_total, s.pcg_iters);
            if (s.active && s.dq_inf < s.tol) {
                s.final_update = s.dq_inf;
                s.converged = 1;
                s.active = 0;
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
                        s.active = 0;
                        atomicCAS(err, 0, kErrLineSearch);
                    }
                }
            }
            break;
        case kOpNewtonTail: // the loop bound of newton.cpp:16
            if (s.active && s.iterations >= max_iters) s.active = 0;
            break;
        default:
            break;
        }
        act = s.active != 0;
        srch = s.searching != 0;
    }
    const bool any_act = __syncthreads_or(act);
    const bool any_srch = __syncthreads_or(srch);
    if (threadIdx.x == 0) {
        if (ctrl) {
            ctrl->any_active = any_act;
            ctrl->any_searching = any_srch;
            if (op == kOpIterBegin) ++ctrl->exec_newton;
            if (op == kOpAlphaMax) ++ctrl->exec_step;
            if (op == kOpAccept) ++ctrl->exec_ls;
        }
        if (op == kOpReset || op == kOpNewtonTail) set_cond(hd.newton, any_act, hd.graph);
        if (op == kOpNewtonCheck) set_cond(hd.step, any_act, hd.graph);
        if (op == kOpAlphaMax || op == kOpAccept) set_cond(hd.ls, any_srch, hd.graph);
    }
}

// N=1 ADMM frame controller (sim.cpp:221-239).
__global__ void k_frame_ctrl(FrameCtrl* c, int op, const double* dq_part, int P, double h,
                             double l, double theta, int K, double* trace, int trace_cap,
                             CondHandles hd, int* err, const PartState* ps) {
    const double frame = c->frame;
    if (threadIdx.x != 0) return;
    if (op == 0) { // head
        ++c->exec_admm;
        if (c->k > 1) {
            const double nrm = h * l;
            const bool end = c->dq_inf / nrm < theta && 0.0 / nrm < theta && 0.0 / nrm < theta;
            if (trace && c->trace_n < trace_cap) {
                double* row = trace + 8 * c->trace_n;
                row[0] = frame;
                row[1] = 0.0;
                row[2] = c->k;
                row[3] = c->dq_inf;
                row[4] = 0.0;
                row[5] = 0.0;
                row[6] = 1.0;
                row[7] = end ? 1.0 : 0.0;
            }
            ++c->trace_n;
            if (end) {
                c->ended = 1;
                c->admm_iterations = c->k;
            }
        }
        set_cond(hd.admm, !c->ended, hd.graph);
    } else if (op == 1) { // tail: collect the solve, advance k
        double dq = 0.0;
        for (int p = 0; p < P; ++p) {
            dq = fmax(dq, dq_part[p]);
            c->newton_total += ps[p].iterations;
            c->ls_total += ps[p].ls_steps;
        }
        if (!c->ended) c->dq_inf = dq;
        c->k += 1;
        if (!c->ended && c->k > K) {
            c->failed = 1;
            atomicCAS(err, 0, kErrSettle); // run_reference: failed to settle
        }
        set_cond(hd.admm, !c->ended && !c->failed, hd.graph);
    } else { // op 2: init
        c->k = 1;
        c->ended = 0;
        c->failed = 0;
        c->admm_iterations = 0;
        c->dq_inf = 0.0;
        c->trace_n = 0;
        set_cond(hd.admm, true, hd.graph);
    }
}

} // namespace

void launch_scalar(PartState* ps, int P, int op, FrameCtrl* ctrl, CondHandles h, double tol,
                   int max_iters, int* err, cudaStream_t s) {
    DABD_LAUNCH("k_scalar", s,
                k_scalar<<<1, 32, 0, s>>>(ps, P, op, ctrl, h, tol, max_iters, err));
}

void launch_frame_ctrl(FrameCtrl* ctrl, int op, const double* dq_part, int P, double h, double l,
                       double theta, int K, double* trace, int trace_cap, CondHandles hd, int* err,
                       const PartState* ps, cudaStream_t s) {
    DABD_LAUNCH("k_frame_ctrl", s,
                k_frame_ctrl<<<1, 32, 0, s>>>(ctrl, op, dq_part, P, h, l, theta, K, trace,
                                              trace_cap, hd, err, ps));
}

} // namespace dabd_gpu
