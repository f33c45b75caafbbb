// Per-partition scalar control of the batched Newton solve (newton.cpp:16-69)
// as a block-level device function; in graph mode it also steers the
// conditional nodes (cudaGraphSetConditional).
#pragma once

#include "kernels.hpp"

namespace dabd_gpu {

__device__ __forceinline__ void set_cond(unsigned long long h, bool v, int graph) {
    if (graph) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(h), v ? 1u : 0u);
}

// One step of the per-partition scalar control, executed by ALL threads of
// one block (blockDim.x >= P). Shared by k_scalar and the fused kernels that
// finish with a control step (k_energy's line-search accept).
// iter_reset (fused Newton body, kOpReset / kOpNewtonTail only): when the
// Newton loop is about to run another iteration, also take kOpIterBegin's
// resets here (per-partition counters, the active-contact counter
// *iter_reset, exec_newton), so the iteration's body and contact terms can
// run side by side as independent graph branches.
__device__ __forceinline__ void scalar_block(PartState* ps, int P, int op, FrameCtrl* ctrl,
                                             CondHandles hd, double tol, int max_iters, int* err,
                                             int* iter_reset = nullptr) {
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
            s.pcg_total = 0;
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
    if (iter_reset && any_act && (op == kOpReset || op == kOpNewtonTail)) {
        if (p < P) {
            PartState& s = ps[p];
            s.dq_inf = 0.0;
            s.toi_earliest = 2.0;
            s.n_candidates = 0;
            s.n_active_contacts = 0;
        }
        if (threadIdx.x == 0) {
            *iter_reset = 0;
            if (ctrl) ++ctrl->exec_newton;
        }
    }
    if (threadIdx.x == 0) {
        if (ctrl) {
            ctrl->any_active = any_act;
            ctrl->any_searching = any_srch;
            if (op == kOpIterBegin) ++ctrl->exec_newton;
            if (op == kOpAlphaMax) ++ctrl->exec_step;
            if (op == kOpAccept) ++ctrl->exec_ls;
        }
        if (op == kOpReset || op == kOpNewtonTail) set_cond(hd.newton, any_act, hd.graph);
        if (op == kOpNewtonCheck && hd.has_step) set_cond(hd.step, any_act, hd.graph);
        if (op == kOpAlphaMax || op == kOpAccept) set_cond(hd.ls, any_srch, hd.graph);
    }
}

} // namespace dabd_gpu
