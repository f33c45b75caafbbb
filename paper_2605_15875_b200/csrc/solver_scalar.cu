// Per-partition scalar control of the batched Newton solve and the N=1 ADMM
// frame controller. In graph mode these kernels also steer the conditional
// WHILE nodes (cudaGraphSetConditional), so a whole frame runs without a
// host round trip.
#include "kernels.hpp"

#include "instrument.hpp"
#include "scalar_ops.cuh"

namespace dabd_gpu {

namespace {

__global__ void k_scalar(PartState* ps, int P, int op, FrameCtrl* ctrl, CondHandles hd,
                         double tol, int max_iters, int* err, int* iter_reset) {
    scalar_block(ps, P, op, ctrl, hd, tol, max_iters, err, iter_reset);
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

void set_scalar_carveout(int pct) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(k_scalar), cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(k_frame_ctrl), cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();
}

void launch_scalar(PartState* ps, int P, int op, FrameCtrl* ctrl, CondHandles h, double tol,
                   int max_iters, int* err, cudaStream_t s, int* iter_reset) {
    DABD_LAUNCH("k_scalar", s,
                k_scalar<<<1, 32, 0, s>>>(ps, P, op, ctrl, h, tol, max_iters, err, iter_reset));
}

void launch_frame_ctrl(FrameCtrl* ctrl, int op, const double* dq_part, int P, double h, double l,
                       double theta, int K, double* trace, int trace_cap, CondHandles hd, int* err,
                       const PartState* ps, cudaStream_t s) {
    DABD_LAUNCH("k_frame_ctrl", s,
                k_frame_ctrl<<<1, 32, 0, s>>>(ctrl, op, dq_part, P, h, l, theta, K, trace,
                                              trace_cap, hd, err, ps));
}

} // namespace dabd_gpu
