// Host launch wrappers of the solver/ADMM kernels (solver.cu, pcg.cu, solver_scalar.cu).
//
// Kernels that walk a candidate/contact list take its capacity `n` (grid
// size, host) and an optional device-side count `dn`: entries in [*dn, n)
// are padding. That keeps every launch free of host reads, so the whole
// frame can be captured into one CUDA graph.
#pragma once

#include "geometry.cuh"
#include "solver.hpp"

namespace dabd_gpu {

// which: 0 = partitions with an active Newton, 1 = partitions in a line
// search, 2 = every partition.
struct FrameCtrl;
void launch_body_terms(const SolverView& sv, const double* q, bool derivs, int which,
                       cudaStream_t s, int* reset_counter = nullptr, FrameCtrl* iter_begin = nullptr);
void launch_filter(const SolverView& sv, const unsigned long long* keys, int n, const int* dn,
                   KeyFmt fmt, const Box* box, const double* q, int mode, int which,
                   unsigned char* flag, double* val, cudaStream_t s);
void launch_contact_terms(const SolverView& sv, const ContactView& cv, cudaStream_t s);
void launch_contact_select(const SolverView& sv, const ContactView& cv, const Box* box,
                           cudaStream_t s, bool terms = false);
void launch_list_check(const SceneView& sc, const InstView& iv, const double* qref,
                       const double* qt, const double* skin, double* skin_next, double s_min,
                       double grow, ListState* ls, unsigned long long cond, int graph,
                       cudaStream_t s);
void launch_list_commit(int n, const double* iq, double* qref, const double* skin_next,
                        double* skin, cudaStream_t s);
void launch_seg_offsets(const unsigned long long* keys, int n, const int* dn, KeyFmt fmt,
                        int n_inst, int* off, int field, const int* perm, cudaStream_t s);
void launch_make_bkeys(const unsigned long long* keys, int n, const int* dn, KeyFmt fmt,
                       unsigned long long* bkeys, int* idx, cudaStream_t s);
void launch_assemble(const SolverView& sv, const ContactView& cv, double* row_trace,
                     cudaStream_t s);
void launch_precond(const SolverView& sv, cudaStream_t s);
int segsum_chunks(int n);
int energy_chunks(int n); // k_energy blocks for n entries
void launch_segsum_rows(const double* v, int n, const int* rpart, int P, int part_base,
                        double* partial, double* dst, int stride, bool accumulate, cudaStream_t s);
void launch_segsum_keys(const double* v, int n, const int* dn, const unsigned long long* keys,
                        KeyFmt fmt, const int* ipart, int P, int part_base, double* partial,
                        double* dst, int stride, bool accumulate, cudaStream_t s);
void launch_make_trial(const SolverView& sv, bool use_alpha, double alpha, int which,
                       cudaStream_t s);
void launch_dq_inf(const SolverView& sv, cudaStream_t s);
struct CondHandles;
// alpha_max_ctrl != nullptr: the last block also takes kOpAlphaMax (steering hd->ls).
void launch_ccd(const SolverView& sv, const unsigned long long* keys, int n, const int* dn,
                KeyFmt fmt, const Box* box0, const double* q0, const double* q1, int which,
                double* earliest_override, cudaStream_t s, FrameCtrl* alpha_max_ctrl = nullptr,
                const CondHandles* hd = nullptr);
// k_make_trial(alpha 1) + k_list_check + swept k_inst_boxes (margin 0) in one launch.
void launch_toi_reset(PartState* ps, int P, FrameCtrl* ctrl, cudaStream_t s);
void launch_ccd_prep(const SolverView& sv, const double* qref, const double* skin, double* skin_next,
                     double s_min, double grow, ListState* ls, unsigned long long cond, int graph,
                     Box* box, cudaStream_t s);

// Persistent cooperative block-Jacobi PCG over all partitions (pcg.cu).
// pbuf: 12 * n_rows doubles; partials: 3 * pcg_grid_size(n_rows) * P doubles.
int pcg_grid_size(int n_rows);
// Cluster-resident variant: one thread-block cluster (<= 16 CTAs) per partition,
// used while every partition has at most kClusterPcgMaxRows rows.
constexpr int kClusterPcgMaxRows = 4096;
int pcg_cluster_size();
// preferred shared-memory carveout (percent) of the Newton-loop kernels
void set_solver_carveout(int pct);
void set_scalar_carveout(int pct);
struct PcgFuse;
// fuse != nullptr: the fused Newton head (trace/eps/Dinv before, ||dq||_inf and
// the kOpNewtonCheck decision after; see PcgArgs in pcg.cu).
void launch_pcg_cluster(const SolverView& sv, int max_rows_per_part, double* pbuf, double tol,
                        int max_iters, cudaStream_t s, const PcgFuse* fuse = nullptr);
void launch_pcg_persistent(const SolverView& sv, double* pbuf, double* partials, double* rowval,
                           double tol, int max_iters, cudaStream_t s);
// Grid-wide pipelined PCG (one grid barrier per iteration) for partitions
// beyond the cluster kernel: vecs [10][6 n_rows], partials [2][blocks][P][4].
int pcg_grid_blocks();
void launch_pcg_grid(const SolverView& sv, double* vecs, double* partials, double tol, int max_iters,
                     cudaStream_t s, double eta_loose = 0.0, double eta_factor = 0.0);

// Per-partition scalar steps (solver_scalar.cu). `op` selects the update.
enum ScalarOp : int {
    kOpEps = 3,         // eps = 1e-8 * trace / ndof; ++iterations
    kOpAlphaMax = 4,    // alpha_max from toi_earliest; alpha = alpha_max; searching = 1
    kOpAccept = 5,      // line-search decision (newton.cpp:47-62)
    kOpNewtonCheck = 6, // dq_inf < tol -> converged without moving (newton.cpp:30-36)
    kOpIterBegin = 7,   // dq_inf = 0, toi_earliest = 2, n_candidates = 0
    kOpReset = 8,       // start of a solve: active = ndof > 0 (unless ctrl says ended)
    kOpNewtonTail = 9   // end of a Newton iteration: cap at max_iters
};

// Device-side frame control for the captured graph (run_reference semantics,
// sim.cpp:207-247). Conditional handles steer the WHILE nodes; in eager mode
// they are 0 and the host reads the same flags.
struct FrameCtrl {
    int k;               // ADMM iteration counter of the frame
    int ended;           // stop decision taken
    int failed;          // K exhausted without a stop
    int admm_iterations;
    int newton_total, ls_total, pcg_total, max_contacts, max_candidates;
    int any_active, any_searching;
    int trace_n;
    int exec_admm, exec_newton, exec_step, exec_ls; // conditional-body executions
    // multi-partition ADMM frame on the device (k_admm_ctrl): sigma of the
    // last decision (0 running, 1 end, 2 retry with h/2, 3 halving budget
    // spent, -1 device error), whether h may still halve (host-written),
    // executions of the merge-gate and local-solve bodies, and the largest
    // merge-gate candidate count of the attempt (capacity feedback)
    int sigma, can_halve, exec_gate, exec_solve, gate_max;
    double dq_inf;       // max over partitions of the last solve's config delta
    double frame;        // frame index for trace rows (written by the host)
    double attempt;      // attempt index for trace rows (written by the host)
};

struct CondHandles {
    unsigned long long admm = 0, newton = 0, step = 0, ls = 0; // cudaGraphConditionalHandle values
    unsigned long long gate = 0, solve = 0; // multi-partition ADMM frame: IF(k > 1), IF(continue)
    int graph = 0;
    int has_step = 0; // an IF(step) node exists for `step` (not in the flat fused Newton body)
};

struct PcgFuse {
    const double* row_trace; // [n_rows] trace of each assembled diagonal block (k_assemble)
    FrameCtrl* ctrl;
    CondHandles hd;          // hd.step is set from the convergence decision
    double eta_loose = 0.0;  // inexact Newton: loose relative residual (0: off)
    double eta_factor = 0.0; // ... allowed while rms(x) > eta_factor x Newton tol
    bool close_loop = false; // folded Newton tail: end the Newton WHILE when no partition stays active
};

// Fused objective value (solver.cu k_energy): qmode 0 = iq, 1 = line-search
// trial of searching partitions; result into dst (PartState field, stride in
// doubles); accept = also take kOpAccept. partial: energy_chunks(n_rows) +
// energy_chunks(cap) blocks x P doubles.
void launch_energy(const SolverView& sv, const unsigned long long* keys, int cap, const int* dn,
                   KeyFmt fmt, int qmode, int which, double* partial, double* dst, int stride,
                   bool accept, FrameCtrl* ctrl, CondHandles hd, cudaStream_t s, bool apply = false,
                   int tail_max_iters = 0, int* iter_reset = nullptr);
void launch_accept_trial(const SolverView& sv, cudaStream_t s);

void launch_scalar(PartState* ps, int P, int op, FrameCtrl* ctrl, CondHandles h, double tol,
                   int max_iters, int* err, cudaStream_t s, int* iter_reset = nullptr);

// ADMM controller of the N=1 frame (sim.cpp:223-238): op 0 = step head
// (stop test for k > 1), op 1 = step tail (k++, K bound). Writes trace rows.
void launch_frame_ctrl(FrameCtrl* ctrl, int op, const double* dq_part, int P, double h, double l,
                       double theta, int K, double* trace, int trace_cap, CondHandles hd, int* err,
                       const PartState* ps, cudaStream_t s);

} // namespace dabd_gpu
