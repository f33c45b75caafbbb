// Batched local solve on one device: every partition this context owns runs
// its own projected Newton (proj/src/newton.cpp:7-71) on its instance set,
// with its own line search and convergence, inside the same kernels.
//
// Arrays are sorted by (partition, body) so every per-partition quantity is
// a contiguous segment; reductions are fixed-order two-level segment sums,
// so results are bitwise reproducible run to run.
#pragma once

#include "common.cuh"
#include "device_scene.hpp"

namespace dabd_gpu {

constexpr int kEll = 24;   // initial off-diagonal 6x6 blocks per BSR row (SolverView::ell_w grows on kErrEll)
constexpr int kMaxParts = 32;

struct PartState {
    double energy;     // objective at the current iterate
    double trial;      // objective at the current line-search trial
    double alpha;      // current step
    double alpha_max;  // CCD bound (newton.cpp:38-42)
    double dq_inf;     // ||dq||_inf of the current direction
    double tol;        // Newton tolerance theta*h*l
    double eps;        // 1e-8 tr(H)/n (newton.cpp:20-22)
    double trace;
    double final_update;
    double toi_earliest; // CCD min over candidates (2.0 = none)
    double rz, rr, bnorm2, pap;
    int ndof;
    int active;        // Newton still iterating
    int searching;     // line search in progress
    int accepted;      // trial accepted in the last line-search round
    int converged;
    int iterations;
    int ls_steps;
    int pcg_done;
    int pcg_iters;
    int n_active_contacts;
    int n_candidates;
    int pcg_total;     // PCG iterations summed over this Newton solve (balancer cost)
};

// Device-side launch accounting of the PCG kernel (bench.py roofline): the
// launch duration from %globaltimer (first CTA in, last CTA out of the first
// cluster) and the algorithmic bytes of SURVEY.md 8(d):
// I_pcg * [288 * (N_b + 2 E_o) + 504 * N_b] per partition.
struct DevPerf {
    unsigned long long ns;
    unsigned long long launches;
    double bytes;
    unsigned long long iters;
    // clock64 cycles of CTA 0 / warp 0 per PCG phase, summed over iterations
    // (see k_pcg_cluster; dabd_gpu_ctx_pcg_phases); [8] setup, [9] epilogue,
    // [10..15] setup sub-phases: staging issue + first cluster barrier,
    // exchange plan, staging wait, plan barrier, eps + factor, init
    // [16..19] init sub-phases: eps + send plan, warm start, u = Dinv r +
    // barrier, initial SpMV + m
    unsigned long long phase[24];
};

struct SolverView {
    DevPerf* perf = nullptr;
    int pcg_phases = 0; // per-phase clock64 accounting in k_pcg_cluster (DABD_GPU_PCG_PHASES=1)
    SceneView sc;
    int n_inst = 0, n_rows = 0, n_parts = 0, part_base = 0;
    // instances
    const int* ibody = nullptr;
    const int* ipart = nullptr;
    const int* irow = nullptr;
    double* iq = nullptr;     // current iterate [I][6]
    double* iq_try = nullptr; // trial / end configuration [I][6]
    const double* iqt = nullptr;  // q_tilde
    const double* iinvk = nullptr; // 1/kappa_b
    const int* ianc = nullptr;     // anchored (shared) flag
    const double* iz = nullptr;
    const double* iu = nullptr;
    const double* irho = nullptr;
    // body holder masks (single_domain -> kappa_c = 1)
    const uint32_t* bmask = nullptr;
    int single_domain = 1;
    // rows (dynamic instances)
    const int* rinst = nullptr;
    const int* rpart = nullptr;
    double* rgrad = nullptr;  // [R][6]
    double* rdiag = nullptr;  // [R][36]
    double* rdinv = nullptr;  // [R][36]
    double* rval = nullptr;   // [R]
    int* ell_cnt = nullptr;   // [R]
    int* ell_col = nullptr;   // [R][ell_w]
    double* ell_blk = nullptr; // [R][ell_w][36]
    int ell_w = kEll;          // ELL width: coupling blocks a row can hold
    double* x = nullptr;      // dq [R][6]
    double* r = nullptr;
    double* z = nullptr;
    double* p0 = nullptr;
    double* p1 = nullptr;
    double* ap = nullptr;
    // partition offsets
    const int* part_row_off = nullptr;  // [P+1]
    const int* part_inst_off = nullptr; // [P+1]
    PartState* ps = nullptr;
    // params
    double h = 0.01, d_hat = 0.01, kappa_bar = 1e4, kappa_arap = 1e6;
    int project = 1; // PSD-project body and contact blocks (objective.cpp:366, 381)
    int* err = nullptr;
};

// Skin list ("Verlet list") of the local solve: the candidate superset
// built at a reference configuration qref, every instance i carrying its own
// skin s_i (body box grown by d_hat + s_i, point-edge tests by
// d_hat + s_P + s_E). While every vertex of instance i stays within s_i of
// its qref position (infinity norm) at the configurations a Newton iteration
// touches (q and the CCD end q + dq; the trials lie between), every
// candidate of the reference predicate at those configurations (static
// margin d_hat, swept margin 0) is in the list; each use re-applies the
// exact predicate, so detection results equal a fresh broad phase while the
// list is rebuilt only when a body leaves its skin (k_list_check decides on
// the device, a conditional graph node rebuilds).
struct ListState {
    int valid;        // 0: rebuild at the next check
    int rebuild;      // decision of the last check
    int n_rebuilds;
    int n_act;        // active contacts of the current derivative pass
    int invalid_acc;  // OR over the blocks of the running check
    unsigned ticket;
};

// Contacts of the current derivative pass, stored at their skin-list
// position t (list sorted by (a, b, v, e)); flag[t] marks the active ones.
struct ContactView {
    int n = 0;                    // list capacity (grid size)
    const int* dn = nullptr;      // device-side list length
    KeyFmt fmt;
    const unsigned long long* key = nullptr; // list keys, sorted by (a, b, v, e)
    const int* perm_b = nullptr;  // list positions sorted by (b, a, v, e)
    const int* aoff = nullptr;    // [I+1] positions with a == i: [aoff[i], aoff[i+1])
    const int* boff = nullptr;    // [I+1] perm_b positions with b == i
    unsigned char* flag = nullptr; // [cap] active at the current iterate
    int* act = nullptr;           // [cap] active positions (any order)
    ListState* ls = nullptr;      // ls->n_act = number of entries in act
    double* cval = nullptr;       // [cap] weighted barrier value (0 when inactive)
    double* cgrad = nullptr;      // [cap][12] weighted gradient
    // [cap][108] DoF-space blocks of the projected contact Hessian, row-major
    // 6x6 each: TL (point body x point body), BR (edge body x edge body), TR
    // (point body rows x edge body cols); BL = TR^T
    double* cblk = nullptr;
};

} // namespace dabd_gpu
