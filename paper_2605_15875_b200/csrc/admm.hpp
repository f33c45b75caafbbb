// Launchers of the frame-level / consensus-ADMM kernels (admm.cu).
#pragma once

#include "kernels.hpp"
#include "scene.hpp"

namespace dabd_gpu {

void launch_gather(int n, const int* ibody, const double* q, double* iq, cudaStream_t s);
// x[6 n_rows], p2[6 n_rows] from prev = (x_old, p2_old) through map (-1: zero).
void launch_warm_remap(int n_rows, const int* map, const double* prev, int r_old, double* x,
                       double* p2, cudaStream_t s);
void launch_predict(const SceneView& sc, int n, const int* ibody, const double* iq,
                    const double* qd, double h, double gx, double gy, const double* ifs,
                    double* iqt, cudaStream_t s);
void launch_delta_inf(int n_rows, const int* rinst, const int* rpart, int part_base,
                      const double* a, const double* b, double* out, cudaStream_t s);
void launch_masks(const SceneView& sc, const double* q, const double* planes, int np, double w,
                  uint32_t all, uint32_t* masks, int* err, cudaStream_t s);
void launch_vmax(const SceneView& sc, const double* qd, double* out, cudaStream_t s);
// Halo packet of one replica: q[6], u[6], rho.
constexpr int kHaloStride = 13;

void launch_consensus(int ns, const int* sh, const int* ipart, int part_base, const double* iq,
                      double* iu, const double* irho, const double* iz, const double* remote_lo,
                      const double* remote_hi, int n_lo, double* iznext, double* rb, double* sb,
                      double* rloc, double* sloc, int* err, cudaStream_t s);
void launch_pack_halo(int n, const int* inst, const double* iq, const double* iu,
                      const double* irho, double* out, cudaStream_t s);
void launch_select_commit(const SceneView& sc, const uint32_t* bmask, const int* part_rank,
                          const double* gath, size_t stride, double* q, double* qd,
                          cudaStream_t s);
// Owned-body commit records (runtime.cpp:484-506 across ranks): bodies whose
// lowest holder partition lies in [p0, p1) -> (id, q[6], qdot[6]); and the
// inverse over every rank's records.
void launch_pack_owned(const SceneView& sc, const uint32_t* bmask, int p0, int p1, const double* q,
                       const double* qd, double* rec, int* count, cudaStream_t s);
void launch_unpack_owned(int world, const int* counts, const double* gath, size_t stride, double* q,
                         double* qd, cudaStream_t s);
void launch_merged(int n, const int* ianc, const double* iq, const double* iznext, double* out,
                   cudaStream_t s);
void launch_adapt(int n, const int* ianc, double* irho, const double* irho0, const double* rb,
                  const double* sb, const AdaptParams& a, double* iz, const double* iznext,
                  cudaStream_t s, const FrameCtrl* skip_first = nullptr);
void launch_commit(const SceneView& sc, int n, const int* ibody, const int* ipart, const int* ianc,
                   const uint32_t* bmask, double* iq, const double* iznext, const double* q_start,
                   double h, double* q, double* qd, cudaStream_t s);
void launch_accept_copy(int n, const int* ipart, int part_base, const PartState* ps,
                        const double* src, double* dst, cudaStream_t s);

// Device-side instance sets (runtime.cpp:126-236): flags of every
// (partition, body) pair in partition-major order t = p * nb + b: in the
// partition, dynamic in it, a replica past the body's lowest holder (a
// shared-pair second). w: when vmax is given, the overlap width
// max(2 v_max h, w_min) (runtime.cpp:556-560) is formed on the device.
void launch_inst_flags(const SceneView& sc, const uint32_t* masks, int P, int p0, int* f_all, int* f_dyn,
                       int* f_sh, cudaStream_t s);
// counts: [0] instances, [1] rows, [2] shared pairs, [3, 3 + P] instance
// offsets per partition, [4 + P, 5 + 2P] row offsets
void launch_inst_counts(int P, int nb, const int* f_all, const int* f_dyn, const int* f_sh, const int* s_all,
                        const int* s_dyn, const int* s_sh, int* counts, cudaStream_t s);
struct InstOut {
    int *ibody, *ipart, *irow, *rinst, *rpart, *stat, *ianc, *shared, *wmap, *rowtab, *pio, *pro;
    double *invk, *rho, *rho0;
};
void launch_inst_scatter(const SceneView& sc, const uint32_t* masks, int P, int p0, const int* f_all,
                         const int* f_dyn, const int* f_sh, const int* s_all, const int* s_dyn,
                         const int* s_sh, double beta, const double* rho_carry, const int* rowtab_prev,
                         InstOut o, cudaStream_t s);
// rho carry (runtime.cpp:481-482): NaN everywhere, then each replica's rho
void launch_rho_carry(int n_inst, int nb, const int* ibody, const int* ianc, const double* irho,
                      double* carry, cudaStream_t s);
void launch_masks_w(const SceneView& sc, const double* q, const double* planes, int np, const double* vmax,
                    double h, double w_min, double* w_out, uint32_t all, uint32_t* masks, int* err,
                    cudaStream_t s);

// Device fan-in across ranks (admm.cu k_fan_*): records [world][rec_stride]
// and flags [world] in every rank's buffer, peers' buffers mapped by IPC.
struct FanView {
    int rank = 0, world = 1, rec_stride = 0;
    double* peer_rec[32] = {};              // slot array of every rank's buffer (own included)
    unsigned long long* peer_flag[32] = {}; // flags of every rank's buffer
    const unsigned long long* local_flag = nullptr;
    const double* local_rec = nullptr;
    unsigned long long* seq = nullptr; // local round counter (device)
};
void launch_fan_post(const FanView& f, const double* rec, int rec_len, cudaStream_t s);
void launch_fan_wait(const FanView& f, cudaStream_t s);
void launch_fan_record(int P, const double* dq, const double* rloc, const double* sloc, const double* gate,
                       const int* err, double* rec, cudaStream_t s);
void launch_pack_halo_par(int n, const int* inst, const double* iq, const double* iu, const double* irho,
                          double* pub, const FrameCtrl* pc, int side, size_t reg, cudaStream_t s);
void launch_consensus_par(int ns, const int* sh, const int* ipart, int part_base, const double* iq, double* iu,
                          const double* irho, const double* iz, const double* peer_lo, const double* peer_hi,
                          int n_lo, double* iznext, double* rb, double* sb, double* rloc, double* sloc, int* err,
                          const FrameCtrl* pc, size_t reg, cudaStream_t s);

// Device controller of the multi-partition consensus-ADMM frame
// (runtime.cpp:316-476 and the controller round trip 572-638 for the
// partitions of one context). ops: kAdmmInit, kAdmmHead (IF(gate) = k > 1;
// gate TOIs <- 2, r/s partials <- 0), kAdmmDecide (stop test of
// consensus.cpp:54-64 over every partition's dq, r, s and merge-gate TOI,
// trace row, sigma; IF(solve), WHILE), kAdmmTail (collect the local solve:
// dq, Newton totals, partition costs; k++).
enum AdmmCtrlOp { kAdmmInit = 0, kAdmmHead = 1, kAdmmDecide = 2, kAdmmTail = 3 };
struct AdmmCtrlArgs {
    FrameCtrl* c = nullptr;
    double* gate = nullptr;      // [P] earliest merge-gate TOI (2.0 = none)
    double* rloc = nullptr;      // [P] primal residual
    double* sloc = nullptr;      // [P] dual residual
    double* dq = nullptr;        // [P] last local solve's ||q - q_before||_inf
    const double* dq_new = nullptr; // [P] delta_inf output of the solve just done
    double* cost = nullptr;      // [P] balancer cost of the attempt
    const PartState* ps = nullptr;
    const int* gate_count = nullptr; // merge-gate candidate count (device)
    int* err = nullptr;
    double* trace = nullptr;
    int trace_cap = 0;
    int P = 0, K = 0;
    double h = 0.0, l = 0.0, theta = 0.0;
    CondHandles hd;
    // partition-per-GPU runs: every rank's fan-in record [world][stride]
    // (n_parts, fail, then dq, r, s, earliest TOI per partition) decides
    const double* fan_rec = nullptr;
    int fan_world = 0, fan_stride = 0;
};
void launch_admm_ctrl(const AdmmCtrlArgs& a, int op, cudaStream_t s);

} // namespace dabd_gpu
