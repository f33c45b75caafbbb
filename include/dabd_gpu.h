/* dabd_gpu: B200-native (sm_100a) distributed ADMM affine-body dynamics.
 *
 * C ABI of the hot path of arxiv/paper_2605_15875 (`dabd`). It keeps the
 * conventions of the reference's C API (proj/include/dabd.h:25-70,
 * proj/src/capi.cpp:16-34): status codes, opaque handles freed by the caller,
 * a thread-local last-error string, no exceptions across the ABI, null
 * arguments -> INVALID, blocking calls. Plain pointers and sizes only.
 *
 * Every array is FP64/int32 and host-resident unless stated otherwise.
 * Configurations are [n_bodies][6] row-major q = [p_x, p_y, A00, A01, A10,
 * A11] (proj/include/dabd/types.hpp:18). Contact pairs are int32[4] =
 * (body_a, body_b, point_index, edge_index), lexicographically sorted like
 * ContactPair::operator< (proj/include/dabd/geometry.hpp:31-36).
 *
 * Replaced reference interfaces (file:line relative to /root/reference/proj):
 *   dabd_gpu_scene_create        make_affine_body / SceneData   src/body.cpp:96-118, include/dabd/scene.hpp:15-56
 *   dabd_gpu_broad_phase         broad_phase / broad_phase_swept include/dabd/geometry.hpp:47-58
 *   dabd_gpu_narrow_phase        narrow_phase                    include/dabd/geometry.hpp:61-63
 *   dabd_gpu_ccd_toi             ccd_toi_scene                   include/dabd/geometry.hpp:72-74
 *   dabd_gpu_holder_masks        body_holder_mask                include/dabd/partition.hpp:43-45
 *   dabd_gpu_objective           LocalObjective::value/derivatives include/dabd/objective.hpp:34-75
 *   dabd_gpu_newton_solve        newton_solve                    include/dabd/newton.hpp:25-26
 *   dabd_gpu_consensus_step      consensus_update, dual_update, *_residual_inf, adapt_rho
 *                                                                include/dabd/consensus.hpp:13-55
 *   dabd_gpu_check_stopping      check_stopping                  src/consensus.cpp:54-64
 *   dabd_gpu_timestep_apply      TimestepController              include/dabd/consensus.hpp:60-87
 *   dabd_gpu_contact3d_terms     3D extension of contact_energy  src/energy.cpp:63-94 (PT / EE, no reference)
 *   dabd_gpu_ccd3d               3D extension of ccd_toi          src/geometry.cpp:232-341 (no reference)
 *   dabd_gpu_broad_phase3d       3D extension of broad_phase      src/geometry.cpp:106-208 (no reference)
 *   dabd_gpu_sim3d_*             3D extension of run_reference    src/sim.cpp:186-249 + newton.cpp:7-71 (no reference)
 *   dabd_gpu_balancer_*          Balancer, imbalance_metric, pd_update, balance_factor
 *                                                                include/dabd/balance.hpp:9-56
 *   dabd_gpu_run_frames          run_reference (workers==0)      src/sim.cpp:186-249
 *                                WorkerSession/ControllerSession frame loop  src/runtime.cpp:110-694
 */
#ifndef DABD_GPU_H
#define DABD_GPU_H

#include <stddef.h>
#include <stdint.h>

#if defined(_WIN32)
#define DABD_GPU_API __declspec(dllexport)
#else
#define DABD_GPU_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dabd_gpu_status {
    DABD_GPU_OK = 0,
    DABD_GPU_ERR_IO = 1,
    DABD_GPU_ERR_PARSE = 2,
    DABD_GPU_ERR_INVALID = 3, /* bad arguments, too-small output capacity */
    DABD_GPU_ERR_RUNTIME = 4, /* CUDA/NCCL failure or a solver error the reference throws */
} dabd_gpu_status;

/* SimParams (include/dabd/params.hpp:8-15), same field order. */
typedef struct dabd_gpu_sim_params {
    double h;
    double gravity_x, gravity_y;
    double arap_stiffness;
    double barrier_stiffness;
    double d_hat;
    double theta;
    double scene_scale;
} dabd_gpu_sim_params;

/* AdaptParams (include/dabd/params.hpp:26-32). */
typedef struct dabd_gpu_adapt_params {
    double beta, tau, mu, sigma_min, sigma_max;
    int adapt_enabled;
} dabd_gpu_adapt_params;

/* Remaining SceneData knobs (include/dabd/scene.hpp:21-36). */
typedef struct dabd_gpu_run_params {
    double w_min;
    int admm_max_iterations; /* K */
    int newton_cap;
    int max_halvings;
    int force_split_frames;
} dabd_gpu_run_params;

/* Linear-solver knobs of the B200 local solve (block-Jacobi PCG replaces
 * SimplicialLDLT, src/newton.cpp:25). */
typedef struct dabd_gpu_solver_params {
    double pcg_rel_tol; /* ||r||_2 <= tol * ||b||_2 */
    int pcg_max_iters;
} dabd_gpu_solver_params;

typedef struct dabd_gpu_frame_stats {
    int committed;        /* 1 when the frame committed */
    int attempts;         /* 1 + AbortRetry halvings */
    double h;             /* step actually used */
    int admm_iterations;  /* k at End (>= 2) */
    int newton_iterations;/* summed over partitions and solves */
    int line_search_steps;
    int pcg_iterations;
    int max_contacts;     /* largest active set seen */
    int max_candidates;
    int exact_retries;    /* Newton solves redone at the exact-solve PCG limit after a
                             line-search collapse (newton.cpp:56-58); 0 on a clean frame */
    int capacity_retries; /* work redone after a capacity grew (candidate list, BSR row width) */
    /* Host wall-clock seconds, as the reference's worker timers
     * (runtime.cpp:117-124, 399-402, 466-475; sim.hpp:44-47): local Newton
     * solves, collision work of the consensus step (merge gate), waiting on
     * peer ranks, and the whole frame (t_compute = t_frame - t_sync). For a
     * run_reference context t_solve = t_frame. */
    double t_solve, t_coll, t_sync, t_frame;
} dabd_gpu_frame_stats;

/* Inter-GPU exchange of a partition-per-GPU run; replaces
 * the reference's Transport (include/dabd/transport.hpp:15-40) on the data
 * path. Rank r owns partitions [part_offsets[r], part_offsets[r+1]) and
 * creates its context with exactly that range. All pointers handed to the
 * callbacks are DEVICE pointers on `stream` (a cudaStream_t); a callback
 * returns 0 on success and must leave the results ordered before later work
 * on `stream` (e.g. NCCL on that stream).
 *   halo: send n_lo doubles from send_lo to rank-1 and receive n_lo from it
 *         into recv_lo; likewise n_hi with rank+1. Both sides always agree on
 *         the counts (they derive them from the same replicated holder masks);
 *         a zero count means no transfer on that side.
 *   allgather: every rank contributes `count` doubles; recv holds
 *         world * count doubles in rank order. */
typedef struct dabd_gpu_comm {
    void* user;
    int (*halo)(void* user, const double* send_lo, double* recv_lo, size_t n_lo,
                const double* send_hi, double* recv_hi, size_t n_hi, uintptr_t stream);
    int (*allgather)(void* user, const double* send, double* recv, size_t count,
                     uintptr_t stream);
    int rank;
    int world;
    const int* part_offsets; /* world + 1 entries, copied */
} dabd_gpu_comm;

/* Balancer::Options + SceneData::balance_enabled (include/dabd/balance.hpp:24-29,
 * scene.hpp:31-32). dp_max <= 0: w/2 per frame. */
typedef struct dabd_gpu_balance_params {
    int enabled;
    double kp, kd, smoothing, dp_max;
} dabd_gpu_balance_params;

typedef struct dabd_gpu_scene dabd_gpu_scene;
typedef struct dabd_gpu_balancer dabd_gpu_balancer;
typedef struct dabd_gpu_ctx dabd_gpu_ctx;

DABD_GPU_API const char* dabd_gpu_version(void);
DABD_GPU_API const char* dabd_gpu_last_error(void);

/* ---- scene -------------------------------------------------------------
 * Body b owns loops [body_loop_start[b], body_loop_start[b+1]); loop l owns
 * world-space vertices [loop_vert_start[l], loop_vert_start[l+1]) of
 * verts_xy. qdot is [n_bodies][6]. */
DABD_GPU_API dabd_gpu_status dabd_gpu_scene_create(int n_bodies, const int* body_loop_start,
                                                   const int* loop_vert_start,
                                                   const double* verts_xy, const double* density,
                                                   const int* is_static, const double* arap_scale,
                                                   const double* qdot, dabd_gpu_scene** out);
DABD_GPU_API void dabd_gpu_scene_free(dabd_gpu_scene* scene);
DABD_GPU_API dabd_gpu_status dabd_gpu_scene_set_params(dabd_gpu_scene* scene,
                                                       const dabd_gpu_sim_params* sim,
                                                       const dabd_gpu_adapt_params* adapt,
                                                       const dabd_gpu_run_params* run);
/* planes: n_planes x (point_x, point_y, normal_x, normal_y). */
DABD_GPU_API dabd_gpu_status dabd_gpu_scene_set_planes(dabd_gpu_scene* scene, int n_planes,
                                                       const double* planes);
DABD_GPU_API dabd_gpu_status dabd_gpu_scene_set_force_split(dabd_gpu_scene* scene, int body,
                                                            double fx, double fy);
/* PD load balancing of the interface planes between frames (runtime.cpp:537-552):
 * each committed frame's per-partition compute costs drive Balancer::update,
 * whose shifted planes partition the next frame. */
DABD_GPU_API dabd_gpu_status dabd_gpu_scene_set_balance(dabd_gpu_scene* scene,
                                                        const dabd_gpu_balance_params* p);
DABD_GPU_API dabd_gpu_status dabd_gpu_scene_counts(const dabd_gpu_scene* scene, int* n_bodies,
                                                   int* n_verts);
/* rest_xy [n_verts][2], vert_start [n_bodies+1], q [n][6], mass [n], M [n][36]. */
DABD_GPU_API dabd_gpu_status dabd_gpu_scene_bodies(const dabd_gpu_scene* scene, double* rest_xy,
                                                   int* vert_start, double* q, double* mass,
                                                   double* mass_matrix);

/* ---- device context ------------------------------------------------------
 * A context owns all device memory for one GPU and the partitions
 * [part_begin, part_end) of a `num_workers`-way slab decomposition
 * (num_workers == 0 selects the single-domain run_reference semantics). */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_create(const dabd_gpu_scene* scene, int device,
                                                 int num_workers, int part_begin, int part_end,
                                                 dabd_gpu_ctx** out);
DABD_GPU_API void dabd_gpu_ctx_free(dabd_gpu_ctx* ctx);
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_set_solver(dabd_gpu_ctx* ctx,
                                                     const dabd_gpu_solver_params* p);
/* Inexact Newton inside frames (the cluster PCG of partitions up to 4096
 * rows): a Newton direction may stop at the relative residual `eta` (instead
 * of pcg_rel_tol) while its root-mean-square entry exceeds `factor` x the
 * Newton tolerance theta h l (so ||dq||_inf does too): a direction that can
 * decide convergence (newton.cpp:30-36) is always solved to pcg_rel_tol, and
 * a loose one ends a line search (newton.cpp:56-62) only on a step shortened
 * below 1 / factor. eta <= pcg_rel_tol (e.g. 0) turns it off. Default: 1e-3,
 * factor 1 for single-domain contexts (num_workers == 0), off for consensus
 * contexts (their stop test reads residuals of the local solutions);
 * dabd_gpu_newton_solve always solves every direction to pcg_rel_tol. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_set_inexact(dabd_gpu_ctx* ctx, double eta, double factor);
/* Stream (cudaStream_t as uintptr_t) the context launches on; 0 = own stream. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_set_stream(dabd_gpu_ctx* ctx, uintptr_t stream);
/* Join a partition-per-GPU run (comm == NULL leaves it). Required when the
 * context's partition range is not [0, num_workers). The callbacks are
 * called from the thread that calls dabd_gpu_run_frames. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_set_comm(dabd_gpu_ctx* ctx, const dabd_gpu_comm* comm);

/* Exchange path of a joined context: 0 single process, 1 halo callback,
 * 2 peer-memory halo (the neighbours' published packets mapped through CUDA
 * IPC and loaded by the consensus kernel; DABD_GPU_P2P_HALO=0 disables it),
 * 3 the same plus the device ADMM loop: every rank's controller fan-in record
 * and the ordering barriers through IPC-mapped peer slots and device flags,
 * the attempt one captured graph per rank (DABD_GPU_FANIN=0 disables it). */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_comm_mode(dabd_gpu_ctx* ctx, int* mode);

/* ---- parity entry points (identical-input comparisons with the oracle) ---
 * subset == NULL means all bodies. q_end == NULL: static broad phase. On
 * capacity overflow the call returns INVALID and writes the needed count. */
DABD_GPU_API dabd_gpu_status dabd_gpu_broad_phase(dabd_gpu_ctx* ctx, const double* q,
                                                  const double* q_end, double margin,
                                                  const int* subset, int n_subset, int* pairs,
                                                  int capacity, int* count);
DABD_GPU_API dabd_gpu_status dabd_gpu_narrow_phase(dabd_gpu_ctx* ctx, const double* q,
                                                   const int* candidates, int n_candidates,
                                                   double d_hat, int* out_pairs, double* out_d,
                                                   int* count);
DABD_GPU_API dabd_gpu_status dabd_gpu_ccd_toi(dabd_gpu_ctx* ctx, const double* q0,
                                              const double* q1, const int* subset, int n_subset,
                                              double* toi);
DABD_GPU_API dabd_gpu_status dabd_gpu_holder_masks(dabd_gpu_ctx* ctx, const double* q,
                                                   int n_planes, const double* planes, double w,
                                                   uint32_t* masks);

/* One consensus step for n split bodies with two replicas each (lower holder
 * first; the k_consensus / k_adapt kernels of the ADMM frame):
 * z = sum rho (q + u) / sum rho (consensus_update, consensus.cpp:9-21),
 * u' = (u + q) - z per replica (dual_update, :23-25), r = max |q - z| over
 * both replicas, s = max |z - z_prev| (:27-36), rho' = adapt_rho(rho, r, s,
 * rho0) (:44-52; rho' = rho when adapt->adapt_enabled == 0). q, u, u_new:
 * [n][2][6]; z_prev, z: [n][6]; rho, rho0, r, s, rho_next: [n]. */
DABD_GPU_API dabd_gpu_status dabd_gpu_consensus_step(int device, int n, const double* q,
                                                     const double* u, const double* rho,
                                                     const double* z_prev, const double* rho0,
                                                     const dabd_gpu_adapt_params* adapt, double* z,
                                                     double* u_new, double* r, double* s,
                                                     double* rho_next);

/* The controller's stop rule (consensus.cpp:54-64), the function the
 * multi-partition frame evaluates: *end = 1 iff dq / (h l), r / (h l) and
 * s / (h l) are all strictly below theta and every merge-gate toi is exactly
 * 1.0 (n_tois may be 0). */
DABD_GPU_API dabd_gpu_status dabd_gpu_check_stopping(double dq, double r, double s,
                                                     const double* tois, int n_tois, double h,
                                                     double l, double theta, int* end);
/* TimestepController (consensus.hpp:60-87) driven by a sequence of frame
 * outcomes: events[i] = 0 a failed frame (h /= 2; more than max_halvings
 * failures in a row is DABD_GPU_RUNTIME), 1 a committed frame
 * (h = min(h0, 2 h)). h_after[i] = h after event i. */
DABD_GPU_API dabd_gpu_status dabd_gpu_timestep_apply(double h0, int max_halvings, const int* events,
                                                     int n_events, double* h_after);

/* Penetration audit of a configuration: intersection_test
 * (proj/src/geometry.cpp:389-454; strict vertex / loop-centroid containment
 * and proper edge crossings over body pairs with overlapping AABBs) and the
 * minimum point-edge distance of proj/tests/support/oracles.cpp:153-173 over
 * ordered pairs a != b that are not both static. q == NULL audits the
 * context's current device state (no host copy). result = 1 iff some pair
 * interpenetrates; n_violations (nullable) counts those pairs. min_distance
 * (nullable) is computed when cutoff > 0 and is exact whenever it is below
 * the cutoff (DBL_MAX when no pair comes within reach). */
DABD_GPU_API dabd_gpu_status dabd_gpu_audit(dabd_gpu_ctx* ctx, const double* q, const int* subset,
                                            int n_subset, double cutoff, int* result,
                                            int* n_violations, double* min_distance);

/* LocalObjective over `local` bodies with per-local kappa and q_tilde and
 * optional anchors (body, z[6], u[6], rho). holder_mask (per body) may be
 * NULL for single-domain weights. mode 0: value; 1: value without anchors;
 * 2: value + gradient [n_dof] + dense PSD-projected Hessian [n_dof^2] (test
 * sizes only); 3: as 2 without projection. */
DABD_GPU_API dabd_gpu_status dabd_gpu_objective(dabd_gpu_ctx* ctx, int n_local, const int* local,
                                                const double* kappa, const double* q_tilde,
                                                int n_anchor, const int* anchor_body,
                                                const double* anchor_zu, const double* anchor_rho,
                                                const uint32_t* holder_mask,
                                                const dabd_gpu_sim_params* sim, const double* q,
                                                int mode, double* value, double* grad,
                                                double* hess_dense, int* active, int* candidates);
/* newton_solve (newton.cpp:7-71) on the device; q [n][6] updated in place. */
DABD_GPU_API dabd_gpu_status dabd_gpu_newton_solve(
    dabd_gpu_ctx* ctx, int n_local, const int* local, const double* kappa, const double* q_tilde,
    int n_anchor, const int* anchor_body, const double* anchor_zu, const double* anchor_rho,
    const uint32_t* holder_mask, const dabd_gpu_sim_params* sim, double* q, int max_iters,
    double tol, int* iterations, double* final_update_inf, int* converged, int* line_search_steps);

/* ---- stepping -------------------------------------------------------------
 * Advances the device-resident global state by n_frames committed frames
 * (run_reference semantics when the context was created with 0 workers,
 * the consensus-ADMM runtime semantics otherwise). stats: n_frames entries
 * or NULL. */
DABD_GPU_API dabd_gpu_status dabd_gpu_run_frames(dabd_gpu_ctx* ctx, int n_frames,
                                                 dabd_gpu_frame_stats* stats);
DABD_GPU_API dabd_gpu_status dabd_gpu_set_state(dabd_gpu_ctx* ctx, const double* q,
                                                const double* qdot);
DABD_GPU_API dabd_gpu_status dabd_gpu_get_state(dabd_gpu_ctx* ctx, double* q, double* qdot);
/* Final adapted rho per body (NaN where the body is not shared), after a frame. */
DABD_GPU_API dabd_gpu_status dabd_gpu_get_rho(dabd_gpu_ctx* ctx, double* rho);
/* Interface planes the next frame partitions with: (num_workers-1) x (px, py, nx, ny). */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_get_planes(dabd_gpu_ctx* ctx, double* planes);
/* Per-partition compute costs of the last committed frame (num_workers
 * entries; 0 before the first commit or with balancing off). The reference
 * feeds wall-clock worker times (runtime.cpp:674); batched partitions share
 * kernels, so the cost is the deterministic row-weighted work of the
 * partition's Newton + PCG iterations. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_partition_costs(dabd_gpu_ctx* ctx, double* costs);
/* ADMM trace rows since the last call: (frame, attempt, k, dq, r, s, min_toi,
 * sigma) doubles; returns the number of rows written (<= capacity). */
DABD_GPU_API dabd_gpu_status dabd_gpu_take_trace(dabd_gpu_ctx* ctx, double* rows, int capacity,
                                                 int* count);

/* ---- 3D affine-body contact terms ----------------------
 * The reference is 2D; this is its contact_energy (energy.cpp:63-94) for 3D
 * affine bodies (q = [p(3), A row-major(9)], x = A xbar + p) and the two 3D
 * primitive pairs: kind 0 point-triangle (rest: p of body a, t0 t1 t2 of body
 * b), kind 1 edge-edge (rest: a0 a1 of body a, b0 b1 of body b). Per pair k
 * (host arrays): qa/qb [n][12], rest [n][4][3] -> distance d [n], closest-
 * feature type [n] (PT: 0-2 vertex, 3-5 edge t0t1/t1t2/t2t0, 6 face; EE: 0-3
 * vertex pairs a0b0/a0b1/a1b0/a1b1, 4-5 a0/a1 vs edge b, 6-7 b0/b1 vs edge a,
 * 8 line-line), value = weight * b(d) with the log barrier of energy.cpp:50-61
 * (0 for d >= d_hat), grad [n][24] (body a then b) and, when hess != NULL,
 * hess [n][24][24] (the objective.cpp:12-17 clamp when project != 0).
 * Computed on `device`; RUNTIME when a pair has d <= 0. Parity unpinned: no
 * reference implements 3D (oracle/geometry3d.cpp restates it independently). */
DABD_GPU_API dabd_gpu_status dabd_gpu_contact3d_terms(int device, int n, const int* kind,
                                                      const double* qa, const double* qb,
                                                      const double* rest, double d_hat,
                                                      double kappa, double weight, int project,
                                                      double* d, int* dtype, double* value,
                                                      double* grad, double* hess);

/* CCD of the same 3D pairs while both bodies move linearly from (qa0, qb0) to
 * (qa1, qb1) (so every point moves linearly): additive CCD (conservative
 * advancement on the distance), toi [n] = 1.0 when the pair stays apart over
 * [0, 1], else a time at which it still keeps 10% of its starting gap; the
 * line-search bound is min(toi) like ccd_toi_scene (geometry.cpp:322-341).
 * 0.0 when a pair already touches. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ccd3d(int device, int n, const int* kind, const double* qa0,
                                            const double* qa1, const double* qb0,
                                            const double* qb1, const double* rest, double* toi);

/* Mass moments of a 3D affine body from a closed, outward-oriented triangle
 * surface (verts [n_verts][3], tris [n_tris][3]): moments10 = density * (V,
 * s_x, s_y, s_z, S_xx, S_xy, S_xz, S_yy, S_yz, S_zz) about the rest centroid
 * (s = 0 by construction), centroid [3] (the body's initial translation, as
 * make_affine_body re-centres, body.cpp:96-118), volume. Host only. */
DABD_GPU_API dabd_gpu_status dabd_gpu_body3d_moments(int n_verts, const double* verts, int n_tris,
                                                     const int* tris, double density,
                                                     double* moments10, double* centroid,
                                                     double* volume);
/* Body terms of n 12-DoF bodies (energy.cpp:7-48 in 3D): value = 1/2 (q -
 * qt)^T M (q - qt) + scale * w ||A^T A - I||_F^2 with M from moments10, w [n]
 * (kappa * volume * arap_scale), scale (h^2 in the objective); grad [n][12],
 * hess [n][12][12] (nullable; clamped like objective.cpp:143-167 when
 * project != 0). */
DABD_GPU_API dabd_gpu_status dabd_gpu_body3d_terms(int device, int n, const double* q,
                                                   const double* qt, const double* moments10,
                                                   const double* w, double scale, int project,
                                                   double* value, double* grad, double* hess);

/* 3D broad phase (geometry.cpp:106-208 in 3D): candidate pairs between n
 * bodies at q [n][12] (q_end [n][12] nullable: swept), each body a closed
 * triangle mesh in rest coordinates (vert_start [n+1] into verts [nv][3],
 * tri_start [n+1] into tris [nt][3], edge_start [n+1] into edges [ne][2],
 * local vertex indices). Body boxes inflated by margin, sweep on lo.x (ties by
 * id), 3D overlap; per overlapping pair, both orders, point box vs inflated
 * triangle box -> (0, a, b, vertex, triangle); once per pair (a < b), edge box
 * vs inflated edge box -> (1, a, b, edge, edge). pairs [capacity][5] sorted
 * lexicographically; INVALID with the needed count when capacity is short. */
DABD_GPU_API dabd_gpu_status dabd_gpu_broad_phase3d(int device, int n_bodies, const double* q,
                                                    const double* q_end, const int* vert_start,
                                                    const double* verts, const int* tri_start,
                                                    const int* tris, const int* edge_start,
                                                    const int* edges, double margin, int* pairs,
                                                    int capacity, int* count);

/* ---- 3D affine-body scene stepping -------------------
 * run_reference (sim.cpp:186-249) with newton.cpp:7-71 for 12-DoF bodies on
 * the 3D primitives above: predict q~ = q + h qdot + h^2 g, then Newton on
 * 1/2 (q - q~)^T M (q - q~) + h^2 kappa_arap vol ||A^T A - I||^2 + h^2 sum b(d)
 * (PSD-projected terms, eps I of newton.cpp:20-24, a block-Jacobi PCG on
 * 12x12 blocks, the CCD bound 0.9 toi and halving line search). Bodies as in
 * dabd_gpu_broad_phase3d (rest vertices about each body's centroid),
 * moments10 / volume from dabd_gpu_body3d_moments, q0 / qd0 [n][12]. No
 * reference frame exists to compare with (the reference is 2D). */
typedef struct dabd_gpu_sim3d dabd_gpu_sim3d;
typedef struct {
    double h;
    double gravity[3];
    double d_hat, kappa, kappa_arap;
    double theta, scene_scale; /* Newton tolerance theta h l on ||dq||_inf */
    int newton_cap;
    double pcg_rel_tol;
    int pcg_max_iters;
} dabd_gpu_sim3d_params;
typedef struct {
    int newton_iterations, line_search_steps, pcg_iterations, max_candidates, converged;
    double min_distance; /* over the pairs within d_hat at the committed state (0: none) */
} dabd_gpu_sim3d_stats;
DABD_GPU_API dabd_gpu_status dabd_gpu_sim3d_create(int device, int n_bodies, const int* vert_start,
                                                   const double* verts, const int* tri_start,
                                                   const int* tris, const int* edge_start,
                                                   const int* edges, const int* is_static,
                                                   const double* moments10, const double* volume,
                                                   const double* q0, const double* qd0,
                                                   const dabd_gpu_sim3d_params* params,
                                                   dabd_gpu_sim3d** out);
DABD_GPU_API void dabd_gpu_sim3d_free(dabd_gpu_sim3d* sim);
DABD_GPU_API dabd_gpu_status dabd_gpu_sim3d_run(dabd_gpu_sim3d* sim, int frames, dabd_gpu_sim3d_stats* stats);
DABD_GPU_API dabd_gpu_status dabd_gpu_sim3d_get_state(dabd_gpu_sim3d* sim, double* q, double* qd);
DABD_GPU_API dabd_gpu_status dabd_gpu_sim3d_set_state(dabd_gpu_sim3d* sim, const double* q, const double* qd);
/* The Newton system of the next frame's first iteration at the current state:
 * H [12R][12R] (dense, + eps I), g [12R] and the PCG direction dq [12R] for
 * the R dynamic bodies in body order; *rows = R. Buffers sized for 12 n. */
DABD_GPU_API dabd_gpu_status dabd_gpu_sim3d_system(dabd_gpu_sim3d* sim, double* H, double* g, double* dq,
                                                   int* rows);

/* ---- PD load balancer (host control logic, no device) ----------------------
 * balance.cpp:8-83: imbalance T = (eta-1)/(eta+1), eta = tau_i/tau_j (times
 * must be > 0, else RUNTIME); dp = kp T + kd (T - T_prev) clamped to
 * +-dp_max when dp_max > 0; balance factor = mean/max. The stateful balancer
 * smooths the times (EMA), shifts each plane along its normal and keeps w of
 * clearance to its neighbours; planes: n_planes x (px, py, nx, ny) in/out. */
DABD_GPU_API dabd_gpu_status dabd_gpu_imbalance_metric(double tau_i, double tau_j, double* out);
DABD_GPU_API dabd_gpu_status dabd_gpu_pd_update(double t, double t_prev, double kp, double kd,
                                                double dp_max, double* out);
DABD_GPU_API dabd_gpu_status dabd_gpu_balance_factor(const double* times, int n, double* out);
DABD_GPU_API dabd_gpu_status dabd_gpu_balancer_create(int num_workers,
                                                      const dabd_gpu_balance_params* p,
                                                      dabd_gpu_balancer** out);
DABD_GPU_API void dabd_gpu_balancer_free(dabd_gpu_balancer* b);
DABD_GPU_API dabd_gpu_status dabd_gpu_balancer_update(dabd_gpu_balancer* b, const double* times,
                                                      int n_planes, double* planes, double w,
                                                      double* applied);

/* ---- instrumentation (bench.py) ---------------------------------------------
 * Total dabd_gpu kernel launches so far (CUB library kernels excluded), and
 * CUDA-event timing of every launch of one named kernel (e.g. "k_pcg_spmv");
 * name == NULL disables. read() synchronises nothing: call after the work. */
DABD_GPU_API dabd_gpu_status dabd_gpu_launch_count(long long* count);
DABD_GPU_API dabd_gpu_status dabd_gpu_kernel_timer_enable(const char* kernel_name);
/* Device-side accounting of the PCG kernel since the last reset: summed
 * launch durations (%globaltimer, ns), launches, algorithmic bytes
 * (I_pcg * [288 (N_b + 2 E_o) + 504 N_b]) and iterations.
 * Valid inside captured graphs, where CUDA events cannot bracket a node. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_pcg_perf(dabd_gpu_ctx* ctx, int reset, double* ns,
                                                   long long* launches, double* bytes,
                                                   long long* iterations);
/* Cycles (clock64, CTA 0 / warp 0 of the cluster PCG) spent per phase of a
 * PCG iteration since the last reset, summed over iterations: [0] local
 * m = Dinv w + partials, [1] CTA reduction + DSMEM push, [2] arrive,
 * [3] local-column SpMV, [4] barrier wait, [5] fold + scalars, [6] remote
 * SpMV + recurrences, [7] iterations counted, [8] setup (staging, fused
 * preconditioner, exchange plan) and [9] epilogue cycles per launch, summed,
 * [10..15] setup sub-phases (staging issue + first cluster barrier, exchange
 * plan, staging wait, plan barrier, eps + factor, init), [16..19] init
 * sub-phases (eps + send plan, warm start, u = Dinv r + cluster barrier,
 * initial SpMV + m). cycles: 24 doubles. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_pcg_phases(dabd_gpu_ctx* ctx, int reset, double* cycles);
/* Skin-list counters of the local solve (no reference counterpart; the
 * reference runs a fresh broad phase per detect, geometry.cpp:161-208):
 * rebuilds since the context's instance set was last (re)built, the current
 * list length (candidate superset) and the largest per-instance skin. */
DABD_GPU_API dabd_gpu_status dabd_gpu_ctx_list_stats(dabd_gpu_ctx* ctx, long long* rebuilds,
                                                     int* length, double* delta);
/* "name launches total_ms;" per timed kernel ("*" times every kernel). */
DABD_GPU_API dabd_gpu_status dabd_gpu_kernel_timer_report(char* buf, int capacity);
DABD_GPU_API dabd_gpu_status dabd_gpu_kernel_timer_read(double* total_ms, long long* launches,
                                                        double* algorithmic_bytes);

#ifdef __cplusplus
}
#endif

#endif /* DABD_GPU_H */
