// C ABI (include/dabd_gpu.h). Conventions follow proj/src/capi.cpp:16-34:
// thread-local last error, no exceptions across the boundary, null -> INVALID.
#include "dabd_gpu.h"

#include "admm.hpp"
#include "body3d.hpp"
#include "broad3d.hpp"
#include "contact3d.hpp"
#include "engine.hpp"
#include "sim3d.hpp"
#include "instrument.hpp"
#include "scene.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

using dabd_gpu::Engine;
using dabd_gpu::HostScene;

struct dabd_gpu_scene {
    HostScene s;
};

struct dabd_gpu_balancer {
    dabd_gpu::Balancer b;
    int workers = 0;
};

struct dabd_gpu_ctx {
    std::unique_ptr<Engine> e;
};

struct dabd_gpu_sim3d {
    std::unique_ptr<dabd_gpu::Sim3d> s;
};

namespace {

dabd_gpu::BalanceOpts to_balance(const dabd_gpu_balance_params& p) {
    dabd_gpu::BalanceOpts o;
    o.enabled = p.enabled != 0;
    o.kp = p.kp;
    o.kd = p.kd;
    o.smoothing = p.smoothing;
    o.dp_max = p.dp_max;
    return o;
}

thread_local std::string g_last_error;

void set_error(const std::string& m) { g_last_error = m; }

template <typename Fn>
dabd_gpu_status guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const dabd_gpu::InvalidArg& e) {
        set_error(e.what());
        return DABD_GPU_ERR_INVALID;
    } catch (const std::exception& e) {
        set_error(e.what());
        return DABD_GPU_ERR_RUNTIME;
    }
}

dabd_gpu_status null_arg() {
    set_error("null argument");
    return DABD_GPU_ERR_INVALID;
}

dabd_gpu::SimParams to_sim(const dabd_gpu_sim_params& p) {
    dabd_gpu::SimParams s;
    s.h = p.h;
    s.gravity[0] = p.gravity_x;
    s.gravity[1] = p.gravity_y;
    s.arap_stiffness = p.arap_stiffness;
    s.barrier_stiffness = p.barrier_stiffness;
    s.d_hat = p.d_hat;
    s.theta = p.theta;
    s.scene_scale = p.scene_scale;
    return s;
}

Engine::ObjectiveIn objective_in(int n_local, const int* local, const double* kappa,
                                 const double* q_tilde, int n_anchor, const int* anchor_body,
                                 const double* anchor_zu, const double* anchor_rho,
                                 const uint32_t* holder_mask, const dabd_gpu_sim_params* sim) {
    Engine::ObjectiveIn in;
    in.n_local = n_local;
    in.local = local;
    in.kappa = kappa;
    in.q_tilde = q_tilde;
    in.n_anchor = n_anchor;
    in.anchor_body = anchor_body;
    in.anchor_zu = anchor_zu;
    in.anchor_rho = anchor_rho;
    in.holder_mask = holder_mask;
    in.sim = to_sim(*sim);
    return in;
}

} // namespace

extern "C" {

const char* dabd_gpu_version(void) { return "0.1.0"; }

const char* dabd_gpu_last_error(void) { return g_last_error.c_str(); }

dabd_gpu_status dabd_gpu_scene_create(int n_bodies, const int* bls, const int* lvs,
                                      const double* verts, const double* density,
                                      const int* is_static, const double* arap_scale,
                                      const double* qdot, dabd_gpu_scene** out) {
    if (!out || n_bodies < 0) return null_arg();
    if (n_bodies > 0 && (!bls || !lvs || !verts || !density || !is_static || !arap_scale || !qdot))
        return null_arg();
    return guarded([&] {
        auto sc = std::make_unique<dabd_gpu_scene>();
        sc->s = dabd_gpu::build_scene(n_bodies, bls, lvs, verts, density, is_static, arap_scale, qdot);
        *out = sc.release();
        return DABD_GPU_OK;
    });
}

void dabd_gpu_scene_free(dabd_gpu_scene* scene) { delete scene; }

dabd_gpu_status dabd_gpu_scene_set_params(dabd_gpu_scene* scene, const dabd_gpu_sim_params* sim,
                                          const dabd_gpu_adapt_params* adapt,
                                          const dabd_gpu_run_params* run) {
    if (!scene || !sim || !adapt || !run) return null_arg();
    return guarded([&] {
        dabd_gpu::SimParams s = to_sim(*sim);
        s.validate();
        dabd_gpu::AdaptParams a;
        a.beta = adapt->beta;
        a.tau = adapt->tau;
        a.mu = adapt->mu;
        a.sigma_min = adapt->sigma_min;
        a.sigma_max = adapt->sigma_max;
        a.adapt_enabled = adapt->adapt_enabled != 0;
        a.validate();
        if (run->admm_max_iterations < 2 || run->newton_cap < 1 || run->max_halvings < 0)
            throw dabd_gpu::InvalidArg("scene: invalid iteration limits");
        scene->s.params = s;
        scene->s.adapt = a;
        scene->s.w_min = run->w_min;
        scene->s.admm_max_iterations = run->admm_max_iterations;
        scene->s.newton_cap = run->newton_cap;
        scene->s.max_halvings = run->max_halvings;
        scene->s.force_split_frames = run->force_split_frames;
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_scene_set_planes(dabd_gpu_scene* scene, int n, const double* planes) {
    if (!scene || n < 0 || (n > 0 && !planes)) return null_arg();
    return guarded([&] {
        scene->s.planes.clear();
        for (int i = 0; i < n; ++i) {
            dabd_gpu::PlaneH p{planes[4 * i], planes[4 * i + 1], planes[4 * i + 2], planes[4 * i + 3]};
            if (std::abs(std::sqrt(p.nx * p.nx + p.ny * p.ny) - 1.0) > 1e-9)
                throw dabd_gpu::InvalidArg("partition_scene: plane normal must be unit length");
            scene->s.planes.push_back(p);
        }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_scene_set_force_split(dabd_gpu_scene* scene, int body, double fx,
                                               double fy) {
    if (!scene) return null_arg();
    if (body < 0 || body >= scene->s.nb) {
        set_error("force split body out of range");
        return DABD_GPU_ERR_INVALID;
    }
    scene->s.force_split[body] = {fx, fy};
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_scene_set_balance(dabd_gpu_scene* scene, const dabd_gpu_balance_params* p) {
    if (!scene || !p) return null_arg();
    scene->s.balance = to_balance(*p);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_scene_counts(const dabd_gpu_scene* scene, int* nb, int* nv) {
    if (!scene || !nb || !nv) return null_arg();
    *nb = scene->s.nb;
    *nv = scene->s.nv;
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_scene_bodies(const dabd_gpu_scene* scene, double* rest_xy,
                                      int* vert_start, double* q, double* mass, double* mm) {
    if (!scene) return null_arg();
    const HostScene& s = scene->s;
    if (rest_xy) std::memcpy(rest_xy, s.rest.data(), s.rest.size() * sizeof(double));
    if (vert_start) std::memcpy(vert_start, s.vstart.data(), s.vstart.size() * sizeof(int));
    if (q) std::memcpy(q, s.q0.data(), s.q0.size() * sizeof(double));
    if (mass) std::memcpy(mass, s.mass.data(), s.mass.size() * sizeof(double));
    if (mm)
        for (int b = 0; b < s.nb; ++b) s.full_mass_matrix(b, mm + 36 * b);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_ctx_create(const dabd_gpu_scene* scene, int device, int num_workers,
                                    int part_begin, int part_end, dabd_gpu_ctx** out) {
    if (!scene || !out) return null_arg();
    return guarded([&] {
        auto c = std::make_unique<dabd_gpu_ctx>();
        c->e = std::make_unique<Engine>(scene->s, device, num_workers, part_begin, part_end);
        *out = c.release();
        return DABD_GPU_OK;
    });
}

void dabd_gpu_ctx_free(dabd_gpu_ctx* ctx) { delete ctx; }

dabd_gpu_status dabd_gpu_ctx_set_solver(dabd_gpu_ctx* ctx, const dabd_gpu_solver_params* p) {
    if (!ctx || !p) return null_arg();
    if (!(p->pcg_rel_tol > 0.0) || p->pcg_max_iters < 1) {
        set_error("invalid solver parameters");
        return DABD_GPU_ERR_INVALID;
    }
    ctx->e->set_solver(p->pcg_rel_tol, p->pcg_max_iters);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_ctx_set_inexact(dabd_gpu_ctx* ctx, double eta, double factor) {
    if (!ctx) return null_arg();
    if (!(eta >= 0.0) || !(factor >= 1.0)) {
        set_error("invalid inexact-Newton parameters (eta >= 0, factor >= 1)");
        return DABD_GPU_ERR_INVALID;
    }
    ctx->e->set_inexact(eta, factor);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_ctx_set_stream(dabd_gpu_ctx* ctx, uintptr_t stream) {
    if (!ctx) return null_arg();
    return guarded([&] {
        ctx->e->set_stream(reinterpret_cast<cudaStream_t>(stream));
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_ctx_set_comm(dabd_gpu_ctx* ctx, const dabd_gpu_comm* comm) {
    if (!ctx) return null_arg();
    return guarded([&] {
        dabd_gpu::Comm c;
        if (comm) {
            if (!comm->halo || !comm->allgather || !comm->part_offsets || comm->world < 1 ||
                comm->rank < 0 || comm->rank >= comm->world)
                throw dabd_gpu::InvalidArg("comm: missing callbacks or bad rank/world");
            c.user = comm->user;
            c.halo = comm->halo;
            c.allgather = comm->allgather;
            c.rank = comm->rank;
            c.world = comm->world;
            c.part_offsets.assign(comm->part_offsets, comm->part_offsets + comm->world + 1);
        }
        ctx->e->set_comm(comm ? &c : nullptr);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_broad_phase(dabd_gpu_ctx* ctx, const double* q, const double* q_end,
                                     double margin, const int* subset, int n_subset, int* pairs,
                                     int capacity, int* count) {
    if (!ctx || !q || !count || (capacity > 0 && !pairs)) return null_arg();
    return guarded([&] {
        const std::vector<int> out = ctx->e->broad_phase(q, q_end, margin, subset, n_subset);
        const int n = static_cast<int>(out.size() / 4);
        *count = n;
        if (n > capacity) {
            set_error("capacity too small");
            return DABD_GPU_ERR_INVALID;
        }
        if (n) std::memcpy(pairs, out.data(), out.size() * sizeof(int));
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_narrow_phase(dabd_gpu_ctx* ctx, const double* q, const int* cand, int n,
                                      double d_hat, int* out_pairs, double* out_d, int* count) {
    if (!ctx || !q || !count || (n > 0 && (!cand || !out_pairs || !out_d))) return null_arg();
    return guarded([&] {
        std::vector<int> pairs;
        std::vector<double> d;
        ctx->e->narrow_phase(q, cand, n, d_hat, pairs, d);
        *count = static_cast<int>(d.size());
        if (!d.empty()) {
            std::memcpy(out_pairs, pairs.data(), pairs.size() * sizeof(int));
            std::memcpy(out_d, d.data(), d.size() * sizeof(double));
        }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_ccd_toi(dabd_gpu_ctx* ctx, const double* q0, const double* q1,
                                 const int* subset, int n_subset, double* toi) {
    if (!ctx || !q0 || !q1 || !toi) return null_arg();
    return guarded([&] {
        *toi = ctx->e->ccd_toi(q0, q1, subset, n_subset);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_holder_masks(dabd_gpu_ctx* ctx, const double* q, int n_planes,
                                      const double* planes, double w, uint32_t* masks) {
    if (!ctx || !q || !masks || n_planes < 0 || (n_planes > 0 && !planes)) return null_arg();
    return guarded([&] {
        ctx->e->holder_masks(q, n_planes, planes, w, masks);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_audit(dabd_gpu_ctx* ctx, const double* q, const int* subset, int n_subset,
                               double cutoff, int* result, int* n_violations, double* min_distance) {
    if (!ctx || !result || n_subset < 0 || !(cutoff >= 0.0)) return null_arg();
    return guarded([&] {
        const dabd_gpu::AuditResult r = ctx->e->audit(q, subset, n_subset, cutoff);
        *result = r.violations > 0 ? 1 : 0;
        if (n_violations) *n_violations = r.violations;
        if (min_distance) *min_distance = r.min_distance;
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_objective(dabd_gpu_ctx* ctx, int n_local, const int* local,
                                   const double* kappa, const double* q_tilde, int n_anchor,
                                   const int* anchor_body, const double* anchor_zu,
                                   const double* anchor_rho, const uint32_t* holder_mask,
                                   const dabd_gpu_sim_params* sim, const double* q, int mode,
                                   double* value, double* grad, double* hess_dense, int* active,
                                   int* candidates) {
    if (!ctx || !sim || !q || !value || !active || !candidates || n_local < 0) return null_arg();
    if (n_local > 0 && (!local || !kappa || !q_tilde)) return null_arg();
    if (n_anchor > 0 && (!anchor_body || !anchor_zu || !anchor_rho)) return null_arg();
    return guarded([&] {
        ctx->e->objective(objective_in(n_local, local, kappa, q_tilde, n_anchor, anchor_body,
                                       anchor_zu, anchor_rho, holder_mask, sim),
                          q, mode, value, grad, hess_dense, active, candidates);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_newton_solve(dabd_gpu_ctx* ctx, int n_local, const int* local,
                                      const double* kappa, const double* q_tilde, int n_anchor,
                                      const int* anchor_body, const double* anchor_zu,
                                      const double* anchor_rho, const uint32_t* holder_mask,
                                      const dabd_gpu_sim_params* sim, double* q, int max_iters,
                                      double tol, int* iterations, double* final_update_inf,
                                      int* converged, int* line_search_steps) {
    if (!ctx || !sim || !q || !iterations || !final_update_inf || !converged || !line_search_steps)
        return null_arg();
    if (n_local > 0 && (!local || !kappa || !q_tilde)) return null_arg();
    if (n_anchor > 0 && (!anchor_body || !anchor_zu || !anchor_rho)) return null_arg();
    return guarded([&] {
        const dabd_gpu::NewtonResult r = ctx->e->newton_solve(
            objective_in(n_local, local, kappa, q_tilde, n_anchor, anchor_body, anchor_zu,
                         anchor_rho, holder_mask, sim),
            q, max_iters, tol);
        *iterations = r.iterations;
        *final_update_inf = r.final_update;
        *converged = r.converged;
        *line_search_steps = r.ls_steps;
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_run_frames(dabd_gpu_ctx* ctx, int n_frames, dabd_gpu_frame_stats* stats) {
    if (!ctx || n_frames < 0) return null_arg();
    return guarded([&] {
        std::vector<dabd_gpu::FrameStats> st(n_frames);
        ctx->e->run_frames(n_frames, st.data());
        if (stats)
            for (int f = 0; f < n_frames; ++f) {
                dabd_gpu_frame_stats& o = stats[f];
                o.committed = st[f].committed;
                o.attempts = st[f].attempts;
                o.h = st[f].h;
                o.admm_iterations = st[f].admm_iterations;
                o.newton_iterations = st[f].newton_iterations;
                o.line_search_steps = st[f].line_search_steps;
                o.pcg_iterations = st[f].pcg_iterations;
                o.max_contacts = st[f].max_contacts;
                o.max_candidates = st[f].max_candidates;
                o.exact_retries = st[f].exact_retries;
                o.capacity_retries = st[f].capacity_retries;
                o.t_solve = st[f].t_solve;
                o.t_coll = st[f].t_coll;
                o.t_sync = st[f].t_sync;
                o.t_frame = st[f].t_frame;
            }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_set_state(dabd_gpu_ctx* ctx, const double* q, const double* qdot) {
    if (!ctx || !q || !qdot) return null_arg();
    return guarded([&] {
        ctx->e->set_state(q, qdot);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_get_state(dabd_gpu_ctx* ctx, double* q, double* qdot) {
    if (!ctx) return null_arg();
    return guarded([&] {
        ctx->e->get_state(q, qdot);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_get_rho(dabd_gpu_ctx* ctx, double* rho) {
    if (!ctx || !rho) return null_arg();
    ctx->e->get_rho(rho);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_ctx_comm_mode(dabd_gpu_ctx* ctx, int* mode) {
    if (!ctx || !mode) return null_arg();
    *mode = ctx->e->comm_mode();
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_ctx_get_planes(dabd_gpu_ctx* ctx, double* planes) {
    if (!ctx || !planes) return null_arg();
    const std::vector<double> p = ctx->e->planes();
    std::copy(p.begin(), p.end(), planes);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_ctx_partition_costs(dabd_gpu_ctx* ctx, double* costs) {
    if (!ctx || !costs) return null_arg();
    const std::vector<double>& c = ctx->e->partition_costs();
    std::copy(c.begin(), c.end(), costs);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_contact3d_terms(int device, int n, const int* kind, const double* qa,
                                         const double* qb, const double* rest, double d_hat,
                                         double kappa, double weight, int project, double* d,
                                         int* dtype, double* value, double* grad, double* hess) {
    if (n < 0) return null_arg();
    if (n > 0 && (!kind || !qa || !qb || !rest || !d || !dtype || !value || !grad)) return null_arg();
    if (!(d_hat > 0.0)) {
        set_error("contact3d: d_hat must be > 0");
        return DABD_GPU_ERR_INVALID;
    }
    return guarded([&] {
        for (int k = 0; k < n; ++k)
            if (kind[k] != 0 && kind[k] != 1) throw dabd_gpu::InvalidArg("contact3d: kind must be 0 (PT) or 1 (EE)");
        if (n == 0) return DABD_GPU_OK;
        CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t s = nullptr;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        dabd_gpu::DBuf<int> dk, dt, derr;
        dabd_gpu::DBuf<double> dqa, dqb, dr, dd, dv, dg, dh;
        dk.upload(kind, n, s);
        dqa.upload(qa, 12 * static_cast<size_t>(n), s);
        dqb.upload(qb, 12 * static_cast<size_t>(n), s);
        dr.upload(rest, 12 * static_cast<size_t>(n), s);
        dd.resize(n);
        dt.resize(n);
        dv.resize(n);
        dg.resize(24 * static_cast<size_t>(n));
        if (hess) dh.resize(576 * static_cast<size_t>(n));
        derr.resize(1);
        derr.zero(s);
        dabd_gpu::Contact3dArgs a{n, dk.get(), dqa.get(), dqb.get(), dr.get(), d_hat, kappa, weight,
                                  project, dd.get(), dt.get(), dv.get(), dg.get(),
                                  hess ? dh.get() : nullptr, derr.get()};
        dabd_gpu::launch_contact3d(a, s);
        CUDA_CHECK(cudaGetLastError());
        int err = 0;
        CUDA_CHECK(cudaMemcpyAsync(d, dd.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(dtype, dt.get(), n * sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(value, dv.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(grad, dg.get(), 24 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (hess)
            CUDA_CHECK(cudaMemcpyAsync(hess, dh.get(), 576 * static_cast<size_t>(n) * sizeof(double),
                                       cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(&err, derr.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamDestroy(s));
        if (err) throw dabd_gpu::Error("contact3d: a pair has d <= 0 (interpenetration)");
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_ccd3d(int device, int n, const int* kind, const double* qa0, const double* qa1,
                               const double* qb0, const double* qb1, const double* rest, double* toi) {
    if (n < 0) return null_arg();
    if (n > 0 && (!kind || !qa0 || !qa1 || !qb0 || !qb1 || !rest || !toi)) return null_arg();
    return guarded([&] {
        for (int k = 0; k < n; ++k)
            if (kind[k] != 0 && kind[k] != 1) throw dabd_gpu::InvalidArg("ccd3d: kind must be 0 (PT) or 1 (EE)");
        if (n == 0) return DABD_GPU_OK;
        CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t s = nullptr;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const size_t m = 12 * static_cast<size_t>(n);
        dabd_gpu::DBuf<int> dk;
        dabd_gpu::DBuf<double> a0, a1, b0, b1, dr, dt;
        dk.upload(kind, n, s);
        a0.upload(qa0, m, s);
        a1.upload(qa1, m, s);
        b0.upload(qb0, m, s);
        b1.upload(qb1, m, s);
        dr.upload(rest, m, s);
        dt.resize(n);
        dabd_gpu::Ccd3dArgs a{n, dk.get(), a0.get(), a1.get(), b0.get(), b1.get(), dr.get(), dt.get()};
        dabd_gpu::launch_ccd3d(a, s);
        CUDA_CHECK(cudaGetLastError());
        CUDA_CHECK(cudaMemcpyAsync(toi, dt.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamDestroy(s));
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_body3d_moments(int n_verts, const double* verts, int n_tris, const int* tris,
                                        double density, double* moments10, double* centroid,
                                        double* volume) {
    if (!verts || !tris || !moments10 || n_verts < 4 || n_tris < 4) return null_arg();
    return guarded([&] {
        const dabd_gpu::Moments3 m = dabd_gpu::polyhedron_moments(n_verts, verts, n_tris, tris, density);
        std::copy(m.mom, m.mom + 10, moments10);
        if (centroid) std::copy(m.centroid, m.centroid + 3, centroid);
        if (volume) *volume = m.volume;
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_body3d_terms(int device, int n, const double* q, const double* qt,
                                      const double* moments10, const double* w, double scale,
                                      int project, double* value, double* grad, double* hess) {
    if (n < 0) return null_arg();
    if (n > 0 && (!q || !qt || !moments10 || !w || !value || !grad)) return null_arg();
    return guarded([&] {
        if (n == 0) return DABD_GPU_OK;
        CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t s = nullptr;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const size_t m12 = 12 * static_cast<size_t>(n);
        dabd_gpu::DBuf<double> dq, dqt, dm, dw, dv, dg, dh;
        dq.upload(q, m12, s);
        dqt.upload(qt, m12, s);
        dm.upload(moments10, 10 * static_cast<size_t>(n), s);
        dw.upload(w, n, s);
        dv.resize(n);
        dg.resize(m12);
        if (hess) dh.resize(144 * static_cast<size_t>(n));
        dabd_gpu::Body3dArgs a{n, dq.get(), dqt.get(), dm.get(), dw.get(), scale, project,
                               dv.get(), dg.get(), hess ? dh.get() : nullptr};
        dabd_gpu::launch_body3d(a, s);
        CUDA_CHECK(cudaGetLastError());
        CUDA_CHECK(cudaMemcpyAsync(value, dv.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(grad, dg.get(), m12 * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (hess)
            CUDA_CHECK(cudaMemcpyAsync(hess, dh.get(), 144 * static_cast<size_t>(n) * sizeof(double),
                                       cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaStreamDestroy(s));
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_broad_phase3d(int device, int n, const double* q, const double* q_end,
                                       const int* vert_start, const double* verts, const int* tri_start,
                                       const int* tris, const int* edge_start, const int* edges,
                                       double margin, int* pairs, int capacity, int* count) {
    if (n < 0 || !count || (n > 0 && (!q || !vert_start || !verts || !tri_start || !tris || !edge_start || !edges)) ||
        (capacity > 0 && !pairs))
        return null_arg();
    return guarded([&] {
        *count = 0;
        if (n < 2) return DABD_GPU_OK;
        const int nv = vert_start[n], nt = tri_start[n], ne = edge_start[n];
        int maxp = 1;
        for (int b = 0; b < n; ++b) {
            if (vert_start[b + 1] < vert_start[b] || tri_start[b + 1] < tri_start[b] || edge_start[b + 1] < edge_start[b])
                throw dabd_gpu::InvalidArg("broad_phase3d: offsets must be non-decreasing");
            const int nvb = vert_start[b + 1] - vert_start[b];
            for (int t = 3 * tri_start[b]; t < 3 * tri_start[b + 1]; ++t)
                if (tris[t] < 0 || tris[t] >= nvb) throw dabd_gpu::InvalidArg("broad_phase3d: triangle vertex out of range");
            for (int e = 2 * edge_start[b]; e < 2 * edge_start[b + 1]; ++e)
                if (edges[e] < 0 || edges[e] >= nvb) throw dabd_gpu::InvalidArg("broad_phase3d: edge vertex out of range");
            maxp = std::max({maxp, nvb, tri_start[b + 1] - tri_start[b], edge_start[b + 1] - edge_start[b]});
        }
        auto bits = [](int x) {
            int b = 1;
            while ((1ll << b) < x) ++b;
            return b;
        };
        dabd_gpu::Key3Fmt f;
        f.bb = bits(n);
        f.pb = bits(maxp);
        if (f.total_bits() > 64) throw dabd_gpu::InvalidArg("broad_phase3d: body / primitive counts exceed the key width");
        CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t s = nullptr;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        dabd_gpu::DBuf<double> dq, dqe, dv;
        dabd_gpu::DBuf<int> dvs, dts, dt, des, de;
        dq.upload(q, 12 * static_cast<size_t>(n), s);
        if (q_end) dqe.upload(q_end, 12 * static_cast<size_t>(n), s);
        dvs.upload(vert_start, n + 1, s);
        dv.upload(verts, 3 * static_cast<size_t>(std::max(nv, 1)), s);
        dts.upload(tri_start, n + 1, s);
        dt.upload(tris, 3 * static_cast<size_t>(std::max(nt, 1)), s);
        des.upload(edge_start, n + 1, s);
        de.upload(edges, 2 * static_cast<size_t>(std::max(ne, 1)), s);
        dabd_gpu::Broad3dView v{n, dq.get(), q_end ? dqe.get() : nullptr, dvs.get(), dv.get(), dts.get(),
                                dt.get(), des.get(), de.get(), margin};
        const std::vector<unsigned long long> keys = dabd_gpu::broad_phase3d(v, f, s);
        CUDA_CHECK(cudaStreamDestroy(s));
        *count = static_cast<int>(keys.size());
        if (*count > capacity) {
            set_error("broad_phase3d: capacity too small (needed count written)");
            return DABD_GPU_ERR_INVALID;
        }
        for (size_t k = 0; k < keys.size(); ++k) {
            int* o = pairs + 5 * k;
            f.unpack(keys[k], o[0], o[1], o[2], o[3], o[4]);
        }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_check_stopping(double dq, double r, double s, const double* tois, int n_tois,
                                        double h, double l, double theta, int* end) {
    if (!end || n_tois < 0 || (n_tois > 0 && !tois)) return null_arg();
    return guarded([&] {
        *end = dabd_gpu::check_stopping(dq, r, s, tois, n_tois, h, l, theta) ? 1 : 0;
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_timestep_apply(double h0, int max_halvings, const int* events, int n_events,
                                        double* h_after) {
    if (n_events < 0 || (n_events > 0 && (!events || !h_after))) return null_arg();
    return guarded([&] {
        dabd_gpu::TimestepController ts(h0, max_halvings);
        for (int i = 0; i < n_events; ++i) {
            if (events[i] == 0) ts.on_frame_failed();
            else ts.on_frame_committed();
            h_after[i] = ts.h();
        }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_consensus_step(int device, int n, const double* q, const double* u,
                                        const double* rho, const double* z_prev, const double* rho0,
                                        const dabd_gpu_adapt_params* adapt, double* z, double* u_new,
                                        double* r, double* s, double* rho_next) {
    if (n < 0 || !adapt) return null_arg();
    if (n > 0 && (!q || !u || !rho || !z_prev || !rho0 || !z || !u_new || !r || !s || !rho_next))
        return null_arg();
    return guarded([&] {
        if (n == 0) return DABD_GPU_OK;
        for (int i = 0; i < n; ++i)
            if (!(rho[i] > 0.0)) throw dabd_gpu::Error("consensus_update: rho must be > 0");
        CUDA_CHECK(cudaSetDevice(device));
        cudaStream_t st = nullptr;
        CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const int I = 2 * n; // replica instances 2i (partition 0), 2i + 1 (partition 1)
        std::vector<double> hrho(I), hrho0(I), hz(6 * static_cast<size_t>(I));
        std::vector<int> hpart(I), hsh(I), hanc(I, 1);
        for (int i = 0; i < n; ++i)
            for (int h = 0; h < 2; ++h) {
                const int k = 2 * i + h;
                hrho[k] = rho[i];
                hrho0[k] = rho0[i];
                hpart[k] = h;
                hsh[k] = k;
                for (int c = 0; c < 6; ++c) hz[6 * k + c] = z_prev[6 * i + c];
            }
        dabd_gpu::DBuf<double> dq, du, drho, drho0, dz, dzn, drb, dsb, drl, dsl;
        dabd_gpu::DBuf<int> dpart, dsh, danc, derr;
        dq.upload(q, 6 * static_cast<size_t>(I), st);
        du.upload(u, 6 * static_cast<size_t>(I), st);
        drho.upload(hrho, st);
        drho0.upload(hrho0, st);
        dz.upload(hz, st);
        dzn.resize(6 * static_cast<size_t>(I));
        drb.resize(I);
        dsb.resize(I);
        drl.resize(2);
        dsl.resize(2);
        drl.zero(st);
        dsl.zero(st);
        dpart.upload(hpart, st);
        dsh.upload(hsh, st);
        danc.upload(hanc, st);
        derr.resize(1);
        derr.zero(st);
        dabd_gpu::launch_consensus(n, dsh.get(), dpart.get(), 0, dq.get(), du.get(), drho.get(), dz.get(),
                                   nullptr, nullptr, 0, dzn.get(), drb.get(), dsb.get(), drl.get(), dsl.get(),
                                   derr.get(), st);
        dabd_gpu::AdaptParams ap;
        ap.beta = adapt->beta;
        ap.tau = adapt->tau;
        ap.mu = adapt->mu;
        ap.sigma_min = adapt->sigma_min;
        ap.sigma_max = adapt->sigma_max;
        ap.adapt_enabled = adapt->adapt_enabled != 0;
        dabd_gpu::launch_adapt(I, danc.get(), drho.get(), drho0.get(), drb.get(), dsb.get(), ap, dz.get(),
                               dzn.get(), st);
        CUDA_CHECK(cudaGetLastError());
        const std::vector<double> zn = dzn.to_host(st), un = du.to_host(st), rb = drb.to_host(st),
                                  sb = dsb.to_host(st), rn = drho.to_host(st);
        const std::vector<int> e = derr.to_host(st);
        CUDA_CHECK(cudaStreamDestroy(st));
        if (e[0] != 0) throw dabd_gpu::Error("consensus: replica rho mismatch");
        for (int i = 0; i < n; ++i) {
            for (int c = 0; c < 6; ++c) z[6 * i + c] = zn[12 * i + c];
            for (int c = 0; c < 12; ++c) u_new[12 * i + c] = un[12 * i + c];
            r[i] = rb[2 * i];
            s[i] = sb[2 * i];
            rho_next[i] = rn[2 * i];
        }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_imbalance_metric(double tau_i, double tau_j, double* out) {
    if (!out) return null_arg();
    return guarded([&] {
        *out = dabd_gpu::imbalance_metric(tau_i, tau_j);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_pd_update(double t, double t_prev, double kp, double kd, double dp_max,
                                   double* out) {
    if (!out) return null_arg();
    *out = dabd_gpu::pd_update(t, t_prev, kp, kd, dp_max);
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_balance_factor(const double* times, int n, double* out) {
    if (!out || n < 0 || (n > 0 && !times)) return null_arg();
    return guarded([&] {
        *out = dabd_gpu::balance_factor(std::vector<double>(times, times + n));
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_balancer_create(int num_workers, const dabd_gpu_balance_params* p,
                                         dabd_gpu_balancer** out) {
    if (!p || !out || num_workers < 1) return null_arg();
    return guarded([&] {
        auto b = std::make_unique<dabd_gpu_balancer>();
        b->b = dabd_gpu::Balancer(num_workers, to_balance(*p));
        b->workers = num_workers;
        *out = b.release();
        return DABD_GPU_OK;
    });
}

void dabd_gpu_balancer_free(dabd_gpu_balancer* b) { delete b; }

dabd_gpu_status dabd_gpu_balancer_update(dabd_gpu_balancer* b, const double* times, int n_planes,
                                         double* planes, double w, double* applied) {
    if (!b || !times || n_planes < 0 || (n_planes > 0 && !planes)) return null_arg();
    return guarded([&] {
        std::vector<dabd_gpu::PlaneH> pl(n_planes);
        for (int k = 0; k < n_planes; ++k) pl[k] = {planes[4 * k], planes[4 * k + 1], planes[4 * k + 2], planes[4 * k + 3]};
        const std::vector<double> dp =
            b->b.update(std::vector<double>(times, times + b->workers), pl, w);
        for (int k = 0; k < n_planes; ++k) {
            planes[4 * k] = pl[k].px;
            planes[4 * k + 1] = pl[k].py;
            planes[4 * k + 2] = pl[k].nx;
            planes[4 * k + 3] = pl[k].ny;
            if (applied) applied[k] = dp[k];
        }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_take_trace(dabd_gpu_ctx* ctx, double* rows, int capacity, int* count) {
    if (!ctx || !count || (capacity > 0 && !rows)) return null_arg();
    return guarded([&] {
        const std::vector<dabd_gpu::TraceRow> t = ctx->e->take_trace();
        const int n = std::min<int>(capacity, static_cast<int>(t.size()));
        *count = n;
        for (int i = 0; i < n; ++i) std::memcpy(rows + 8 * i, &t[i], 8 * sizeof(double));
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_launch_count(long long* count) {
    if (!count) return null_arg();
    *count = dabd_gpu::launch_counter().load();
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_kernel_timer_enable(const char* name) {
    dabd_gpu::KernelTimer::get().enable(name ? name : "");
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_ctx_pcg_perf(dabd_gpu_ctx* ctx, int reset, double* ns,
                                      long long* launches, double* bytes, long long* iterations) {
    if (!ctx || !ns || !launches || !bytes || !iterations) return null_arg();
    return guarded([&] {
        const dabd_gpu::DevPerf p = ctx->e->read_perf(reset != 0);
        *ns = static_cast<double>(p.ns);
        *launches = static_cast<long long>(p.launches);
        *bytes = p.bytes;
        *iterations = static_cast<long long>(p.iters);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_ctx_pcg_phases(dabd_gpu_ctx* ctx, int reset, double* cycles) {
    if (!ctx || !cycles) return null_arg();
    return guarded([&] {
        const dabd_gpu::DevPerf p = ctx->e->read_perf(reset != 0);
        for (int k = 0; k < 24; ++k) cycles[k] = static_cast<double>(p.phase[k]);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_ctx_list_stats(dabd_gpu_ctx* ctx, long long* rebuilds, int* length,
                                       double* delta) {
    if (!ctx || !rebuilds || !length || !delta) return null_arg();
    return guarded([&] {
        ctx->e->list_stats(rebuilds, length, delta);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_kernel_timer_report(char* buf, int capacity) {
    if (!buf || capacity < 1) return null_arg();
    const std::string r = dabd_gpu::KernelTimer::get().report();
    std::strncpy(buf, r.c_str(), static_cast<size_t>(capacity) - 1);
    buf[capacity - 1] = '\0';
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_kernel_timer_read(double* total_ms, long long* launches,
                                           double* algorithmic_bytes) {
    if (!total_ms || !launches || !algorithmic_bytes) return null_arg();
    *algorithmic_bytes = dabd_gpu::KernelTimer::get().bytes();
    *total_ms = dabd_gpu::KernelTimer::get().total_ms();
    *launches = dabd_gpu::KernelTimer::get().count();
    return DABD_GPU_OK;
}

dabd_gpu_status dabd_gpu_sim3d_create(int device, int n, const int* vert_start, const double* verts,
                                      const int* tri_start, const int* tris, const int* edge_start, const int* edges,
                                      const int* is_static, const double* moments10, const double* volume,
                                      const double* q0, const double* qd0, const dabd_gpu_sim3d_params* p,
                                      dabd_gpu_sim3d** out) {
    if (!out || !p || n < 1 || !vert_start || !verts || !tri_start || !tris || !edge_start || !edges || !is_static ||
        !moments10 || !volume || !q0 || !qd0)
        return null_arg();
    *out = nullptr;
    return guarded([&] {
        if (!(p->h > 0.0) || !(p->d_hat > 0.0) || !(p->kappa > 0.0) || !(p->theta > 0.0) || p->newton_cap < 1 ||
            !(p->pcg_rel_tol > 0.0) || p->pcg_max_iters < 1)
            throw dabd_gpu::InvalidArg("sim3d: invalid parameters");
        for (int b = 0; b < n; ++b) {
            const int nvb = vert_start[b + 1] - vert_start[b];
            if (nvb < 1 || tri_start[b + 1] < tri_start[b] || edge_start[b + 1] < edge_start[b])
                throw dabd_gpu::InvalidArg("sim3d: offsets must be non-decreasing, every body needs vertices");
            for (int t = 3 * tri_start[b]; t < 3 * tri_start[b + 1]; ++t)
                if (tris[t] < 0 || tris[t] >= nvb) throw dabd_gpu::InvalidArg("sim3d: triangle vertex out of range");
            for (int e = 2 * edge_start[b]; e < 2 * edge_start[b + 1]; ++e)
                if (edges[e] < 0 || edges[e] >= nvb) throw dabd_gpu::InvalidArg("sim3d: edge vertex out of range");
        }
        dabd_gpu::Sim3dParams sp;
        sp.h = p->h;
        for (int k = 0; k < 3; ++k) sp.gravity[k] = p->gravity[k];
        sp.d_hat = p->d_hat;
        sp.kappa = p->kappa;
        sp.kappa_arap = p->kappa_arap;
        sp.theta = p->theta;
        sp.scene_scale = p->scene_scale;
        sp.newton_cap = p->newton_cap;
        sp.pcg_rel_tol = p->pcg_rel_tol;
        sp.pcg_max_iters = p->pcg_max_iters;
        auto h = std::make_unique<dabd_gpu_sim3d>();
        h->s = std::make_unique<dabd_gpu::Sim3d>(device, n, vert_start, verts, tri_start, tris, edge_start, edges,
                                                 is_static, moments10, volume, q0, qd0, sp);
        *out = h.release();
        return DABD_GPU_OK;
    });
}

void dabd_gpu_sim3d_free(dabd_gpu_sim3d* sim) { delete sim; }

dabd_gpu_status dabd_gpu_sim3d_run(dabd_gpu_sim3d* sim, int frames, dabd_gpu_sim3d_stats* stats) {
    if (!sim || frames < 0 || (frames > 0 && !stats)) return null_arg();
    return guarded([&] {
        for (int f = 0; f < frames; ++f) {
            const dabd_gpu::Sim3dStats s = sim->s->frame();
            stats[f] = dabd_gpu_sim3d_stats{s.newton_iterations, s.line_search_steps, s.pcg_iterations,
                                            s.max_candidates, s.converged, s.min_distance};
        }
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_sim3d_get_state(dabd_gpu_sim3d* sim, double* q, double* qd) {
    if (!sim || !q || !qd) return null_arg();
    return guarded([&] {
        sim->s->state(q, qd);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_sim3d_set_state(dabd_gpu_sim3d* sim, const double* q, const double* qd) {
    if (!sim || !q || !qd) return null_arg();
    return guarded([&] {
        sim->s->set_state(q, qd);
        return DABD_GPU_OK;
    });
}

dabd_gpu_status dabd_gpu_sim3d_system(dabd_gpu_sim3d* sim, double* H, double* g, double* dq, int* rows) {
    if (!sim || !H || !g || !dq || !rows) return null_arg();
    return guarded([&] {
        *rows = sim->s->system(H, g, dq);
        return DABD_GPU_OK;
    });
}

} // extern "C"
