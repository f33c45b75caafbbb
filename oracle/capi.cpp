// TEST INFRASTRUCTURE ONLY (see oracle.hpp). Flat C entry points so the
// Python tests can drive the oracle through ctypes. Error convention mirrors
// proj/src/capi.cpp:16-34 (status code + thread-local last error).
#include "oracle.hpp"

#include <cstring>
#include <memory>

using namespace oracle;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Configs to_configs(const double* q, int n) {
    Configs c(n);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 6; ++k) c[i][k] = q[6 * i + k];
    return c;
}

void from_configs(const Configs& c, double* q) {
    for (size_t i = 0; i < c.size(); ++i)
        for (int k = 0; k < 6; ++k) q[6 * i + k] = c[i][k];
}

std::vector<int> to_vec(const int* p, int n) {
    return p && n > 0 ? std::vector<int>(p, p + n) : std::vector<int>();
}

void write_pairs(const std::vector<ContactPair>& v, int* pairs, double* d, int cap, int* count) {
    *count = static_cast<int>(v.size());
    if (static_cast<int>(v.size()) > cap) throw Error("capacity too small");
    for (size_t i = 0; i < v.size(); ++i) {
        pairs[4 * i + 0] = v[i].body_a;
        pairs[4 * i + 1] = v[i].body_b;
        pairs[4 * i + 2] = v[i].point_index;
        pairs[4 * i + 3] = v[i].edge_index;
        if (d) d[i] = v[i].d;
    }
}

std::vector<ContactPair> read_pairs(const int* pairs, int n) {
    std::vector<ContactPair> v(n);
    for (int i = 0; i < n; ++i) {
        v[i].body_a = pairs[4 * i];
        v[i].body_b = pairs[4 * i + 1];
        v[i].point_index = pairs[4 * i + 2];
        v[i].edge_index = pairs[4 * i + 3];
    }
    return v;
}

SimParams params_from(const double* s8) {
    SimParams p;
    p.h = s8[0];
    p.gravity = {s8[1], s8[2]};
    p.arap_stiffness = s8[3];
    p.barrier_stiffness = s8[4];
    p.d_hat = s8[5];
    p.theta = s8[6];
    p.scene_scale = s8[7];
    return p;
}

LocalObjective make_objective(const Scene* s, int n_local, const int* local, const double* kappa,
                              const double* q_tilde, int n_anchor, const int* anchor_body,
                              const double* anchor_zu, const double* anchor_rho,
                              const uint32_t* holder_mask, const double* sim8) {
    std::vector<int> loc(local, local + n_local);
    std::vector<double> kap(kappa, kappa + n_local);
    std::vector<Vec6> qt(n_local);
    for (int i = 0; i < n_local; ++i)
        for (int k = 0; k < 6; ++k) qt[i][k] = q_tilde[6 * i + k];
    std::vector<SharedAnchor> an(n_anchor);
    for (int i = 0; i < n_anchor; ++i) {
        an[i].body = anchor_body[i];
        for (int k = 0; k < 6; ++k) {
            an[i].z[k] = anchor_zu[12 * i + k];
            an[i].u[k] = anchor_zu[12 * i + 6 + k];
        }
        an[i].rho = anchor_rho[i];
    }
    std::vector<uint32_t> hm;
    if (holder_mask) hm.assign(holder_mask, holder_mask + s->bodies.size());
    return LocalObjective::assemble(s->bodies, loc, kap, qt, an, hm, params_from(sim8));
}

} // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

// Body specs (the JSON-level BodySpec of scene.cpp:81-98), flattened:
// body b owns loops [body_loop_start[b], body_loop_start[b+1]); loop l owns
// vertices [loop_vert_start[l], loop_vert_start[l+1]) of verts (world xy).
void* oracle_scene_new(int n_bodies, const int* body_loop_start, const int* loop_vert_start,
                       const double* verts, const double* density, const int* is_static,
                       const double* arap_scale, const double* qdot) {
    Scene* s = nullptr;
    const int rc = guarded([&] {
        auto sc = std::make_unique<Scene>();
        for (int b = 0; b < n_bodies; ++b) {
            std::vector<Loop> loops;
            for (int l = body_loop_start[b]; l < body_loop_start[b + 1]; ++l) {
                Loop lp;
                for (int v = loop_vert_start[l]; v < loop_vert_start[l + 1]; ++v)
                    lp.push_back({verts[2 * v], verts[2 * v + 1]});
                loops.push_back(lp);
            }
            AffineBody body = make_affine_body(b, loops, density[b], is_static[b] != 0);
            body.arap_scale = arap_scale[b];
            for (int k = 0; k < 6; ++k) body.q_dot[k] = qdot[6 * b + k];
            sc->bodies.push_back(std::move(body));
        }
        s = sc.release();
    });
    return rc == 0 ? s : nullptr;
}

void oracle_scene_free(void* s) { delete static_cast<Scene*>(s); }

int oracle_scene_set_params(void* sp, const double* sim8, const double* adapt5,
                            int adapt_enabled, int K, int newton_cap, int max_halvings,
                            double w_min, int n_planes, const double* planes4,
                            int force_split_frames) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        s->params = params_from(sim8);
        s->adapt.beta = adapt5[0];
        s->adapt.tau = adapt5[1];
        s->adapt.mu = adapt5[2];
        s->adapt.sigma_min = adapt5[3];
        s->adapt.sigma_max = adapt5[4];
        s->adapt.adapt_enabled = adapt_enabled != 0;
        s->params.validate();
        s->adapt.validate();
        s->admm_max_iterations = K;
        s->newton_cap = newton_cap;
        s->max_halvings = max_halvings;
        s->w_min = w_min;
        s->planes.clear();
        for (int i = 0; i < n_planes; ++i)
            s->planes.push_back({{planes4[4 * i], planes4[4 * i + 1]},
                                 {planes4[4 * i + 2], planes4[4 * i + 3]}});
        s->force_split_frames = force_split_frames;
    });
}

// Replaces the initial state (AffineBody::q, q_dot) so drivers start from it.
int oracle_scene_set_state(void* sp, const double* q, const double* qdot) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        for (size_t b = 0; b < s->bodies.size(); ++b)
            for (int k = 0; k < 6; ++k) {
                s->bodies[b].q[k] = q[6 * b + k];
                s->bodies[b].q_dot[k] = qdot[6 * b + k];
            }
    });
}

int oracle_scene_set_force_split(void* sp, int body, double fx, double fy) {
    return guarded([&] { static_cast<Scene*>(sp)->replica_force_split[body] = {fx, fy}; });
}

int oracle_scene_counts(void* sp, int* n_bodies, int* n_verts) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        *n_bodies = static_cast<int>(s->bodies.size());
        int v = 0;
        for (const auto& b : s->bodies) v += b.vertex_count();
        *n_verts = v;
    });
}

// rest_xy[2V] flattened in body order, vert_start[n+1], q[6n], mass[n],
// M[36n] row-major, rest_area[n].
int oracle_scene_bodies(void* sp, double* rest_xy, int* vert_start, double* q, double* mass,
                        double* mm, double* rest_area) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        int v = 0;
        for (size_t b = 0; b < s->bodies.size(); ++b) {
            const AffineBody& body = s->bodies[b];
            vert_start[b] = v;
            for (const Vec2& x : body.flat) {
                rest_xy[2 * v] = x.x;
                rest_xy[2 * v + 1] = x.y;
                ++v;
            }
            for (int k = 0; k < 6; ++k) q[6 * b + k] = body.q[k];
            mass[b] = body.mass;
            std::memcpy(mm + 36 * b, body.mass_matrix.m, 36 * sizeof(double));
            rest_area[b] = body.rest_area;
        }
        vert_start[s->bodies.size()] = v;
    });
}

int oracle_broad_phase(void* sp, const double* q, const double* q_end, double margin,
                       const int* subset, int n_subset, int* pairs, int cap, int* count) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        const int n = static_cast<int>(s->bodies.size());
        const Configs qa = to_configs(q, n);
        std::vector<ContactPair> out;
        if (q_end) {
            const Configs qe = to_configs(q_end, n);
            out = broad_phase_swept(s->bodies, qa, qe, margin, to_vec(subset, n_subset));
        } else {
            out = broad_phase(s->bodies, qa, margin, to_vec(subset, n_subset));
        }
        write_pairs(out, pairs, nullptr, cap, count);
    });
}

int oracle_narrow_phase(void* sp, const double* q, const int* cand, int n_cand, double d_hat,
                        int* out_pairs, double* out_d, int* count) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        const Configs qa = to_configs(q, static_cast<int>(s->bodies.size()));
        const auto out = narrow_phase(read_pairs(cand, n_cand), s->bodies, qa, d_hat);
        write_pairs(out, out_pairs, out_d, n_cand, count);
    });
}

int oracle_ccd_toi(void* sp, const double* q0, const double* q1, const int* subset,
                   int n_subset, double* toi) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        const int n = static_cast<int>(s->bodies.size());
        *toi = ccd_toi_scene(s->bodies, to_configs(q0, n), to_configs(q1, n),
                             to_vec(subset, n_subset));
    });
}

int oracle_ccd_toi_pairs(void* sp, const double* q0, const double* q1, const int* cand,
                         int n_cand, double* toi) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        const int n = static_cast<int>(s->bodies.size());
        *toi = ccd_toi(s->bodies, to_configs(q0, n), to_configs(q1, n), read_pairs(cand, n_cand));
    });
}

int oracle_holder_masks(void* sp, const double* q, int n_planes, const double* planes4,
                        double w, uint32_t* masks) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        std::vector<Plane> pl;
        for (int i = 0; i < n_planes; ++i)
            pl.push_back({{planes4[4 * i], planes4[4 * i + 1]}, {planes4[4 * i + 2], planes4[4 * i + 3]}});
        const uint32_t all = (n_planes + 1) >= 32 ? 0xffffffffu : ((1u << (n_planes + 1)) - 1u);
        for (size_t b = 0; b < s->bodies.size(); ++b) {
            Vec6 qq;
            for (int k = 0; k < 6; ++k) qq[k] = q[6 * b + k];
            masks[b] = s->bodies[b].is_static ? all : body_holder_mask(s->bodies[b], qq, pl, w);
        }
    });
}

int oracle_max_vertex_speed(void* sp, const double* qdot, double* out) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        for (size_t b = 0; b < s->bodies.size(); ++b) {
            Vec6 v;
            for (int k = 0; k < 6; ++k) v[k] = qdot[6 * b + k];
            out[b] = max_vertex_speed(s->bodies[b], v);
        }
    });
}

int oracle_intersection_test(void* sp, const double* q, const int* subset, int n_subset,
                             int* result) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        *result = intersection_test(s->bodies, to_configs(q, static_cast<int>(s->bodies.size())),
                                    to_vec(subset, n_subset))
                      ? 1
                      : 0;
    });
}

int oracle_min_pair_distance(void* sp, const double* q, const int* subset, int n_subset,
                             int skip_static_pairs, double* out) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        *out = min_pair_distance(s->bodies, to_configs(q, static_cast<int>(s->bodies.size())),
                                 to_vec(subset, n_subset), skip_static_pairs != 0);
    });
}

int oracle_predicted_position(void* sp, const double* q, const double* qdot, const double* f,
                              double h, double* out) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        for (size_t b = 0; b < s->bodies.size(); ++b) {
            Vec6 qq, vv, ff;
            for (int k = 0; k < 6; ++k) {
                qq[k] = q[6 * b + k];
                vv[k] = qdot[6 * b + k];
                ff[k] = f[6 * b + k];
            }
            const Vec6 r = s->bodies[b].is_static
                               ? qq
                               : predicted_position(qq, vv, ff, h, s->bodies[b].mass_matrix);
            for (int k = 0; k < 6; ++k) out[6 * b + k] = r[k];
        }
    });
}

int oracle_point_edge_distance(const double* x6, int with_hess, double* d, double* grad6,
                               double* hess36) {
    return guarded([&] {
        const PointEdgeDistance r =
            point_edge_distance({x6[0], x6[1]}, {x6[2], x6[3]}, {x6[4], x6[5]}, with_hess != 0);
        *d = r.d;
        for (int k = 0; k < 6; ++k) grad6[k] = r.grad[k];
        std::memcpy(hess36, r.hess.m, 36 * sizeof(double));
    });
}

int oracle_barrier(double d, double d_hat, double kappa, double* out3) {
    return guarded([&] {
        const BarrierValue b = barrier_energy(d, d_hat, kappa);
        out3[0] = b.value;
        out3[1] = b.dvalue;
        out3[2] = b.ddvalue;
    });
}

int oracle_inertia_energy(const double* q, const double* qt, const double* m36, double* val,
                          double* grad6) {
    return guarded([&] {
        Vec6 a, b;
        Mat6 m;
        for (int k = 0; k < 6; ++k) {
            a[k] = q[k];
            b[k] = qt[k];
        }
        std::memcpy(m.m, m36, 36 * sizeof(double));
        const BodyEnergy e = inertia_energy(a, b, m);
        *val = e.value;
        for (int k = 0; k < 6; ++k) grad6[k] = e.grad[k];
    });
}

int oracle_arap_energy(const double* q, double kappa, double area, double* val, double* grad6,
                       double* hess36) {
    return guarded([&] {
        Vec6 a;
        for (int k = 0; k < 6; ++k) a[k] = q[k];
        const BodyEnergy e = arap_energy(a, kappa, area);
        *val = e.value;
        for (int k = 0; k < 6; ++k) grad6[k] = e.grad[k];
        std::memcpy(hess36, e.hess.m, 36 * sizeof(double));
    });
}

int oracle_contact_energy(void* sp, const double* q, int a, int b, int v, int e, double d_hat,
                          double kappa, double* val, double* grad12, double* hess144) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        Vec6 qa, qb;
        for (int k = 0; k < 6; ++k) {
            qa[k] = q[6 * a + k];
            qb[k] = q[6 * b + k];
        }
        const PairEnergy r =
            contact_energy(s->bodies[a], qa, s->bodies[b], qb, v, e, d_hat, kappa);
        *val = r.value;
        for (int k = 0; k < 12; ++k) grad12[k] = r.grad[k];
        std::memcpy(hess144, r.hess.m, 144 * sizeof(double));
    });
}

int oracle_clamp_psd(int n, const double* in, double* out) {
    return guarded([&] {
        if (n == 6) {
            Mat6 m;
            std::memcpy(m.m, in, 36 * sizeof(double));
            const Mat6 r = clamp_psd<6>(m);
            std::memcpy(out, r.m, 36 * sizeof(double));
        } else if (n == 12) {
            Mat12 m;
            std::memcpy(m.m, in, 144 * sizeof(double));
            const Mat12 r = clamp_psd<12>(m);
            std::memcpy(out, r.m, 144 * sizeof(double));
        } else {
            throw Error("clamp_psd: n must be 6 or 12");
        }
    });
}

// Objective evaluation. mode 0: value only (with anchors), 1: value without
// anchors, 2: derivatives (dense hessian out, n_dof^2), 3: derivatives
// without PSD projection.
int oracle_objective(void* sp, int n_local, const int* local, const double* kappa,
                     const double* q_tilde, int n_anchor, const int* anchor_body,
                     const double* anchor_zu, const double* anchor_rho,
                     const uint32_t* holder_mask, const double* sim8, const double* q, int mode,
                     double* value, double* grad, double* hess_dense, int* n_dofs,
                     int* active, int* candidates) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        const LocalObjective obj = make_objective(s, n_local, local, kappa, q_tilde, n_anchor,
                                                  anchor_body, anchor_zu, anchor_rho,
                                                  holder_mask, sim8);
        const Configs qq = to_configs(q, static_cast<int>(s->bodies.size()));
        *n_dofs = obj.num_dofs();
        if (mode <= 1) {
            *value = obj.value(qq, mode == 0);
            obj.contact_counts(qq, *active, *candidates);
            return;
        }
        const auto der = obj.derivatives(qq, mode == 2);
        *value = der.value;
        *active = der.active_contacts;
        *candidates = der.candidate_pairs;
        const int nd = obj.num_dofs();
        if (grad)
            for (int i = 0; i < nd; ++i) grad[i] = der.grad[i];
        if (hess_dense) {
            for (int i = 0; i < nd * nd; ++i) hess_dense[i] = 0.0;
            for (int b = 0; b < der.hess.nb; ++b)
                for (int r = 0; r < 6; ++r)
                    for (int c = 0; c < 6; ++c)
                        hess_dense[(6 * b + r) * nd + 6 * b + c] = der.hess.diag[b](r, c);
            for (const auto& kv : der.hess.off)
                for (int r = 0; r < 6; ++r)
                    for (int c = 0; c < 6; ++c)
                        hess_dense[(6 * kv.first.first + r) * nd + 6 * kv.first.second + c] =
                            kv.second(r, c);
        }
    });
}

int oracle_newton_solve(void* sp, int n_local, const int* local, const double* kappa,
                        const double* q_tilde, int n_anchor, const int* anchor_body,
                        const double* anchor_zu, const double* anchor_rho,
                        const uint32_t* holder_mask, const double* sim8, double* q,
                        int max_iters, double tol, int* iterations, double* final_update,
                        int* converged, int* ls_steps) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        const LocalObjective obj = make_objective(s, n_local, local, kappa, q_tilde, n_anchor,
                                                  anchor_body, anchor_zu, anchor_rho,
                                                  holder_mask, sim8);
        Configs qq = to_configs(q, static_cast<int>(s->bodies.size()));
        NewtonOptions no;
        no.max_iters = max_iters;
        no.tol = tol;
        const NewtonReport r = newton_solve(obj, qq, no);
        from_configs(qq, q);
        *iterations = r.iterations;
        *final_update = r.final_update_inf;
        *converged = r.converged ? 1 : 0;
        *ls_steps = r.line_search_steps;
    });
}

// Runs N=1 (workers == 0: run_reference semantics) or the distributed
// semantics with `workers` partitions. Outputs: q_traj/qdot_traj [frames][6n],
// h[frames], stats [frames][5] (attempts, admm, newton, ls, h as double
// stored separately), trace rows [cap][8] (frame, attempt, k, dq, r, s, toi,
// sigma), rho_final[n].
int oracle_run(void* sp, int workers, int frames, double* q_traj, double* qdot_traj,
               double* h_traj, int* stats4, double* trace8, int trace_cap, int* trace_count,
               double* rho_final) {
    return guarded([&] {
        Scene* s = static_cast<Scene*>(sp);
        const Trajectory t = workers == 0 ? run_reference(*s, frames) : run_distributed(*s, workers, frames);
        const size_t n = s->bodies.size();
        for (size_t f = 0; f < t.q.size(); ++f) {
            from_configs(t.q[f], q_traj + f * 6 * n);
            from_configs(t.q_dot[f], qdot_traj + f * 6 * n);
            h_traj[f] = t.h[f];
            stats4[4 * f + 0] = t.stats[f].attempts;
            stats4[4 * f + 1] = t.stats[f].admm_iterations;
            stats4[4 * f + 2] = t.stats[f].newton_iterations;
            stats4[4 * f + 3] = t.stats[f].line_search_steps;
        }
        *trace_count = static_cast<int>(t.trace.size());
        for (size_t i = 0; i < t.trace.size() && static_cast<int>(i) < trace_cap; ++i) {
            const IterTrace& it = t.trace[i];
            double* r = trace8 + 8 * i;
            r[0] = it.frame;
            r[1] = it.attempt;
            r[2] = it.k;
            r[3] = it.dq_inf;
            r[4] = it.r_inf;
            r[5] = it.s_inf;
            r[6] = it.min_toi;
            r[7] = it.sigma;
        }
        if (rho_final) {
            for (size_t b = 0; b < n; ++b)
                rho_final[b] = b < t.rho_final.size() ? t.rho_final[b] : std::nan("");
        }
    });
}

} // extern "C"

// ---- consensus step (consensus.cpp:9-52, runtime.cpp:361-397) ----------------
// TEST INFRASTRUCTURE: n split bodies with two replicas each (lower holder
// first): z = consensus_update, u' = dual_update per replica, r = primal
// residual over both replicas, s = dual residual against z_prev, rho' =
// adapt_rho (skipped when adapt5[5] == 0).
extern "C" int oracle_consensus_step(int n, const double* q, const double* u, const double* rho,
                                     const double* z_prev, const double* rho0, const double* adapt6,
                                     double* z, double* u_new, double* r, double* s, double* rho_next) {
    using namespace oracle;
    return guarded([&] {
        AdaptParams ap;
        ap.beta = adapt6[0];
        ap.tau = adapt6[1];
        ap.mu = adapt6[2];
        ap.sigma_min = adapt6[3];
        ap.sigma_max = adapt6[4];
        ap.adapt_enabled = adapt6[5] != 0.0;
        for (int i = 0; i < n; ++i) {
            std::vector<Vec6> rq(2), rqu(2);
            for (int h = 0; h < 2; ++h)
                for (int c = 0; c < 6; ++c) {
                    rq[h][c] = q[12 * i + 6 * h + c];
                    rqu[h][c] = q[12 * i + 6 * h + c] + u[12 * i + 6 * h + c];
                }
            const Vec6 zi = consensus_update(rqu, {rho[i], rho[i]});
            Vec6 zp;
            for (int c = 0; c < 6; ++c) {
                z[6 * i + c] = zi[c];
                zp[c] = z_prev[6 * i + c];
            }
            for (int h = 0; h < 2; ++h) {
                Vec6 uh;
                for (int c = 0; c < 6; ++c) uh[c] = u[12 * i + 6 * h + c];
                const Vec6 un = dual_update(uh, rq[h], zi);
                for (int c = 0; c < 6; ++c) u_new[12 * i + 6 * h + c] = un[c];
            }
            r[i] = primal_residual_inf(rq, zi);
            s[i] = dual_residual_inf(zi, zp);
            rho_next[i] = ap.adapt_enabled ? adapt_rho(rho[i], r[i], s[i], ap, rho0[i]) : rho[i];
        }
    });
}

// consensus.cpp:9-21 with arbitrary replica weights: qu [n][6], rho [n].
extern "C" int oracle_consensus_update(int n, const double* qu, const double* rho, double* z) {
    return guarded([&] {
        std::vector<Vec6> v(n);
        for (int i = 0; i < n; ++i)
            for (int c = 0; c < 6; ++c) v[i][c] = qu[6 * i + c];
        const Vec6 zz = consensus_update(v, rho ? std::vector<double>(rho, rho + n) : std::vector<double>());
        for (int c = 0; c < 6; ++c) z[c] = zz[c];
    });
}

// consensus.cpp:38-52
extern "C" int oracle_init_rho(double mass, double beta, double* out) {
    return guarded([&] { *out = init_rho(mass, beta); });
}

extern "C" int oracle_adapt_rho(double rho, double r, double s, const double* adapt6, double rho0,
                                double* out) {
    return guarded([&] {
        AdaptParams ap;
        ap.beta = adapt6[0];
        ap.tau = adapt6[1];
        ap.mu = adapt6[2];
        ap.sigma_min = adapt6[3];
        ap.sigma_max = adapt6[4];
        ap.adapt_enabled = adapt6[5] != 0.0;
        *out = adapt_rho(rho, r, s, ap, rho0);
    });
}

// consensus.cpp:54-64
extern "C" int oracle_check_stopping(double dq, double r, double s, const double* tois, int n, double h,
                                     double l, double theta, int* end) {
    return guarded([&] {
        *end = check_stopping(dq, r, s, std::vector<double>(tois, tois + n), h, l, theta) ? 1 : 0;
    });
}

// consensus.hpp:60-87: events 0 = failed frame, 1 = committed frame.
extern "C" int oracle_timestep_apply(double h0, int max_halvings, const int* events, int n,
                                     double* h_after) {
    return guarded([&] {
        TimestepController ts(h0, max_halvings);
        for (int i = 0; i < n; ++i) {
            if (events[i] == 0) ts.on_frame_failed();
            else ts.on_frame_committed();
            h_after[i] = ts.h();
        }
    });
}

// partition.cpp:131-138 on two holder masks.
extern "C" int oracle_contact_replication(uint32_t mask_a, uint32_t mask_b, int* kc) {
    return guarded([&] {
        PartitionLayout L;
        L.holder_mask = {mask_a, mask_b};
        *kc = contact_replication(L, 0, 1);
    });
}
