// TEST INFRASTRUCTURE ONLY (see oracle.hpp). Restates proj/src/partition.cpp,
// consensus.cpp, the N=1 driver run_reference (sim.cpp:186-249) and the
// distributed runtime semantics (runtime.cpp:110-694) in the shape of the
// sequential replay oracle (tests/support/replay.cpp:11-169), extended with
// what the replay lacks: w from the current q_dot (runtime.cpp:556-560),
// the replica force split (runtime.cpp:252-262), per-worker z/u/rho state and
// AbortRetry/Fail with time-step halving (runtime.cpp:603-642).
#include "oracle.hpp"

#include <algorithm>
#include <bit>
#include <cstdlib>
#include <exception>
#include <limits>
#include <thread>

namespace oracle {

// One std::thread per worker, as the reference runs its workers
// (sim.cpp:281-322): fn(i) for i in [0, n) on up to
// worker_threads() threads. Each worker's work touches only its own state;
// results are combined by the caller in worker order, so the outcome is
// independent of the thread count. ORACLE_THREADS=1 runs sequentially.
int worker_threads() {
    if (const char* e = std::getenv("ORACLE_THREADS")) return std::max(1, std::atoi(e));
    return std::max(1u, std::thread::hardware_concurrency());
}

template <typename Fn>
void for_workers(int n, Fn&& fn) {
    const int t = std::min(n, worker_threads());
    if (t <= 1) {
        for (int i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::exception_ptr> errs(n);
    std::vector<std::thread> pool;
    for (int k = 0; k < t; ++k)
        pool.emplace_back([&, k] {
            for (int i = k; i < n; i += t) {
                try {
                    fn(i);
                } catch (...) {
                    errs[i] = std::current_exception();
                }
            }
        });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e); // the lowest worker's error, like a sequential run
}

// partition.cpp:9-11
double overlap_width(double v_max, double h, double w_min) {
    return std::max(2.0 * v_max * h, w_min);
}

int PartitionLayout::kappa_b(int body) const { return std::popcount(holder_mask[body]); }

std::vector<int> PartitionLayout::holders_of(int body) const {
    std::vector<int> out;
    for (int i = 0; i < num_workers; ++i)
        if (holder_mask[body] & (1u << i)) out.push_back(i);
    return out;
}

// partition.cpp:36-67
uint32_t body_holder_mask(const AffineBody& body, const Vec6& q,
                          const std::vector<Plane>& planes, double w) {
    const Aabb box = body_aabb(body, q);
    int hit = -1;
    for (size_t k = 0; k < planes.size(); ++k) {
        double lo = std::numeric_limits<double>::max();
        double hi = -lo;
        for (int corner = 0; corner < 4; ++corner) {
            const Vec2 c{(corner & 1) ? box.hi.x : box.lo.x, (corner & 2) ? box.hi.y : box.lo.y};
            const double s = dot(c - planes[k].point, planes[k].normal);
            lo = std::min(lo, s);
            hi = std::max(hi, s);
        }
        if (lo <= w / 2.0 && hi >= -w / 2.0) {
            if (hit >= 0)
                throw Error("partition: body AABB wider than a region (straddles two interfaces)");
            hit = static_cast<int>(k);
        }
    }
    if (hit >= 0) return (1u << hit) | (1u << (hit + 1));
    const Vec2 c{q[0], q[1]};
    int region = 0;
    for (const Plane& p : planes)
        if (dot(c - p.point, p.normal) <= 0.0) ++region;
    return 1u << region;
}

// partition.cpp:69-129
PartitionLayout partition_scene(const std::vector<AffineBody>& bodies, const Configs& q,
                                const std::vector<Plane>& planes, int nw, double h,
                                double w_min, double v_max_override) {
    if (nw < 1 || nw > 32) throw Error("partition_scene: worker count must be in [1, 32]");
    if (static_cast<int>(planes.size()) != nw - 1)
        throw Error("partition_scene: need exactly num_workers - 1 planes");
    PartitionLayout L;
    L.num_workers = nw;
    L.planes = planes;
    for (const Plane& p : planes)
        if (std::abs(norm(p.normal) - 1.0) > 1e-9)
            throw Error("partition_scene: plane normal must be unit length");
    double v_max = v_max_override;
    if (v_max < 0.0) {
        v_max = 0.0;
        for (const AffineBody& b : bodies)
            if (!b.is_static) v_max = std::max(v_max, max_vertex_speed(b, b.q_dot));
    }
    L.w = overlap_width(v_max, h, w_min);
    const uint32_t all = nw == 32 ? 0xffffffffu : ((1u << nw) - 1u);
    L.holder_mask.assign(bodies.size(), 0);
    L.internal_bodies.resize(nw);
    L.shared_bodies.resize(nw);
    L.local_bodies.resize(nw);
    L.neighbors.resize(nw);
    for (size_t b = 0; b < bodies.size(); ++b)
        L.holder_mask[b] = bodies[b].is_static ? all : body_holder_mask(bodies[b], q[b], planes, L.w);
    for (size_t b = 0; b < bodies.size(); ++b) {
        const uint32_t m = L.holder_mask[b];
        for (int i = 0; i < nw; ++i) {
            if (!(m & (1u << i))) continue;
            L.local_bodies[i].push_back(static_cast<int>(b));
            if (bodies[b].is_static) continue;
            if (std::popcount(m) == 1)
                L.internal_bodies[i].push_back(static_cast<int>(b));
            else
                L.shared_bodies[i].push_back(static_cast<int>(b));
        }
    }
    for (int k = 0; k + 1 < nw; ++k) {
        L.neighbors[k].push_back(k + 1);
        L.neighbors[k + 1].push_back(k);
    }
    for (auto& n : L.neighbors) std::sort(n.begin(), n.end());
    return L;
}

// partition.cpp:131-138
int contact_replication(const PartitionLayout& L, int a, int b) {
    const int kc = std::popcount(L.holder_mask[a] & L.holder_mask[b]);
    if (kc == 0)
        throw Error("contact_replication: no worker sees both bodies (overlap width too small)");
    return kc;
}

// consensus.cpp:9-21
Vec6 consensus_update(const std::vector<Vec6>& qu, const std::vector<double>& rho) {
    if (qu.empty() || qu.size() != rho.size())
        throw Error("consensus_update: need matching, non-empty replica lists");
    Vec6 num = zero6();
    double den = 0.0;
    for (size_t i = 0; i < qu.size(); ++i) {
        if (!(rho[i] > 0.0)) throw Error("consensus_update: rho must be > 0");
        for (int k = 0; k < 6; ++k) num[k] += rho[i] * qu[i][k];
        den += rho[i];
    }
    Vec6 z;
    for (int k = 0; k < 6; ++k) z[k] = num[k] / den;
    return z;
}

// consensus.cpp:23-25
Vec6 dual_update(const Vec6& u, const Vec6& q, const Vec6& z) {
    Vec6 o;
    for (int k = 0; k < 6; ++k) o[k] = (u[k] + q[k]) - z[k];
    return o;
}

// consensus.cpp:27-36
double primal_residual_inf(const std::vector<Vec6>& reps, const Vec6& z) {
    double best = 0.0;
    for (const Vec6& q : reps)
        for (int k = 0; k < 6; ++k) best = std::max(best, std::abs(q[k] - z[k]));
    return best;
}

double dual_residual_inf(const Vec6& zn, const Vec6& zp) {
    double best = 0.0;
    for (int k = 0; k < 6; ++k) best = std::max(best, std::abs(zn[k] - zp[k]));
    return best;
}

// consensus.cpp:38-42
double init_rho(double mass, double beta) {
    if (!(mass > 0.0) || !(beta > 0.0)) throw Error("init_rho: mass and beta must be > 0");
    return beta * mass;
}

// consensus.cpp:44-52
double adapt_rho(double rho, double r, double s, const AdaptParams& p, double rho0) {
    double next = rho;
    if (r > p.mu * s)
        next = p.tau * rho;
    else if (s > p.mu * r)
        next = rho / p.tau;
    return std::clamp(next, p.sigma_min * rho0, p.sigma_max * rho0);
}

// consensus.cpp:54-64
bool check_stopping(double dq, double r, double s, const std::vector<double>& tois, double h,
                    double l, double theta) {
    const double norm_ = h * l;
    bool end = dq / norm_ < theta && r / norm_ < theta && s / norm_ < theta;
    for (double t : tois)
        if (t != 1.0) end = false;
    return end;
}

// consensus.cpp:66-75
double merge_ccd_gate(const std::vector<AffineBody>& bodies, const Configs& ql,
                      const std::vector<int>& shared, const std::vector<Vec6>& z,
                      const std::vector<int>& local_subset) {
    if (shared.size() != z.size()) throw Error("merge_ccd_gate: shared/z size mismatch");
    Configs merged = ql;
    for (size_t i = 0; i < shared.size(); ++i) merged[shared[i]] = z[i];
    return ccd_toi_scene(bodies, ql, merged, local_subset);
}

// consensus.cpp:77-86
void finalize_merge(Configs& q, Configs& qd, const Configs& q_start, double h,
                    const std::vector<int>& shared, const std::vector<Vec6>& z,
                    const std::vector<int>& dyn, bool gate_passed) {
    if (!gate_passed) throw Error("finalize_merge: called without a passed merge gate");
    if (shared.size() != z.size()) throw Error("finalize_merge: shared/z size mismatch");
    for (size_t i = 0; i < shared.size(); ++i) q[shared[i]] = z[i];
    for (int b : dyn)
        for (int k = 0; k < 6; ++k) qd[b][k] = (q[b][k] - q_start[b][k]) / h;
}

Configs Scene::initial_configs() const {
    Configs q(bodies.size());
    for (size_t i = 0; i < bodies.size(); ++i) q[i] = bodies[i].q;
    return q;
}

Configs Scene::initial_velocities() const {
    Configs v(bodies.size());
    for (size_t i = 0; i < bodies.size(); ++i) v[i] = bodies[i].q_dot;
    return v;
}

// sim.cpp:186-249
Trajectory run_reference(const Scene& scene, int frames) {
    const auto& bodies = scene.bodies;
    const int nb = static_cast<int>(bodies.size());
    Configs q = scene.initial_configs(), qd = scene.initial_velocities();
    std::vector<int> local_all, local_dyn;
    std::vector<uint32_t> mask(nb, 1u);
    for (int b = 0; b < nb; ++b) {
        local_all.push_back(b);
        if (!bodies[b].is_static) local_dyn.push_back(b);
    }
    const SimParams& P = scene.params;
    NewtonOptions no;
    no.max_iters = scene.newton_cap;
    no.tol = P.theta * P.h * P.scene_scale;
    Trajectory traj;
    for (int f = 0; f < frames; ++f) {
        const Configs q_start = q;
        std::vector<Vec6> qt;
        std::vector<double> kap;
        for (int b : local_all) {
            kap.push_back(1.0);
            qt.push_back(bodies[b].is_static
                             ? q[b]
                             : predicted_position(q[b], qd[b], gravity_force(bodies[b], P.gravity),
                                                  P.h, bodies[b].mass_matrix));
        }
        FrameStat st;
        st.h = P.h;
        double dq_inf = 0.0;
        bool ended = false;
        for (int k = 1; k <= scene.admm_max_iterations; ++k) {
            if (k > 1) {
                const bool end = check_stopping(dq_inf, 0.0, 0.0, {1.0}, P.h, P.scene_scale, P.theta);
                IterTrace it;
                it.frame = f;
                it.k = k;
                it.dq_inf = dq_inf;
                it.sigma = end ? 1 : 0;
                traj.trace.push_back(it);
                if (end) {
                    ended = true;
                    st.admm_iterations = k;
                    break;
                }
            }
            const LocalObjective obj =
                LocalObjective::assemble(bodies, local_all, kap, qt, {}, mask, P);
            const Configs q_before = q;
            const NewtonReport r = newton_solve(obj, q, no);
            st.newton_iterations += r.iterations;
            st.line_search_steps += r.line_search_steps;
            dq_inf = obj.config_delta_inf(q, q_before);
        }
        if (!ended) throw Error("run_reference: Newton stepping failed to settle");
        finalize_merge(q, qd, q_start, P.h, {}, {}, local_dyn, true);
        traj.q.push_back(q);
        traj.q_dot.push_back(qd);
        traj.h.push_back(P.h);
        traj.stats.push_back(st);
    }
    return traj;
}

// runtime.cpp:110-694 with global replicated state.
Trajectory run_distributed(const Scene& scene, int nw, int frames) {
    const auto& bodies = scene.bodies;
    const int nb = static_cast<int>(bodies.size());
    if (nw < 1 || nw > 32) throw Error("run_distributed: worker count must be in [1, 32]");
    if (static_cast<int>(scene.planes.size()) < nw - 1)
        throw Error("controller: scene has too few interface planes");
    const std::vector<Plane> planes(scene.planes.begin(), scene.planes.begin() + (nw - 1));
    const uint32_t everyone = nw == 32 ? 0xffffffffu : ((1u << nw) - 1u);
    Configs q = scene.initial_configs(), qd = scene.initial_velocities();
    std::vector<double> rho_carry(nb, std::numeric_limits<double>::quiet_NaN());
    TimestepController ts(scene.params.h, scene.max_halvings);
    Trajectory traj;

    for (int f = 0; f < frames; ++f) {
        int attempt = 0;
        while (true) {
            FrameStat st;
            st.attempts = attempt + 1;
            const double h = ts.h();
            st.h = h;
            double v_max = 0.0; // runtime.cpp:556-560
            for (int b = 0; b < nb; ++b)
                if (!bodies[b].is_static) v_max = std::max(v_max, max_vertex_speed(bodies[b], qd[b]));
            const double w = overlap_width(v_max, h, scene.w_min);
            std::vector<uint32_t> mask(nb, 0);
            for (int b = 0; b < nb; ++b)
                mask[b] = bodies[b].is_static ? everyone : body_holder_mask(bodies[b], q[b], planes, w);

            SimParams fp = scene.params;
            fp.h = h;
            NewtonOptions no;
            no.max_iters = scene.newton_cap;
            no.tol = fp.theta * h * fp.scene_scale;

            struct Worker {
                std::vector<int> local_all, local_dyn, shared;
                std::vector<Vec6> qt_of;
                std::vector<Vec6> z, u;
                std::vector<double> rho, rho0;
                Configs wq;
                double dq = 0.0;
            };
            std::vector<Worker> W(nw);
            for (int i = 0; i < nw; ++i) {
                Worker& wk = W[i];
                wk.wq = q;
                wk.qt_of.assign(nb, zero6());
                for (int b = 0; b < nb; ++b) {
                    if (!(mask[b] & (1u << i))) continue;
                    wk.local_all.push_back(b);
                    if (bodies[b].is_static) {
                        wk.qt_of[b] = q[b];
                        continue;
                    }
                    wk.local_dyn.push_back(b);
                    if (std::popcount(mask[b]) >= 2) wk.shared.push_back(b);
                    Vec6 fext = gravity_force(bodies[b], fp.gravity);
                    const auto split = scene.replica_force_split.find(b);
                    const bool active = scene.force_split_frames < 0 || f < scene.force_split_frames;
                    if (split != scene.replica_force_split.end() && active &&
                        std::popcount(mask[b]) >= 2) {
                        const int lowest = std::countr_zero(mask[b]);
                        const double sign = i == lowest ? 1.0 : -1.0;
                        fext[0] += sign * split->second.x;
                        fext[1] += sign * split->second.y;
                    }
                    wk.qt_of[b] = predicted_position(q[b], qd[b], fext, h, bodies[b].mass_matrix);
                }
                const size_t ns = wk.shared.size();
                wk.z.resize(ns);
                wk.u.assign(ns, zero6());
                wk.rho.resize(ns);
                wk.rho0.resize(ns);
                for (size_t s = 0; s < ns; ++s) {
                    const int b = wk.shared[s];
                    wk.z[s] = wk.qt_of[b];
                    wk.rho0[s] = init_rho(bodies[b].mass, scene.adapt.beta);
                    wk.rho[s] = std::isnan(rho_carry[b]) ? wk.rho0[s] : rho_carry[b];
                }
            }
            auto slot = [&](int i, int b) {
                const auto& sh = W[i].shared;
                const auto it = std::lower_bound(sh.begin(), sh.end(), b);
                if (it == sh.end() || *it != b) throw Error("protocol error: missing replica state");
                return static_cast<int>(it - sh.begin());
            };

            bool ended = false, retry = false;
            std::vector<std::vector<Vec6>> z_commit(nw);
            for (int k = 1; k <= scene.admm_max_iterations; ++k) {
                if (k > 1) {
                    // consensus / dual / residual per worker (runtime.cpp:361-397)
                    std::vector<std::vector<Vec6>> z_next(nw);
                    std::vector<std::vector<double>> rb(nw), sb(nw);
                    std::vector<double> r_loc(nw, 0.0), s_loc(nw, 0.0), toi(nw, 1.0);
                    std::vector<std::vector<Vec6>> u_new(nw);
                    for (int i = 0; i < nw; ++i) {
                        Worker& wk = W[i];
                        const size_t ns = wk.shared.size();
                        z_next[i].resize(ns);
                        rb[i].assign(ns, 0.0);
                        sb[i].assign(ns, 0.0);
                        u_new[i] = wk.u;
                        for (size_t s = 0; s < ns; ++s) {
                            const int b = wk.shared[s];
                            std::vector<Vec6> rq, rqu;
                            std::vector<double> rr;
                            for (int hw = 0; hw < nw; ++hw) {
                                if (!(mask[b] & (1u << hw))) continue;
                                const int hs = slot(hw, b);
                                if (W[hw].rho[hs] != wk.rho[s])
                                    throw Error("protocol error: replica rho mismatch");
                                Vec6 qu;
                                for (int c = 0; c < 6; ++c) qu[c] = W[hw].wq[b][c] + W[hw].u[hs][c];
                                rq.push_back(W[hw].wq[b]);
                                rqu.push_back(qu);
                                rr.push_back(W[hw].rho[hs]);
                            }
                            z_next[i][s] = consensus_update(rqu, rr);
                            u_new[i][s] = dual_update(wk.u[s], wk.wq[b], z_next[i][s]);
                            rb[i][s] = primal_residual_inf(rq, z_next[i][s]);
                            sb[i][s] = dual_residual_inf(z_next[i][s], wk.z[s]);
                            r_loc[i] = std::max(r_loc[i], rb[i][s]);
                            s_loc[i] = std::max(s_loc[i], sb[i][s]);
                        }
                    }
                    for (int i = 0; i < nw; ++i) W[i].u = u_new[i];
                    for_workers(nw, [&](int i) {
                        toi[i] = merge_ccd_gate(bodies, W[i].wq, W[i].shared, z_next[i], W[i].local_all);
                    });
                    // controller (runtime.cpp:586-619)
                    IterTrace it;
                    it.frame = f;
                    it.attempt = attempt;
                    it.k = k;
                    it.min_toi = 1.0;
                    for (int i = 0; i < nw; ++i) {
                        it.dq_inf = std::max(it.dq_inf, W[i].dq);
                        it.r_inf = std::max(it.r_inf, r_loc[i]);
                        it.s_inf = std::max(it.s_inf, s_loc[i]);
                        it.min_toi = std::min(it.min_toi, toi[i]);
                    }
                    const bool end = check_stopping(it.dq_inf, it.r_inf, it.s_inf, toi, h,
                                                    fp.scene_scale, fp.theta);
                    if (end) {
                        it.sigma = 1;
                    } else if (k == scene.admm_max_iterations) {
                        it.sigma = ts.halvings() < scene.max_halvings ? 2 : 3;
                    } else {
                        it.sigma = 0;
                    }
                    traj.trace.push_back(it);
                    if (it.sigma == 1) {
                        z_commit = z_next;
                        st.admm_iterations = k;
                        ended = true;
                        break;
                    }
                    if (it.sigma == 3)
                        throw Error("frame failed: halving budget exhausted with a blocked merge");
                    if (it.sigma == 2) {
                        ts.on_frame_failed();
                        retry = true;
                        break;
                    }
                    if (scene.adapt.adapt_enabled)
                        for (int i = 0; i < nw; ++i)
                            for (size_t s = 0; s < W[i].shared.size(); ++s)
                                W[i].rho[s] = adapt_rho(W[i].rho[s], rb[i][s], sb[i][s],
                                                        scene.adapt, W[i].rho0[s]);
                    for (int i = 0; i < nw; ++i) W[i].z = z_next[i];
                }
                // local solves (runtime.cpp:465-475), one thread per worker
                std::vector<NewtonReport> reps(nw);
                for_workers(nw, [&](int i) {
                    Worker& wk = W[i];
                    std::vector<double> kap;
                    std::vector<Vec6> qt;
                    for (int b : wk.local_all) {
                        kap.push_back(std::popcount(mask[b]));
                        qt.push_back(wk.qt_of[b]);
                    }
                    std::vector<SharedAnchor> an;
                    for (size_t s = 0; s < wk.shared.size(); ++s) {
                        SharedAnchor a;
                        a.body = wk.shared[s];
                        a.z = wk.z[s];
                        a.u = wk.u[s];
                        a.rho = wk.rho[s];
                        an.push_back(a);
                    }
                    std::vector<uint32_t> hm(nb, 0);
                    for (int b : wk.local_all) hm[b] = mask[b];
                    const LocalObjective obj =
                        LocalObjective::assemble(bodies, wk.local_all, kap, qt, an, hm, fp);
                    const Configs before = wk.wq;
                    reps[i] = newton_solve(obj, wk.wq, no);
                    wk.dq = obj.config_delta_inf(wk.wq, before);
                });
                for (int i = 0; i < nw; ++i) {
                    st.newton_iterations += reps[i].iterations;
                    st.line_search_steps += reps[i].line_search_steps;
                }
            }
            if (retry) {
                ++attempt;
                continue;
            }
            if (!ended) throw Error("controller: frame ended without a decision");
            // commit (runtime.cpp:481-506, 646-677)
            std::fill(rho_carry.begin(), rho_carry.end(), std::numeric_limits<double>::quiet_NaN());
            Configs qn = q, qdn = qd;
            for (int i = 0; i < nw; ++i) {
                Worker& wk = W[i];
                for (size_t s = 0; s < wk.shared.size(); ++s)
                    if (std::countr_zero(mask[wk.shared[s]]) == i) rho_carry[wk.shared[s]] = wk.rho[s];
                Configs qi = wk.wq, qdi = qd;
                finalize_merge(qi, qdi, q, h, wk.shared, z_commit[i], wk.local_dyn, true);
                for (int b : wk.local_dyn) {
                    if (std::countr_zero(mask[b]) != i) continue;
                    qn[b] = qi[b];
                    qdn[b] = qdi[b];
                }
            }
            q = qn;
            qd = qdn;
            ts.on_frame_committed();
            traj.q.push_back(q);
            traj.q_dot.push_back(qd);
            traj.h.push_back(h);
            traj.stats.push_back(st);
            break;
        }
    }
    traj.rho_final = rho_carry;
    return traj;
}

} // namespace oracle
