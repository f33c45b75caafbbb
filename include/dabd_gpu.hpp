/* dabd_gpu.hpp: the reference's C++ scene / step / parameter API over the C ABI.
 *
 * Header-only C++17 adapter in the vocabulary of the reference
 * (proj/include/dabd/{params,scene,sim,partition}.hpp) so a host program written
 * against `dabd::` drops onto the B200 path by switching the namespace to
 * `dabd::gpu::` and linking libdabd_gpu.so. Every computation runs in the
 * sm_100a kernels behind include/dabd_gpu.h; this file only marshals host
 * buffers, owns the handles (RAII) and writes the reference's output files.
 *
 *   reference (file:line, /root/reference/proj)          here
 *   SimParams, AdaptParams   include/dabd/params.hpp:8-41  SimParams, AdaptParams
 *   Plane                    include/dabd/partition.hpp:13-16  Plane
 *   SceneData                include/dabd/scene.hpp:15-56  SceneData (bodies as world loops, the
 *                                                          form scene JSON and make_affine_body take)
 *   make_scenario            src/scene.cpp:345-557         make_scenario (funnel-analog,
 *                                                          drop-grid-N, density-sweep-R, pile-1k)
 *   run_reference            src/sim.cpp:186-249           run_reference
 *   run_distributed          src/sim.cpp:264-432           run_distributed (all workers on one GPU)
 *   write_snapshot / read_snapshot / load_trajectory
 *                            src/sim.cpp:34-108            same names, same byte layout
 *   write_metrics_csv        src/sim.cpp:110-137           same name, same header and columns
 *   mse_to_reference         src/sim.cpp:14-28             same name
 *   SceneData::balance       scene.hpp:31-32, balance.hpp:24-29  (planes move between frames)
 *   broad_phase, ccd_toi_scene, body_holder_mask, intersection_test
 *                            include/dabd/geometry.hpp:47-74, partition.hpp:43-45, geometry.cpp:389
 *
 * Errors: a non-OK status from the C ABI throws dabd::gpu::Error carrying
 * dabd_gpu_last_error(), like dabd::Error (types.hpp:41-44).
 */
#ifndef DABD_GPU_HPP
#define DABD_GPU_HPP

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dabd_gpu.h"

namespace dabd {
namespace gpu {

using Vec2 = std::array<double, 2>;
using Vec6 = std::array<double, 6>;  // q = [p_x, p_y, A00, A01, A10, A11] (types.hpp:18)
using Loop = std::vector<Vec2>;
using Configs = std::vector<Vec6>;

class Error : public std::runtime_error {
  public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

inline void check(dabd_gpu_status s) {
    if (s != DABD_GPU_OK) throw Error(std::string("dabd_gpu: ") + dabd_gpu_last_error());
}

/* params.hpp:8-23, same defaults. */
struct SimParams {
    double h = 0.01;
    Vec2 gravity{0.0, -9.81};
    double arap_stiffness = 1e6;
    double barrier_stiffness = 1e4;
    double d_hat = 0.01;
    double theta = 1e-3;
    double scene_scale = 1.0;
};

/* params.hpp:26-41. */
struct AdaptParams {
    double beta = 1.0, tau = 2.0, mu = 5.0, sigma_min = 1e-3, sigma_max = 1e3;
    bool adapt_enabled = true;
};

/* partition.hpp:13-16: interface plane between workers k and k+1. */
struct Plane {
    Vec2 point{0.0, 0.0};
    Vec2 normal{1.0, 0.0};
};

/* One body as scene.cpp:81-98 reads it: world-space loops, built by
 * make_affine_body (body.cpp:96-118) on the library side. */
struct Body {
    std::vector<Loop> loops;
    double density = 1000.0;
    Vec6 velocity{0, 0, 0, 0, 0, 0};
    bool is_static = false;
    double arap_scale = 1.0;
};

/* scene.hpp:15-56. */
struct SceneData {
    std::string name = "scene";
    std::vector<Body> bodies;
    SimParams params;
    AdaptParams adapt;
    std::vector<Plane> planes;
    double w_min = 0.1;
    int frames = 100;
    int admm_max_iterations = 300;
    int newton_cap = 32;
    int max_halvings = 4;
    bool balance_enabled = false;
    struct BalanceOptions { // balance.hpp:24-29
        double kp = 0.0, kd = 0.0, smoothing = 0.5, dp_max = 0.0;
    } balance;
    std::map<int, Vec2> replica_force_split;
    int force_split_frames = -1;
    uint64_t seed = 0;

    int dynamic_count() const {
        int n = 0;
        for (const Body& b : bodies) n += b.is_static ? 0 : 1;
        return n;
    }
};

/* sim.hpp:13-17. */
struct Trajectory {
    std::vector<Configs> q;
    std::vector<Configs> q_dot;
    std::vector<double> h;
};

/* sim.hpp:25-40. Partitions batched in one context share one host clock, so
 * every worker column of a commit row carries the context's frame compute /
 * sync seconds (dabd_gpu_frame_stats t_frame - t_sync, t_sync); the
 * iteration rows leave them empty. */
struct MetricsRow {
    int64_t frame = 0;
    int32_t attempt = 0;
    int32_t k = 0;
    double r_inf = 0.0;
    double s_inf = 0.0;
    double min_toi = 1.0;
    int active_contacts = 0;
    int candidate_pairs = 0;
    double mse = std::numeric_limits<double>::quiet_NaN();
    bool commit_row = false;
    std::vector<double> dq_inf;
    std::vector<int> newton_iters;
    std::vector<double> t_compute;
    std::vector<double> t_sync;
};

/* sim.hpp:42-53 plus the device counters of dabd_gpu_frame_stats. */
struct FrameStats {
    int64_t frame = 0;
    int attempts = 1;
    double h = 0.0;
    int admm_iterations = 0;
    int newton_iterations = 0;
    int line_search_steps = 0;
    int pcg_iterations = 0;
    int max_contacts = 0;
    int max_candidates = 0;
    int exact_retries = 0;
    int capacity_retries = 0;
    double t_solve = 0.0, t_coll = 0.0, t_sync = 0.0, t_frame = 0.0; // sim.hpp:44-47
};

/* sim.hpp:55-61. */
struct RunResult {
    Trajectory trajectory;
    std::vector<MetricsRow> metrics;
    std::vector<FrameStats> frames;
    int intersection_violations = 0;
    std::vector<double> rho;  // final adapted rho per body (NaN: not shared)
};

/* sim.hpp:63-71 (InProc only: the transport is replaced by batched kernels). */
struct RunOptions {
    int workers = 1;
    std::string out_dir;
    const Trajectory* reference = nullptr;
    bool audit = false;
    int device = 0;
};

/* sim.hpp:98-103. */
struct Snapshot {
    int64_t frame = 0;
    std::vector<int> ids;
    std::vector<Vec6> q;
    std::vector<Vec6> q_dot;
};

// ---------------------------------------------------------------------------
// RAII handles
// ---------------------------------------------------------------------------

/* dabd_gpu_scene: the body table built from the world loops. */
class Scene {
  public:
    explicit Scene(const SceneData& s) : n_(static_cast<int>(s.bodies.size())) {
        std::vector<int> body_loop{0}, loop_vert{0}, is_static;
        std::vector<double> verts, density, arap, qdot;
        for (const Body& b : s.bodies) {
            for (const Loop& l : b.loops) {
                for (const Vec2& v : l) verts.insert(verts.end(), {v[0], v[1]});
                loop_vert.push_back(static_cast<int>(verts.size() / 2));
            }
            body_loop.push_back(static_cast<int>(loop_vert.size()) - 1);
            density.push_back(b.density);
            is_static.push_back(b.is_static ? 1 : 0);
            arap.push_back(b.arap_scale);
            qdot.insert(qdot.end(), b.velocity.begin(), b.velocity.end());
        }
        check(dabd_gpu_scene_create(n_, body_loop.data(), loop_vert.data(), verts.data(),
                                    density.data(), is_static.data(), arap.data(), qdot.data(),
                                    &h_));
        const dabd_gpu_sim_params sim = to_c(s.params);
        const dabd_gpu_adapt_params ad{s.adapt.beta,      s.adapt.tau,       s.adapt.mu,
                                       s.adapt.sigma_min, s.adapt.sigma_max, s.adapt.adapt_enabled};
        const dabd_gpu_run_params run{s.w_min, s.admm_max_iterations, s.newton_cap, s.max_halvings,
                                      s.force_split_frames};
        check(dabd_gpu_scene_set_params(h_, &sim, &ad, &run));
        std::vector<double> pl;
        for (const Plane& p : s.planes) pl.insert(pl.end(), {p.point[0], p.point[1], p.normal[0], p.normal[1]});
        check(dabd_gpu_scene_set_planes(h_, static_cast<int>(s.planes.size()),
                                        pl.empty() ? nullptr : pl.data()));
        const dabd_gpu_balance_params bal{s.balance_enabled ? 1 : 0, s.balance.kp, s.balance.kd,
                                          s.balance.smoothing, s.balance.dp_max};
        check(dabd_gpu_scene_set_balance(h_, &bal));
        for (const auto& [body, f] : s.replica_force_split)
            check(dabd_gpu_scene_set_force_split(h_, body, f[0], f[1]));
        int nv = 0;
        check(dabd_gpu_scene_counts(h_, &n_, &nv));
        rest_.resize(2 * static_cast<size_t>(nv));
        vstart_.resize(n_ + 1);
        q0_.resize(n_);
        mass_.resize(n_);
        mm_.resize(36 * static_cast<size_t>(n_));
        check(dabd_gpu_scene_bodies(h_, rest_.data(), vstart_.data(), q0_.data()->data(),
                                    mass_.data(), mm_.data()));
        for (const Body& b : s.bodies) is_static_.push_back(b.is_static);
    }
    ~Scene() { dabd_gpu_scene_free(h_); }
    Scene(const Scene&) = delete;
    Scene& operator=(const Scene&) = delete;

    static dabd_gpu_sim_params to_c(const SimParams& p) {
        return {p.h, p.gravity[0], p.gravity[1], p.arap_stiffness, p.barrier_stiffness, p.d_hat,
                p.theta, p.scene_scale};
    }
    const dabd_gpu_scene* handle() const { return h_; }
    int size() const { return n_; }
    /* SceneData::initial_configs (scene.hpp:38-42): centroid translation, A = I. */
    const Configs& initial_configs() const { return q0_; }
    const std::vector<double>& mass() const { return mass_; }
    const std::vector<bool>& is_static() const { return is_static_; }

  private:
    dabd_gpu_scene* h_ = nullptr;
    int n_ = 0;
    std::vector<double> rest_, mass_, mm_;
    std::vector<int> vstart_;
    Configs q0_;
    std::vector<bool> is_static_;
};

/* dabd_gpu_ctx: one GPU's engine. workers == 0 selects run_reference
 * semantics, workers >= 1 the consensus-ADMM runtime over `workers` slabs. */
class Context {
  public:
    Context(const Scene& scene, int device = 0, int workers = 0) : n_(scene.size()) {
        check(dabd_gpu_ctx_create(scene.handle(), device, workers, 0, workers > 0 ? workers : 1, &h_));
    }
    ~Context() { dabd_gpu_ctx_free(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    dabd_gpu_ctx* handle() { return h_; }
    void set_solver(double pcg_rel_tol, int pcg_max_iters) {
        const dabd_gpu_solver_params p{pcg_rel_tol, pcg_max_iters};
        check(dabd_gpu_ctx_set_solver(h_, &p));
    }
    std::vector<dabd_gpu_frame_stats> run_frames(int n) {
        std::vector<dabd_gpu_frame_stats> st(n > 0 ? n : 1);
        check(dabd_gpu_run_frames(h_, n, st.data()));
        st.resize(n);
        return st;
    }
    void state(Configs& q, Configs& q_dot) {
        q.resize(n_);
        q_dot.resize(n_);
        check(dabd_gpu_get_state(h_, q.data()->data(), q_dot.data()->data()));
    }
    void set_state(const Configs& q, const Configs& q_dot) {
        check(dabd_gpu_set_state(h_, q.data()->data(), q_dot.data()->data()));
    }
    std::vector<double> rho() {
        std::vector<double> r(n_ > 0 ? n_ : 1);
        check(dabd_gpu_get_rho(h_, r.data()));
        r.resize(n_);
        return r;
    }
    /* (frame, attempt, k, dq, r, s, min_toi, sigma) rows; sigma 1 = End. */
    std::vector<std::array<double, 8>> take_trace() {
        std::vector<std::array<double, 8>> rows(1 << 14);
        int cnt = 0;
        check(dabd_gpu_take_trace(h_, rows.data()->data(), static_cast<int>(rows.size()), &cnt));
        rows.resize(cnt);
        return rows;
    }
    /* intersection_test (geometry.cpp:389-454) of the device-resident state. */
    bool intersection_test() {
        int res = 0;
        check(dabd_gpu_audit(h_, nullptr, nullptr, 0, 0.0, &res, nullptr, nullptr));
        return res != 0;
    }

  private:
    dabd_gpu_ctx* h_ = nullptr;
    int n_ = 0;
};

// ---------------------------------------------------------------------------
// Files (sim.cpp:34-137): same names, same layouts
// ---------------------------------------------------------------------------

inline std::string frame_path(const std::string& dir, int64_t frame) {
    char name[32];
    std::snprintf(name, sizeof(name), "frame_%04lld.bin", static_cast<long long>(frame));
    return dir + "/" + name;
}

/* [u64 frame][u64 n_dynamic][per dynamic body: u64 id, 6 f64 q, 6 f64 q_dot]. */
inline void write_snapshot(const std::string& path, int64_t frame, const std::vector<bool>& is_static,
                           const Configs& q, const Configs& q_dot) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("snapshot: cannot open " + path);
    auto put_u64 = [&](uint64_t v) { out.write(reinterpret_cast<const char*>(&v), 8); };
    auto put_f64 = [&](double v) { out.write(reinterpret_cast<const char*>(&v), 8); };
    uint64_t n = 0;
    for (bool s : is_static) n += s ? 0 : 1;
    put_u64(static_cast<uint64_t>(frame));
    put_u64(n);
    for (size_t b = 0; b < is_static.size(); ++b) {
        if (is_static[b]) continue;
        put_u64(static_cast<uint64_t>(b));
        for (int i = 0; i < 6; ++i) put_f64(q[b][i]);
        for (int i = 0; i < 6; ++i) put_f64(q_dot[b][i]);
    }
}

inline Snapshot read_snapshot(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error("snapshot: cannot open " + path);
    auto get_u64 = [&]() {
        uint64_t v = 0;
        in.read(reinterpret_cast<char*>(&v), 8);
        return v;
    };
    auto get_f64 = [&]() {
        double v = 0;
        in.read(reinterpret_cast<char*>(&v), 8);
        return v;
    };
    Snapshot snap;
    snap.frame = static_cast<int64_t>(get_u64());
    const uint64_t n = get_u64();
    for (uint64_t i = 0; i < n && in; ++i) {
        snap.ids.push_back(static_cast<int>(get_u64()));
        Vec6 q, qd;
        for (int j = 0; j < 6; ++j) q[j] = get_f64();
        for (int j = 0; j < 6; ++j) qd[j] = get_f64();
        snap.q.push_back(q);
        snap.q_dot.push_back(qd);
    }
    if (!in) throw Error("snapshot: truncated file " + path);
    return snap;
}

/* sim.cpp:53-78: static bodies keep their initial configuration. */
inline Trajectory load_trajectory(const std::string& dir, const Configs& initial) {
    Trajectory traj;
    for (int64_t frame = 0;; ++frame) {
        const std::string path = frame_path(dir, frame);
        if (!std::filesystem::exists(path)) break;
        const Snapshot snap = read_snapshot(path);
        Configs q = initial, qd(initial.size(), Vec6{});
        for (size_t i = 0; i < snap.ids.size(); ++i) {
            const int id = snap.ids[i];
            if (id < 0 || id >= static_cast<int>(initial.size()))
                throw Error("load_trajectory: snapshot body id out of range");
            q[id] = snap.q[i];
            qd[id] = snap.q_dot[i];
        }
        traj.q.push_back(std::move(q));
        traj.q_dot.push_back(std::move(qd));
        traj.h.push_back(0.0);
    }
    if (traj.q.empty()) throw Error("load_trajectory: no snapshots in " + dir);
    return traj;
}

inline void write_metrics_csv(const std::string& path, const std::vector<MetricsRow>& rows,
                              int workers) {
    std::ofstream out(path);
    if (!out) throw Error("metrics: cannot open " + path);
    out << "frame,attempt,k,committed,r_inf,s_inf,min_toi,active_contacts,candidate_pairs,mse";
    for (int i = 0; i < workers; ++i) out << ",dq_inf_w" << i;
    for (int i = 0; i < workers; ++i) out << ",newton_w" << i;
    for (int i = 0; i < workers; ++i) out << ",t_compute_w" << i;
    for (int i = 0; i < workers; ++i) out << ",t_sync_w" << i;
    out << "\n";
    out.precision(17);
    auto col = [&](const auto& v, int i) {
        out << ',';
        if (i < static_cast<int>(v.size())) out << v[i];
    };
    for (const MetricsRow& r : rows) {
        out << r.frame << ',' << r.attempt << ',' << r.k << ',' << (r.commit_row ? 1 : 0) << ','
            << r.r_inf << ',' << r.s_inf << ',' << r.min_toi << ',' << r.active_contacts << ','
            << r.candidate_pairs << ',';
        if (!std::isnan(r.mse)) out << r.mse;
        for (int i = 0; i < workers; ++i) col(r.dq_inf, i);
        for (int i = 0; i < workers; ++i) col(r.newton_iters, i);
        for (int i = 0; i < workers; ++i) col(r.t_compute, i);
        for (int i = 0; i < workers; ++i) col(r.t_sync, i);
        out << "\n";
    }
}

/* sim.cpp:14-28: mean squared error over the dynamic DoF. */
inline double mse_to_reference(const std::vector<bool>& is_static, const Configs& q,
                               const Configs& q_ref) {
    double sum = 0.0;
    int64_t entries = 0;
    for (size_t b = 0; b < is_static.size(); ++b) {
        if (is_static[b]) continue;
        for (int i = 0; i < 6; ++i) {
            const double d = q[b][i] - q_ref[b][i];
            sum += d * d;
        }
        entries += 6;
    }
    return entries > 0 ? sum / static_cast<double>(entries) : 0.0;
}

// ---------------------------------------------------------------------------
// Drivers (sim.cpp:186-432)
// ---------------------------------------------------------------------------

/* run_reference (sim.cpp:186-249): one CUDA graph per frame on `device`. */
inline Trajectory run_reference(const SceneData& scene, const std::string& out_dir = "",
                                int device = 0) {
    Scene sc(scene);
    Context ctx(sc, device, 0);
    if (!out_dir.empty()) std::filesystem::create_directories(out_dir);
    Trajectory traj;
    for (int64_t f = 0; f < scene.frames; ++f) {
        const dabd_gpu_frame_stats st = ctx.run_frames(1)[0];
        Configs q, qd;
        ctx.state(q, qd);
        if (!out_dir.empty()) write_snapshot(frame_path(out_dir, f), f, sc.is_static(), q, qd);
        traj.q.push_back(std::move(q));
        traj.q_dot.push_back(std::move(qd));
        traj.h.push_back(st.h);
    }
    return traj;
}

/* run_distributed (sim.cpp:264-432): the controller + worker semantics of
 * runtime.cpp:110-694 with all `workers` partitions batched on one GPU.
 * metrics.csv rows come from the device ADMM trace (one row per k). */
inline RunResult run_distributed(const SceneData& scene, const RunOptions& options) {
    Scene sc(scene);
    Context ctx(sc, options.device, options.workers);
    if (!options.out_dir.empty()) std::filesystem::create_directories(options.out_dir);
    RunResult res;
    for (int64_t f = 0; f < scene.frames; ++f) {
        const dabd_gpu_frame_stats st = ctx.run_frames(1)[0];
        Configs q, qd;
        ctx.state(q, qd);
        for (const auto& t : ctx.take_trace()) {
            MetricsRow row;
            row.frame = static_cast<int64_t>(t[0]);
            row.attempt = static_cast<int32_t>(t[1]);
            row.k = static_cast<int32_t>(t[2]);
            row.dq_inf.assign(1, t[3]);
            row.r_inf = t[4];
            row.s_inf = t[5];
            row.min_toi = t[6];
            row.commit_row = t[7] == 1.0;
            if (row.commit_row && options.reference && f < static_cast<int64_t>(options.reference->q.size()))
                row.mse = mse_to_reference(sc.is_static(), q, options.reference->q[f]);
            if (row.commit_row) {
                row.t_compute.assign(options.workers, st.t_frame - st.t_sync);
                row.t_sync.assign(options.workers, st.t_sync);
            }
            res.metrics.push_back(std::move(row));
        }
        FrameStats fs;
        fs.frame = f;
        fs.attempts = st.attempts;
        fs.h = st.h;
        fs.admm_iterations = st.admm_iterations;
        fs.newton_iterations = st.newton_iterations;
        fs.line_search_steps = st.line_search_steps;
        fs.pcg_iterations = st.pcg_iterations;
        fs.max_contacts = st.max_contacts;
        fs.max_candidates = st.max_candidates;
        fs.exact_retries = st.exact_retries;
        fs.capacity_retries = st.capacity_retries;
        fs.t_solve = st.t_solve;
        fs.t_coll = st.t_coll;
        fs.t_sync = st.t_sync;
        fs.t_frame = st.t_frame;
        res.frames.push_back(fs);
        if (options.audit && ctx.intersection_test()) ++res.intersection_violations;
        if (!options.out_dir.empty())
            write_snapshot(frame_path(options.out_dir, f), f, sc.is_static(), q, qd);
        res.trajectory.q.push_back(std::move(q));
        res.trajectory.q_dot.push_back(std::move(qd));
        res.trajectory.h.push_back(st.h);
    }
    res.rho = ctx.rho();
    if (!options.out_dir.empty())
        write_metrics_csv(options.out_dir + "/metrics.csv", res.metrics, options.workers);
    return res;
}

// ---------------------------------------------------------------------------
// Geometry / partition entry points (geometry.hpp:47-74, partition.hpp:43-45)
// ---------------------------------------------------------------------------

struct ContactPair {
    int a, b, v, e;  // point of body a against edge e of body b (geometry.hpp:25-36)
};

/* broad_phase (q_end empty) / broad_phase_swept over all bodies. */
inline std::vector<ContactPair> broad_phase(Context& ctx, const Configs& q, double margin,
                                            const Configs& q_end = {}) {
    int cap = 4096;
    for (;;) {
        std::vector<ContactPair> out(cap);
        int cnt = 0;
        const dabd_gpu_status s =
            dabd_gpu_broad_phase(ctx.handle(), q.data()->data(), q_end.empty() ? nullptr : q_end.data()->data(),
                                 margin, nullptr, 0, &out.data()->a, cap, &cnt);
        if (s == DABD_GPU_ERR_INVALID && cnt > cap) {
            cap = cnt;
            continue;
        }
        check(s);
        out.resize(cnt);
        return out;
    }
}

/* ccd_toi_scene (geometry.hpp:72-74): 1.0 exactly iff no impact. */
inline double ccd_toi_scene(Context& ctx, const Configs& q0, const Configs& q1) {
    double t = 1.0;
    check(dabd_gpu_ccd_toi(ctx.handle(), q0.data()->data(), q1.data()->data(), nullptr, 0, &t));
    return t;
}

/* body_holder_mask (partition.hpp:43-45) for every body. */
inline std::vector<uint32_t> body_holder_masks(Context& ctx, const Configs& q,
                                               const std::vector<Plane>& planes, double w) {
    std::vector<double> pl;
    for (const Plane& p : planes) pl.insert(pl.end(), {p.point[0], p.point[1], p.normal[0], p.normal[1]});
    std::vector<uint32_t> masks(q.size());
    check(dabd_gpu_holder_masks(ctx.handle(), q.data()->data(), static_cast<int>(planes.size()),
                                pl.empty() ? nullptr : pl.data(), w, masks.data()));
    return masks;
}

// ---------------------------------------------------------------------------
// Built-in scenarios (scene.cpp:18-32, 345-557; same arithmetic as scene.py)
// ---------------------------------------------------------------------------

/* splitmix64 jitter stream (scene.cpp:18-32). */
class JitterRng {
  public:
    explicit JitterRng(uint64_t seed) : state_(seed ? seed : 0x9E3779B97F4A7C15ull) {}
    double uniform(double lo, double hi) {
        state_ += 0x9E3779B97F4A7C15ull;
        uint64_t z = state_;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
        return lo + u * (hi - lo);
    }

  private:
    uint64_t state_;
};

inline Loop box_loop(Vec2 c, Vec2 h) {
    return {{c[0] + -h[0], c[1] + -h[1]}, {c[0] + h[0], c[1] + -h[1]},
            {c[0] + h[0], c[1] + h[1]},   {c[0] + -h[0], c[1] + h[1]}};
}

inline Loop thick_segment_loop(Vec2 a, Vec2 b, double thickness) {
    double dx = b[0] - a[0], dy = b[1] - a[1];
    const double nrm = std::sqrt(dx * dx + dy * dy);
    dx = dx / nrm;
    dy = dy / nrm;
    const double nx = -dy, ny = dx, s = 0.5 * thickness, tx = s * nx, ty = s * ny;
    Loop loop{{a[0] - tx, a[1] - ty}, {b[0] - tx, b[1] - ty}, {b[0] + tx, b[1] + ty}, {a[0] + tx, a[1] + ty}};
    double area = 0.0;
    for (size_t i = 0; i < loop.size(); ++i) {
        const Vec2& p = loop[i];
        const Vec2& q = loop[(i + 1) % loop.size()];
        area += (p[0] * q[1] - q[0] * p[1]) / 2.0;
    }
    if (area < 0.0) std::reverse(loop.begin(), loop.end());
    return loop;
}

namespace detail {
inline void drop_params(SceneData& s, double l) {
    s.params.h = 0.01;
    s.params.gravity = {0.0, -10.0};
    s.params.arap_stiffness = 1e8;
    s.params.barrier_stiffness = 1e4;
    s.params.d_hat = 0.01;
    s.params.theta = 1e-3;
    s.params.scene_scale = l;
}

inline SceneData funnel_analog(double density, uint64_t seed) {
    SceneData s;
    s.name = "funnel-analog";
    s.frames = 100;
    s.seed = seed;
    s.params.h = 0.01;
    s.params.gravity = {0.0, -10.0};
    s.params.arap_stiffness = 1e8;
    s.params.barrier_stiffness = 1e5;
    s.params.d_hat = 0.01;
    s.params.theta = 3e-4;
    s.params.scene_scale = 4.0;
    s.planes = {Plane{{0.0, 0.0}, {-1.0, 0.0}}};
    s.w_min = 0.5;
    Body st;
    st.loops = {box_loop({0.0, -0.06}, {1.3, 0.06}), thick_segment_loop({-1.24, -0.02}, {-2.0, 0.78}, 0.12),
                thick_segment_loop({1.24, -0.02}, {2.0, 0.78}, 0.12)};
    st.is_static = true;
    s.bodies.push_back(st);
    JitterRng rng(seed);
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 8; ++c) {
            double cx = -0.98 + 0.28 * c, cy = 0.145 + 0.45 * r;
            cx += rng.uniform(-0.012, 0.012);
            cy += rng.uniform(-0.005, 0.005);
            Body b;
            b.loops = {box_loop({cx, cy}, {0.12, 0.12})};
            b.density = density;
            s.bodies.push_back(b);
        }
    return s;
}

inline SceneData drop_grid(int slabs, uint64_t seed) {
    SceneData s;
    s.name = "drop-grid-" + std::to_string(slabs);
    s.frames = 100;
    s.seed = seed;
    drop_params(s, 2.0 * slabs);
    s.w_min = 0.4;
    const double width = 2.0 * slabs;
    for (int k = 1; k < slabs; ++k) s.planes.push_back(Plane{{-width / 2.0 + 2.0 * k, 0.0}, {-1.0, 0.0}});
    Body st;
    st.loops = {box_loop({0.0, -0.06}, {width / 2.0 + 0.2, 0.06}),
                box_loop({-width / 2.0 - 0.14, 0.8}, {0.06, 0.8}),
                box_loop({width / 2.0 + 0.14, 0.8}, {0.06, 0.8})};
    st.is_static = true;
    s.bodies.push_back(st);
    JitterRng rng(seed);
    for (int sl = 0; sl < slabs; ++sl) {
        const double x0 = -width / 2.0 + 2.0 * sl + 0.35;
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
                double cx = x0 + 0.43 * c, cy = 0.35 + 0.42 * r;
                cx += rng.uniform(-0.02, 0.02);
                cy += rng.uniform(-0.02, 0.02);
                Body b;
                b.loops = {box_loop({cx, cy}, {0.12, 0.12})};
                s.bodies.push_back(b);
            }
    }
    return s;
}

/* scene.py:lattice_pile: boxes dropped into a container. */
inline SceneData lattice_pile(const std::string& name, int rows, int cols, int slabs, double half,
                              double spacing, double jitter, uint64_t seed, double slab_width,
                              double l) {
    if (slab_width <= 0.0) slab_width = cols * spacing;
    const double width = slab_width * slabs;
    SceneData s;
    s.name = name;
    s.frames = 100;
    s.seed = seed;
    drop_params(s, l > 0.0 ? l : std::max(2.0, width));
    s.w_min = 0.4;
    for (int k = 1; k < slabs; ++k) s.planes.push_back(Plane{{-width / 2.0 + slab_width * k, 0.0}, {-1.0, 0.0}});
    const double hw = width / 2.0, wall_h = rows * spacing + 1.0;
    Body st;
    st.loops = {box_loop({0.0, -0.06}, {hw + 0.2, 0.06}), box_loop({-hw - 0.14, wall_h / 2.0}, {0.06, wall_h / 2.0}),
                box_loop({hw + 0.14, wall_h / 2.0}, {0.06, wall_h / 2.0})};
    st.is_static = true;
    s.bodies.push_back(st);
    JitterRng rng(seed);
    const double y0 = half + 0.02;
    for (int sl = 0; sl < slabs; ++sl) {
        const double x0 = -width / 2.0 + slab_width * sl + 0.5 * (slab_width - (cols - 1) * spacing);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) {
                double cx = x0 + spacing * c, cy = y0 + spacing * r;
                cx += rng.uniform(-jitter, jitter);
                cy += rng.uniform(-jitter, jitter);
                Body b;
                b.loops = {box_loop({cx, cy}, {half, half})};
                s.bodies.push_back(b);
            }
    }
    return s;
}
}  // namespace detail

/* make_scenario (scene.cpp:538-557) for the builtins the C++ side needs. */
inline SceneData make_scenario(const std::string& name) {
    if (name == "funnel-analog") return detail::funnel_analog(1000.0, 7);
    const std::string dg = "drop-grid-", ds = "density-sweep-";
    if (name.rfind(dg, 0) == 0) return detail::drop_grid(std::stoi(name.substr(dg.size())), 11);
    if (name.rfind(ds, 0) == 0) {
        SceneData s = detail::funnel_analog(std::stod(name.substr(ds.size())), 7);
        s.name = name;
        return s;
    }
    if (name == "pile-1k") return detail::lattice_pile(name, 25, 40, 1, 0.05, 0.13, 0.005, 11, 0.0, 6.0);
    if (name == "pour-10k") return detail::lattice_pile(name, 50, 25, 8, 0.03, 0.075, 0.004, 11, 2.0, 0.0);
    throw Error("unknown scenario '" + name + "'");
}

}  // namespace gpu
}  // namespace dabd

#endif /* DABD_GPU_HPP */
