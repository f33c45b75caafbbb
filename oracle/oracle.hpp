// ============================================================================
// TEST INFRASTRUCTURE ONLY -- NOT PART OF THE PRODUCT.
//
// CPU restatement of the reference hot path (arxiv/paper_2605_15875, `dabd`)
// used as the parity checker for the B200 kernels. Only tests/, the smoke()
// entry and bench.py's cpu_baseline leg may load it. The product library
// (paper_2605_15875_b200/libdabd_gpu.so) never links or calls it.
//
// Each function cites the reference file:line it restates (paths relative to
// /root/reference/proj). The reference cannot be compiled in this container
// (Eigen3 and the vendored single headers are absent), so the
// third-party pieces (Eigen LDLT/SelfAdjointEigenSolver/SimplicialLDLT) are
// replaced by a pivoted 6x6 LDLT, cyclic Jacobi and a block-sparse Cholesky;
// those are parity-pinned only at tolerance level by the reference's own
// known-answer tests (ported in tests/test_oracle_*.py).
//
// Build: -O3 -ffp-contract=off (x86-64 SSE2, no FMA), matching the reference
// build which has no -march flag (proj/CMakeLists.txt:1-13).
// ============================================================================
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

struct Error : std::runtime_error {
    explicit Error(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------------------
// L0 types (types.hpp:10-42)
// ---------------------------------------------------------------------------
struct Vec2 {
    double x = 0.0, y = 0.0;
};
inline Vec2 operator+(Vec2 a, Vec2 b) { return {a.x + b.x, a.y + b.y}; }
inline Vec2 operator-(Vec2 a, Vec2 b) { return {a.x - b.x, a.y - b.y}; }
inline Vec2 operator*(double s, Vec2 a) { return {s * a.x, s * a.y}; }
inline Vec2 operator/(Vec2 a, double s) { return {a.x / s, a.y / s}; }
inline double dot(Vec2 a, Vec2 b) { return a.x * b.x + a.y * b.y; }
inline double sqnorm(Vec2 a) { return a.x * a.x + a.y * a.y; }
inline double norm(Vec2 a) { return std::sqrt(sqnorm(a)); }
inline double cross2(Vec2 a, Vec2 b) { return a.x * b.y - a.y * b.x; }
inline Vec2 vmin(Vec2 a, Vec2 b) { return {std::min(a.x, b.x), std::min(a.y, b.y)}; }
inline Vec2 vmax(Vec2 a, Vec2 b) { return {std::max(a.x, b.x), std::max(a.y, b.y)}; }

using Vec6 = std::array<double, 6>;
using Vec12 = std::array<double, 12>;

// Row-major dense N x N.
template <int N>
struct MatN {
    double m[N * N];
    MatN() { for (int i = 0; i < N * N; ++i) m[i] = 0.0; }
    double& operator()(int r, int c) { return m[r * N + c]; }
    double operator()(int r, int c) const { return m[r * N + c]; }
    static MatN identity() {
        MatN a;
        for (int i = 0; i < N; ++i) a(i, i) = 1.0;
        return a;
    }
};
using Mat6 = MatN<6>;
using Mat12 = MatN<12>;

inline Vec6 zero6() { return Vec6{0, 0, 0, 0, 0, 0}; }

// world_point: A*xbar + p with A=[[q2,q3],[q4,q5]] (types.hpp:19-30).
inline Vec2 world_point(const Vec6& q, Vec2 xb) {
    return {(q[2] * xb.x + q[3] * xb.y) + q[0], (q[4] * xb.x + q[5] * xb.y) + q[1]};
}

// ---------------------------------------------------------------------------
// Params (params.hpp:8-41)
// ---------------------------------------------------------------------------
struct SimParams {
    double h = 0.01;
    Vec2 gravity{0.0, -9.81};
    double arap_stiffness = 1e6;
    double barrier_stiffness = 1e4;
    double d_hat = 0.01;
    double theta = 1e-3;
    double scene_scale = 1.0;
    void validate() const;
};

struct AdaptParams {
    double beta = 1.0, tau = 2.0, mu = 5.0, sigma_min = 1e-3, sigma_max = 1e3;
    bool adapt_enabled = true;
    void validate() const;
};

// ---------------------------------------------------------------------------
// Body (body.hpp:16-91, body.cpp)
// ---------------------------------------------------------------------------
struct Aabb {
    Vec2 lo, hi;
    bool overlaps(const Aabb& o) const {
        return lo.x <= o.hi.x && o.lo.x <= hi.x && lo.y <= o.hi.y && o.lo.y <= hi.y;
    }
    Aabb inflated(double r) const { return {lo - Vec2{r, r}, hi + Vec2{r, r}}; }
    Aabb merged(const Aabb& o) const { return {vmin(lo, o.lo), vmax(hi, o.hi)}; }
};

using Loop = std::vector<Vec2>;
using Configs = std::vector<Vec6>;

struct PolygonMoments {
    double area = 0, sx = 0, sy = 0, sxx = 0, sxy = 0, syy = 0;
};
PolygonMoments loop_moments(const Loop& loop);
PolygonMoments loops_moments(const std::vector<Loop>& loops);

struct AffineBody {
    int id = -1;
    std::vector<Loop> rest_loops;
    Vec6 q = zero6();
    Vec6 q_dot = zero6();
    double density = 1.0;
    double mass = 0.0;
    Mat6 mass_matrix;
    double rest_area = 0.0;
    bool is_static = false;
    double arap_scale = 1.0;
    // Flattened vertex cache (rest_vertex/rest_edge of body.cpp:49-69).
    std::vector<Vec2> flat;
    std::vector<int> next; // flat index of the second endpoint of edge e
    int vertex_count() const { return static_cast<int>(flat.size()); }
    int edge_count() const { return vertex_count(); }
    Vec2 rest_vertex(int v) const { return flat.at(v); }
    void rest_edge(int e, Vec2& a, Vec2& b) const {
        a = flat.at(e);
        b = flat.at(next.at(e));
    }
    void build_flat();
};

void build_mass_matrix(const std::vector<Loop>& loops, double density, double& mass,
                       Mat6& m);
AffineBody make_affine_body(int id, const std::vector<Loop>& world_loops, double density,
                            bool is_static);
Vec6 predicted_position(const Vec6& q, const Vec6& q_dot, const Vec6& f_ext, double h,
                        const Mat6& mass_matrix);
Vec6 gravity_force(const AffineBody& body, Vec2 gravity);
Aabb body_aabb(const AffineBody& body, const Vec6& q);
double max_vertex_speed(const AffineBody& body, const Vec6& q_dot);

// ---------------------------------------------------------------------------
// Geometry (geometry.hpp, geometry.cpp)
// ---------------------------------------------------------------------------
struct PointEdgeDistance {
    double d = 0.0;
    Vec6 grad = zero6();
    Mat6 hess;
};
PointEdgeDistance point_edge_distance(Vec2 p, Vec2 e0, Vec2 e1, bool with_hessian = true);

struct ContactPair {
    int body_a = -1, body_b = -1, point_index = -1, edge_index = -1;
    double d = 0.0;
    double kappa_c = 1.0;
    friend bool operator<(const ContactPair& l, const ContactPair& r) {
        if (l.body_a != r.body_a) return l.body_a < r.body_a;
        if (l.body_b != r.body_b) return l.body_b < r.body_b;
        if (l.point_index != r.point_index) return l.point_index < r.point_index;
        return l.edge_index < r.edge_index;
    }
};

std::vector<ContactPair> broad_phase(const std::vector<AffineBody>& bodies,
                                     const Configs& q, double d_hat,
                                     const std::vector<int>& subset = {});
std::vector<ContactPair> broad_phase_swept(const std::vector<AffineBody>& bodies,
                                           const Configs& start, const Configs& end,
                                           double margin, const std::vector<int>& subset = {});
std::vector<ContactPair> narrow_phase(const std::vector<ContactPair>& cand,
                                      const std::vector<AffineBody>& bodies,
                                      const Configs& q, double d_hat);
double pair_impact_time(Vec2 p0, Vec2 p1, Vec2 a0, Vec2 a1, Vec2 b0, Vec2 b1);
double ccd_toi(const std::vector<AffineBody>& bodies, const Configs& start,
               const Configs& end, const std::vector<ContactPair>& cand);
double ccd_toi_scene(const std::vector<AffineBody>& bodies, const Configs& start,
                     const Configs& end, const std::vector<int>& subset = {});
double min_pair_distance(const std::vector<AffineBody>& bodies, const Configs& q,
                         const std::vector<int>& subset, bool skip_static_pairs);
bool intersection_test(const std::vector<AffineBody>& bodies, const Configs& q,
                       const std::vector<int>& subset = {});

// ---------------------------------------------------------------------------
// Energy (energy.hpp, energy.cpp)
// ---------------------------------------------------------------------------
struct BodyEnergy {
    double value = 0.0;
    Vec6 grad = zero6();
    Mat6 hess;
};
struct PairEnergy {
    double value = 0.0;
    Vec12 grad{};
    Mat12 hess;
};
struct BarrierValue {
    double value = 0.0, dvalue = 0.0, ddvalue = 0.0;
};
BodyEnergy inertia_energy(const Vec6& q, const Vec6& q_tilde, const Mat6& m);
BodyEnergy arap_energy(const Vec6& q, double kappa, double rest_area);
BarrierValue barrier_energy(double d, double d_hat, double kappa);
PairEnergy contact_energy(const AffineBody& pb, const Vec6& qa, const AffineBody& eb,
                          const Vec6& qb, int point_index, int edge_index, double d_hat,
                          double kappa);

// Symmetric eigen-clamp (objective.cpp:12-17) via cyclic Jacobi.
template <int N>
MatN<N> clamp_psd(const MatN<N>& a);

// ---------------------------------------------------------------------------
// Objective (objective.hpp, objective.cpp)
// ---------------------------------------------------------------------------
struct SharedAnchor {
    int body = -1;
    Vec6 z = zero6();
    Vec6 u = zero6();
    double rho = 0.0;
};

// Block-sparse symmetric matrix over 6x6 body blocks (replaces the Eigen
// triplet SparseMatrix; duplicate contributions sum in insertion order,
// as setFromTriplets does).
struct BlockMatrix {
    int nb = 0;
    std::vector<Mat6> diag;
    std::map<std::pair<int, int>, Mat6> off; // (r, c), r != c, both stored
    void add(int r, int c, const Mat6& blk);
    double trace() const;
};

class LocalObjective {
  public:
    static LocalObjective assemble(const std::vector<AffineBody>& bodies,
                                   std::vector<int> local, std::vector<double> kappa_b,
                                   std::vector<Vec6> q_tilde,
                                   std::vector<SharedAnchor> anchors,
                                   std::vector<uint32_t> holder_mask,
                                   const SimParams& params);
    double value(const Configs& q, bool with_anchors = true) const;
    struct Derivatives {
        double value = 0.0;
        std::vector<double> grad;
        BlockMatrix hess;
        int active_contacts = 0;
        int candidate_pairs = 0;
    };
    Derivatives derivatives(const Configs& q, bool project_psd = true) const;
    int num_dofs() const { return num_dofs_; }
    const std::vector<int>& local_bodies() const { return local_; }
    const std::vector<AffineBody>& bodies() const { return *bodies_; }
    const SimParams& params() const { return params_; }
    void apply_step(Configs& q, const std::vector<double>& delta, double alpha) const;
    double config_delta_inf(const Configs& a, const Configs& b) const;
    std::vector<ContactPair> active_contacts(const Configs& q) const {
        return detect(q, nullptr);
    }
    void contact_counts(const Configs& q, int& active, int& candidates) const;
    double contact_weight(int a, int b) const;

  private:
    std::vector<ContactPair> detect(const Configs& q, int* candidates) const;
    const std::vector<AffineBody>* bodies_ = nullptr;
    std::vector<int> local_;
    std::vector<double> inv_kappa_;
    std::vector<Vec6> q_tilde_;
    std::vector<int> anchor_of_;
    std::vector<SharedAnchor> anchors_;
    std::vector<uint32_t> holder_mask_;
    std::vector<int> dof_offset_;
    std::vector<int> local_pos_;
    int num_dofs_ = 0;
    SimParams params_;
};

// ---------------------------------------------------------------------------
// Newton (newton.hpp, newton.cpp)
// ---------------------------------------------------------------------------
struct NewtonReport {
    int iterations = 0;
    double final_update_inf = 0.0;
    bool converged = false;
    int line_search_steps = 0;
};
struct NewtonOptions {
    int max_iters = 32;
    double tol = 1e-6;
    double armijo_c = 0.0;
};
NewtonReport newton_solve(const LocalObjective& obj, Configs& q, const NewtonOptions& opt);
// Solves (H + eps I) x = rhs with a block Cholesky on a minimum-degree
// ordering of the body graph (stand-in for Eigen::SimplicialLDLT).
std::vector<double> block_sparse_solve(const BlockMatrix& h, double eps,
                                       const std::vector<double>& rhs);

// ---------------------------------------------------------------------------
// Partition / consensus (partition.cpp, consensus.cpp)
// ---------------------------------------------------------------------------
struct Plane {
    Vec2 point{0.0, 0.0};
    Vec2 normal{1.0, 0.0};
};
double overlap_width(double v_max, double h, double w_min);
uint32_t body_holder_mask(const AffineBody& body, const Vec6& q,
                          const std::vector<Plane>& planes, double w);

struct PartitionLayout {
    int num_workers = 1;
    double w = 0.0;
    std::vector<Plane> planes;
    std::vector<uint32_t> holder_mask;
    std::vector<std::vector<int>> internal_bodies, shared_bodies, local_bodies, neighbors;
    int kappa_b(int body) const;
    std::vector<int> holders_of(int body) const;
    bool is_shared(int body) const { return kappa_b(body) >= 2; }
};
PartitionLayout partition_scene(const std::vector<AffineBody>& bodies, const Configs& q,
                                const std::vector<Plane>& planes, int num_workers,
                                double h, double w_min, double v_max_override = -1.0);
int contact_replication(const PartitionLayout& layout, int a, int b);

Vec6 consensus_update(const std::vector<Vec6>& q_plus_u, const std::vector<double>& rho);
Vec6 dual_update(const Vec6& u, const Vec6& q, const Vec6& z);
double primal_residual_inf(const std::vector<Vec6>& replica_q, const Vec6& z);
double dual_residual_inf(const Vec6& z_new, const Vec6& z_prev);
double init_rho(double mass, double beta);
double adapt_rho(double rho, double r_inf, double s_inf, const AdaptParams& p, double rho0);
bool check_stopping(double dq, double r, double s, const std::vector<double>& tois,
                    double h, double l, double theta);
double merge_ccd_gate(const std::vector<AffineBody>& bodies, const Configs& q_local,
                      const std::vector<int>& shared, const std::vector<Vec6>& z,
                      const std::vector<int>& local_subset);
void finalize_merge(Configs& q, Configs& q_dot, const Configs& q_start, double h,
                    const std::vector<int>& shared, const std::vector<Vec6>& z,
                    const std::vector<int>& dynamic_local, bool gate_passed);

class TimestepController {
  public:
    TimestepController(double h0, int max_halvings = 4)
        : h0_(h0), h_(h0), max_halvings_(max_halvings) {}
    double h() const { return h_; }
    int halvings() const { return halvings_; }
    double on_frame_failed() {
        if (halvings_ >= max_halvings_)
            throw Error("adaptive_timestep: frame failed after max halvings");
        h_ /= 2.0;
        ++halvings_;
        return h_;
    }
    void on_frame_committed() {
        h_ = std::min(h0_, 2.0 * h_);
        halvings_ = 0;
    }

  private:
    double h0_, h_;
    int halvings_ = 0, max_halvings_;
};

// ---------------------------------------------------------------------------
// Scene + drivers (scene.hpp, sim.cpp:186-249, runtime.cpp:110-694,
// tests/support/replay.cpp:11-169)
// ---------------------------------------------------------------------------
struct Scene {
    std::vector<AffineBody> bodies;
    SimParams params;
    AdaptParams adapt;
    std::vector<Plane> planes;
    double w_min = 0.1;
    int frames = 100;
    int admm_max_iterations = 300;
    int newton_cap = 32;
    int max_halvings = 4;
    std::map<int, Vec2> replica_force_split;
    int force_split_frames = -1;
    Configs initial_configs() const;
    Configs initial_velocities() const;
};

struct FrameStat {
    int attempts = 1;
    double h = 0.0;
    int admm_iterations = 0;
    int newton_iterations = 0;  // summed over workers and solves
    int line_search_steps = 0;
};

struct IterTrace {
    int frame = 0, attempt = 0, k = 0;
    double dq_inf = 0, r_inf = 0, s_inf = 0, min_toi = 1.0;
    int sigma = 0; // 0 continue, 1 end, 2 abort-retry, 3 fail
};

struct Trajectory {
    std::vector<Configs> q, q_dot;
    std::vector<double> h;
    std::vector<FrameStat> stats;
    std::vector<IterTrace> trace;
    std::vector<double> rho_final; // per body, NaN when not shared at the end
};

Trajectory run_reference(const Scene& scene, int frames);
Trajectory run_distributed(const Scene& scene, int workers, int frames);

} // namespace oracle
