// TEST INFRASTRUCTURE ONLY (see oracle.hpp). Restates proj/src/energy.cpp,
// objective.cpp and newton.cpp; clamp_psd and the sparse solve stand in for
// Eigen (SelfAdjointEigenSolver, SimplicialLDLT), parity-pinned at tolerance.
#include "oracle.hpp"

#include <algorithm>
#include <bit>
#include <set>

namespace oracle {

// ---------------------------------------------------------------------------
// energy.cpp
// ---------------------------------------------------------------------------

// energy.cpp:7-15
BodyEnergy inertia_energy(const Vec6& q, const Vec6& qt, const Mat6& m) {
    BodyEnergy out;
    Vec6 diff, md;
    for (int i = 0; i < 6; ++i) diff[i] = q[i] - qt[i];
    for (int i = 0; i < 6; ++i) {
        double s = 0.0;
        for (int k = 0; k < 6; ++k) s += m(i, k) * diff[k];
        md[i] = s;
    }
    double dd = 0.0;
    for (int i = 0; i < 6; ++i) dd += diff[i] * md[i];
    out.value = 0.5 * dd;
    out.grad = md;
    out.hess = m;
    return out;
}

// energy.cpp:17-48
BodyEnergy arap_energy(const Vec6& q, double kappa, double rest_area) {
    BodyEnergy out;
    const double a[2][2] = {{q[2], q[3]}, {q[4], q[5]}};
    double g[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            g[i][j] = (a[0][i] * a[0][j] + a[1][i] * a[1][j]) - (i == j ? 1.0 : 0.0);
    const double w = kappa * rest_area;
    out.value = w * (g[0][0] * g[0][0] + g[1][0] * g[1][0] + g[0][1] * g[0][1] +
                     g[1][1] * g[1][1]);
    const double w4 = 4.0 * w;
    double ag[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) ag[i][j] = a[i][0] * g[0][j] + a[i][1] * g[1][j];
    out.grad[2] = w4 * ag[0][0];
    out.grad[3] = w4 * ag[0][1];
    out.grad[4] = w4 * ag[1][0];
    out.grad[5] = w4 * ag[1][1];
    double aat[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) aat[i][j] = a[i][0] * a[j][0] + a[i][1] * a[j][1];
    const int slot[2][2] = {{2, 3}, {4, 5}};
    for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l)
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) {
                    double v = 0.0;
                    if (i == k) v += g[j][l];
                    v += a[i][l] * a[k][j];
                    if (j == l) v += aat[i][k];
                    out.hess(slot[k][l], slot[i][j]) = w4 * v;
                }
    return out;
}

// energy.cpp:50-61
BarrierValue barrier_energy(double d, double d_hat, double kappa) {
    if (d <= 0.0) throw Error("barrier_energy: d <= 0 (barrier domain violated)");
    BarrierValue out;
    if (d >= d_hat) return out;
    const double gap = d - d_hat;
    const double lg = std::log(d / d_hat);
    out.value = -kappa * gap * gap * lg;
    out.dvalue = -kappa * (2.0 * gap * lg + gap * gap / d);
    out.ddvalue = -kappa * (2.0 * lg + 2.0 * gap / d + gap * (d + d_hat) / (d * d));
    return out;
}

// energy.cpp:63-94
PairEnergy contact_energy(const AffineBody& pb, const Vec6& qa, const AffineBody& eb,
                          const Vec6& qb, int pi, int ei, double d_hat, double kappa) {
    PairEnergy out;
    const Vec2 rv = pb.rest_vertex(pi);
    Vec2 r0, r1;
    eb.rest_edge(ei, r0, r1);
    const Vec2 p = world_point(qa, rv), e0 = world_point(qb, r0), e1 = world_point(qb, r1);
    const PointEdgeDistance dist = point_edge_distance(p, e0, e1);
    if (dist.d >= d_hat) return out;
    const BarrierValue b = barrier_energy(dist.d, d_hat, kappa);
    out.value = b.value;
    double t[6][12] = {};
    auto put_j = [&t](int row, int col, Vec2 xb) {
        t[row][col + 0] = 1.0;
        t[row + 1][col + 1] = 1.0;
        t[row][col + 2] = xb.x;
        t[row][col + 3] = xb.y;
        t[row + 1][col + 4] = xb.x;
        t[row + 1][col + 5] = xb.y;
    };
    put_j(0, 0, rv);
    put_j(2, 6, r0);
    put_j(4, 6, r1);
    Vec12 gd{};
    for (int c = 0; c < 12; ++c) {
        double s = 0.0;
        for (int r = 0; r < 6; ++r) s += t[r][c] * dist.grad[r];
        gd[c] = s;
    }
    for (int c = 0; c < 12; ++c) out.grad[c] = b.dvalue * gd[c];
    double ht[6][12]; // H_d * t
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 12; ++c) {
            double s = 0.0;
            for (int k = 0; k < 6; ++k) s += dist.hess(r, k) * t[k][c];
            ht[r][c] = s;
        }
    for (int i = 0; i < 12; ++i)
        for (int j = 0; j < 12; ++j) {
            double s = 0.0;
            for (int k = 0; k < 6; ++k) s += t[k][i] * ht[k][j];
            out.hess(i, j) = b.ddvalue * (gd[i] * gd[j]) + b.dvalue * s;
        }
    return out;
}

// ---------------------------------------------------------------------------
// clamp_psd (objective.cpp:12-17): cyclic Jacobi eigendecomposition.
// ---------------------------------------------------------------------------
template <int N>
MatN<N> clamp_psd(const MatN<N>& in) {
    MatN<N> a = in;
    MatN<N> v = MatN<N>::identity();
    double total = 0.0;
    for (int i = 0; i < N * N; ++i) total += a.m[i] * a.m[i];
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < N; ++p)
            for (int q = p + 1; q < N; ++q) off += a(p, q) * a(p, q);
        if (off == 0.0 || off <= 1e-34 * total) break;
        for (int p = 0; p < N; ++p)
            for (int q = p + 1; q < N; ++q) {
                const double apq = a(p, q);
                if (apq == 0.0) continue;
                const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
                double t;
                if (std::abs(theta) > 1e150)
                    t = 0.5 / theta;
                else
                    t = (theta >= 0.0 ? 1.0 : -1.0) /
                        (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0);
                const double s = t * c;
                for (int k = 0; k < N; ++k) { // columns p, q
                    const double akp = a(k, p), akq = a(k, q);
                    a(k, p) = c * akp - s * akq;
                    a(k, q) = s * akp + c * akq;
                }
                for (int k = 0; k < N; ++k) { // rows p, q
                    const double apk = a(p, k), aqk = a(q, k);
                    a(p, k) = c * apk - s * aqk;
                    a(q, k) = s * apk + c * aqk;
                }
                a(p, q) = 0.0;
                a(q, p) = 0.0;
                for (int k = 0; k < N; ++k) {
                    const double vkp = v(k, p), vkq = v(k, q);
                    v(k, p) = c * vkp - s * vkq;
                    v(k, q) = s * vkp + c * vkq;
                }
            }
    }
    double lam[N];
    for (int i = 0; i < N; ++i) lam[i] = std::max(a(i, i), 0.0);
    MatN<N> out;
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
            double s = 0.0;
            for (int k = 0; k < N; ++k) s += v(i, k) * lam[k] * v(j, k);
            out(i, j) = s;
        }
    return out;
}
template MatN<6> clamp_psd<6>(const MatN<6>&);
template MatN<12> clamp_psd<12>(const MatN<12>&);

// ---------------------------------------------------------------------------
// BlockMatrix
// ---------------------------------------------------------------------------
void BlockMatrix::add(int r, int c, const Mat6& blk) {
    Mat6* dst;
    if (r == c) {
        dst = &diag[r];
    } else {
        dst = &off[{r, c}];
    }
    for (int i = 0; i < 36; ++i) dst->m[i] += blk.m[i];
}

double BlockMatrix::trace() const {
    double s = 0.0;
    for (int b = 0; b < nb; ++b)
        for (int i = 0; i < 6; ++i) s += diag[b](i, i);
    return s;
}

// ---------------------------------------------------------------------------
// LocalObjective (objective.cpp:21-230)
// ---------------------------------------------------------------------------
LocalObjective LocalObjective::assemble(const std::vector<AffineBody>& bodies,
                                        std::vector<int> local, std::vector<double> kappa_b,
                                        std::vector<Vec6> q_tilde,
                                        std::vector<SharedAnchor> anchors,
                                        std::vector<uint32_t> holder_mask,
                                        const SimParams& params) {
    params.validate();
    if (local.size() != kappa_b.size() || local.size() != q_tilde.size())
        throw Error("LocalObjective: body/kappa/q_tilde size mismatch");
    LocalObjective obj;
    obj.bodies_ = &bodies;
    obj.params_ = params;
    obj.holder_mask_ = std::move(holder_mask);
    std::vector<size_t> order(local.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return local[a] < local[b]; });
    for (size_t i : order) {
        obj.local_.push_back(local[i]);
        obj.inv_kappa_.push_back(1.0 / kappa_b[i]);
        obj.q_tilde_.push_back(q_tilde[i]);
    }
    obj.local_pos_.assign(bodies.size(), -1);
    obj.anchor_of_.assign(obj.local_.size(), -1);
    obj.dof_offset_.assign(obj.local_.size(), -1);
    int dof = 0;
    for (size_t i = 0; i < obj.local_.size(); ++i) {
        const int b = obj.local_[i];
        if (b < 0 || b >= static_cast<int>(bodies.size()))
            throw Error("LocalObjective: body index out of range");
        if (obj.local_pos_[b] != -1) throw Error("LocalObjective: duplicate local body");
        obj.local_pos_[b] = static_cast<int>(i);
        if (!bodies[b].is_static) {
            obj.dof_offset_[i] = dof;
            dof += 6;
        }
    }
    obj.num_dofs_ = dof;
    std::sort(anchors.begin(), anchors.end(),
              [](const SharedAnchor& a, const SharedAnchor& b) { return a.body < b.body; });
    for (const SharedAnchor& an : anchors) {
        const int pos = an.body >= 0 && an.body < static_cast<int>(bodies.size())
                            ? obj.local_pos_[an.body]
                            : -1;
        if (pos < 0) throw Error("LocalObjective: anchor for a body not on this worker");
        if (bodies[an.body].is_static) throw Error("LocalObjective: anchor on a static body");
        if (obj.anchor_of_[pos] != -1) throw Error("LocalObjective: duplicate anchor for one body");
        obj.anchor_of_[pos] = static_cast<int>(obj.anchors_.size());
        obj.anchors_.push_back(an);
    }
    return obj;
}

double LocalObjective::contact_weight(int a, int b) const {
    if (holder_mask_.empty()) return 1.0;
    const int kc = std::popcount(holder_mask_[a] & holder_mask_[b]);
    if (kc == 0)
        throw Error("LocalObjective: contact pair visible to no worker (overlap too small)");
    return 1.0 / kc;
}

std::vector<ContactPair> LocalObjective::detect(const Configs& q, int* candidates) const {
    auto cand = broad_phase(*bodies_, q, params_.d_hat, local_);
    cand.erase(std::remove_if(cand.begin(), cand.end(),
                              [this](const ContactPair& p) {
                                  return (*bodies_)[p.body_a].is_static &&
                                         (*bodies_)[p.body_b].is_static;
                              }),
               cand.end());
    if (candidates) *candidates = static_cast<int>(cand.size());
    auto active = narrow_phase(cand, *bodies_, q, params_.d_hat);
    for (ContactPair& p : active) p.kappa_c = 1.0 / contact_weight(p.body_a, p.body_b);
    return active;
}

void LocalObjective::contact_counts(const Configs& q, int& active, int& candidates) const {
    active = static_cast<int>(detect(q, &candidates).size());
}

static double sqn6(const Vec6& v) {
    double s = 0.0;
    for (int i = 0; i < 6; ++i) s += v[i] * v[i];
    return s;
}

double LocalObjective::value(const Configs& q, bool with_anchors) const {
    const double h2 = params_.h * params_.h;
    double total = 0.0;
    for (size_t i = 0; i < local_.size(); ++i) {
        const AffineBody& body = (*bodies_)[local_[i]];
        if (body.is_static) continue;
        const Vec6& qb = q[local_[i]];
        double e = inertia_energy(qb, q_tilde_[i], body.mass_matrix).value;
        e += h2 * arap_energy(qb, params_.arap_stiffness * body.arap_scale, body.rest_area).value;
        total += inv_kappa_[i] * e;
        if (with_anchors && anchor_of_[i] >= 0) {
            const SharedAnchor& a = anchors_[anchor_of_[i]];
            Vec6 d;
            for (int k = 0; k < 6; ++k) d[k] = (qb[k] - a.z[k]) + a.u[k];
            total += 0.5 * a.rho * sqn6(d);
        }
    }
    for (const ContactPair& p : detect(q, nullptr)) {
        const double w = 1.0 / p.kappa_c;
        const double b = barrier_energy(p.d, params_.d_hat, params_.barrier_stiffness).value;
        total += h2 * w * b;
    }
    return total;
}

LocalObjective::Derivatives LocalObjective::derivatives(const Configs& q, bool project) const {
    const double h2 = params_.h * params_.h;
    Derivatives out;
    out.grad.assign(num_dofs_, 0.0);
    out.hess.nb = num_dofs_ / 6;
    out.hess.diag.assign(out.hess.nb, Mat6());
    for (size_t i = 0; i < local_.size(); ++i) {
        const AffineBody& body = (*bodies_)[local_[i]];
        if (body.is_static) continue;
        const Vec6& qb = q[local_[i]];
        const int dof = dof_offset_[i];
        const BodyEnergy in = inertia_energy(qb, q_tilde_[i], body.mass_matrix);
        const BodyEnergy ar =
            arap_energy(qb, params_.arap_stiffness * body.arap_scale, body.rest_area);
        const double ik = inv_kappa_[i];
        double value = ik * (in.value + h2 * ar.value);
        Vec6 grad;
        Mat6 hess;
        for (int k = 0; k < 6; ++k) grad[k] = ik * (in.grad[k] + h2 * ar.grad[k]);
        for (int k = 0; k < 36; ++k) hess.m[k] = ik * (in.hess.m[k] + h2 * ar.hess.m[k]);
        if (anchor_of_[i] >= 0) {
            const SharedAnchor& a = anchors_[anchor_of_[i]];
            Vec6 d;
            for (int k = 0; k < 6; ++k) d[k] = (qb[k] - a.z[k]) + a.u[k];
            value += 0.5 * a.rho * sqn6(d);
            for (int k = 0; k < 6; ++k) grad[k] += a.rho * d[k];
            for (int k = 0; k < 6; ++k) hess(k, k) += a.rho * 1.0;
        }
        out.value += value;
        for (int k = 0; k < 6; ++k) out.grad[dof + k] += grad[k];
        out.hess.add(dof / 6, dof / 6, project ? clamp_psd<6>(hess) : hess);
    }
    int candidates = 0;
    const auto contacts = detect(q, &candidates);
    out.candidate_pairs = candidates;
    out.active_contacts = static_cast<int>(contacts.size());
    for (const ContactPair& p : contacts) {
        const AffineBody& ba = (*bodies_)[p.body_a];
        const AffineBody& bb = (*bodies_)[p.body_b];
        const double w = h2 / p.kappa_c;
        const PairEnergy e = contact_energy(ba, q[p.body_a], bb, q[p.body_b], p.point_index,
                                            p.edge_index, params_.d_hat,
                                            params_.barrier_stiffness);
        out.value += w * e.value;
        Mat12 hw;
        for (int k = 0; k < 144; ++k) hw.m[k] = w * e.hess.m[k];
        const Mat12 hess = project ? clamp_psd<12>(hw) : hw;
        const int da = ba.is_static ? -1 : dof_offset_[local_pos_[p.body_a]];
        const int db = bb.is_static ? -1 : dof_offset_[local_pos_[p.body_b]];
        auto sub = [&hess](int r0, int c0) {
            Mat6 s;
            for (int r = 0; r < 6; ++r)
                for (int c = 0; c < 6; ++c) s(r, c) = hess(r0 + r, c0 + c);
            return s;
        };
        if (da >= 0) {
            for (int k = 0; k < 6; ++k) out.grad[da + k] += w * e.grad[k];
            out.hess.add(da / 6, da / 6, sub(0, 0));
        }
        if (db >= 0) {
            for (int k = 0; k < 6; ++k) out.grad[db + k] += w * e.grad[6 + k];
            out.hess.add(db / 6, db / 6, sub(6, 6));
        }
        if (da >= 0 && db >= 0) {
            out.hess.add(da / 6, db / 6, sub(0, 6));
            out.hess.add(db / 6, da / 6, sub(6, 0));
        }
    }
    return out;
}

void LocalObjective::apply_step(Configs& q, const std::vector<double>& d, double alpha) const {
    for (size_t i = 0; i < local_.size(); ++i) {
        if (dof_offset_[i] < 0) continue;
        for (int k = 0; k < 6; ++k) q[local_[i]][k] += alpha * d[dof_offset_[i] + k];
    }
}

double LocalObjective::config_delta_inf(const Configs& a, const Configs& b) const {
    double best = 0.0;
    for (size_t i = 0; i < local_.size(); ++i) {
        if (dof_offset_[i] < 0) continue;
        double m = 0.0;
        for (int k = 0; k < 6; ++k) m = std::max(m, std::abs(a[local_[i]][k] - b[local_[i]][k]));
        best = std::max(best, m);
    }
    return best;
}

// ---------------------------------------------------------------------------
// Block-sparse Cholesky with minimum-degree ordering (SimplicialLDLT stand-in)
// ---------------------------------------------------------------------------
namespace {

bool chol6(const Mat6& a, Mat6& l) {
    l = Mat6();
    for (int j = 0; j < 6; ++j) {
        double s = a(j, j);
        for (int k = 0; k < j; ++k) s -= l(j, k) * l(j, k);
        if (!(s > 0.0)) return false;
        const double d = std::sqrt(s);
        l(j, j) = d;
        for (int i = j + 1; i < 6; ++i) {
            double t = a(i, j);
            for (int k = 0; k < j; ++k) t -= l(i, k) * l(j, k);
            l(i, j) = t / d;
        }
    }
    return true;
}

// X = B * L^{-T}  (solve X L^T = B)
Mat6 right_solve_lt(const Mat6& b, const Mat6& l) {
    Mat6 x;
    for (int r = 0; r < 6; ++r)
        for (int j = 0; j < 6; ++j) {
            double s = b(r, j);
            for (int k = 0; k < j; ++k) s -= x(r, k) * l(j, k);
            x(r, j) = s / l(j, j);
        }
    return x;
}

} // namespace

std::vector<double> block_sparse_solve(const BlockMatrix& h, double eps,
                                       const std::vector<double>& rhs) {
    const int n = h.nb;
    std::vector<std::set<int>> adj(n);
    for (const auto& kv : h.off) {
        adj[kv.first.first].insert(kv.first.second);
        adj[kv.first.second].insert(kv.first.first);
    }
    // Minimum-degree elimination on the block graph.
    std::set<std::pair<int, int>> pq;
    for (int i = 0; i < n; ++i) pq.insert({static_cast<int>(adj[i].size()), i});
    std::vector<int> perm, iperm(n, -1);
    std::vector<std::vector<int>> col(n); // structure in original ids
    perm.reserve(n);
    while (!pq.empty()) {
        const int v = pq.begin()->second;
        pq.erase(pq.begin());
        iperm[v] = static_cast<int>(perm.size());
        perm.push_back(v);
        std::vector<int> nb(adj[v].begin(), adj[v].end());
        col[v] = nb;
        for (int u : nb) {
            pq.erase({static_cast<int>(adj[u].size()), u});
            adj[u].erase(v);
            for (int w2 : nb)
                if (w2 != u) adj[u].insert(w2);
            pq.insert({static_cast<int>(adj[u].size()), u});
        }
        adj[v].clear();
    }
    // Numeric factorization (right-looking, new ordering).
    std::vector<Mat6> dblk(n);
    std::vector<std::vector<int>> cs(n); // column structure, new ids, ascending
    std::map<std::pair<int, int>, Mat6> lo;  // (i, j) i > j, new ids
    for (int k = 0; k < n; ++k) {
        dblk[k] = h.diag[perm[k]];
        for (int i = 0; i < 6; ++i) dblk[k](i, i) += eps;
        for (int u : col[perm[k]]) cs[k].push_back(iperm[u]);
        std::sort(cs[k].begin(), cs[k].end());
    }
    for (const auto& kv : h.off) {
        const int i = iperm[kv.first.first], j = iperm[kv.first.second];
        if (i > j) lo[{i, j}] = kv.second;
    }
    std::vector<Mat6> lkk(n);
    for (int k = 0; k < n; ++k) {
        if (!chol6(dblk[k], lkk[k])) throw Error("newton_solve: factorization failed");
        std::vector<Mat6*> lik(cs[k].size());
        for (size_t a = 0; a < cs[k].size(); ++a) {
            Mat6& blk = lo[{cs[k][a], k}];
            blk = right_solve_lt(blk, lkk[k]);
            lik[a] = &blk;
        }
        for (size_t a = 0; a < cs[k].size(); ++a) {
            const int i = cs[k][a];
            for (size_t b = 0; b <= a; ++b) {
                const int j = cs[k][b];
                Mat6* dst = (i == j) ? &dblk[i] : &lo[{i, j}];
                const Mat6& li = *lik[a];
                const Mat6& lj = *lik[b];
                for (int r = 0; r < 6; ++r)
                    for (int c = 0; c < 6; ++c) {
                        double s = 0.0;
                        for (int t = 0; t < 6; ++t) s += li(r, t) * lj(c, t);
                        (*dst)(r, c) -= s;
                    }
            }
        }
    }
    // Solve.
    std::vector<double> y(6 * n);
    for (int k = 0; k < n; ++k)
        for (int i = 0; i < 6; ++i) y[6 * k + i] = rhs[6 * perm[k] + i];
    for (int k = 0; k < n; ++k) {
        double* yk = &y[6 * k];
        for (int i = 0; i < 6; ++i) {
            double s = yk[i];
            for (int t = 0; t < i; ++t) s -= lkk[k](i, t) * yk[t];
            yk[i] = s / lkk[k](i, i);
        }
        for (int i : cs[k]) {
            const Mat6& l = lo[{i, k}];
            for (int r = 0; r < 6; ++r) {
                double s = 0.0;
                for (int t = 0; t < 6; ++t) s += l(r, t) * yk[t];
                y[6 * i + r] -= s;
            }
        }
    }
    for (int k = n - 1; k >= 0; --k) {
        double* yk = &y[6 * k];
        for (int i : cs[k]) {
            const Mat6& l = lo[{i, k}];
            for (int t = 0; t < 6; ++t) {
                double s = 0.0;
                for (int r = 0; r < 6; ++r) s += l(r, t) * y[6 * i + r];
                yk[t] -= s;
            }
        }
        for (int i = 5; i >= 0; --i) {
            double s = yk[i];
            for (int t = i + 1; t < 6; ++t) s -= lkk[k](t, i) * yk[t];
            yk[i] = s / lkk[k](i, i);
        }
    }
    std::vector<double> x(6 * n);
    for (int k = 0; k < n; ++k)
        for (int i = 0; i < 6; ++i) x[6 * perm[k] + i] = y[6 * k + i];
    return x;
}

// newton.cpp:7-71
NewtonReport newton_solve(const LocalObjective& obj, Configs& q, const NewtonOptions& opt) {
    NewtonReport rep;
    if (obj.num_dofs() == 0) {
        rep.converged = true;
        return rep;
    }
    double energy = obj.value(q);
    for (int iter = 0; iter < opt.max_iters; ++iter) {
        const auto der = obj.derivatives(q);
        ++rep.iterations;
        const double eps = 1e-8 * der.hess.trace() / obj.num_dofs();
        std::vector<double> rhs(der.grad.size());
        for (size_t i = 0; i < rhs.size(); ++i) rhs[i] = -der.grad[i];
        const std::vector<double> dq = block_sparse_solve(der.hess, eps, rhs);
        double dq_inf = 0.0;
        for (double v : dq) dq_inf = std::max(dq_inf, std::abs(v));
        if (dq_inf < opt.tol) {
            rep.final_update_inf = dq_inf;
            rep.converged = true;
            break;
        }
        Configs q_end = q;
        obj.apply_step(q_end, dq, 1.0);
        const double alpha_max = ccd_toi_scene(obj.bodies(), q, q_end, obj.local_bodies());
        double alpha = alpha_max;
        double slope = 0.0;
        for (size_t i = 0; i < dq.size(); ++i) slope += der.grad[i] * dq[i];
        bool accepted = false;
        while (alpha >= 1e-12) {
            Configs q_try = q;
            obj.apply_step(q_try, dq, alpha);
            const double trial = obj.value(q_try);
            if (trial < energy + opt.armijo_c * alpha * slope) {
                q = std::move(q_try);
                energy = trial;
                accepted = true;
                break;
            }
            alpha *= 0.5;
            ++rep.line_search_steps;
        }
        if (!accepted)
            throw Error("newton_solve: line search failed below 1e-12 (non-descent direction)");
        rep.final_update_inf = alpha * dq_inf;
        if (rep.final_update_inf < opt.tol) {
            rep.converged = true;
            break;
        }
    }
    return rep;
}

} // namespace oracle
