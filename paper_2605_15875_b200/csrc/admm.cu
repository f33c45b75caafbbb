// Frame-level and consensus-ADMM kernels: state gather, prediction, holder
// masks, overlap width, consensus/dual/residuals, rho adaptation, merge
// targets and the commit (proj/src/consensus.cpp:9-86, partition.cpp:36-67,
// body.cpp:120-161, runtime.cpp:241-277, 361-397, 457-506).
#include "admm.hpp"

#include "instrument.hpp"

namespace dabd_gpu {

namespace {

constexpr int kB = 128;

__global__ void k_gather(int n, const int* ibody, const double* q, double* iq) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 6 * n; t += gridDim.x * blockDim.x)
        iq[t] = q[6 * ibody[t / 6] + t % 6];
}

// PCG warm-start vectors carried to a new instance set: row r takes the
// previous row map[r] (same (partition, body)) or starts from zero. prev holds
// the previous x (6 R_old) followed by the previous p2 (6 R_old).
__global__ void k_warm_remap(int n_rows, const int* map, const double* prev, int r_old, double* x,
                             double* p2) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 6 * n_rows; t += gridDim.x * blockDim.x) {
        const int m = map[t / 6];
        const size_t e = 6 * static_cast<size_t>(m) + t % 6;
        x[t] = m >= 0 ? prev[e] : 0.0;
        p2[t] = m >= 0 ? prev[6 * static_cast<size_t>(r_old) + e] : 0.0;
    }
}

// q_tilde = q + h qdot + h^2 M^{-1} f, f = m g (+ replica force split) on the
// translation slots (body.cpp:120-134, runtime.cpp:252-264).
__global__ void k_predict(SceneView sc, int n, const int* ibody, const double* iq,
                          const double* qd, double h, double gx, double gy, const double* ifs,
                          double* iqt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int b = ibody[i];
        const double* q = iq + 6 * i;
        double* o = iqt + 6 * i;
        if (sc.is_static[b]) {
            for (int k = 0; k < 6; ++k) o[k] = q[k];
            continue;
        }
        double f0 = sc.mass[b] * gx, f1 = sc.mass[b] * gy;
        if (ifs) {
            f0 += ifs[2 * i];
            f1 += ifs[2 * i + 1];
        }
        const double* mi = sc.minv + 3 * b;
        double x[6];
        x[0] = f0 * mi[0];
        x[2] = f0 * mi[1];
        x[3] = f0 * mi[2];
        x[1] = f1 * mi[0];
        x[4] = f1 * mi[1];
        x[5] = f1 * mi[2];
        const double h2 = xmul(h, h);
        const double* v = qd + 6 * b;
        for (int k = 0; k < 6; ++k) o[k] = xadd(xadd(q[k], xmul(h, v[k])), xmul(h2, x[k]));
    }
}

__global__ void k_delta_inf(int n_rows, const int* rinst, const int* rpart, int part_base,
                            const double* a, const double* b, double* out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        const int i = rinst[r];
        double m = 0.0;
        for (int k = 0; k < 6; ++k) m = fmax(m, fabs(a[6 * i + k] - b[6 * i + k]));
        atomic_max_nonneg(&out[rpart[r] - part_base], m);
    }
}

// body_holder_mask (partition.cpp:36-67), bit-exact.
__global__ void k_masks(SceneView sc, const double* q, const double* planes, int np, double w,
                        uint32_t all, uint32_t* masks, int* err, const double* vmax_dev = nullptr,
                        double h = 0.0, double w_min = 0.0, double* w_out = nullptr) {
    if (vmax_dev) { // overlap width on the device: max(2 v_max h, w_min), host rounding (runtime.cpp:556-560)
        const double x = xmul(xmul(2.0, *vmax_dev), h);
        w = x < w_min ? w_min : x;
        if (w_out && blockIdx.x == 0 && threadIdx.x == 0) *w_out = w;
    }
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < sc.nb; b += gridDim.x * blockDim.x) {
        if (sc.is_static[b]) {
            masks[b] = all;
            continue;
        }
        const double* qb = q + 6 * b;
        V2 lo{1.7976931348623157e308, 1.7976931348623157e308}, hi{-1.7976931348623157e308,
                                                                  -1.7976931348623157e308};
        for (int v = sc.vstart[b]; v < sc.vstart[b + 1]; ++v) {
            const double2 r = sc.rest[v];
            const V2 x = world_point(qb, V2{r.x, r.y});
            lo = vmin(lo, x);
            hi = vmax(hi, x);
        }
        const double hw = xdiv(w, 2.0);
        int hit = -1;
        bool bad = false;
        for (int k = 0; k < np; ++k) {
            const V2 pt{planes[4 * k], planes[4 * k + 1]}, nn{planes[4 * k + 2], planes[4 * k + 3]};
            double slo = 1.7976931348623157e308, shi = -1.7976931348623157e308;
            for (int corner = 0; corner < 4; ++corner) {
                const V2 c{(corner & 1) ? hi.x : lo.x, (corner & 2) ? hi.y : lo.y};
                const double s = vdot(vsub(c, pt), nn);
                slo = fmin(slo, s);
                shi = fmax(shi, s);
            }
            if (slo <= hw && shi >= -hw) {
                if (hit >= 0) bad = true;
                hit = k;
            }
        }
        if (bad) {
            raise(err, kErrStraddle);
            masks[b] = 0;
            continue;
        }
        if (hit >= 0) {
            masks[b] = (1u << hit) | (1u << (hit + 1));
            continue;
        }
        const V2 c{qb[0], qb[1]};
        int region = 0;
        for (int k = 0; k < np; ++k) {
            const V2 pt{planes[4 * k], planes[4 * k + 1]}, nn{planes[4 * k + 2], planes[4 * k + 3]};
            if (vdot(vsub(c, pt), nn) <= 0.0) ++region;
        }
        masks[b] = 1u << region;
    }
}

// max_vertex_speed over dynamic bodies (body.cpp:151-161), exact max.
__global__ void k_vmax(SceneView sc, const double* qd, double* out) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < sc.nb; b += gridDim.x * blockDim.x) {
        if (sc.is_static[b]) continue;
        const double* v = qd + 6 * b;
        double best = 0.0;
        for (int k = sc.vstart[b]; k < sc.vstart[b + 1]; ++k) {
            const double2 r = sc.rest[k];
            const double vx = xadd(xadd(v[0], xmul(v[2], r.x)), xmul(v[3], r.y));
            const double vy = xadd(xadd(v[1], xmul(v[4], r.x)), xmul(v[5], r.y));
            best = fmax(best, xsqrt(xadd(xmul(vx, vx), xmul(vy, vy))));
        }
        atomic_max_nonneg(out, best);
    }
}

// Consensus over the two replicas of each shared body (consensus.cpp:9-36,
// runtime.cpp:365-397): z = sum rho (q + u) / sum rho in ascending worker
// order, u' = u + q - z, r_b, s_b.
//
// A replica handle v >= 0 is a local instance; v < 0 is the halo packet
// -1 - v received from the neighbouring rank (q[6], u[6], rho). Both ranks of
// a cross-GPU pair evaluate the same expression in the same (ascending
// partition) order, so they agree on z bit for bit; each updates only its
// own replica.
struct Replica {
    const double* q;
    double* u;
    double rho;
    int inst; // -1 when remote
};

// Remote packets j < n_lo come from rank - 1 (at remote_lo), the others from
// rank + 1 (at remote_hi, index j - n_lo). With the peer-memory halo these
// are the neighbours' own published buffers (CUDA IPC mappings: NVLink loads
// on a multi-GPU box), so the exchange is fused into this kernel's reads.
__device__ __forceinline__ Replica replica(int v, const double* iq, double* iu, const double* irho,
                                           const double* remote_lo, const double* remote_hi, int n_lo) {
    if (v >= 0) return Replica{iq + 6 * v, iu + 6 * v, irho[v], v};
    const int j = -1 - v;
    const double* p = j < n_lo ? remote_lo + kHaloStride * j : remote_hi + kHaloStride * (j - n_lo);
    return Replica{p, const_cast<double*>(p + 6), p[12], -1};
}

__global__ void k_consensus(int ns, const int* sh, const int* ipart, int part_base,
                            const double* iq, double* iu, const double* irho, const double* iz,
                            const double* remote_lo, const double* remote_hi, int n_lo,
                            double* iznext, double* rb, double* sb, double* rloc, double* sloc,
                            int* err, const FrameCtrl* pc = nullptr, size_t reg = 0) {
    if (pc) { // device ADMM loop: the neighbours' publish regions of this iteration's parity
        const int par = pc->k & 1;
        if (remote_lo) remote_lo += (1 * 2 + par) * reg;
        if (remote_hi) remote_hi += (0 * 2 + par) * reg;
    }
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
        const Replica a = replica(sh[2 * s], iq, iu, irho, remote_lo, remote_hi, n_lo);
        const Replica b = replica(sh[2 * s + 1], iq, iu, irho, remote_lo, remote_hi, n_lo);
        if (a.rho != b.rho) raise(err, kErrReplica);
        double z[6];
        const double den = xadd(xadd(0.0, a.rho), b.rho);
        for (int k = 0; k < 6; ++k) {
            const double qu0 = xadd(a.q[k], a.u[k]);
            const double qu1 = xadd(b.q[k], b.u[k]);
            const double num = xadd(xadd(0.0, xmul(a.rho, qu0)), xmul(b.rho, qu1));
            z[k] = xdiv(num, den);
        }
        double rmax = 0.0;
        for (int k = 0; k < 6; ++k) {
            rmax = fmax(rmax, fabs(xsub(a.q[k], z[k])));
            rmax = fmax(rmax, fabs(xsub(b.q[k], z[k])));
        }
        const int mine[2] = {a.inst, b.inst};
        for (int side = 0; side < 2; ++side) {
            const int i = mine[side];
            if (i < 0) continue;
            double sm = 0.0;
            for (int k = 0; k < 6; ++k) {
                sm = fmax(sm, fabs(xsub(z[k], iz[6 * i + k])));
                iu[6 * i + k] = xsub(xadd(iu[6 * i + k], iq[6 * i + k]), z[k]);
                iznext[6 * i + k] = z[k];
            }
            rb[i] = rmax;
            sb[i] = sm;
            const int p = ipart[i] - part_base;
            atomic_max_nonneg(&rloc[p], rmax);
            atomic_max_nonneg(&sloc[p], sm);
        }
    }
}

// Halo packets of the local replicas a neighbouring rank pairs with.
__global__ void k_pack_halo(int n, const int* inst, const double* iq, const double* iu,
                            const double* irho, double* out, const FrameCtrl* pc = nullptr, int side = 0,
                            size_t reg = 0) {
    if (pc) out += (side * 2 + (pc->k & 1)) * reg; // [side][parity] publish region
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int i = inst[j];
        double* o = out + kHaloStride * j;
        for (int k = 0; k < 6; ++k) {
            o[k] = iq[6 * i + k];
            o[6 + k] = iu[6 * i + k];
        }
        o[12] = irho[i];
    }
}

// After the commit all-gather: every dynamic body takes the state written by
// the rank that holds its lowest partition (runtime.cpp:484-506 "the lowest
// holder commits").
__global__ void k_select_commit(SceneView sc, const uint32_t* bmask, const int* part_rank,
                                const double* gath, size_t stride, double* q, double* qd) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < sc.nb; b += gridDim.x * blockDim.x) {
        if (sc.is_static[b]) continue;
        const int r = part_rank[__ffs(bmask[b]) - 1];
        const double* src = gath + stride * r;
        for (int k = 0; k < 6; ++k) {
            q[6 * b + k] = src[6 * b + k];
            qd[6 * b + k] = src[6 * sc.nb + 6 * b + k];
        }
    }
}

// Candidate merged state: shared replicas moved to z (consensus.cpp:66-75).
__global__ void k_merged(int n, const int* ianc, const double* iq, const double* iznext,
                         double* out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 6 * n; t += gridDim.x * blockDim.x)
        out[t] = ianc[t / 6] ? iznext[t] : iq[t];
}

// consensus.cpp:44-52 applied per shared replica (runtime.cpp:457-461),
// followed by z = z_next (runtime.cpp:462).
__global__ void k_adapt(int n, const int* ianc, double* irho, const double* irho0, const double* rb,
                        const double* sb, double tau, double mu, double smin, double smax,
                        int enabled, double* iz, const double* iznext, const FrameCtrl* skip_first) {
    if (skip_first && skip_first->k == 1) return; // device ADMM frame: no consensus before the first solve
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (!ianc[i]) continue;
        if (enabled) {
            const double rho = irho[i], r = rb[i], s = sb[i], r0 = irho0[i];
            double next = rho;
            if (r > mu * s)
                next = tau * rho;
            else if (s > mu * r)
                next = rho / tau;
            const double lo = smin * r0, hi = smax * r0;
            irho[i] = next < lo ? lo : (hi < next ? hi : next);
        }
        for (int k = 0; k < 6; ++k) iz[6 * i + k] = iznext[6 * i + k];
    }
}

// Commit (consensus.cpp:77-86, runtime.cpp:484-506): shared replicas take z,
// qdot = (q - q_start) / h, the lowest-rank holder writes the global state.
__global__ void k_commit(SceneView sc, int n, const int* ibody, const int* ipart, const int* ianc,
                         const uint32_t* bmask, double* iq, const double* iznext,
                         const double* q_start, double h, double* q, double* qd) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int b = ibody[i];
        if (sc.is_static[b]) continue;
        double* qi = iq + 6 * i;
        if (ianc[i])
            for (int k = 0; k < 6; ++k) qi[k] = iznext[6 * i + k];
        const bool owner = bmask == nullptr || (__ffs(bmask[b]) - 1) == ipart[i];
        if (!owner) continue;
        for (int k = 0; k < 6; ++k) {
            q[6 * b + k] = qi[k];
            qd[6 * b + k] = xdiv(xsub(qi[k], q_start[6 * b + k]), h);
        }
    }
}

__global__ void k_accept_copy(int n, const int* ipart, int part_base, const PartState* ps,
                              const double* src, double* dst) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 6 * n; t += gridDim.x * blockDim.x)
        if (ps[ipart[t / 6] - part_base].accepted) dst[t] = src[t];
}


// ---- device-side instance sets (runtime.cpp:126-236) ----------------------
__global__ void k_inst_flags(SceneView sc, const uint32_t* masks, int P, int p0, int* f_all, int* f_dyn,
                             int* f_sh) {
    const long long n = static_cast<long long>(P) * sc.nb;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(t / sc.nb), b = static_cast<int>(t - static_cast<long long>(p) * sc.nb);
        const uint32_t m = masks[b];
        const int in = static_cast<int>((m >> (p0 + p)) & 1u);
        const int dyn = in && !sc.is_static[b];
        f_all[t] = in;
        f_dyn[t] = dyn;
        f_sh[t] = dyn && __popc(m) >= 2 && (p0 + p) != __ffs(m) - 1;
    }
}

__global__ void k_inst_counts(int P, int nb, const int* f_all, const int* f_dyn, const int* f_sh,
                              const int* s_all, const int* s_dyn, const int* s_sh, int* counts) {
    const long long n = static_cast<long long>(P) * nb;
    const long long last = n - 1;
    if (threadIdx.x == 0) {
        counts[0] = n ? s_all[last] + f_all[last] : 0;
        counts[1] = n ? s_dyn[last] + f_dyn[last] : 0;
        counts[2] = n ? s_sh[last] + f_sh[last] : 0;
    }
    for (int p = threadIdx.x; p <= P; p += blockDim.x) {
        const long long t = static_cast<long long>(p) * nb;
        counts[3 + p] = p < P ? (n ? s_all[t] : 0) : (n ? s_all[last] + f_all[last] : 0);
        counts[4 + P + p] = p < P ? (n ? s_dyn[t] : 0) : (n ? s_dyn[last] + f_dyn[last] : 0);
    }
}

__global__ void k_inst_scatter(SceneView sc, const uint32_t* masks, int P, int p0, const int* f_all,
                               const int* f_dyn, const int* f_sh, const int* s_all, const int* s_dyn,
                               const int* s_sh, double beta, const double* rho_carry,
                               const int* rowtab_prev, InstOut o) {
    const int nb = sc.nb;
    const long long n = static_cast<long long>(P) * nb;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int dyn = f_dyn[t];
        o.rowtab[t] = dyn ? s_dyn[t] : -1;
        if (!f_all[t]) continue;
        const int p = static_cast<int>(t / nb), b = static_cast<int>(t - static_cast<long long>(p) * nb);
        const uint32_t m = masks[b];
        const int i = s_all[t];
        const int kb = __popc(m);
        o.ibody[i] = b;
        o.ipart[i] = p0 + p;
        o.invk[i] = 1.0 / kb;
        const int anc = dyn && kb >= 2;
        o.ianc[i] = anc;
        const double r0 = anc ? xmul(beta, sc.mass[b]) : 0.0; // init_rho (consensus.cpp:38-42)
        o.rho0[i] = r0;
        o.rho[i] = anc ? (isnan(rho_carry[b]) ? r0 : rho_carry[b]) : 0.0;
        if (dyn) {
            const int row = s_dyn[t];
            o.irow[i] = row;
            o.rinst[row] = i;
            o.rpart[row] = p0 + p;
            o.wmap[row] = rowtab_prev ? rowtab_prev[t] : -1;
        } else {
            o.irow[i] = -1;
            o.stat[i - s_dyn[t]] = i;
        }
        if (f_sh[t]) { // (first replica, this replica) in instance order
            const int j = s_sh[t];
            const int lowp = __ffs(m) - 1 - p0;
            o.shared[2 * j] = s_all[static_cast<long long>(lowp) * nb + b];
            o.shared[2 * j + 1] = i;
        }
    }
}

__global__ void k_rho_carry(int n_inst, int nb, const int* ibody, const int* ianc, const double* irho,
                            double* carry) {
    const int t0 = blockIdx.x * blockDim.x + threadIdx.x, st = gridDim.x * blockDim.x;
    for (int b = t0; b < nb; b += st) carry[b] = __longlong_as_double(0x7ff8000000000000ll);
    __syncthreads();
    // replicas carry equal rho (k_consensus checks it): any one may stand in;
    // a grid-stride pass after a grid-wide NaN fill needs the fill first, so
    // the fill and the writes run in one block
    for (int i = t0; i < n_inst; i += st)
        if (ianc[i]) carry[ibody[i]] = irho[i];
}

__global__ void k_pack_owned(SceneView sc, const uint32_t* bmask, int p0, int p1, const double* q,
                             const double* qd, double* rec, int* count) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < sc.nb; b += gridDim.x * blockDim.x) {
        if (sc.is_static[b]) continue;
        const int owner = __ffs(bmask[b]) - 1;
        if (owner < p0 || owner >= p1) continue;
        double* o = rec + 13 * static_cast<size_t>(atomicAdd(count, 1)); // slot order is irrelevant: keyed by id
        o[0] = b;
        for (int k = 0; k < 6; ++k) {
            o[1 + k] = q[6 * b + k];
            o[7 + k] = qd[6 * b + k];
        }
    }
}

__global__ void k_unpack_owned(int world, const int* counts, const double* gath, size_t stride, double* q,
                               double* qd) {
    for (int r = 0; r < world; ++r) {
        const double* g = gath + stride * r;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < counts[r]; i += gridDim.x * blockDim.x) {
            const double* rc = g + 13 * static_cast<size_t>(i);
            const int b = static_cast<int>(rc[0]);
            for (int k = 0; k < 6; ++k) {
                q[6 * b + k] = rc[1 + k];
                qd[6 * b + k] = rc[7 + k];
            }
        }
    }
}

// ---- device fan-in across ranks (partition-per-GPU device ADMM loop) ------
// Every rank owns a fan-in buffer [world][rec_len] records + [world] flags,
// mapped into every peer (CUDA IPC). post: this rank's record (if any) into
// slot `rank` of every peer's buffer, a system fence, then the flag = the
// next sequence number; wait: until every flag of the local buffer reached
// the local sequence number. Every rank posts the same sequence of rounds.
__global__ void k_fan_post(FanView f, const double* rec, int rec_len) {
    if (threadIdx.x != 0) return;
    const unsigned long long seq = ++(*f.seq);
    for (int r = 0; r < f.world; ++r) {
        double* dst = f.peer_rec[r] + static_cast<size_t>(f.rank) * f.rec_stride;
        for (int k = 0; k < rec_len; ++k) dst[k] = rec[k];
    }
    __threadfence_system();
    for (int r = 0; r < f.world; ++r)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f.peer_flag[r] + f.rank), "l"(seq) : "memory");
}

__global__ void k_fan_wait(FanView f) {
    if (threadIdx.x != 0) return;
    const unsigned long long seq = *f.seq;
    for (int r = 0; r < f.world; ++r) {
        while (true) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f.local_flag + r) : "memory");
            if (v >= seq) break;
            __nanosleep(200);
        }
    }
    __threadfence_system();
}

// this rank's fan-in record: (n_parts, fail, then per partition dq, r, s, earliest TOI)
__global__ void k_fan_record(int P, const double* dq, const double* rloc, const double* sloc,
                             const double* gate, const int* err, double* rec) {
    if (threadIdx.x != 0) return;
    rec[0] = P;
    rec[1] = *err != 0 ? 1.0 : 0.0;
    for (int p = 0; p < P; ++p) {
        rec[2 + 4 * p] = dq[p];
        rec[3 + 4 * p] = rloc[p];
        rec[4 + 4 * p] = sloc[p];
        rec[5 + 4 * p] = gate[p];
    }
}

__device__ __forceinline__ void admm_cond(unsigned long long h, bool v, int graph) {
    if (graph) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(h), v ? 1u : 0u);
}

// one warp; lane p < P handles partition p where partitions are independent
__global__ void k_admm_ctrl(AdmmCtrlArgs a, int op) {
    FrameCtrl* c = a.c;
    const int lane = threadIdx.x;
    const bool graph = a.hd.graph != 0;
    if (op == kAdmmInit) {
        if (lane == 0) {
            c->k = 1;
            c->ended = c->failed = 0;
            c->sigma = 0;
            c->admm_iterations = 0;
            c->trace_n = 0;
            c->newton_total = c->ls_total = c->pcg_total = 0;
            c->exec_admm = c->exec_gate = c->exec_solve = 0;
            c->exec_newton = c->exec_step = c->exec_ls = 0;
            c->gate_max = 0;
            admm_cond(a.hd.admm, true, graph);
        }
        for (int p = lane; p < a.P; p += 32) {
            a.dq[p] = 0.0;
            a.cost[p] = 0.0;
        }
        return;
    }
    if (op == kAdmmHead) {
        const bool gate = c->k > 1;
        for (int p = lane; p < a.P; p += 32) {
            a.gate[p] = 2.0;
            a.rloc[p] = 0.0;
            a.sloc[p] = 0.0;
        }
        if (lane == 0) {
            ++c->exec_admm;
            admm_cond(a.hd.gate, gate, graph);
            admm_cond(a.hd.solve, !gate, graph); // k = 1: straight to the local solve
        }
        return;
    }
    if (op == kAdmmDecide) {
        if (lane != 0) return;
        ++c->exec_gate;
        const int gc = *a.gate_count;
        if (gc > c->gate_max) c->gate_max = gc;
        int sigma = 0;
        bool fail = *a.err != 0;
        if (a.fan_rec)
            for (int rk = 0; rk < a.fan_world; ++rk) fail = fail || a.fan_rec[static_cast<size_t>(rk) * a.fan_stride + 1] != 0.0;
        if (fail) {
            sigma = -1;
        } else {
            // runtime.cpp:586-619: every partition's (dq, r, s, earliest TOI),
            // of every rank in partition order when the frame is distributed
            double dq = 0.0, r = 0.0, sres = 0.0, toi = 1.0;
            bool all_one = true;
            auto take = [&](double dqp, double rp, double sp, double e) {
                const double t = e > 1.0 ? 1.0 : fmin(1.0, __dmul_rn(0.9, e));
                dq = fmax(dq, dqp);
                r = fmax(r, rp);
                sres = fmax(sres, sp);
                toi = fmin(toi, t);
                all_one = all_one && t == 1.0;
            };
            if (a.fan_rec) {
                for (int rk = 0; rk < a.fan_world; ++rk) {
                    const double* rc = a.fan_rec + static_cast<size_t>(rk) * a.fan_stride;
                    for (int p = 0; p < static_cast<int>(rc[0]); ++p)
                        take(rc[2 + 4 * p], rc[3 + 4 * p], rc[4 + 4 * p], rc[5 + 4 * p]);
                }
            } else {
                for (int p = 0; p < a.P; ++p) take(a.dq[p], a.rloc[p], a.sloc[p], a.gate[p]);
            }
            const double nrm = __dmul_rn(a.h, a.l); // consensus.cpp:54-64
            const bool end = __ddiv_rn(dq, nrm) < a.theta && __ddiv_rn(r, nrm) < a.theta &&
                             __ddiv_rn(sres, nrm) < a.theta && all_one;
            if (end) sigma = 1;
            else if (c->k == a.K) sigma = c->can_halve ? 2 : 3;
            if (a.trace && c->trace_n < a.trace_cap) {
                double* row = a.trace + 8 * c->trace_n;
                row[0] = c->frame;
                row[1] = c->attempt;
                row[2] = c->k;
                row[3] = dq;
                row[4] = r;
                row[5] = sres;
                row[6] = toi;
                row[7] = sigma;
            }
            ++c->trace_n;
            if (sigma == 1) {
                c->ended = 1;
                c->admm_iterations = c->k;
            }
        }
        c->sigma = sigma;
        admm_cond(a.hd.solve, sigma == 0, graph);
        admm_cond(a.hd.admm, sigma == 0, graph);
        return;
    }
    // kAdmmTail
    __shared__ int s_err;
    if (lane == 0) {
        ++c->exec_solve;
        s_err = *a.err;
    }
    __syncwarp();
    for (int p = lane; p < a.P; p += 32) {
        const PartState& s = a.ps[p];
        a.dq[p] = a.dq_new[p];
        // balancer cost (engine.cu partition_cost)
        const double rows = s.ndof / 6.0;
        a.cost[p] += fmax(1.0, s.iterations * (rows + 2.0 * s.n_active_contacts) + s.pcg_total * rows);
    }
    if (lane == 0) {
        for (int p = 0; p < a.P; ++p) {
            c->newton_total += a.ps[p].iterations;
            c->ls_total += a.ps[p].ls_steps;
        }
        c->k += 1;
        if (s_err != 0 && !a.fan_rec) { // distributed: the next fan-in carries the failure to every rank
            c->sigma = -1;
            admm_cond(a.hd.admm, false, graph);
        }
    }
}

} // namespace

void launch_gather(int n, const int* ibody, const double* q, double* iq, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_gather", s, k_gather<<<grid_for(6ll * n, kB), kB, 0, s>>>(n, ibody, q, iq));
}

void launch_warm_remap(int n_rows, const int* map, const double* prev, int r_old, double* x,
                       double* p2, cudaStream_t s) {
    if (n_rows == 0) return;
    DABD_LAUNCH("k_warm_remap", s, k_warm_remap<<<grid_for(6ll * n_rows, kB), kB, 0, s>>>(n_rows, map, prev, r_old, x, p2));
}

void launch_predict(const SceneView& sc, int n, const int* ibody, const double* iq,
                    const double* qd, double h, double gx, double gy, const double* ifs,
                    double* iqt, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_predict", s, k_predict<<<grid_for(n, kB), kB, 0, s>>>(sc, n, ibody, iq, qd, h, gx, gy, ifs, iqt));
}

void launch_delta_inf(int n_rows, const int* rinst, const int* rpart, int part_base,
                      const double* a, const double* b, double* out, cudaStream_t s) {
    if (n_rows == 0) return;
    DABD_LAUNCH("k_delta_inf", s, k_delta_inf<<<grid_for(n_rows, kB), kB, 0, s>>>(n_rows, rinst, rpart, part_base, a, b, out));
}

void launch_masks(const SceneView& sc, const double* q, const double* planes, int np, double w,
                  uint32_t all, uint32_t* masks, int* err, cudaStream_t s) {
    if (sc.nb == 0) return;
    DABD_LAUNCH("k_masks", s, k_masks<<<grid_for(sc.nb, kB), kB, 0, s>>>(sc, q, planes, np, w, all, masks, err));
}

void launch_vmax(const SceneView& sc, const double* qd, double* out, cudaStream_t s) {
    if (sc.nb == 0) return;
    DABD_LAUNCH("k_vmax", s, k_vmax<<<grid_for(sc.nb, kB), kB, 0, s>>>(sc, qd, out));
}

void launch_consensus(int ns, const int* sh, const int* ipart, int part_base, const double* iq,
                      double* iu, const double* irho, const double* iz, const double* remote_lo,
                      const double* remote_hi, int n_lo, double* iznext, double* rb, double* sb,
                      double* rloc, double* sloc, int* err, cudaStream_t s) {
    if (ns == 0) return;
    DABD_LAUNCH("k_consensus", s, k_consensus<<<grid_for(ns, kB), kB, 0, s>>>(ns, sh, ipart, part_base, iq, iu, irho, iz,
                                                                             remote_lo, remote_hi, n_lo, iznext, rb,
                                                                             sb, rloc, sloc, err));
}

void launch_pack_halo(int n, const int* inst, const double* iq, const double* iu,
                      const double* irho, double* out, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_pack_halo", s, k_pack_halo<<<grid_for(n, kB), kB, 0, s>>>(n, inst, iq, iu, irho, out));
}

void launch_select_commit(const SceneView& sc, const uint32_t* bmask, const int* part_rank,
                          const double* gath, size_t stride, double* q, double* qd,
                          cudaStream_t s) {
    if (sc.nb == 0) return;
    DABD_LAUNCH("k_select_commit", s, k_select_commit<<<grid_for(sc.nb, kB), kB, 0, s>>>(sc, bmask, part_rank, gath, stride, q, qd));
}

void launch_merged(int n, const int* ianc, const double* iq, const double* iznext, double* out,
                   cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_merged", s, k_merged<<<grid_for(6ll * n, kB), kB, 0, s>>>(n, ianc, iq, iznext, out));
}

void launch_adapt(int n, const int* ianc, double* irho, const double* irho0, const double* rb,
                  const double* sb, const AdaptParams& a, double* iz, const double* iznext,
                  cudaStream_t s, const FrameCtrl* skip_first) {
    if (n == 0) return;
    DABD_LAUNCH("k_adapt", s, k_adapt<<<grid_for(n, kB), kB, 0, s>>>(n, ianc, irho, irho0, rb, sb, a.tau, a.mu, a.sigma_min,
                                           a.sigma_max, a.adapt_enabled ? 1 : 0, iz, iznext, skip_first));
}

void launch_commit(const SceneView& sc, int n, const int* ibody, const int* ipart, const int* ianc,
                   const uint32_t* bmask, double* iq, const double* iznext, const double* q_start,
                   double h, double* q, double* qd, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_commit", s, k_commit<<<grid_for(n, kB), kB, 0, s>>>(sc, n, ibody, ipart, ianc, bmask, iq, iznext, q_start,
                                            h, q, qd));
}

void launch_accept_copy(int n, const int* ipart, int part_base, const PartState* ps,
                        const double* src, double* dst, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_accept_copy", s, k_accept_copy<<<grid_for(6ll * n, kB), kB, 0, s>>>(n, ipart, part_base, ps, src, dst));
}

void launch_admm_ctrl(const AdmmCtrlArgs& a, int op, cudaStream_t s) {
    DABD_LAUNCH("k_admm_ctrl", s, k_admm_ctrl<<<1, 32, 0, s>>>(a, op));
}

void launch_inst_flags(const SceneView& sc, const uint32_t* masks, int P, int p0, int* f_all, int* f_dyn,
                       int* f_sh, cudaStream_t s) {
    const long long n = static_cast<long long>(P) * sc.nb;
    if (n == 0) return;
    DABD_LAUNCH("k_inst_flags", s, k_inst_flags<<<grid_for(n, 256), 256, 0, s>>>(sc, masks, P, p0, f_all, f_dyn, f_sh));
}

void launch_inst_counts(int P, int nb, const int* f_all, const int* f_dyn, const int* f_sh, const int* s_all,
                        const int* s_dyn, const int* s_sh, int* counts, cudaStream_t s) {
    DABD_LAUNCH("k_inst_counts", s, k_inst_counts<<<1, 64, 0, s>>>(P, nb, f_all, f_dyn, f_sh, s_all, s_dyn, s_sh, counts));
}

void launch_inst_scatter(const SceneView& sc, const uint32_t* masks, int P, int p0, const int* f_all,
                         const int* f_dyn, const int* f_sh, const int* s_all, const int* s_dyn,
                         const int* s_sh, double beta, const double* rho_carry, const int* rowtab_prev,
                         InstOut o, cudaStream_t s) {
    const long long n = static_cast<long long>(P) * sc.nb;
    if (n == 0) return;
    DABD_LAUNCH("k_inst_scatter", s, k_inst_scatter<<<grid_for(n, 256), 256, 0, s>>>(sc, masks, P, p0, f_all, f_dyn, f_sh, s_all,
                                                                        s_dyn, s_sh, beta, rho_carry, rowtab_prev, o));
}

void launch_rho_carry(int n_inst, int nb, const int* ibody, const int* ianc, const double* irho,
                      double* carry, cudaStream_t s) {
    if (nb == 0) return;
    DABD_LAUNCH("k_rho_carry", s, k_rho_carry<<<1, 1024, 0, s>>>(n_inst, nb, ibody, ianc, irho, carry));
}

void launch_masks_w(const SceneView& sc, const double* q, const double* planes, int np, const double* vmax,
                    double h, double w_min, double* w_out, uint32_t all, uint32_t* masks, int* err,
                    cudaStream_t s) {
    if (sc.nb == 0) return;
    DABD_LAUNCH("k_masks", s, k_masks<<<grid_for(sc.nb, kB), kB, 0, s>>>(sc, q, planes, np, 0.0, all, masks, err, vmax, h,
                                                                   w_min, w_out));
}

void launch_pack_owned(const SceneView& sc, const uint32_t* bmask, int p0, int p1, const double* q,
                       const double* qd, double* rec, int* count, cudaStream_t s) {
    if (sc.nb == 0) return;
    DABD_LAUNCH("k_pack_owned", s, k_pack_owned<<<grid_for(sc.nb, kB), kB, 0, s>>>(sc, bmask, p0, p1, q, qd, rec, count));
}

void launch_unpack_owned(int world, const int* counts, const double* gath, size_t stride, double* q,
                         double* qd, cudaStream_t s) {
    DABD_LAUNCH("k_unpack_owned", s, k_unpack_owned<<<64, kB, 0, s>>>(world, counts, gath, stride, q, qd));
}

void launch_fan_post(const FanView& f, const double* rec, int rec_len, cudaStream_t s) {
    DABD_LAUNCH("k_fan_post", s, k_fan_post<<<1, 32, 0, s>>>(f, rec, rec_len));
}

void launch_fan_wait(const FanView& f, cudaStream_t s) {
    DABD_LAUNCH("k_fan_wait", s, k_fan_wait<<<1, 32, 0, s>>>(f));
}

void launch_fan_record(int P, const double* dq, const double* rloc, const double* sloc, const double* gate,
                       const int* err, double* rec, cudaStream_t s) {
    DABD_LAUNCH("k_fan_record", s, k_fan_record<<<1, 32, 0, s>>>(P, dq, rloc, sloc, gate, err, rec));
}

void launch_pack_halo_par(int n, const int* inst, const double* iq, const double* iu, const double* irho,
                          double* pub, const FrameCtrl* pc, int side, size_t reg, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_pack_halo", s, k_pack_halo<<<grid_for(n, kB), kB, 0, s>>>(n, inst, iq, iu, irho, pub, pc, side, reg));
}

void launch_consensus_par(int ns, const int* sh, const int* ipart, int part_base, const double* iq, double* iu,
                          const double* irho, const double* iz, const double* peer_lo, const double* peer_hi,
                          int n_lo, double* iznext, double* rb, double* sb, double* rloc, double* sloc, int* err,
                          const FrameCtrl* pc, size_t reg, cudaStream_t s) {
    if (ns == 0) return;
    DABD_LAUNCH("k_consensus", s, k_consensus<<<grid_for(ns, kB), kB, 0, s>>>(ns, sh, ipart, part_base, iq, iu, irho, iz,
                                                                          peer_lo, peer_hi, n_lo, iznext, rb, sb,
                                                                          rloc, sloc, err, pc, reg));
}

} // namespace dabd_gpu
