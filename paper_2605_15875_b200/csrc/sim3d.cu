// 3D affine-body scene stepping (sim3d.hpp). Single domain: predict
// (body.cpp:120-134 in 3D), then newton.cpp:7-71 on
//   E(q) = 1/2 (q - q~)^T M (q - q~) + h^2 w ||A^T A - I||^2 + h^2 sum_c b(d_c)
// with the 3D primitives: body terms (contact3d.cu k_body3d), candidate
// point-triangle / edge-edge pairs (broad3d.cu), barrier terms with the
// PSD-projected 24x24 pair Hessian (k_contact3d) and additive CCD (k_ccd3d).
// The Newton system is a 12x12-block BSR over the dynamic bodies, assembled in
// a fixed order (no floating-point atomics) and solved by a block-Jacobi PCG
// in one thread block (3D scenes here are tens to hundreds of bodies).
#include "sim3d.hpp"

#include "broad3d.hpp"
#include "contact3d.hpp"
#include "instrument.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <map>

namespace dabd_gpu {

namespace {

constexpr int kPT = 1024; // PCG block size

__global__ void k_predict3(int n, const int* is_static, const double* q, const double* qd, double h, double gx,
                           double gy, double gz, double* qt) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    for (int k = 0; k < 12; ++k) {
        double v = q[12 * b + k];
        if (!is_static[b]) {
            v += h * qd[12 * b + k];
            if (k < 3) v += h * h * (k == 0 ? gx : (k == 1 ? gy : gz));
        }
        qt[12 * b + k] = v;
    }
}

// key -> (kind, a, b) and the four rest points (PT: vertex of a, triangle of
// b; EE: edge of a, edge of b)
__global__ void k_expand3(int nk, const unsigned long long* keys, int bb, int pb, const int* vstart,
                          const double* verts, const int* tstart, const int* tris, const int* estart,
                          const int* edges, int* kind, int* ka, int* kb, double* rest) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nk) return;
    unsigned long long key = keys[k];
    const unsigned long long mp = (1ull << pb) - 1ull, mb = (1ull << bb) - 1ull;
    const int pbi = static_cast<int>(key & mp);
    key >>= pb;
    const int pa = static_cast<int>(key & mp);
    key >>= pb;
    const int b = static_cast<int>(key & mb);
    key >>= bb;
    const int a = static_cast<int>(key & mb);
    key >>= bb;
    const int kd = static_cast<int>(key);
    kind[k] = kd;
    ka[k] = a;
    kb[k] = b;
    int vid[4];
    if (kd == 0) {
        vid[0] = vstart[a] + pa;
        const int* t = tris + 3 * (tstart[b] + pbi);
        for (int i = 0; i < 3; ++i) vid[1 + i] = vstart[b] + t[i];
    } else {
        const int* e0 = edges + 2 * (estart[a] + pa);
        const int* e1 = edges + 2 * (estart[b] + pbi);
        vid[0] = vstart[a] + e0[0];
        vid[1] = vstart[a] + e0[1];
        vid[2] = vstart[b] + e1[0];
        vid[3] = vstart[b] + e1[1];
    }
    for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) rest[12 * k + 3 * i + c] = verts[3 * vid[i] + c];
}

__global__ void k_gather3(int nk, const int* ka, const int* kb, const double* q0, const double* q1, double* qa,
                          double* qb) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 12 * nk) return;
    const int k = t / 12, c = t - 12 * k;
    qa[t] = q0[12 * ka[k] + c];
    qb[t] = q1[12 * kb[k] + c];
}

// y = x + alpha d on dynamic bodies (static bodies keep x)
__global__ void k_axpy3(int n, const int* is_static, const double* x, const double* d, double alpha, double* y) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 12 * n) return;
    y[t] = is_static[t / 12] ? x[t] : x[t] + alpha * d[t];
}

// Deterministic single-block sum / max / min of up to two arrays.
template <int OP> // 0 sum, 1 max |.|, 2 min
__global__ void k_reduce3(int n1, const double* v1, const int* mask1, int n2, const double* v2, double* out) {
    __shared__ double sh[256];
    double acc = OP == 2 ? DBL_MAX : 0.0;
    for (int i = threadIdx.x; i < n1 + n2; i += 256) {
        double v;
        if (i < n1) {
            if (mask1 && mask1[i]) continue; // static bodies carry no energy / step
            v = v1[i];
        } else {
            v = v2[i - n1];
        }
        if (OP == 0) acc += v;
        else if (OP == 1) acc = fmax(acc, fabs(v));
        else acc = fmin(acc, v);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double a = sh[threadIdx.x], b = sh[threadIdx.x + w];
            sh[threadIdx.x] = OP == 0 ? a + b : (OP == 1 ? fmax(a, b) : fmin(a, b));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// one block of 144 threads per BSR block: body Hessian (diagonal blocks) plus
// the listed pair-Hessian quarters in list order
__global__ void k_assemble3(int nblk, const int* blk_body, const double* bhess, const int* cptr, const int* centry,
                            const double* chess, double* blk) {
    const int bi = blockIdx.x;
    if (bi >= nblk) return;
    const int e = threadIdx.x, r = e / 12, c = e - 12 * r;
    double v = blk_body[bi] >= 0 ? bhess[144 * static_cast<size_t>(blk_body[bi]) + e] : 0.0;
    for (int t = cptr[bi]; t < cptr[bi + 1]; ++t) {
        const int k = centry[t] >> 2, part = centry[t] & 3;
        const int ro = (part == 1 || part == 3) ? 12 : 0, co = (part == 1 || part == 2) ? 12 : 0;
        v += chess[576 * static_cast<size_t>(k) + 24 * (ro + r) + co + c];
    }
    blk[144 * static_cast<size_t>(bi) + e] = v;
}

// rhs = -(body gradient + pair gradients) per row, fixed order
__global__ void k_rhs3(int R, const int* body_of_row, const double* bgrad, const int* gptr, const int* gentry,
                       const double* cgrad, double* rhs) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 12 * R) return;
    const int i = t / 12, c = t - 12 * i;
    double v = bgrad[12 * body_of_row[i] + c];
    for (int u = gptr[i]; u < gptr[i + 1]; ++u) {
        const int k = gentry[u] >> 1, side = gentry[u] & 1;
        v += cgrad[24 * static_cast<size_t>(k) + 12 * side + c];
    }
    rhs[t] = -v;
}

__device__ double block_sum(double v, double* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < kPT / 32 ? sh[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) sh[32] = t;
    }
    __syncthreads();
    return sh[32];
}

// Block-Jacobi PCG on the BSR system (diagonal block first in every row) with
// eps I of newton.cpp:20-24 added to the diagonal; the whole solve in one
// block. work: Dinv [R][144], r, z, p, ap [12 R].
__global__ void __launch_bounds__(kPT) k_pcg3(int R, const int* bptr, const int* bcol, const double* blk,
                                              const double* rhs, double* x, double* work, double tol, int max_iters,
                                              int* iters_out, int* err) {
    __shared__ double sh[33];
    const int N = 12 * R;
    double* dinv = work;
    double* r = work + 144 * static_cast<size_t>(R);
    double* z = r + N;
    double* p = z + N;
    double* ap = p + N;
    double tr = 0.0;
    for (int i = threadIdx.x; i < R; i += kPT)
        for (int c = 0; c < 12; ++c) tr += blk[144 * static_cast<size_t>(bptr[i]) + 13 * c];
    const double eps = 1e-8 * block_sum(tr, sh) / N;
    for (int i = threadIdx.x; i < R; i += kPT) { // (D + eps I)^-1 by Cholesky
        double L[12][12];
        const double* d = blk + 144 * static_cast<size_t>(bptr[i]);
        for (int j = 0; j < 12; ++j) {
            double s = d[13 * j] + eps;
            for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
            if (!(s > 0.0)) atomicCAS(err, 0, 2);
            L[j][j] = sqrt(fmax(s, 1e-300));
            for (int m = j + 1; m < 12; ++m) {
                double t = d[12 * m + j];
                for (int k = 0; k < j; ++k) t -= L[m][k] * L[j][k];
                L[m][j] = t / L[j][j];
            }
        }
        double* o = dinv + 144 * static_cast<size_t>(i);
        for (int c = 0; c < 12; ++c) { // column c of (L L^T)^-1: forward then backward substitution
            double y[12];
            for (int m = 0; m < 12; ++m) {
                double t = m == c ? 1.0 : 0.0;
                for (int k = 0; k < m; ++k) t -= L[m][k] * y[k];
                y[m] = t / L[m][m];
            }
            for (int m = 11; m >= 0; --m) {
                double t = y[m];
                for (int k = m + 1; k < 12; ++k) t -= L[k][m] * y[k];
                y[m] = t / L[m][m];
            }
            for (int m = 0; m < 12; ++m) o[12 * m + c] = y[m];
        }
    }
    __syncthreads();
    auto precond = [&](const double* in, double* out) {
        for (int t = threadIdx.x; t < N; t += kPT) {
            const int i = t / 12, c = t - 12 * i;
            const double* di = dinv + 144 * static_cast<size_t>(i) + 12 * c;
            double v = 0.0;
            for (int k = 0; k < 12; ++k) v += di[k] * in[12 * i + k];
            out[t] = v;
        }
    };
    double bb = 0.0;
    for (int t = threadIdx.x; t < N; t += kPT) {
        x[t] = 0.0;
        r[t] = rhs[t];
        bb += rhs[t] * rhs[t];
    }
    bb = block_sum(bb, sh);
    precond(r, z);
    __syncthreads();
    double rz = 0.0;
    for (int t = threadIdx.x; t < N; t += kPT) {
        p[t] = z[t];
        rz += r[t] * z[t];
    }
    rz = block_sum(rz, sh);
    int it = 0;
    while (bb > 0.0 && it < max_iters) {
        double pap = 0.0;
        for (int t = threadIdx.x; t < N; t += kPT) {
            const int i = t / 12, c = t - 12 * i;
            double v = 0.0;
            for (int bk = bptr[i]; bk < bptr[i + 1]; ++bk) {
                const double* m = blk + 144 * static_cast<size_t>(bk) + 12 * c;
                const double* pv = p + 12 * bcol[bk];
                for (int k = 0; k < 12; ++k) v += m[k] * pv[k];
            }
            v += eps * p[t];
            ap[t] = v;
            pap += p[t] * v;
        }
        pap = block_sum(pap, sh);
        const double alpha = rz / pap;
        double rr = 0.0;
        for (int t = threadIdx.x; t < N; t += kPT) {
            x[t] += alpha * p[t];
            r[t] -= alpha * ap[t];
            rr += r[t] * r[t];
        }
        rr = block_sum(rr, sh);
        ++it;
        if (rr <= tol * tol * bb || !(pap > 0.0)) break;
        precond(r, z);
        __syncthreads();
        double rz2 = 0.0;
        for (int t = threadIdx.x; t < N; t += kPT) rz2 += r[t] * z[t];
        rz2 = block_sum(rz2, sh);
        const double beta = rz2 / rz;
        rz = rz2;
        for (int t = threadIdx.x; t < N; t += kPT) p[t] = z[t] + beta * p[t];
        __syncthreads();
    }
    if (threadIdx.x == 0) *iters_out = it;
}

// row solution -> body step (static bodies 0)
__global__ void k_scatter_dq(int n, const int* row_of, const double* x, double* dq) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 12 * n) return;
    const int b = t / 12, rw = row_of[b];
    dq[t] = rw >= 0 ? x[12 * rw + (t - 12 * b)] : 0.0;
}

__global__ void k_velocity3(int n, const int* is_static, const double* q, const double* q0, double h, double* qd) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 12 * n) return;
    qd[t] = is_static[t / 12] ? 0.0 : (q[t] - q0[t]) / h;
}

int grid(long long n, int b) { return static_cast<int>(std::max(1ll, (n + b - 1) / b)); }

int bits_for(int x) {
    int b = 1;
    while ((1ll << b) < x) ++b;
    return b;
}

} // namespace

Sim3d::Sim3d(int device, int n, const int* vstart, const double* verts, const int* tstart, const int* tris,
             const int* estart, const int* edges, const int* is_static, const double* moments,
             const double* volume, const double* q0, const double* qd0, const Sim3dParams& p)
    : device_(device), n_(n), p_(p) {
    if (n < 1) throw InvalidArg("sim3d: no bodies");
    CUDA_CHECK(cudaSetDevice(device));
    CUDA_CHECK(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
    is_static_.assign(is_static, is_static + n);
    row_of_.assign(n, -1);
    int maxp = 1;
    for (int b = 0; b < n; ++b) {
        if (!is_static_[b]) {
            row_of_[b] = R_++;
            body_of_row_.push_back(b);
        }
        maxp = std::max({maxp, vstart[b + 1] - vstart[b], tstart[b + 1] - tstart[b], estart[b + 1] - estart[b]});
    }
    bb_bits_ = bits_for(n);
    pb_bits_ = bits_for(maxp);
    if (1 + 2 * bb_bits_ + 2 * pb_bits_ > 64) throw InvalidArg("sim3d: scene too large for the candidate key");
    vstart_.upload(vstart, n + 1, s_);
    tstart_.upload(tstart, n + 1, s_);
    estart_.upload(estart, n + 1, s_);
    verts_.upload(verts, 3 * static_cast<size_t>(std::max(vstart[n], 1)), s_);
    tris_.upload(tris, 3 * static_cast<size_t>(std::max(tstart[n], 1)), s_);
    edges_.upload(edges, 2 * static_cast<size_t>(std::max(estart[n], 1)), s_);
    stat_d_.upload(is_static_, s_);
    row_of_d_.upload(row_of_, s_);
    moments_.upload(moments, 10 * static_cast<size_t>(n), s_);
    std::vector<double> w(n);
    for (int b = 0; b < n; ++b) w[b] = p.kappa_arap * volume[b];
    w_.upload(w, s_);
    const size_t m = 12 * static_cast<size_t>(n);
    for (DBuf<double>* b : {&q_, &qd_, &qt_, &qstart_, &dq_, &qtry_, &bgrad_}) b->resize(m);
    q_.upload(q0, m, s_);
    qd_.upload(qd0, m, s_);
    bval_.resize(n);
    bhess_.resize(144 * static_cast<size_t>(n));
    red_.resize(4);
    cerr_.resize(1);
    cerr_.zero(s_);
    pin_.resize(4);
    pin_i_.resize(4);
    CUDA_CHECK(cudaStreamSynchronize(s_));
}

Sim3d::~Sim3d() {
    if (s_) cudaStreamDestroy(s_);
}

void Sim3d::state(double* q, double* qd) const {
    const size_t m = 12 * static_cast<size_t>(n_);
    CUDA_CHECK(cudaMemcpyAsync(q, q_.get(), m * sizeof(double), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(qd, qd_.get(), m * sizeof(double), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
}

void Sim3d::set_state(const double* q, const double* qd) {
    const size_t m = 12 * static_cast<size_t>(n_);
    q_.upload(q, m, s_);
    qd_.upload(qd, m, s_);
    CUDA_CHECK(cudaStreamSynchronize(s_));
}

// candidate pairs over [q0, q1] (q1 = nullptr: static) inflated by margin,
// expanded to per-pair kind, bodies and rest points
int Sim3d::candidates(const double* q0, const double* q1, double margin, Contacts& c) {
    Broad3dView v{n_, q0, q1, vstart_.get(), verts_.get(), tstart_.get(), tris_.get(), estart_.get(), edges_.get(),
                  margin};
    Key3Fmt f;
    f.bb = bb_bits_;
    f.pb = pb_bits_;
    c.n = broad_phase3d_device(v, f, c.keys, s_);
    const size_t k = std::max(c.n, 1);
    for (DBuf<int>* b : {&c.kind, &c.a, &c.b, &c.dtype}) b->resize(k);
    for (DBuf<double>* b : {&c.qa, &c.qb}) b->resize(12 * k);
    c.rest.resize(12 * k);
    c.d.resize(k);
    c.value.resize(k);
    c.grad.resize(24 * k);
    if (c.n > 0)
        DABD_LAUNCH("k_expand3", s_, k_expand3<<<grid(c.n, 128), 128, 0, s_>>>(
                                         c.n, c.keys.get(), bb_bits_, pb_bits_, vstart_.get(), verts_.get(),
                                         tstart_.get(), tris_.get(), estart_.get(), edges_.get(), c.kind.get(),
                                         c.a.get(), c.b.get(), c.rest.get()));
    return c.n;
}

void Sim3d::contact_terms(Contacts& c, const double* q, bool hess) {
    if (c.n == 0) return;
    if (hess) c.hess.resize(576 * static_cast<size_t>(c.n));
    DABD_LAUNCH("k_gather3", s_, k_gather3<<<grid(12ll * c.n, 128), 128, 0, s_>>>(c.n, c.a.get(), c.b.get(), q, q,
                                                                                  c.qa.get(), c.qb.get()));
    Contact3dArgs a{c.n, c.kind.get(), c.qa.get(), c.qb.get(), c.rest.get(), p_.d_hat, p_.kappa,
                    p_.h * p_.h, 1, c.d.get(), c.dtype.get(), c.value.get(), c.grad.get(),
                    hess ? c.hess.get() : nullptr, cerr_.get()};
    launch_contact3d(a, s_);
}

// E(q) over the dynamic bodies and the pairs of c (c must cover every pair
// within d_hat at q); *bad: some pair at or below zero distance
double Sim3d::energy(const double* q, Contacts& c, bool* bad) {
    cerr_.zero(s_);
    Body3dArgs ba{n_, q, qt_.get(), moments_.get(), w_.get(), p_.h * p_.h, 1, bval_.get(), bgrad_.get(), nullptr};
    launch_body3d(ba, s_);
    contact_terms(c, q, false);
    DABD_LAUNCH("k_reduce3", s_, (k_reduce3<0><<<1, 256, 0, s_>>>(n_, bval_.get(), stat_d_.get(), c.n, c.value.get(),
                                                                   red_.get())));
    CUDA_CHECK(cudaMemcpyAsync(pin_.get(), red_.get(), sizeof(double), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 2, cerr_.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
    *bad = pin_i_[2] != 0;
    return pin_[0];
}

// BSR pattern and fixed-order contribution lists from the pairs of c
void Sim3d::assemble(Contacts& c) {
    std::vector<int> ka(std::max(c.n, 1)), kb(std::max(c.n, 1));
    if (c.n) {
        CUDA_CHECK(cudaMemcpyAsync(ka.data(), c.a.get(), c.n * sizeof(int), cudaMemcpyDeviceToHost, s_));
        CUDA_CHECK(cudaMemcpyAsync(kb.data(), c.b.get(), c.n * sizeof(int), cudaMemcpyDeviceToHost, s_));
        CUDA_CHECK(cudaStreamSynchronize(s_));
    }
    std::vector<std::map<int, std::vector<int>>> rows(R_); // row -> col row -> entries (k << 2 | part)
    std::vector<std::vector<int>> gl(R_);                  // row -> (k << 1 | side)
    for (int i = 0; i < R_; ++i) rows[i][i];                // diagonal block first (smallest key is not i in general)
    for (int k = 0; k < c.n; ++k) {
        const int ra = row_of_[ka[k]], rb = row_of_[kb[k]];
        if (ra >= 0) {
            rows[ra][ra].push_back(k << 2 | 0);
            gl[ra].push_back(k << 1 | 0);
        }
        if (rb >= 0) {
            rows[rb][rb].push_back(k << 2 | 1);
            gl[rb].push_back(k << 1 | 1);
        }
        if (ra >= 0 && rb >= 0 && ra != rb) {
            rows[ra][rb].push_back(k << 2 | 2);
            rows[rb][ra].push_back(k << 2 | 3);
        }
    }
    h_bptr_.assign(1, 0);
    h_bcol_.clear();
    std::vector<int> blk_body, cptr(1, 0), centry, gptr(1, 0), gentry;
    for (int i = 0; i < R_; ++i) {
        // diagonal first, then ascending columns
        auto emit = [&](int col, const std::vector<int>& e) {
            h_bcol_.push_back(col);
            blk_body.push_back(col == i ? body_of_row_[i] : -1);
            centry.insert(centry.end(), e.begin(), e.end());
            cptr.push_back(static_cast<int>(centry.size()));
        };
        emit(i, rows[i][i]);
        for (const auto& kv : rows[i])
            if (kv.first != i) emit(kv.first, kv.second);
        h_bptr_.push_back(static_cast<int>(h_bcol_.size()));
        gentry.insert(gentry.end(), gl[i].begin(), gl[i].end());
        gptr.push_back(static_cast<int>(gentry.size()));
    }
    const int nblk = static_cast<int>(h_bcol_.size());
    bptr_.upload(h_bptr_, s_);
    bcol_.upload(h_bcol_, s_);
    DBuf<int> bbody;
    bbody.upload(blk_body, s_);
    contrib_ptr_.upload(cptr, s_);
    contrib_.upload(centry.empty() ? std::vector<int>{0} : centry, s_);
    gcontrib_ptr_.upload(gptr, s_);
    gcontrib_.upload(gentry.empty() ? std::vector<int>{0} : gentry, s_);
    DBuf<int> bor;
    bor.upload(body_of_row_, s_);
    blk_.resize(144 * static_cast<size_t>(nblk));
    rhs_.resize(12 * static_cast<size_t>(R_));
    Body3dArgs ba{n_, q_.get(), qt_.get(), moments_.get(), w_.get(), p_.h * p_.h, 1, bval_.get(), bgrad_.get(),
                  bhess_.get()};
    launch_body3d(ba, s_);
    DABD_LAUNCH("k_assemble3", s_, k_assemble3<<<nblk, 144, 0, s_>>>(nblk, bbody.get(), bhess_.get(), contrib_ptr_.get(),
                                                                      contrib_.get(), c.n ? c.hess.get() : nullptr,
                                                                      blk_.get()));
    DABD_LAUNCH("k_rhs3", s_, k_rhs3<<<grid(12ll * R_, 128), 128, 0, s_>>>(R_, bor.get(), bgrad_.get(), gcontrib_ptr_.get(),
                                                                          gcontrib_.get(), c.n ? c.grad.get() : nullptr,
                                                                          rhs_.get()));
    CUDA_CHECK(cudaStreamSynchronize(s_)); // the pattern buffers above are local
}

int Sim3d::solve() {
    x_.resize(12 * static_cast<size_t>(R_));
    pcg_scratch_.resize(144 * static_cast<size_t>(R_) + 4 * 12 * static_cast<size_t>(R_));
    DBuf<int> it, err;
    it.resize(1);
    err.resize(1);
    err.zero(s_);
    DABD_LAUNCH("k_pcg3", s_, k_pcg3<<<1, kPT, 0, s_>>>(R_, bptr_.get(), bcol_.get(), blk_.get(), rhs_.get(), x_.get(),
                                                       pcg_scratch_.get(), p_.pcg_rel_tol, p_.pcg_max_iters,
                                                       it.get(), err.get()));
    DABD_LAUNCH("k_scatter_dq", s_, k_scatter_dq<<<grid(12ll * n_, 128), 128, 0, s_>>>(n_, row_of_d_.get(), x_.get(),
                                                                                       dq_.get()));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get(), it.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 1, err.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
    if (pin_i_[1]) throw Error("sim3d: a diagonal block is not positive definite");
    last_pcg_iters_ = pin_i_[0];
    return pin_i_[0];
}

double Sim3d::dq_inf() {
    DABD_LAUNCH("k_reduce3", s_, (k_reduce3<1><<<1, 256, 0, s_>>>(12 * n_, dq_.get(), nullptr, 0, nullptr, red_.get())));
    CUDA_CHECK(cudaMemcpyAsync(pin_.get(), red_.get(), sizeof(double), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
    return pin_[0];
}

// sim.cpp:207-247 (single domain) with newton.cpp:7-71, in 3D
Sim3dStats Sim3d::frame() {
    Sim3dStats st;
    const size_t m = 12 * static_cast<size_t>(n_);
    CUDA_CHECK(cudaMemcpyAsync(qstart_.get(), q_.get(), m * sizeof(double), cudaMemcpyDeviceToDevice, s_));
    DABD_LAUNCH("k_predict3", s_, k_predict3<<<grid(n_, 128), 128, 0, s_>>>(n_, stat_d_.get(), q_.get(), qd_.get(), p_.h,
                                                                           p_.gravity[0], p_.gravity[1], p_.gravity[2],
                                                                           qt_.get()));
    const double tol = p_.theta * p_.h * p_.scene_scale;
    for (int it = 0; it < p_.newton_cap && R_ > 0; ++it) {
        ++st.newton_iterations;
        candidates(q_.get(), nullptr, p_.d_hat, c0_);
        st.max_candidates = std::max(st.max_candidates, c0_.n);
        bool bad = false;
        const double e0 = energy(q_.get(), c0_, &bad);
        if (bad) throw Error("sim3d: a pair is at zero distance");
        contact_terms(c0_, q_.get(), true);
        assemble(c0_);
        st.pcg_iterations += solve();
        const double dmax = dq_inf();
        if (dmax < tol) { // newton.cpp:30-36
            st.converged = 1;
            break;
        }
        // CCD bound over [q, q + dq] (newton.cpp:38-42, geometry.cpp:333-334)
        DABD_LAUNCH("k_axpy3", s_, k_axpy3<<<grid(12ll * n_, 128), 128, 0, s_>>>(n_, stat_d_.get(), q_.get(), dq_.get(),
                                                                                1.0, qtry_.get()));
        candidates(q_.get(), qtry_.get(), 0.0, cs_);
        double toi = 2.0;
        if (cs_.n > 0) {
            DBuf<double> qa1, qb1, t;
            qa1.resize(12 * static_cast<size_t>(cs_.n));
            qb1.resize(12 * static_cast<size_t>(cs_.n));
            t.resize(cs_.n);
            DABD_LAUNCH("k_gather3", s_, k_gather3<<<grid(12ll * cs_.n, 128), 128, 0, s_>>>(
                                             cs_.n, cs_.a.get(), cs_.b.get(), q_.get(), q_.get(), cs_.qa.get(), cs_.qb.get()));
            DABD_LAUNCH("k_gather3", s_, k_gather3<<<grid(12ll * cs_.n, 128), 128, 0, s_>>>(
                                             cs_.n, cs_.a.get(), cs_.b.get(), qtry_.get(), qtry_.get(), qa1.get(), qb1.get()));
            Ccd3dArgs ca{cs_.n, cs_.kind.get(), cs_.qa.get(), qa1.get(), cs_.qb.get(), qb1.get(), cs_.rest.get(), t.get()};
            launch_ccd3d(ca, s_);
            DABD_LAUNCH("k_reduce3", s_, (k_reduce3<2><<<1, 256, 0, s_>>>(cs_.n, t.get(), nullptr, 0, nullptr, red_.get())));
            CUDA_CHECK(cudaMemcpyAsync(pin_.get(), red_.get(), sizeof(double), cudaMemcpyDeviceToHost, s_));
            CUDA_CHECK(cudaStreamSynchronize(s_));
            toi = pin_[0];
        }
        double alpha = toi > 1.0 ? 1.0 : std::min(1.0, 0.9 * toi);
        // every pair within d_hat anywhere on [q, q + alpha dq]: one superset for all trials
        DABD_LAUNCH("k_axpy3", s_, k_axpy3<<<grid(12ll * n_, 128), 128, 0, s_>>>(n_, stat_d_.get(), q_.get(), dq_.get(),
                                                                                alpha, qtry_.get()));
        candidates(q_.get(), qtry_.get(), p_.d_hat, cs_);
        bool accepted = false;
        while (true) { // newton.cpp:47-62 (armijo_c = 0: pure decrease)
            DABD_LAUNCH("k_axpy3", s_, k_axpy3<<<grid(12ll * n_, 128), 128, 0, s_>>>(n_, stat_d_.get(), q_.get(),
                                                                                    dq_.get(), alpha, qtry_.get()));
            bool tbad = false;
            const double e1 = energy(qtry_.get(), cs_, &tbad);
            if (!tbad && e1 < e0) {
                accepted = true;
                break;
            }
            alpha *= 0.5;
            ++st.line_search_steps;
            if (!(alpha >= 1e-12)) break;
        }
        if (!accepted) throw Error("sim3d: line search failed below 1e-12");
        std::swap(q_, qtry_);
        if (alpha * dmax < tol) {
            st.converged = 1;
            break;
        }
    }
    DABD_LAUNCH("k_velocity3", s_, k_velocity3<<<grid(12ll * n_, 128), 128, 0, s_>>>(n_, stat_d_.get(), q_.get(),
                                                                                    qstart_.get(), p_.h, qd_.get()));
    // minimum distance over the pairs within d_hat at the committed state
    candidates(q_.get(), nullptr, p_.d_hat, c0_);
    if (c0_.n > 0) {
        contact_terms(c0_, q_.get(), false);
        DABD_LAUNCH("k_reduce3", s_, (k_reduce3<2><<<1, 256, 0, s_>>>(c0_.n, c0_.d.get(), nullptr, 0, nullptr, red_.get())));
        CUDA_CHECK(cudaMemcpyAsync(pin_.get(), red_.get(), sizeof(double), cudaMemcpyDeviceToHost, s_));
    }
    CUDA_CHECK(cudaStreamSynchronize(s_));
    st.min_distance = c0_.n > 0 ? pin_[0] : 0.0;
    return st;
}

int Sim3d::system(double* H, double* g, double* dq) {
    DABD_LAUNCH("k_predict3", s_, k_predict3<<<grid(n_, 128), 128, 0, s_>>>(n_, stat_d_.get(), q_.get(), qd_.get(), p_.h,
                                                                           p_.gravity[0], p_.gravity[1], p_.gravity[2],
                                                                           qt_.get()));
    candidates(q_.get(), nullptr, p_.d_hat, c0_);
    contact_terms(c0_, q_.get(), true);
    assemble(c0_);
    solve();
    const int N = 12 * R_;
    std::vector<double> blk(blk_.size()), rhs(N), x(N);
    CUDA_CHECK(cudaMemcpy(blk.data(), blk_.get(), blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(rhs.data(), rhs_.get(), N * sizeof(double), cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaMemcpy(x.data(), x_.get(), N * sizeof(double), cudaMemcpyDeviceToHost));
    std::fill(H, H + static_cast<size_t>(N) * N, 0.0);
    double tr = 0.0;
    for (int i = 0; i < R_; ++i)
        for (int c = 0; c < 12; ++c) tr += blk[144 * static_cast<size_t>(h_bptr_[i]) + 13 * c];
    const double eps = 1e-8 * tr / std::max(N, 1);
    for (int i = 0; i < R_; ++i)
        for (int bk = h_bptr_[i]; bk < h_bptr_[i + 1]; ++bk)
            for (int r = 0; r < 12; ++r)
                for (int c = 0; c < 12; ++c)
                    H[static_cast<size_t>(12 * i + r) * N + 12 * h_bcol_[bk] + c] = blk[144 * static_cast<size_t>(bk) + 12 * r + c];
    for (int t = 0; t < N; ++t) {
        H[static_cast<size_t>(t) * N + t] += eps;
        g[t] = -rhs[t];
        dq[t] = x[t];
    }
    return R_;
}

} // namespace dabd_gpu
