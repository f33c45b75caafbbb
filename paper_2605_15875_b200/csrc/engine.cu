// Engine: host orchestration of the B200 hot path (see engine.hpp).
#include "engine.hpp"

#include "admm.hpp"
#include "instrument.hpp"

#include <cub/cub.cuh>

#include <algorithm>
#include <bit>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <limits>
#include <functional>
#include <numeric>

namespace dabd_gpu {

namespace {

const char* err_text(int code) {
    switch (code) {
    case kErrStraddle: return "partition: body AABB wider than a region (straddles two interfaces)";
    case kErrTouching: return "ccd_toi: start configuration already touching/intersecting";
    case kErrBarrierDomain: return "barrier_energy: d <= 0 (barrier domain violated)";
    case kErrDegenerateEdge: return "point_edge_distance: degenerate edge (e0 == e1)";
    case kErrCapacity: return "capacity exceeded (contact candidate list)";
    case kErrEll: return "capacity exceeded (BSR row couples more bodies than the ELL width)";
    case kErrSettle: return "run_reference: Newton stepping failed to settle";
    case kErrNoHolder: return "LocalObjective: contact pair visible to no worker (overlap too small)";
    case kErrFactor: return "newton_solve: factorization failed (non-SPD diagonal block)";
    case kErrLineSearch: return "newton_solve: line search failed below 1e-12 (non-descent direction)";
    case kErrReplica: return "protocol error: replica rho mismatch";
    default: return "device error";
    }
}

constexpr int kPsStride = sizeof(PartState) / sizeof(double);
static_assert(sizeof(PartState) % sizeof(double) == 0, "PartState must be 8-byte strided");

double* ps_field(PartState* ps, double PartState::*f) { return &(ps->*f); }

// A partition's compute cost for the balancer: the reference feeds the
// worker's wall-clock compute time (runtime.cpp:674); partitions batched in
// shared kernels have no separable clock, so the cost is the deterministic
// row-weighted work of its solves: every Newton iteration touches its rows
// and contact blocks, every PCG iteration its rows. Floored at 1 so the
// imbalance metric's positivity holds for an empty partition.
double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double partition_cost(const PartState& s) {
    const double rows = s.ndof / 6.0;
    return std::max(1.0, s.iterations * (rows + 2.0 * s.n_active_contacts) + s.pcg_total * rows);
}

} // namespace

// DABD_GPU_ADMM_PROFILE=1: host-side phase clock of the multi-partition
// frame (synchronises the stream at every mark; a probe, never on in bench).
namespace {
struct AdmmProfile {
    bool on = std::getenv("DABD_GPU_ADMM_PROFILE") != nullptr;
    double t[12] = {};
    long long n[12] = {};
    std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    void mark(int slot, cudaStream_t s) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        t[slot] += std::chrono::duration<double, std::milli>(now - last).count();
        ++n[slot];
        last = now;
    }
    ~AdmmProfile() {
        if (!on) return;
        static const char* names[12] = {"frame_setup(rest)", "consensus+gate|capture", "decision", "newton|graph",
                                        "delta_inf", "commit", "other", "setup:masks", "setup:instances",
                                        "setup:prepare_solver(rest)", "prep:det_prepare", "prep:resizes"};
        for (int i = 0; i < 12; ++i)
            std::fprintf(stderr, "admm_profile %-15s %10.3f ms %8lld marks\n", names[i], t[i], n[i]);
    }
};
AdmmProfile& admm_prof() {
    static AdmmProfile p;
    return p;
}
} // namespace

Engine::Engine(const HostScene& hs, int device, int W, int pb, int pe) : hs_(hs), device_(device) {
    if (W < 0 || W > 32) throw InvalidArg("ctx: worker count must be in [0, 32]");
    if (W == 0) {
        W_ = 0;
        p0_ = 0;
        p1_ = 1;
    } else {
        if (!(0 <= pb && pb < pe && pe <= W)) throw InvalidArg("ctx: bad partition range");
        if (static_cast<int>(hs.planes.size()) < W - 1)
            throw InvalidArg("controller: scene has too few interface planes");
        W_ = W;
        p0_ = pb;
        p1_ = pe;
    }
    P_ = p1_ - p0_;
    CUDA_CHECK(cudaSetDevice(device));
    CUDA_CHECK(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
    own_stream_ = true;
    ds_.upload(hs_, s_);
    q_.upload(hs_.q0, s_);
    qd_.upload(hs_.qdot0, s_);
    q_start_.resize(6 * std::max(hs_.nb, 1));
    rho_carry_.assign(hs_.nb, std::numeric_limits<double>::quiet_NaN());
    tsc_ = TimestepController(hs_.params.h, hs_.max_halvings);
    if (W_ > 0) {
        planes_cur_.assign(hs_.planes.begin(), hs_.planes.begin() + (W_ - 1));
        balancer_ = Balancer(W_, hs_.balance);
        part_cost_.assign(W_, 0.0);
    }
    ps_.resize(P_);
    ps_h_.resize(P_);
    scal_a_.resize(P_);
    scal_b_.resize(P_);
    gate_.resize(P_);
    rloc_.resize(P_);
    sloc_.resize(P_);
    err_.resize(1);
    err_.zero(s_);
    pin_i_.resize(16);
    pin_d_.resize(256); // [0,32) gate, [32,64) r, [64,96) s, [96,128) dq, [128,160) 2.0 fill
    cellmax_.resize(1);
    nsel_.resize(1);
    ctrl_.resize(1);
    ctrl_.zero(s_);
    ctrl_h_.resize(1);
    perf_.resize(1);
    perf_.zero(s_);
    lstate_.resize(1);
    lstate_h_.resize(1);
    invalidate_list();
    trace_dev_.resize(8 * static_cast<size_t>(trace_cap_));
    qd_start_.resize(6 * std::max(hs_.nb, 1));
    if (const char* e = std::getenv("DABD_GPU_NO_GRAPH")) use_graph_ = e[0] == '0';
    if (const char* e = std::getenv("DABD_GPU_PCG_PHASES")) {
        // "1": CTA 0 / warp 0; "1:<cta>:<warp>": the timed thread is lane 0
        // of that warp of that CTA (per-CTA timelines, tools/pcg_phases.py)
        int cta = 0, w = 0;
        if (e[0] == '1') {
            std::sscanf(e, "1:%d:%d", &cta, &w);
            pcg_phases_ = 1 + 256 * cta + 16 * w;
        }
    }
    {
        int carve = -1; // driver default unless asked (experiment: DABD_GPU_CARVEOUT=100)
        if (const char* e = std::getenv("DABD_GPU_CARVEOUT")) carve = std::atoi(e);
        if (carve >= 0) {
            set_solver_carveout(carve);
            set_scalar_carveout(carve);
        }
    }
    if (const char* e = std::getenv("DABD_GPU_ADMM_HOST")) admm_device_ = e[0] != '1';
    // inexact Newton: on by default for single-domain frames only (a
    // consensus frame's stop test reads residuals built from the local
    // solutions, which the loose directions would perturb at the scale it
    // tests); dabd_gpu_ctx_set_inexact overrides
    eta_loose_ = W_ == 0 ? 1e-3 : 0.0;
    if (const char* e = std::getenv("DABD_GPU_PCG_ETA")) eta_loose_ = std::atof(e);
    if (const char* e = std::getenv("DABD_GPU_PCG_ETA_FACTOR")) eta_factor_ = std::atof(e);
    if (const char* e = std::getenv("DABD_SKIN_MIN")) skin_min_ = std::atof(e);
    if (const char* e = std::getenv("DABD_SKIN_GROW")) skin_grow_ = std::atof(e);
    sync();
}

Engine::~Engine() {
    if (exec_) cudaGraphExecDestroy(exec_);
    if (newton_exec_) cudaGraphExecDestroy(newton_exec_);
    if (admm_exec_) cudaGraphExecDestroy(admm_exec_);
    for (cudaStream_t s : cap_streams_) cudaStreamDestroy(s);
    for (cudaStream_t s : side_streams_) cudaStreamDestroy(s);
    if (peer_lo_) cudaIpcCloseMemHandle(const_cast<double*>(peer_lo_));
    if (peer_hi_) cudaIpcCloseMemHandle(const_cast<double*>(peer_hi_));
    for (void* ptr : fan_opened_) cudaIpcCloseMemHandle(ptr);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (own_stream_ && s_) cudaStreamDestroy(s_);
}

void Engine::set_stream(cudaStream_t s) {
    sync();
    if (own_stream_ && s_) cudaStreamDestroy(s_);
    own_stream_ = false;
    s_ = s;
    if (s_ == nullptr) {
        CUDA_CHECK(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
        own_stream_ = true;
    }
}

void Engine::set_comm(const Comm* c) {
    sync();
    // drop a previous run's peer mappings
    if (peer_lo_) cudaIpcCloseMemHandle(const_cast<double*>(peer_lo_));
    if (peer_hi_) cudaIpcCloseMemHandle(const_cast<double*>(peer_hi_));
    cudaGetLastError();
    peer_lo_ = peer_hi_ = nullptr;
    p2p_ = false;
    close_fanin();
    halo_parity_ = 0;
    if (!c) {
        distributed_ = false;
        comm_ = Comm{};
        return;
    }
    if (W_ == 0) throw InvalidArg("comm: a run_reference context (0 workers) has no exchange");
    const std::vector<int>& o = c->part_offsets;
    if (static_cast<int>(o.size()) != c->world + 1 || o.front() != 0 || o.back() != W_)
        throw InvalidArg("comm: part_offsets must cover [0, num_workers)");
    for (int r = 0; r < c->world; ++r)
        if (o[r] >= o[r + 1]) throw InvalidArg("comm: every rank needs at least one partition");
    if (o[c->rank] != p0_ || o[c->rank + 1] != p1_)
        throw InvalidArg("comm: the context's partition range differs from part_offsets[rank]");
    comm_ = *c;
    distributed_ = c->world > 1;
    std::vector<int> pr(W_);
    for (int r = 0; r < c->world; ++r)
        for (int p = o[r]; p < o[r + 1]; ++p) pr[p] = r;
    part_rank_.upload(pr, s_);
    sync();
    if (distributed_) setup_p2p();
    if (distributed_ && p2p_) setup_fanin();
}

// One all-gather of a single value: every rank's earlier work on its stream
// is complete (gloo stages through the host) or ordered (NCCL) before any
// rank's later work.
void Engine::comm_barrier() {
    rec_.resize(1);
    rec_all_.resize(comm_.world);
    if (comm_.allgather(comm_.user, rec_.get(), rec_all_.get(), 1, reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: barrier failed");
}

void Engine::setup_p2p() {
    p2p_ = false;
    if (const char* e = std::getenv("DABD_GPU_P2P_HALO"))
        if (e[0] == '0') return;
    // capacity: every body could be split (packets per region)
    pub_cap_ = static_cast<size_t>(std::max(hs_.nb, 1));
    pub_.resize(4 * kHaloStride * pub_cap_);
    // IPC handle (64 bytes = 8 doubles) + a success flag, all-gathered
    std::vector<double> rec(9, 0.0);
    cudaIpcMemHandle_t mine{};
    bool ok = cudaIpcGetMemHandle(&mine, pub_.get()) == cudaSuccess;
    cudaGetLastError();
    std::memcpy(rec.data(), &mine, sizeof(mine));
    rec[8] = ok ? 1.0 : 0.0;
    rec_.upload(rec, s_);
    rec_all_.resize(9 * comm_.world);
    if (comm_.allgather(comm_.user, rec_.get(), rec_all_.get(), 9, reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: all-gather failed");
    std::vector<double> all = rec_all_.to_host(s_);
    void* lo = nullptr;
    void* hi = nullptr;
    auto open = [&](int r, void** out) {
        if (r < 0 || r >= comm_.world) return true;
        if (all[9 * r + 8] == 0.0) return false;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, all.data() + 9 * r, sizeof(h));
        const bool good = cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
        cudaGetLastError();
        return good;
    };
    ok = ok && open(comm_.rank - 1, &lo) && open(comm_.rank + 1, &hi);
    // every rank must agree, or all fall back to the halo callback
    rec_.upload(std::vector<double>{ok ? 1.0 : 0.0}, s_);
    rec_all_.resize(comm_.world);
    if (comm_.allgather(comm_.user, rec_.get(), rec_all_.get(), 1, reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: all-gather failed");
    all = rec_all_.to_host(s_);
    bool every = true;
    for (int r = 0; r < comm_.world; ++r) every = every && all[r] != 0.0;
    if (!every) {
        if (lo) cudaIpcCloseMemHandle(lo);
        if (hi) cudaIpcCloseMemHandle(hi);
        cudaGetLastError();
        return;
    }
    peer_lo_ = static_cast<const double*>(lo);
    peer_hi_ = static_cast<const double*>(hi);
    p2p_ = true;
}

void Engine::close_fanin() {
    for (void* ptr : fan_opened_) cudaIpcCloseMemHandle(ptr);
    fan_opened_.clear();
    cudaGetLastError();
    fan_ok_ = false;
}

// Every rank's fan-in buffer mapped into every peer (the partition-per-GPU
// device ADMM loop's controller fan-in and ordering barriers; runtime.cpp:
// 586-619 without a host round trip). All ranks agree or none uses it.
void Engine::setup_fanin() {
    close_fanin();
    if (const char* e = std::getenv("DABD_GPU_FANIN"))
        if (e[0] == '0') return;
    const int world = comm_.world;
    if (world > 32) return;
    const size_t rec_bytes = sizeof(double) * kFanStride * static_cast<size_t>(world);
    fan_buf_.resize(rec_bytes + sizeof(unsigned long long) * world);
    fan_buf_.zero(s_);
    fan_rec_local_.resize(kFanStride);
    fan_seq_.resize(1);
    fan_seq_.zero(s_);
    sync();
    std::vector<double> rec(9, 0.0);
    cudaIpcMemHandle_t mine{};
    bool ok = cudaIpcGetMemHandle(&mine, fan_buf_.get()) == cudaSuccess;
    cudaGetLastError();
    std::memcpy(rec.data(), &mine, sizeof(mine));
    rec[8] = ok ? 1.0 : 0.0;
    rec_.upload(rec, s_);
    rec_all_.resize(9 * world);
    if (comm_.allgather(comm_.user, rec_.get(), rec_all_.get(), 9, reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: all-gather failed");
    std::vector<double> all = rec_all_.to_host(s_);
    FanView f;
    f.rank = comm_.rank;
    f.world = world;
    f.rec_stride = kFanStride;
    for (int r = 0; r < world && ok; ++r) {
        unsigned char* base = nullptr;
        if (r == comm_.rank) {
            base = fan_buf_.get();
        } else {
            if (all[9 * r + 8] == 0.0) {
                ok = false;
                break;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, all.data() + 9 * r, sizeof(h));
            void* ptr = nullptr;
            ok = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
            cudaGetLastError();
            if (!ok) break;
            fan_opened_.push_back(ptr);
            base = static_cast<unsigned char*>(ptr);
        }
        f.peer_rec[r] = reinterpret_cast<double*>(base);
        f.peer_flag[r] = reinterpret_cast<unsigned long long*>(base + rec_bytes);
    }
    f.local_rec = reinterpret_cast<const double*>(fan_buf_.get());
    f.local_flag = reinterpret_cast<const unsigned long long*>(fan_buf_.get() + rec_bytes);
    f.seq = fan_seq_.get();
    rec_.upload(std::vector<double>{ok ? 1.0 : 0.0}, s_);
    rec_all_.resize(world);
    if (comm_.allgather(comm_.user, rec_.get(), rec_all_.get(), 1, reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: all-gather failed");
    all = rec_all_.to_host(s_);
    bool every = true;
    for (int r = 0; r < world; ++r) every = every && all[r] != 0.0;
    if (!every) {
        close_fanin();
        return;
    }
    fan_view_ = f;
    fan_ok_ = true;
}

void Engine::exchange_halo() {
    const int n = n_halo_lo_ + n_halo_hi_;
    const size_t lo = static_cast<size_t>(kHaloStride) * n_halo_lo_;
    const size_t hi = static_cast<size_t>(kHaloStride) * n_halo_hi_;
    if (p2p_) {
        if (static_cast<size_t>(std::max(n_halo_lo_, n_halo_hi_)) > pub_cap_)
            throw Error("comm: peer halo capacity exceeded");
        // publish into [side][parity], barrier, then k_consensus reads the
        // neighbours' regions in place: rank-1's hi side, rank+1's lo side
        const size_t reg = static_cast<size_t>(kHaloStride) * pub_cap_;
        const int par = halo_parity_;
        halo_parity_ ^= 1;
        double* my_lo = pub_.get() + (0 * 2 + par) * reg;
        double* my_hi = pub_.get() + (1 * 2 + par) * reg;
        launch_pack_halo(n_halo_lo_, halo_inst_.get(), iq_.get(), iu_.get(), irho_.get(), my_lo, s_);
        launch_pack_halo(n_halo_hi_, halo_inst_.get() + n_halo_lo_, iq_.get(), iu_.get(), irho_.get(), my_hi, s_);
        comm_barrier();
        remote_lo_ = peer_lo_ ? peer_lo_ + (1 * 2 + par) * reg : nullptr;
        remote_hi_ = peer_hi_ ? peer_hi_ + (0 * 2 + par) * reg : nullptr;
        return;
    }
    launch_pack_halo(n, halo_inst_.get(), iq_.get(), iu_.get(), irho_.get(), hsend_.get(), s_);
    if (comm_.halo(comm_.user, hsend_.get(), hrecv_.get(), lo, hsend_.get() + lo, hrecv_.get() + lo,
                   hi, reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: halo exchange failed");
    remote_lo_ = hrecv_.get();
    remote_hi_ = hrecv_.get() + lo;
}

std::vector<double> Engine::allgather_host(const std::vector<double>& mine) {
    // fixed record width so every rank passes the same count
    int pmax = 0;
    for (int r = 0; r < comm_.world; ++r)
        pmax = std::max(pmax, comm_.part_offsets[r + 1] - comm_.part_offsets[r]);
    const size_t count = 2 + 4 * static_cast<size_t>(pmax);
    std::vector<double> rec(mine);
    rec.resize(count, 0.0);
    rec_.upload(rec, s_);
    rec_all_.resize(count * comm_.world);
    if (comm_.allgather(comm_.user, rec_.get(), rec_all_.get(), count,
                        reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: all-gather failed");
    return rec_all_.to_host(s_);
}

void Engine::commit_gather() {
    // Each rank publishes only the bodies it owns (its partitions hold the
    // body's lowest holder, the replica whose copy wins): a count all-gather,
    // then records (id, q, qdot) at the largest rank's count
    const int nb = hs_.nb;
    own_cnt_.resize(1);
    own_cnt_.zero(s_);
    own_rec_.resize(13 * static_cast<size_t>(std::max(nb, 1)));
    launch_pack_owned(ds_.view(), bmask_.get(), p0_, p1_, q_.get(), qd_.get(), own_rec_.get(), own_cnt_.get(), s_);
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 12, own_cnt_.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    sync();
    const std::vector<double> counts = allgather_host({static_cast<double>(pin_i_[12])});
    const size_t cstride = counts.size() / comm_.world;
    int cmax = 0;
    std::vector<int> cnt(comm_.world);
    for (int r = 0; r < comm_.world; ++r) {
        cnt[r] = static_cast<int>(counts[cstride * r]);
        cmax = std::max(cmax, cnt[r]);
    }
    if (cmax == 0) return;
    const size_t stride = 13 * static_cast<size_t>(cmax);
    own_rec_.resize(std::max(own_rec_.size(), stride));
    gath_.resize(stride * comm_.world);
    if (comm_.allgather(comm_.user, own_rec_.get(), gath_.get(), stride, reinterpret_cast<uintptr_t>(s_)) != 0)
        throw Error("comm: commit all-gather failed");
    own_cnts_.upload(cnt, s_);
    launch_unpack_owned(comm_.world, own_cnts_.get(), gath_.get(), stride, q_.get(), qd_.get(), s_);
}

void Engine::check_err(const char* where) {
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get(), err_.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
    const int code = pin_i_[0];
    if (code != 0) {
        err_.zero(s_);
        CUDA_CHECK(cudaStreamSynchronize(s_));
        throw DeviceError(std::string(err_text(code)) + " [" + where + "]", code);
    }
}

void Engine::sync() {
    CUDA_CHECK(cudaStreamSynchronize(s_));
    check_err("sync");
}

// ---------------------------------------------------------------------------
// instance sets
// ---------------------------------------------------------------------------
void Engine::build_instances(const std::vector<std::vector<int>>& per_part, const uint32_t* masks,
                             bool single_domain) {
    // (partition, body) of every row of the outgoing set: the PCG warm start
    // of a row that survives into the new set is carried over (per partition,
    // so N ranks and one GPU hand a partition the same starting guess);
    // every other row starts from zero
    std::vector<std::pair<long long, int>> old_keys(h_rinst_.size());
    for (size_t r = 0; r < h_rinst_.size(); ++r)
        old_keys[r] = {(static_cast<long long>(h_rpart_[r]) << 32) | h_ibody_[h_rinst_[r]], static_cast<int>(r)};
    if (h_rinst_.empty() && rowtab_valid_ && n_rows_ > 0) {
        // the outgoing set came from the device builder: its (partition,
        // body) -> row table stands in for the host lists
        const std::vector<int> tab = rowtab_.to_host(s_);
        const int nb = std::max(hs_.nb, 1);
        for (size_t t = 0; t < tab.size(); ++t)
            if (tab[t] >= 0)
                old_keys.push_back({(static_cast<long long>(p0_ + static_cast<int>(t / nb)) << 32) |
                                        static_cast<long long>(t % nb),
                                    tab[t]});
    }
    std::sort(old_keys.begin(), old_keys.end());
    const int r_old = n_rows_;
    h_ibody_.clear();
    h_ipart_.clear();
    h_irow_.clear();
    h_rinst_.clear();
    h_rpart_.clear();
    h_stat_.clear();
    h_pio_.assign(P_ + 1, 0);
    h_pro_.assign(P_ + 1, 0);
    for (int p = 0; p < P_; ++p) {
        h_pio_[p] = static_cast<int>(h_ibody_.size());
        h_pro_[p] = static_cast<int>(h_rinst_.size());
        for (int b : per_part[p]) {
            const int i = static_cast<int>(h_ibody_.size());
            h_ibody_.push_back(b);
            h_ipart_.push_back(p0_ + p);
            if (hs_.is_static[b]) {
                h_irow_.push_back(-1);
                h_stat_.push_back(i);
            } else {
                h_irow_.push_back(static_cast<int>(h_rinst_.size()));
                h_rinst_.push_back(i);
                h_rpart_.push_back(p0_ + p);
            }
        }
    }
    h_pio_[P_] = static_cast<int>(h_ibody_.size());
    h_pro_[P_] = static_cast<int>(h_rinst_.size());
    n_inst_ = static_cast<int>(h_ibody_.size());
    n_rows_ = static_cast<int>(h_rinst_.size());
    n_stat_ = static_cast<int>(h_stat_.size());
    {
        // (partition, body) -> row table of this set, so a device-built set
        // that follows carries the PCG warm start exactly as a host one would
        const int nb = std::max(hs_.nb, 1);
        std::vector<int> tab(static_cast<size_t>(P_) * nb, -1);
        for (int r = 0; r < n_rows_; ++r) tab[static_cast<size_t>(h_rpart_[r] - p0_) * nb + h_ibody_[h_rinst_[r]]] = r;
        rowtab_.upload(tab, s_);
        rowtab_valid_ = true;
    }
    if (n_inst_ >= (1 << 22)) throw InvalidArg("too many body instances for the candidate key");
    single_domain_ = single_domain;
    invalidate_list();
    ref_ready_ = false; // the N=1 frame graph refers to the previous instance set
    graph_ok_ = false;
    ibody_.upload(h_ibody_, s_);
    ipart_.upload(h_ipart_, s_);
    irow_.upload(h_irow_, s_);
    rinst_.upload(h_rinst_, s_);
    rpart_.upload(h_rpart_, s_);
    stat_.upload(h_stat_, s_);
    pio_.upload(h_pio_, s_);
    pro_.upload(h_pro_, s_);
    const size_t I = std::max(n_inst_, 1), R = std::max(n_rows_, 1);
    for (DBuf<double>* b : {&iq_, &iqtry_, &iqt_, &iz_, &iu_, &iznext_, &iqbefore_, &qref_})
        b->resize(6 * I);
    for (DBuf<double>* b : {&iinvk_, &irho_, &irho0_, &rb_, &sb_, &iskin_, &iskin_next_}) b->resize(I);
    ianc_.resize(I);
    ianc_.zero(s_);
    iu_.zero(s_);
    {
        std::vector<int> map(R, -1);
        bool carried = false;
        for (int r = 0; r < n_rows_; ++r) {
            const long long key = (static_cast<long long>(h_rpart_[r]) << 32) | h_ibody_[h_rinst_[r]];
            const auto it = std::lower_bound(old_keys.begin(), old_keys.end(), std::make_pair(key, -1));
            if (it != old_keys.end() && it->first == key) {
                map[r] = it->second;
                carried = true;
            }
        }
        if (carried) { // old rows (x, p2) out of the way before the buffers are reused
            warm_prev_.resize(12 * static_cast<size_t>(r_old));
            CUDA_CHECK(cudaMemcpyAsync(warm_prev_.get(), x_.get(), 6 * r_old * sizeof(double),
                                       cudaMemcpyDeviceToDevice, s_));
            CUDA_CHECK(cudaMemcpyAsync(warm_prev_.get() + 6 * r_old, pbuf_.get(), 6 * r_old * sizeof(double),
                                       cudaMemcpyDeviceToDevice, s_));
        }
        for (DBuf<double>* b : {&rgrad_, &x_, &r_, &z_, &p0v_, &p1v_, &ap_}) b->resize(6 * R);
        pbuf_.resize(12 * R);
        if (carried) {
            warm_map_.upload(map, s_);
            launch_warm_remap(n_rows_, warm_map_.get(), warm_prev_.get(), r_old, x_.get(), pbuf_.get(), s_);
        } else {
            x_.zero(s_);
            pbuf_.zero(s_);
        }
    }
    rdiag_.resize(36 * R);
    rdinv_.resize(36 * R);
    rval_.resize(R);
    rowtmp_.resize(R);
    rowtmp2_.resize(R);
    ell_cnt_.resize(R);
    ell_col_.resize(R * ell_w_);
    ell_blk_.resize(R * ell_w_ * 36);
    partial_.resize(static_cast<size_t>(segsum_chunks(std::max(n_inst_ * 64, 1 << 16))) * P_ + P_);
    if (masks) {
        bmask_.upload(masks, hs_.nb, s_);
    } else {
        bmask_.resize(std::max(hs_.nb, 1));
    }
    aoff_.resize(I + 1);
    boff_.resize(I + 1);
}

// Device-side instance set of a multi-partition attempt (runtime.cpp:126-236,
// partition.cpp:69-129): the same sets, order and per-instance constants as
// build_instances + frame_admm's host loops (instances sorted by (partition,
// body), rows = dynamic instances, static list, 1/kappa_b, anchor flags,
// rho0 = beta m_b and the carried rho, the shared-replica pairs, the PCG
// warm-start map by (partition, body)), from flags of every (partition, body)
// pair and three exclusive scans. One read-back: the counts (and w).
int Engine::build_instances_device(const uint32_t* masks_dev, double* w_out) {
    const int nb = hs_.nb;
    const size_t n = static_cast<size_t>(P_) * std::max(nb, 1);
    for (DBuf<int>* b : {&fl_all_, &fl_dyn_, &fl_sh_, &sc_all_, &sc_dyn_, &sc_sh_}) b->resize(n);
    if (rowtab_.size() != n) rowtab_valid_ = false;
    rowtab_.resize(n);
    rowtab_prev_.resize(n);
    inst_cnt_.resize(5 + 2 * static_cast<size_t>(P_));
    inst_cnt_h_.resize(8 + 2 * static_cast<size_t>(P_));
    launch_inst_flags(ds_.view(), masks_dev, P_, p0_, fl_all_.get(), fl_dyn_.get(), fl_sh_.get(), s_);
    size_t tb = 0;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, fl_all_.get(), sc_all_.get(), static_cast<int>(n)));
    scan_temp_.resize(std::max<size_t>(tb, 1));
    for (int k = 0; k < 3; ++k) {
        const int* in = k == 0 ? fl_all_.get() : k == 1 ? fl_dyn_.get() : fl_sh_.get();
        int* out = k == 0 ? sc_all_.get() : k == 1 ? sc_dyn_.get() : sc_sh_.get();
        size_t t2 = tb;
        CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scan_temp_.get(), t2, in, out, static_cast<int>(n), s_));
    }
    launch_inst_counts(P_, nb, fl_all_.get(), fl_dyn_.get(), fl_sh_.get(), sc_all_.get(), sc_dyn_.get(),
                       sc_sh_.get(), inst_cnt_.get(), s_);
    CUDA_CHECK(cudaMemcpyAsync(inst_cnt_h_.get(), inst_cnt_.get(), (5 + 2 * P_) * sizeof(int),
                               cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_d_.get() + 160, gate_.get() + 1, sizeof(double), cudaMemcpyDeviceToHost, s_));
    sync(); // the only host read of the instance build
    if (w_out) *w_out = pin_d_[160];
    const int I = inst_cnt_h_[0], R = inst_cnt_h_[1], ns = inst_cnt_h_[2];
    if (I >= (1 << 22)) throw InvalidArg("too many body instances for the candidate key");
    h_pio_.assign(inst_cnt_h_.get() + 3, inst_cnt_h_.get() + 4 + P_);
    h_pro_.assign(inst_cnt_h_.get() + 4 + P_, inst_cnt_h_.get() + 5 + 2 * P_);
    // host mirrors of the per-instance lists are not built on this path
    h_ibody_.clear();
    h_ipart_.clear();
    h_irow_.clear();
    h_rinst_.clear();
    h_rpart_.clear();
    h_stat_.clear();
    const int r_old = n_rows_;
    n_inst_ = I;
    n_rows_ = R;
    n_stat_ = I - R;
    single_domain_ = false;
    invalidate_list();
    ref_ready_ = false;
    graph_ok_ = false;
    const size_t Ic = std::max(I, 1), Rc = std::max(R, 1);
    for (DBuf<int>* b : {&ibody_, &ipart_, &irow_, &ianc_}) b->resize(Ic);
    rinst_.resize(Rc);
    rpart_.resize(Rc);
    stat_.resize(std::max(I - R, 1));
    pio_.resize(P_ + 1);
    pro_.resize(P_ + 1);
    shared_inst_.resize(2 * static_cast<size_t>(std::max(ns, 1)));
    warm_map_.resize(Rc);
    for (DBuf<double>* b : {&iq_, &iqtry_, &iqt_, &iz_, &iu_, &iznext_, &iqbefore_, &qref_}) b->resize(6 * Ic);
    for (DBuf<double>* b : {&iinvk_, &irho_, &irho0_, &rb_, &sb_, &iskin_, &iskin_next_}) b->resize(Ic);
    iu_.zero(s_);
    // the previous rows' (x, p2) out of the way before the buffers are reused
    const bool carry = rowtab_valid_ && r_old > 0;
    if (carry) {
        warm_prev_.resize(12 * static_cast<size_t>(r_old));
        CUDA_CHECK(cudaMemcpyAsync(warm_prev_.get(), x_.get(), 6 * r_old * sizeof(double), cudaMemcpyDeviceToDevice, s_));
        CUDA_CHECK(cudaMemcpyAsync(warm_prev_.get() + 6 * r_old, pbuf_.get(), 6 * r_old * sizeof(double),
                                   cudaMemcpyDeviceToDevice, s_));
        std::swap(rowtab_, rowtab_prev_);
    }
    InstOut o{ibody_.get(), ipart_.get(), irow_.get(), rinst_.get(), rpart_.get(), stat_.get(), ianc_.get(),
              shared_inst_.get(), warm_map_.get(), rowtab_.get(), pio_.get(), pro_.get(),
              iinvk_.get(), irho_.get(), irho0_.get()};
    launch_inst_scatter(ds_.view(), masks_dev, P_, p0_, fl_all_.get(), fl_dyn_.get(), fl_sh_.get(), sc_all_.get(),
                        sc_dyn_.get(), sc_sh_.get(), hs_.adapt.beta, rho_carry_d_.get(),
                        carry ? rowtab_prev_.get() : nullptr, o, s_);
    rowtab_valid_ = true;
    CUDA_CHECK(cudaMemcpyAsync(pio_.get(), inst_cnt_.get() + 3, (P_ + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s_));
    CUDA_CHECK(cudaMemcpyAsync(pro_.get(), inst_cnt_.get() + 4 + P_, (P_ + 1) * sizeof(int),
                               cudaMemcpyDeviceToDevice, s_));
    for (DBuf<double>* b : {&rgrad_, &x_, &r_, &z_, &p0v_, &p1v_, &ap_}) b->resize(6 * Rc);
    pbuf_.resize(12 * Rc);
    if (carry) {
        launch_warm_remap(R, warm_map_.get(), warm_prev_.get(), r_old, x_.get(), pbuf_.get(), s_);
    } else {
        x_.zero(s_);
        pbuf_.zero(s_);
    }
    rdiag_.resize(36 * Rc);
    rdinv_.resize(36 * Rc);
    rval_.resize(Rc);
    rowtmp_.resize(Rc);
    rowtmp2_.resize(Rc);
    ell_cnt_.resize(Rc);
    ell_col_.resize(Rc * ell_w_);
    ell_blk_.resize(Rc * ell_w_ * 36);
    partial_.resize(static_cast<size_t>(segsum_chunks(std::max(I * 64, 1 << 16))) * P_ + P_);
    bmask_.resize(std::max(nb, 1));
    if (nb) CUDA_CHECK(cudaMemcpyAsync(bmask_.get(), masks_dev, nb * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s_));
    aoff_.resize(Ic + 1);
    boff_.resize(Ic + 1);
    return ns;
}

void Engine::gather_iq(const double* q_dev) {
    launch_gather(n_inst_, ibody_.get(), q_dev, iq_.get(), s_);
}

SolverView Engine::view() {
    SolverView v;
    v.sc = ds_.view();
    v.n_inst = n_inst_;
    v.n_rows = n_rows_;
    v.n_parts = P_;
    v.part_base = p0_;
    v.ibody = ibody_.get();
    v.ipart = ipart_.get();
    v.irow = irow_.get();
    v.iq = iq_.get();
    v.iq_try = iqtry_.get();
    v.iqt = iqt_.get();
    v.iinvk = iinvk_.get();
    v.ianc = ianc_.get();
    v.iz = iz_.get();
    v.iu = iu_.get();
    v.irho = irho_.get();
    v.bmask = bmask_.get();
    v.single_domain = single_domain_ ? 1 : 0;
    v.rinst = rinst_.get();
    v.rpart = rpart_.get();
    v.rgrad = rgrad_.get();
    v.rdiag = rdiag_.get();
    v.rdinv = rdinv_.get();
    v.rval = rval_.get();
    v.ell_cnt = ell_cnt_.get();
    v.ell_col = ell_col_.get();
    v.ell_blk = ell_blk_.get();
    v.ell_w = ell_w_;
    v.x = x_.get();
    v.r = r_.get();
    v.z = z_.get();
    v.p0 = p0v_.get();
    v.p1 = p1v_.get();
    v.ap = ap_.get();
    v.part_row_off = pro_.get();
    v.part_inst_off = pio_.get();
    v.ps = ps_.get();
    v.h = frame_params_.h;
    v.d_hat = frame_params_.d_hat;
    v.kappa_bar = frame_params_.barrier_stiffness;
    v.kappa_arap = frame_params_.arap_stiffness;
    v.project = project_;
    v.perf = perf_.get();
    v.pcg_phases = pcg_phases_;
    v.err = err_.get();
    return v;
}

ContactView Engine::cview() {
    ContactView c;
    c.n = cap_;              // list capacity
    c.dn = det_.d_count();   // device-side list length
    c.fmt = cfmt_;
    c.key = det_.keys();
    c.perm_b = perm_b_.get();
    c.aoff = aoff_.get();
    c.boff = boff_.get();
    c.flag = cflag_.get();
    c.act = act_.get();
    c.ls = lstate_.get();
    c.cval = cval_.get();
    c.cgrad = cgrad_.get();
    c.cblk = cblk_.get();
    return c;
}

InstView Engine::iview(const double* q0, const double* q1) {
    InstView v;
    v.n = n_inst_;
    v.body = ibody_.get();
    v.part = ipart_.get();
    v.q0 = q0;
    v.q1 = q1;
    return v;
}

// ---------------------------------------------------------------------------
// local solve: enqueue-only building blocks (no host reads, capturable)
// ---------------------------------------------------------------------------
void Engine::prepare_solver() {
    ++solver_epoch_; // buffers, sizes and frame parameters may change: recapture the Newton graph
    // per-partition constants (ndof) live in PartState; kOpReset keeps them
    for (int p = 0; p < P_; ++p) {
        PartState& s = ps_h_[p];
        std::memset(&s, 0, sizeof(PartState));
        s.ndof = 6 * (h_pro_[p + 1] - h_pro_[p]);
        s.toi_earliest = 2.0;
        s.alpha = 1.0;
    }
    CUDA_CHECK(cudaMemcpyAsync(ps_.get(), ps_h_.get(), P_ * sizeof(PartState),
                               cudaMemcpyHostToDevice, s_));
    const int want = std::max(cap_, 48 * std::max(n_inst_, 1) + 4096);
    admm_prof().mark(9, s_);
    if (want != cap_ || det_.cap() != want || det_fmt_n_ != n_inst_) {
        cap_ = want;
        det_.prepare(n_inst_, ds_.max_verts, cap_);
        det_fmt_n_ = n_inst_;
        graph_ok_ = false;
    }
    admm_prof().mark(10, s_);
    const size_t C = static_cast<size_t>(cap_);
    const size_t before = cflag_.capacity() + act_.capacity() + cblk_.capacity();
    cflag_.resize(C);
    sval_.resize(C);
    act_.resize(C);
    cval_.resize(C);
    cgrad_.resize(12 * C);
    cblk_.resize(108 * C);
    invalidate_list();
    bkey_.resize(C);
    bkey_sorted_.resize(C);
    bidx_.resize(C);
    perm_b_.resize(C);
    partial_.resize(static_cast<size_t>(std::max(segsum_chunks(std::max(cap_, n_rows_)),
                                                 energy_chunks(cap_) + energy_chunks(n_rows_))) * P_ + P_);
    // (x_ / pbuf_, the PCG warm start, are (re)initialised by build_instances)
    pcg_part_.resize(std::max(3 * static_cast<size_t>(pcg_grid_size(std::max(n_rows_, 1))),
                              8 * static_cast<size_t>(pcg_grid_blocks())) * P_);
    if (max_part_rows() > kClusterPcgMaxRows) pcg_vec_.resize(60 * static_cast<size_t>(std::max(n_rows_, 1)));
    (void)pcg_cluster_size(); // resolve cluster attributes before any graph capture
    box_.resize(std::max(n_inst_, 1));
    admm_prof().mark(11, s_);
    size_t t1 = 0, t2 = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, t2, bkey_.get(), bkey_sorted_.get(),
                                               bidx_.get(), perm_b_.get(), cap_, 0,
                                               det_.fmt().total_bits()));
    temp_bytes_ = std::max(t1, t2);
    temp_.resize(temp_bytes_);
    if (cflag_.capacity() + act_.capacity() + cblk_.capacity() != before) graph_ok_ = false;
    cfmt_ = det_.fmt();
}

void Engine::enq_superset(const double* q0, const double* q1, bool swept) {
    det_.enqueue(ds_.view(), iview(q0, q1), stat_.get(), n_stat_, swept,
                 frame_params_.d_hat, err_.get(), s_);
}

void Engine::invalidate_list() {
    ListState ls{};
    ls.valid = 0;
    CUDA_CHECK(cudaStreamSynchronize(s_)); // lstate_h_ doubles as the read-back buffer
    lstate_h_[0] = ls;
    rebuilds_seen_ = 0;
    CUDA_CHECK(cudaMemcpyAsync(lstate_.get(), lstate_h_.get(), sizeof(ListState),
                               cudaMemcpyHostToDevice, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
}

// Skin list rebuild at qref = iq with the margin k_list_check wrote
// (d_hat + 2 delta): the detector's static broad phase, the a-segment
// offsets, and the b-sorted permutation with its segment offsets.
void Engine::enq_list_rebuild() {
    launch_list_commit(n_inst_, iq_.get(), qref_.get(), iskin_next_.get(), iskin_.get(), s_);
    InstView iv = iview(iq_.get(), iq_.get());
    iv.skin = iskin_.get();
    det_.enqueue(ds_.view(), iv, stat_.get(), n_stat_, false,
                 frame_params_.d_hat, err_.get(), s_);
    launch_seg_offsets(det_.keys(), cap_, det_.d_count(), cfmt_, n_inst_, aoff_.get(), 0, nullptr, s_);
    launch_make_bkeys(det_.keys(), cap_, det_.d_count(), cfmt_, bkey_.get(), bidx_.get(), s_);
    size_t tb = temp_bytes_;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(temp_.get(), tb, bkey_.get(), bkey_sorted_.get(),
                                               bidx_.get(), perm_b_.get(), cap_, 0,
                                               cfmt_.total_bits(), s_));
    launch_seg_offsets(det_.keys(), cap_, det_.d_count(), cfmt_, n_inst_, boff_.get(), 1,
                       perm_b_.get(), s_);
}

// The list must cover iq and q1 (the CCD end point; the trials lie between).
// fused_ccd: q1 = iq + dq is formed by the check itself (k_ccd_prep), which
// also writes the swept CCD boxes.
void Engine::enq_list_ensure(const double* q1, bool fused_ccd) {
    const bool graph = hd_.graph != 0;
    const unsigned long long h = graph ? new_cond_handle() : 0ull;
    if (fused_ccd)
        launch_ccd_prep(view(), qref_.get(), iskin_.get(), iskin_next_.get(),
                        skin_min_ * frame_params_.d_hat, skin_grow_, lstate_.get(), h, graph ? 1 : 0,
                        nullptr, s_); // k_ccd runs without body boxes (the swept point/edge test implies them)
    else
        launch_list_check(ds_.view(), iview(iq_.get(), q1), qref_.get(), iqt_.get(), iskin_.get(),
                          iskin_next_.get(), skin_min_ * frame_params_.d_hat, skin_grow_,
                          lstate_.get(), h, graph ? 1 : 0, s_);
    if (graph) {
        add_cond_node(h, false, cap_level_ + 1, [&] { enq_list_rebuild(); }, false);
    } else {
        CUDA_CHECK(cudaMemcpyAsync(lstate_h_.get(), lstate_.get(), sizeof(ListState),
                                   cudaMemcpyDeviceToHost, s_));
        CUDA_CHECK(cudaStreamSynchronize(s_));
        if (lstate_h_[0].rebuild) enq_list_rebuild();
    }
}

// Objective value of every flagged partition (fused k_energy): qmode 0 at
// iq, 1 at the line-search trial; accept = take kOpAccept afterwards.
void Engine::enq_energy(int qmode, int which, double PartState::*field, bool accept) {
    launch_energy(view(), det_.keys(), cap_, det_.d_count(), cfmt_, qmode, which, partial_.get(),
                  ps_field(ps_.get(), field), kPsStride, accept, ctrl_.get(), hd_, s_);
}

// fused: the trace sum, kOpEps and the preconditioner factor are left to
// the fused cluster PCG (pcg_fused()).
// fused (graph path of a Newton iteration): kOpIterBegin rides on the body
// terms, the contact selection recomputes body boxes and evaluates the
// contact terms in place: body -> select+terms -> assemble -> fused PCG.
void Engine::enq_derivatives(bool fused) {
    SolverView v = view();
    const ContactView cv = cview();
    if (fused) {
        // body terms and contact terms as two independent branches (kOpIterBegin's
        // resets ran in the kOpReset / kOpNewtonTail that decided this iteration)
        const cudaStream_t side = side_stream();
        CUDA_CHECK(cudaEventRecord(ev_fork_, s_));
        CUDA_CHECK(cudaStreamWaitEvent(side, ev_fork_, 0));
        launch_body_terms(v, iq_.get(), true, 0, side);
        launch_contact_select(v, cv, nullptr, s_, true);
        CUDA_CHECK(cudaEventRecord(ev_join_, side));
        CUDA_CHECK(cudaStreamWaitEvent(s_, ev_join_, 0));
        launch_assemble(v, cv, rowtmp_.get(), s_);
        return;
    }
    launch_inst_boxes(v.sc, iview(iq_.get(), iq_.get()), false, frame_params_.d_hat, box_.get(),
                      cellmax_.get(), s_);
    launch_body_terms(v, iq_.get(), true, 0, s_, &lstate_.get()->n_act);
    launch_contact_select(v, cv, box_.get(), s_);
    launch_contact_terms(v, cv, s_);
    launch_assemble(v, cv, rowtmp_.get(), s_);
    launch_segsum_rows(rowtmp_.get(), n_rows_, rpart_.get(), P_, p0_, partial_.get(),
                       ps_field(ps_.get(), &PartState::trace), kPsStride, false, s_);
    launch_scalar(ps_.get(), P_, kOpEps, ctrl_.get(), hd_, 0.0, 0, err_.get(), s_);
    if (project_) launch_precond(v, s_); // unprojected blocks (objective mode 3) may be indefinite
}

int Engine::max_part_rows() const {
    int max_rows = 0;
    for (int p = 0; p < P_; ++p) max_rows = std::max(max_rows, h_pro_[p + 1] - h_pro_[p]);
    return max_rows;
}

bool Engine::pcg_fused() const {
    return n_rows_ > 0 && project_ && max_part_rows() <= kClusterPcgMaxRows &&
           !std::getenv("DABD_GPU_NO_FUSED_PCG");
}

void Engine::enq_pcg(bool fused) {
    if (n_rows_ == 0) return;
    const int max_rows = max_part_rows();
    if (max_rows <= kClusterPcgMaxRows) {
        // small partitions: one thread-block cluster per partition (DSMEM dots)
        PcgFuse f{rowtmp_.get(), ctrl_.get(), hd_, inexact_ ? eta_loose_ : 0.0, eta_factor_, tail_max_iters_ > 0};
        launch_pcg_cluster(view(), max_rows, pbuf_.get(), pcg_tol_, pcg_max_, s_, fused ? &f : nullptr);
    } else {
        static const bool grid_kernel = [] {
            const char* e = std::getenv("DABD_GPU_PCG_GRID");
            return !e || e[0] != '0';
        }();
        if (grid_kernel) { // one grid barrier per iteration (pipelined CG); vectors sized in prepare_solver
            launch_pcg_grid(view(), pcg_vec_.get(), pcg_part_.get(), pcg_tol_, pcg_max_, s_,
                            inexact_ ? eta_loose_ : 0.0, eta_factor_);
        } else {
            launch_pcg_persistent(view(), pbuf_.get(), pcg_part_.get(), rowtmp_.get(), pcg_tol_,
                              pcg_max_, s_);
        }
    }
}

// newton.cpp:16-69, one iteration for every partition still active.
void Engine::enq_newton_head(int max_iters) {
    SolverView v = view();
    const bool fused = pcg_fused();
    if (!fused) launch_scalar(ps_.get(), P_, kOpIterBegin, ctrl_.get(), hd_, 0.0, max_iters, err_.get(), s_);
    enq_derivatives(fused);
    enq_pcg(fused);
    if (fused) return; // ||dq||_inf and kOpNewtonCheck ran inside the PCG kernel
    launch_dq_inf(v, s_);
    launch_scalar(ps_.get(), P_, kOpNewtonCheck, ctrl_.get(), hd_, 0.0, max_iters, err_.get(), s_);
}

// CCD bound over [q, q + dq] on the swept superset (newton.cpp:38-42).
void Engine::enq_newton_ccd() {
    SolverView v = view();
    if (pcg_fused()) {
        // k_ccd forms q + dq itself (q1 == nullptr) and needs no body boxes, so
        // it runs beside k_ccd_prep (skin check of the list) as a second branch:
        // [k_ccd(+kOpAlphaMax) || k_ccd_prep] IF(rebuild) { rebuild, toi reset,
        // k_ccd(+kOpAlphaMax) over the new list }. The first k_ccd's result is
        // discarded when the list was stale (rare); decisions are the same.
        const bool graph = hd_.graph != 0;
        const unsigned long long h = graph ? new_cond_handle() : 0ull;
        auto ccd = [&](cudaStream_t st) {
            launch_ccd(view(), det_.keys(), cap_, det_.d_count(), cfmt_, nullptr, iq_.get(), nullptr, 0,
                       nullptr, st, ctrl_.get(), &hd_);
        };
        const cudaStream_t side = side_stream();
        CUDA_CHECK(cudaEventRecord(ev_fork_, s_));
        CUDA_CHECK(cudaStreamWaitEvent(side, ev_fork_, 0));
        ccd(side);
        launch_ccd_prep(v, qref_.get(), iskin_.get(), iskin_next_.get(), skin_min_ * frame_params_.d_hat,
                        skin_grow_, lstate_.get(), h, graph ? 1 : 0, nullptr, s_);
        CUDA_CHECK(cudaEventRecord(ev_join_, side));
        CUDA_CHECK(cudaStreamWaitEvent(s_, ev_join_, 0));
        auto rerun = [&] {
            enq_list_rebuild();
            launch_toi_reset(ps_.get(), P_, ctrl_.get(), s_);
            ccd(s_);
        };
        if (graph) {
            // launch accounting: executed rebuilds count the plain rebuild's
            // nodes (the toi reset and the second k_ccd go uncounted)
            const long long keep = rebuild_nodes_;
            add_cond_node(h, false, cap_level_ + 1, rerun, false);
            if (keep > 0) rebuild_nodes_ = keep;
        } else {
            CUDA_CHECK(cudaMemcpyAsync(lstate_h_.get(), lstate_.get(), sizeof(ListState),
                                       cudaMemcpyDeviceToHost, s_));
            CUDA_CHECK(cudaStreamSynchronize(s_));
            if (lstate_h_[0].rebuild) rerun();
        }
        return;
    }
    launch_make_trial(v, false, 1.0, 0, s_);
    enq_list_ensure(iqtry_.get());
    launch_inst_boxes(v.sc, iview(iq_.get(), iqtry_.get()), true, 0.0, box_.get(), cellmax_.get(),
                      s_);
    launch_ccd(v, det_.keys(), cap_, det_.d_count(), cfmt_, box_.get(), iq_.get(), iqtry_.get(), 0,
               nullptr, s_);
    launch_scalar(ps_.get(), P_, kOpAlphaMax, ctrl_.get(), hd_, 0.0, 0, err_.get(), s_);
}

// One backtracking trial (newton.cpp:47-59) for every partition still searching.
void Engine::enq_ls_trial() {
    SolverView v = view();
    // small instance sets: the energy kernel's last block also applies the
    // accepted step (one launch per trial instead of two)
    const bool fuse = n_inst_ <= kFuseAcceptMaxInst;
    // captured fused body (cap_newton): the last trial also takes the Newton
    // tail when the accepted step is applied in the same kernel
    const int tail = hd_.graph && pcg_fused() && fuse ? tail_max_iters_ : 0;
    launch_energy(v, det_.keys(), cap_, det_.d_count(), cfmt_, 1, 1, partial_.get(),
                  ps_field(ps_.get(), &PartState::trial), kPsStride, true, ctrl_.get(), hd_, s_, fuse, tail,
                  tail ? iter_reset() : nullptr);
    if (!fuse) launch_accept_trial(v, s_);
}

int* Engine::iter_reset() { return pcg_fused() ? &lstate_.get()->n_act : nullptr; }

// Second stream of the current capture level (or of eager execution) for
// independent branches inside one Newton iteration.
cudaStream_t Engine::side_stream() {
    const int idx = cap_level_ + 1;
    while (static_cast<int>(side_streams_.size()) <= idx) {
        cudaStream_t s;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        side_streams_.push_back(s);
    }
    if (!ev_fork_) {
        CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        CUDA_CHECK(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    return side_streams_[idx];
}

void Engine::enq_solve_begin(double tol) {
    launch_scalar(ps_.get(), P_, kOpReset, ctrl_.get(), hd_, tol, 0, err_.get(), s_, iter_reset());
    enq_list_ensure(iq_.get());
    enq_energy(0, 0, &PartState::energy);
}

FrameCtrl Engine::read_ctrl() {
    CUDA_CHECK(cudaMemcpyAsync(ctrl_h_.get(), ctrl_.get(), sizeof(FrameCtrl),
                               cudaMemcpyDeviceToHost, s_));
    check_err("newton");
    return ctrl_h_[0];
}

// Host-driven variant (parity entry points, multi-partition ADMM frames).
NewtonResult Engine::newton_batch(int max_iters, double tol, bool reset_ctrl) {
    hd_ = CondHandles{};
    if (reset_ctrl) CUDA_CHECK(cudaMemsetAsync(ctrl_.get(), 0, sizeof(FrameCtrl), s_));
    enq_solve_begin(tol);
    FrameCtrl c = read_ctrl();
    for (int iter = 0; iter < max_iters && c.any_active; ++iter) {
        enq_newton_head(max_iters);
        c = read_ctrl();
        if (c.any_active) {
            enq_newton_ccd();
            c = read_ctrl();
            for (int t = 0; t < 80 && c.any_searching; ++t) {
                enq_ls_trial();
                c = read_ctrl();
            }
        }
        launch_scalar(ps_.get(), P_, kOpNewtonTail, ctrl_.get(), hd_, 0.0, max_iters, err_.get(), s_,
                      iter_reset());
        c = read_ctrl();
    }
    CUDA_CHECK(cudaMemcpyAsync(ps_h_.get(), ps_.get(), P_ * sizeof(PartState),
                               cudaMemcpyDeviceToHost, s_));
    check_err("newton: end");
    NewtonResult res;
    res.converged = 1;
    for (int p = 0; p < P_; ++p) {
        res.iterations += ps_h_[p].iterations;
        res.ls_steps += ps_h_[p].ls_steps;
        res.converged &= ps_h_[p].converged;
        res.final_update = std::max(res.final_update, ps_h_[p].final_update);
    }
    res.pcg_iters = c.pcg_total;
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 2, &lstate_.get()->n_act, sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 3, det_.d_count(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    sync();
    n_contacts_ = pin_i_[2];
    n_super_ = pin_i_[3];
    return res;
}

// Captured batched Newton solve for the multi-partition ADMM frame: the
// same conditional-node structure as the N=1 frame (cap_newton), captured
// once per solver epoch (instance set / capacities / h of the current
// attempt) and replayed for every ADMM iteration: one host synchronisation
// per local solve instead of several per Newton iteration.
NewtonResult Engine::newton_graph(int max_iters, double tol, const std::function<void()>& tail) {
    if (!newton_exec_ || newton_epoch_ != solver_epoch_ || newton_tol_ != tol || newton_max_ != max_iters) {
        KernelTimer::get().suspend(true);
        hd_ = CondHandles{};
        hd_.graph = 1;
        for (long long& v : nodes_inc_) v = 0;
        const long long c0 = launch_counter().load();
        CUDA_CHECK(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal));
        try {
            cap_newton(max_iters, tol, 0);
        } catch (...) {
            cudaGraph_t g;
            cudaStreamEndCapture(s_, &g);
            KernelTimer::get().suspend(false);
            hd_ = CondHandles{};
            throw;
        }
        cudaGraph_t g;
        CUDA_CHECK(cudaStreamEndCapture(s_, &g));
        KernelTimer::get().suspend(false);
        newton_total_ = launch_counter().load() - c0;
        launch_counter() -= newton_total_; // captured, not executed
        for (int k = 0; k < 4; ++k) newton_inc_[k] = nodes_inc_[k];
        // same topology as the last capture (the usual case: a new frame with
        // new buffers or h): update the executable graph in place, which is
        // much cheaper than instantiating it again
        bool updated = false;
        if (newton_exec_) {
            cudaGraphExecUpdateResultInfo info;
            updated = cudaGraphExecUpdate(newton_exec_, g, &info) == cudaSuccess;
            if (!updated) {
                cudaGetLastError();
                cudaGraphExecDestroy(newton_exec_);
                newton_exec_ = nullptr;
            }
        }
        if (!updated) CUDA_CHECK(cudaGraphInstantiate(&newton_exec_, g, 0));
        CUDA_CHECK(cudaGraphDestroy(g));
        hd_ = CondHandles{};
        newton_epoch_ = solver_epoch_;
        newton_tol_ = tol;
        newton_max_ = max_iters;
    }
    CUDA_CHECK(cudaMemsetAsync(ctrl_.get(), 0, sizeof(FrameCtrl), s_));
    CUDA_CHECK(cudaGraphLaunch(newton_exec_, s_));
    if (tail) tail();
    CUDA_CHECK(cudaMemcpyAsync(ps_h_.get(), ps_.get(), P_ * sizeof(PartState), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(lstate_h_.get(), lstate_.get(), sizeof(ListState), cudaMemcpyDeviceToHost, s_));
    const FrameCtrl c = read_ctrl(); // synchronises, raises a device error
    const long long rebuilds = lstate_h_[0].n_rebuilds - rebuilds_seen_;
    rebuilds_seen_ = lstate_h_[0].n_rebuilds;
    count_launch(rebuilds * rebuild_nodes_ + newton_total_ - newton_inc_[0] +
                 static_cast<long long>(c.exec_newton) * (newton_inc_[0] - newton_inc_[1]) +
                 static_cast<long long>(c.exec_step) * (newton_inc_[1] - newton_inc_[2]) +
                 static_cast<long long>(c.exec_ls) * newton_inc_[2]);
    NewtonResult res;
    res.converged = 1;
    for (int p = 0; p < P_; ++p) {
        res.iterations += ps_h_[p].iterations;
        res.ls_steps += ps_h_[p].ls_steps;
        res.converged &= ps_h_[p].converged;
        res.final_update = std::max(res.final_update, ps_h_[p].final_update);
    }
    res.pcg_iters = c.pcg_total;
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 2, &lstate_.get()->n_act, sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 3, det_.d_count(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    sync();
    n_contacts_ = pin_i_[2];
    n_super_ = pin_i_[3];
    return res;
}

// ---------------------------------------------------------------------------
// CUDA-graph capture helpers (conditional WHILE / IF nodes, CUDA 12.4+)
// ---------------------------------------------------------------------------
unsigned long long Engine::new_cond_handle() {
    cudaStreamCaptureStatus st;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CUDA_CHECK(cudaStreamGetCaptureInfo(s_, &st, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle h;
    CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    return static_cast<unsigned long long>(h);
}

void Engine::add_cond_node(unsigned long long h, bool is_while, int level,
                           const std::function<void()>& body, bool account) {
    cudaStreamCaptureStatus st;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CUDA_CHECK(cudaStreamGetCaptureInfo(s_, &st, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = static_cast<cudaGraphConditionalHandle>(h);
    p.conditional.type = is_while ? cudaGraphCondTypeWhile : cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    CUDA_CHECK(cudaGraphAddNode(&node, g, deps, nd, &p));
    CUDA_CHECK(cudaStreamUpdateCaptureDependencies(s_, &node, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t bg = p.conditional.phGraph_out[0];
    cudaStream_t saved = s_;
    const int saved_level = cap_level_;
    s_ = cap_stream(level);
    cap_level_ = level;
    CUDA_CHECK(cudaStreamBeginCaptureToGraph(s_, bg, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed));
    const long long before = launch_counter().load();
    body();
    const long long inc = launch_counter().load() - before;
    if (account) {
        if (level < 8) nodes_inc_[level] = inc;
    } else { // list rebuild: counted per executed rebuild, not per enclosing body
        rebuild_nodes_ = inc;
        launch_counter() -= inc;
    }
    cudaGraph_t out;
    CUDA_CHECK(cudaStreamEndCapture(s_, &out));
    s_ = saved;
    cap_level_ = saved_level;
}

cudaStream_t Engine::cap_stream(int level) {
    while (static_cast<int>(cap_streams_.size()) <= level) {
        cudaStream_t s;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        cap_streams_.push_back(s);
    }
    return cap_streams_[level];
}

// Captured Newton solve: Reset -> superset -> energy -> WHILE(active) {
//   head; IF(active) { CCD; WHILE(searching) { trial } }; tail }.
void Engine::cap_newton(int max_iters, double tol, int level) {
    hd_.newton = new_cond_handle();
    enq_solve_begin(tol);
    // fused body, small sets: the tail (newton.cpp:16's loop bound, the WHILE
    // condition, the next iteration's resets) rides on the last line-search
    // trial, and the PCG epilogue closes the loop when nothing stays active
    const bool folded_tail = pcg_fused() && n_inst_ <= kFuseAcceptMaxInst;
    tail_max_iters_ = folded_tail ? max_iters : 0;
    // flat fused body: no IF(step) node around the CCD and the line search.
    // After a converged PCG the CCD finds no active partition, its
    // kOpAlphaMax clears `searching` and the WHILE(ls) body never runs, so the
    // node only saved two short launches once per solve while costing its own
    // evaluation on every iteration. Launch accounting keeps the step level
    // (kOpAlphaMax counts exec_step once per executed CCD).
    static const bool flat_env = [] {
        const char* e = std::getenv("DABD_GPU_STEP_IF");
        return !(e && e[0] == '1');
    }();
    const bool flat = flat_env && pcg_fused();
    static const bool flat_ls = [] { // DABD_GPU_LS_FIRST_FLAT=0: the first trial inside WHILE(ls) too
        const char* e = std::getenv("DABD_GPU_LS_FIRST_FLAT");
        return !(e && e[0] == '0');
    }();
    add_cond_node(hd_.newton, true, level, [&] {
        auto step_body = [&] {
            hd_.ls = new_cond_handle();
            enq_newton_ccd();
            add_cond_node(hd_.ls, true, level + 2, [&] { enq_ls_trial(); });
        };
        if (flat) {
            hd_.step = 0;
            hd_.has_step = 0;
            enq_newton_head(max_iters);
            const long long before = launch_counter().load();
            if (flat_ls) {
                // the first line-search trial unconditionally (every iteration
                // tries alpha_max; with nothing searching it evaluates nothing
                // and its kOpAccept leaves every partition as it was), then
                // WHILE(ls) only for the halvings: the loop node is entered by
                // ~13% of the iterations
                hd_.ls = new_cond_handle();
                enq_newton_ccd();
                const long long b1 = launch_counter().load();
                enq_ls_trial();
                const long long first = launch_counter().load() - b1;
                launch_counter() -= first; // counted per executed trial through exec_ls x the ls body
                add_cond_node(hd_.ls, true, level + 2, [&] { enq_ls_trial(); });
            } else {
                step_body();
            }
            if (level + 1 < 8) nodes_inc_[level + 1] = launch_counter().load() - before;
        } else {
            hd_.step = new_cond_handle(); // set by kOpNewtonCheck inside the head
            hd_.has_step = 1;
            enq_newton_head(max_iters);
            add_cond_node(hd_.step, false, level + 1, step_body);
        }
        if (!folded_tail)
            launch_scalar(ps_.get(), P_, kOpNewtonTail, ctrl_.get(), hd_, 0.0, max_iters, err_.get(), s_,
                          iter_reset());
    });
    tail_max_iters_ = 0;
}


std::vector<double> Engine::delta_inf(const double* a, const double* b) {
    gate_.zero(s_);
    launch_delta_inf(n_rows_, rinst_.get(), rpart_.get(), p0_, a, b, gate_.get(), s_);
    std::vector<double> out = gate_.to_host(s_);
    out.resize(P_);
    return out;
}

// ---------------------------------------------------------------------------
// parity entry points
// ---------------------------------------------------------------------------
static std::vector<int> subset_sorted(const int* subset, int n, int nb) {
    std::vector<int> sub;
    if (subset && n > 0) {
        sub.assign(subset, subset + n);
        for (int b : sub)
            if (b < 0 || b >= nb) throw InvalidArg("subset body index out of range");
    } else {
        sub.resize(nb);
        std::iota(sub.begin(), sub.end(), 0);
    }
    std::sort(sub.begin(), sub.end());
    if (std::adjacent_find(sub.begin(), sub.end()) != sub.end())
        throw InvalidArg("subset has duplicate bodies");
    return sub;
}

std::vector<int> Engine::broad_phase(const double* q, const double* q_end, double margin,
                                     const int* subset, int n_subset) {
    const std::vector<int> sub = subset_sorted(subset, n_subset, hs_.nb);
    std::vector<std::vector<int>> per(P_);
    per[0] = sub;
    build_instances(per, nullptr, true);
    DBuf<double> gq, gqe;
    gq.upload(q, 6 * static_cast<size_t>(hs_.nb), s_);
    gather_iq(gq.get());
    const double* q1 = iq_.get();
    if (q_end) {
        gqe.upload(q_end, 6 * static_cast<size_t>(hs_.nb), s_);
        launch_gather(n_inst_, ibody_.get(), gqe.get(), iqtry_.get(), s_);
        q1 = iqtry_.get();
    }
    const int n = det_gate_.build(ds_.view(), iview(iq_.get(), q1), stat_.get(),
                                  n_stat_, q_end != nullptr, margin,
                                  ds_.max_verts, s_);
    std::vector<unsigned long long> keys(n);
    if (n) {
        CUDA_CHECK(cudaMemcpyAsync(keys.data(), det_gate_.keys(), n * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, s_));
    }
    sync();
    std::vector<int> out(4 * static_cast<size_t>(n));
    const KeyFmt f = det_gate_.fmt();
    for (int t = 0; t < n; ++t) {
        int a, b, v, e;
        f.unpack(keys[t], a, b, v, e);
        out[4 * t] = h_ibody_[a];
        out[4 * t + 1] = h_ibody_[b];
        out[4 * t + 2] = v;
        out[4 * t + 3] = e;
    }
    return out;
}

void Engine::narrow_phase(const double* q, const int* cand, int n, double d_hat,
                          std::vector<int>& pairs, std::vector<double>& d) {
    pairs.clear();
    d.clear();
    if (n <= 0) return;
    for (int t = 0; t < n; ++t) {
        const int a = cand[4 * t], b = cand[4 * t + 1];
        if (a < 0 || a >= hs_.nb || b < 0 || b >= hs_.nb) throw InvalidArg("candidate body out of range");
        if (cand[4 * t + 2] < 0 || cand[4 * t + 2] >= hs_.vstart[a + 1] - hs_.vstart[a] ||
            cand[4 * t + 3] < 0 || cand[4 * t + 3] >= hs_.vstart[b + 1] - hs_.vstart[b])
            throw InvalidArg("candidate primitive index out of range");
    }
    DBuf<double> gq, dd;
    DBuf<int> gc, fl;
    gq.upload(q, 6 * static_cast<size_t>(hs_.nb), s_);
    gc.upload(cand, 4 * static_cast<size_t>(n), s_);
    dd.resize(n);
    fl.resize(n);
    launch_narrow_bodies(ds_.view(), gq.get(), gc.get(), n, d_hat, dd.get(), fl.get(), err_.get(), s_);
    std::vector<double> hd = dd.to_host(s_);
    std::vector<int> hf = fl.to_host(s_);
    check_err("narrow_phase");
    for (int t = 0; t < n; ++t)
        if (hf[t]) {
            pairs.insert(pairs.end(), cand + 4 * t, cand + 4 * t + 4);
            d.push_back(hd[t]);
        }
}

double Engine::ccd_toi(const double* q0, const double* q1, const int* subset, int n_subset) {
    const std::vector<int> sub = subset_sorted(subset, n_subset, hs_.nb);
    std::vector<std::vector<int>> per(P_);
    per[0] = sub;
    build_instances(per, nullptr, true);
    DBuf<double> g0, g1;
    g0.upload(q0, 6 * static_cast<size_t>(hs_.nb), s_);
    g1.upload(q1, 6 * static_cast<size_t>(hs_.nb), s_);
    gather_iq(g0.get());
    launch_gather(n_inst_, ibody_.get(), g1.get(), iqtry_.get(), s_);
    const int n = det_gate_.build(ds_.view(), iview(iq_.get(), iqtry_.get()), stat_.get(),
                                  n_stat_, true, 0.0, ds_.max_verts, s_);
    std::vector<double> init(P_, 2.0);
    gate_.upload(init, s_);
    // margin-0 swept candidates are exactly the reference set; the filter
    // inside k_ccd re-applies the same predicate with the detector's boxes.
    launch_ccd(view(), det_gate_.keys(), n, nullptr, det_gate_.fmt(), det_gate_.boxes(), iq_.get(),
               iqtry_.get(), 2, gate_.get(), s_);
    std::vector<double> e = gate_.to_host(s_);
    check_err("ccd_toi");
    const double earliest = e[0];
    if (earliest > 1.0) return 1.0;
    return std::min(1.0, 0.9 * earliest);
}

AuditResult Engine::audit(const double* q, const int* subset, int n_subset, double cutoff) {
    const std::vector<int> sub = subset_sorted(subset, n_subset, hs_.nb);
    const double* qd = q_.get();
    if (q) {
        audit_q_.upload(q, 6 * static_cast<size_t>(hs_.nb), s_);
        qd = audit_q_.get();
    }
    return auditor_.run(ds_.view(), qd, sub, cutoff, s_);
}

void Engine::holder_masks(const double* q, int np, const double* planes, double w, uint32_t* out) {
    if (hs_.nb == 0) return;
    DBuf<double> gq, gp;
    DBuf<uint32_t> gm;
    gq.upload(q, 6 * static_cast<size_t>(hs_.nb), s_);
    gp.resize(std::max(4 * np, 4));
    if (np > 0) gp.upload(planes, 4 * static_cast<size_t>(np), s_);
    gm.resize(hs_.nb);
    const uint32_t all = (np + 1) >= 32 ? 0xffffffffu : ((1u << (np + 1)) - 1u);
    launch_masks(ds_.view(), gq.get(), gp.get(), np, w, all, gm.get(), err_.get(), s_);
    gm.download(out, hs_.nb, s_);
    sync();
}

void Engine::objective(const ObjectiveIn& in, const double* q, int mode, double* value,
                       double* grad, double* hess_dense, int* active, int* candidates) {
    in.sim.validate();
    frame_params_ = in.sim;
    std::vector<int> order(in.n_local);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return in.local[a] < in.local[b]; });
    std::vector<std::vector<int>> per(P_);
    for (int k : order) {
        if (in.local[k] < 0 || in.local[k] >= hs_.nb) throw InvalidArg("LocalObjective: body index out of range");
        per[0].push_back(in.local[k]);
    }
    if (std::adjacent_find(per[0].begin(), per[0].end()) != per[0].end())
        throw InvalidArg("LocalObjective: duplicate local body");
    build_instances(per, in.holder_mask, in.holder_mask == nullptr);
    const int I = n_inst_;
    std::vector<double> qt(6 * I), invk(I), z(6 * I, 0.0), u(6 * I, 0.0), rho(I, 0.0);
    std::vector<int> anc(I, 0);
    for (int i = 0; i < I; ++i) {
        const int k = order[i];
        for (int c = 0; c < 6; ++c) qt[6 * i + c] = in.q_tilde[6 * k + c];
        invk[i] = 1.0 / in.kappa[k];
    }
    for (int a = 0; a < in.n_anchor; ++a) {
        const int b = in.anchor_body[a];
        const auto it = std::lower_bound(per[0].begin(), per[0].end(), b);
        if (b < 0 || b >= hs_.nb || it == per[0].end() || *it != b)
            throw InvalidArg("LocalObjective: anchor for a body not on this worker");
        if (hs_.is_static[b]) throw InvalidArg("LocalObjective: anchor on a static body");
        const int i = static_cast<int>(it - per[0].begin());
        if (anc[i]) throw InvalidArg("LocalObjective: duplicate anchor for one body");
        anc[i] = mode == 1 ? 0 : 1;
        for (int c = 0; c < 6; ++c) {
            z[6 * i + c] = in.anchor_zu[12 * a + c];
            u[6 * i + c] = in.anchor_zu[12 * a + 6 + c];
        }
        rho[i] = in.anchor_rho[a];
    }
    iqt_.upload(qt, s_);
    iinvk_.upload(invk, s_);
    iz_.upload(z, s_);
    iu_.upload(u, s_);
    irho_.upload(rho, s_);
    ianc_.upload(anc, s_);
    DBuf<double> gq;
    gq.upload(q, 6 * static_cast<size_t>(hs_.nb), s_);
    gather_iq(gq.get());
    ref_ready_ = false;
    prepare_solver();
    hd_ = CondHandles{};
    CUDA_CHECK(cudaMemsetAsync(ctrl_.get(), 0, sizeof(FrameCtrl), s_));
    launch_scalar(ps_.get(), P_, kOpReset, ctrl_.get(), hd_, 0.0, 0, err_.get(), s_);
    enq_list_ensure(iq_.get());
    if (mode <= 1) {
        enq_energy(0, 2, &PartState::energy);
        enq_derivatives(); // counts only
        CUDA_CHECK(cudaMemcpyAsync(ps_h_.get(), ps_.get(), P_ * sizeof(PartState),
                                   cudaMemcpyDeviceToHost, s_));
        CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 2, &lstate_.get()->n_act, sizeof(int),
                                   cudaMemcpyDeviceToHost, s_));
        sync();
        *value = ps_h_[0].energy;
        *active = pin_i_[2];
        *candidates = ps_h_[0].n_candidates;
        return;
    }
    // derivatives (value as the sum of body and contact terms)
    project_ = mode == 2 ? 1 : 0;
    enq_derivatives();
    project_ = 1;
    CUDA_CHECK(cudaMemcpyAsync(ps_h_.get(), ps_.get(), P_ * sizeof(PartState),
                               cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 2, &lstate_.get()->n_act, sizeof(int),
                               cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 3, det_.d_count(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    std::vector<double> rv = rval_.to_host(s_);
    std::vector<double> cv = cval_.to_host(s_);
    sync();
    n_contacts_ = pin_i_[2];
    double val = 0.0;
    for (int r = 0; r < n_rows_; ++r) val += rv[r];
    for (int c = 0; c < std::min(pin_i_[3], cap_); ++c) val += cv[c]; // 0 off the active set
    *value = val;
    *active = n_contacts_;
    *candidates = ps_h_[0].n_candidates;
    const int nd = 6 * n_rows_;
    if (grad) {
        std::vector<double> g = rgrad_.to_host(s_);
        std::copy(g.begin(), g.begin() + nd, grad);
    }
    if (hess_dense) {
        std::vector<double> dg = rdiag_.to_host(s_);
        std::vector<int> cnt = ell_cnt_.to_host(s_), col = ell_col_.to_host(s_);
        std::vector<double> blk = ell_blk_.to_host(s_);
        std::fill(hess_dense, hess_dense + static_cast<size_t>(nd) * nd, 0.0);
        for (int r = 0; r < n_rows_; ++r) {
            for (int a = 0; a < 6; ++a)
                for (int c = 0; c < 6; ++c)
                    hess_dense[static_cast<size_t>(6 * r + a) * nd + 6 * r + c] = dg[36 * r + 6 * a + c];
            for (int t = 0; t < cnt[r]; ++t) {
                const int cc = col[r * ell_w_ + t];
                for (int a = 0; a < 6; ++a)
                    for (int c = 0; c < 6; ++c)
                        hess_dense[static_cast<size_t>(6 * r + a) * nd + 6 * cc + c] =
                            blk[(static_cast<size_t>(r) * ell_w_ + t) * 36 + 6 * a + c];
            }
        }
    }
}

NewtonResult Engine::newton_solve(const ObjectiveIn& in, double* q, int max_iters, double tol) {
    double dummy_v;
    int da, dc;
    // Reuse objective() for the instance/anchor setup (mode 0 evaluates once).
    objective(in, q, 0, &dummy_v, nullptr, nullptr, &da, &dc);
    inexact_ = false; // newton.cpp:7-71 as the reference solves it: every direction to pcg_tol_
    NewtonResult r;
    try {
        r = newton_batch(max_iters, tol);
    } catch (...) {
        inexact_ = true;
        throw;
    }
    inexact_ = true;
    std::vector<double> iq = iq_.to_host(s_);
    for (int i = 0; i < n_inst_; ++i) {
        const int b = h_ibody_[i];
        if (hs_.is_static[b]) continue;
        for (int c = 0; c < 6; ++c) q[6 * b + c] = iq[6 * i + c];
    }
    return r;
}

// ---------------------------------------------------------------------------
// frames
// ---------------------------------------------------------------------------
void Engine::set_state(const double* q, const double* qd) {
    q_.upload(q, 6 * static_cast<size_t>(hs_.nb), s_);
    qd_.upload(qd, 6 * static_cast<size_t>(hs_.nb), s_);
    sync();
}

void Engine::get_state(double* q, double* qd) {
    if (q) q_.download(q, 6 * static_cast<size_t>(hs_.nb), s_);
    if (qd) qd_.download(qd, 6 * static_cast<size_t>(hs_.nb), s_);
    sync();
}

std::vector<double> Engine::planes() const {
    std::vector<double> out;
    for (const PlaneH& p : planes_cur_) out.insert(out.end(), {p.px, p.py, p.nx, p.ny});
    return out;
}

void Engine::get_rho(double* rho) const {
    if (carry_on_device_) {
        const std::vector<double> c = rho_carry_d_.to_host(s_);
        std::copy(c.begin(), c.begin() + hs_.nb, rho);
        return;
    }
    std::copy(rho_carry_.begin(), rho_carry_.end(), rho);
}

std::vector<TraceRow> Engine::take_trace() {
    std::vector<TraceRow> t;
    t.swap(trace_);
    return t;
}

void Engine::run_frames(int n, FrameStats* stats) {
    for (int f = 0; f < n; ++f) {
        const NvtxRange range(W_ == 0 ? "dabd.frame_reference" : "dabd.frame_admm");
        const auto t0 = std::chrono::steady_clock::now();
        FrameStats st = W_ == 0 ? frame_reference() : frame_admm(static_cast<int>(frame_counter_));
        st.t_frame = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (W_ == 0) st.t_solve = st.t_frame; // the whole N=1 frame is one solve graph (sim.cpp:207-247)
        ++frame_counter_;
        if (stats) stats[f] = st;
    }
}

// ---------------------------------------------------------------------------
// N = 1 frame (sim.cpp:207-247), captured once into a CUDA graph
// ---------------------------------------------------------------------------
void Engine::enq_reference_frame(bool graph) {
    const SimParams& P = frame_params_;
    const double h = P.h;
    const size_t nq = 6 * static_cast<size_t>(hs_.nb);
    CUDA_CHECK(cudaMemcpyAsync(q_start_.get(), q_.get(), nq * sizeof(double),
                               cudaMemcpyDeviceToDevice, s_));
    CUDA_CHECK(cudaMemcpyAsync(qd_start_.get(), qd_.get(), nq * sizeof(double),
                               cudaMemcpyDeviceToDevice, s_));
    gather_iq(q_.get());
    launch_predict(ds_.view(), n_inst_, ibody_.get(), iq_.get(), qd_.get(), h, P.gravity[0],
                   P.gravity[1], nullptr, iqt_.get(), s_);
    const double tol = P.theta * h * P.scene_scale;
    auto admm_step = [&](int level) {
        launch_frame_ctrl(ctrl_.get(), 0, gate_.get(), P_, h, P.scene_scale, P.theta,
                          hs_.admm_max_iterations, trace_dev_.get(), trace_cap_, hd_, err_.get(),
                          ps_.get(), s_);
        CUDA_CHECK(cudaMemcpyAsync(iqbefore_.get(), iq_.get(), 6 * n_inst_ * sizeof(double),
                                   cudaMemcpyDeviceToDevice, s_));
        if (graph) {
            cap_newton(hs_.newton_cap, tol, level);
        } else {
            newton_batch(hs_.newton_cap, tol, false);
        }
        CUDA_CHECK(cudaMemsetAsync(gate_.get(), 0, P_ * sizeof(double), s_));
        launch_delta_inf(n_rows_, rinst_.get(), rpart_.get(), p0_, iq_.get(), iqbefore_.get(),
                         gate_.get(), s_);
        launch_frame_ctrl(ctrl_.get(), 1, gate_.get(), P_, h, P.scene_scale, P.theta,
                          hs_.admm_max_iterations, trace_dev_.get(), trace_cap_, hd_, err_.get(),
                          ps_.get(), s_);
    };
    if (graph) {
        hd_.admm = new_cond_handle();
        launch_frame_ctrl(ctrl_.get(), 2, gate_.get(), P_, h, P.scene_scale, P.theta,
                          hs_.admm_max_iterations, trace_dev_.get(), trace_cap_, hd_, err_.get(),
                          ps_.get(), s_);
        add_cond_node(hd_.admm, true, 0, [&] { admm_step(1); });
    } else {
        launch_frame_ctrl(ctrl_.get(), 2, gate_.get(), P_, h, P.scene_scale, P.theta,
                          hs_.admm_max_iterations, trace_dev_.get(), trace_cap_, hd_, err_.get(),
                          ps_.get(), s_);
        for (int k = 1; k <= hs_.admm_max_iterations + 1; ++k) {
            const FrameCtrl c = read_ctrl();
            if (c.ended || c.failed) break;
            admm_step(0);
        }
    }
    launch_commit(ds_.view(), n_inst_, ibody_.get(), ipart_.get(), ianc_.get(), nullptr, iq_.get(),
                  iznext_.get(), q_start_.get(), h, q_.get(), qd_.get(), s_);
}

void Engine::capture_reference_graph() {
    if (exec_) {
        cudaGraphExecDestroy(exec_);
        exec_ = nullptr;
    }
    KernelTimer::get().suspend(true);
    hd_ = CondHandles{};
    hd_.graph = 1;
    CUDA_CHECK(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal));
    try {
        const long long c0 = launch_counter().load();
        for (long long& v : nodes_inc_) v = 0;
        enq_reference_frame(true);
        nodes_total_ = launch_counter().load() - c0;
        launch_counter() -= nodes_total_; // captured, not executed
    } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(s_, &g);
        KernelTimer::get().suspend(false);
        hd_ = CondHandles{};
        throw;
    }
    cudaGraph_t g;
    CUDA_CHECK(cudaStreamEndCapture(s_, &g));
    KernelTimer::get().suspend(false);
    CUDA_CHECK(cudaGraphInstantiate(&exec_, g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
    hd_ = CondHandles{};
    graph_ok_ = true;
}

// kErrCapacity: the contact-candidate list; kErrEll: the BSR row width. The
// caller has restored the state the failed work started from.
bool Engine::grow_capacity(int code) {
    if (code == kErrCapacity) {
        cap_ *= 2;
        det_fmt_n_ = -1;
        prepare_solver();
    } else if (code == kErrEll) {
        ell_w_ *= 2;
        const size_t R = std::max(n_rows_, 1);
        ell_col_.resize(R * ell_w_);
        ell_blk_.resize(R * ell_w_ * 36);
        ++solver_epoch_;
    } else {
        return false;
    }
    graph_ok_ = false;
    return true;
}

// sim.cpp:186-249
FrameStats Engine::frame_reference() {
    frame_params_ = hs_.params;
    if (!ref_ready_) {
        std::vector<std::vector<int>> per(1);
        per[0].resize(hs_.nb);
        std::iota(per[0].begin(), per[0].end(), 0);
        build_instances(per, nullptr, true);
        std::vector<double> invk(std::max(n_inst_, 1), 1.0);
        iinvk_.upload(invk, s_);
        prepare_solver();
        ref_ready_ = true;
        graph_ok_ = false;
    }
    FrameStats st;
    st.h = frame_params_.h;
    const long long exact0 = exact_retries_, cap0 = capacity_retries_;
    bool exact_retry = false;
    SolverRestore restore(*this); // the exact-solve retry's PCG limits never outlive the frame
    const size_t nq = 6 * static_cast<size_t>(hs_.nb);
    auto restart = [&] { // back to the frame start
        err_.zero(s_);
        CUDA_CHECK(cudaMemcpyAsync(q_.get(), q_start_.get(), nq * sizeof(double), cudaMemcpyDeviceToDevice, s_));
        CUDA_CHECK(cudaMemcpyAsync(qd_.get(), qd_start_.get(), nq * sizeof(double), cudaMemcpyDeviceToDevice, s_));
    };
    for (int grows = 0;;) {
        FrameCtrl init{};
        init.frame = static_cast<double>(frame_counter_);
        ctrl_h_[0] = init;
        CUDA_CHECK(cudaMemcpyAsync(ctrl_.get(), ctrl_h_.get(), sizeof(FrameCtrl),
                                   cudaMemcpyHostToDevice, s_));
        int code = 0;
        if (use_graph_ && hs_.nb > 0) {
            if (!graph_ok_) capture_reference_graph();
            CUDA_CHECK(cudaGraphLaunch(exec_, s_));
            graph_replayed_ = true;
        } else {
            // the eager frame reads device errors mid-frame (check_err): the
            // recoverable ones take the same restart path as the graph's
            try {
                enq_reference_frame(false);
            } catch (const DeviceError& e) {
                if (e.code != kErrCapacity && e.code != kErrEll && e.code != kErrLineSearch) throw;
                code = e.code;
            }
        }
        if (code == 0) {
            CUDA_CHECK(cudaMemcpyAsync(ctrl_h_.get(), ctrl_.get(), sizeof(FrameCtrl),
                                       cudaMemcpyDeviceToHost, s_));
            CUDA_CHECK(cudaMemcpyAsync(pin_i_.get(), err_.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
            CUDA_CHECK(cudaMemcpyAsync(lstate_h_.get(), lstate_.get(), sizeof(ListState),
                                       cudaMemcpyDeviceToHost, s_));
            CUDA_CHECK(cudaStreamSynchronize(s_));
            code = pin_i_[0];
        }
        if ((code == kErrCapacity || code == kErrEll) && grows < kMaxGrows) {
            // grow the capacity that overflowed, restore the frame start and
            // redo it; past the budget check_err below reports the overflow
            restart();
            grow_capacity(code);
            ++grows;
            ++capacity_retries_;
            continue;
        }
        if (code == kErrLineSearch && !exact_retry) {
            // newton.cpp:56-58's collapse after an iterative solve: redo the
            // frame from its start with the PCG at the exact-solve limit (see
            // frame_admm) before reporting the reference's error
            restart();
            exact_retry = true;
            set_solver(1e-14, std::max(pcg_max_, 50000));
            ++exact_retries_;
            continue;
        }
        check_err("frame_reference"); // any other device error, or an overflow past the budget
        break;
    }
    const FrameCtrl& c = ctrl_h_[0];
    if (graph_replayed_) { // kernels the replay executed: nodes per body x body executions
        const long long rebuilds = lstate_h_[0].n_rebuilds - rebuilds_seen_;
        count_launch(rebuilds * rebuild_nodes_ + nodes_total_ - nodes_inc_[0] +
                     static_cast<long long>(c.exec_admm) * (nodes_inc_[0] - nodes_inc_[1]) +
                     static_cast<long long>(c.exec_newton) * (nodes_inc_[1] - nodes_inc_[2]) +
                     static_cast<long long>(c.exec_step) * (nodes_inc_[2] - nodes_inc_[3]) +
                     static_cast<long long>(c.exec_ls) * nodes_inc_[3]);
        graph_replayed_ = false;
    }
    rebuilds_seen_ = lstate_h_[0].n_rebuilds;
    if (c.failed || !c.ended) throw Error("run_reference: Newton stepping failed to settle");
    st.exact_retries = static_cast<int>(exact_retries_ - exact0);
    st.capacity_retries = static_cast<int>(capacity_retries_ - cap0);
    st.admm_iterations = c.admm_iterations;
    st.newton_iterations = c.newton_total;
    st.line_search_steps = c.ls_total;
    st.pcg_iterations = c.pcg_total;
    const int nt = std::min(c.trace_n, trace_cap_);
    if (nt > 0) {
        std::vector<double> rows(8 * static_cast<size_t>(nt));
        CUDA_CHECK(cudaMemcpy(rows.data(), trace_dev_.get(), rows.size() * sizeof(double),
                              cudaMemcpyDeviceToHost));
        for (int i = 0; i < nt; ++i)
            trace_.push_back({rows[8 * i], rows[8 * i + 1], rows[8 * i + 2], rows[8 * i + 3],
                              rows[8 * i + 4], rows[8 * i + 5], rows[8 * i + 6], rows[8 * i + 7]});
    }
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 2, &lstate_.get()->n_act, sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 3, det_.d_count(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    sync();
    st.max_contacts = pin_i_[2];
    st.max_candidates = pin_i_[3];
    st.committed = 1;
    return st;
}

// ---------------------------------------------------------------------------
// Multi-partition ADMM attempt as one captured graph (runtime.cpp:316-476 and
// the controller round trip 572-638, for the partitions of this context):
//
//   init; WHILE(sigma == 0) {
//     head                       (IF(gate) = k > 1; TOIs <- 2, r, s <- 0)
//     IF(gate)  { consensus, merge targets, merge-gate broad phase + CCD,
//                 decide: stop test, trace row, sigma, IF(solve), WHILE }
//     IF(solve) { adapt rho + z (k > 1), q_before, Newton solve (nested
//                 conditional graph), delta_inf, tail: dq, totals, costs, k++ }
//   }
//
// Instance sets and capacities change per attempt, so the graph is captured
// per attempt (an in-place update when the topology is unchanged) and read
// back once. Recoverable device errors (contact-list, BSR-width or gate
// capacity; the line-search collapse of an iterative solve) redo the attempt
// from its start, which is deterministic.
int Engine::admm_attempt_device(int frame, int attempt, double h, double tol, int I, int ns,
                                FrameStats& st, std::vector<double>& cost, int& grows, bool& exact) {
    const SimParams& P = frame_params_;
    AdmmProfile& prof = admm_prof();
    prof.mark(0, s_);
    if (gate_cap_ == 0) gate_cap_ = 64 * std::max(I, 1);
    det_gate_.ensure(I, ds_.max_verts, gate_cap_);
    admm_dq_.resize(std::max(P_, 1));
    admm_dqnew_.resize(std::max(P_, 1));
    admm_cost_.resize(std::max(P_, 1));
    admm_cost_h_.resize(std::max(P_, 1));
    FrameCtrl init{};
    init.frame = static_cast<double>(frame);
    init.attempt = static_cast<double>(attempt);
    init.can_halve = tsc_.can_halve() ? 1 : 0;
    ctrl_h_[0] = init;
    CUDA_CHECK(cudaMemcpyAsync(ctrl_.get(), ctrl_h_.get(), sizeof(FrameCtrl), cudaMemcpyHostToDevice, s_));
    err_.zero(s_);

    AdmmCtrlArgs a;
    a.c = ctrl_.get();
    a.gate = gate_.get();
    a.rloc = rloc_.get();
    a.sloc = sloc_.get();
    a.dq = admm_dq_.get();
    a.dq_new = admm_dqnew_.get();
    a.cost = admm_cost_.get();
    a.ps = ps_.get();
    a.gate_count = det_gate_.d_count();
    a.err = err_.get();
    a.trace = trace_dev_.get();
    a.trace_cap = trace_cap_;
    a.P = P_;
    a.K = hs_.admm_max_iterations;
    a.h = h;
    a.l = P.scene_scale;
    a.theta = P.theta;
    const bool dist = distributed_;
    if (dist) {
        if (!p2p_ || !fan_ok_) throw Error("admm: the device loop of a distributed frame needs the peer-memory paths");
        if (static_cast<size_t>(std::max(n_halo_lo_, n_halo_hi_)) > pub_cap_)
            throw Error("comm: peer halo capacity exceeded");
        a.fan_rec = fan_view_.local_rec;
        a.fan_world = comm_.world;
        a.fan_stride = kFanStride;
    }

    KernelTimer::get().suspend(true);
    hd_ = CondHandles{};
    hd_.graph = 1;
    for (long long& v : nodes_inc_) v = 0;
    const long long c0 = launch_counter().load();
    long long total = 0;
    CUDA_CHECK(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal));
    try {
        hd_.admm = new_cond_handle();
        a.hd = hd_;
        launch_admm_ctrl(a, kAdmmInit, s_);
        add_cond_node(hd_.admm, true, 0, [&] {
            hd_.gate = new_cond_handle();
            hd_.solve = new_cond_handle();
            a.hd = hd_;
            launch_admm_ctrl(a, kAdmmHead, s_);
            add_cond_node(hd_.gate, false, 1, [&] {
                if (dist) {
                    // split-body packets into this iteration's [side][parity]
                    // publish regions, the ordering barrier, then k_consensus
                    // reads the neighbours' packets in place over peer memory
                    const size_t reg = static_cast<size_t>(kHaloStride) * pub_cap_;
                    launch_pack_halo_par(n_halo_lo_, halo_inst_.get(), iq_.get(), iu_.get(), irho_.get(), pub_.get(),
                                         ctrl_.get(), 0, reg, s_);
                    launch_pack_halo_par(n_halo_hi_, halo_inst_.get() + n_halo_lo_, iq_.get(), iu_.get(), irho_.get(),
                                         pub_.get(), ctrl_.get(), 1, reg, s_);
                    launch_fan_post(fan_view_, nullptr, 0, s_);
                    launch_fan_wait(fan_view_, s_);
                    launch_consensus_par(ns, shared_inst_.get(), ipart_.get(), p0_, iq_.get(), iu_.get(), irho_.get(),
                                         iz_.get(), peer_lo_, peer_hi_, n_halo_lo_, iznext_.get(), rb_.get(),
                                         sb_.get(), rloc_.get(), sloc_.get(), err_.get(), ctrl_.get(), reg, s_);
                } else {
                    launch_consensus(ns, shared_inst_.get(), ipart_.get(), p0_, iq_.get(), iu_.get(),
                                     irho_.get(), iz_.get(), nullptr, nullptr, 0, iznext_.get(), rb_.get(),
                                     sb_.get(), rloc_.get(), sloc_.get(), err_.get(), s_);
                }
                // merge gate per partition (consensus.cpp:66-75): fixed-capacity
                // broad phase, CCD over its device count
                launch_merged(I, ianc_.get(), iq_.get(), iznext_.get(), iqtry_.get(), s_);
                det_gate_.enqueue(ds_.view(), iview(iq_.get(), iqtry_.get()), stat_.get(),
                                  n_stat_, true, 0.0, err_.get(), s_);
                launch_ccd(view(), det_gate_.keys(), det_gate_.cap(), det_gate_.d_count(), det_gate_.fmt(),
                           det_gate_.boxes(), iq_.get(), iqtry_.get(), 2, gate_.get(), s_);
                if (dist) { // controller fan-in (runtime.cpp:586-601) through peer memory
                    launch_fan_record(P_, admm_dq_.get(), rloc_.get(), sloc_.get(), gate_.get(), err_.get(),
                                      fan_rec_local_.get(), s_);
                    launch_fan_post(fan_view_, fan_rec_local_.get(), 2 + 4 * P_, s_);
                    launch_fan_wait(fan_view_, s_);
                }
                launch_admm_ctrl(a, kAdmmDecide, s_);
            });
            add_cond_node(hd_.solve, false, 2, [&] {
                launch_adapt(I, ianc_.get(), irho_.get(), irho0_.get(), rb_.get(), sb_.get(), hs_.adapt,
                             iz_.get(), iznext_.get(), s_, ctrl_.get());
                if (I) CUDA_CHECK(cudaMemcpyAsync(iqbefore_.get(), iq_.get(), 6 * I * sizeof(double),
                                                  cudaMemcpyDeviceToDevice, s_));
                cap_newton(hs_.newton_cap, tol, 3);
                CUDA_CHECK(cudaMemsetAsync(admm_dqnew_.get(), 0, P_ * sizeof(double), s_));
                launch_delta_inf(n_rows_, rinst_.get(), rpart_.get(), p0_, iq_.get(), iqbefore_.get(),
                                 admm_dqnew_.get(), s_);
                launch_admm_ctrl(a, kAdmmTail, s_);
            });
        });
        total = launch_counter().load() - c0;
        launch_counter() -= total; // captured, not executed
    } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(s_, &g);
        if (g) cudaGraphDestroy(g);
        KernelTimer::get().suspend(false);
        hd_ = CondHandles{};
        throw;
    }
    cudaGraph_t g;
    CUDA_CHECK(cudaStreamEndCapture(s_, &g));
    KernelTimer::get().suspend(false);
    hd_ = CondHandles{};
    bool updated = false;
    if (admm_exec_) {
        cudaGraphExecUpdateResultInfo info;
        updated = cudaGraphExecUpdate(admm_exec_, g, &info) == cudaSuccess;
        if (!updated) {
            cudaGetLastError();
            cudaGraphExecDestroy(admm_exec_);
            admm_exec_ = nullptr;
        }
    }
    if (!updated) CUDA_CHECK(cudaGraphInstantiate(&admm_exec_, g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
    const long long inc[6] = {nodes_inc_[0], nodes_inc_[1], nodes_inc_[2], nodes_inc_[3], nodes_inc_[4],
                              nodes_inc_[5]};
    prof.mark(1, s_);

    const NvtxRange range("dabd.solve.admm_attempt");
    const auto t0 = std::chrono::steady_clock::now();
    CUDA_CHECK(cudaGraphLaunch(admm_exec_, s_));
    CUDA_CHECK(cudaMemcpyAsync(ctrl_h_.get(), ctrl_.get(), sizeof(FrameCtrl), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get(), err_.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 9, det_gate_.d_count(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(lstate_h_.get(), lstate_.get(), sizeof(ListState), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 3, det_.d_count(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(admm_cost_h_.get(), admm_cost_.get(), P_ * sizeof(double), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
    st.t_solve += seconds_since(t0);
    prof.mark(3, s_);
    const FrameCtrl c = ctrl_h_[0];
    // kernels the replay executed: per conditional body its own nodes x its
    // executions (levels: 0 ADMM body, 1 gate, 2 solve, 3 Newton, 4 step, 5 ls)
    const long long rebuilds = lstate_h_[0].n_rebuilds - rebuilds_seen_;
    rebuilds_seen_ = lstate_h_[0].n_rebuilds;
    count_launch(rebuilds * rebuild_nodes_ + (total - inc[0]) +
                 static_cast<long long>(c.exec_admm) * (inc[0] - inc[1] - inc[2]) +
                 static_cast<long long>(c.exec_gate) * inc[1] +
                 static_cast<long long>(c.exec_solve) * (inc[2] - inc[3]) +
                 static_cast<long long>(c.exec_newton) * (inc[3] - inc[4]) +
                 static_cast<long long>(c.exec_step) * (inc[4] - inc[5]) +
                 static_cast<long long>(c.exec_ls) * inc[5]);
    int code = pin_i_[0];
    if (dist) {
        // every rank ran the same rounds; agree on the outcome: a recoverable
        // error anywhere redoes the attempt everywhere (each rank grows what
        // overflowed locally; a line-search collapse anywhere arms the exact
        // solve everywhere, as one context would), anything else fails all
        const std::vector<double> all = allgather_host({static_cast<double>(code)});
        const size_t stride = all.size() / comm_.world;
        bool any = false, fatal = false, ls = false;
        for (int r = 0; r < comm_.world; ++r) {
            const int cr = static_cast<int>(all[stride * r]);
            any = any || cr != 0;
            ls = ls || cr == kErrLineSearch;
            fatal = fatal || (cr != 0 && cr != kErrCapacity && cr != kErrEll && cr != kErrLineSearch);
        }
        if (any) {
            err_.zero(s_);
            if (fatal || grows >= kMaxGrows || (ls && exact)) {
                sync();
                if (code != 0) throw DeviceError(std::string(err_text(code)) + " [admm frame]", code);
                throw Error("admm: a peer rank failed");
            }
            const int gate_count = std::max(pin_i_[9], c.gate_max);
            if (code == kErrCapacity && gate_count > gate_cap_) gate_cap_ = 2 * gate_count;
            else if (code == kErrCapacity || code == kErrEll) grow_capacity(code);
            if (ls && !exact) {
                set_solver(1e-14, std::max(pcg_max_, 50000));
                exact = true;
                ++exact_retries_;
            }
            ++grows;
            ++capacity_retries_;
            return 0;
        }
    }
    if (code != 0) {
        err_.zero(s_);
        const int gate_count = std::max(pin_i_[9], c.gate_max); // the largest gate of the attempt
        if (code == kErrCapacity && gate_count > gate_cap_ && grows < kMaxGrows) {
            gate_cap_ = 2 * gate_count; // merge-gate candidates overflowed its fixed capacity
            ++grows;
            ++capacity_retries_;
            return 0;
        }
        if ((code == kErrCapacity || code == kErrEll) && grows < kMaxGrows) {
            grow_capacity(code);
            ++grows;
            ++capacity_retries_;
            return 0;
        }
        if (code == kErrLineSearch && !exact) {
            set_solver(1e-14, std::max(pcg_max_, 50000));
            exact = true;
            ++exact_retries_;
            return 0;
        }
        sync();
        throw DeviceError(std::string(err_text(code)) + " [admm frame]", code);
    }
    // the gate's sort cost follows its capacity: shrink it (with hysteresis)
    // towards twice the most candidates an iteration found
    if (4 * c.gate_max < gate_cap_ && gate_cap_ > 8192) gate_cap_ = std::max(8192, 2 * c.gate_max);
    const int nt = std::min(c.trace_n, trace_cap_);
    if (nt > 0) {
        std::vector<double> rows(8 * static_cast<size_t>(nt));
        CUDA_CHECK(cudaMemcpy(rows.data(), trace_dev_.get(), rows.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int i = 0; i < nt; ++i)
            trace_.push_back({rows[8 * i], rows[8 * i + 1], rows[8 * i + 2], rows[8 * i + 3], rows[8 * i + 4],
                              rows[8 * i + 5], rows[8 * i + 6], rows[8 * i + 7]});
    }
    st.newton_iterations += c.newton_total;
    st.line_search_steps += c.ls_total;
    st.pcg_iterations += c.pcg_total;
    st.max_contacts = std::max(st.max_contacts, lstate_h_[0].n_act);
    st.max_candidates = std::max(st.max_candidates, pin_i_[3]);
    for (int p = 0; p < P_; ++p) cost[p] += admm_cost_h_[p];
    if (c.sigma == 1) {
        st.admm_iterations = c.admm_iterations;
        return 1;
    }
    if (c.sigma == 2) return 2;
    if (c.sigma == 3) throw Error("frame failed: halving budget exhausted with a blocked merge");
    throw Error("controller: frame ended without a decision");
}

// runtime.cpp:110-694 on replicated global state with every partition of
// this context solved in the same batched kernels.
FrameStats Engine::frame_admm(int frame) {
    AdmmProfile& prof = admm_prof();
    prof.mark(6, s_);
    const int nb = hs_.nb;
    // PD balancer step on the previous committed frame's partition costs;
    // the shifted planes take effect in this frame's partitioning
    // (runtime.cpp:543-552, applied by every worker at runtime.cpp:97-103)
    if (hs_.balance.enabled && have_costs_ && W_ > 1) balancer_.update(part_cost_, planes_cur_, w_last_);
    const std::vector<PlaneH>& planes = planes_cur_;
    std::vector<double> hplanes;
    for (const PlaneH& p : planes) hplanes.insert(hplanes.end(), {p.px, p.py, p.nx, p.ny});
    DBuf<double> dplanes;
    dplanes.resize(std::max<size_t>(hplanes.size(), 4));
    if (!hplanes.empty()) dplanes.upload(hplanes, s_);
    const uint32_t everyone = W_ == 32 ? 0xffffffffu : ((1u << W_) - 1u);
    int attempt = 0;
    FrameStats st;
    const long long exact0 = exact_retries_, cap0 = capacity_retries_;
    SolverRestore frame_restore(*this); // an exact-solve retry's PCG limits end with the frame
    int dev_grows = 0;
    bool dev_exact = false;
    while (true) {
        st.attempts = attempt + 1;
        const double h = tsc_.h();
        st.h = h;
        frame_params_ = hs_.params;
        frame_params_.h = h;
        const SimParams& P = frame_params_;
        std::vector<double> cost(P_, 0.0); // this attempt's per-partition compute cost
        // the whole attempt on the device: instance sets, constants and the
        // ADMM loop (no force split: its per-frame host table stays host-side)
        const bool split_active =
            !hs_.force_split.empty() && (hs_.force_split_frames < 0 || frame < hs_.force_split_frames);
        const bool device_attempt = admm_device_ && use_graph_ && !distributed_ && !split_active;
        if (device_attempt) {
            if (!carry_on_device_) {
                rho_carry_d_.resize(std::max(nb, 1));
                rho_carry_d_.upload(rho_carry_, s_);
                carry_on_device_ = true;
            }
            gate_.resize(std::max(P_, 2));
            gate_.zero(s_);
            launch_vmax(ds_.view(), qd_.get(), gate_.get(), s_);
            masks_d_.resize(std::max(nb, 1));
            launch_masks_w(ds_.view(), q_.get(), dplanes.get(), W_ - 1, gate_.get(), h, hs_.w_min, gate_.get() + 1,
                           everyone, masks_d_.get(), err_.get(), s_);
            prof.mark(7, s_);
            double w = 0.0;
            const int ns = build_instances_device(masks_d_.get(), &w); // synchronises once
            w_last_ = w;
            check_err("frame: holder masks");
            prof.mark(8, s_);
            prepare_solver();
            prof.mark(9, s_);
            const int I = n_inst_;
            const size_t nq = 6 * static_cast<size_t>(nb);
            if (nq) CUDA_CHECK(cudaMemcpyAsync(q_start_.get(), q_.get(), nq * sizeof(double), cudaMemcpyDeviceToDevice, s_));
            gather_iq(q_.get());
            launch_predict(ds_.view(), I, ibody_.get(), iq_.get(), qd_.get(), h, P.gravity[0], P.gravity[1], nullptr,
                           iqt_.get(), s_);
            if (I) CUDA_CHECK(cudaMemcpyAsync(iz_.get(), iqt_.get(), 6 * I * sizeof(double), cudaMemcpyDeviceToDevice, s_));
            const double tol = P.theta * h * P.scene_scale;
            const int r = n_rows_ > 0 ? admm_attempt_device(frame, attempt, h, tol, I, ns, st, cost, dev_grows, dev_exact)
                                      : -1;
            if (r == 0) continue; // a capacity grew / the exact-solve retry is armed: redo the attempt
            if (r == 2) {         // blocked merge at K: h halves (runtime.cpp:603-642)
                tsc_.on_frame_failed();
                ++attempt;
                continue;
            }
            if (r == 1) {
                // rho carry + commit (runtime.cpp:481-506), on the device
                launch_rho_carry(I, nb, ibody_.get(), ianc_.get(), irho_.get(), rho_carry_d_.get(), s_);
                launch_commit(ds_.view(), I, ibody_.get(), ipart_.get(), ianc_.get(), bmask_.get(), iq_.get(),
                              iznext_.get(), q_start_.get(), h, q_.get(), qd_.get(), s_);
                if (hs_.balance.enabled && W_ > 1) {
                    for (int p = 0; p < P_; ++p) part_cost_[p0_ + p] = cost[p];
                    have_costs_ = true;
                }
                sync();
                prof.mark(5, s_);
                tsc_.on_frame_committed();
                st.exact_retries = static_cast<int>(exact_retries_ - exact0);
                st.capacity_retries = static_cast<int>(capacity_retries_ - cap0);
                st.committed = 1;
                return st;
            }
            // no dynamic instance: nothing to solve; fall through to the host path
        }
        if (carry_on_device_) { // the host path owns the carry from here
            rho_carry_ = rho_carry_d_.to_host(s_);
            rho_carry_.resize(nb);
            carry_on_device_ = false;
        }
        // overlap width from the current velocities (runtime.cpp:556-560)
        gate_.zero(s_);
        launch_vmax(ds_.view(), qd_.get(), gate_.get(), s_);
        const double v_max = gate_.to_host(s_)[0];
        const double w = std::max(2.0 * v_max * h, hs_.w_min);
        w_last_ = w;
        // holder masks (partition.cpp:36-67)
        DBuf<uint32_t> dm;
        dm.resize(std::max(nb, 1));
        launch_masks(ds_.view(), q_.get(), dplanes.get(), W_ - 1, w, everyone, dm.get(), err_.get(), s_);
        std::vector<uint32_t> mask = dm.to_host(s_);
        check_err("frame: holder masks");
        prof.mark(7, s_);
        mask.resize(nb);
        // local sets per partition (runtime.cpp:212-236)
        std::vector<std::vector<int>> per(P_);
        for (int b = 0; b < nb; ++b)
            for (int p = 0; p < P_; ++p)
                if (mask[b] & (1u << (p0_ + p))) per[p].push_back(b);
        prof.mark(0, s_);
        build_instances(per, mask.data(), false);
        prof.mark(8, s_);
        prepare_solver();
        prof.mark(9, s_);
        const int I = n_inst_;
        std::vector<double> invk(std::max(I, 1)), rho(std::max(I, 1), 0.0), rho0(std::max(I, 1), 0.0),
            fs(2 * std::max(I, 1), 0.0);
        std::vector<int> anc(std::max(I, 1), 0);
        bool any_split = false;
        h_shared_inst_.clear();
        std::vector<int> first_inst(nb, -1);
        for (int i = 0; i < I; ++i) {
            const int b = h_ibody_[i];
            const int kb = std::popcount(mask[b]);
            invk[i] = 1.0 / kb;
            if (hs_.is_static[b] || kb < 2) continue;
            anc[i] = 1;
            rho0[i] = hs_.adapt.beta * hs_.mass[b]; // init_rho (consensus.cpp:38-42)
            rho[i] = std::isnan(rho_carry_[b]) ? rho0[i] : rho_carry_[b];
            const auto it = hs_.force_split.find(b);
            const bool active = hs_.force_split_frames < 0 || frame < hs_.force_split_frames;
            if (it != hs_.force_split.end() && active) {
                const int lowest = std::countr_zero(mask[b]);
                const double sign = h_ipart_[i] == lowest ? 1.0 : -1.0;
                fs[2 * i] = sign * it->second.first;
                fs[2 * i + 1] = sign * it->second.second;
                any_split = true;
            }
            if (first_inst[b] < 0) {
                first_inst[b] = i;
            } else {
                h_shared_inst_.push_back(first_inst[b]);
                h_shared_inst_.push_back(i);
            }
        }
        // replicas whose partner partition lives on a neighbouring rank
        // (partition-per-GPU runs): lo side = shared with p0-1, hi side =
        // shared with p1; both lists in instance (= body) order, which the
        // neighbour derives identically from the same masks.
        h_halo_inst_.clear();
        std::vector<int> hi_list;
        for (int i = 0; i < I; ++i) {
            if (!anc[i]) continue;
            const int b = h_ibody_[i];
            const int lo = std::countr_zero(mask[b]), hi = 31 - std::countl_zero(mask[b]);
            if (lo < p0_) h_halo_inst_.push_back(i);
            else if (hi >= p1_) hi_list.push_back(i);
        }
        n_halo_lo_ = static_cast<int>(h_halo_inst_.size());
        n_halo_hi_ = static_cast<int>(hi_list.size());
        if ((n_halo_lo_ || n_halo_hi_) && !distributed_)
            throw Error("ctx: the partition range needs dabd_gpu_ctx_set_comm (neighbour partitions are remote)");
        for (int j = 0; j < n_halo_lo_; ++j) { // remote replica first (lower partition)
            h_shared_inst_.push_back(-1 - j);
            h_shared_inst_.push_back(h_halo_inst_[j]);
        }
        for (int j = 0; j < n_halo_hi_; ++j) {
            h_shared_inst_.push_back(hi_list[j]);
            h_shared_inst_.push_back(-1 - (n_halo_lo_ + j));
        }
        h_halo_inst_.insert(h_halo_inst_.end(), hi_list.begin(), hi_list.end());
        const int ns = static_cast<int>(h_shared_inst_.size() / 2);
        if (distributed_) {
            const size_t nh = std::max<size_t>(h_halo_inst_.size(), 1);
            halo_inst_.upload(h_halo_inst_.empty() ? std::vector<int>{0} : h_halo_inst_, s_);
            hsend_.resize(kHaloStride * nh);
            hrecv_.resize(kHaloStride * nh);
        }
        iinvk_.upload(invk.data(), std::max(I, 1), s_);
        irho_.upload(rho.data(), std::max(I, 1), s_);
        irho0_.upload(rho0.data(), std::max(I, 1), s_);
        ianc_.upload(anc.data(), std::max(I, 1), s_);
        shared_inst_.upload(h_shared_inst_.empty() ? std::vector<int>{0, 0} : h_shared_inst_, s_);
        if (any_split) ifs_.upload(fs, s_);
        const size_t nq = 6 * static_cast<size_t>(nb);
        if (nq) CUDA_CHECK(cudaMemcpyAsync(q_start_.get(), q_.get(), nq * sizeof(double),
                                           cudaMemcpyDeviceToDevice, s_));
        gather_iq(q_.get());
        launch_predict(ds_.view(), I, ibody_.get(), iq_.get(), qd_.get(), h, P.gravity[0],
                       P.gravity[1], any_split ? ifs_.get() : nullptr, iqt_.get(), s_);
        // warm start z = q_tilde, u = 0 (runtime.cpp:267-277)
        if (I) CUDA_CHECK(cudaMemcpyAsync(iz_.get(), iqt_.get(), 6 * I * sizeof(double),
                                          cudaMemcpyDeviceToDevice, s_));
        iu_.zero(s_);
        const double tol = P.theta * h * P.scene_scale;
        std::vector<double> dq(P_, 0.0);
        bool ended = false, retry = false;
        prof.mark(0, s_);
        // A local failure on one rank must not leave its peers blocked in a
        // collective: it is carried to the next agreement point instead.
        std::string fail;
        // partition-per-GPU: the host built the sets (remote replicas, halo
        // lists); the k-loop itself runs on the device when every rank mapped
        // the peer-memory paths (the same decision on every rank)
        const bool device_loop = distributed_ && p2p_ && fan_ok_ && admm_device_ && use_graph_;
        if (device_loop) {
            const int r = admm_attempt_device(frame, attempt, h, tol, I, ns, st, cost, dev_grows, dev_exact);
            if (r == 0) continue; // recoverable error somewhere: redo the attempt on every rank
            if (r == 2) {
                tsc_.on_frame_failed();
                retry = true;
            } else {
                ended = true;
            }
        }
        for (int k = 1; !device_loop && k <= hs_.admm_max_iterations; ++k) {
            if (k > 1) {
                std::vector<double> earliest(P_, 2.0), rl(P_, 0.0), sl(P_, 0.0);
                try {
                    if (!fail.empty()) throw Error(fail);
                    const NvtxRange range("dabd.coll");
                    const auto tc = std::chrono::steady_clock::now();
                    rloc_.zero(s_);
                    sloc_.zero(s_);
                    if (distributed_) {
                        const auto ts = std::chrono::steady_clock::now();
                        exchange_halo();
                        st.t_sync += seconds_since(ts);
                    } else {
                        remote_lo_ = remote_hi_ = nullptr;
                    }
                    launch_consensus(ns, shared_inst_.get(), ipart_.get(), p0_, iq_.get(),
                                     iu_.get(), irho_.get(), iz_.get(), remote_lo_, remote_hi_,
                                     n_halo_lo_, iznext_.get(),
                                     rb_.get(), sb_.get(), rloc_.get(), sloc_.get(), err_.get(), s_);
                    // merge CCD gate per partition (consensus.cpp:66-75): a
                    // fixed-capacity broad phase and the CCD over its device
                    // count, then ONE readback of (earliest TOI, r, s, error)
                    launch_merged(I, ianc_.get(), iq_.get(), iznext_.get(), iqtry_.get(), s_);
                    if (gate_cap_ == 0) gate_cap_ = 64 * std::max(I, 1);
                    det_gate_.ensure(I, ds_.max_verts, gate_cap_);
                    det_gate_.enqueue(ds_.view(), iview(iq_.get(), iqtry_.get()), stat_.get(),
                                      n_stat_, true, 0.0, err_.get(), s_);
                    for (int p = 0; p < P_; ++p) pin_d_[128 + p] = 2.0;
                    CUDA_CHECK(cudaMemcpyAsync(gate_.get(), pin_d_.get() + 128, P_ * sizeof(double),
                                               cudaMemcpyHostToDevice, s_));
                    launch_ccd(view(), det_gate_.keys(), det_gate_.cap(), det_gate_.d_count(),
                               det_gate_.fmt(), det_gate_.boxes(), iq_.get(), iqtry_.get(), 2,
                               gate_.get(), s_);
                    CUDA_CHECK(cudaMemcpyAsync(pin_d_.get(), gate_.get(), P_ * sizeof(double),
                                               cudaMemcpyDeviceToHost, s_));
                    CUDA_CHECK(cudaMemcpyAsync(pin_d_.get() + 32, rloc_.get(), P_ * sizeof(double),
                                               cudaMemcpyDeviceToHost, s_));
                    CUDA_CHECK(cudaMemcpyAsync(pin_d_.get() + 64, sloc_.get(), P_ * sizeof(double),
                                               cudaMemcpyDeviceToHost, s_));
                    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 8, err_.get(), sizeof(int),
                                               cudaMemcpyDeviceToHost, s_));
                    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 9, det_gate_.d_count(), sizeof(int),
                                               cudaMemcpyDeviceToHost, s_));
                    sync();
                    // the gate's sort cost follows its capacity: shrink it (with
                    // hysteresis) towards twice the candidates actually found
                    if (pin_i_[8] == 0 && 4 * pin_i_[9] < gate_cap_ && gate_cap_ > 8192)
                        gate_cap_ = std::max(8192, 2 * pin_i_[9]);
                    if (pin_i_[8] == kErrCapacity) { // grow and redo this gate with the counted build
                        err_.zero(s_);
                        const int nc = det_gate_.build(ds_.view(), iview(iq_.get(), iqtry_.get()),
                                                       stat_.get(), n_stat_,
                                                       true, 0.0, ds_.max_verts, s_);
                        gate_cap_ = det_gate_.cap();
                        gate_.upload(earliest, s_);
                        launch_ccd(view(), det_gate_.keys(), nc, nullptr, det_gate_.fmt(),
                                   det_gate_.boxes(), iq_.get(), iqtry_.get(), 2, gate_.get(), s_);
                        earliest = gate_.to_host(s_);
                        check_err("admm: consensus/gate");
                    } else if (pin_i_[8] != 0) {
                        const int code = pin_i_[8];
                        err_.zero(s_);
                        sync();
                        throw Error(std::string(err_text(code)) + " [admm: consensus/gate]");
                    } else {
                        for (int p = 0; p < P_; ++p) earliest[p] = pin_d_[p];
                    }
                    for (int p = 0; p < P_; ++p) {
                        rl[p] = pin_d_[32 + p];
                        sl[p] = pin_d_[64 + p];
                    }
                    st.t_coll += seconds_since(tc); // consensus + merge gate (runtime.cpp:399-402)
                    prof.mark(1, s_);
                } catch (const Error& e) {
                    if (!distributed_) throw;
                    if (fail.empty()) fail = e.what();
                }
                if (distributed_) {
                    // controller fan-in (runtime.cpp:586-619): every rank
                    // sees every partition's (dq, r, s, earliest TOI).
                    std::vector<double> rec = {static_cast<double>(P_), fail.empty() ? 0.0 : 1.0};
                    for (int p = 0; p < P_; ++p) rec.insert(rec.end(), {dq[p], rl[p], sl[p], earliest[p]});
                    const NvtxRange range("dabd.sync.fanin");
                    const auto ts = std::chrono::steady_clock::now();
                    const std::vector<double> all = allgather_host(rec);
                    st.t_sync += seconds_since(ts); // controller fan-in (runtime.cpp:586-601)
                    const size_t stride = all.size() / comm_.world;
                    dq.clear(), rl.clear(), sl.clear(), earliest.clear();
                    bool any_fail = false;
                    for (int r = 0; r < comm_.world; ++r) {
                        const double* x = all.data() + stride * r;
                        any_fail = any_fail || x[1] != 0.0;
                        for (int p = 0; p < static_cast<int>(x[0]); ++p) {
                            dq.push_back(x[2 + 4 * p]);
                            rl.push_back(x[3 + 4 * p]);
                            sl.push_back(x[4 + 4 * p]);
                            earliest.push_back(x[5 + 4 * p]);
                        }
                    }
                    if (any_fail)
                        throw Error(fail.empty() ? std::string("admm: a peer rank failed") : fail);
                }
                TraceRow row{static_cast<double>(frame), static_cast<double>(attempt),
                             static_cast<double>(k), 0.0, 0.0, 0.0, 1.0, 0.0};
                const int np = static_cast<int>(earliest.size());
                std::vector<double> tois(np);
                for (int p = 0; p < np; ++p) {
                    tois[p] = earliest[p] > 1.0 ? 1.0 : std::min(1.0, 0.9 * earliest[p]);
                    row.dq = std::max(row.dq, dq[p]);
                    row.r = std::max(row.r, rl[p]);
                    row.s = std::max(row.s, sl[p]);
                    row.toi = std::min(row.toi, tois[p]);
                }
                const bool end =
                    check_stopping(row.dq, row.r, row.s, tois, h, P.scene_scale, P.theta);
                if (end) row.sigma = 1;
                else if (k == hs_.admm_max_iterations) row.sigma = tsc_.can_halve() ? 2 : 3;
                trace_.push_back(row);
                if (row.sigma == 1) {
                    st.admm_iterations = k;
                    ended = true;
                    break;
                }
                if (row.sigma == 3) throw Error("frame failed: halving budget exhausted with a blocked merge");
                if (row.sigma == 2) {
                    tsc_.on_frame_failed();
                    retry = true;
                    break;
                }
                launch_adapt(I, ianc_.get(), irho_.get(), irho0_.get(), rb_.get(), sb_.get(),
                             hs_.adapt, iz_.get(), iznext_.get(), s_);
                prof.mark(2, s_);
            }
            if (!fail.empty()) continue;
            try {
                if (I) CUDA_CHECK(cudaMemcpyAsync(iqbefore_.get(), iq_.get(), 6 * I * sizeof(double),
                                                  cudaMemcpyDeviceToDevice, s_));
                // ||q - q_before||_inf per partition rides on the Newton readback
                auto dq_tail = [&] {
                    gate_.zero(s_);
                    launch_delta_inf(n_rows_, rinst_.get(), rpart_.get(), p0_, iq_.get(), iqbefore_.get(),
                                     gate_.get(), s_);
                    CUDA_CHECK(cudaMemcpyAsync(pin_d_.get() + 96, gate_.get(), P_ * sizeof(double),
                                               cudaMemcpyDeviceToHost, s_));
                };
                const bool fused_dq = use_graph_ && n_rows_ > 0;
                auto solve = [&] {
                    return use_graph_ ? newton_graph(hs_.newton_cap, tol, fused_dq ? dq_tail : std::function<void()>{})
                                      : newton_batch(hs_.newton_cap, tol);
                };
                // Capacity overflow inside the solve (contact list, BSR row
                // width): grow and redo the solve from its start. newton.cpp:
                // 56-58's line-search collapse: the reference solves exactly
                // (SimplicialLDLT); an iterative solve to a relative residual
                // can leave error in near-null directions that keeps
                // ||dq||_inf above tol where the exact step would stop, so the
                // solve is redone once with the PCG at the exact-solve limit
                // before the error is reported.
                NewtonResult r;
                SolverRestore restore(*this);
                for (int grows = 0, exact = 0;;) {
                    try {
                        const NvtxRange range("dabd.solve");
                        const auto tn = std::chrono::steady_clock::now();
                        r = solve();
                        st.t_solve += seconds_since(tn); // runtime.cpp:466-468
                        break;
                    } catch (const DeviceError& e) {
                        const bool cap = (e.code == kErrCapacity || e.code == kErrEll) && grows < kMaxGrows;
                        const bool ls = e.code == kErrLineSearch && !exact;
                        if (!cap && !ls) throw;
                        if (I) CUDA_CHECK(cudaMemcpyAsync(iq_.get(), iqbefore_.get(), 6 * I * sizeof(double),
                                                          cudaMemcpyDeviceToDevice, s_));
                        if (cap) {
                            grow_capacity(e.code);
                            ++grows;
                            ++capacity_retries_;
                        } else {
                            set_solver(1e-14, std::max(pcg_max_, 50000));
                            exact = 1;
                            ++exact_retries_;
                        }
                    }
                }
                st.newton_iterations += r.iterations;
                st.line_search_steps += r.ls_steps;
                st.pcg_iterations += r.pcg_iters;
                for (int p = 0; p < P_; ++p) cost[p] += partition_cost(ps_h_[p]);
                st.max_contacts = std::max(st.max_contacts, n_contacts_);
                st.max_candidates = std::max(st.max_candidates, n_super_);
                prof.mark(3, s_);
                if (fused_dq) {
                    for (int p = 0; p < P_; ++p) dq[p] = pin_d_[96 + p];
                } else {
                    dq = n_rows_ ? delta_inf(iq_.get(), iqbefore_.get()) : std::vector<double>(P_, 0.0);
                }
                prof.mark(4, s_);
            } catch (const Error& e) {
                if (!distributed_) throw;
                fail = e.what();
            }
        }
        if (retry) {
            ++attempt;
            continue;
        }
        if (!ended) throw Error("controller: frame ended without a decision");
        // rho carry + commit (runtime.cpp:481-506)
        std::vector<double> rho_now = irho_.to_host(s_);
        std::fill(rho_carry_.begin(), rho_carry_.end(), std::numeric_limits<double>::quiet_NaN());
        // Replicas carry equal rho (k_consensus checks it), so any local
        // replica may stand in for the lowest holder's.
        for (int i = 0; i < I; ++i)
            if (anc[i]) rho_carry_[h_ibody_[i]] = rho_now[i];
        launch_commit(ds_.view(), I, ibody_.get(), ipart_.get(), ianc_.get(), bmask_.get(),
                      iq_.get(), iznext_.get(), q_start_.get(), h, q_.get(), qd_.get(), s_);
        if (distributed_) {
            const NvtxRange range("dabd.sync.commit");
            const auto ts = std::chrono::steady_clock::now();
            commit_gather();
            sync();
            st.t_sync += seconds_since(ts);
        }
        if (hs_.balance.enabled && W_ > 1) {
            // every rank needs every partition's cost (runtime.cpp:674-675)
            const std::vector<double> all = distributed_ ? allgather_host(cost) : cost;
            if (distributed_) { // fixed-width records, one per rank (allgather_host)
                const size_t stride = all.size() / comm_.world;
                for (int r = 0; r < comm_.world; ++r)
                    for (int p = comm_.part_offsets[r]; p < comm_.part_offsets[r + 1]; ++p)
                        part_cost_[p] = all[stride * r + (p - comm_.part_offsets[r])];
            } else {
                for (int p = 0; p < P_; ++p) part_cost_[p0_ + p] = all[p];
            }
            have_costs_ = true;
        }
        sync();
        prof.mark(5, s_);
        tsc_.on_frame_committed();
        st.exact_retries = static_cast<int>(exact_retries_ - exact0);
        st.capacity_retries = static_cast<int>(capacity_retries_ - cap0);
        st.committed = 1;
        return st;
    }
}

} // namespace dabd_gpu

namespace dabd_gpu {

void Engine::list_stats(long long* rebuilds, int* length, double* delta) {
    CUDA_CHECK(cudaMemcpyAsync(lstate_h_.get(), lstate_.get(), sizeof(ListState),
                               cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaMemcpyAsync(pin_i_.get() + 4, det_.d_count(), sizeof(int), cudaMemcpyDeviceToHost, s_));
    sync();
    *rebuilds = lstate_h_[0].n_rebuilds;
    *length = pin_i_[4];
    std::vector<double> sk = iskin_.to_host(s_);
    double m = 0.0;
    for (int i = 0; i < n_inst_; ++i) m = std::max(m, sk[i]);
    *delta = m;
}

DevPerf Engine::read_perf(bool reset) {
    DevPerf h{};
    CUDA_CHECK(cudaMemcpyAsync(&h, perf_.get(), sizeof(DevPerf), cudaMemcpyDeviceToHost, s_));
    CUDA_CHECK(cudaStreamSynchronize(s_));
    if (reset) {
        perf_.zero(s_);
        CUDA_CHECK(cudaStreamSynchronize(s_));
    }
    return h;
}

} // namespace dabd_gpu
