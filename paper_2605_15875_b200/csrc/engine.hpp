// The per-GPU engine behind the C ABI: owns every device buffer, runs the
// batched local solves, the consensus ADMM iteration and the frame loop.
// Host control follows proj/src/runtime.cpp:110-694 (worker + controller
// collapsed onto replicated global state) and
// proj/src/sim.cpp:186-249 (num_workers == 0).
#pragma once

#include "audit.hpp"
#include "geometry.cuh"
#include "kernels.hpp"
#include "admm.hpp"
#include "balance.hpp"
#include "controller.hpp"
#include "scene.hpp"
#include "solver.hpp"

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace dabd_gpu {

struct FrameStats {
    int committed = 0, attempts = 1;
    double h = 0.0;
    int admm_iterations = 0, newton_iterations = 0, line_search_steps = 0, pcg_iterations = 0;
    int max_contacts = 0, max_candidates = 0;
    int exact_retries = 0;    // solves redone at the exact-solve PCG limit (line-search collapse)
    int capacity_retries = 0; // work redone after a capacity grew (list / ELL width)
    // host wall-clock seconds (runtime.cpp:117-124, 399-402, 466-475): local
    // Newton solves, consensus + merge-gate collision work, waiting on
    // exchanges with peer ranks, the whole frame (compute = frame - sync)
    double t_solve = 0.0, t_coll = 0.0, t_sync = 0.0, t_frame = 0.0;
};

struct TraceRow {
    double frame, attempt, k, dq, r, s, toi, sigma;
};

struct NewtonResult {
    int iterations = 0, ls_steps = 0, pcg_iters = 0, converged = 0;
    double final_update = 0.0;
};

// Inter-rank exchange of a partition-per-GPU run (dabd_gpu_comm in
// include/dabd_gpu.h). Device pointers, ordered on the engine's stream.
struct Comm {
    void* user = nullptr;
    int (*halo)(void*, const double*, double*, size_t, const double*, double*, size_t,
                uintptr_t) = nullptr;
    int (*allgather)(void*, const double*, double*, size_t, uintptr_t) = nullptr;
    int rank = 0, world = 1;
    std::vector<int> part_offsets; // world + 1
};

class Engine {
  public:
    Engine(const HostScene& hs, int device, int num_workers, int part_begin, int part_end);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void set_stream(cudaStream_t s);
    void set_comm(const Comm* c);
    void set_solver(double tol, int max_iters) {
        pcg_tol_ = tol;
        pcg_max_ = max_iters;
        graph_ok_ = false; // the captured frame bakes the PCG arguments in
        ++solver_epoch_;
    }
    cudaStream_t stream() const { return s_; }
    int comm_mode() const {
        if (!distributed_) return 0;
        if (!p2p_) return 1;
        return fan_ok_ && admm_device_ && use_graph_ ? 3 : 2;
    }
    const HostScene& scene() const { return hs_; }

    // ---- parity entry points (host arrays) ----
    std::vector<int> broad_phase(const double* q, const double* q_end, double margin,
                                 const int* subset, int n_subset);
    void narrow_phase(const double* q, const int* cand, int n, double d_hat,
                      std::vector<int>& pairs, std::vector<double>& d);
    double ccd_toi(const double* q0, const double* q1, const int* subset, int n_subset);
    void holder_masks(const double* q, int n_planes, const double* planes, double w,
                      uint32_t* masks);
    struct ObjectiveIn {
        int n_local;
        const int* local;
        const double* kappa;
        const double* q_tilde;
        int n_anchor;
        const int* anchor_body;
        const double* anchor_zu;
        const double* anchor_rho;
        const uint32_t* holder_mask;
        SimParams sim;
    };
    void objective(const ObjectiveIn& in, const double* q, int mode, double* value, double* grad,
                   double* hess_dense, int* active, int* candidates);
    NewtonResult newton_solve(const ObjectiveIn& in, double* q, int max_iters, double tol);
    // intersection_test + minimum distance (audit.cu); q == nullptr audits
    // the device-resident current state.
    AuditResult audit(const double* q, const int* subset, int n_subset, double cutoff);

    // ---- stepping ----
    void run_frames(int n, FrameStats* stats);
    void set_state(const double* q, const double* qd);
    void get_state(double* q, double* qd);
    void get_rho(double* rho) const;
    std::vector<TraceRow> take_trace();
    // interface planes in use ((W-1) x (px, py, nx, ny)) and the per-partition
    // compute costs of the last committed frame that fed the balancer
    std::vector<double> planes() const;
    const std::vector<double>& partition_costs() const { return part_cost_; }
    // PCG launch accounting since the last reset (device %globaltimer, SURVEY 8(d) bytes).
    DevPerf read_perf(bool reset);
    void list_stats(long long* rebuilds, int* length, double* delta);

  private:
    // instance sets ----------------------------------------------------------
    void build_instances(const std::vector<std::vector<int>>& per_part, const uint32_t* masks,
                         bool single_domain);
    void gather_iq(const double* q_dev);
    SolverView view();
    ContactView cview();
    InstView iview(const double* q0, const double* q1);
    void check_err(const char* where);
    void sync();

    // local solve (enqueue-only, capturable) -----------------------------------
    void prepare_solver();
    void enq_superset(const double* q0, const double* q1, bool swept);
    void enq_list_ensure(const double* q1, bool fused_ccd = false);
    void enq_list_rebuild();
    void invalidate_list();
    void enq_energy(int qmode, int which, double PartState::*field, bool accept = false);
    void enq_derivatives(bool fused = false);
    void enq_pcg(bool fused = false);
    int max_part_rows() const;
    bool pcg_fused() const;
    int* iter_reset(); // kOpIterBegin's resets ride on kOpReset / kOpNewtonTail (fused head)
    cudaStream_t side_stream();
    void enq_newton_head(int max_iters);
    void enq_newton_ccd();
    void enq_ls_trial();
    void enq_solve_begin(double tol);
    FrameCtrl read_ctrl();
    NewtonResult newton_batch(int max_iters, double tol, bool reset_ctrl = true);
    // tail: enqueued after the graph launch, before the one readback sync
    NewtonResult newton_graph(int max_iters, double tol, const std::function<void()>& tail = {});
    std::vector<double> delta_inf(const double* a, const double* b);

    // CUDA graphs with conditional nodes -------------------------------------
    unsigned long long new_cond_handle();
    void add_cond_node(unsigned long long h, bool is_while, int level,
                       const std::function<void()>& body, bool account = true);
    cudaStream_t cap_stream(int level);
    void cap_newton(int max_iters, double tol, int level);
    void enq_reference_frame(bool graph);
    void capture_reference_graph();

    // frames -----------------------------------------------------------------
    FrameStats frame_reference();
    FrameStats frame_admm(int frame_index);
    // One attempt of the multi-partition frame as ONE captured graph (no
    // host round trip per ADMM iteration): 1 = ended, 2 = retry with h / 2,
    // 0 = a capacity grew or the exact-solve retry was armed (redo the
    // attempt); throws on any other device error.
    int admm_attempt_device(int frame, int attempt, double h, double tol, int I, int ns,
                            FrameStats& st, std::vector<double>& cost, int& grows, bool& exact);
    cudaGraphExec_t admm_exec_ = nullptr;
    DBuf<double> admm_dq_, admm_dqnew_, admm_cost_;
    PinnedBuf<double> admm_cost_h_;
    bool admm_device_ = true; // DABD_GPU_ADMM_HOST=1: the host-driven ADMM loop

    HostScene hs_;
    DeviceScene ds_;
    int device_ = 0;
    int W_ = 0, p0_ = 0, p1_ = 1, P_ = 1;
    cudaStream_t s_ = nullptr;
    bool own_stream_ = false;
    double pcg_tol_ = 1e-10;
    int pcg_max_ = 4000;
    // Inexact Newton inside frames (cluster PCG): a Newton direction may stop
    // at the relative residual eta_loose_ while its rms entry exceeds
    // eta_factor_ x the Newton tolerance; the directions that decide
    // convergence are solved to pcg_tol_. 0 = off (default for consensus
    // contexts; 1e-4 for single-domain ones, set in the constructor). The
    // standalone newton_solve parity entry point always solves to pcg_tol_.
    double eta_loose_ = 0.0, eta_factor_ = 1.0;
    bool inexact_ = true;

    // global replicated state
    DBuf<double> q_, qd_, q_start_;
    std::vector<double> rho_carry_; // host, NaN = none
    TimestepController tsc_; // h of the next attempt (consensus.hpp:60-87)
    long long frame_counter_ = 0;
    std::vector<TraceRow> trace_;
    long long exact_retries_ = 0;       // Newton solves redone at the exact-solve PCG limit
    long long capacity_retries_ = 0;    // frames / solves redone after a capacity grew
    static constexpr int kMaxGrows = 8; // capacity doublings per frame before the overflow is an error
    // restores the PCG limits a retry changed, on every exit path
    struct SolverRestore {
        Engine& e;
        double tol;
        int max;
        explicit SolverRestore(Engine& en) : e(en), tol(en.pcg_tol_), max(en.pcg_max_) {}
        ~SolverRestore() {
            if (e.pcg_tol_ != tol || e.pcg_max_ != max) e.set_solver(tol, max);
        }
    };
    DBuf<double> warm_prev_;            // previous instance set's (x, p2) while remapping
    DBuf<int> warm_map_;
    std::vector<cudaStream_t> side_streams_; // per capture level: independent branches
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    // PD load balancer of the planes (runtime.cpp:537-552, 674-675)
    std::vector<PlaneH> planes_cur_;
    Balancer balancer_;
    std::vector<double> part_cost_; // [W_] last committed frame
    bool have_costs_ = false;
    double w_last_ = 0.0;

    // instance set (host mirrors + device)
    int n_inst_ = 0, n_rows_ = 0, n_stat_ = 0;
    // Device-side instance sets (runtime.cpp:126-236, partition.cpp:69-129):
    // holder masks -> (partition, body) flags -> scans -> scatter, with one
    // read-back of the counts. Returns the number of shared-replica pairs;
    // host mirrors h_ibody_ ... are not filled (only h_pio_ / h_pro_).
    int build_instances_device(const uint32_t* masks_dev, double* w_out);
    DBuf<int> fl_all_, fl_dyn_, fl_sh_, sc_all_, sc_dyn_, sc_sh_, rowtab_, rowtab_prev_, inst_cnt_;
    PinnedBuf<int> inst_cnt_h_;
    DBuf<unsigned char> scan_temp_;
    bool rowtab_valid_ = false;
    DBuf<double> rho_carry_d_;   // device rho carry (NaN = none), authoritative when carry_on_device_
    bool carry_on_device_ = false;
    DBuf<uint32_t> masks_d_;
    bool single_domain_ = true;
    std::vector<int> h_ibody_, h_ipart_, h_irow_, h_rinst_, h_rpart_, h_stat_;
    std::vector<int> h_pio_, h_pro_;
    DBuf<int> ibody_, ipart_, irow_, rinst_, rpart_, stat_, pio_, pro_, ianc_;
    DBuf<double> iq_, iqtry_, iqt_, iinvk_, iz_, iu_, irho_, irho0_, iznext_, iqbefore_;
    DBuf<uint32_t> bmask_;
    DBuf<double> rgrad_, rdiag_, rdinv_, rval_, x_, r_, z_, p0v_, p1v_, ap_, rowtmp_, rowtmp2_;
    DBuf<int> ell_cnt_, ell_col_;
    int ell_w_ = kEll; // ELL width, doubled on kErrEll (a row coupling more bodies)
    bool grow_capacity(int code); // kErrCapacity / kErrEll: grow, true if grown
    DBuf<double> ell_blk_;
    DBuf<PartState> ps_;
    PinnedBuf<PartState> ps_h_;
    DBuf<double> scal_a_, scal_b_, partial_, gate_;
    DBuf<int> err_;
    PinnedBuf<int> pin_i_;
    PinnedBuf<double> pin_d_;

    // detection
    Detector det_;       // superset for the local solve
    Detector det_gate_;  // merge gate / parity
    int gate_cap_ = 0;   // fixed merge-gate candidate capacity (grown on kErrCapacity)
    int n_super_ = 0;
    DBuf<Box> box_;
    DBuf<double> cellmax_;
    DBuf<unsigned char> cflag_;
    DBuf<double> sval_;
    DBuf<unsigned long long> ckey_, bkey_, bkey_sorted_;
    DBuf<int> bidx_, perm_b_, aoff_, boff_, nsel_;
    DBuf<double> cval_, cgrad_, cblk_;
    DBuf<int> act_;
    // skin list (ListState in solver.hpp): det_ holds the list keys
    DBuf<double> qref_, iskin_, iskin_next_;
    double skin_min_ = 0.5;  // x d_hat
    double skin_grow_ = 1.5;
    DBuf<ListState> lstate_;
    PinnedBuf<ListState> lstate_h_;
    long long rebuild_nodes_ = 0; // kernels in one captured rebuild body
    long long rebuilds_seen_ = 0; // ListState::n_rebuilds at the last frame end
    int cap_level_ = -1;          // capture level of s_ while capturing (-1: top)
    DBuf<unsigned char> temp_;
    int n_contacts_ = 0;
    KeyFmt cfmt_;

    // ADMM shared bodies: [ns][2] replica handles in ascending partition
    // order, >= 0 a local instance, < 0 the halo packet -1 - v (remote rank).
    std::vector<int> h_shared_inst_;
    DBuf<int> shared_inst_;
    // partition-per-GPU exchange
    bool distributed_ = false;
    Comm comm_;
    std::vector<int> h_halo_inst_;    // local instances packed: lo side then hi side
    int n_halo_lo_ = 0, n_halo_hi_ = 0;
    DBuf<int> halo_inst_, part_rank_;
    DBuf<double> hsend_, hrecv_, rec_, rec_all_, gath_;
    void exchange_halo();
    // Peer-memory halo (SURVEY 8(e) "direct P2P halo reads"): every rank
    // publishes its packets in a device buffer the neighbours map through
    // CUDA IPC; k_consensus loads the neighbours' packets directly.
    // pub_ regions: [side lo/hi][parity] x pub_cap_ packets.
    void setup_p2p();
    void comm_barrier();
    // Device fan-in (partition-per-GPU device ADMM loop): every rank's buffer
    // [world][kFanStride] records + [world] flags, mapped into every peer.
    static constexpr int kFanStride = 2 + 4 * kMaxParts;
    static constexpr int kFuseAcceptMaxInst = 4096; // k_energy's last block applies accepted steps up to this
    int tail_max_iters_ = 0; // while capturing a folded-tail Newton body: its iteration cap
    void setup_fanin();
    void close_fanin();
    DBuf<unsigned char> fan_buf_;
    DBuf<double> fan_rec_local_;
    DBuf<unsigned long long> fan_seq_;
    FanView fan_view_;
    std::vector<void*> fan_opened_;
    bool fan_ok_ = false;
    DBuf<double> pub_;
    size_t pub_cap_ = 0;
    const double* peer_lo_ = nullptr; // rank - 1's pub_ (mapped)
    const double* peer_hi_ = nullptr; // rank + 1's pub_ (mapped)
    bool p2p_ = false;
    int halo_parity_ = 0;
    const double* remote_lo_ = nullptr; // what k_consensus reads this iteration
    const double* remote_hi_ = nullptr;
    std::vector<double> allgather_host(const std::vector<double>& mine);
    void commit_gather();
    DBuf<int> own_cnt_, own_cnts_;
    DBuf<double> own_rec_;
    DBuf<double> rloc_, sloc_, rb_, sb_;
    DBuf<double> ifs_; // per-instance force split (fx, fy)
    SimParams frame_params_;
    int project_ = 1;
    DBuf<double> pbuf_, pcg_part_, pcg_vec_;
    DBuf<DevPerf> perf_;
    Auditor auditor_;
    DBuf<double> audit_q_;
    int pcg_phases_ = 0;

    // fixed capacities (graph-safe) and the captured N=1 frame
    int cap_ = 0;
    int det_fmt_n_ = -1;
    size_t temp_bytes_ = 0;
    DBuf<FrameCtrl> ctrl_;
    PinnedBuf<FrameCtrl> ctrl_h_;
    CondHandles hd_;
    cudaGraphExec_t exec_ = nullptr;
    // captured Newton solve of the ADMM frame (newton_graph)
    cudaGraphExec_t newton_exec_ = nullptr;
    long long solver_epoch_ = 0, newton_epoch_ = -1;
    double newton_tol_ = 0.0;
    int newton_max_ = 0;
    long long newton_inc_[4] = {}, newton_total_ = 0;
    bool graph_ok_ = false;
    bool use_graph_ = true;
    bool ref_ready_ = false;
    long long nodes_inc_[8] = {};  // kernels captured per conditional level (inclusive)
    long long nodes_total_ = 0;
    bool graph_replayed_ = false;
    std::vector<cudaStream_t> cap_streams_;
    DBuf<double> trace_dev_;
    int trace_cap_ = 4096;
    DBuf<double> qd_start_;

  public:
    void set_inexact(double eta, double factor) {
        eta_loose_ = eta;
        eta_factor_ = factor;
        graph_ok_ = false;
        ++solver_epoch_;
    }
    void set_use_graph(bool on) {
        use_graph_ = on;
        graph_ok_ = false;
        ++solver_epoch_;
    }
};

} // namespace dabd_gpu
