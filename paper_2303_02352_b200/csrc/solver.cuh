// solver.cuh -- per-rank solver object behind the C ABI: the device
// hierarchy, the flexible-CG state and the captured iteration graph.
#pragma once

#include <array>
#include <memory>
#include <vector>

#include "amg.cuh"
#include "p2p.cuh"

namespace pb {

// Fused level-0 zero-start sweep written by the FCG update (solve.cu).
struct ZeroStart {
    double* x = nullptr;
    const uint8_t* pid = nullptr;  // STEN level 0: pattern byte per row ...
    const double* ptab = nullptr;  // ... and the per-pattern l1 diagonal
    const double* pinv = nullptr;  // ... and its reciprocal (ddiv_recip)
    const double* l1 = nullptr;    // otherwise the l1 array
    double omega = 1.0;
};

// Device-resident FCG scalars (Alg. 1 lines 11-15), read once per iteration.
struct FcgState {
    double alpha, beta, gamma, rho;  // current dots / rho_i
    double c, a;                     // gamma_i/rho_{i-1}, alpha_i/rho_i
    double rr, rr0;                  // |r_{i+1}|^2, |r_0|^2
    int it;                          // iterations completed
    int status;                      // 0 ok, 1 breakdown
    int stop;                        // multi-rank: r_it met the stopping test, no update
};

// Timed kernel classes (level 0): 0 l1-Jacobi sweep, 1 residual,
// 2 SpMV + dot triple, 3 FCG vector update; kLevelClass + k: level k's own
// V-cycle work (everything between entering level k and leaving it, minus
// level k+1's cycle; two intervals per V-cycle), for k < kTimedLevels.
constexpr int kLevelClass = 4;
constexpr int kTimedLevels = 16;
constexpr int kNumClasses = kLevelClass + kTimedLevels;

struct KernelClassTiming {
    int64_t launches = 0;
    double ms = 0.0;
    double bytes_per_launch = 0.0;
};

class Solver {
public:
    explicit Solver(Runtime& rt);
    ~Solver();

    void setup(std::vector<int64_t> starts, DBuf<int64_t>&& rp, DBuf<int64_t>&& col, DBuf<double>&& val,
               int64_t nnz, const double* d_w0, const SetupConfig& cfg);
    // Flexible PCG on device vectors (owned block).  Returns iterations.
    void solve(const double* d_b, double* d_u, const CycleConfig& cc, double rtol, int max_iters,
               bool precflag, pairamg_solve_stats* st);
    void vcycle(const double* d_r, double* d_x, const CycleConfig& cc);
    void spmv(int level, const double* d_x, double* d_y);
    // Hierarchy::warnings plus validate_cycle_config's (cycle.cpp:7-13) for
    // the cycle configuration of the last solve / V-cycle.
    std::vector<std::string> warnings() const;

    Runtime& rt;
    Hierarchy h;
    bool ready = false;
    bool timing = false;
    bool overlap = true;  // halo exchange overlapped with interior rows (else exchange, then all rows)
    bool mr_device_loop_ok() const;
    bool loop_ok = true;  // single-rank solves run as one graph with a device-side stopping test
    bool p2p_ = true;         // NVLink direct-store exchanges (else NCCL)
    int halo_grid_ = 0;       // CTA cap of interior kernels on halo levels (0 = uncapped)
    P2PGather dots_gather_;   // NVLink allgather of the per-iteration dot partials
    P2PSegGather rep_gather_; // NVLink gather of the first replicated level's right-hand side
    std::array<KernelClassTiming, kNumClasses> ktime{};
    int64_t last_launches = 0;
    std::string cycle_warning;

private:
    // enqueue helpers (host-side pointer bookkeeping; graph-capturable)
    void smooth(int k, bool zero_start, int nu, const double* rhs, double*& xcur, double*& xoth, double omega,
                bool time_l0);
    void apply(int k, const SellOpArgs& o, int kclass);
    void apply_on(Level& L, const SellOpArgs& o, int kclass);
    void exchange(Level& L, const double* x, cudaStream_t st);
    bool split_launch(const Level& L) const;
    void shared_gpu_fence();
    int interior_cap(const Level& L) const;  // CTA cap of the interior launch next to a halo exchange
    Level& lvl(int k);  // replicated copy for k >= h.rep_level, else the distributed level
    void vcycle_enqueue(int k, const double* rhs, double*& out, const CycleConfig& cc);
    void iteration_enqueue(const CycleConfig& cc, bool precflag);
    bool zs_fused(const CycleConfig& cc, bool precflag);
    ZeroStart zero_start_args(const CycleConfig& cc);
    bool zs_pending_ = false;  // level-0 x1 of the next V-cycle is already formed
    int zs_level_ = -1;        // coarse level whose x1 the last restriction formed
    void reduce_dots_enqueue(bool fused_norm);
    void reduce_norm_enqueue(bool init_rr0);
    void ensure_vectors();
    void ensure_events(int kclass, int idx);
    void begin_time(int kclass);
    void end_time(int kclass);
    void collect_times();
    void destroy_graph();

    cudaStream_t s_;
    int64_t n_ = 0, next_ = 0;
    DBuf<double> u_, r_, w_, v_, d_, q_;
    DBuf<double> partials_, stage_, local_, gathered_;
    DBuf<FcgState> state_;
    FcgState* h_state_ = nullptr;  // pinned
    int max_blocks_ = 0;
    int dots_grid_ = 0;  // partial triples of the last SpMV+dots enqueue
    double* w_out_ = nullptr;      // buffer holding w_i after the captured V-cycle
    cudaGraphExec_t graph_ = nullptr;
    CycleConfig graph_cc_{};
    bool graph_prec_ = true;
    bool graph_timing_ = false;
    // whole-solve graph: conditional WHILE node around the captured iteration
    cudaGraphExec_t loop_graph_ = nullptr;
    CycleConfig loop_cc_{};
    bool loop_prec_ = true;
    double loop_rtol_ = 0.0;
    int loop_maxit_ = 0;
    DBuf<double> hist_;
    void ensure_loop_graph(const CycleConfig& cc, bool precflag, double rtol, int max_iters);
    int64_t per_iter_launches_ = 0;
    int reductions_per_iter_ = 0, halos_per_iter_ = 0;  // cross-rank exchanges per FCG iteration
    double halo_bytes_per_iter_ = 0.0;
    double cap_rtol_ = 0.0;  // stopping test captured into the multi-rank iteration graph
    int cap_maxit_ = 0;
    std::vector<cudaEvent_t> ev_pool_;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    // per-class event pairs recorded in the captured iteration
    std::array<std::vector<std::pair<cudaEvent_t, cudaEvent_t>>, kNumClasses> tev_{};
    std::array<int, kNumClasses> tcount_{};
    std::array<int, kNumClasses> topen_{};
    int64_t launches_ = 0;
};

}  // namespace pb
