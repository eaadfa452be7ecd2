// pairamg_b200.hpp -- header-only C++ mirror of the reference's hot-path API
// (namespace pairamg in /root/reference/proj/src/pairamg) over the C ABI of
// libpairamg_b200.so.  Same names, argument meaning and error behaviour:
//   pairamg::ErrorCode / pairamg::Error        types.hpp:13-35
//   pairamg::Partition::uniform                 runtime.hpp:15-28, runtime.cpp:13-22
//   pairamg::SetupConfig / CycleConfig          amg.hpp:17-23, cycle.hpp:7-12
//   pairamg::MatchingTrace (replay / record)    amg.hpp:13-23, amg.cpp:182-220
//   pairamg::SolveConfig / SolveStats           SPEC.md:468-477 (pcg.cpp absent)
//   pairamg::b200::Solver::setup                setup_hierarchy, amg.hpp:84-85
//   pairamg::b200::Solver::solve                pcg_solve
//   pairamg::b200::Solver::vcycle / spmv        vcycle_apply cycle.hpp:31-32, spmv_dist dist.hpp:83-86
//   pairamg::b200::Solver::summary              hierarchy_summary, amg.cpp:297-313
// Failures throw pairamg::Error carrying the ErrorCode, like the reference.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pairamg_b200.h"

namespace pairamg {

using index_t = std::int64_t;
using real_t = double;

enum class ErrorCode {
    invalid_argument,
    contract_violation,
    missing_row,
    singular_smoother,
    stagnation,
    breakdown,
    deadlock,
    parse_error,
    io_error,
    internal,
};

class Error : public std::runtime_error {
public:
    Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
    ErrorCode code() const noexcept { return code_; }

private:
    ErrorCode code_;
};

inline void check(pairamg_status s) {
    if (s != PAIRAMG_OK)
        throw Error(static_cast<ErrorCode>(static_cast<int>(s) - 1), pairamg_last_error());
}

struct Partition {
    index_t global_n = 0;
    std::vector<index_t> starts;
    static Partition uniform(index_t n, int nranks) {
        Partition p;
        p.global_n = n;
        p.starts.resize(static_cast<size_t>(nranks) + 1);
        for (int r = 0; r <= nranks; ++r) p.starts[r] = (n / nranks) * r + std::min<index_t>(n % nranks, r);
        return p;
    }
    index_t begin(int r) const { return starts[r]; }
    index_t end(int r) const { return starts[r + 1]; }
    index_t extent(int r) const { return starts[r + 1] - starts[r]; }
};

// Recorded pairwise matchings (global mates, one array per pairwise step).
struct MatchingTrace {
    std::vector<std::vector<index_t>> steps;
};

struct SetupConfig {
    int aggregation_exponent = 3;
    index_t coarse_size_target = 40;
    int max_levels = 40;
    const MatchingTrace* replay = nullptr;
    MatchingTrace* record = nullptr;
};

struct CycleConfig {
    int pre_sweeps = 4;
    int post_sweeps = 4;
    int coarsest_sweeps = 20;
    real_t relax_weight = 1.0;
};

struct SolveConfig {
    real_t rtol = 1e-6;
    int max_iters = 1000;
    bool precflag = true;
};

struct SolveStats {
    int iterations = 0;
    real_t final_relres = 0.0;
    bool converged = false;
    std::vector<real_t> history;
    double t_solve = 0.0;
};

namespace b200 {

// One rank: a GPU plus (nranks > 1) an NCCL communicator.
class Runtime {
public:
    Runtime(int device, int rank, int nranks, const std::vector<uint8_t>& nccl_id = {}) : rank_(rank), nranks_(nranks) {
        check(pairamg_runtime_create(device, rank, nranks, nccl_id.empty() ? nullptr : nccl_id.data(), &h_));
    }
    ~Runtime() { pairamg_runtime_destroy(h_); }
    Runtime(const Runtime&) = delete;
    Runtime& operator=(const Runtime&) = delete;
    static std::vector<uint8_t> unique_id() {
        std::vector<uint8_t> id(128);
        check(pairamg_comm_unique_id(id.data()));
        return id;
    }
    // ranks that are threads of this process (spawn_ranks): one id for all of them
    static std::vector<uint8_t> local_id() {
        std::vector<uint8_t> id(128);
        check(pairamg_comm_local_id(id.data()));
        return id;
    }
    int rank() const { return rank_; }
    int nranks() const { return nranks_; }
    pairamg_runtime* get() const { return h_; }

private:
    pairamg_runtime* h_ = nullptr;
    int rank_, nranks_;
};

class Solver {
public:
    explicit Solver(Runtime& rt) : rt_(rt) { check(pairamg_solver_create(rt.get(), &h_)); }
    ~Solver() { pairamg_solver_destroy(h_); }
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;

    // Owned row block in the reference CsrMatrix layout (global columns).
    void setup(const Partition& part, const std::vector<index_t>& row_ptr, const std::vector<index_t>& col_idx,
               const std::vector<real_t>& values, const std::vector<real_t>* w0 = nullptr,
               const SetupConfig& cfg = {}) {
        pairamg_setup_config c;
        pairamg_default_setup_config(&c);
        c.aggregation_exponent = cfg.aggregation_exponent;
        c.coarse_size_target = cfg.coarse_size_target;
        c.max_levels = cfg.max_levels;
        std::vector<const int64_t*> mates;
        std::vector<int64_t> sizes;
        if (cfg.replay) {
            for (const auto& m : cfg.replay->steps) {
                mates.push_back(m.data());
                sizes.push_back(static_cast<int64_t>(m.size()));
            }
            c.replay_steps = static_cast<int>(mates.size());
            c.replay_mates = mates.data();
            c.replay_sizes = sizes.data();
        }
        check(pairamg_setup(h_, part.global_n, part.starts.data(), part.extent(rt_.rank()), row_ptr.data(),
                            col_idx.data(), values.data(), w0 ? w0->data() : nullptr, &c));
        if (cfg.record) {  // this rank's owned block of every step (the reference records on rank 0 only)
            int steps = 0;
            check(pairamg_num_matchings(h_, &steps));
            cfg.record->steps.clear();
            for (int t = 0; t < steps; ++t) {
                int64_t n = 0;
                check(pairamg_matching_export(h_, t, &n, nullptr));
                std::vector<index_t> m(static_cast<size_t>(n));
                check(pairamg_matching_export(h_, t, &n, m.data()));
                cfg.record->steps.push_back(std::move(m));
            }
        }
    }

    // Hierarchy::warnings (amg.hpp:56) + validate_cycle_config's (cycle.cpp:7-13).
    std::vector<std::string> warnings() const {
        int n = 0;
        check(pairamg_setup_warnings(h_, &n));
        std::vector<std::string> out;
        for (int i = 0; i < n; ++i) {
            size_t len = 0;
            check(pairamg_setup_warning(h_, i, nullptr, 0, &len));
            std::string w(len + 1, '\0');
            check(pairamg_setup_warning(h_, i, w.data(), w.size(), nullptr));
            w.resize(len);
            out.push_back(std::move(w));
        }
        return out;
    }

    SolveStats solve(const std::vector<real_t>& b, std::vector<real_t>& u, const CycleConfig& cc = {},
                     const SolveConfig& sc = {}) {
        SolveStats out;
        out.history.assign(static_cast<size_t>(sc.max_iters) + 1, 0.0);
        pairamg_solve_stats st{};
        st.history = out.history.data();
        st.history_cap = static_cast<int>(out.history.size());
        const pairamg_cycle_config c{cc.pre_sweeps, cc.post_sweeps, cc.coarsest_sweeps, cc.relax_weight};
        const pairamg_solve_config s{sc.rtol, sc.max_iters, sc.precflag ? 1 : 0};
        check(pairamg_solve(h_, b.data(), u.data(), &c, &s, &st));
        out.iterations = st.iterations;
        out.final_relres = st.final_relres;
        out.converged = st.converged != 0;
        out.history.resize(static_cast<size_t>(st.iterations) + 1);
        out.t_solve = st.t_solve_s;
        return out;
    }

    std::vector<real_t> vcycle(const std::vector<real_t>& r, const CycleConfig& cc = {}) {
        std::vector<real_t> x(r.size());
        const pairamg_cycle_config c{cc.pre_sweeps, cc.post_sweeps, cc.coarsest_sweeps, cc.relax_weight};
        check(pairamg_vcycle(h_, r.data(), x.data(), &c, 0));
        return x;
    }

    std::vector<real_t> spmv(int level, const std::vector<real_t>& x) {
        int64_t rows = 0;
        check(pairamg_level_info(h_, level, nullptr, nullptr, nullptr, &rows, nullptr));
        std::vector<real_t> y(static_cast<size_t>(rows));
        check(pairamg_spmv(h_, level, x.data(), y.data(), 0));
        return y;
    }

    // hierarchy_summary (amg.cpp:297-313), same format.
    std::string summary() const {
        int nl = 0;
        double opc = 0;
        check(pairamg_hierarchy_info(h_, &nl, &opc));
        std::string s = "level        rows          nnz\n";
        char buf[96];
        for (int k = 0; k < nl; ++k) {
            int64_t rows = 0, nnz = 0;
            check(pairamg_level_info(h_, k, &rows, &nnz, nullptr, nullptr, nullptr));
            std::snprintf(buf, sizeof buf, "%5d%13lld%13lld\n", k + 1, static_cast<long long>(rows),
                          static_cast<long long>(nnz));
            s += buf;
        }
        std::snprintf(buf, sizeof buf, "levels %d, operator complexity %.4f\n", nl, opc);
        return s + buf;
    }

    pairamg_solver* get() const { return h_; }

private:
    Runtime& rt_;
    pairamg_solver* h_ = nullptr;
};

}  // namespace b200
}  // namespace pairamg
