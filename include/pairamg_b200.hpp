// pairamg_b200.hpp -- header-only C++ mirror of the reference's hot-path API
// (namespace pairamg in /root/reference/proj/src/pairamg) over the C ABI of
// libpairamg_b200.so.  Same names, argument meaning and error behaviour:
//   pairamg::ErrorCode / pairamg::Error        types.hpp:13-35
//   pairamg::Partition::uniform                 runtime.hpp:15-28, runtime.cpp:13-22
//   pairamg::SetupConfig / CycleConfig          amg.hpp:17-23, cycle.hpp:7-12
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

struct SetupConfig {
    int aggregation_exponent = 3;
    index_t coarse_size_target = 40;
    int max_levels = 40;
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
        const pairamg_setup_config c{cfg.aggregation_exponent, cfg.coarse_size_target, cfg.max_levels};
        check(pairamg_setup(h_, part.global_n, part.starts.data(), part.extent(rt_.rank()), row_ptr.data(),
                            col_idx.data(), values.data(), w0 ? w0->data() : nullptr, &c));
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
