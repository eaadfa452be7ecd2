// C++ host example over the drop-in boundary: the reference's usage flow
// (Appendix A, "x <- bcmgx(A, b, p, precflag)") written against
// include/pairamg_b200.hpp.  Built and run by tests/test_cpp_host.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "pairamg_b200.hpp"

int main(int argc, char** argv) {
    const int nd = argc > 1 ? std::atoi(argv[1]) : 24;
    const pairamg::index_t n = static_cast<pairamg::index_t>(nd) * nd * nd;
    pairamg::b200::Runtime rt(0, 0, 1);
    const auto part = pairamg::Partition::uniform(n, 1);
    // generate the owned rows with the library's host generator
    const int64_t nnz = pairamg_poisson_nnz(7, nd, nd, nd, 0, n);
    std::vector<pairamg::index_t> rp(static_cast<size_t>(n) + 1), ci(static_cast<size_t>(nnz));
    std::vector<double> va(static_cast<size_t>(nnz));
    pairamg::check(pairamg_poisson_host(7, nd, nd, nd, 0, n, rp.data(), ci.data(), va.data()));
    pairamg::b200::Solver solver(rt);
    pairamg::SetupConfig cfg;
    cfg.coarse_size_target = 40 * nd;
    solver.setup(part, rp, ci, va, nullptr, cfg);
    std::printf("%s", solver.summary().c_str());
    std::vector<double> b(static_cast<size_t>(n), 1.0), u(static_cast<size_t>(n), 0.0);
    const auto st = solver.solve(b, u);
    std::printf("iterations %d relres %.3e converged %d\n", st.iterations, st.final_relres, st.converged ? 1 : 0);
    // error behaviour mirrors pairamg::Error
    try {
        pairamg::b200::Solver bad(rt);
        bad.solve(b, u);
        return 2;
    } catch (const pairamg::Error& e) {
        std::printf("caught %d: %s\n", static_cast<int>(e.code()), e.what());
        if (e.code() != pairamg::ErrorCode::contract_violation) return 3;
    }
    return st.converged ? 0 : 1;
}
