// ref_driver.cpp -- TEST INFRASTRUCTURE: drives the reference's own compiled
// objects (csr, runtime, dist, matching, amg, cycle from
// /root/reference/proj/src/pairamg) through oracle_api.h.
//
// The reference ships no Krylov solver, no problem generator and no C API
// (pcg.cpp, problem.cpp, capi.cpp are listed in src/CMakeLists.txt:11-21 but
// absent).  This file restates only those two missing pieces:
//   * the 7/27-point Poisson generator per SPEC.md:512-557 (lexicographic,
//     x fastest, diagonal 6 (26), off-diagonals -1, b = 1);
//   * Notay's flexible PCG, PAPER.md:86-115 (Alg. 1) with SPEC.md:474-482,
//     built only from the reference's own spmv_dist / dot_dist /
//     vcycle_apply (dist.cpp:128-199, 412-421; cycle.cpp:86-112).
// Everything else (setup_hierarchy, matching, Galerkin, V-cycle, halo SpMV)
// is the unmodified reference code, run as p ranks on p threads by
// spawn_ranks (runtime.cpp:92-152).  Compiled by oracle/Makefile into
// oracle/_ref/libpairamg_ref.so; never linked into the product.
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pairamg/amg.hpp"
#include "pairamg/cycle.hpp"
#include "pairamg/dist.hpp"
#include "pairamg/mm_io.hpp"

#include "oracle_api.h"

using namespace pairamg;

namespace {

thread_local std::string g_err;
thread_local int g_status = 0;

struct RankState {
    DistMatrix A;
    DistVector b;
    DistVector w0;
    Hierarchy h;
};

struct Session {
    orc_config cfg;
    index_t n = 0;
    CsrMatrix global;  // only for orc_create_csr
    std::vector<RankState> ranks;
    MatchingTrace trace;
    bool setup_done = false;
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_status = 0;
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        g_status = static_cast<int>(e.code()) + 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_status = static_cast<int>(ErrorCode::internal) + 1;
    }
    return g_status;
}

// Owned rows of the stencil operator on an nx*ny*nz grid, global columns
// ascending (27-point uses 26/-1, SURVEY 8c restatement 1).
CsrMatrix gen_rows(int stencil, index_t nx, index_t ny, index_t nz, index_t begin, index_t end) {
    CsrMatrix L(end - begin, nx * ny * nz);
    const int r = 1;
    L.col_idx.reserve(static_cast<std::size_t>((end - begin) * (stencil == 27 ? 27 : 7)));
    L.values.reserve(L.col_idx.capacity());
    for (index_t row = begin; row < end; ++row) {
        const index_t i = row % nx, j = (row / nx) % ny, k = row / (nx * ny);
        for (int dk = -r; dk <= r; ++dk)
            for (int dj = -r; dj <= r; ++dj)
                for (int di = -r; di <= r; ++di) {
                    const int manhattan = std::abs(di) + std::abs(dj) + std::abs(dk);
                    if (stencil == 7 && manhattan > 1) continue;
                    const index_t ii = i + di, jj = j + dj, kk = k + dk;
                    if (ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz) continue;
                    L.col_idx.push_back(ii + nx * (jj + ny * kk));
                    L.values.push_back(manhattan == 0 ? (stencil == 27 ? 26.0 : 6.0) : -1.0);
                }
        L.row_ptr[row - begin + 1] = static_cast<index_t>(L.col_idx.size());
    }
    return L;
}

template <typename F>
void run(Session& s, F&& program) {
    RuntimeOptions opts;
    opts.nranks = s.cfg.nranks;
    opts.deadlock_timeout = std::chrono::milliseconds(600000);
    spawn_ranks(opts, program);
}

SetupConfig setup_cfg(Session& s, bool record) {
    SetupConfig c;
    c.aggregation_exponent = s.cfg.aggregation_exponent;
    c.coarse_size_target = s.cfg.coarse_size_target;
    c.max_levels = s.cfg.max_levels;
    c.record = record ? &s.trace : nullptr;
    return c;
}

CycleConfig cycle_cfg(const Session& s) {
    CycleConfig c;
    c.pre_sweeps = s.cfg.pre_sweeps;
    c.post_sweeps = s.cfg.post_sweeps;
    c.coarsest_sweeps = s.cfg.coarsest_sweeps;
    c.relax_weight = s.cfg.relax_weight;
    return c;
}

void init_session(Session& s) {
    if (s.cfg.matching_mode != 0)
        throw Error(ErrorCode::invalid_argument,
                    "reference driver: only the reference strict-weight matching exists");
    s.ranks.resize(static_cast<std::size_t>(s.cfg.nranks));
    const Partition part = Partition::uniform(s.n, s.cfg.nranks);
    run(s, [&](RankCtx& ctx) {
        RankState& st = s.ranks[ctx.rank()];
        st.A.part = part;
        st.A.global_ncols = s.n;
        if (s.cfg.stencil == 0)
            st.A = distribute_matrix(ctx, s.global, part);
        else
            st.A.local = gen_rows(s.cfg.stencil, s.cfg.nx, s.cfg.ny, s.cfg.nz, part.begin(ctx.rank()),
                                  part.end(ctx.rank()));
        st.b = DistVector::constant(part, ctx, 1.0);
        st.w0 = DistVector::constant(part, ctx, 1.0);
    });
}

// Assemble a level-k global object on the caller from per-rank pieces.
void gather_rows(const std::vector<const CsrMatrix*>& blocks, int64_t* row_ptr, int64_t* col,
                 double* val) {
    int64_t row = 0, off = 0;
    if (row_ptr) row_ptr[0] = 0;
    for (const CsrMatrix* B : blocks) {
        for (index_t i = 0; i < B->nrows; ++i) {
            for (index_t t = B->row_ptr[i]; t < B->row_ptr[i + 1]; ++t) {
                if (col) col[off] = B->col_idx[t];
                if (val) val[off] = B->values[t];
                ++off;
            }
            ++row;
            if (row_ptr) row_ptr[row] = off;
        }
    }
}

Session* S(void* h) {
    if (!h) throw Error(ErrorCode::invalid_argument, "null session");
    return static_cast<Session*>(h);
}

Session* S_setup(void* h) {
    Session* s = S(h);
    if (!s->setup_done) throw Error(ErrorCode::contract_violation, "setup not run");
    return s;
}

}  // namespace

extern "C" {

void orc_default_config(orc_config* c) {
    std::memset(c, 0, sizeof *c);
    c->stencil = 7;
    c->nx = c->ny = c->nz = 16;
    c->nranks = 1;
    c->aggregation_exponent = 3;
    c->coarse_size_target = 40;
    c->max_levels = 40;
    c->matching_mode = 0;
    c->pre_sweeps = 4;
    c->post_sweeps = 4;
    c->coarsest_sweeps = 20;
    c->relax_weight = 1.0;
    c->rtol = 1e-6;
    c->max_iters = 1000;
    c->precflag = 1;
    c->threads = 1;
}

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_last_status(void) { return g_status; }

void* orc_create(const orc_config* cfg) {
    Session* s = nullptr;
    const int rc = guarded([&] {
        auto up = std::make_unique<Session>();
        up->cfg = *cfg;
        if (cfg->stencil != 7 && cfg->stencil != 27)
            throw Error(ErrorCode::invalid_argument, "stencil must be 7 or 27");
        up->n = cfg->nx * cfg->ny * cfg->nz;
        init_session(*up);
        s = up.release();
    });
    return rc == 0 ? s : nullptr;
}

void* orc_create_csr(const orc_config* cfg, int64_t n, const int64_t* row_ptr, const int64_t* col,
                     const double* val) {
    Session* s = nullptr;
    const int rc = guarded([&] {
        auto up = std::make_unique<Session>();
        up->cfg = *cfg;
        up->cfg.stencil = 0;
        up->n = n;
        up->global = CsrMatrix(n, n);
        for (index_t i = 0; i <= n; ++i) up->global.row_ptr[i] = row_ptr[i];
        up->global.col_idx.assign(col, col + row_ptr[n]);
        up->global.values.assign(val, val + row_ptr[n]);
        up->global.validate();
        init_session(*up);
        s = up.release();
    });
    return rc == 0 ? s : nullptr;
}

void orc_destroy(void* h) { delete static_cast<Session*>(h); }

int64_t orc_global_n(void* h) { return S(h)->n; }

int64_t orc_global_nnz(void* h) {
    int64_t nnz = 0;
    for (const auto& r : S(h)->ranks) nnz += r.A.local.nnz();
    return nnz;
}

int orc_export_input(void* h, int64_t* row_ptr, int64_t* col, double* val) {
    return guarded([&] {
        Session* s = S(h);
        std::vector<const CsrMatrix*> blocks;
        for (const auto& r : s->ranks) blocks.push_back(&r.A.local);
        gather_rows(blocks, row_ptr, col, val);
    });
}

int orc_setup(void* h) {
    return guarded([&] {
        Session* s = S(h);
        s->trace.steps.clear();
        run(*s, [&](RankCtx& ctx) {
            RankState& st = s->ranks[ctx.rank()];
            st.h = setup_hierarchy(ctx, st.A, st.w0, setup_cfg(*s, true));
        });
        s->setup_done = true;
    });
}

int orc_num_levels(void* h) {
    Session* s = S(h);
    return s->setup_done ? s->ranks[0].h.nl() : 0;
}

double orc_opc(void* h) { return S(h)->ranks[0].h.opc; }

int orc_get_setup_stats(void* h, orc_setup_stats* out) {
    return guarded([&] {
        Session* s = S_setup(h);
        // Rank 0's timers (all ranks run in lock-step).
        const SetupStats& st = s->ranks[0].h.stats;
        out->t_total = st.t_total;
        out->t_matching = st.t_matching;
        out->t_spmm = st.t_spmm;
        out->t_spmm_comm = st.t_spmm_comm;
        out->matching_messages = 0;
        out->rc_messages = 0;
        for (const auto& r : s->ranks) {
            out->matching_messages += r.h.stats.matching_messages;
            out->rc_messages += r.h.stats.rc_messages;
        }
    });
}

int orc_level_size(void* h, int level, int64_t* n, int64_t* nnz) {
    return guarded([&] {
        Session* s = S_setup(h);
        const Hierarchy& H = s->ranks[0].h;
        if (level < 0 || level >= H.nl()) throw Error(ErrorCode::invalid_argument, "level");
        *n = H.level_sizes[level];
        *nnz = H.level_nnz[level];
    });
}

int orc_level_partition(void* h, int level, int64_t* starts) {
    return guarded([&] {
        Session* s = S_setup(h);
        const Partition& p = s->ranks[0].h.levels.at(level).A.part;
        for (std::size_t r = 0; r < p.starts.size(); ++r) starts[r] = p.starts[r];
    });
}

int orc_export_level(void* h, int level, int64_t* row_ptr, int64_t* col, double* val, double* w,
                     double* l1) {
    return guarded([&] {
        Session* s = S_setup(h);
        std::vector<const CsrMatrix*> blocks;
        int64_t off = 0;
        for (const auto& r : s->ranks) {
            const Level& L = r.h.levels.at(level);
            blocks.push_back(&L.A.local);
            for (std::size_t i = 0; i < L.w.local.size(); ++i) {
                if (w) w[off + i] = L.w.local[i];
                if (l1) l1[off + i] = L.m_l1.local[i];
            }
            off += static_cast<int64_t>(L.w.local.size());
        }
        gather_rows(blocks, row_ptr, col, val);
    });
}

int orc_export_prolongator(void* h, int level, int64_t* col, double* val) {
    return guarded([&] {
        Session* s = S_setup(h);
        if (level < 1) throw Error(ErrorCode::invalid_argument, "prolongator level must be >= 1");
        std::vector<const CsrMatrix*> blocks;
        for (const auto& r : s->ranks) blocks.push_back(&r.h.levels.at(level).P_block);
        for (const CsrMatrix* B : blocks)
            for (index_t i = 0; i < B->nrows; ++i)
                if (B->row_ptr[i + 1] - B->row_ptr[i] != 1)
                    throw Error(ErrorCode::internal, "prolongator row without exactly one entry");
        gather_rows(blocks, nullptr, col, val);
    });
}

int orc_num_matchings(void* h) { return static_cast<int>(S(h)->trace.steps.size()); }

int64_t orc_matching_size(void* h, int step) {
    Session* s = S(h);
    if (step < 0 || step >= static_cast<int>(s->trace.steps.size())) return -1;
    return static_cast<int64_t>(s->trace.steps[static_cast<std::size_t>(step)].size());
}

int orc_export_matching(void* h, int step, int64_t* mate) {
    return guarded([&] {
        Session* s = S_setup(h);
        const auto& m = s->trace.steps.at(static_cast<std::size_t>(step));
        std::copy(m.begin(), m.end(), mate);
    });
}

int orc_spmv(void* h, int level, const double* x, double* y) {
    return guarded([&] {
        Session* s = S_setup(h);
        run(*s, [&](RankCtx& ctx) {
            const Level& L = s->ranks[ctx.rank()].h.levels.at(level);
            const index_t b = L.A.part.begin(ctx.rank());
            DistVector xv{L.A.part, std::vector<real_t>(x + b, x + L.A.part.end(ctx.rank()))};
            DistVector yv = spmv_dist(ctx, L.A, xv, *L.spmv_plan, true);
            std::copy(yv.local.begin(), yv.local.end(), y + b);
        });
    });
}

int orc_vcycle(void* h, const double* r, double* x) {
    return guarded([&] {
        Session* s = S_setup(h);
        const CycleConfig cc = cycle_cfg(*s);
        run(*s, [&](RankCtx& ctx) {
            const Hierarchy& H = s->ranks[ctx.rank()].h;
            const Partition& part = H.levels[0].A.part;
            const index_t b = part.begin(ctx.rank());
            DistVector rv{part, std::vector<real_t>(r + b, r + part.end(ctx.rank()))};
            DistVector xv = vcycle_apply(ctx, H, cc, rv, 0);
            std::copy(xv.local.begin(), xv.local.end(), x + b);
        });
    });
}

// Notay flexible PCG, PAPER.md:86-115 (Algorithm 1).
// Iteration k is counted when r_k is formed; stop at the first k with
// |r_k|/|r_0| < rtol (r_1 after the initialisation block is k = 1) or at
// max_iters.  Per iteration: one V-cycle, one SpMV, one reduction of the
// dot triple (alpha, beta, gamma), the rho update and four vector updates.
// Vector-update operation order (also used by the CUDA path):
//   d = w - (gamma/rho_prev) d;  q = v - (gamma/rho_prev) q;
//   u = u + (alpha/rho) d;       r = r - (alpha/rho) q.
int64_t orc_build_weights(int64_t n, const int64_t* rp, const int64_t* col, const double* val,
                          const double* w, int64_t* grp, int64_t* gcol, double* gw) {
    int64_t out = -1;
    guarded([&] {
        CsrMatrix B(n, n);
        for (index_t i = 0; i <= n; ++i) B.row_ptr[i] = rp[i];
        B.col_idx.assign(col, col + rp[n]);
        B.values.assign(val, val + rp[n]);
        const WeightedGraph g = build_weights(B, std::span<const real_t>(w, static_cast<std::size_t>(n)));
        for (index_t i = 0; i <= n; ++i) grp[i] = g.adj.row_ptr[i];
        std::copy(g.adj.col_idx.begin(), g.adj.col_idx.end(), gcol);
        std::copy(g.adj.values.begin(), g.adj.values.end(), gw);
        out = g.adj.nnz();
    });
    return out;
}

int orc_match_graph(int64_t n, const int64_t* rp, const int64_t* col, const double* w, int mode,
                    int64_t* mate) {
    return guarded([&] {
        if (mode != 0)
            throw Error(ErrorCode::invalid_argument, "reference suitor has only the strict acceptor");
        WeightedGraph g;
        g.n = n;
        g.adj = CsrMatrix(n, n);
        for (index_t i = 0; i <= n; ++i) g.adj.row_ptr[i] = rp[i];
        g.adj.col_idx.assign(col, col + rp[n]);
        g.adj.values.assign(w, w + rp[n]);
        const Matching m = suitor_match(g);
        std::copy(m.mate.begin(), m.mate.end(), mate);
    });
}

int orc_set_solve(void* h, double rtol, int max_iters) {
    return guarded([&] {
        Session* s = S(h);
        s->cfg.rtol = rtol;
        s->cfg.max_iters = max_iters;
    });
}

int orc_solve(void* h, const double* b, double* u, double* hist, int hist_cap, int* iters,
              double* relres, double* t_solve) {
    return guarded([&] {
        Session* s = S(h);
        if (s->cfg.precflag && !s->setup_done)
            throw Error(ErrorCode::contract_violation, "setup not run");
        const CycleConfig cc = cycle_cfg(*s);
        std::vector<double> history;
        int it_out = 0;
        double rel_out = 0.0;
        const auto t0 = std::chrono::steady_clock::now();
        run(*s, [&](RankCtx& ctx) {
            RankState& st = s->ranks[ctx.rank()];
            const Partition& part = st.A.part;
            const index_t beg = part.begin(ctx.rank());
            const std::size_t nl = static_cast<std::size_t>(part.extent(ctx.rank()));
            const HaloPlan& plan =
                s->cfg.precflag ? *st.h.levels[0].spmv_plan : ensure_spmv_plan(ctx, st.A);
            const DistMatrix& A = s->cfg.precflag ? st.h.levels[0].A : st.A;
            DistVector bv = b ? DistVector{part, std::vector<real_t>(b + beg, b + beg + nl)} : st.b;
            DistVector uu = DistVector::zeros(part, ctx);
            auto apply_B = [&](const DistVector& r) {
                return s->cfg.precflag ? vcycle_apply(ctx, st.h, cc, r, 0) : r;
            };
            // r0 = b - A u0
            DistVector r = spmv_dist(ctx, A, uu, plan, true);
            for (std::size_t i = 0; i < nl; ++i) r.local[i] = bv.local[i] - r.local[i];
            const double rnorm0 = norm2_dist(ctx, r);
            std::vector<double> hloc{1.0};
            int k = 0;
            double rel = 1.0;
            if (rnorm0 != 0.0) {
                DistVector w = apply_B(r);
                DistVector d = w;
                DistVector v = spmv_dist(ctx, A, w, plan, true);
                DistVector q = v;
                const double alpha = dot_dist(ctx, w, r);
                double rho = dot_dist(ctx, w, v);
                if (rho == 0.0 || !std::isfinite(rho))
                    throw Error(ErrorCode::breakdown, "fcg: breakdown at iteration 0");
                const double a0 = alpha / rho;
                for (std::size_t i = 0; i < nl; ++i) {
                    uu.local[i] = uu.local[i] + a0 * d.local[i];
                    r.local[i] = r.local[i] - a0 * q.local[i];
                }
                k = 1;
                rel = norm2_dist(ctx, r) / rnorm0;
                hloc.push_back(rel);
                while (!(rel < s->cfg.rtol) && k < s->cfg.max_iters) {
                    w = apply_B(r);
                    spmv_dist(ctx, A, w, plan, true, v);
                    const double al = dot_dist(ctx, w, r);
                    const double be = dot_dist(ctx, w, v);
                    const double ga = dot_dist(ctx, w, q);
                    const double rho_new = be - ga * ga / rho;
                    if (rho_new == 0.0 || !std::isfinite(rho_new))
                        throw Error(ErrorCode::breakdown,
                                    "fcg: breakdown at iteration " + std::to_string(k));
                    const double c = ga / rho;
                    const double a = al / rho_new;
                    for (std::size_t i = 0; i < nl; ++i) {
                        d.local[i] = w.local[i] - c * d.local[i];
                        q.local[i] = v.local[i] - c * q.local[i];
                        uu.local[i] = uu.local[i] + a * d.local[i];
                        r.local[i] = r.local[i] - a * q.local[i];
                    }
                    rho = rho_new;
                    ++k;
                    rel = norm2_dist(ctx, r) / rnorm0;
                    hloc.push_back(rel);
                }
            }
            if (u) std::copy(uu.local.begin(), uu.local.end(), u + beg);
            if (ctx.rank() == 0) {
                history = hloc;
                it_out = k;
                rel_out = rel;
            }
        });
        const double dt =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (t_solve) *t_solve = dt;
        if (iters) *iters = it_out;
        if (relres) *relres = rel_out;
        if (hist)
            for (int i = 0; i < hist_cap && i < static_cast<int>(history.size()); ++i)
                hist[i] = history[i];
    });
}


void* orc_mm_load(const char* path) {
    CsrMatrix* out = nullptr;
    guarded([&] { out = new CsrMatrix(read_matrix_market(std::string(path))); });
    return out;
}

void orc_mm_info(void* m, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
    const CsrMatrix& A = *static_cast<CsrMatrix*>(m);
    *nrows = A.nrows;
    *ncols = A.ncols;
    *nnz = static_cast<int64_t>(A.col_idx.size());
}

void orc_mm_export(void* m, int64_t* row_ptr, int64_t* col, double* val) {
    const CsrMatrix& A = *static_cast<CsrMatrix*>(m);
    std::memcpy(row_ptr, A.row_ptr.data(), 8 * A.row_ptr.size());
    std::memcpy(col, A.col_idx.data(), 8 * A.col_idx.size());
    std::memcpy(val, A.values.data(), 8 * A.values.size());
}

void orc_mm_free(void* m) { delete static_cast<CsrMatrix*>(m); }

void* orc_spgemm(int64_t an, int64_t am, const int64_t* a_rp, const int64_t* a_col, const double* a_val, int64_t bm,
                 const int64_t* b_rp, const int64_t* b_col, const double* b_val) {
    CsrMatrix* out = nullptr;
    guarded([&] {
        CsrMatrix A(an, am), B(am, bm);
        A.row_ptr.assign(a_rp, a_rp + an + 1);
        A.col_idx.assign(a_col, a_col + a_rp[an]);
        A.values.assign(a_val, a_val + a_rp[an]);
        B.row_ptr.assign(b_rp, b_rp + am + 1);
        B.col_idx.assign(b_col, b_col + b_rp[am]);
        B.values.assign(b_val, b_val + b_rp[am]);
        out = new CsrMatrix(spgemm_local(A, B));
    });
    return out;
}

int orc_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_ptr, const int64_t* col,
                 const double* val) {
    return guarded([&] {
        CsrMatrix A(nrows, ncols);
        A.row_ptr.assign(row_ptr, row_ptr + nrows + 1);
        A.col_idx.assign(col, col + row_ptr[nrows]);
        A.values.assign(val, val + row_ptr[nrows]);
        write_matrix_market(std::string(path), A);
    });
}

}  // extern "C"
