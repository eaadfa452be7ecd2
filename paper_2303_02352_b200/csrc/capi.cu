// capi.cu -- the extern "C" boundary (include/pairamg_b200.h).  Every entry
// point converts pb::Error / CUDA / NCCL failures into a pairamg_status and a
// thread-local message, mirroring the reference's exception-carrying
// ErrorCode (types.hpp:13-35) and the absent capi.cpp (src/CMakeLists.txt:20).
#include <cub/cub.cuh>

#include <cstring>
#include <set>
#include <string>

#include "mmio.cuh"
#include "pairamg_b200.h"
#include "spgemm.cuh"
#include "solver.cuh"

struct pairamg_solver;
struct pairamg_runtime {
    std::unique_ptr<pb::Runtime> rt;
    std::set<pairamg_solver*> solvers;  // live solvers: released before the runtime goes
};

struct pairamg_solver {
    pairamg_runtime* rt = nullptr;
    std::unique_ptr<pb::Solver> s;
};

namespace {

thread_local std::string g_err;

template <typename F>
pairamg_status guarded(F&& f) {
    try {
        f();
        return PAIRAMG_OK;
    } catch (const pb::Error& e) {
        g_err = e.what();
        return e.code();
    } catch (const std::bad_alloc& e) {
        g_err = std::string("out of memory: ") + e.what();
        return PAIRAMG_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PAIRAMG_INTERNAL;
    }
}

pb::Solver& S(pairamg_solver* s) {
    if (!s) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null solver");
    if (!s->s) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "solver used after its runtime was destroyed");
    PB_CUDA(cudaSetDevice(s->rt->rt->device()));
    return *s->s;
}

pb::SetupConfig setup_cfg(const pairamg_setup_config* c) {
    pb::SetupConfig o;
    if (c) {
        o.aggregation_exponent = c->aggregation_exponent;
        o.coarse_size_target = c->coarse_size_target;
        o.max_levels = c->max_levels;
        if (c->replay_steps < 0) pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: replay_steps must be >= 0");
        if (c->replay_steps > 0 && (!c->replay_mates || !c->replay_sizes))
            pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: replay_steps > 0 needs replay_mates and replay_sizes");
        for (int t = 0; t < c->replay_steps; ++t) {
            o.replay.push_back(c->replay_mates[t]);
            o.replay_sizes.push_back(c->replay_sizes[t]);
        }
        if (c->storage < PAIRAMG_STORAGE_AUTO || c->storage > PAIRAMG_STORAGE_CODED)
            pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: unknown storage format " + std::to_string(c->storage));
        o.storage = c->storage;
        if (c->replicate_rows < 0) pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: replicate_rows must be >= 0");
        o.replicate_rows = c->replicate_rows;
        o.setup_overlap = c->setup_overlap != 0;
    }
    return o;
}

pb::CycleConfig cycle_cfg(const pairamg_cycle_config* c) {
    pb::CycleConfig o;
    if (c) {
        o.pre_sweeps = c->pre_sweeps;
        o.post_sweeps = c->post_sweeps;
        o.coarsest_sweeps = c->coarsest_sweeps;
        o.relax_weight = c->relax_weight;
    }
    return o;
}

// CsrMatrix::validate (csr.cpp:56-78) on the device: row_ptr[0] == 0,
// non-decreasing, columns strictly increasing and in [0, ncols).
__global__ void k_validate(const int64_t* __restrict__ rp, const int64_t* __restrict__ col, int64_t n,
                           int64_t ncols, unsigned long long* __restrict__ bad_row) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = rp[i], e = rp[i + 1];
    bool ok = (i > 0 || b == 0) && b <= e;
    for (int64_t t = b; ok && t < e; ++t) {
        const int64_t c = col[t];
        if (c < 0 || c >= ncols || (t > b && col[t - 1] >= c)) ok = false;
    }
    if (!ok) atomicMin(bad_row, static_cast<unsigned long long>(i));
}

void check_partition(const pb::Runtime& rt, int64_t global_n, const int64_t* starts, int64_t n_local) {
    if (!starts) pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: part_starts is null");
    const int p = rt.nranks();
    if (starts[0] != 0 || starts[p] != global_n)
        pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup: partition does not span [0, global_n)");
    for (int r = 0; r < p; ++r)
        if (starts[r + 1] < starts[r]) pb::fail(PAIRAMG_INVALID_ARGUMENT, "partition: negative block size");
    if (starts[rt.rank() + 1] - starts[rt.rank()] != n_local)
        pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup: n_local does not match the partition extent");
}

void setup_impl(pairamg_solver* s, int64_t global_n, const int64_t* starts, int64_t n_local, int64_t nnz,
                pb::DBuf<int64_t>&& rp, pb::DBuf<int64_t>&& col, pb::DBuf<double>&& val, const double* d_w0,
                const pairamg_setup_config* cfg) {
    pb::Solver& sv = S(s);
    cudaStream_t st = sv.rt.stream();
    check_partition(sv.rt, global_n, starts, n_local);
    if (n_local > 0) {
        pb::DBuf<unsigned long long> bad(1, st);
        PB_CUDA(cudaMemsetAsync(bad.get(), 0xff, 8, st));
        k_validate<<<pb::blocks_for(n_local, 256), 256, 0, st>>>(rp.get(), col.get(), n_local, global_n, bad.get());
        PB_CHECK_LAUNCH();
        unsigned long long h = 0;
        int64_t last = 0;
        PB_CUDA(cudaMemcpyAsync(&h, bad.get(), 8, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaMemcpyAsync(&last, rp.get() + n_local, 8, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaStreamSynchronize(st));
        if (h != ~0ULL)
            pb::fail(PAIRAMG_CONTRACT_VIOLATION, "csr: invalid row " + std::to_string(h) +
                                                     " (row_ptr order, or columns not strictly increasing / out of range)");
        if (last != nnz) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "csr: row_ptr[nrows] != nnz");
    }
    std::vector<int64_t> part(starts, starts + sv.rt.nranks() + 1);
    sv.setup(std::move(part), std::move(rp), std::move(col), std::move(val), nnz, d_w0, setup_cfg(cfg));
}

// ---- Poisson generator ----
__host__ __device__ inline int row_len(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t row) {
    const int64_t i = row % nx, j = (row / nx) % ny, k = row / (nx * ny);
    const int ax = 1 + (i > 0) + (i < nx - 1), ay = 1 + (j > 0) + (j < ny - 1), az = 1 + (k > 0) + (k < nz - 1);
    return stencil == 27 ? ax * ay * az : 1 + (ax - 1) + (ay - 1) + (az - 1);
}

// Variable-coefficient operator (a workload for the general storage paths,
// no reference counterpart): cell coefficient k_c from a hash of (seed, c) --
// 1 + (h mod levels) for levels > 0 (few distinct entry values), else a
// continuous value in [0.5, 1.5) (every value distinct).  Coupling of
// neighbours i, j: -(k_i + k_j)/2; diagonal: the sum over all stencil
// directions of (k_i + k_j)/2, with k_i for directions leaving the grid
// (Dirichlet), in direction order -- an SPD M-matrix.  levels < 0 = Poisson.
struct Coef {
    int levels = -1;
    uint64_t seed = 0;
};

__host__ __device__ inline double cell_coef(int64_t c, const Coef& cf) {
    uint64_t z = cf.seed + 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(c + 1);  // splitmix64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    if (cf.levels > 0) return 1.0 + static_cast<double>(z % static_cast<uint64_t>(cf.levels));
    return 0.5 + static_cast<double>(z >> 11) * 0x1p-53;
}

__host__ __device__ inline void fill_row(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t row,
                                         int64_t* col, double* val, Coef cf = Coef()) {
    const int64_t i = row % nx, j = (row / nx) % ny, k = row / (nx * ny);
    const bool var = cf.levels >= 0;
    const double ki = var ? cell_coef(row, cf) : 0.0;
    double diag = 0.0;
    int o = 0, od = 0;
    for (int dk = -1; dk <= 1; ++dk)
        for (int dj = -1; dj <= 1; ++dj)
            for (int di = -1; di <= 1; ++di) {
                const int man = (di != 0) + (dj != 0) + (dk != 0);
                if (stencil == 7 && man > 1) continue;
                const int64_t ii = i + di, jj = j + dj, kk = k + dk;
                const bool in = !(ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz);
                if (var && man > 0) {
                    const double c = in ? (ki + cell_coef(ii + nx * (jj + ny * kk), cf)) * 0.5 : ki;
                    diag = diag + c;
                    if (in) val[o] = -c;
                }
                if (!in) continue;
                col[o] = ii + nx * (jj + ny * kk);
                if (man == 0) od = o;
                if (!var) val[o] = man == 0 ? (stencil == 27 ? 26.0 : 6.0) : -1.0;
                ++o;
            }
    if (var) val[od] = diag;
}

__global__ void k_poisson_len(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t b, int64_t m,
                              int64_t* __restrict__ rp) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < m) rp[r] = row_len(stencil, nx, ny, nz, b + r);
    if (r == m) rp[m] = 0;
}

__global__ void k_poisson_fill(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t b, int64_t m,
                               const int64_t* __restrict__ rp, int64_t* __restrict__ col, double* __restrict__ val,
                               Coef cf) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < m) fill_row(stencil, nx, ny, nz, b + r, col + rp[r], val + rp[r], cf);
}

void generate_host(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t b, int64_t e, int64_t* row_ptr,
                   int64_t* col, double* val, Coef cf) {
    if (stencil != 7 && stencil != 27) pb::fail(PAIRAMG_INVALID_ARGUMENT, "stencil must be 7 or 27");
    if (b < 0 || e < b || e > nx * ny * nz) pb::fail(PAIRAMG_INVALID_ARGUMENT, "row range");
    row_ptr[0] = 0;
    for (int64_t r = b; r < e; ++r) {
        fill_row(stencil, nx, ny, nz, r, col + row_ptr[r - b], val + row_ptr[r - b], cf);
        row_ptr[r - b + 1] = row_ptr[r - b] + row_len(stencil, nx, ny, nz, r);
    }
}

void generate_device(pairamg_runtime* rt, int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t b, int64_t e,
                     int64_t* d_rp, int64_t* d_col, double* d_val, Coef cf) {
    if (!rt) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null runtime");
    if (stencil != 7 && stencil != 27) pb::fail(PAIRAMG_INVALID_ARGUMENT, "stencil must be 7 or 27");
    if (b < 0 || e < b || e > nx * ny * nz) pb::fail(PAIRAMG_INVALID_ARGUMENT, "row range");
    PB_CUDA(cudaSetDevice(rt->rt->device()));
    cudaStream_t st = rt->rt->stream();
    const int64_t m = e - b;
    k_poisson_len<<<pb::blocks_for(m + 1, 256), 256, 0, st>>>(stencil, nx, ny, nz, b, m, d_rp);
    PB_CHECK_LAUNCH();
    size_t bytes = 0;
    PB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, d_rp, d_rp, m + 1, st));
    pb::DBuf<uint8_t> tmp(bytes ? bytes : 1, st);
    PB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, d_rp, d_rp, m + 1, st));
    if (m) k_poisson_fill<<<pb::blocks_for(m, 256), 256, 0, st>>>(stencil, nx, ny, nz, b, m, d_rp, d_col, d_val, cf);
    PB_CHECK_LAUNCH();
    PB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

extern "C" {

void pairamg_default_setup_config(pairamg_setup_config* c) {
    std::memset(c, 0, sizeof *c);
    c->aggregation_exponent = 3;
    c->coarse_size_target = 40;
    c->max_levels = 40;
    c->replay_steps = 0;
    c->replay_mates = nullptr;
    c->replay_sizes = nullptr;
    c->storage = PAIRAMG_STORAGE_AUTO;
    c->replicate_rows = 2500000;
    c->setup_overlap = 0;
}

void pairamg_default_cycle_config(pairamg_cycle_config* c) {
    c->pre_sweeps = 4;
    c->post_sweeps = 4;
    c->coarsest_sweeps = 20;
    c->relax_weight = 1.0;
}

void pairamg_default_solve_config(pairamg_solve_config* c) {
    c->rtol = 1e-6;
    c->max_iters = 1000;
    c->precflag = 1;
}

const char* pairamg_status_name(pairamg_status s) {
    switch (s) {  // error_code_name (types.hpp:37-51)
        case PAIRAMG_OK: return "ok";
        case PAIRAMG_INVALID_ARGUMENT: return "invalid_argument";
        case PAIRAMG_CONTRACT_VIOLATION: return "contract_violation";
        case PAIRAMG_MISSING_ROW: return "missing_row";
        case PAIRAMG_SINGULAR_SMOOTHER: return "singular_smoother";
        case PAIRAMG_STAGNATION: return "stagnation";
        case PAIRAMG_BREAKDOWN: return "breakdown";
        case PAIRAMG_DEADLOCK: return "deadlock";
        case PAIRAMG_PARSE_ERROR: return "parse_error";
        case PAIRAMG_IO_ERROR: return "io_error";
        case PAIRAMG_INTERNAL: return "internal";
    }
    return "unknown";
}

const char* pairamg_last_error(void) { return g_err.c_str(); }
int pairamg_abi_version(void) { return PAIRAMG_B200_ABI_VERSION; }

pairamg_status pairamg_comm_local_id(uint8_t id[128]) {
    return guarded([&] {
        if (!id) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null id");
        pb::make_local_id(id);
    });
}

pairamg_status pairamg_comm_unique_id(uint8_t id[128]) {
    return guarded([&] {
        ncclUniqueId uid;
        PB_NCCL(ncclGetUniqueId(&uid));
        std::memcpy(id, uid.internal, 128);
    });
}

pairamg_status pairamg_runtime_create(int device, int rank, int nranks, const uint8_t* id, pairamg_runtime** out) {
    return guarded([&] {
        if (!out) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null out");
        auto r = std::make_unique<pairamg_runtime>();
        r->rt = std::make_unique<pb::Runtime>(device, rank, nranks, id);
        *out = r.release();
    });
}

// Either destruction order is safe: destroying a runtime first releases the
// device state of every solver created on it (the handles stay valid, later
// calls fail with CONTRACT_VIOLATION, pairamg_solver_destroy frees them).
pairamg_status pairamg_runtime_destroy(pairamg_runtime* rt) {
    return guarded([&] {
        if (!rt) return;
        if (rt->rt) cudaSetDevice(rt->rt->device());
        for (pairamg_solver* s : rt->solvers) {
            s->s.reset();
            s->rt = nullptr;
        }
        delete rt;
    });
}

pairamg_status pairamg_solver_create(pairamg_runtime* rt, pairamg_solver** out) {
    return guarded([&] {
        if (!rt || !out) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null runtime/out");
        PB_CUDA(cudaSetDevice(rt->rt->device()));
        auto s = std::make_unique<pairamg_solver>();
        s->rt = rt;
        s->s = std::make_unique<pb::Solver>(*rt->rt);
        rt->solvers.insert(s.get());
        *out = s.release();
    });
}

pairamg_status pairamg_solver_destroy(pairamg_solver* s) {
    return guarded([&] {
        if (s && s->rt) {
            cudaSetDevice(s->rt->rt->device());
            s->rt->solvers.erase(s);
        }
        delete s;
    });
}

pairamg_status pairamg_setup(pairamg_solver* s, int64_t global_n, const int64_t* part_starts, int64_t n_local,
                             const int64_t* row_ptr, const int64_t* col_idx, const double* values, const double* w0,
                             const pairamg_setup_config* cfg) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (n_local < 0 || !row_ptr) pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: bad CSR arguments");
        cudaStream_t st = sv.rt.stream();
        const int64_t nnz = row_ptr[n_local];
        if (nnz < 0 || (nnz > 0 && (!col_idx || !values)))
            pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: bad CSR arguments");
        pb::DBuf<int64_t> rp(static_cast<size_t>(n_local + 1), st), col(static_cast<size_t>(nnz), st);
        pb::DBuf<double> val(static_cast<size_t>(nnz), st), w(w0 ? static_cast<size_t>(n_local) : 0, st);
        PB_CUDA(cudaMemcpyAsync(rp.get(), row_ptr, 8 * (n_local + 1), cudaMemcpyHostToDevice, st));
        if (nnz) {
            PB_CUDA(cudaMemcpyAsync(col.get(), col_idx, 8 * nnz, cudaMemcpyHostToDevice, st));
            PB_CUDA(cudaMemcpyAsync(val.get(), values, 8 * nnz, cudaMemcpyHostToDevice, st));
        }
        if (w0 && n_local) PB_CUDA(cudaMemcpyAsync(w.get(), w0, 8 * n_local, cudaMemcpyHostToDevice, st));
        setup_impl(s, global_n, part_starts, n_local, nnz, std::move(rp), std::move(col), std::move(val),
                   w0 ? w.get() : nullptr, cfg);
    });
}

pairamg_status pairamg_setup_device(pairamg_solver* s, int64_t global_n, const int64_t* part_starts, int64_t n_local,
                                    int64_t nnz_local, const int64_t* d_row_ptr, const int64_t* d_col_idx,
                                    const double* d_values, const double* d_w0, const pairamg_setup_config* cfg) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        cudaStream_t st = sv.rt.stream();
        if (n_local < 0 || nnz_local < 0) pb::fail(PAIRAMG_INVALID_ARGUMENT, "setup: bad sizes");
        pb::DBuf<int64_t> rp(static_cast<size_t>(n_local + 1), st), col(static_cast<size_t>(nnz_local), st);
        pb::DBuf<double> val(static_cast<size_t>(nnz_local), st);
        PB_CUDA(cudaMemcpyAsync(rp.get(), d_row_ptr, 8 * (n_local + 1), cudaMemcpyDeviceToDevice, st));
        if (nnz_local) {
            PB_CUDA(cudaMemcpyAsync(col.get(), d_col_idx, 8 * nnz_local, cudaMemcpyDeviceToDevice, st));
            PB_CUDA(cudaMemcpyAsync(val.get(), d_values, 8 * nnz_local, cudaMemcpyDeviceToDevice, st));
        }
        setup_impl(s, global_n, part_starts, n_local, nnz_local, std::move(rp), std::move(col), std::move(val), d_w0,
                   cfg);
    });
}

pairamg_status pairamg_solve_device(pairamg_solver* s, const double* d_b, double* d_u, const pairamg_cycle_config* ccfg,
                                    const pairamg_solve_config* scfg, pairamg_solve_stats* stats) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        pairamg_solve_config sc;
        pairamg_default_solve_config(&sc);
        if (scfg) sc = *scfg;
        sv.solve(d_b, d_u, cycle_cfg(ccfg), sc.rtol, sc.max_iters, sc.precflag != 0, stats);
    });
}

pairamg_status pairamg_solve(pairamg_solver* s, const double* b, double* u, const pairamg_cycle_config* ccfg,
                             const pairamg_solve_config* scfg, pairamg_solve_stats* stats) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "solve: setup not run");
        cudaStream_t st = sv.rt.stream();
        const int64_t n = sv.h.levels[0]->A.n;
        pb::DBuf<double> db(static_cast<size_t>(n), st), du(static_cast<size_t>(n), st);
        // the copies are timed on the solver stream (events), apart from the solve
        cudaEvent_t ev[4];
        for (auto& e : ev) PB_CUDA(cudaEventCreate(&e));
        PB_CUDA(cudaEventRecord(ev[0], st));
        if (n) {
            PB_CUDA(cudaMemcpyAsync(db.get(), b, 8 * n, cudaMemcpyHostToDevice, st));
            PB_CUDA(cudaMemcpyAsync(du.get(), u, 8 * n, cudaMemcpyHostToDevice, st));
        }
        PB_CUDA(cudaEventRecord(ev[1], st));
        pairamg_solve_config sc;
        pairamg_default_solve_config(&sc);
        if (scfg) sc = *scfg;
        sv.solve(db.get(), du.get(), cycle_cfg(ccfg), sc.rtol, sc.max_iters, sc.precflag != 0, stats);
        PB_CUDA(cudaEventRecord(ev[2], st));
        if (n) PB_CUDA(cudaMemcpyAsync(u, du.get(), 8 * n, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaEventRecord(ev[3], st));
        PB_CUDA(cudaStreamSynchronize(st));
        float h2d = 0.f, d2h = 0.f;
        PB_CUDA(cudaEventElapsedTime(&h2d, ev[0], ev[1]));
        PB_CUDA(cudaEventElapsedTime(&d2h, ev[2], ev[3]));
        for (auto& e : ev) cudaEventDestroy(e);
        if (stats) {
            stats->t_h2d_s = h2d * 1e-3;
            stats->t_d2h_s = d2h * 1e-3;
        }
    });
}

pairamg_status pairamg_vcycle(pairamg_solver* s, const double* r, double* x, const pairamg_cycle_config* ccfg,
                              int is_device) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "vcycle: setup not run");
        cudaStream_t st = sv.rt.stream();
        const int64_t n = sv.h.levels[0]->A.n;
        if (is_device) {
            sv.vcycle(r, x, cycle_cfg(ccfg));
            return;
        }
        pb::DBuf<double> dr(static_cast<size_t>(n), st), dx(static_cast<size_t>(n), st);
        if (n) PB_CUDA(cudaMemcpyAsync(dr.get(), r, 8 * n, cudaMemcpyHostToDevice, st));
        sv.vcycle(dr.get(), dx.get(), cycle_cfg(ccfg));
        if (n) PB_CUDA(cudaMemcpyAsync(x, dx.get(), 8 * n, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaStreamSynchronize(st));
    });
}

pairamg_status pairamg_spmv(pairamg_solver* s, int level, const double* x, double* y, int is_device) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "spmv: setup not run");
        if (level < 0 || level >= sv.h.nl()) pb::fail(PAIRAMG_INVALID_ARGUMENT, "spmv: level out of range");
        cudaStream_t st = sv.rt.stream();
        const int64_t n = sv.h.levels[level]->A.n;
        if (is_device) {
            sv.spmv(level, x, y);
            return;
        }
        pb::DBuf<double> dx(static_cast<size_t>(n), st), dy(static_cast<size_t>(n), st);
        if (n) PB_CUDA(cudaMemcpyAsync(dx.get(), x, 8 * n, cudaMemcpyHostToDevice, st));
        sv.spmv(level, dx.get(), dy.get());
        if (n) PB_CUDA(cudaMemcpyAsync(y, dy.get(), 8 * n, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaStreamSynchronize(st));
    });
}

pairamg_status pairamg_hierarchy_info(pairamg_solver* s, int* nlevels, double* opc) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup not run");
        if (nlevels) *nlevels = sv.h.nl();
        if (opc) *opc = sv.h.opc;
    });
}

pairamg_status pairamg_level_info(pairamg_solver* s, int level, int64_t* global_rows, int64_t* global_nnz,
                                  int64_t* row_begin, int64_t* local_rows, int64_t* local_nnz) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup not run");
        if (level < 0 || level >= sv.h.nl()) pb::fail(PAIRAMG_INVALID_ARGUMENT, "level out of range");
        const pb::DevMatrix& A = sv.h.levels[level]->A;
        if (global_rows) *global_rows = sv.h.level_sizes[level];
        if (global_nnz) *global_nnz = sv.h.level_nnz[level];
        if (row_begin) *row_begin = A.row_begin;
        if (local_rows) *local_rows = A.n;
        if (local_nnz) *local_nnz = A.nnz;
    });
}

pairamg_status pairamg_level_storage(pairamg_solver* s, int level, int* format) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup not run");
        if (level < 0 || level >= sv.h.nl()) pb::fail(PAIRAMG_INVALID_ARGUMENT, "level out of range");
        if (!format) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null format");
        const pb::Level& L = *sv.h.levels[level];
        *format = L.A.halo.n_halo > 0 && L.sell_int.nrows > 0 ? L.sell_int.format : L.sell_all.format;
    });
}

pairamg_status pairamg_level_export(pairamg_solver* s, int level, int64_t* row_ptr, int64_t* col, double* val,
                                    double* w, double* l1) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup not run");
        if (level < 0 || level >= sv.h.nl()) pb::fail(PAIRAMG_INVALID_ARGUMENT, "level out of range");
        const pb::Level& L = *sv.h.levels[level];
        cudaStream_t st = sv.rt.stream();
        const int64_t n = L.A.n, nnz = L.A.nnz;
        if (row_ptr) PB_CUDA(cudaMemcpyAsync(row_ptr, L.A.rp.get(), 8 * (n + 1), cudaMemcpyDeviceToHost, st));
        if (col && nnz) {
            pb::DBuf<int64_t> g(static_cast<size_t>(nnz), st);
            pb::global_columns(L.A, g.get(), st);
            PB_CUDA(cudaMemcpyAsync(col, g.get(), 8 * nnz, cudaMemcpyDeviceToHost, st));
            PB_CUDA(cudaStreamSynchronize(st));
        }
        if (val && nnz) PB_CUDA(cudaMemcpyAsync(val, L.A.val.get(), 8 * nnz, cudaMemcpyDeviceToHost, st));
        if (w && n) PB_CUDA(cudaMemcpyAsync(w, L.w.get(), 8 * n, cudaMemcpyDeviceToHost, st));
        if (l1 && n) PB_CUDA(cudaMemcpyAsync(l1, L.l1.get(), 8 * n, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaStreamSynchronize(st));
    });
}

pairamg_status pairamg_prolongator_export(pairamg_solver* s, int level, int64_t* col, double* val) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup not run");
        if (level < 1 || level >= sv.h.nl()) pb::fail(PAIRAMG_INVALID_ARGUMENT, "prolongator level must be >= 1");
        const pb::Level& C = *sv.h.levels[level];
        const int64_t nf = sv.h.levels[level - 1]->A.n;
        cudaStream_t st = sv.rt.stream();
        if (col && nf) {
            std::vector<int32_t> lc(static_cast<size_t>(nf));
            PB_CUDA(cudaMemcpyAsync(lc.data(), C.pcol.get(), 4 * nf, cudaMemcpyDeviceToHost, st));
            PB_CUDA(cudaStreamSynchronize(st));
            for (int64_t i = 0; i < nf; ++i) col[i] = C.A.row_begin + lc[static_cast<size_t>(i)];
        }
        if (val && nf) PB_CUDA(cudaMemcpyAsync(val, C.pval.get(), 8 * nf, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaStreamSynchronize(st));
    });
}

pairamg_status pairamg_num_matchings(pairamg_solver* s, int* steps) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        *steps = static_cast<int>(sv.h.matchings.size());
    });
}

pairamg_status pairamg_matching_export(pairamg_solver* s, int step, int64_t* n, int64_t* mate) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (step < 0 || step >= static_cast<int>(sv.h.matchings.size()))
            pb::fail(PAIRAMG_INVALID_ARGUMENT, "matching step out of range");
        const auto& m = sv.h.matchings[static_cast<size_t>(step)];
        if (n) *n = static_cast<int64_t>(m.size());
        if (mate && m.size()) {
            PB_CUDA(cudaMemcpyAsync(mate, m.get(), 8 * m.size(), cudaMemcpyDeviceToHost, sv.rt.stream()));
            PB_CUDA(cudaStreamSynchronize(sv.rt.stream()));
        }
    });
}

pairamg_status pairamg_get_setup_stats(pairamg_solver* s, pairamg_setup_stats* out) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!sv.ready) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "setup not run");
        const auto& st = sv.h.stats;
        out->t_total = st.t_total;
        out->t_matching = st.t_matching;
        out->t_spmm = st.t_spmm;
        out->t_spmm_comm = st.t_spmm_comm;
        out->matching_messages = st.matching_messages;
        out->rc_messages = st.rc_messages;
        out->levels = sv.h.nl();
        out->opc = sv.h.opc;
    });
}

pairamg_status pairamg_setup_warnings(pairamg_solver* s, int* count) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (!count) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null count");
        *count = static_cast<int>(sv.warnings().size());
    });
}

pairamg_status pairamg_setup_warning(pairamg_solver* s, int i, char* buf, size_t cap, size_t* len) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        const std::vector<std::string> w = sv.warnings();
        if (i < 0 || i >= static_cast<int>(w.size())) pb::fail(PAIRAMG_INVALID_ARGUMENT, "warning index out of range");
        const std::string& m = w[static_cast<size_t>(i)];
        if (len) *len = m.size();
        if (buf && cap) {
            const size_t k = std::min(cap - 1, m.size());
            std::memcpy(buf, m.data(), k);
            buf[k] = 0;
        }
    });
}

pairamg_status pairamg_match_graph(pairamg_runtime* rt, int64_t n, const int64_t* row_ptr, const int64_t* col,
                                   const double* weight, int64_t* mate) {
    return guarded([&] {
        if (!rt || n < 0 || !row_ptr) pb::fail(PAIRAMG_INVALID_ARGUMENT, "match_graph: bad arguments");
        PB_CUDA(cudaSetDevice(rt->rt->device()));
        cudaStream_t st = rt->rt->stream();
        const int64_t m = row_ptr[n];
        std::vector<int32_t> c32(static_cast<size_t>(m));
        for (int64_t t = 0; t < m; ++t) {
            if (col[t] < 0 || col[t] >= n) pb::fail(PAIRAMG_CONTRACT_VIOLATION, "match_graph: column out of range");
            c32[static_cast<size_t>(t)] = static_cast<int32_t>(col[t]);
        }
        pb::DBuf<int64_t> drp(static_cast<size_t>(n + 1), st), dm(static_cast<size_t>(n), st);
        pb::DBuf<int32_t> dc(static_cast<size_t>(m), st);
        pb::DBuf<double> dw(static_cast<size_t>(m), st);
        PB_CUDA(cudaMemcpyAsync(drp.get(), row_ptr, 8 * (n + 1), cudaMemcpyHostToDevice, st));
        if (m) {
            PB_CUDA(cudaMemcpyAsync(dc.get(), c32.data(), 4 * m, cudaMemcpyHostToDevice, st));
            PB_CUDA(cudaMemcpyAsync(dw.get(), weight, 8 * m, cudaMemcpyHostToDevice, st));
        }
        if (n) pb::suitor_match_device(drp.get(), dc.get(), dw.get(), n, dm.get(), st);
        if (n) PB_CUDA(cudaMemcpyAsync(mate, dm.get(), 8 * n, cudaMemcpyDeviceToHost, st));
        PB_CUDA(cudaStreamSynchronize(st));
    });
}

pairamg_status pairamg_set_kernel_timing(pairamg_solver* s, int enabled) {
    return guarded([&] { S(s).timing = enabled != 0; });
}

pairamg_status pairamg_kernel_timing(pairamg_solver* s, int kclass, int64_t* launches, double* ms,
                                     double* bytes_per_launch) {
    return guarded([&] {
        pb::Solver& sv = S(s);
        if (kclass < 0 || kclass >= pb::kNumClasses) pb::fail(PAIRAMG_INVALID_ARGUMENT, "kernel class out of range");
        if (launches) *launches = sv.ktime[kclass].launches;
        if (ms) *ms = sv.ktime[kclass].ms;
        if (bytes_per_launch) *bytes_per_launch = sv.ktime[kclass].bytes_per_launch;
    });
}

pairamg_status pairamg_launch_count(pairamg_solver* s, int64_t* launches) {
    return guarded([&] { *launches = S(s).last_launches; });
}

void* pairamg_solver_stream(pairamg_solver* s) {
    if (!s || !s->s) return nullptr;
    return reinterpret_cast<void*>(s->s->rt.stream());
}

int64_t pairamg_poisson_nnz(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t b, int64_t e) {
    int64_t z = 0;
    for (int64_t r = b; r < e; ++r) z += row_len(stencil, nx, ny, nz, r);
    return z;
}

pairamg_status pairamg_poisson_host(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t b, int64_t e,
                                    int64_t* row_ptr, int64_t* col, double* val) {
    return guarded([&] { generate_host(stencil, nx, ny, nz, b, e, row_ptr, col, val, Coef()); });
}

pairamg_status pairamg_poisson_device(pairamg_runtime* rt, int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t b,
                                      int64_t e, int64_t* d_rp, int64_t* d_col, double* d_val) {
    return guarded([&] { generate_device(rt, stencil, nx, ny, nz, b, e, d_rp, d_col, d_val, Coef()); });
}

pairamg_status pairamg_varcoef_host(int stencil, int64_t nx, int64_t ny, int64_t nz, int levels, uint64_t seed,
                                    int64_t b, int64_t e, int64_t* row_ptr, int64_t* col, double* val) {
    return guarded([&] {
        if (levels < 0) pb::fail(PAIRAMG_INVALID_ARGUMENT, "varcoef: levels must be >= 0");
        Coef cf;
        cf.levels = levels;
        cf.seed = seed;
        generate_host(stencil, nx, ny, nz, b, e, row_ptr, col, val, cf);
    });
}

pairamg_status pairamg_varcoef_device(pairamg_runtime* rt, int stencil, int64_t nx, int64_t ny, int64_t nz, int levels,
                                      uint64_t seed, int64_t b, int64_t e, int64_t* d_rp, int64_t* d_col,
                                      double* d_val) {
    return guarded([&] {
        if (levels < 0) pb::fail(PAIRAMG_INVALID_ARGUMENT, "varcoef: levels must be >= 0");
        Coef cf;
        cf.levels = levels;
        cf.seed = seed;
        generate_device(rt, stencil, nx, ny, nz, b, e, d_rp, d_col, d_val, cf);
    });
}

}  // extern "C"

// ---- MatrixMarket -----------------------------------------------------------

struct pairamg_mm {
    pb::HostCsr A;
};

namespace {
void mm_block(pairamg_mm* m, int64_t b, int64_t e) {
    if (!m) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null matrix handle");
    if (b < 0 || e < b || e > m->A.nrows)
        pb::fail(PAIRAMG_CONTRACT_VIOLATION, "distribute_matrix: row block outside the matrix");
}
}  // namespace

extern "C" {

pairamg_status pairamg_mm_open(const char* path, pairamg_mm** out, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
    return guarded([&] {
        if (!path || !out) pb::fail(PAIRAMG_INVALID_ARGUMENT, "null path/out");
        *out = nullptr;
        auto m = std::make_unique<pairamg_mm>();
        m->A = pb::read_matrix_market(path);
        if (nrows) *nrows = m->A.nrows;
        if (ncols) *ncols = m->A.ncols;
        if (nnz) *nnz = static_cast<int64_t>(m->A.col.size());
        *out = m.release();
    });
}

pairamg_status pairamg_mm_rows(pairamg_mm* m, int64_t b, int64_t e, int64_t* nnz_local) {
    return guarded([&] {
        mm_block(m, b, e);
        if (nnz_local) *nnz_local = m->A.row_ptr[static_cast<size_t>(e)] - m->A.row_ptr[static_cast<size_t>(b)];
    });
}

pairamg_status pairamg_mm_copy_rows(pairamg_mm* m, int64_t b, int64_t e, int64_t* row_ptr, int64_t* col, double* val) {
    return guarded([&] {
        mm_block(m, b, e);
        const int64_t base = m->A.row_ptr[static_cast<size_t>(b)];
        const int64_t end = m->A.row_ptr[static_cast<size_t>(e)];
        if (row_ptr)
            for (int64_t i = 0; i <= e - b; ++i) row_ptr[i] = m->A.row_ptr[static_cast<size_t>(b + i)] - base;
        if (col) std::memcpy(col, m->A.col.data() + base, 8 * static_cast<size_t>(end - base));
        if (val) std::memcpy(val, m->A.val.data() + base, 8 * static_cast<size_t>(end - base));
    });
}

pairamg_status pairamg_spgemm(pairamg_runtime* rt, int64_t an, int64_t am, const int64_t* a_rp, const int64_t* a_col,
                              const double* a_val, int64_t bm, const int64_t* b_rp, const int64_t* b_col,
                              const double* b_val, pairamg_mm** out, int64_t* nnz) {
    return guarded([&] {
        if (!rt || !rt->rt || !out || !a_rp || !b_rp) pb::fail(PAIRAMG_INVALID_ARGUMENT, "spgemm: null argument");
        *out = nullptr;
        PB_CUDA(cudaSetDevice(rt->rt->device()));
        auto m = std::make_unique<pairamg_mm>();
        m->A = pb::spgemm(an, am, a_rp, a_col, a_val, bm, b_rp, b_col, b_val, rt->rt->stream());
        if (nnz) *nnz = static_cast<int64_t>(m->A.col.size());
        *out = m.release();
    });
}

pairamg_status pairamg_mm_close(pairamg_mm* m) {
    delete m;
    return PAIRAMG_OK;
}

pairamg_status pairamg_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                                const int64_t* col, const double* val) {
    return guarded([&] {
        if (!path || nrows < 0 || ncols < 0 || (nrows > 0 && (!row_ptr || ((!col || !val) && row_ptr[nrows] > 0))))
            pb::fail(PAIRAMG_INVALID_ARGUMENT, "mm_write: bad arguments");
        pb::write_matrix_market(path, nrows, ncols, row_ptr, col, val);
    });
}

}  // extern "C"
