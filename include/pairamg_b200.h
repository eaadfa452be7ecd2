/*
 * pairamg_b200.h -- C-ABI drop-in boundary of the B200-native AMG-FCG hot path.
 *
 * The reference ("pairamg", /root/reference/proj) declares an exported C
 * shared library `add_library(pairamg SHARED capi.cpp)` with public headers
 * in proj/include (src/CMakeLists.txt:20-23) whose error categories are
 * "mirrored by the C API" (types.hpp:12), but neither capi.cpp nor include/
 * exists.  This header is therefore the C surface of the reference's C++
 * hot-path API, one entry point per reference function it replaces:
 *
 *   pairamg_runtime_create     <- spawn_ranks / RankCtx        (runtime.hpp:71-136)
 *   pairamg_setup              <- setup_hierarchy               (amg.hpp:84-85, amg.cpp:144-295)
 *   pairamg_solve              <- pcg_solve (absent)
 *   pairamg_vcycle             <- vcycle_apply                  (cycle.hpp:31-32, cycle.cpp:86-112)
 *   pairamg_spmv               <- spmv_dist                     (dist.hpp:83-86, dist.cpp:128-199)
 *   pairamg_hierarchy_info /
 *   pairamg_level_info         <- Hierarchy::level_sizes/level_nnz/opc, hierarchy_summary
 *                                                               (amg.hpp:49-58, amg.cpp:297-313)
 *   pairamg_level_export       <- Level{A, w, m_l1}             (amg.hpp:27-38)
 *   pairamg_prolongator_export <- Level::P_block                (amg.hpp:36)
 *   pairamg_matching_export    <- SetupConfig::record / MatchingTrace (amg.hpp:13-23, amg.cpp:207-220)
 *   pairamg_get_setup_stats    <- SetupStats                    (amg.hpp:40-47)
 *   pairamg_status_name        <- error_code_name               (types.hpp:37-51)
 *
 * Conventions:
 *  - One pairamg_runtime per rank; rank r drives GPU `device` from one host
 *    thread.  With nranks > 1 the ranks are separate processes (or threads)
 *    joined by an NCCL unique id obtained on one rank with
 *    pairamg_comm_unique_id and broadcast by the caller.  Calls on a solver
 *    are rank-collective, in the same order on every rank (runtime.hpp:84).
 *  - Inputs use the reference's data layout: the rank's owned row block of a
 *    row-block partition (Partition, runtime.hpp:15-28) in CSR with int64
 *    row_ptr and GLOBAL int64 column ids, strictly ascending per row
 *    (csr.hpp:10-11), f64 values.  Host arrays are caller-owned and copied
 *    in; device state is library-owned.  *_device variants take pointers in
 *    the runtime device's global memory instead.
 *  - Every function returns a pairamg_status; on failure
 *    pairamg_last_error() returns a thread-local message.  Status values are
 *    0 = ok followed by the reference ErrorCode values in declaration order
 *    (types.hpp:13-24).
 *  - All calls are synchronous with respect to the host.
 */
#ifndef PAIRAMG_B200_H
#define PAIRAMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAIRAMG_B200_ABI_VERSION 2

/* ErrorCode (types.hpp:13-24), shifted by one; 0 = success. */
typedef enum pairamg_status {
    PAIRAMG_OK = 0,
    PAIRAMG_INVALID_ARGUMENT = 1,
    PAIRAMG_CONTRACT_VIOLATION = 2,
    PAIRAMG_MISSING_ROW = 3,
    PAIRAMG_SINGULAR_SMOOTHER = 4,
    PAIRAMG_STAGNATION = 5,
    PAIRAMG_BREAKDOWN = 6,
    PAIRAMG_DEADLOCK = 7,
    PAIRAMG_PARSE_ERROR = 8,
    PAIRAMG_IO_ERROR = 9,
    PAIRAMG_INTERNAL = 10
} pairamg_status;

/* Solve-time storage of a level's rows (B200 extension, no reference
 * counterpart).  Every format reproduces each entry's column and value
 * exactly and sums rows in CSR order, so results are bitwise equal; the
 * format only decides which kernels run and how many bytes they move. */
typedef enum pairamg_storage {
    PAIRAMG_STORAGE_AUTO = -1, /* STEN, else PAT (rows > 16 entries), DICT, PAT, CODED, PLAIN */
    PAIRAMG_STORAGE_PLAIN = 0, /* SELL-32, int32 column + f64 value per entry */
    PAIRAMG_STORAGE_DICT = 1,  /* one byte per entry into <= 255 (column - row, value) pairs */
    PAIRAMG_STORAGE_PAT = 2,   /* one byte per row into <= 255 row patterns */
    PAIRAMG_STORAGE_STEN = 3,  /* one byte per row: subset of one main stencil pattern */
    PAIRAMG_STORAGE_CODED = 4  /* SELL-32, one 32-bit (column - row, value code) word per entry */
} pairamg_storage;

/* SetupConfig (amg.hpp:17-23).  Matching ties are broken by the total order
 * key(e) = (w(e), -min(e), -max(e)) (hard part 1); the
 * reference's sequential Suitor keeps the incumbent on equal weights
 * (matching.cpp:82), so on coarse steps of odd grids the two may pick
 * different matchings.  `replay` reproduces any recorded matching exactly. */
typedef struct pairamg_setup_config {
    int aggregation_exponent; /* s: pairwise steps composed per level (default 3) */
    int64_t coarse_size_target; /* stop when global rows <= this (default 40) */
    int max_levels;             /* default 40 */
    /* SetupConfig::replay / MatchingTrace (amg.hpp:13-23, amg.cpp:182-197):
     * replay_steps > 0 skips the matching kernels; pairwise step t takes its
     * matching from replay_mates[t], the GLOBAL mate of every global row of
     * that step's fine level (replay_sizes[t] entries, -1 = unmatched), e.g.
     * the reference's MatchingTrace::steps or pairamg_matching_export.  A
     * mate outside the rank's owned block is CONTRACT_VIOLATION ("replayed
     * matching crosses the rank partition"), too few steps is
     * CONTRACT_VIOLATION ("matching trace exhausted").  Host pointers. */
    int replay_steps;
    const int64_t* const* replay_mates;
    const int64_t* replay_sizes;
    /* B200 extensions (no reference counterpart): */
    int storage;             /* pairamg_storage; default PAIRAMG_STORAGE_AUTO.  A forced
                                format falls back to PLAIN on rows it cannot encode. */
    int64_t replicate_rows;  /* nranks > 1: coarse levels with <= this many global rows
                                are also held in full on every rank (default 2500000; 0 = off);
                                the first such level must also have <= 8 x this many nonzeros */
    int setup_overlap;       /* nranks > 1: P's halo exchange on the communication stream
                                while R, w_next and the composed P are built (default 0:
                                measured no gain) */
} pairamg_setup_config;

/* CycleConfig (cycle.hpp:7-12). */
typedef struct pairamg_cycle_config {
    int pre_sweeps;      /* default 4 */
    int post_sweeps;     /* default 4 */
    int coarsest_sweeps; /* default 20 */
    double relax_weight; /* default 1.0 */
} pairamg_cycle_config;

/* SolveConfig. */
typedef struct pairamg_solve_config {
    double rtol;   /* default 1e-6 */
    int max_iters; /* default 1000 */
    int precflag;  /* 1 = AMG V-cycle preconditioner, 0 = identity */
} pairamg_solve_config;

/* SolveStats.  history (optional, caller-owned, capacity
 * history_cap) receives |r_k|/|r_0| for k = 0..iterations. */
typedef struct pairamg_solve_stats {
    int iterations;
    int converged;
    double final_relres;
    double rnorm0;
    double t_solve_s; /* device time of the solve (CUDA events) */
    double* history;
    int history_cap;
    /* pairamg_solve (host buffers) only: device time of the b/u0 upload and
     * of the u download (CUDA events on the solver stream); 0 otherwise. */
    double t_h2d_s, t_d2h_s;
    /* cross-rank exchanges of the FCG reduction per iteration (contract: 1;
     * SPEC.md:477) and halo exchanges per iteration, from CommStats deltas. */
    int reductions_per_iter;
    int halo_exchanges_per_iter;
    double halo_bytes_per_iter; /* halo values this rank receives per iteration (8 B each) */
} pairamg_solve_stats;

/* SetupStats (amg.hpp:40-47) plus the hierarchy summary. */
typedef struct pairamg_setup_stats {
    double t_total, t_matching, t_spmm, t_spmm_comm; /* seconds */
    int64_t matching_messages; /* transport activity during matching (contract: 0) */
    int64_t rc_messages;       /* transport activity during R*C (contract: 0) */
    int levels;
    double opc;
} pairamg_setup_stats;

typedef struct pairamg_runtime pairamg_runtime;
typedef struct pairamg_solver pairamg_solver;

void pairamg_default_setup_config(pairamg_setup_config* cfg);
void pairamg_default_cycle_config(pairamg_cycle_config* cfg);
void pairamg_default_solve_config(pairamg_solve_config* cfg);

const char* pairamg_status_name(pairamg_status s);
const char* pairamg_last_error(void);
int pairamg_abi_version(void);

/* ---- runtime (spawn_ranks / RankCtx, runtime.hpp:71-136) ---- */
/* 128-byte NCCL unique id, to be broadcast to every rank by the caller. */
pairamg_status pairamg_comm_unique_id(uint8_t id[128]);
/* spawn_ranks analogue (runtime.cpp:92-152): a 128-byte id for ranks that are
 * threads of ONE process.  Passed to pairamg_runtime_create by every rank
 * thread, it joins them through an in-process hub instead of NCCL: host
 * collectives meet in shared memory (with the reference's deadlock timeout,
 * PAIRAMG_DEADLOCK), device data moves by peer copies and the solve-path
 * exchanges by the same P2P store/flag kernels as across processes.  Ranks
 * may share one GPU (device argument equal), e.g. to run a multi-rank setup
 * and solve on a single B200. */
pairamg_status pairamg_comm_local_id(uint8_t id[128]);
/* nranks == 1: id may be NULL and no communicator is created. */
pairamg_status pairamg_runtime_create(int device, int rank, int nranks, const uint8_t* id,
                                      pairamg_runtime** out);
pairamg_status pairamg_runtime_destroy(pairamg_runtime* rt);

/* ---- solver ---- */
pairamg_status pairamg_solver_create(pairamg_runtime* rt, pairamg_solver** out);
pairamg_status pairamg_solver_destroy(pairamg_solver* s);

/* setup_hierarchy(ctx, A, w0, cfg) (amg.hpp:84-85).  part_starts: nranks+1
 * row starts of the fine partition (the rank owns [part_starts[rank],
 * part_starts[rank+1])); n_local = that extent; row_ptr (n_local+1),
 * col_idx/values (row_ptr[n_local]) in the reference CsrMatrix layout with
 * global columns.  w0 may be NULL (all ones).  cfg may be NULL
 * (defaults). */
pairamg_status pairamg_setup(pairamg_solver* s, int64_t global_n, const int64_t* part_starts,
                             int64_t n_local, const int64_t* row_ptr, const int64_t* col_idx,
                             const double* values, const double* w0,
                             const pairamg_setup_config* cfg);
pairamg_status pairamg_setup_device(pairamg_solver* s, int64_t global_n, const int64_t* part_starts,
                                    int64_t n_local, int64_t nnz_local, const int64_t* d_row_ptr,
                                    const int64_t* d_col_idx, const double* d_values,
                                    const double* d_w0, const pairamg_setup_config* cfg);

/* Flexible PCG: u = A^{-1} b to rtol.  u holds u0 on entry
 * (NULL-free: pass zeros for u0 = 0).  Owned block of b and u. */
pairamg_status pairamg_solve(pairamg_solver* s, const double* b_local, double* u_local,
                             const pairamg_cycle_config* ccfg, const pairamg_solve_config* scfg,
                             pairamg_solve_stats* stats);
pairamg_status pairamg_solve_device(pairamg_solver* s, const double* d_b_local, double* d_u_local,
                                    const pairamg_cycle_config* ccfg,
                                    const pairamg_solve_config* scfg, pairamg_solve_stats* stats);

/* x = B r, one V-cycle from level 0 (vcycle_apply). is_device selects pointer space. */
pairamg_status pairamg_vcycle(pairamg_solver* s, const double* r_local, double* x_local,
                              const pairamg_cycle_config* ccfg, int is_device);
/* y = A^k x on level k (spmv_dist with the level's halo plan). */
pairamg_status pairamg_spmv(pairamg_solver* s, int level, const double* x_local, double* y_local,
                            int is_device);

/* ---- hierarchy introspection / parity export (all host arrays) ---- */
pairamg_status pairamg_hierarchy_info(pairamg_solver* s, int* nlevels, double* opc);
pairamg_status pairamg_level_info(pairamg_solver* s, int level, int64_t* global_rows,
                                  int64_t* global_nnz, int64_t* row_begin, int64_t* local_rows,
                                  int64_t* local_nnz);
/* Solve-time storage of level k's owned rows (pairamg_storage: 0 PLAIN,
 * 1 DICT, 2 PAT, 3 STEN, 4 CODED) -- for the interior row set when the level
 * has halo traffic.  All formats give bitwise-equal results; this only
 * reports which kernels run. */
pairamg_status pairamg_level_storage(pairamg_solver* s, int level, int* format);
/* Owned rows of A^k: row_ptr (local_rows+1), col (local_nnz, GLOBAL ids,
 * ascending), val; w^k and the l1 diagonal (local_rows).  Any pointer may be NULL. */
pairamg_status pairamg_level_export(pairamg_solver* s, int level, int64_t* row_ptr, int64_t* col,
                                    double* val, double* w, double* l1);
/* Composed prolongator into level k >= 1: one entry per owned fine row of
 * level k-1 (global coarse column, value). */
pairamg_status pairamg_prolongator_export(pairamg_solver* s, int level, int64_t* col, double* val);
/* Pairwise matching of setup step `step` on the owned block: *n receives the
 * owned vertex count; mate (may be NULL) receives global mates, -1 = unmatched. */
pairamg_status pairamg_num_matchings(pairamg_solver* s, int* steps);
pairamg_status pairamg_matching_export(pairamg_solver* s, int step, int64_t* n, int64_t* mate);
pairamg_status pairamg_get_setup_stats(pairamg_solver* s, pairamg_setup_stats* out);
/* Hierarchy::warnings (amg.hpp:56, amg.cpp:230-234) plus the cycle-config
 * warning of validate_cycle_config (cycle.cpp:7-13): *count receives the
 * number; pairamg_setup_warning copies warning i (NUL-terminated, truncated
 * to cap bytes) and returns its full length in *len (either may be NULL). */
pairamg_status pairamg_setup_warnings(pairamg_solver* s, int* count);
pairamg_status pairamg_setup_warning(pairamg_solver* s, int i, char* buf, size_t cap, size_t* len);

/* ---- matching KAT hook ---- */
/* suitor_match (matching.cpp:62-100) under the total-order tie rule, run by
 * the setup's parallel Suitor kernels on a caller graph: host CSR (n+1 row
 * pointers, local column ids, symmetric, weights aligned with columns;
 * self loops ignored).  mate (n) receives partners, -1 = unmatched. */
pairamg_status pairamg_match_graph(pairamg_runtime* rt, int64_t n, const int64_t* row_ptr, const int64_t* col,
                                   const double* weight, int64_t* mate);

/* ---- measurement hooks ---- */
/* Per-kernel-class device time accumulated over the last solve (CUDA events
 * around every launch of the class when timing was enabled):
 * class 0 = level-0 smoother sweeps, 1 = level-0 residual, 2 = level-0 outer
 * SpMV+dots, 3 = FCG vector updates, 4 + k (k < 16) = level k's own
 * V-cycle work (two intervals per cycle: entry to restriction, return from
 * level k+1 to exit).  *launches and *ms may be NULL. */
pairamg_status pairamg_set_kernel_timing(pairamg_solver* s, int enabled);
pairamg_status pairamg_kernel_timing(pairamg_solver* s, int kclass, int64_t* launches, double* ms,
                                     double* bytes_per_launch);
/* Number of library kernel launches enqueued by the last solve. */
pairamg_status pairamg_launch_count(pairamg_solver* s, int64_t* launches);
/* cudaStream_t the solver launches on (for caller-side events). */
void* pairamg_solver_stream(pairamg_solver* s);

/* ---- problem generator ---- */
/* Owned rows [row_begin, row_end) of the 7- or 27-point Poisson operator on an
 * nx*ny*nz grid (lexicographic, x fastest; diagonal 6 or 26, off-diagonals -1).
 * Host variant: caller allocates row_ptr (rows+1), col/val (nnz from
 * pairamg_poisson_nnz).  Device variant: pointers in device memory. */
int64_t pairamg_poisson_nnz(int stencil, int64_t nx, int64_t ny, int64_t nz, int64_t row_begin,
                            int64_t row_end);
pairamg_status pairamg_poisson_host(int stencil, int64_t nx, int64_t ny, int64_t nz,
                                    int64_t row_begin, int64_t row_end, int64_t* row_ptr,
                                    int64_t* col, double* val);
pairamg_status pairamg_poisson_device(pairamg_runtime* rt, int stencil, int64_t nx, int64_t ny,
                                      int64_t nz, int64_t row_begin, int64_t row_end,
                                      int64_t* d_row_ptr, int64_t* d_col, double* d_val);
/* Variable-coefficient workload (no reference counterpart; exercises the
 * general storage paths): same sparsity as the Poisson operator, cell
 * coefficients k_c = 1 + (hash(seed, c) mod levels) for levels > 0 (a few
 * distinct entry values) or continuous in [0.5, 1.5) for levels = 0 (all
 * distinct); couplings -(k_i + k_j)/2, diagonal = sum over the stencil
 * directions of (k_i + k_j)/2 with k_i across the Dirichlet boundary. */
pairamg_status pairamg_varcoef_host(int stencil, int64_t nx, int64_t ny, int64_t nz, int levels,
                                    uint64_t seed, int64_t row_begin, int64_t row_end,
                                    int64_t* row_ptr, int64_t* col, double* val);
pairamg_status pairamg_varcoef_device(pairamg_runtime* rt, int stencil, int64_t nx, int64_t ny,
                                      int64_t nz, int levels, uint64_t seed, int64_t row_begin,
                                      int64_t row_end, int64_t* d_row_ptr, int64_t* d_col,
                                      double* d_val);

/* ---- MatrixMarket ingest / distribute (mm_io.cpp:26-110, csr.cpp:24-54,
 *      dist.cpp:349-363) ---- */
/* Parse a coordinate MatrixMarket file (real | integer | pattern; general |
 * symmetric | skew-symmetric; symmetric storage expanded) into a host CSR with
 * rows sorted by column; duplicates and malformed lines are
 * PAIRAMG_PARSE_ERROR ("path:line: msg"), an unreadable file PAIRAMG_IO_ERROR. */
typedef struct pairamg_mm pairamg_mm;
pairamg_status pairamg_mm_open(const char* path, pairamg_mm** out, int64_t* nrows, int64_t* ncols,
                               int64_t* nnz);
/* Rows [row_begin, row_end) as a rank's DistMatrix block (distribute_matrix):
 * nnz of the block, then local row_ptr (rows+1, from 0), global col, val. */
pairamg_status pairamg_mm_rows(pairamg_mm* m, int64_t row_begin, int64_t row_end, int64_t* nnz_local);
pairamg_status pairamg_mm_copy_rows(pairamg_mm* m, int64_t row_begin, int64_t row_end, int64_t* row_ptr,
                                    int64_t* col, double* val);
pairamg_status pairamg_mm_close(pairamg_mm* m);
/* General sparse product C = A*B on rt's GPU (spgemm_local, csr.cpp:206-272;
 * SURVEY 8f row 4): A is a_nrows x a_ncols, B is a_ncols x b_ncols, host CSR
 * arrays; per output entry the products a_ik*b_kj are summed in encounter
 * order (A row, then B row), the first assigned -- bitwise the reference.
 * The result is a host-CSR handle read with pairamg_mm_rows/copy_rows and
 * freed with pairamg_mm_close. */
pairamg_status pairamg_spgemm(pairamg_runtime* rt, int64_t a_nrows, int64_t a_ncols, const int64_t* a_row_ptr,
                              const int64_t* a_col, const double* a_val, int64_t b_ncols,
                              const int64_t* b_row_ptr, const int64_t* b_col, const double* b_val,
                              pairamg_mm** out, int64_t* nnz);
/* Write "coordinate real general" with %.17g values (write_matrix_market). */
pairamg_status pairamg_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                                const int64_t* col, const double* val);

#ifdef __cplusplus
}
#endif
#endif
