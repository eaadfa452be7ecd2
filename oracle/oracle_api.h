/*
 * oracle_api.h -- C interface shared by the two CPU checkers under oracle/.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product library
 * (paper_2303_02352_b200/) includes, links or calls this.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs load the two implementations:
 *
 *   oracle/_build/libpairamg_oracle.so  -- pairamg_oracle.c, a plain-C
 *       restatement of the reference algorithm (single process, p row blocks
 *       emulated), with each function citing the reference file:line.
 *   oracle/_ref/libpairamg_ref.so       -- the reference's own seven C++
 *       translation units (/root/reference/proj/src/pairamg/ *.cpp) compiled
 *       unmodified with the reference Release flags, plus ref_driver.cpp
 *       (the Poisson generator and Alg.-1 FCG, which the reference lacks:
 *       pcg.cpp / problem.cpp are absent).
 *
 * Both export exactly this API, so a test can run the same case through
 * both and compare bit patterns.
 */
#ifndef PAIRAMG_ORACLE_API_H
#define PAIRAMG_ORACLE_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_config {
    /* problem: stencil 7 or 27 on an nx*ny*nz grid (lexicographic, x fastest)
     * or 0 for a caller-supplied CSR (orc_create_csr). */
    int stencil;
    int64_t nx, ny, nz;
    int nranks; /* row-block partition Partition::uniform (runtime.cpp:13-22) */
    /* SetupConfig (amg.hpp:17-23) */
    int aggregation_exponent;
    int64_t coarse_size_target;
    int max_levels;
    /* matching tie rule: 0 = reference strict-weight acceptor
     * (matching.cpp:82), 1 = total order key (w, -min, -max) (SURVEY 7 hard
     * part 1).  The compiled reference only implements 0. */
    int matching_mode;
    /* CycleConfig (cycle.hpp:7-12) */
    int pre_sweeps, post_sweeps, coarsest_sweeps;
    double relax_weight;
    /* SolveConfig */
    double rtol;
    int max_iters;
    int precflag; /* 1 = AMG V-cycle, 0 = identity */
    int threads;  /* ref driver: ranks run as threads (always nranks); oracle: ignored */
} orc_config;

typedef struct orc_setup_stats {
    double t_total, t_matching, t_spmm, t_spmm_comm; /* SetupStats amg.hpp:40-47 */
    int64_t matching_messages, rc_messages;
} orc_setup_stats;

void orc_default_config(orc_config* cfg);

/* Generates the Poisson system (b = 1, u0 = 0, w0 = 1). */
void* orc_create(const orc_config* cfg);
/* Caller-supplied global CSR (int64 indices, strictly ascending columns). */
void* orc_create_csr(const orc_config* cfg, int64_t n, const int64_t* row_ptr,
                     const int64_t* col, const double* val);
void orc_destroy(void* h);
const char* orc_last_error(void);
/* Error code of the last failure: ErrorCode (types.hpp:13-24) + 1, 0 = ok. */
int orc_last_status(void);

int64_t orc_global_n(void* h);
int64_t orc_global_nnz(void* h);
/* Matrix of the input system, assembled globally. */
int orc_export_input(void* h, int64_t* row_ptr, int64_t* col, double* val);

int orc_setup(void* h);
int orc_num_levels(void* h);
double orc_opc(void* h);
int orc_get_setup_stats(void* h, orc_setup_stats* out);
/* level sizes: rows and nnz of A^k (global). */
int orc_level_size(void* h, int level, int64_t* n, int64_t* nnz);
/* Level k partition starts (nranks+1 entries). */
int orc_level_partition(void* h, int level, int64_t* starts);
/* A^k assembled globally (row_ptr n+1, col nnz, val nnz), w^k, l1 diag. */
int orc_export_level(void* h, int level, int64_t* row_ptr, int64_t* col, double* val,
                     double* w, double* l1);
/* Composed prolongator into level k (k >= 1): one entry per fine row. */
int orc_export_prolongator(void* h, int level, int64_t* col, double* val);
/* Pairwise matchings in setup order (global mates, -1 = unmatched). */
int orc_num_matchings(void* h);
int64_t orc_matching_size(void* h, int step);
int orc_export_matching(void* h, int step, int64_t* mate);

/* Matching kernels on a caller graph (KAT hooks):
 * orc_build_weights: build_weights (matching.cpp:28-60) of a square block
 *   with smooth vector w -> graph CSR (diagonal removed) in grp/gcol/gw
 *   (capacity nnz), returns the edge count (or -1).
 * orc_match_graph: suitor_match (matching.cpp:62-100) on a weighted graph CSR
 *   (symmetric, no self loops); mode as orc_config.matching_mode. */
int64_t orc_build_weights(int64_t n, const int64_t* rp, const int64_t* col, const double* val,
                          const double* w, int64_t* grp, int64_t* gcol, double* gw);
int orc_match_graph(int64_t n, const int64_t* rp, const int64_t* col, const double* w, int mode,
                    int64_t* mate);

/* MatrixMarket (reference checker only: read_matrix_market, mm_io.cpp:26-88,
 * through the reference's own CsrMatrix::from_triplets).  orc_mm_load returns
 * NULL on error (orc_last_status / orc_last_error). */
void* orc_mm_load(const char* path);
void orc_mm_info(void* m, int64_t* nrows, int64_t* ncols, int64_t* nnz);
void orc_mm_export(void* m, int64_t* row_ptr, int64_t* col, double* val);
void orc_mm_free(void* m);
/* spgemm_local(A, B) (csr.cpp:206-279) -> a CsrMatrix handle read with
 * orc_mm_info / orc_mm_export / orc_mm_free; NULL on error. */
void* orc_spgemm(int64_t an, int64_t am, const int64_t* a_rp, const int64_t* a_col, const double* a_val, int64_t bm,
                 const int64_t* b_rp, const int64_t* b_col, const double* b_val);
/* write_matrix_market (mm_io.cpp:90-110) of a CSR. */
int orc_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_ptr, const int64_t* col,
                 const double* val);

/* y = A^k x (global vectors). */
int orc_spmv(void* h, int level, const double* x, double* y);
/* x = B r, one V-cycle from level 0 (global vectors). */
int orc_vcycle(void* h, const double* r, double* x);
/* Flexible PCG on the input system, b = ones unless b != NULL.
 * u (global, may be NULL) receives the solution; hist (cap entries) the
 * relative residual history |r_k|/|r_0| for k = 0..iters. */
/* Change the solve parameters of an existing session (SolveConfig). */
int orc_set_solve(void* h, double rtol, int max_iters);
int orc_solve(void* h, const double* b, double* u, double* hist, int hist_cap, int* iters,
              double* relres, double* t_solve);

#ifdef __cplusplus
}
#endif
#endif
