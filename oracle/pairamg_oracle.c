/*
 * pairamg_oracle.c -- TEST INFRASTRUCTURE: plain-C restatement of the
 * reference AMG-FCG path (BootCMatchGX "pairamg", /root/reference/proj).
 *
 * This is the parity checker for the CUDA library, not part of it.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 * Parity of this restatement is pinned against the reference itself: the
 * reference's seven C++ units are compiled unmodified into
 * oracle/_ref/libpairamg_ref.so (oracle/Makefile) and tests/test_oracle.py
 * requires bit-identical hierarchies, matchings, V-cycles and residual
 * histories between the two (matching_mode 0), plus the SURVEY-pinned golden
 * numbers in tests/golden/.
 *
 * Global-view emulation of p row blocks.  Every quantity the reference
 * computes per rank is either block-local (matching on the diagonal block,
 * aggregate numbering, P, R, R*C) or partition-independent by construction
 * (spmv_dist sums each row in ascending global column order, dist.cpp:164-187;
 * spgemm_local sums each entry in ascending inner index, csr.cpp:206-272), so
 * one process holding global arrays reproduces the distributed result bit for
 * bit.  The only explicitly per-rank arithmetic is dot_dist (dist.cpp:299-306:
 * sequential per-rank partial, then rank-ascending allreduce,
 * runtime.cpp:243-259), which is emulated as such.
 *
 * Floating point: built with -ffp-contract=off (no FMA) to match the
 * reference's Release objects, which contain no FMA.
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oracle_api.h"

/* ErrorCode (types.hpp:13-24) + 1 */
enum {
    ST_OK = 0,
    ST_INVALID_ARGUMENT,
    ST_CONTRACT_VIOLATION,
    ST_MISSING_ROW,
    ST_SINGULAR_SMOOTHER,
    ST_STAGNATION,
    ST_BREAKDOWN,
    ST_DEADLOCK,
    ST_PARSE_ERROR,
    ST_IO_ERROR,
    ST_INTERNAL
};

static _Thread_local char g_err[512];
static _Thread_local int g_status;

static int fail(int st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    g_status = st;
    return st;
}

#define CHECK(x)                   \
    do {                           \
        int rc__ = (x);            \
        if (rc__) return rc__;     \
    } while (0)

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) {
        fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
        abort();
    }
    return p;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---------------------------------------------------------------- CSR --- */

/* CsrMatrix (csr.hpp:12-41): global int64 columns, strictly ascending. */
typedef struct {
    int64_t n, ncols, nnz;
    int64_t* rp;
    int64_t* ci;
    double* va;
} csr_t;

static void csr_alloc(csr_t* A, int64_t n, int64_t ncols, int64_t nnz) {
    A->n = n;
    A->ncols = ncols;
    A->nnz = nnz;
    A->rp = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    A->ci = xmalloc(sizeof(int64_t) * (size_t)nnz);
    A->va = xmalloc(sizeof(double) * (size_t)nnz);
    A->rp[0] = 0;
}

static void csr_free(csr_t* A) {
    free(A->rp);
    free(A->ci);
    free(A->va);
    memset(A, 0, sizeof *A);
}

/* CsrMatrix::validate (csr.cpp:56-78) */
static int csr_validate(const csr_t* A) {
    if (A->rp[0] != 0) return fail(ST_CONTRACT_VIOLATION, "csr: row_ptr[0] != 0");
    for (int64_t i = 0; i < A->n; ++i) {
        if (A->rp[i] > A->rp[i + 1])
            return fail(ST_CONTRACT_VIOLATION, "csr: row_ptr not non-decreasing");
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            if (A->ci[k] < 0 || A->ci[k] >= A->ncols)
                return fail(ST_CONTRACT_VIOLATION, "csr: column %lld out of range in row %lld",
                            (long long)A->ci[k], (long long)i);
            if (k > A->rp[i] && A->ci[k - 1] >= A->ci[k])
                return fail(ST_CONTRACT_VIOLATION, "csr: columns not strictly increasing in row %lld",
                            (long long)i);
        }
    }
    return 0;
}

/* spmv_local / spmv_dist row loop (csr.cpp:100-117, dist.cpp:164-187):
 * sum = 0.0; sum += a_ij * x_j in CSR (ascending global column) order. */
static void spmv(const csr_t* A, const double* x, double* y) {
    for (int64_t i = 0; i < A->n; ++i) {
        double sum = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) sum += A->va[k] * x[A->ci[k]];
        y[i] = sum;
    }
}

/* Stable insertion sort of (col, val) pairs by col; rows here are short. */
static void stable_sort_pairs(int64_t* c, double* v, int64_t m) {
    for (int64_t a = 1; a < m; ++a) {
        int64_t kc = c[a];
        double kv = v[a];
        int64_t b = a - 1;
        while (b >= 0 && c[b] > kc) {
            c[b + 1] = c[b];
            v[b + 1] = v[b];
            --b;
        }
        c[b + 1] = kc;
        v[b + 1] = kv;
    }
}

/* Merge a stably sorted contribution list: per column the first contribution
 * is assigned and later ones added in encounter order, output ascending --
 * exactly HashAccumulator::add + extract_sorted (csr.cpp:145-172) and
 * merge_row (csr.cpp:186-202). Returns the merged length. */
static int64_t merge_sorted(int64_t* c, double* v, int64_t m) {
    int64_t out = 0, i = 0;
    while (i < m) {
        int64_t col = c[i];
        double sum = v[i];
        ++i;
        while (i < m && c[i] == col) {
            sum += v[i];
            ++i;
        }
        c[out] = col;
        v[out] = sum;
        ++out;
    }
    return out;
}

/* ---------------------------------------------------------- partition --- */

/* Partition::uniform (runtime.cpp:13-22) */
static void partition_uniform(int64_t n, int p, int64_t* starts) {
    for (int r = 0; r <= p; ++r) starts[r] = (n / p) * r + (n % p < r ? n % p : r);
}

/* --------------------------------------------------------- hierarchy --- */

typedef struct {
    csr_t A;          /* level operator, global rows/cols */
    int64_t* starts;  /* row partition, nranks+1 */
    double* w;        /* smooth vector */
    double* l1;       /* l1-Jacobi diagonal */
    /* transfer from the finer level (k >= 1) */
    int64_t* pcol;    /* composed P: one entry per fine row, global coarse col */
    double* pval;
    csr_t R;          /* R = P^T: coarse rows, fine global cols ascending */
} level_t;

typedef struct {
    orc_config cfg;
    csr_t A0;
    int64_t* starts0;
    int nl;
    level_t* lv;
    int nmatch;
    int64_t** match; /* recorded global mates per pairwise step */
    int64_t* match_n;
    int setup_done;
    orc_setup_stats stats;
} session_t;

static void level_free(level_t* L) {
    csr_free(&L->A);
    free(L->starts);
    free(L->w);
    free(L->l1);
    free(L->pcol);
    free(L->pval);
    csr_free(&L->R);
}

static void hierarchy_free(session_t* s) {
    for (int k = 0; k < s->nl; ++k) level_free(&s->lv[k]);
    free(s->lv);
    s->lv = NULL;
    s->nl = 0;
    for (int i = 0; i < s->nmatch; ++i) free(s->match[i]);
    free(s->match);
    free(s->match_n);
    s->match = NULL;
    s->match_n = NULL;
    s->nmatch = 0;
    s->setup_done = 0;
}

/* ---------------------------------------------------------- matching --- */

/* suitor_match (matching.cpp:62-100) on a graph CSR (local ids, no self
 * loops).  Ascending proposers; each bids on its heaviest neighbour that
 * would accept, smallest index on ties (strict '>' scan); the displaced
 * suitor re-bids; mate = mutual suitors.  mode 0: the reference acceptor
 * `wv > suitor_weight[v]` (matching.cpp:82); mode 1: the acceptor compares
 * the total order key(e) = (w, -min(e), -max(e)) (SURVEY.md 7 hard part 1). */
static void suitor_run(int64_t n, const int64_t* grp, const int64_t* gci, const double* gw, int mode,
                       int64_t* mate) {
    int64_t* suitor = xmalloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    double* sw = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t v = 0; v < n; ++v) {
        suitor[v] = -1;
        sw[v] = -INFINITY;
        mate[v] = -1;
    }
    for (int64_t u = 0; u < n; ++u) {
        int64_t current = u;
        while (current != -1) {
            int64_t partner = -1;
            double best = -INFINITY;
            for (int64_t t = grp[current]; t < grp[current + 1]; ++t) {
                const int64_t v = gci[t];
                const double wv = gw[t];
                int accept;
                if (mode == 0) {
                    accept = wv > sw[v];
                } else {
                    const int64_t s = suitor[v];
                    if (s == -1 || wv > sw[v]) {
                        accept = s == -1 ? (wv > sw[v]) : 1;
                    } else if (wv < sw[v]) {
                        accept = 0;
                    } else {
                        const int64_t mn_c = current < v ? current : v, mx_c = current < v ? v : current;
                        const int64_t mn_s = s < v ? s : v, mx_s = s < v ? v : s;
                        accept = mn_c < mn_s || (mn_c == mn_s && mx_c < mx_s);
                    }
                }
                if (accept && wv > best) {
                    best = wv;
                    partner = v;
                }
            }
            if (partner == -1) break;
            const int64_t displaced = suitor[partner];
            suitor[partner] = current;
            sw[partner] = best;
            current = displaced;
        }
    }
    for (int64_t v = 0; v < n; ++v) {
        const int64_t s = suitor[v];
        if (s != -1 && suitor[s] == v) mate[v] = s;
    }
    free(suitor);
    free(sw);
}

int orc_match_graph(int64_t n, const int64_t* rp, const int64_t* col, const double* w, int mode,
                    int64_t* mate) {
    suitor_run(n, rp, col, w, mode, mate);
    return 0;
}

/* build_weights (matching.cpp:28-60) on a square block (local columns). */
int64_t orc_build_weights(int64_t n, const int64_t* rp, const int64_t* col, const double* val,
                          const double* w, int64_t* grp, int64_t* gcol, double* gw) {
    double* diag = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        diag[i] = 0.0;
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t)
            if (col[t] == i) diag[i] = val[t];
    }
    int64_t pos = 0;
    grp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            const int64_t j = col[t];
            if (j == i) continue;
            const double num = 2.0 * val[t] * w[i] * w[j];
            const double den = diag[i] * w[i] * w[i] + diag[j] * w[j] * w[j];
            double weight = 1.0 - num / den;
            if (!isfinite(weight)) weight = -1e300;
            gcol[pos] = j;
            gw[pos] = weight;
            ++pos;
        }
        grp[i + 1] = pos;
    }
    free(diag);
    return pos;
}

/* Decoupled matching of one rank's diagonal block [b, e) of A (global rows):
 * extract_diagonal_block (matching.cpp:8-26), build_weights
 * (matching.cpp:28-60), suitor_match (matching.cpp:62-100).  mate is local
 * (0..e-b-1, -1 unmatched).  matching_mode 1 replaces only the acceptor test
 * of matching.cpp:82 by the total order key(e) = (w, -min, -max). */
static void match_block(const csr_t* A, int64_t b, int64_t e, const double* w, int mode,
                        int64_t* mate) {
    const int64_t n = e - b;
    /* block graph: local columns in [0, n), diagonal removed */
    int64_t* grp = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t m = 0;
    double* diag = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        diag[i] = 0.0;
        for (int64_t t = A->rp[b + i]; t < A->rp[b + i + 1]; ++t) {
            const int64_t j = A->ci[t];
            if (j >= b && j < e) {
                if (j - b == i)
                    diag[i] = A->va[t];
                else
                    ++m;
            }
        }
    }
    int64_t* gci = xmalloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    double* gw = xmalloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    int64_t pos = 0;
    grp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double* wl = w + b;
        for (int64_t t = A->rp[b + i]; t < A->rp[b + i + 1]; ++t) {
            const int64_t jg = A->ci[t];
            if (jg < b || jg >= e) continue;
            const int64_t j = jg - b;
            if (j == i) continue; /* no self-loops */
            const double num = 2.0 * A->va[t] * wl[i] * wl[j];
            const double den = diag[i] * wl[i] * wl[i] + diag[j] * wl[j] * wl[j];
            double weight = 1.0 - num / den;
            if (!isfinite(weight)) weight = -1e300; /* kClampedWeight, matching.hpp:29 */
            gci[pos] = j;
            gw[pos] = weight;
            ++pos;
        }
        grp[i + 1] = pos;
    }

    suitor_run(n, grp, gci, gw, mode, mate);
    free(grp);
    free(diag);
    free(gci);
    free(gw);
}

/* build_pairwise_prolongator (amg.cpp:38-77) for one rank block: aggregates
 * numbered by smallest member; values w_i/sqrt(w_i^2+w_j^2) (1/sqrt 2 when the
 * norm is 0) or w_i/|w_i| (1 when w_i == 0).  Writes local aggregate ids. */
static int64_t pairwise_prolongator(const int64_t* mate, const double* w, int64_t n,
                                    int64_t* agg, double* val) {
    int64_t naggs = 0;
    for (int64_t i = 0; i < n; ++i) agg[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        agg[i] = naggs;
        if (mate[i] != -1) agg[mate[i]] = naggs;
        ++naggs;
    }
    for (int64_t i = 0; i < n; ++i) {
        const int64_t j = mate[i];
        if (j == -1) {
            val[i] = w[i] == 0.0 ? 1.0 : w[i] / fabs(w[i]);
        } else {
            const double norm = sqrt(w[i] * w[i] + w[j] * w[j]);
            val[i] = norm == 0.0 ? 1.0 / sqrt(2.0) : w[i] / norm;
        }
    }
    return naggs;
}

/* transpose_block (amg.cpp:87-108), global form: R row c lists the fine
 * rows of aggregate c in ascending fine index. */
static void transpose_p(const int64_t* pcol, const double* pval, int64_t nf, int64_t nc, csr_t* R) {
    csr_alloc(R, nc, nf, nf);
    for (int64_t c = 0; c <= nc; ++c) R->rp[c] = 0;
    for (int64_t i = 0; i < nf; ++i) ++R->rp[pcol[i] + 1];
    for (int64_t c = 0; c < nc; ++c) R->rp[c + 1] += R->rp[c];
    int64_t* next = xmalloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
    for (int64_t c = 0; c < nc; ++c) next[c] = R->rp[c];
    for (int64_t i = 0; i < nf; ++i) {
        const int64_t slot = next[pcol[i]]++;
        R->ci[slot] = i;
        R->va[slot] = pval[i];
    }
    free(next);
}

/* galerkin_product (amg.cpp:110-142): C = A*P by spmm_dist/spgemm_local
 * (dist.cpp:208-297, csr.cpp:206-272) with P one entry per row, then
 * A_c = R*C with R = transpose_block(P) (communication-free). */
static void galerkin(const csr_t* A, const int64_t* pcol, const double* pval, int64_t nc,
                     csr_t* Ac) {
    const int64_t n = A->n;
    /* C = A*P: row i gets (pcol[j], a_ij*pval[j]) in ascending j, merged. */
    csr_t Cm;
    csr_alloc(&Cm, n, nc, A->nnz);
    int64_t off = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t s = off;
        for (int64_t t = A->rp[i]; t < A->rp[i + 1]; ++t) {
            const int64_t j = A->ci[t];
            Cm.ci[off] = pcol[j];
            Cm.va[off] = A->va[t] * pval[j];
            ++off;
        }
        stable_sort_pairs(Cm.ci + s, Cm.va + s, off - s);
        off = s + merge_sorted(Cm.ci + s, Cm.va + s, off - s);
        Cm.rp[i + 1] = off;
    }
    Cm.nnz = off;
    csr_t R;
    transpose_p(pcol, pval, n, nc, &R);
    /* A_c = R*C: coarse row c collects R_ci * C_i,: over fine i ascending. */
    int64_t cap = Cm.nnz > 0 ? Cm.nnz : 1;
    csr_alloc(Ac, nc, nc, 0);
    Ac->ci = realloc(Ac->ci, sizeof(int64_t) * (size_t)cap);
    Ac->va = realloc(Ac->va, sizeof(double) * (size_t)cap);
    int64_t bufcap = 64;
    int64_t* bc = xmalloc(sizeof(int64_t) * (size_t)bufcap);
    double* bv = xmalloc(sizeof(double) * (size_t)bufcap);
    off = 0;
    for (int64_t c = 0; c < nc; ++c) {
        int64_t m = 0;
        for (int64_t t = R.rp[c]; t < R.rp[c + 1]; ++t) {
            const int64_t i = R.ci[t];
            const double r = R.va[t];
            for (int64_t u = Cm.rp[i]; u < Cm.rp[i + 1]; ++u) {
                if (m == bufcap) {
                    bufcap *= 2;
                    bc = realloc(bc, sizeof(int64_t) * (size_t)bufcap);
                    bv = realloc(bv, sizeof(double) * (size_t)bufcap);
                }
                bc[m] = Cm.ci[u];
                bv[m] = r * Cm.va[u];
                ++m;
            }
        }
        stable_sort_pairs(bc, bv, m);
        m = merge_sorted(bc, bv, m);
        if (off + m > cap) {
            while (off + m > cap) cap *= 2;
            Ac->ci = realloc(Ac->ci, sizeof(int64_t) * (size_t)cap);
            Ac->va = realloc(Ac->va, sizeof(double) * (size_t)cap);
        }
        memcpy(Ac->ci + off, bc, sizeof(int64_t) * (size_t)m);
        memcpy(Ac->va + off, bv, sizeof(double) * (size_t)m);
        off += m;
        Ac->rp[c + 1] = off;
    }
    Ac->nnz = off;
    free(bc);
    free(bv);
    csr_free(&R);
    csr_free(&Cm);
}

/* l1_diagonal_dist (cycle.cpp:15-35) */
static int l1_diagonal(const csr_t* A, double* d) {
    for (int64_t i = 0; i < A->n; ++i) {
        double acc = 0.0;
        for (int64_t t = A->rp[i]; t < A->rp[i + 1]; ++t) {
            if (A->ci[t] == i)
                acc += A->va[t];
            else
                acc += fabs(A->va[t]);
        }
        if (acc == 0.0)
            return fail(ST_SINGULAR_SMOOTHER, "l1_diagonal_dist: zero diagonal weight at global row %lld",
                        (long long)i);
        d[i] = acc;
    }
    return 0;
}

static void csr_copy(const csr_t* A, csr_t* B) {
    csr_alloc(B, A->n, A->ncols, A->nnz);
    memcpy(B->rp, A->rp, sizeof(int64_t) * (size_t)(A->n + 1));
    memcpy(B->ci, A->ci, sizeof(int64_t) * (size_t)A->nnz);
    memcpy(B->va, A->va, sizeof(double) * (size_t)A->nnz);
}

static void record_match(session_t* s, const int64_t* gm, int64_t n) {
    s->match = realloc(s->match, sizeof(int64_t*) * (size_t)(s->nmatch + 1));
    s->match[s->nmatch] = xmalloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    memcpy(s->match[s->nmatch], gm, sizeof(int64_t) * (size_t)n);
    s->match_n = realloc(s->match_n, sizeof(int64_t) * (size_t)(s->nmatch + 1));
    s->match_n[s->nmatch] = n;
    ++s->nmatch;
}

/* setup_hierarchy (amg.cpp:144-295). */
static int setup_hierarchy(session_t* s) {
    const orc_config* cfg = &s->cfg;
    const int p = cfg->nranks;
    if (cfg->aggregation_exponent < 1)
        return fail(ST_INVALID_ARGUMENT, "setup: aggregation exponent must be >= 1");
    if (cfg->max_levels < 1) return fail(ST_INVALID_ARGUMENT, "setup: max_levels must be >= 1");
    hierarchy_free(s);
    const double t0 = now_s();
    memset(&s->stats, 0, sizeof s->stats);

    s->lv = calloc((size_t)cfg->max_levels, sizeof(level_t));
    level_t* L0 = &s->lv[0];
    csr_copy(&s->A0, &L0->A);
    L0->starts = xmalloc(sizeof(int64_t) * (size_t)(p + 1));
    memcpy(L0->starts, s->starts0, sizeof(int64_t) * (size_t)(p + 1));
    L0->w = xmalloc(sizeof(double) * (size_t)L0->A.n);
    for (int64_t i = 0; i < L0->A.n; ++i) L0->w[i] = 1.0; /* w0 = 1 */
    s->nl = 1;

    while (s->nl < cfg->max_levels && s->lv[s->nl - 1].A.n > cfg->coarse_size_target) {
        level_t* Lf = &s->lv[s->nl - 1];
        const int level_index = s->nl;
        /* A_pair / w_pair (amg.cpp:168-169); A_pair is formed lazily: the
         * pairwise Galerkin product of the last step of a multi-step level is
         * discarded by the reference (amg.cpp:261-264), so it is skipped. */
        const csr_t* A_pair = &Lf->A;
        csr_t A_pair_own;
        int own_pair = 0;
        int64_t npair = Lf->A.n;
        int64_t* part = xmalloc(sizeof(int64_t) * (size_t)(p + 1));
        memcpy(part, Lf->starts, sizeof(int64_t) * (size_t)(p + 1));
        double* w_pair = xmalloc(sizeof(double) * (size_t)npair);
        memcpy(w_pair, Lf->w, sizeof(double) * (size_t)npair);
        int nsteps = 0;
        int64_t* comp_col = NULL; /* composed P (amg.cpp:79-85), fine rows of Lf */
        double* comp_val = NULL;

        for (int step = 0; step < cfg->aggregation_exponent; ++step) {
            if (npair <= cfg->coarse_size_target) break;
            if (step > 0 && A_pair == NULL) {
                /* unreachable: A_pair materialised below when a next step runs */
            }
            const double tm = now_s();
            int64_t* gm = xmalloc(sizeof(int64_t) * (size_t)npair);
            int64_t* counts = xmalloc(sizeof(int64_t) * (size_t)p);
            int64_t* agg = xmalloc(sizeof(int64_t) * (size_t)npair);
            double* pv = xmalloc(sizeof(double) * (size_t)npair);
            for (int r = 0; r < p; ++r) {
                const int64_t b = part[r], e = part[r + 1];
                match_block(A_pair, b, e, w_pair, cfg->matching_mode, gm + b);
                counts[r] = pairwise_prolongator(gm + b, w_pair + b, e - b, agg + b, pv + b);
                for (int64_t i = b; i < e; ++i)
                    if (gm[i] != -1) gm[i] += b;
            }
            s->stats.t_matching += now_s() - tm;
            record_match(s, gm, npair);
            /* allgather_partition (amg.cpp:19-27) */
            int64_t* cpart = xmalloc(sizeof(int64_t) * (size_t)(p + 1));
            cpart[0] = 0;
            for (int r = 0; r < p; ++r) cpart[r + 1] = cpart[r] + counts[r];
            const int64_t nc = cpart[p];
            if (nc == npair) {
                free(gm); free(counts); free(agg); free(pv); free(cpart); free(part); free(w_pair);
                free(comp_col); free(comp_val);
                if (own_pair) csr_free(&A_pair_own);
                return fail(ST_STAGNATION, "setup: coarsening stagnated at level %d (empty matching)",
                            level_index);
            }
            /* global coarse column (shift_columns, amg.cpp:29-34) */
            for (int r = 0; r < p; ++r)
                for (int64_t i = part[r]; i < part[r + 1]; ++i) agg[i] += cpart[r];
            /* w_next = R w (amg.cpp:244-247), ascending fine index */
            double* wn = xmalloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
            for (int64_t c = 0; c < nc; ++c) wn[c] = 0.0;
            for (int64_t i = 0; i < npair; ++i) wn[agg[i]] += pv[i] * w_pair[i];
            /* compose left to right: ((P1*P2)*P3) (amg.cpp:79-85 via spgemm_local) */
            if (step == 0) {
                comp_col = agg;
                comp_val = pv;
                agg = NULL;
                pv = NULL;
            } else {
                for (int64_t i = 0; i < Lf->A.n; ++i) {
                    const int64_t c = comp_col[i];
                    comp_val[i] = comp_val[i] * pv[c];
                    comp_col[i] = agg[c];
                }
            }
            ++nsteps;
            /* pairwise Galerkin (amg.cpp:240) only if the next step needs it
             * or this single step is the whole level */
            const int more = (step + 1 < cfg->aggregation_exponent) && (nc > cfg->coarse_size_target);
            const int single = !more && nsteps == 1;
            if (more || single) {
                const double tg = now_s();
                csr_t Anew;
                const int64_t* pc = step == 0 ? comp_col : agg;
                const double* pvv = step == 0 ? comp_val : pv;
                galerkin(A_pair, pc, pvv, nc, &Anew);
                s->stats.t_spmm += now_s() - tg;
                if (own_pair) csr_free(&A_pair_own);
                A_pair_own = Anew;
                own_pair = 1;
                A_pair = &A_pair_own;
            }
            free(agg);
            free(pv);
            free(gm);
            free(counts);
            free(part);
            part = cpart;
            free(w_pair);
            w_pair = wn;
            npair = nc;
        }
        if (nsteps == 0) {
            free(part);
            free(w_pair);
            if (own_pair) csr_free(&A_pair_own);
            break;
        }
        level_t* Lc = &s->lv[s->nl];
        memset(Lc, 0, sizeof *Lc);
        if (nsteps == 1) {
            Lc->A = A_pair_own; /* amg.cpp:261-262 */
            own_pair = 0;
        } else {
            const double tg = now_s();
            galerkin(&Lf->A, comp_col, comp_val, npair, &Lc->A); /* amg.cpp:263-264 */
            s->stats.t_spmm += now_s() - tg;
            if (own_pair) csr_free(&A_pair_own);
        }
        Lc->starts = part;
        Lc->w = w_pair;
        Lc->pcol = comp_col;
        Lc->pval = comp_val;
        transpose_p(comp_col, comp_val, Lf->A.n, npair, &Lc->R);
        ++s->nl;
    }

    int64_t nnz0 = s->lv[0].A.nnz;
    double opc = 0.0;
    for (int k = 0; k < s->nl; ++k) {
        level_t* L = &s->lv[k];
        L->l1 = xmalloc(sizeof(double) * (size_t)(L->A.n > 0 ? L->A.n : 1));
        CHECK(l1_diagonal(&L->A, L->l1));
        opc += (double)L->A.nnz / (double)nnz0; /* amg.cpp:286-289 */
    }
    (void)opc;
    s->stats.t_total = now_s() - t0;
    s->setup_done = 1;
    return 0;
}

/* ------------------------------------------------------------- cycle --- */

/* l1_jacobi_sweeps (cycle.cpp:37-62). x0 == NULL: zero start. */
static void jacobi(const level_t* L, const double* r, double* x, int have_x0, int nu, double omega,
                   double* tmp) {
    const int64_t n = L->A.n;
    if (!have_x0)
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    if (nu == 0) return;
    int sweep = 0;
    if (!have_x0) {
        for (int64_t i = 0; i < n; ++i) x[i] = omega * r[i] / L->l1[i];
        ++sweep;
    }
    for (; sweep < nu; ++sweep) {
        spmv(&L->A, x, tmp);
        for (int64_t i = 0; i < n; ++i) x[i] += omega * (r[i] - tmp[i]) / L->l1[i];
    }
}

/* vcycle_apply (cycle.cpp:86-112) with restrict_to_coarse (cycle.cpp:64-75)
 * and prolongate_add (cycle.cpp:77-84). */
static void vcycle(const session_t* s, int k, const double* r, double* x) {
    const level_t* L = &s->lv[k];
    const orc_config* c = &s->cfg;
    const int64_t n = L->A.n;
    double* tmp = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (k == s->nl - 1) {
        jacobi(L, r, x, 0, c->coarsest_sweeps, c->relax_weight, tmp);
        free(tmp);
        return;
    }
    jacobi(L, r, x, 0, c->pre_sweeps, c->relax_weight, tmp);
    spmv(&L->A, x, tmp);
    for (int64_t i = 0; i < n; ++i) tmp[i] = r[i] - tmp[i];
    const level_t* Lc = &s->lv[k + 1];
    const int64_t nc = Lc->A.n;
    double* rc = xmalloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
    double* e = xmalloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
    for (int64_t cc = 0; cc < nc; ++cc) {
        double sum = 0.0;
        for (int64_t t = Lc->R.rp[cc]; t < Lc->R.rp[cc + 1]; ++t) sum += Lc->R.va[t] * tmp[Lc->R.ci[t]];
        rc[cc] = sum;
    }
    vcycle(s, k + 1, rc, e);
    for (int64_t i = 0; i < n; ++i) x[i] += Lc->pval[i] * e[Lc->pcol[i]];
    jacobi(L, r, x, 1, c->post_sweeps, c->relax_weight, tmp);
    free(rc);
    free(e);
    free(tmp);
}

/* dot_dist (dist.cpp:299-306): per-rank sequential partial, then the
 * rank-ascending allreduce_sum (runtime.cpp:243-259). */
static double dot_dist(const session_t* s, const int64_t* starts, const double* x, const double* y) {
    double acc = 0.0;
    for (int r = 0; r < s->cfg.nranks; ++r) {
        double partial = 0.0;
        for (int64_t i = starts[r]; i < starts[r + 1]; ++i) partial += x[i] * y[i];
        acc += partial;
    }
    return acc;
}

/* ----------------------------------------------------------- public --- */

void orc_default_config(orc_config* c) {
    memset(c, 0, sizeof *c);
    c->stencil = 7;
    c->nx = c->ny = c->nz = 16;
    c->nranks = 1;
    c->aggregation_exponent = 3;
    c->coarse_size_target = 40; /* SetupConfig default, amg.hpp:19 */
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

const char* orc_last_error(void) { return g_err; }
int orc_last_status(void) { return g_status; }

/* Poisson generator, restated from SPEC.md:512-557 (the reference's
 * problem.cpp is absent): lexicographic rows (x fastest), diagonal 6 (7-point)
 * or 26 (27-point), -1 per in-grid neighbour, ascending columns. */
static void gen_poisson(int stencil, int64_t nx, int64_t ny, int64_t nz, csr_t* A) {
    const int64_t n = nx * ny * nz;
    const int64_t per = stencil == 27 ? 27 : 7;
    csr_alloc(A, n, n, n * per);
    int64_t off = 0;
    for (int64_t row = 0; row < n; ++row) {
        const int64_t i = row % nx, j = (row / nx) % ny, k = row / (nx * ny);
        for (int dk = -1; dk <= 1; ++dk)
            for (int dj = -1; dj <= 1; ++dj)
                for (int di = -1; di <= 1; ++di) {
                    const int man = abs(di) + abs(dj) + abs(dk);
                    if (stencil == 7 && man > 1) continue;
                    const int64_t ii = i + di, jj = j + dj, kk = k + dk;
                    if (ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz) continue;
                    A->ci[off] = ii + nx * (jj + ny * kk);
                    A->va[off] = man == 0 ? (stencil == 27 ? 26.0 : 6.0) : -1.0;
                    ++off;
                }
        A->rp[row + 1] = off;
    }
    A->nnz = off;
}

static session_t* new_session(const orc_config* cfg) {
    if (cfg->nranks < 1) {
        fail(ST_INVALID_ARGUMENT, "spawn_ranks: nranks must be >= 1");
        return NULL;
    }
    session_t* s = calloc(1, sizeof *s);
    s->cfg = *cfg;
    return s;
}

void* orc_create(const orc_config* cfg) {
    if (cfg->stencil != 7 && cfg->stencil != 27) {
        fail(ST_INVALID_ARGUMENT, "stencil must be 7 or 27");
        return NULL;
    }
    session_t* s = new_session(cfg);
    if (!s) return NULL;
    gen_poisson(cfg->stencil, cfg->nx, cfg->ny, cfg->nz, &s->A0);
    s->starts0 = xmalloc(sizeof(int64_t) * (size_t)(cfg->nranks + 1));
    partition_uniform(s->A0.n, cfg->nranks, s->starts0);
    g_status = 0;
    return s;
}

void* orc_create_csr(const orc_config* cfg, int64_t n, const int64_t* rp, const int64_t* ci,
                     const double* va) {
    session_t* s = new_session(cfg);
    if (!s) return NULL;
    s->cfg.stencil = 0;
    csr_alloc(&s->A0, n, n, rp[n]);
    memcpy(s->A0.rp, rp, sizeof(int64_t) * (size_t)(n + 1));
    memcpy(s->A0.ci, ci, sizeof(int64_t) * (size_t)rp[n]);
    memcpy(s->A0.va, va, sizeof(double) * (size_t)rp[n]);
    if (csr_validate(&s->A0)) {
        csr_free(&s->A0);
        free(s);
        return NULL;
    }
    s->starts0 = xmalloc(sizeof(int64_t) * (size_t)(cfg->nranks + 1));
    partition_uniform(n, cfg->nranks, s->starts0);
    g_status = 0;
    return s;
}

void orc_destroy(void* h) {
    session_t* s = h;
    if (!s) return;
    hierarchy_free(s);
    csr_free(&s->A0);
    free(s->starts0);
    free(s);
}

int64_t orc_global_n(void* h) { return ((session_t*)h)->A0.n; }
int64_t orc_global_nnz(void* h) { return ((session_t*)h)->A0.nnz; }

int orc_export_input(void* h, int64_t* rp, int64_t* ci, double* va) {
    session_t* s = h;
    memcpy(rp, s->A0.rp, sizeof(int64_t) * (size_t)(s->A0.n + 1));
    memcpy(ci, s->A0.ci, sizeof(int64_t) * (size_t)s->A0.nnz);
    memcpy(va, s->A0.va, sizeof(double) * (size_t)s->A0.nnz);
    return 0;
}

int orc_setup(void* h) {
    g_status = 0;
    return setup_hierarchy((session_t*)h);
}

int orc_num_levels(void* h) { return ((session_t*)h)->nl; }

double orc_opc(void* h) {
    session_t* s = h;
    double opc = 0.0;
    for (int k = 0; k < s->nl; ++k) opc += (double)s->lv[k].A.nnz / (double)s->lv[0].A.nnz;
    return opc;
}

int orc_get_setup_stats(void* h, orc_setup_stats* out) {
    *out = ((session_t*)h)->stats;
    return 0;
}

static int need_setup(session_t* s, int level) {
    if (!s->setup_done) return fail(ST_CONTRACT_VIOLATION, "setup not run");
    if (level < 0 || level >= s->nl) return fail(ST_INVALID_ARGUMENT, "level out of range");
    return 0;
}

int orc_level_size(void* h, int level, int64_t* n, int64_t* nnz) {
    session_t* s = h;
    CHECK(need_setup(s, level));
    *n = s->lv[level].A.n;
    *nnz = s->lv[level].A.nnz;
    return 0;
}

int orc_level_partition(void* h, int level, int64_t* starts) {
    session_t* s = h;
    CHECK(need_setup(s, level));
    memcpy(starts, s->lv[level].starts, sizeof(int64_t) * (size_t)(s->cfg.nranks + 1));
    return 0;
}

int orc_export_level(void* h, int level, int64_t* rp, int64_t* ci, double* va, double* w,
                     double* l1) {
    session_t* s = h;
    CHECK(need_setup(s, level));
    const level_t* L = &s->lv[level];
    if (rp) memcpy(rp, L->A.rp, sizeof(int64_t) * (size_t)(L->A.n + 1));
    if (ci) memcpy(ci, L->A.ci, sizeof(int64_t) * (size_t)L->A.nnz);
    if (va) memcpy(va, L->A.va, sizeof(double) * (size_t)L->A.nnz);
    if (w) memcpy(w, L->w, sizeof(double) * (size_t)L->A.n);
    if (l1) memcpy(l1, L->l1, sizeof(double) * (size_t)L->A.n);
    return 0;
}

int orc_export_prolongator(void* h, int level, int64_t* col, double* val) {
    session_t* s = h;
    CHECK(need_setup(s, level));
    if (level < 1) return fail(ST_INVALID_ARGUMENT, "prolongator level must be >= 1");
    const int64_t nf = s->lv[level - 1].A.n;
    memcpy(col, s->lv[level].pcol, sizeof(int64_t) * (size_t)nf);
    memcpy(val, s->lv[level].pval, sizeof(double) * (size_t)nf);
    return 0;
}

int orc_num_matchings(void* h) { return ((session_t*)h)->nmatch; }

int64_t orc_matching_size(void* h, int step) {
    session_t* s = h;
    return (step < 0 || step >= s->nmatch) ? -1 : s->match_n[step];
}

int orc_export_matching(void* h, int step, int64_t* mate) {
    session_t* s = h;
    if (step < 0 || step >= s->nmatch) return fail(ST_INVALID_ARGUMENT, "matching step out of range");
    memcpy(mate, s->match[step], sizeof(int64_t) * (size_t)s->match_n[step]);
    return 0;
}

int orc_spmv(void* h, int level, const double* x, double* y) {
    session_t* s = h;
    CHECK(need_setup(s, level));
    spmv(&s->lv[level].A, x, y);
    return 0;
}

int orc_vcycle(void* h, const double* r, double* x) {
    session_t* s = h;
    CHECK(need_setup(s, 0));
    vcycle(s, 0, r, x);
    return 0;
}

/* Flexible PCG (Alg. 1), same iteration
 * convention and vector-update order as ref_driver.cpp's orc_solve. */
int orc_set_solve(void* h, double rtol, int max_iters) {
    session_t* s = h;
    s->cfg.rtol = rtol;
    s->cfg.max_iters = max_iters;
    return 0;
}

int orc_solve(void* h, const double* b, double* u_out, double* hist, int hist_cap, int* iters,
              double* relres, double* t_solve) {
    session_t* s = h;
    const orc_config* c = &s->cfg;
    if (c->precflag && !s->setup_done) return fail(ST_CONTRACT_VIOLATION, "setup not run");
    const csr_t* A = &s->A0;
    const int64_t* starts = s->starts0;
    const int64_t n = A->n;
    const double t0 = now_s();
    double* u = calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    double* r = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* w = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* v = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* d = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* q = xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int k = 0, rc = 0;
    double rel = 1.0;
    if (hist && hist_cap > 0) hist[0] = 1.0;
    spmv(A, u, r);
    for (int64_t i = 0; i < n; ++i) r[i] = (b ? b[i] : 1.0) - r[i];
    const double rnorm0 = sqrt(dot_dist(s, starts, r, r));
    if (rnorm0 != 0.0) {
        if (c->precflag)
            vcycle(s, 0, r, w);
        else
            memcpy(w, r, sizeof(double) * (size_t)n);
        memcpy(d, w, sizeof(double) * (size_t)n);
        spmv(A, w, v);
        memcpy(q, v, sizeof(double) * (size_t)n);
        const double alpha = dot_dist(s, starts, w, r);
        double rho = dot_dist(s, starts, w, v);
        if (rho == 0.0 || !isfinite(rho)) {
            rc = fail(ST_BREAKDOWN, "fcg: breakdown at iteration 0");
            goto out;
        }
        const double a0 = alpha / rho;
        for (int64_t i = 0; i < n; ++i) {
            u[i] = u[i] + a0 * d[i];
            r[i] = r[i] - a0 * q[i];
        }
        k = 1;
        rel = sqrt(dot_dist(s, starts, r, r)) / rnorm0;
        if (hist && hist_cap > 1) hist[1] = rel;
        while (!(rel < c->rtol) && k < c->max_iters) {
            if (c->precflag)
                vcycle(s, 0, r, w);
            else
                memcpy(w, r, sizeof(double) * (size_t)n);
            spmv(A, w, v);
            const double al = dot_dist(s, starts, w, r);
            const double be = dot_dist(s, starts, w, v);
            const double ga = dot_dist(s, starts, w, q);
            const double rho_new = be - ga * ga / rho;
            if (rho_new == 0.0 || !isfinite(rho_new)) {
                rc = fail(ST_BREAKDOWN, "fcg: breakdown at iteration %d", k);
                goto out;
            }
            const double cc = ga / rho;
            const double a = al / rho_new;
            for (int64_t i = 0; i < n; ++i) {
                d[i] = w[i] - cc * d[i];
                q[i] = v[i] - cc * q[i];
                u[i] = u[i] + a * d[i];
                r[i] = r[i] - a * q[i];
            }
            rho = rho_new;
            ++k;
            rel = sqrt(dot_dist(s, starts, r, r)) / rnorm0;
            if (hist && k < hist_cap) hist[k] = rel;
        }
    }
out:
    if (t_solve) *t_solve = now_s() - t0;
    if (iters) *iters = k;
    if (relres) *relres = rel;
    if (u_out) memcpy(u_out, u, sizeof(double) * (size_t)n);
    free(u);
    free(r);
    free(w);
    free(v);
    free(d);
    free(q);
    return rc;
}
