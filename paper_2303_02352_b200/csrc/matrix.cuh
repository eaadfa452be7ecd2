// matrix.cuh -- device data layout of one rank's share of a hierarchy level.
//
// HBM layout (per level, per rank):
//   DevMatrix  : owned rows in CSR, int64 row_ptr, int32 LOCAL column ids
//                ([0,n) owned, [n, n+n_halo) halo slots), f64 values.  Each
//                row keeps the reference's column order (ascending GLOBAL id,
//                csr.hpp:10-11), so every per-row sum runs in the reference
//                order (dist.cpp:164-187).
//   HaloPlan   : HaloPlan (dist.hpp:50-65): sorted global ids of the halo
//                slots (recv_ids), per-peer receive ranges, per-peer send
//                lists of owned local ids, a packed send buffer.
//   Sell       : the solve-time copy of a row set in SELL-32 (slices of 32
//                consecutive rows stored column-major, padded per slice to
//                the slice's longest row, pad column = -1).  One warp owns a
//                slice, one lane a row: every val/col load of a warp is one
//                contiguous 256 B / 128 B transaction and the lane's sum runs
//                over its row in CSR order, bitwise equal to spmv_local.
//                Interior and boundary rows get separate Sells so halo
//                exchange overlaps interior rows (dist.cpp:190-198).
#pragma once

#include <vector>

#include "common.cuh"
#include "runtime.cuh"

namespace pb {

struct HaloPlan {
    int64_t n_halo = 0;
    DBuf<int64_t> recv_gid;                  // sorted global ids of the halo slots
    std::vector<int> recv_peers;             // source ranks, ascending
    std::vector<int64_t> recv_off;           // npeers+1 offsets into the halo region
    std::vector<int> send_peers;             // destination ranks, ascending
    std::vector<int64_t> send_off;           // npeers+1 offsets into send_idx
    DBuf<int32_t> send_idx;                  // owned local ids to pack, per peer
    DBuf<double> send_buf;                   // packed values
    DBuf<int64_t> send_buf_i64;              // packed ids (setup-time P exchange)
    bool has_traffic() const { return n_halo > 0 || !send_peers.empty(); }
};

struct DevMatrix {
    int64_t n = 0;          // owned rows
    int64_t nnz = 0;
    int64_t row_begin = 0;  // global id of owned row 0 (= owned column range begin)
    int64_t n_global = 0;
    std::vector<int64_t> starts;  // row partition (nranks+1)
    DBuf<int64_t> rp;
    DBuf<int32_t> col;
    DBuf<double> val;
    HaloPlan halo;
    DBuf<int32_t> boundary_rows;  // rows with at least one halo column (ascending)
    DBuf<int32_t> interior_rows;  // the others (ascending); empty when no halo
    int64_t n_boundary = 0;
};

struct Sell {
    // PAT  : one byte per ROW naming its row pattern (the row's full sequence
    //        of (column - row, value) entries; <= 255 distinct patterns); the
    //        pattern table (16-byte records) and the per-pattern l1 diagonal
    //        live in global memory (L1-resident).  Preferred when it applies.
    // DICT : one byte per entry (<= 255 distinct (column - row, value)).
    // PLAIN: int32 column + f64 value per entry.
    // STEN : every row an order-preserving subset of one main pattern: PAT's
    //        byte per row names the subset (absent-record mask + l1 diagonal);
    //        the main records and the per-pattern data travel as a kernel
    //        parameter.  Preferred whenever it applies (sell_sten.cuh).
    enum Format { kPlain = 0, kDict = 1, kPat = 2, kSten = 3, kCoded = 4 };
    int format = kPlain;
    int64_t nrows = 0, nslices = 0, padded_nnz = 0;
    DBuf<int64_t> slice_off;  // nslices+1; elements (PLAIN) or 32-bit code words (DICT), multiples of 32
    DBuf<int32_t> col;        // PLAIN: padded local column ids, -1 = pad
    DBuf<double> val;         // PLAIN: values
    DBuf<uint32_t> code;      // DICT: 4 one-byte codes per word, 0xFF = pad; [slice][word][lane]
    int words = 0;            // DICT: words per row (uniform)
    DBuf<ulonglong2> dict;    // DICT: 256 records {value bits, column - row}; [255] = pad {0, 0}
    std::vector<ulonglong2> hdict;  // DICT: host copy, passed to the kernels as a __grid_constant__ parameter
    int ndict = 0;
    DBuf<uint8_t> pid;        // PAT: pattern id per row (indexed by row id)
    DBuf<ulonglong2> ptab;    // PAT: pattern records {value bits, column - row}
    DBuf<int2> pmeta;         // PAT: {first record, length} per pattern
    DBuf<double> pdiag;       // PAT: l1 diagonal per pattern (bitwise = l1_diagonal)
    DBuf<double> pinv;        // RN(1 / pdiag) per pattern (ddiv_recip; 0 = divide)
    int npat = 0, maxlen = 0;
    std::vector<ulonglong2> hptab;  // PAT host copies (STEN conversion)
    std::vector<int2> hpmeta;
    std::vector<double> hpdiag;
    int sten_L = 0, sten_offmin = 0, sten_offmax = 0;  // STEN: main pattern
    std::vector<int> sten_off;
    std::vector<double> sten_val;
    std::vector<uint32_t> sten_mask;  // per pattern: absent main records (L <= 32)
    std::vector<unsigned long long> sten_mask64;  // the same, any L <= 64
    int64_t xlen = 0;         // gathered vector length (owned + halo slots)
    DBuf<int32_t> rows;       // row id of each SELL row; empty = row0 + index
    int64_t row0 = 0;
};

// Operators of the SELL kernels (sell.cu)
enum SellOp { kSpmv = 0, kJacobi = 1, kResid = 2 };

struct SellOpArgs {
    int op = kSpmv;
    const double* x = nullptr;  // iterate (gathered)
    double* y = nullptr;        // output rows
    const double* r = nullptr;  // right-hand side
    const double* d = nullptr;  // l1 diagonal
    double omega = 1.0;
    int max_grid = 0;               // STEN: cap on CTAs (grid-stride), 0 = one CTA per row block
};

// ---- sparse.cu ----
// Global-column CSR (int64 row_ptr / col, device) of the owned rows ->
// DevMatrix with local columns and a halo plan (build_rows_to_receive +
// exchange_requests + build_spmv_plan, dist.cpp:45-120).  Takes ownership
// of the buffers.
void localize(Runtime& rt, DevMatrix& M, DBuf<int64_t>&& rp, DBuf<int64_t>&& gcol,
              DBuf<double>&& val, int64_t nnz);
// Global ids of M's columns (export).
void global_columns(const DevMatrix& M, int64_t* d_out, cudaStream_t s);
// ---- sell.cu ----
// SELL-32 copy of the rows listed in `rows` (nullptr = all rows); DICT
// encoding when allowed and the rows have <= 255 distinct (col-row, value).
// PAT is tried first (needs the level's l1 diagonal to verify the per-pattern
// diagonal bitwise), then DICT, then PLAIN.
void build_sell(const DevMatrix& M, const int32_t* rows, int64_t nrows, Sell& out, cudaStream_t s,
                int storage = -1, const double* l1 = nullptr);
// One byte per value into <= 256 distinct values (exact bits); false (and
// nothing built) when there are more.
bool build_value_codes(const double* v, int64_t n, DBuf<uint8_t>& code, std::vector<double>& table, cudaStream_t s);
double sell_bytes(const Sell& S);               // stored matrix bytes of the format
double sell_op_bytes(const Sell& S, int op);    // algorithmic bytes of one launch (op, or -1 = spmv+dots)
// l1_diagonal_dist (cycle.cpp:15-35); throws singular_smoother.
void l1_diagonal(const DevMatrix& M, double* d_out, cudaStream_t s);
// x_halo[h] <- owner's x for every halo slot (pack, NCCL send/recv). On `s`.
void halo_exchange(Runtime& rt, HaloPlan& H, const double* x_owned, double* x_halo, cudaStream_t s);
// Same for an (int64, f64) pair of per-row arrays (setup-time P exchange).
void halo_exchange_pair(Runtime& rt, HaloPlan& H, const int64_t* a_owned, int64_t* a_halo,
                        const double* b_owned, double* b_halo, cudaStream_t s);

// Apply one operator (SellOp) on a Sell; all row sums in CSR order, exactly rounded.
void sell_apply(const Sell& S, const SellOpArgs& o, cudaStream_t s);
// v = A w plus per-block partials of (w.r, w.v, w.q) (FCG lines 10-13).
// Returns the number of partial triples written.
// cap > 0: at most cap CTAs (STEN grid-strides; leaves SM slots to concurrent kernels).
int sell_spmv_dots(const Sell& S, const double* w, double* v, const double* r, const double* q,
                   double* partials, int max_blocks, cudaStream_t s, int cap = 0);
int sell_dots_grid(const Sell& S, int cap = 0);
// Halo delivered by NVLink direct stores (p2p.cu): where the boundary rows of
// a split launch find it and how they learn it has arrived.
struct HaloSrc {
    const unsigned long long* flags = nullptr;  // flag slot per sender rank
    int nfrom = 0;
    int from[8] = {};
    const double* staging = nullptr;            // parity stride nhalo
    int64_t nhalo = 0;
    unsigned long long* ctr = nullptr;          // [0] exchanges done, [3] boundary blocks done,
                                                // [4] pushes done, [5] push blocks done
    // fused push (npeers > 0): this rank's boundary values go to the
    // neighbours from the first blocks of the same launch
    bool fused = false;
    int npeers = 0;
    int64_t off[9] = {};                        // send_off
    double* dst[8] = {};                        // peer staging + my offset (parity 0)
    int64_t stride[8] = {};                     // peer parity stride
    unsigned long long* pflag[8] = {};          // peer flag slot of this rank
    const int32_t* send_idx = nullptr;
};
// Interior (contiguous STEN) + boundary (STEN) rows in one launch; the
// boundary blocks wait for the neighbours' pushes of this exchange.
bool sell_split_ok(const Sell& interior, const Sell& boundary);
// The row set runs the 27-point marching kernels (sell_sten.cuh): contiguous
// rows, full 3x3x3 main pattern, large enough for two waves of 4 CTAs/SM.
bool sell_march_ok(const Sell& S);
// STEN with a main pattern of up to 64 records (split-launch boundary rows
// only); false (S unusable) when the rows do not nest into one.
bool build_sten_wide(const DevMatrix& M, const int32_t* rows, int64_t nrows, Sell& S, cudaStream_t s,
                     const double* l1);
void sell_apply_split(const Sell& interior, const Sell& boundary, const SellOpArgs& o, const HaloSrc& hs,
                      cudaStream_t s);
int sell_split_dots_grid(const Sell& interior, const Sell& boundary);
int sell_spmv_dots_split(const Sell& interior, const Sell& boundary, const double* w, double* v, const double* r,
                         const double* q, double* partials, int max_blocks, const HaloSrc& hs, cudaStream_t s);
// The coarsest level's zero start + nu-1 l1-Jacobi sweeps in one cluster
// launch (halo-free STEN, <= 16384 rows); false when not applicable.
bool sell_coarse_solve(const Sell& S, const double* rhs, double* x, int nu, double omega, cudaStream_t s);

}  // namespace pb
