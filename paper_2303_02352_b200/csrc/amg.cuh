// amg.cuh -- the device-resident AMG hierarchy (Hierarchy / Level,
// amg.hpp:27-58) and the entry points of setup.cu / solve.cu.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "matrix.cuh"
#include "p2p.cuh"

namespace pb {

struct SetupConfig {  // SetupConfig (amg.hpp:17-23)
    int aggregation_exponent = 3;
    int64_t coarse_size_target = 40;
    int max_levels = 40;
    // replay (MatchingTrace, amg.hpp:13-23): global mates per pairwise step
    std::vector<const int64_t*> replay;
    std::vector<int64_t> replay_sizes;
    int storage = -1;                  // pairamg_storage (-1 auto)
    int64_t replicate_rows = 2500000;  // nranks > 1: replicate coarse levels up to this size
    bool setup_overlap = false;        // nranks > 1: P halo exchange on the comm stream
};

struct CycleConfig {  // CycleConfig (cycle.hpp:7-12)
    int pre_sweeps = 4, post_sweeps = 4, coarsest_sweeps = 20;
    double relax_weight = 1.0;
};

struct Level {
    DevMatrix A;
    DBuf<double> w;   // smooth vector
    DBuf<double> l1;  // l1-Jacobi diagonal
    // transfer from the finer level (k >= 1): block prolongator, local ids
    DBuf<int32_t> pcol;  // per fine row of level k-1: local coarse row
    DBuf<double> pval;
    DBuf<int64_t> rrp;   // R = P^T: local coarse rows -> local fine rows ascending
    DBuf<int32_t> rcol;
    DBuf<double> rval;
    // solve-time byte codes of pval / rval (<= 256 distinct values each)
    DBuf<uint8_t> pcode, rcode;
    std::vector<double> ptab, rtab;
    // solve-time layout
    Sell sell_all;           // all rows (no halo)
    Sell sell_int, sell_bnd; // interior / boundary rows (halo present)
    Sell sell_bndw;          // boundary rows as wide STEN (split launches) when sell_bnd is not STEN
    const Sell& split_bnd() const { return sell_bnd.format == Sell::kSten ? sell_bnd : sell_bndw; }
    // V-cycle work vectors
    DBuf<double> x, xt;      // n + n_halo (ping-pong iterates)
    DBuf<double> rhs, res;   // n
    P2PHalo p2p;             // NVLink direct-store halo exchange (multi-rank)
    ~Level() { p2p_destroy(p2p); }
};

struct SetupStats {  // SetupStats (amg.hpp:40-47)
    double t_total = 0, t_matching = 0, t_spmm = 0, t_spmm_comm = 0;
    int64_t matching_messages = 0, rc_messages = 0;
};

struct Hierarchy {
    std::vector<std::unique_ptr<Level>> levels;
    std::vector<int64_t> level_sizes, level_nnz;  // global
    double opc = 1.0;
    SetupStats stats;
    std::vector<std::string> warnings;
    std::vector<DBuf<int64_t>> matchings;  // owned-block global mates per pairwise step
    int nl() const { return static_cast<int>(levels.size()); }

    // Coarse-level replication (nranks > 1): levels >= rep_level are also held
    // in full on every rank (rep[k - rep_level]); the V-cycle gathers the
    // restricted right-hand side once (padded ncclAllGather) and runs those
    // levels redundantly without halo traffic.  Row sums are the same, so the
    // result is bit-identical to the distributed cycle.
    int rep_level = -1;
    std::vector<std::unique_ptr<Level>> rep;
    std::vector<int64_t> rep_counts, rep_offsets;  // owned rows of level rep_level per rank
    int64_t rep_max = 0;
    DBuf<double> rep_send, rep_recv;                // rep_max, nranks * rep_max
};

// Replicate every level whose global size is <= max_rows (nranks > 1).
void replicate_coarse_levels(Runtime& rt, Hierarchy& h, int64_t max_rows, int storage);
// Padded allgather of per-rank segments (counts[r] elements each) into a
// contiguous vector on `s` (graph-capturable).
void gather_segments(Runtime& rt, const double* d_local, int64_t count, double* sendbuf, double* recvbuf,
                     int64_t maxcount, const std::vector<int64_t>& offsets, const std::vector<int64_t>& counts,
                     double* d_out, cudaStream_t s);

// Parallel Suitor on a weighted graph CSR already on the device (the
// k_suitor / k_mate kernels of the setup; exposed for matching KATs).
void suitor_match_device(const int64_t* rp, const int32_t* col, const double* w, int64_t n, int64_t* mate,
                         cudaStream_t s);

// setup_hierarchy (amg.cpp:144-295) on the device.  The input is the owned
// row block in global-column CSR (device buffers, ownership taken).
void setup_hierarchy(Runtime& rt, Hierarchy& h, std::vector<int64_t> starts, DBuf<int64_t>&& rp,
                     DBuf<int64_t>&& gcol, DBuf<double>&& val, int64_t nnz, const double* d_w0,
                     const SetupConfig& cfg);

}  // namespace pb
