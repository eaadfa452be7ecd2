// p2p.cuh -- halo exchange by direct NVLink stores into the neighbours'
// memory (CUDA IPC), replacing NCCL send/recv on the solve path.
//
// Measured on the B200 pair: a 512 KB NCCL send/recv takes ~51 us alone and
// ~255 us next to an HBM-bound kernel, so at level 0 of a 256^3 slab the
// exchange finished only after the interior rows (halo trace).
// Here the sender's pack kernel stores its boundary values straight into the
// receiver's staging buffer (one per level, double-buffered by exchange
// parity) and raises a per-sender flag with a system-scope release; the
// receiver's unpack kernel waits for the flag, copies staging -> halo slots.
// Parity double-buffering needs no acknowledgement: a sender can be at most
// one exchange ahead (its next exchange needs the receiver's data of this
// one).  Both kernels run on the communication stream.
#pragma once

#include <vector>

#include "matrix.cuh"

namespace pb {

struct P2PHalo {
    bool ok = false;
    int64_t n_halo = 0;
    double* staging = nullptr;                 // 2 * n_halo (cudaMalloc, IPC-exported)
    unsigned long long* flags = nullptr;       // nranks slots (cudaMalloc, IPC-exported); slot = sender
    std::vector<double*> peer_staging;         // per send peer: its staging + my offset (parity 0)
    std::vector<int64_t> peer_stride;          // per send peer: its n_halo (parity stride)
    std::vector<unsigned long long*> peer_flag;  // per send peer: its flags[my rank]
    std::vector<void*> opened;                 // IPC mappings to close
    DBuf<unsigned long long> ctr;              // [0] exchanges received, [2] pull / [3] split blocks done, [4] pushes, [5] push blocks done
    DBuf<double*> d_peer_staging;              // device copies of the per-peer tables
    DBuf<int64_t> d_peer_stride;
    DBuf<unsigned long long*> d_peer_flag;
    DBuf<int> d_recv_from;                     // recv peer ranks (flags to wait for)
};

// Collective over the ranks sharing the level; leaves P.ok = false (NCCL
// path stays) when IPC is unavailable.
void p2p_setup(Runtime& rt, const HaloPlan& H, P2PHalo& P, cudaStream_t s);
void p2p_destroy(P2PHalo& P);
// Close this rank's mappings of peer buffers (no free); see p2p.cu.
void p2p_close_imports(P2PHalo& P);
// x_halo <- the owners' x (push from every rank, then pull), on stream s.
void p2p_exchange(const HaloPlan& H, P2PHalo& P, const double* x_owned, double* x_halo, cudaStream_t s);
// Push only: the consumer is a split launch reading the staging slot itself
// (sell_apply_split / sell_spmv_dots_split with p2p_halo_src).
void p2p_push(const HaloPlan& H, P2PHalo& P, const double* x_owned, cudaStream_t s);
HaloSrc p2p_halo_src(const HaloPlan& H, P2PHalo& P);

// Small allgather (the FCG dot partials) by NVLink stores: every rank writes
// its K doubles into every rank's mailbox (parity double-buffered), raises
// its flag there, waits for all flags, copies the mailbox out in rank order.
struct P2PGather {
    bool ok = false;
    int nranks = 0, rank = 0, kmax = 0;
    double* mail = nullptr;                      // 2 * nranks * kmax (IPC-exported)
    unsigned long long* flags = nullptr;         // nranks (IPC-exported)
    std::vector<double*> peer_mail;              // per rank (own: local pointer)
    std::vector<unsigned long long*> peer_flags;
    std::vector<void*> opened;
    DBuf<unsigned long long> ctr;                // [0] gathers done
    DBuf<double*> d_peer_mail;
    DBuf<unsigned long long*> d_peer_flags;
    ~P2PGather();
};

void p2p_gather_setup(Runtime& rt, P2PGather& G, int kmax, cudaStream_t s);

// Segment allgather into one replicated vector (the restricted right-hand
// side entering the first replicated coarse level): every rank stores its
// rows [off, off + cnt) straight into every rank's copy of the vector over
// NVLink, raises its flag there and waits for all flags.  Single-buffered:
// consecutive gathers must be separated by a collective step (the FCG dot
// allgather of every iteration does it; Solver::vcycle adds one).
constexpr int kSegMaxRanks = 16;
struct P2PSegGather {
    bool ok = false;
    int nranks = 0, rank = 0;
    int64_t total = 0;
    double* buf = nullptr;                       // total doubles (IPC-exported): the gathered vector
    unsigned long long* flags = nullptr;         // nranks (IPC-exported), slot = sender
    std::vector<double*> peer_buf;               // per rank (own: buf)
    std::vector<unsigned long long*> peer_flags;
    std::vector<void*> opened;
    DBuf<unsigned long long> ctr;                // [0] gathers done, [1] blocks done
    ~P2PSegGather();
};
// Collective; leaves G.ok = false (NCCL stays) when IPC is unavailable.
void p2p_seg_setup(Runtime& rt, P2PSegGather& G, int64_t total, cudaStream_t s);
void p2p_seg_destroy(P2PSegGather& G);
void p2p_seg_close_imports(P2PSegGather& G);
// G.buf[off + i] = src[i] on every rank, all ranks' segments present when the
// kernel completes (stream s, graph-capturable).
void p2p_seg_gather(P2PSegGather& G, const double* src, int64_t cnt, int64_t off, cudaStream_t s);
// recv[r*K + k] = rank r's send[k], on stream s (device-side, graph-capturable).
void p2p_allgather(P2PGather& G, const double* send, double* recv, int K, cudaStream_t s);

}  // namespace pb

