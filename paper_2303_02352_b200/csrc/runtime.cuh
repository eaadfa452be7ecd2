// runtime.cuh -- one rank = one host thread (or process) driving one GPU.
//
// Replaces the reference's in-process mailbox runtime (RankCtx,
// runtime.hpp:71-108; runtime.cpp:57-289) with two transports behind the
// same collective interface:
//
//  * NCCL (one process or thread per GPU, joined by an NCCL unique id):
//      send/recv (tags 101/102)  -> ncclSend/ncclRecv inside ncclGroupStart/End
//      allgather                 -> ncclAllGather
//      alltoallv                 -> counts by ncclAllGather, payload by grouped send/recv
//      allreduce_sum             -> ncclAllGather + rank-ascending sum, which keeps the
//                                   reference's deterministic cross-rank order
//                                   (runtime.cpp:250-258)
//  * LOCAL (ranks are threads of one process, as the reference's
//    spawn_ranks, runtime.cpp:92-152; joined by an id from
//    pairamg_comm_local_id): host collectives meet in a shared hub (mutex +
//    condition variable, generation barrier, a deadlock timeout like the
//    reference's timed receive, runtime.cpp:184-205); device payloads are
//    copied peer-to-peer between the ranks' buffers.  Several ranks may share
//    one GPU, which lets every multi-rank path run on a single B200.  The
//    solve-time exchanges (halos, dot allgather, replicated-rhs gather) use
//    the same NVLink/P2P flag protocol as across processes (p2p.cu), with raw
//    pointers instead of CUDA IPC handles.
//
// CommStats (runtime.hpp:42-54) is kept as instrumentation.
#pragma once

#include <nccl.h>

#include <memory>
#include <vector>

#include "common.cuh"

namespace pb {

#define PB_NCCL(call)                                                                          \
    do {                                                                                       \
        ncclResult_t r__ = (call);                                                             \
        if (r__ != ncclSuccess)                                                                \
            ::pb::fail(PAIRAMG_INTERNAL, std::string("NCCL error ") + ncclGetErrorString(r__) + \
                                             " at " __FILE__ ":" + std::to_string(__LINE__));  \
    } while (0)

struct CommStats {
    int64_t p2p_messages = 0, p2p_bytes = 0;
    int64_t collective_messages = 0, collective_bytes = 0;
    int64_t allgathers = 0, alltoallvs = 0, allreduces = 0;
    // solve-path exchanges enqueued on a stream (counted at enqueue; a
    // captured graph replays exactly what was counted while capturing)
    int64_t device_reductions = 0;  // FCG dot / norm allgathers
    int64_t halo_exchanges = 0;     // halo exchanges of x (any transport)
    int64_t halo_bytes = 0;         // halo values received by those exchanges (8 B each)
    int64_t total_messages() const { return p2p_messages + collective_messages; }
};

struct LocalHub;  // runtime.cu

// 128-byte rank-join ids: an NCCL unique id, or a LOCAL hub id (magic prefix).
bool is_local_id(const uint8_t* id);
void make_local_id(uint8_t id[128]);

class Runtime {
public:
    Runtime(int device, int rank, int nranks, const uint8_t* id);
    ~Runtime();
    Runtime(const Runtime&) = delete;
    Runtime& operator=(const Runtime&) = delete;

    int device() const { return device_; }
    int rank() const { return rank_; }
    int nranks() const { return nranks_; }
    ncclComm_t nccl() const { return comm_; }
    bool local() const { return hub_ != nullptr; }
    // Every rank of a LOCAL runtime on the same GPU: kernels whose blocks wait
    // for a peer rank must then not be mixed with long grids (no split launches).
    bool shared_device() const { return shared_device_; }
    cudaStream_t stream() const { return stream_; }
    cudaStream_t comm_stream() const { return comm_stream_; }
    CommStats& stats() { return stats_; }

    // Host-level collectives (setup path; synchronize the compute stream).
    std::vector<int64_t> allgather_i64(int64_t x);
    // nranks * n bytes: every rank's blob in rank order.
    std::vector<uint8_t> allgather_bytes(const void* data, size_t n);
    int64_t allreduce_sum_i64(int64_t x);
    // alltoallv of int64 id lists (setup only): chunks[d] goes to rank d; the
    // result holds what every source rank sent to us, in rank order.
    std::vector<std::vector<int64_t>> alltoallv_i64(const std::vector<std::vector<int64_t>>& chunks);
    // Setup-time allgather of `bytes` device bytes per rank into recv
    // (nranks * bytes, rank order), on the compute stream; synchronous.
    void allgather_dev(const void* send, void* recv, size_t bytes);
    // Setup-time point-to-point exchange of device buffers: sends[i] (bytes
    // send_bytes[i]) goes to rank send_to[i]; recvs[i] (recv_bytes[i]) comes
    // from rank recv_from[i].  Ordered after earlier work on s; synchronous
    // for LOCAL runtimes, enqueued on s for NCCL.  Pairs must match across ranks.
    void exchange_dev(const std::vector<int>& send_to, const std::vector<const void*>& sends,
                      const std::vector<size_t>& send_bytes, const std::vector<int>& recv_from,
                      const std::vector<void*>& recvs, const std::vector<size_t>& recv_bytes, cudaStream_t s);
    void barrier();
    // Synchronise stream s, polling NCCL's asynchronous error state and a
    // deadlock timeout (PAIRAMG_NCCL_TIMEOUT_S, default 600 s) while waiting,
    // as the reference's timed receive does (runtime.cpp:184-205): a peer
    // failure or a hang becomes PAIRAMG_INTERNAL / PAIRAMG_DEADLOCK instead of
    // blocking forever.  A plain cudaStreamSynchronize for one rank.
    void wait(cudaStream_t s);

    // Device-level: gather `count` doubles from every rank into recv
    // (nranks*count), enqueued on stream s (graph-capturable; NCCL only).
    void allgather_f64(const double* send, double* recv, size_t count, cudaStream_t s);

private:
    void warmup();
    // LOCAL: publish `mine`, wait for every rank, return all ranks' pointers;
    // the caller must call hub_release() once it no longer reads them.
    const std::vector<const void*>& hub_gather(const void* mine);
    void hub_release();
    int device_ = 0, rank_ = 0, nranks_ = 1;
    ncclComm_t comm_ = nullptr;
    std::shared_ptr<LocalHub> hub_;
    bool shared_device_ = false;
    cudaStream_t stream_ = nullptr, comm_stream_ = nullptr;
    CommStats stats_;
};

}  // namespace pb
