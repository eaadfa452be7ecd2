// runtime.cuh -- one rank = one GPU = one host thread (or process).
//
// Replaces the reference's in-process mailbox runtime (RankCtx,
// runtime.hpp:71-108; runtime.cpp:57-289) with NCCL over NVLink/NVSwitch:
//   send/recv (tags 101/102)  -> ncclSend/ncclRecv inside ncclGroupStart/End
//   allgather                 -> ncclAllGather
//   alltoallv                 -> counts by ncclAllGather, payload by grouped send/recv
//   allreduce_sum             -> ncclAllGather + rank-ascending sum, which keeps the
//                                reference's deterministic cross-rank order
//                                (runtime.cpp:250-258)
// CommStats (runtime.hpp:42-54) is kept as instrumentation.
#pragma once

#include <nccl.h>

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
    int64_t total_messages() const { return p2p_messages + collective_messages; }
};

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

    // Device-level: gather `count` doubles from every rank into recv
    // (nranks*count), enqueued on stream s (graph-capturable).
    void allgather_f64(const double* send, double* recv, size_t count, cudaStream_t s);

private:
    void warmup();
    int device_ = 0, rank_ = 0, nranks_ = 1;
    ncclComm_t comm_ = nullptr;
    cudaStream_t stream_ = nullptr, comm_stream_ = nullptr;
    CommStats stats_;
};

}  // namespace pb
