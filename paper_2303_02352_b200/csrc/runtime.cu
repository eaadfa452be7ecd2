// runtime.cu -- NCCL-backed rank runtime (see runtime.cuh).
#include "runtime.cuh"

#include <cstring>

namespace pb {

Runtime::Runtime(int device, int rank, int nranks, const uint8_t* id)
    : device_(device), rank_(rank), nranks_(nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks)
        fail(PAIRAMG_INVALID_ARGUMENT, "runtime: need 0 <= rank < nranks");
    PB_CUDA(cudaSetDevice(device));
    // The halo stream gets the highest priority: its pack + NCCL blocks are
    // dispatched ahead of the remaining interior-row blocks, so the exchange
    // overlaps the interior pass instead of queueing behind it.
    int prio_lo = 0, prio_hi = 0;
    PB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    PB_CUDA(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, prio_lo));
    PB_CUDA(cudaStreamCreateWithPriority(&comm_stream_, cudaStreamNonBlocking, prio_hi));
    // Keep freed stream-ordered allocations cached in the pool.
    cudaMemPool_t pool;
    PB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    PB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    if (nranks > 1) {
        if (!id) fail(PAIRAMG_INVALID_ARGUMENT, "runtime: NCCL unique id required for nranks > 1");
        ncclUniqueId uid;
        static_assert(sizeof(uid.internal) == 128, "NCCL unique id size");
        std::memcpy(uid.internal, id, 128);
        PB_NCCL(ncclCommInitRank(&comm_, nranks, uid, rank));
        warmup();
    }
}

// NCCL connects peers lazily, on the first collective / send-recv between
// them (buffers, IPC handles, proxy threads).  One tiny all-pairs exchange
// plus the collective kinds the library uses moves that one-time cost from
// the first setup into runtime creation.
void Runtime::warmup() {
    DBuf<double> buf(static_cast<size_t>(4 * nranks_), stream_);
    buf.zero(stream_);
    PB_NCCL(ncclGroupStart());
    for (int d = 0; d < nranks_; ++d) {
        if (d == rank_) continue;
        PB_NCCL(ncclSend(buf.get() + d, 1, ncclDouble, d, comm_, stream_));
        PB_NCCL(ncclRecv(buf.get() + nranks_ + d, 1, ncclDouble, d, comm_, stream_));
    }
    PB_NCCL(ncclGroupEnd());
    PB_NCCL(ncclAllGather(buf.get(), buf.get() + 2 * nranks_, 1, ncclDouble, comm_, stream_));
    PB_NCCL(ncclAllReduce(buf.get(), buf.get() + 3 * nranks_, 1, ncclDouble, ncclSum, comm_, stream_));
    PB_CUDA(cudaStreamSynchronize(stream_));
}

Runtime::~Runtime() {
    cudaSetDevice(device_);
    if (comm_) ncclCommDestroy(comm_);
    if (stream_) cudaStreamDestroy(stream_);
    if (comm_stream_) cudaStreamDestroy(comm_stream_);
}

std::vector<int64_t> Runtime::allgather_i64(int64_t x) {
    std::vector<int64_t> out(static_cast<size_t>(nranks_), x);
    if (nranks_ == 1) return out;
    stats_.allgathers += 1;
    stats_.collective_messages += nranks_ - 1;
    stats_.collective_bytes += 8 * (nranks_ - 1);
    DBuf<int64_t> d(static_cast<size_t>(nranks_) + 1, stream_);
    PB_CUDA(cudaMemcpyAsync(d.get() + nranks_, &x, 8, cudaMemcpyHostToDevice, stream_));
    PB_NCCL(ncclAllGather(d.get() + nranks_, d.get(), 1, ncclInt64, comm_, stream_));
    PB_CUDA(cudaMemcpyAsync(out.data(), d.get(), 8 * nranks_, cudaMemcpyDeviceToHost, stream_));
    PB_CUDA(cudaStreamSynchronize(stream_));
    return out;
}

std::vector<uint8_t> Runtime::allgather_bytes(const void* data, size_t n) {
    std::vector<uint8_t> out(static_cast<size_t>(nranks_) * n);
    if (nranks_ == 1) {
        std::memcpy(out.data(), data, n);
        return out;
    }
    stats_.allgathers += 1;
    DBuf<uint8_t> d(static_cast<size_t>(nranks_ + 1) * n, stream_);
    PB_CUDA(cudaMemcpyAsync(d.get() + nranks_ * n, data, n, cudaMemcpyHostToDevice, stream_));
    PB_NCCL(ncclAllGather(d.get() + nranks_ * n, d.get(), n, ncclUint8, comm_, stream_));
    PB_CUDA(cudaMemcpyAsync(out.data(), d.get(), static_cast<size_t>(nranks_) * n, cudaMemcpyDeviceToHost, stream_));
    PB_CUDA(cudaStreamSynchronize(stream_));
    return out;
}

int64_t Runtime::allreduce_sum_i64(int64_t x) {
    if (nranks_ == 1) return x;
    stats_.allreduces += 1;
    int64_t acc = 0;
    for (int64_t v : allgather_i64(x)) acc += v;  // rank-ascending (runtime.cpp:265-280)
    stats_.allgathers -= 1;
    return acc;
}

std::vector<std::vector<int64_t>> Runtime::alltoallv_i64(
    const std::vector<std::vector<int64_t>>& chunks) {
    const int p = nranks_;
    std::vector<std::vector<int64_t>> out(static_cast<size_t>(p));
    if (static_cast<int>(chunks.size()) != p)
        fail(PAIRAMG_CONTRACT_VIOLATION, "alltoallv: need one chunk per rank");
    out[rank_] = chunks[rank_];
    if (p == 1) return out;
    stats_.alltoallvs += 1;
    // counts matrix by allgather (row r = what rank r sends to each rank)
    std::vector<int64_t> mine(p);
    for (int d = 0; d < p; ++d) mine[d] = static_cast<int64_t>(chunks[d].size());
    DBuf<int64_t> dc(static_cast<size_t>(p) * p + p, stream_);
    PB_CUDA(cudaMemcpyAsync(dc.get() + p * p, mine.data(), 8 * p, cudaMemcpyHostToDevice, stream_));
    PB_NCCL(ncclAllGather(dc.get() + p * p, dc.get(), p, ncclInt64, comm_, stream_));
    std::vector<int64_t> counts(static_cast<size_t>(p) * p);
    PB_CUDA(cudaMemcpyAsync(counts.data(), dc.get(), 8 * p * p, cudaMemcpyDeviceToHost, stream_));
    PB_CUDA(cudaStreamSynchronize(stream_));
    int64_t send_total = 0, recv_total = 0;
    for (int d = 0; d < p; ++d) {
        if (d == rank_) continue;
        send_total += counts[rank_ * p + d];
        recv_total += counts[d * p + rank_];
    }
    DBuf<int64_t> sbuf(static_cast<size_t>(send_total), stream_), rbuf(static_cast<size_t>(recv_total), stream_);
    {
        std::vector<int64_t> flat;
        flat.reserve(static_cast<size_t>(send_total));
        for (int d = 0; d < p; ++d)
            if (d != rank_) flat.insert(flat.end(), chunks[d].begin(), chunks[d].end());
        if (send_total)
            PB_CUDA(cudaMemcpyAsync(sbuf.get(), flat.data(), 8 * send_total, cudaMemcpyHostToDevice, stream_));
    }
    PB_NCCL(ncclGroupStart());
    int64_t so = 0, ro = 0;
    for (int d = 0; d < p; ++d) {
        if (d == rank_) continue;
        const int64_t sc = counts[rank_ * p + d], rc = counts[d * p + rank_];
        if (sc) {
            PB_NCCL(ncclSend(sbuf.get() + so, static_cast<size_t>(sc), ncclInt64, d, comm_, stream_));
            stats_.collective_messages += 1;
            stats_.collective_bytes += 8 * sc;
        }
        if (rc) PB_NCCL(ncclRecv(rbuf.get() + ro, static_cast<size_t>(rc), ncclInt64, d, comm_, stream_));
        so += sc;
        ro += rc;
    }
    PB_NCCL(ncclGroupEnd());
    std::vector<int64_t> flat(static_cast<size_t>(recv_total));
    if (recv_total)
        PB_CUDA(cudaMemcpyAsync(flat.data(), rbuf.get(), 8 * recv_total, cudaMemcpyDeviceToHost, stream_));
    PB_CUDA(cudaStreamSynchronize(stream_));
    ro = 0;
    for (int s = 0; s < p; ++s) {
        if (s == rank_) continue;
        const int64_t rc = counts[s * p + rank_];
        out[s].assign(flat.begin() + ro, flat.begin() + ro + rc);
        ro += rc;
    }
    return out;
}

void Runtime::allgather_f64(const double* send, double* recv, size_t count, cudaStream_t s) {
    if (nranks_ == 1) {
        PB_CUDA(cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, s));
        return;
    }
    PB_NCCL(ncclAllGather(send, recv, count, ncclDouble, comm_, s));
}

}  // namespace pb
