// runtime.cu -- NCCL-backed and in-process (LOCAL) rank runtimes (see runtime.cuh).
#include "runtime.cuh"

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <thread>

#include <cuda.h>
#include <unistd.h>

namespace pb {

// ---- LOCAL transport: the in-process hub (spawn_ranks, runtime.cpp:92-152) ----

namespace {
constexpr char kLocalMagic[16] = "PAIRAMG-LOCAL-1";
}

bool is_local_id(const uint8_t* id) { return id && std::memcmp(id, kLocalMagic, sizeof kLocalMagic) == 0; }

void make_local_id(uint8_t id[128]) {
    static std::atomic<uint64_t> seq{0};
    std::memset(id, 0, 128);
    std::memcpy(id, kLocalMagic, sizeof kLocalMagic);
    const uint64_t v[3] = {static_cast<uint64_t>(getpid()), seq.fetch_add(1) + 1, std::random_device{}()};
    std::memcpy(id + 16, v, sizeof v);
}

struct LocalHub {
    int nranks = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    int joined = 0;
    bool aborted = false;
    std::string why;
    std::vector<const void*> slot;

    // Generation barrier with the reference's deadlock semantics: a peer
    // that never arrives (or left) fails the wait instead of hanging.
    void wait_all(int rank) {
        static const int timeout_s = env_int("PAIRAMG_LOCAL_TIMEOUT_S", 600);
        std::unique_lock<std::mutex> lk(m);
        if (aborted) fail(PAIRAMG_DEADLOCK, "rank " + std::to_string(rank) + ": " + why);
        const uint64_t g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return gen != g || aborted; })) {
            aborted = true;
            why = "collective timed out after " + std::to_string(timeout_s) + " s (a peer rank never arrived)";
            cv.notify_all();
        }
        if (gen == g) fail(PAIRAMG_DEADLOCK, "rank " + std::to_string(rank) + ": " + why);
    }
    void abort(const std::string& w) {
        std::lock_guard<std::mutex> lk(m);
        if (!aborted) {
            aborted = true;
            why = w;
        }
        cv.notify_all();
    }
};

namespace {
std::mutex g_hubs_m;
std::map<std::string, std::weak_ptr<LocalHub>> g_hubs;

std::shared_ptr<LocalHub> join_hub(const uint8_t* id, int nranks) {
    const std::string key(reinterpret_cast<const char*>(id), 128);
    std::lock_guard<std::mutex> lk(g_hubs_m);
    std::shared_ptr<LocalHub> h = g_hubs[key].lock();
    if (!h) {
        h = std::make_shared<LocalHub>();
        h->nranks = nranks;
        h->slot.assign(static_cast<size_t>(nranks), nullptr);
        g_hubs[key] = h;
    }
    if (h->nranks != nranks) fail(PAIRAMG_INVALID_ARGUMENT, "runtime: ranks of one local id disagree on nranks");
    if (++h->joined == nranks) g_hubs.erase(key);  // every rank holds it now
    return h;
}
}  // namespace

// Lazy kernel loading (CUDA 12 default) may synchronise the context at a
// kernel's first launch; with several ranks in one context, a rank spinning
// on a peer's halo flag would then deadlock the peer's first launch.
static bool lazy_module_loading() {
    using Fn = CUresult (*)(CUmoduleLoadingMode*);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
        cudaGetLastError();
        return true;  // unknown: assume the default (lazy)
    }
    CUmoduleLoadingMode m = CU_MODULE_LAZY_LOADING;
    if (reinterpret_cast<Fn>(p)(&m) != CUDA_SUCCESS) return true;
    return m == CU_MODULE_LAZY_LOADING;
}

const std::vector<const void*>& Runtime::hub_gather(const void* mine) {
    {
        std::lock_guard<std::mutex> lk(hub_->m);
        hub_->slot[static_cast<size_t>(rank_)] = mine;
    }
    hub_->wait_all(rank_);
    return hub_->slot;
}

void Runtime::hub_release() { hub_->wait_all(rank_); }

void Runtime::wait(cudaStream_t s) {
    if (!comm_) {
        PB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    static const int timeout_s = env_int("PAIRAMG_NCCL_TIMEOUT_S", 600);
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) PB_CUDA(q);
        ncclResult_t ae = ncclSuccess;
        PB_NCCL(ncclCommGetAsyncError(comm_, &ae));
        if (ae != ncclSuccess && ae != ncclInProgress) {
            ncclCommAbort(comm_);
            comm_ = nullptr;
            fail(PAIRAMG_INTERNAL, "rank " + std::to_string(rank_) + ": NCCL asynchronous error " +
                                       ncclGetErrorString(ae) + " (a peer rank failed?)");
        }
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(timeout_s)) {
            ncclCommAbort(comm_);
            comm_ = nullptr;
            fail(PAIRAMG_DEADLOCK, "rank " + std::to_string(rank_) + ": collective did not complete in " +
                                       std::to_string(timeout_s) + " s");
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

void Runtime::barrier() {
    if (nranks_ == 1) return;
    if (hub_) {
        hub_->wait_all(rank_);
        return;
    }
    allreduce_sum_i64(0);
}

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
        if (!id) fail(PAIRAMG_INVALID_ARGUMENT, "runtime: a unique id (NCCL or local) is required for nranks > 1");
        if (is_local_id(id)) {
            hub_ = join_hub(id, nranks);
            const std::vector<int64_t> devs = allgather_i64(device);
            for (int r = 0; r < nranks; ++r) {
                const int d = static_cast<int>(devs[static_cast<size_t>(r)]);
                if (r != rank && d == device) shared_device_ = true;
                if (d != device) {  // peer copies and stores between the ranks' GPUs
                    int can = 0;
                    PB_CUDA(cudaDeviceCanAccessPeer(&can, device, d));
                    if (can) {
                        const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
                        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) PB_CUDA(e);
                        cudaGetLastError();
                    }
                }
            }
            // every rank on this GPU drives two streams; CUDA maps streams onto
            // CUDA_DEVICE_MAX_CONNECTIONS hardware queues (default 8), and two
            // streams sharing a queue serialise -- a rank's spinning halo wait
            // queued ahead of a peer's push would then never finish
            int on_dev = 0;
            for (int64_t d : devs) on_dev += d == device ? 1 : 0;
            const char* mc = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
            const int conns = mc && *mc ? std::atoi(mc) : 8;
            if (shared_device_ && 2 * on_dev > conns) {
                hub_->abort("too few hardware queues for the ranks sharing a GPU");
                fail(PAIRAMG_INVALID_ARGUMENT,
                     "runtime: " + std::to_string(on_dev) + " ranks on one GPU need CUDA_DEVICE_MAX_CONNECTIONS >= " +
                         std::to_string(2 * on_dev) + " (set before the process initialises CUDA; max 32): two "
                         "streams per rank, and streams sharing a hardware queue serialise a peer's halo push "
                         "behind a rank's wait");
            }
            if (shared_device_ && lazy_module_loading()) {
                hub_->abort("lazy module loading with ranks sharing a GPU");
                fail(PAIRAMG_INVALID_ARGUMENT,
                     "runtime: ranks sharing one GPU need CUDA_MODULE_LOADING=EAGER (set before the process "
                     "initialises CUDA): with lazy loading, a rank's first launch of a kernel can wait for a "
                     "context synchronisation that a peer rank's halo wait blocks");
            }
        } else {
            ncclUniqueId uid;
            static_assert(sizeof(uid.internal) == 128, "NCCL unique id size");
            std::memcpy(uid.internal, id, 128);
            PB_NCCL(ncclCommInitRank(&comm_, nranks, uid, rank));
            warmup();
        }
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
    wait(stream_);
}

Runtime::~Runtime() {
    cudaSetDevice(device_);
    if (hub_) hub_->abort("rank " + std::to_string(rank_) + " destroyed its runtime");
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
    if (hub_) {
        const auto& p = hub_gather(&x);
        for (int r = 0; r < nranks_; ++r) out[static_cast<size_t>(r)] = *static_cast<const int64_t*>(p[static_cast<size_t>(r)]);
        hub_release();
        return out;
    }
    DBuf<int64_t> d(static_cast<size_t>(nranks_) + 1, stream_);
    PB_CUDA(cudaMemcpyAsync(d.get() + nranks_, &x, 8, cudaMemcpyHostToDevice, stream_));
    PB_NCCL(ncclAllGather(d.get() + nranks_, d.get(), 1, ncclInt64, comm_, stream_));
    PB_CUDA(cudaMemcpyAsync(out.data(), d.get(), 8 * nranks_, cudaMemcpyDeviceToHost, stream_));
    wait(stream_);
    return out;
}

std::vector<uint8_t> Runtime::allgather_bytes(const void* data, size_t n) {
    std::vector<uint8_t> out(static_cast<size_t>(nranks_) * n);
    if (nranks_ == 1) {
        std::memcpy(out.data(), data, n);
        return out;
    }
    stats_.allgathers += 1;
    if (hub_) {
        const auto& p = hub_gather(data);
        for (int r = 0; r < nranks_; ++r) std::memcpy(out.data() + r * n, p[static_cast<size_t>(r)], n);
        hub_release();
        return out;
    }
    DBuf<uint8_t> d(static_cast<size_t>(nranks_ + 1) * n, stream_);
    PB_CUDA(cudaMemcpyAsync(d.get() + nranks_ * n, data, n, cudaMemcpyHostToDevice, stream_));
    PB_NCCL(ncclAllGather(d.get() + nranks_ * n, d.get(), n, ncclUint8, comm_, stream_));
    PB_CUDA(cudaMemcpyAsync(out.data(), d.get(), static_cast<size_t>(nranks_) * n, cudaMemcpyDeviceToHost, stream_));
    wait(stream_);
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
    if (hub_) {
        const auto& ptr = hub_gather(&chunks);
        for (int q = 0; q < p; ++q) {
            if (q == rank_) continue;
            const auto& theirs = *static_cast<const std::vector<std::vector<int64_t>>*>(ptr[static_cast<size_t>(q)]);
            out[static_cast<size_t>(q)] = theirs[static_cast<size_t>(rank_)];
            if (!chunks[static_cast<size_t>(q)].empty()) {
                stats_.collective_messages += 1;
                stats_.collective_bytes += 8 * static_cast<int64_t>(chunks[static_cast<size_t>(q)].size());
            }
        }
        hub_release();
        return out;
    }
    // counts matrix by allgather (row r = what rank r sends to each rank)
    std::vector<int64_t> mine(p);
    for (int d = 0; d < p; ++d) mine[d] = static_cast<int64_t>(chunks[d].size());
    DBuf<int64_t> dc(static_cast<size_t>(p) * p + p, stream_);
    PB_CUDA(cudaMemcpyAsync(dc.get() + p * p, mine.data(), 8 * p, cudaMemcpyHostToDevice, stream_));
    PB_NCCL(ncclAllGather(dc.get() + p * p, dc.get(), p, ncclInt64, comm_, stream_));
    std::vector<int64_t> counts(static_cast<size_t>(p) * p);
    PB_CUDA(cudaMemcpyAsync(counts.data(), dc.get(), 8 * p * p, cudaMemcpyDeviceToHost, stream_));
    wait(stream_);
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
    wait(stream_);
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
    if (hub_) fail(PAIRAMG_INTERNAL, "allgather_f64: LOCAL runtimes use the P2P gathers on the solve path");
    PB_NCCL(ncclAllGather(send, recv, count, ncclDouble, comm_, s));
}

void Runtime::allgather_dev(const void* send, void* recv, size_t bytes) {
    if (nranks_ == 1) {
        if (bytes) PB_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, stream_));
        wait(stream_);
        return;
    }
    stats_.allgathers += 1;
    if (hub_) {
        wait(stream_);
        const auto& p = hub_gather(send);
        for (int r = 0; r < nranks_; ++r)
            if (bytes)
                PB_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + r * bytes, p[static_cast<size_t>(r)], bytes,
                                        cudaMemcpyDefault, stream_));
        wait(stream_);
        hub_release();
        return;
    }
    PB_NCCL(ncclAllGather(send, recv, bytes, ncclChar, comm_, stream_));
    wait(stream_);
}

namespace {
struct ExchangeView {
    const std::vector<int>* to;
    const std::vector<const void*>* bufs;
    const std::vector<size_t>* bytes;
};
}  // namespace

void Runtime::exchange_dev(const std::vector<int>& send_to, const std::vector<const void*>& sends,
                           const std::vector<size_t>& send_bytes, const std::vector<int>& recv_from,
                           const std::vector<void*>& recvs, const std::vector<size_t>& recv_bytes, cudaStream_t s) {
    for (size_t i = 0; i < send_to.size(); ++i) {
        stats_.p2p_messages += 1;
        stats_.p2p_bytes += static_cast<int64_t>(send_bytes[i]);
    }
    if (hub_) {
        PB_CUDA(cudaStreamSynchronize(s));
        const ExchangeView mine{&send_to, &sends, &send_bytes};
        const auto& p = hub_gather(&mine);
        for (size_t i = 0; i < recv_from.size(); ++i) {
            const ExchangeView& q = *static_cast<const ExchangeView*>(p[static_cast<size_t>(recv_from[i])]);
            size_t k = 0;
            while (k < q.to->size() && (*q.to)[k] != rank_) ++k;
            if (k == q.to->size() || (*q.bytes)[k] != recv_bytes[i])
                fail(PAIRAMG_INTERNAL, "exchange: unmatched send/recv between ranks " + std::to_string(recv_from[i]) +
                                           " and " + std::to_string(rank_));
            if (recv_bytes[i])
                PB_CUDA(cudaMemcpyAsync(recvs[i], (*q.bufs)[k], recv_bytes[i], cudaMemcpyDefault, s));
        }
        PB_CUDA(cudaStreamSynchronize(s));
        hub_release();
        return;
    }
    PB_NCCL(ncclGroupStart());
    for (size_t i = 0; i < send_to.size(); ++i)
        if (send_bytes[i]) PB_NCCL(ncclSend(sends[i], send_bytes[i], ncclChar, send_to[i], comm_, s));
    for (size_t i = 0; i < recv_from.size(); ++i)
        if (recv_bytes[i]) PB_NCCL(ncclRecv(recvs[i], recv_bytes[i], ncclChar, recv_from[i], comm_, s));
    PB_NCCL(ncclGroupEnd());
}

}  // namespace pb
