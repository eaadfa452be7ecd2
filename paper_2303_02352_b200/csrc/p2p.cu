// p2p.cu -- NVLink halo exchange by direct stores (see p2p.cuh).
#include <cstring>

#include "p2p.cuh"

namespace pb {

namespace {

constexpr int kMaxPeers = 8;
constexpr int kPullBlocks = 32;

struct PushArgs {
    int npeers;
    int64_t off[kMaxPeers + 1];  // send_off
    double* dst[kMaxPeers];      // peer staging + my offset
    int64_t stride[kMaxPeers];   // peer parity stride
    unsigned long long* flag[kMaxPeers];
};

struct PullArgs {
    int nrecv;
    int from[kMaxPeers];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel(unsigned long long* p) {
    unsigned long long prev;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(prev) : "l"(p) : "memory");
    return prev;
}

// Every rank pushes its boundary values into each neighbour's staging slot of
// parity (exchange count & 1); the last CTA raises the neighbours' flags.
__global__ void __launch_bounds__(256) k_p2p_push(const double* x, const int32_t* send_idx, int64_t nsend,
                                                   const __grid_constant__ PushArgs pa, unsigned long long* ctr) {
    const unsigned long long e = ctr[4];  // pushes done (== exchanges received on every rank)
    const int64_t par = static_cast<int64_t>(e & 1ull);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nsend;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int p = 0;
        while (p + 1 < pa.npeers && i >= pa.off[p + 1]) ++p;
        pa.dst[p][par * pa.stride[p] + (i - pa.off[p])] = x[send_idx[i]];
    }
    __threadfence_system();
    __syncthreads();
    // every block's stores are system-visible (its fence) before its count;
    // the last block's acq_rel count follows all of them, so its flag
    // stores need no second system fence (as halo_push_block)
    if (threadIdx.x == 0 && atom_add_acq_rel(&ctr[5]) == gridDim.x - 1) {
        ctr[5] = 0;
        ctr[4] = e + 1;
        for (int p = 0; p < pa.npeers; ++p) st_relaxed_sys(pa.flag[p], e + 1);
    }
}

// Wait for every sender's flag of this exchange, then copy the staging slot
// into the halo slots; the last CTA advances the exchange count.
__global__ void __launch_bounds__(256) k_p2p_pull(const double* staging, const unsigned long long* flags, int64_t n_halo,
                                                   const __grid_constant__ PullArgs pl, double* x_halo,
                                                   unsigned long long* ctr) {
    const unsigned long long e = ctr[0];
    if (threadIdx.x == 0) {
        for (int k = 0; k < pl.nrecv; ++k) {
            long long spins = 0;
            while (ld_acquire_sys(flags + pl.from[k]) < e + 1) {
                __nanosleep(64);
                if (++spins == (1ll << 28)) {  // a lost flag must fail loudly, not hang the solve
                    printf("pairamg: p2p halo flag wait timed out\n");
                    __trap();
                }
            }
        }
    }
    __syncthreads();
    const double* src = staging + static_cast<int64_t>(e & 1ull) * n_halo;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_halo;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x_halo[j] = __ldcv(src + j);  // written by a peer GPU: bypass L1
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&ctr[2], 1ull) == gridDim.x - 1) {
        ctr[2] = 0;
        ctr[0] = e + 1;
    }
}

// A device buffer as another rank can map it: a CUDA IPC handle across
// processes, the raw pointer between the threads of one process (LOCAL
// runtimes; same or peer-enabled device).
struct SharedBuf {
    cudaIpcMemHandle_t h;
    void* raw;
};

bool export_buf(const Runtime& rt, void* p, SharedBuf& out) {
    out.raw = p;
    if (rt.local()) return true;
    return cudaIpcGetMemHandle(&out.h, p) == cudaSuccess;
}

bool import_buf(const Runtime& rt, const SharedBuf& in, void** out, std::vector<void*>& opened) {
    if (rt.local()) {
        *out = in.raw;
        return true;
    }
    if (cudaIpcOpenMemHandle(out, in.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    opened.push_back(*out);
    return true;
}

struct Blob {
    SharedBuf staging, flags;
    int64_t n_halo;
    int32_t nrecv;
    int32_t recv_rank[kMaxPeers];
    int64_t recv_off[kMaxPeers];
};

}  // namespace

// Teardown order (CUDA IPC): every importer closes its mappings of a peer's
// buffers before the exporter frees them.  Re-setups do it collectively --
// p2p_close_imports on every rank, a barrier, then the frees (Solver::setup).
void p2p_close_imports(P2PHalo& P) {
    for (void* p : P.opened) cudaIpcCloseMemHandle(p);
    P.opened.clear();
    P.peer_staging.clear();
    P.peer_stride.clear();
    P.peer_flag.clear();
    P.ok = false;
}

void p2p_seg_close_imports(P2PSegGather& G) {
    for (void* p : G.opened) cudaIpcCloseMemHandle(p);
    G.opened.clear();
    G.peer_buf.clear();
    G.peer_flags.clear();
    G.ok = false;
}

void p2p_destroy(P2PHalo& P) {
    for (void* p : P.opened) cudaIpcCloseMemHandle(p);
    P.opened.clear();
    if (P.staging) cudaFree(P.staging);
    if (P.flags) cudaFree(P.flags);
    P.staging = nullptr;
    P.flags = nullptr;
    P.ok = false;
}

void p2p_setup(Runtime& rt, const HaloPlan& H, P2PHalo& P, cudaStream_t s) {
    p2p_destroy(P);
    if (rt.nranks() == 1) return;
    Blob mine;
    std::memset(&mine, 0, sizeof mine);
    bool local_ok = H.recv_peers.size() <= static_cast<size_t>(kMaxPeers) &&
                    H.send_peers.size() <= static_cast<size_t>(kMaxPeers);
    P.n_halo = H.n_halo;
    if (local_ok) {
        local_ok = cudaMalloc(&P.staging, 16 * static_cast<size_t>(std::max<int64_t>(H.n_halo, 1))) == cudaSuccess &&
                   cudaMalloc(&P.flags, 8 * static_cast<size_t>(rt.nranks())) == cudaSuccess &&
                   cudaMemset(P.flags, 0, 8 * static_cast<size_t>(rt.nranks())) == cudaSuccess &&
                   export_buf(rt, P.staging, mine.staging) && export_buf(rt, P.flags, mine.flags);
        cudaGetLastError();
    }
    mine.n_halo = local_ok ? H.n_halo : -1;  // -1: this rank cannot take part
    mine.nrecv = static_cast<int32_t>(std::min<size_t>(H.recv_peers.size(), kMaxPeers));
    for (int i = 0; i < mine.nrecv; ++i) {
        mine.recv_rank[i] = H.recv_peers[static_cast<size_t>(i)];
        mine.recv_off[i] = H.recv_off[static_cast<size_t>(i)];
    }
    const std::vector<uint8_t> all = rt.allgather_bytes(&mine, sizeof(Blob));
    std::vector<Blob> blobs(static_cast<size_t>(rt.nranks()));
    std::memcpy(blobs.data(), all.data(), all.size());
    bool ok = true;
    for (const Blob& b : blobs) ok = ok && b.n_halo >= 0;
    if (ok) {
        for (size_t i = 0; i < H.send_peers.size(); ++i) {
            const Blob& q = blobs[static_cast<size_t>(H.send_peers[i])];
            int64_t off = -1;
            for (int k = 0; k < q.nrecv; ++k)
                if (q.recv_rank[k] == rt.rank()) off = q.recv_off[k];
            void* st = nullptr;
            void* fl = nullptr;
            if (off < 0 || !import_buf(rt, q.staging, &st, P.opened) || !import_buf(rt, q.flags, &fl, P.opened)) {
                ok = false;
                break;
            }
            P.peer_staging.push_back(static_cast<double*>(st) + off);
            P.peer_stride.push_back(q.n_halo);
            P.peer_flag.push_back(static_cast<unsigned long long*>(fl) + rt.rank());
        }
    }
    // every rank must agree, else all fall back to NCCL together
    const bool all_ok = rt.allreduce_sum_i64(ok ? 1 : 0) == rt.nranks();
    if (!all_ok) {
        p2p_destroy(P);
        P.peer_staging.clear();
        P.peer_stride.clear();
        P.peer_flag.clear();
        return;
    }
    P.ctr.alloc(8, s);
    P.ctr.zero(s);
    PB_CUDA(cudaStreamSynchronize(s));
    P.ok = true;
}

namespace {
int p2p_prio() {
    static int prio = [] {
        int lo = 0, hi = 0;
        PB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        return hi;
    }();
    return prio;
}

void launch_push(const HaloPlan& H, P2PHalo& P, const double* x_owned, cudaStream_t s) {
    const int64_t nsend = H.send_off.empty() ? 0 : H.send_off.back();
    PushArgs pa{};
    pa.npeers = static_cast<int>(H.send_peers.size());
    for (int i = 0; i <= pa.npeers; ++i) pa.off[i] = H.send_off[static_cast<size_t>(i)];
    for (int i = 0; i < pa.npeers; ++i) {
        pa.dst[i] = P.peer_staging[static_cast<size_t>(i)];
        pa.stride[i] = P.peer_stride[static_cast<size_t>(i)];
        pa.flag[i] = P.peer_flag[static_cast<size_t>(i)];
    }
    // highest scheduling priority on the launch itself (a stream's priority
    // is not carried into the nodes of a captured graph); a rank with nothing
    // to send still runs it so every rank's exchange counter advances alike
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = p2p_prio();
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.gridDim = dim3(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((nsend + 255) / 256, 2 * kSmCount))));
    PB_CUDA(cudaLaunchKernelEx(&cfg, k_p2p_push, x_owned, static_cast<const int32_t*>(H.send_idx.get()), nsend, pa,
                               P.ctr.get()));
}
}  // namespace

void p2p_push(const HaloPlan& H, P2PHalo& P, const double* x_owned, cudaStream_t s) { launch_push(H, P, x_owned, s); }

HaloSrc p2p_halo_src(const HaloPlan& H, P2PHalo& P) {
    HaloSrc hs;
    hs.flags = P.flags;
    hs.nfrom = static_cast<int>(std::min<size_t>(H.recv_peers.size(), 8));
    for (int i = 0; i < hs.nfrom; ++i) hs.from[i] = H.recv_peers[static_cast<size_t>(i)];
    hs.staging = P.staging;
    hs.nhalo = H.n_halo;
    hs.ctr = P.ctr.get();
    if (H.send_peers.size() <= 8) {
        hs.fused = true;
        hs.npeers = static_cast<int>(H.send_peers.size());
        for (int i = 0; i <= hs.npeers; ++i) hs.off[i] = H.send_off[static_cast<size_t>(i)];
        for (int i = 0; i < hs.npeers; ++i) {
            hs.dst[i] = P.peer_staging[static_cast<size_t>(i)];
            hs.stride[i] = P.peer_stride[static_cast<size_t>(i)];
            hs.pflag[i] = P.peer_flag[static_cast<size_t>(i)];
        }
        hs.send_idx = H.send_idx.get();
    }
    return hs;
}

void p2p_exchange(const HaloPlan& H, P2PHalo& P, const double* x_owned, double* x_halo, cudaStream_t s) {
    launch_push(H, P, x_owned, s);
    PullArgs pl{};
    pl.nrecv = static_cast<int>(H.recv_peers.size());
    for (int i = 0; i < pl.nrecv; ++i) pl.from[i] = H.recv_peers[static_cast<size_t>(i)];
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = p2p_prio();
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.gridDim = dim3(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((H.n_halo + 255) / 256, kPullBlocks))));
    PB_CUDA(cudaLaunchKernelEx(&cfg, k_p2p_pull, static_cast<const double*>(P.staging),
                               static_cast<const unsigned long long*>(P.flags), H.n_halo, pl, x_halo, P.ctr.get()));
}

// ---- small allgather ------------------------------------------------------

namespace {
__global__ void k_p2p_allgather(const double* send, double* recv, int K, int nranks, int rank, double* const* peer_mail,
                                unsigned long long* const* peer_flags, const double* my_mail,
                                const unsigned long long* my_flags, int kmax, unsigned long long* ctr) {
    pdl_wait_only();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long e = ctr[0];
    const int64_t par = static_cast<int64_t>(e & 1ull) * nranks * kmax;
    for (int r = 0; r < nranks; ++r)
        for (int k = 0; k < K; ++k) peer_mail[r][par + rank * kmax + k] = send[k];
    __threadfence_system();
    for (int r = 0; r < nranks; ++r) st_release_sys(peer_flags[r] + rank, e + 1);
    for (int r = 0; r < nranks; ++r) {
        long long spins = 0;
        while (ld_acquire_sys(my_flags + r) < e + 1) {
            __nanosleep(32);
            if (++spins == (1ll << 28)) {
                printf("pairamg: p2p allgather flag wait timed out\n");
                __trap();
            }
        }
    }
    for (int r = 0; r < nranks; ++r)
        for (int k = 0; k < K; ++k) recv[r * K + k] = __ldcv(my_mail + par + r * kmax + k);
    ctr[0] = e + 1;
}
}  // namespace

P2PGather::~P2PGather() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    if (mail) cudaFree(mail);
    if (flags) cudaFree(flags);
}

void p2p_gather_setup(Runtime& rt, P2PGather& G, int kmax, cudaStream_t s) {
    if (rt.nranks() == 1 || G.mail) return;  // set up once per solver (re-setups keep it)
    G.ok = false;
    G.nranks = rt.nranks();
    G.rank = rt.rank();
    G.kmax = kmax;
    struct GBlob {
        SharedBuf mail, flags;
        int32_t ok;
    } mine;
    std::memset(&mine, 0, sizeof mine);
    const size_t mbytes = 8 * 2 * static_cast<size_t>(G.nranks) * kmax;
    mine.ok = cudaMalloc(&G.mail, mbytes) == cudaSuccess && cudaMalloc(&G.flags, 8 * G.nranks) == cudaSuccess &&
              cudaMemset(G.flags, 0, 8 * G.nranks) == cudaSuccess &&
              export_buf(rt, G.mail, mine.mail) && export_buf(rt, G.flags, mine.flags);
    cudaGetLastError();
    const std::vector<uint8_t> all = rt.allgather_bytes(&mine, sizeof mine);
    std::vector<GBlob> blobs(static_cast<size_t>(G.nranks));
    std::memcpy(blobs.data(), all.data(), all.size());
    bool ok = true;
    for (const GBlob& b : blobs) ok = ok && b.ok;
    for (int r = 0; ok && r < G.nranks; ++r) {
        if (r == G.rank) {
            G.peer_mail.push_back(G.mail);
            G.peer_flags.push_back(G.flags);
            continue;
        }
        void* m = nullptr;
        void* f = nullptr;
        if (!import_buf(rt, blobs[static_cast<size_t>(r)].mail, &m, G.opened) ||
            !import_buf(rt, blobs[static_cast<size_t>(r)].flags, &f, G.opened)) {
            ok = false;
            break;
        }
        G.peer_mail.push_back(static_cast<double*>(m));
        G.peer_flags.push_back(static_cast<unsigned long long*>(f));
    }
    if (rt.allreduce_sum_i64(ok ? 1 : 0) != G.nranks) return;  // all or none
    G.ctr.alloc(1, s);
    G.ctr.zero(s);
    G.d_peer_mail.alloc(static_cast<size_t>(G.nranks), s);
    G.d_peer_flags.alloc(static_cast<size_t>(G.nranks), s);
    PB_CUDA(cudaMemcpyAsync(G.d_peer_mail.get(), G.peer_mail.data(), 8 * G.nranks, cudaMemcpyHostToDevice, s));
    PB_CUDA(cudaMemcpyAsync(G.d_peer_flags.get(), G.peer_flags.data(), 8 * G.nranks, cudaMemcpyHostToDevice, s));
    PB_CUDA(cudaStreamSynchronize(s));
    G.ok = true;
}

void p2p_allgather(P2PGather& G, const double* send, double* recv, int K, cudaStream_t s) {
    if (!G.ok || K > G.kmax) fail(PAIRAMG_INTERNAL, "p2p_allgather: not set up");
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = p2p_prio();
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = s;
    PB_CUDA(cudaLaunchKernelEx(&cfg, k_p2p_allgather, send, recv, K, G.nranks, G.rank,
                               static_cast<double* const*>(G.d_peer_mail.get()),
                               static_cast<unsigned long long* const*>(G.d_peer_flags.get()),
                               static_cast<const double*>(G.mail), static_cast<const unsigned long long*>(G.flags),
                               G.kmax, G.ctr.get()));
}

// ---- segment allgather (replicated coarse right-hand side) ----------------

namespace {
struct SegArgs {
    double* buf[kSegMaxRanks];                 // every rank's vector (own: local)
    unsigned long long* flag[kSegMaxRanks];    // every rank's flag array
    const unsigned long long* myflags;
    int nranks, rank;
};

__global__ void __launch_bounds__(256) k_seg_gather(const double* src, int64_t cnt, int64_t off,
                                                    const __grid_constant__ SegArgs a, unsigned long long* ctr) {
    pdl_wait_only();
    const unsigned long long e = ctr[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = src[i];
        for (int r = 0; r < a.nranks; ++r) a.buf[r][off + i] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atom_add_acq_rel(&ctr[1]) == gridDim.x - 1) {  // see k_p2p_push
        ctr[1] = 0;
        for (int r = 0; r < a.nranks; ++r)
            if (r != a.rank) st_relaxed_sys(a.flag[r] + a.rank, e + 1);
        for (int r = 0; r < a.nranks; ++r) {
            if (r == a.rank) continue;
            long long spins = 0;
            while (ld_acquire_sys(a.myflags + r) < e + 1) {
                __nanosleep(64);
                if (++spins == (1ll << 28)) {
                    printf("pairamg: p2p segment gather flag wait timed out\n");
                    __trap();
                }
            }
        }
        ctr[0] = e + 1;
        __threadfence_system();
    }
}
}  // namespace

void p2p_seg_destroy(P2PSegGather& G) {
    for (void* p : G.opened) cudaIpcCloseMemHandle(p);
    G.opened.clear();
    if (G.buf) cudaFree(G.buf);
    if (G.flags) cudaFree(G.flags);
    G.buf = nullptr;
    G.flags = nullptr;
    G.peer_buf.clear();
    G.peer_flags.clear();
    G.ok = false;
}

P2PSegGather::~P2PSegGather() { p2p_seg_destroy(*this); }

void p2p_seg_setup(Runtime& rt, P2PSegGather& G, int64_t total, cudaStream_t s) {
    p2p_seg_destroy(G);
    if (rt.nranks() == 1 || rt.nranks() > kSegMaxRanks) return;
    G.nranks = rt.nranks();
    G.rank = rt.rank();
    G.total = total;
    struct SBlob {
        SharedBuf buf, flags;
        int32_t ok;
    } mine;
    std::memset(&mine, 0, sizeof mine);
    mine.ok = cudaMalloc(&G.buf, 8 * static_cast<size_t>(std::max<int64_t>(total, 1))) == cudaSuccess &&
              cudaMalloc(&G.flags, 8 * G.nranks) == cudaSuccess && cudaMemset(G.flags, 0, 8 * G.nranks) == cudaSuccess &&
              export_buf(rt, G.buf, mine.buf) && export_buf(rt, G.flags, mine.flags);
    cudaGetLastError();
    const std::vector<uint8_t> all = rt.allgather_bytes(&mine, sizeof mine);
    std::vector<SBlob> blobs(static_cast<size_t>(G.nranks));
    std::memcpy(blobs.data(), all.data(), all.size());
    bool ok = true;
    for (const SBlob& b : blobs) ok = ok && b.ok;
    for (int r = 0; ok && r < G.nranks; ++r) {
        if (r == G.rank) {
            G.peer_buf.push_back(G.buf);
            G.peer_flags.push_back(G.flags);
            continue;
        }
        void* m = nullptr;
        void* f = nullptr;
        if (!import_buf(rt, blobs[static_cast<size_t>(r)].buf, &m, G.opened) ||
            !import_buf(rt, blobs[static_cast<size_t>(r)].flags, &f, G.opened)) {
            ok = false;
            break;
        }
        G.peer_buf.push_back(static_cast<double*>(m));
        G.peer_flags.push_back(static_cast<unsigned long long*>(f));
    }
    if (rt.allreduce_sum_i64(ok ? 1 : 0) != G.nranks) {  // all or none
        p2p_seg_destroy(G);
        return;
    }
    G.ctr.alloc(2, s);
    G.ctr.zero(s);
    PB_CUDA(cudaStreamSynchronize(s));
    G.ok = true;
}

void p2p_seg_gather(P2PSegGather& G, const double* src, int64_t cnt, int64_t off, cudaStream_t s) {
    SegArgs a{};
    a.nranks = G.nranks;
    a.rank = G.rank;
    for (int r = 0; r < G.nranks; ++r) {
        a.buf[r] = G.peer_buf[static_cast<size_t>(r)];
        a.flag[r] = G.peer_flags[static_cast<size_t>(r)];
    }
    a.myflags = G.flags;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((cnt + 2047) / 2048, 2 * kSmCount)));
    launch_k<4>(k_seg_gather, grid, 256, 0, s, src, cnt, off, a, G.ctr.get());
    PB_CHECK_LAUNCH();
}

}  // namespace pb
