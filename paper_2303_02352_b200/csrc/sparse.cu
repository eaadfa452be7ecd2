// sparse.cu -- distributed sparse primitives on one rank's device data:
// localization + halo plans (dist.cpp:45-120), halo exchange (the sends /
// receives of spmv_dist, dist.cpp:142-162), SELL-32 construction, the
// SELL apply kernels (spmv_dist row loop dist.cpp:164-187, the l1-Jacobi
// update cycle.cpp:56-60, the V-cycle residual cycle.cpp:101-103) and the
// l1 diagonal (cycle.cpp:15-35).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>

#include "matrix.cuh"

namespace pb {

namespace {

struct OffRange {
    int64_t b, e;
    __host__ __device__ bool operator()(int64_t g) const { return g < b || g >= e; }
};

__global__ void k_map_cols(const int64_t* __restrict__ gcol, int32_t* __restrict__ lcol, int64_t nnz,
                           int64_t b, int64_t e, const int64_t* __restrict__ recv, int64_t nrecv,
                           int64_t n, int* __restrict__ bad) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nnz) return;
    const int64_t g = gcol[t];
    if (g >= b && g < e) {
        lcol[t] = static_cast<int32_t>(g - b);
        return;
    }
    int64_t lo = 0, hi = nrecv;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (recv[mid] < g)
            lo = mid + 1;
        else
            hi = mid;
    }
    if (lo >= nrecv || recv[lo] != g) {
        atomicExch(bad, 1);
        lcol[t] = 0;
        return;
    }
    lcol[t] = static_cast<int32_t>(n + lo);
}

__global__ void k_boundary_flags(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 int64_t n, uint8_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t f = 0;
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t)
        if (col[t] >= n) {
            f = 1;
            break;
        }
    flag[i] = f;
}

__global__ void k_invert(const uint8_t* __restrict__ a, uint8_t* __restrict__ b, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i] ? 0 : 1;
}

__global__ void k_global_cols(const int32_t* __restrict__ col, int64_t nnz, int64_t n, int64_t b,
                              const int64_t* __restrict__ recv, int64_t* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nnz) return;
    const int32_t c = col[t];
    out[t] = c < n ? b + c : recv[c - n];
}

// exchange_requests on the device: the halo ids are sorted, so every owner's
// ids form one contiguous segment; its first index is a lower_bound of the
// owner's first row (one thread per owner).
__global__ void k_owner_segments(const int64_t* __restrict__ ids, int64_t m, const int64_t* __restrict__ starts,
                                 int p, int64_t* __restrict__ seg) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q > p) return;
    const int64_t key = starts[q];
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ids[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    seg[q] = lo;
}

// requested global ids -> owned local ids; flags ids outside [b, e)
__global__ void k_to_local(const int64_t* __restrict__ g, int64_t m, int64_t b, int64_t e, int32_t* __restrict__ out,
                           int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t v = g[i];
    if (v < b || v >= e) atomicExch(bad, 1);
    out[i] = static_cast<int32_t>(v - b);
}

__global__ void k_pack(const int32_t* __restrict__ idx, int64_t m, const double* __restrict__ x,
                       double* __restrict__ buf) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < m) buf[t] = x[idx[t]];
}

__global__ void k_pack_pair(const int32_t* __restrict__ idx, int64_t m, const int64_t* __restrict__ a,
                            const double* __restrict__ b, int64_t* __restrict__ abuf,
                            double* __restrict__ bbuf) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < m) {
        abuf[t] = a[idx[t]];
        bbuf[t] = b[idx[t]];
    }
}

// l1_diagonal_dist (cycle.cpp:15-35): d_i = a_ii + sum_{j != i} |a_ij| in CSR order.
__global__ void k_l1(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                     const double* __restrict__ val, int64_t n, double* __restrict__ d,
                     unsigned long long* __restrict__ zero_row) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
        const double a = val[t];
        acc = dadd(acc, col[t] == i ? a : fabs(a));
    }
    if (acc == 0.0) atomicMin(zero_row, static_cast<unsigned long long>(i));
    d[i] = acc;
}

template <typename F>
void cub_call(F&& f, cudaStream_t s) {
    size_t bytes = 0;
    PB_CUDA(f(nullptr, bytes));
    DBuf<uint8_t> tmp(bytes ? bytes : 1, s);
    PB_CUDA(f(tmp.get(), bytes));
}

int64_t read_i64(const int64_t* d, cudaStream_t s) {
    int64_t h = 0;
    PB_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    return h;
}

// Row ids where flag[i] != 0, ascending.
int64_t select_rows(const uint8_t* flag, int64_t n, DBuf<int32_t>& out, cudaStream_t s) {
    DBuf<int32_t> tmp(static_cast<size_t>(n), s);
    DBuf<int64_t> cnt(1, s);
    thrust::counting_iterator<int32_t> it(0);
    cub_call([&](void* t, size_t& b) {
        return cub::DeviceSelect::Flagged(t, b, it, flag, tmp.get(), cnt.get(), n, s);
    }, s);
    const int64_t m = read_i64(cnt.get(), s);
    out.alloc(static_cast<size_t>(m), s);
    if (m) PB_CUDA(cudaMemcpyAsync(out.get(), tmp.get(), 4 * m, cudaMemcpyDeviceToDevice, s));
    return m;
}

}  // namespace

void localize(Runtime& rt, DevMatrix& M, DBuf<int64_t>&& rp, DBuf<int64_t>&& gcol,
              DBuf<double>&& val, int64_t nnz) {
    NvtxRange nv("setup/localize (halo plan)");
    cudaStream_t s = rt.stream();
    const int p = rt.nranks();
    const int r = rt.rank();
    M.row_begin = M.starts[r];
    M.n = M.starts[r + 1] - M.starts[r];
    M.n_global = M.starts[p];
    M.nnz = nnz;
    if (nnz >= (int64_t(1) << 31) - 1)
        fail(PAIRAMG_INVALID_ARGUMENT, "local nnz exceeds int32 column-slot range; use more ranks");
    const int64_t b = M.row_begin, e = M.starts[r + 1];

    // build_rows_to_receive (dist.cpp:45-55): sorted unique off-range ids.
    HaloPlan& H = M.halo;
    {
        DBuf<int64_t> off(static_cast<size_t>(std::max<int64_t>(nnz, 1)), s);
        DBuf<int64_t> cnt(1, s);
        OffRange pred{b, e};
        cub_call([&](void* t, size_t& bytes) {
            return cub::DeviceSelect::If(t, bytes, gcol.get(), off.get(), cnt.get(), nnz, pred, s);
        }, s);
        const int64_t m = read_i64(cnt.get(), s);
        if (m > 0) {
            DBuf<int64_t> sorted(static_cast<size_t>(m), s);
            cub_call([&](void* t, size_t& bytes) {
                return cub::DeviceRadixSort::SortKeys(t, bytes, off.get(), sorted.get(), m, 0, 64, s);
            }, s);
            cub_call([&](void* t, size_t& bytes) {
                return cub::DeviceSelect::Unique(t, bytes, sorted.get(), off.get(), cnt.get(), m, s);
            }, s);
            H.n_halo = read_i64(cnt.get(), s);
            H.recv_gid.alloc(static_cast<size_t>(H.n_halo), s);
            PB_CUDA(cudaMemcpyAsync(H.recv_gid.get(), off.get(), 8 * H.n_halo, cudaMemcpyDeviceToDevice, s));
        } else {
            H.n_halo = 0;
        }
    }
    if (H.n_halo > 0 && p == 1)
        fail(PAIRAMG_CONTRACT_VIOLATION, "localize: column index outside [0, n) on a single rank");
    if (M.n + H.n_halo >= (int64_t(1) << 31) - 1)
        fail(PAIRAMG_INVALID_ARGUMENT, "local rows + halo exceed int32 range");

    // local column ids
    M.col.alloc(static_cast<size_t>(nnz), s);
    {
        DBuf<int> bad(1, s);
        bad.zero(s);
        if (nnz)
            k_map_cols<<<blocks_for(nnz, 256), 256, 0, s>>>(gcol.get(), M.col.get(), nnz, b, e,
                                                            H.recv_gid.get(), H.n_halo, M.n, bad.get());
        PB_CHECK_LAUNCH();
        int hb = 0;
        PB_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, s));
        PB_CUDA(cudaStreamSynchronize(s));
        if (hb) fail(PAIRAMG_INTERNAL, "localize: halo id lookup failed");
    }
    M.rp = std::move(rp);
    M.val = std::move(val);
    gcol.reset();

    // exchange_requests (dist.cpp:67-91): tell owners what we need -- on the
    // device: owner segments of the sorted ids by binary search, p counts to
    // the host, the id lists peer to peer (no host copy of the ids).
    H.recv_peers.clear();
    H.recv_off.assign(1, 0);
    H.send_peers.clear();
    H.send_off.assign(1, 0);
    if (p > 1) {
        std::vector<int64_t> seg(static_cast<size_t>(p) + 1, 0);
        if (H.n_halo) {
            DBuf<int64_t> dstarts(static_cast<size_t>(p) + 1, s), dseg(static_cast<size_t>(p) + 1, s);
            PB_CUDA(cudaMemcpyAsync(dstarts.get(), M.starts.data(), 8 * (p + 1), cudaMemcpyHostToDevice, s));
            k_owner_segments<<<blocks_for(p + 1, 128), 128, 0, s>>>(H.recv_gid.get(), H.n_halo, dstarts.get(), p,
                                                                   dseg.get());
            PB_CHECK_LAUNCH();
            PB_CUDA(cudaMemcpyAsync(seg.data(), dseg.get(), 8 * (p + 1), cudaMemcpyDeviceToHost, s));
            PB_CUDA(cudaStreamSynchronize(s));
            seg[static_cast<size_t>(p)] = H.n_halo;  // ids >= starts[p] cannot exist (validated columns)
        }
        std::vector<int64_t> want(static_cast<size_t>(p), 0);  // ids this rank requests from each rank
        for (int q = 0; q < p; ++q) want[static_cast<size_t>(q)] = seg[static_cast<size_t>(q) + 1] - seg[static_cast<size_t>(q)];
        if (want[static_cast<size_t>(r)] != 0 || seg[0] != 0)
            fail(PAIRAMG_INTERNAL, "halo plan: owned id in receive set");
        for (int q = 0; q < p; ++q)
            if (want[static_cast<size_t>(q)]) {
                H.recv_peers.push_back(q);
                H.recv_off.push_back(H.recv_off.back() + want[static_cast<size_t>(q)]);
            }
        // counts matrix (row = requester): what every rank asks of us
        const std::vector<uint8_t> all = rt.allgather_bytes(want.data(), 8 * static_cast<size_t>(p));
        std::vector<int64_t> asked(static_cast<size_t>(p), 0);
        for (int q = 0; q < p; ++q) std::memcpy(&asked[static_cast<size_t>(q)], all.data() + (static_cast<size_t>(q) * p + r) * 8, 8);
        for (int q = 0; q < p; ++q)
            if (q != r && asked[static_cast<size_t>(q)]) {
                H.send_peers.push_back(q);
                H.send_off.push_back(H.send_off.back() + asked[static_cast<size_t>(q)]);
            }
        const int64_t nsend = H.send_off.back();
        rt.stats().alltoallvs += 1;
        DBuf<int64_t> gsend(static_cast<size_t>(std::max<int64_t>(nsend, 1)), s);
        std::vector<int> to(H.recv_peers.begin(), H.recv_peers.end()), from(H.send_peers.begin(), H.send_peers.end());
        std::vector<const void*> sb;
        std::vector<void*> rb;
        std::vector<size_t> sn, rn;
        for (size_t i = 0; i < H.recv_peers.size(); ++i) {
            sb.push_back(H.recv_gid.get() + H.recv_off[i]);
            sn.push_back(8 * static_cast<size_t>(H.recv_off[i + 1] - H.recv_off[i]));
        }
        for (size_t i = 0; i < H.send_peers.size(); ++i) {
            rb.push_back(gsend.get() + H.send_off[i]);
            rn.push_back(8 * static_cast<size_t>(H.send_off[i + 1] - H.send_off[i]));
        }
        rt.exchange_dev(to, sb, sn, from, rb, rn, s);
        H.send_idx.alloc(static_cast<size_t>(nsend), s);
        H.send_buf.alloc(static_cast<size_t>(nsend), s);
        if (nsend) {
            DBuf<int> bad(1, s);
            bad.zero(s);
            k_to_local<<<blocks_for(nsend, 256), 256, 0, s>>>(gsend.get(), nsend, b, e, H.send_idx.get(), bad.get());
            PB_CHECK_LAUNCH();
            int hb = 0;
            PB_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, s));
            PB_CUDA(cudaStreamSynchronize(s));
            if (hb) fail(PAIRAMG_INTERNAL, "halo plan: asked for a row we do not own");
        }
    }

    // boundary / interior rows (build_spmv_plan, dist.cpp:109-118)
    M.n_boundary = 0;
    M.boundary_rows.reset();
    M.interior_rows.reset();
    if (H.n_halo > 0) {
        DBuf<uint8_t> flag(static_cast<size_t>(M.n), s), inv(static_cast<size_t>(M.n), s);
        k_boundary_flags<<<blocks_for(M.n, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), M.n, flag.get());
        PB_CHECK_LAUNCH();
        k_invert<<<blocks_for(M.n, 256), 256, 0, s>>>(flag.get(), inv.get(), M.n);
        PB_CHECK_LAUNCH();
        M.n_boundary = select_rows(flag.get(), M.n, M.boundary_rows, s);
        select_rows(inv.get(), M.n, M.interior_rows, s);
    }
    PB_CUDA(cudaStreamSynchronize(s));
}

void global_columns(const DevMatrix& M, int64_t* d_out, cudaStream_t s) {
    if (!M.nnz) return;
    k_global_cols<<<blocks_for(M.nnz, 256), 256, 0, s>>>(M.col.get(), M.nnz, M.n, M.row_begin,
                                                        M.halo.recv_gid.get(), d_out);
    PB_CHECK_LAUNCH();
}

void l1_diagonal(const DevMatrix& M, double* d_out, cudaStream_t s) {
    if (!M.n) return;
    DBuf<unsigned long long> zr(1, s);
    PB_CUDA(cudaMemsetAsync(zr.get(), 0xff, 8, s));
    k_l1<<<blocks_for(M.n, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), M.val.get(), M.n, d_out, zr.get());
    PB_CHECK_LAUNCH();
    unsigned long long h = 0;
    PB_CUDA(cudaMemcpyAsync(&h, zr.get(), 8, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (h != ~0ULL)
        fail(PAIRAMG_SINGULAR_SMOOTHER, "l1_diagonal_dist: zero diagonal weight at global row " +
                                            std::to_string(M.row_begin + static_cast<int64_t>(h)));
}

void halo_exchange(Runtime& rt, HaloPlan& H, const double* x_owned, double* x_halo, cudaStream_t s) {
    if (!H.has_traffic()) return;
    rt.stats().halo_exchanges += 1;
    rt.stats().halo_bytes += 8 * H.n_halo;
    const int64_t nsend = H.send_off.back();
    if (nsend) {
        k_pack<<<blocks_for(nsend, 256), 256, 0, s>>>(H.send_idx.get(), nsend, x_owned, H.send_buf.get());
        PB_CHECK_LAUNCH();
    }
    if (rt.local()) {
        cudaStreamCaptureStatus cs;
        PB_CUDA(cudaStreamIsCapturing(s, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            fail(PAIRAMG_INTERNAL, "halo_exchange: LOCAL runtimes exchange solve-path halos by P2P stores");
    }
    std::vector<int> to(H.send_peers.begin(), H.send_peers.end()), from(H.recv_peers.begin(), H.recv_peers.end());
    std::vector<const void*> sb;
    std::vector<void*> rb;
    std::vector<size_t> sn, rn;
    for (size_t i = 0; i < H.send_peers.size(); ++i) {
        sb.push_back(H.send_buf.get() + H.send_off[i]);
        sn.push_back(8 * static_cast<size_t>(H.send_off[i + 1] - H.send_off[i]));
    }
    for (size_t i = 0; i < H.recv_peers.size(); ++i) {
        rb.push_back(x_halo + H.recv_off[i]);
        rn.push_back(8 * static_cast<size_t>(H.recv_off[i + 1] - H.recv_off[i]));
    }
    rt.exchange_dev(to, sb, sn, from, rb, rn, s);
}

void halo_exchange_pair(Runtime& rt, HaloPlan& H, const int64_t* a_owned, int64_t* a_halo,
                        const double* b_owned, double* b_halo, cudaStream_t s) {
    if (!H.has_traffic()) return;
    const int64_t nsend = H.send_off.back();
    if (H.send_buf_i64.size() < static_cast<size_t>(nsend)) H.send_buf_i64.alloc(static_cast<size_t>(nsend), s);
    if (nsend) {
        k_pack_pair<<<blocks_for(nsend, 256), 256, 0, s>>>(H.send_idx.get(), nsend, a_owned, b_owned,
                                                           H.send_buf_i64.get(), H.send_buf.get());
        PB_CHECK_LAUNCH();
    }
    // ids then values to every peer (two messages per peer, one exchange)
    std::vector<int> to, from;
    std::vector<const void*> sb;
    std::vector<void*> rb;
    std::vector<size_t> sn, rn;
    for (size_t i = 0; i < H.send_peers.size(); ++i) {
        const size_t c = static_cast<size_t>(H.send_off[i + 1] - H.send_off[i]);
        to.push_back(H.send_peers[i]);
        sb.push_back(H.send_buf_i64.get() + H.send_off[i]);
        sn.push_back(8 * c);
    }
    for (size_t i = 0; i < H.recv_peers.size(); ++i) {
        const size_t c = static_cast<size_t>(H.recv_off[i + 1] - H.recv_off[i]);
        from.push_back(H.recv_peers[i]);
        rb.push_back(a_halo + H.recv_off[i]);
        rn.push_back(8 * c);
    }
    rt.exchange_dev(to, sb, sn, from, rb, rn, s);
    to.clear(), from.clear(), sb.clear(), rb.clear(), sn.clear(), rn.clear();
    for (size_t i = 0; i < H.send_peers.size(); ++i) {
        const size_t c = static_cast<size_t>(H.send_off[i + 1] - H.send_off[i]);
        to.push_back(H.send_peers[i]);
        sb.push_back(H.send_buf.get() + H.send_off[i]);
        sn.push_back(8 * c);
    }
    for (size_t i = 0; i < H.recv_peers.size(); ++i) {
        const size_t c = static_cast<size_t>(H.recv_off[i + 1] - H.recv_off[i]);
        from.push_back(H.recv_peers[i]);
        rb.push_back(b_halo + H.recv_off[i]);
        rn.push_back(8 * c);
    }
    rt.exchange_dev(to, sb, sn, from, rb, rn, s);
}

}  // namespace pb
