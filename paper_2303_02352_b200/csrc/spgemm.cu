// spgemm.cu -- general sparse product C = A*B on the device with the
// reference's summation order (spgemm_local, csr.cpp:206-272).
//
// The reference accumulates, per output row, the products a_ik*b_kj in
// encounter order (A row ascending, then B row order): the first product of a
// column is assigned, later ones added (hash path and sort-merge path agree,
// csr.cpp:128-204); columns come out ascending.  Here: every product is
// written once at its encounter position (scan over A entries), a stable
// radix sort on (row, column) keeps encounter order inside each (row,
// column) run, and one thread folds each run left to right with separately
// rounded adds, starting from its first product -- bitwise the reference,
// signed zeros included.  (The pairwise Galerkin product of the hierarchy
// uses the specialised one-nnz-per-row path in setup.cu; this is the general
// operator.)
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "mmio.cuh"
#include "spgemm.cuh"

namespace pb {

namespace {

using ull = unsigned long long;

__global__ void k_rowid(const int64_t* __restrict__ rp, int64_t n, int32_t* __restrict__ rowid) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) rowid[e] = static_cast<int32_t>(i);
}

__global__ void k_contrib_count(const int64_t* __restrict__ a_col, int64_t nnz_a, const int64_t* __restrict__ b_rp,
                                int64_t* __restrict__ cnt) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < nnz_a) cnt[e] = b_rp[a_col[e] + 1] - b_rp[a_col[e]];
}

__global__ void k_contrib_fill(const int32_t* __restrict__ rowid, const int64_t* __restrict__ a_col,
                               const double* __restrict__ a_val, int64_t nnz_a, const int64_t* __restrict__ b_rp,
                               const int64_t* __restrict__ b_col, const double* __restrict__ b_val,
                               const int64_t* __restrict__ off, ull* __restrict__ key, double* __restrict__ val) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= nnz_a) return;
    const int64_t k = a_col[e], b0 = b_rp[k], b1 = b_rp[k + 1];
    const ull rk = static_cast<ull>(rowid[e]) << 32;
    const double av = a_val[e];
    int64_t o = off[e];
    for (int64_t t = b0; t < b1; ++t, ++o) {
        key[o] = rk | static_cast<ull>(b_col[t]);
        val[o] = dmul(av, b_val[t]);
    }
}

__global__ void k_run_heads(const ull* __restrict__ key, int64_t n, uint8_t* __restrict__ head) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// One thread per (row, column) run: left fold from the first product.
__global__ void k_fold_runs(const ull* __restrict__ key, const double* __restrict__ val, const int64_t* __restrict__ start,
                            int64_t nruns, int64_t n, int64_t* __restrict__ col, double* __restrict__ out,
                            int64_t* __restrict__ rowcnt) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const int64_t b = start[r], e = r + 1 < nruns ? start[r + 1] : n;
    double s = val[b];
    for (int64_t j = b + 1; j < e; ++j) s = dadd(s, val[j]);
    out[r] = s;
    col[r] = static_cast<int64_t>(key[b] & 0xFFFFFFFFull);
    atomicAdd(reinterpret_cast<unsigned long long*>(rowcnt + (key[b] >> 32)), 1ull);
}

template <typename F>
void cub_run(F&& f, cudaStream_t s) {
    size_t bytes = 0;
    PB_CUDA(f(nullptr, bytes));
    DBuf<uint8_t> tmp(bytes ? bytes : 1, s);
    PB_CUDA(f(tmp.get(), bytes));
}

}  // namespace

HostCsr spgemm(int64_t an, int64_t am, const int64_t* a_rp, const int64_t* a_col, const double* a_val, int64_t bm,
               const int64_t* b_rp, const int64_t* b_col, const double* b_val, cudaStream_t s) {
    if (an < 0 || am < 0 || bm < 0) fail(PAIRAMG_INVALID_ARGUMENT, "spgemm: negative dimension");
    if (an >= (int64_t(1) << 31) || bm >= (int64_t(1) << 32))
        fail(PAIRAMG_INVALID_ARGUMENT, "spgemm: dimensions exceed the 32-bit key fields");
    const int64_t nnz_a = a_rp[an], nnz_b = b_rp[am];
    for (int64_t e = 0; e < nnz_a; ++e)
        if (a_col[e] < 0 || a_col[e] >= am) fail(PAIRAMG_CONTRACT_VIOLATION, "spgemm: column of A out of range");
    for (int64_t e = 0; e < nnz_b; ++e)
        if (b_col[e] < 0 || b_col[e] >= bm) fail(PAIRAMG_CONTRACT_VIOLATION, "spgemm: column of B out of range");
    HostCsr C;
    C.nrows = an;
    C.ncols = bm;
    C.row_ptr.assign(static_cast<size_t>(an) + 1, 0);
    DBuf<int64_t> arp(static_cast<size_t>(an) + 1, s), acol(std::max<int64_t>(nnz_a, 1), s),
        brp(static_cast<size_t>(am) + 1, s), bcol(std::max<int64_t>(nnz_b, 1), s);
    DBuf<double> aval(std::max<int64_t>(nnz_a, 1), s), bval(std::max<int64_t>(nnz_b, 1), s);
    PB_CUDA(cudaMemcpyAsync(arp.get(), a_rp, 8 * (an + 1), cudaMemcpyHostToDevice, s));
    PB_CUDA(cudaMemcpyAsync(brp.get(), b_rp, 8 * (am + 1), cudaMemcpyHostToDevice, s));
    if (nnz_a) {
        PB_CUDA(cudaMemcpyAsync(acol.get(), a_col, 8 * nnz_a, cudaMemcpyHostToDevice, s));
        PB_CUDA(cudaMemcpyAsync(aval.get(), a_val, 8 * nnz_a, cudaMemcpyHostToDevice, s));
    }
    if (nnz_b) {
        PB_CUDA(cudaMemcpyAsync(bcol.get(), b_col, 8 * nnz_b, cudaMemcpyHostToDevice, s));
        PB_CUDA(cudaMemcpyAsync(bval.get(), b_val, 8 * nnz_b, cudaMemcpyHostToDevice, s));
    }
    if (nnz_a == 0) return C;
    DBuf<int32_t> rowid(static_cast<size_t>(nnz_a), s);
    DBuf<int64_t> off(static_cast<size_t>(nnz_a) + 1, s);
    k_rowid<<<blocks_for(an, 256), 256, 0, s>>>(arp.get(), an, rowid.get());
    k_contrib_count<<<blocks_for(nnz_a, 256), 256, 0, s>>>(acol.get(), nnz_a, brp.get(), off.get());
    PB_CHECK_LAUNCH();
    PB_CUDA(cudaMemsetAsync(off.get() + nnz_a, 0, 8, s));
    cub_run([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, off.get(), off.get(), static_cast<int>(nnz_a + 1), s);
    }, s);
    int64_t T = 0;
    PB_CUDA(cudaMemcpyAsync(&T, off.get() + nnz_a, 8, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (T >= (int64_t(1) << 31)) fail(PAIRAMG_INVALID_ARGUMENT, "spgemm: more than 2^31 products");
    if (T == 0) return C;
    DBuf<ull> key(static_cast<size_t>(T), s), key2(static_cast<size_t>(T), s);
    DBuf<double> val(static_cast<size_t>(T), s), val2(static_cast<size_t>(T), s);
    k_contrib_fill<<<blocks_for(nnz_a, 256), 256, 0, s>>>(rowid.get(), acol.get(), aval.get(), nnz_a, brp.get(),
                                                           bcol.get(), bval.get(), off.get(), key.get(), val.get());
    PB_CHECK_LAUNCH();
    int end_bit = 32;
    while (end_bit < 64 && (ull(1) << (end_bit - 32)) <= static_cast<ull>(an)) ++end_bit;
    cub_run([&](void* t, size_t& b) {  // LSD radix sort: stable, encounter order kept inside equal keys
        return cub::DeviceRadixSort::SortPairs(t, b, key.get(), key2.get(), val.get(), val2.get(), static_cast<int>(T),
                                               0, end_bit, s);
    }, s);
    DBuf<uint8_t> head(static_cast<size_t>(T), s);
    k_run_heads<<<blocks_for(T, 256), 256, 0, s>>>(key2.get(), T, head.get());
    PB_CHECK_LAUNCH();
    DBuf<int64_t> start(static_cast<size_t>(T), s), nsel(1, s);
    cub_run([&](void* t, size_t& b) {
        return cub::DeviceSelect::Flagged(t, b, thrust::counting_iterator<int64_t>(0), head.get(), start.get(),
                                          nsel.get(), static_cast<int>(T), s);
    }, s);
    int64_t nruns = 0;
    PB_CUDA(cudaMemcpyAsync(&nruns, nsel.get(), 8, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    DBuf<int64_t> ccol(static_cast<size_t>(nruns), s), rowcnt(static_cast<size_t>(an) + 1, s);
    DBuf<double> cval(static_cast<size_t>(nruns), s);
    rowcnt.zero(s);
    k_fold_runs<<<blocks_for(nruns, 256), 256, 0, s>>>(key2.get(), val2.get(), start.get(), nruns, T, ccol.get(),
                                                        cval.get(), rowcnt.get());
    PB_CHECK_LAUNCH();
    C.col.resize(static_cast<size_t>(nruns));
    C.val.resize(static_cast<size_t>(nruns));
    std::vector<int64_t> cnt(static_cast<size_t>(an) + 1);
    PB_CUDA(cudaMemcpyAsync(C.col.data(), ccol.get(), 8 * nruns, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaMemcpyAsync(C.val.data(), cval.get(), 8 * nruns, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaMemcpyAsync(cnt.data(), rowcnt.get(), 8 * an, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < an; ++i) C.row_ptr[static_cast<size_t>(i) + 1] = C.row_ptr[static_cast<size_t>(i)] + cnt[static_cast<size_t>(i)];
    return C;
}

}  // namespace pb
