// sell_win.cuh -- DICT operators with the gathered vector staged in shared
// memory by bulk asynchronous copies (included by sell.cu, anonymous
// namespace; uses SellArgs-era helpers from there).
//
// Why: the one-lane-per-row gather kernel is latency bound -- each entry is a
// dependent chain code load -> dictionary lookup -> x gather -> multiply, and
// at the register budget that keeps 64 warps resident ptxas cannot keep more
// than a couple of gathers in flight per warp (ncu: 13 of 22 cycles per
// instruction stalled on L1TEX, DRAM at 44 %).  A DICT row set has few
// distinct column offsets, so for a tile of T consecutive rows every gathered
// x lies in a handful of contiguous segments x[tile + lo_k, tile + T + hi_k)
// ("windows": offsets closer than kWinGap share one).  One thread streams the
// windows, the row's own r/d/q and the tile's code words into shared memory
// with cp.async.bulk (completion on an mbarrier) while the CTA computes the
// previous tile from the other stage; the gathers become shared-memory loads.
// The dictionary records carry the shared-memory index of their window
// (value, base): x of row i for that entry is sx[base + i].
//
// Arithmetic is unchanged (same CSR-order dadd/dmul chain per row, pads add
// +0.0 * own x), so every result is bitwise the one of k_sell.

constexpr int kWinThreads = 256;
constexpr int kWinSmemCap = 200 * 1024;  // dynamic shared memory ceiling of the window kernels

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct WinArgs {
    const uint32_t* code;
    int words;
    int row0, nrows, nslices, ntiles, T;
    int64_t xlen;
    int nwin;
    int lo[kWinMax], len[kWinMax], soff[kWinMax];  // per window: first offset, copied elements, smem offset
    int r_soff, d_soff, q_soff, c_soff, stage;    // smem offsets (doubles), stage size (doubles)
    int al_r, base0;                              // parity of the row-indexed copies; own-x index for row 0
    const double* x;
    double* y;
    const double* r;
    const double* d;
    const double* q;
    double omega;
    double* partials;
};

// Copy src[gs, gs + len) (gs even, clipped to [0, lim)) to dst[0, len) of a
// stage; an odd tail element is stored by the issuing thread (ordered before
// the consumers by its release-arrive).  Returns the bulk bytes.
__device__ __forceinline__ uint32_t win_copy(double* dst, const double* src, int64_t gs, int len, int64_t lim,
                                             uint64_t* bar) {
    const int64_t cs = gs < 0 ? 0 : gs;
    const int64_t ce = gs + len < lim ? gs + len : lim;
    if (ce <= cs) return 0;
    const int64_t n = ce - cs, ne = n & ~int64_t(1);
    double* d = dst + (cs - gs);
    if (ne) bulk_g2s(d, src + cs, static_cast<uint32_t>(ne * 8), bar);
    if (n & 1) d[ne] = src[cs + ne];
    return static_cast<uint32_t>(ne * 8);
}

template <int OP>
__device__ __forceinline__ void win_issue(const WinArgs& a, int t, double* st, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int64_t tr0 = static_cast<int64_t>(a.row0) + static_cast<int64_t>(t) * a.T;
    uint32_t bytes = 0;
    for (int k = 0; k < a.nwin; ++k) {
        const int64_t g = tr0 + a.lo[k];
        bytes += win_copy(st + a.soff[k], a.x, g - (g & 1), a.len[k], a.xlen, bar);
    }
    const int64_t rend = static_cast<int64_t>(a.row0) + a.nrows;
    const int rl = a.T + 2;
    if (OP != kSpmv) bytes += win_copy(st + a.r_soff, a.r, tr0 - a.al_r, rl, rend, bar);
    if (OP == kJacobi) bytes += win_copy(st + a.d_soff, a.d, tr0 - a.al_r, rl, rend, bar);
    if (OP < 0) bytes += win_copy(st + a.q_soff, a.q, tr0 - a.al_r, rl, rend, bar);
    const int64_t w0 = static_cast<int64_t>(t) * a.T * a.words;
    const int64_t wend = static_cast<int64_t>(a.nslices) * 32 * a.words;
    const int64_t nw = (w0 + static_cast<int64_t>(a.T) * a.words < wend ? static_cast<int64_t>(a.T) * a.words : wend - w0);
    bulk_g2s(st + a.c_soff, a.code + w0, static_cast<uint32_t>(nw * 4), bar);
    bytes += static_cast<uint32_t>(nw * 4);
    mbar_arrive_tx(bar, bytes);
}

// Row sum from the staged tile: codes at sc[(slice*W + w)*32 + lane].
__device__ __forceinline__ double win_row_sum(const WinArgs& a, const DictParam<true>& dp, const double* st,
                                              const uint32_t* sc, int i) {
    const int W = a.words;
    const uint32_t* cp = sc + (i >> 5) * W * 32 + (i & 31);
    double sum = 0.0;
    for (int w0 = 0; w0 < W; w0 += 2) {
        const uint32_t wa = cp[w0 * 32];
        const uint32_t wb = w0 + 1 < W ? cp[(w0 + 1) * 32] : 0xFFFFFFFFu;
        double av[8], xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t e = ((j < 4 ? wa : wb) >> (8 * (j & 3))) & 0xFFu;
            const ulonglong2 rec = dp.e[e];
            av[j] = __longlong_as_double(static_cast<long long>(rec.x));
            xv[j] = st[static_cast<int>(rec.y) + i];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) sum = dadd(sum, dmul(av[j], xv[j]));
    }
    return sum;
}

// OP: kSpmv / kJacobi / kResid, or -1 = SpMV + FCG dot triple (w.r, w.v, w.q).
template <int OP>
__global__ void __launch_bounds__(kWinThreads) k_win(WinArgs a, const __grid_constant__ DictParam<true> dp) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockIdx.x < a.ntiles) win_issue<OP>(a, blockIdx.x, smem, &bar[0]);
        if (blockIdx.x + gridDim.x < a.ntiles) win_issue<OP>(a, blockIdx.x + gridDim.x, smem + a.stage, &bar[1]);
    }
    double sa = 0.0, sb = 0.0, sg = 0.0;
    int it = 0;
    for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
        const int s = it & 1;
        mbar_wait(&bar[s], (it >> 1) & 1);
        const double* st = smem + s * a.stage;
        const uint32_t* sc = reinterpret_cast<const uint32_t*>(st + a.c_soff);
        for (int i = threadIdx.x; i < a.T; i += kWinThreads) {
            const int sr = t * a.T + i;
            if (sr >= a.nslices * 32) break;  // whole warp (T and the block are multiples of 32)
            const double sum = win_row_sum(a, dp, st, sc, i);
            if (sr < a.nrows) {
                const int row = a.row0 + sr;
                if (OP == kSpmv) {
                    a.y[row] = sum;
                } else if (OP == kResid) {
                    a.y[row] = dsub(st[a.r_soff + a.al_r + i], sum);
                } else if (OP == kJacobi) {
                    const double xi = st[a.base0 + i];
                    const double ri = st[a.r_soff + a.al_r + i], di = st[a.d_soff + a.al_r + i];
                    a.y[row] = dadd(xi, ddiv(dmul(a.omega, dsub(ri, sum)), di));
                } else {
                    const double wi = st[a.base0 + i];
                    a.y[row] = sum;
                    sa = dadd(sa, dmul(wi, st[a.r_soff + a.al_r + i]));
                    sb = dadd(sb, dmul(wi, sum));
                    sg = dadd(sg, dmul(wi, st[a.q_soff + a.al_r + i]));
                }
            }
        }
        __syncthreads();  // stage s fully consumed
        if (threadIdx.x == 0 && t + 2 * static_cast<int>(gridDim.x) < a.ntiles)
            win_issue<OP>(a, t + 2 * gridDim.x, smem + s * a.stage, &bar[s]);
    }
    if (OP < 0) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int o = 16; o; o >>= 1) {
            sa = dadd(sa, __shfl_down_sync(0xffffffffu, sa, o));
            sb = dadd(sb, __shfl_down_sync(0xffffffffu, sb, o));
            sg = dadd(sg, __shfl_down_sync(0xffffffffu, sg, o));
        }
        __shared__ double red[3][kWinThreads / 32];
        if (lane == 0) {
            red[0][warp] = sa;
            red[1][warp] = sb;
            red[2][warp] = sg;
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            double acc = 0.0;
            for (int k = 0; k < kWinThreads / 32; ++k) acc = dadd(acc, red[threadIdx.x][k]);
            a.partials[blockIdx.x * 3 + threadIdx.x] = acc;
        }
    }
}
