// sell_sten.cuh -- STEN storage: every row is an order-preserving subset of
// ONE main pattern (included by sell.cu, anonymous namespace).
//
// Layout: the main pattern's L <= 32 (column - row, value) records and, per
// row pattern (<= 255, one byte per row as in PAT), the bit mask of main
// records the row lacks plus its l1 diagonal -- all in the constant bank
// (kernel parameter).  Per row only the pattern byte is streamed; the l1
// diagonal stream disappears as in PAT.
//
// Why: in DICT/PAT every gather depends on a per-entry code or record load
// (load -> lookup -> gather -> multiply), so a warp keeps one or two gathers
// in flight and the sweeps are latency bound at ~45 % of HBM bandwidth.
// Here a gather address is row + off[k] with off[k] uniform: all L gathers
// and the row's own operands issue back to back before the first multiply,
// and the multiplies take their value from uniform registers.  Warps whose
// rows all carry the full pattern (the interior) skip the mask selects.
//
// Exactness: a row's sum runs over its own records in CSR order (the mask
// only drops absent records; a dropped add leaves the sum untouched), each
// record's value and column bitwise the CSR one -- the same dadd/dmul chain
// as spmv_local.  Absent records still load x at row + off (clamped into
// [0, xlen) in blocks that touch the vector ends) but never use it.

constexpr int kStenMax = 32;

struct StenParam {
    int off[kStenMax];
    double val[kStenMax];
    uint32_t pmask[256];  // main records absent from the pattern (bit k = record k)
    double pdiag[256];    // l1 diagonal of the pattern (bitwise = l1_diagonal)
    double pinv[256];     // RN(1 / pdiag) for ddiv_recip (0 = divide)
    int neg1;             // every record but the centre (L/2) holds exactly -1.0
};

// Boundary rows of a split launch: the faces of an interior rank reach
// different halo slots, so their merged main pattern can exceed 32 records
// (27-point: 36); the boundary blocks take up to 64 (generic length only).
constexpr int kStenWide = 64;
struct StenParamW {
    int off[kStenWide];
    double val[kStenWide];
    unsigned long long pmask[256];
    double pdiag[256];
    double pinv[256];
    int neg1;
};

struct StenArgs {
    const uint8_t* pid;  // pattern id per row (indexed by row id)
    const int32_t* rows;
    int row0, nrows, xlen;
    int L;
    int safe_lo, safe_hi;  // blocks [safe_lo, safe_hi) gather in range without clamping (contiguous rows)
    int pf_blocks;         // L2 prefetch distance in blocks (0 = off; contiguous rows only)
    int nblk;              // logical row blocks; the grid may be smaller (grid-stride loop)
    int offmax;
    const double* x;
    double* y;
    const double* r;
    double omega;
    const double* q;
    double* partials;
    const double* hsrc;  // boundary rows of a split launch: columns >= nown read hsrc[c - nown]
    int nown;
};

// Row sum over the main pattern; LL = compile-time record count (0 = generic,
// runtime a.L <= kStenMax).  EDGE clamps the gather columns into [0, xlen).
// With LL > 0 the launcher guarantees record LL/2 is the diagonal (offset
// 0, sorted symmetric stencil), so its gather doubles as the row's own x.
template <int LL, bool EDGE, bool HALO = false, typename PT = StenParam, typename MT = uint32_t>
__device__ __forceinline__ double sten_row_sum(const StenArgs& a, const PT& p, int row, MT m, double& own) {
    if constexpr (LL == 0) {
        // generic length: batches of 8 loads (registers, no local-memory array)
        double sum = 0.0;
        for (int k0 = 0; k0 < a.L; k0 += 8) {
            double xv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int c = row + (k0 + j < a.L ? p.off[k0 + j] : 0);
                if (EDGE) c = min(max(c, 0), a.xlen - 1);
                xv[j] = (HALO && c >= a.nown) ? __ldcv(a.hsrc + (c - a.nown)) : a.x[c];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = k0 + j;
                if (k < a.L && !((m >> k) & 1u)) sum = dadd(sum, dmul(p.val[k < a.L ? k : 0], xv[j]));
            }
        }
        return sum;
    } else {
        double xv[LL];
#pragma unroll
        for (int k = 0; k < LL; ++k) {
            int c = row + p.off[k];
            if (EDGE) c = min(max(c, 0), a.xlen - 1);
            xv[k] = a.x[c];  // coherent load: this kernel may start before x's producer completes (PDL)
        }
        double sum = 0.0;
        if (p.neg1) {  // as sten_fold_neg1: -1.0 records subtract (bitwise the same sum)
            if (__all_sync(0xffffffffu, m == 0u)) {
#pragma unroll
                for (int k = 0; k < LL; ++k)
                    sum = k == LL / 2 ? dadd(sum, dmul(p.val[k], xv[k])) : dsub(sum, xv[k]);
            } else {
#pragma unroll
                for (int k = 0; k < LL; ++k)
                    if (!((m >> k) & 1u)) sum = k == LL / 2 ? dadd(sum, dmul(p.val[k], xv[k])) : dsub(sum, xv[k]);
            }
        } else if (__all_sync(0xffffffffu, m == 0u)) {
#pragma unroll
            for (int k = 0; k < LL; ++k) sum = dadd(sum, dmul(p.val[k], xv[k]));
        } else {
#pragma unroll
            for (int k = 0; k < LL; ++k) {
                const double pr = dmul(p.val[k], xv[k]);
                if (!((m >> k) & 1u)) sum = dadd(sum, pr);
            }
        }
        own = xv[LL / 2];
        return sum;
    }
}

template <int LL, bool HALO = false, typename PT = StenParam, typename MT = uint32_t>
__device__ __forceinline__ double sten_sum(const StenArgs& a, const PT& p, int row, MT m, bool edge, double& own) {
    return edge ? sten_row_sum<LL, true, HALO, PT, MT>(a, p, row, m, own)
                : sten_row_sum<LL, false, HALO, PT, MT>(a, p, row, m, own);
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Streams the block pf_blocks ahead will touch first (its r rows, pattern
// bytes and the x rows its largest offset reaches) into L2, so those first
// touches overlap this block's latency instead of starting when it runs.
template <int OP, int BR = 256>
__device__ __forceinline__ void sten_prefetch(const StenArgs& a, const double* own, int blk) {
    if (a.pf_blocks <= 0 || threadIdx.x != 0) return;
    const int b = blk + a.pf_blocks;
    const int64_t first = static_cast<int64_t>(b) * BR;
    if (first >= a.nrows) return;
    const int64_t row = a.row0 + first;
    const int64_t xr = (row + a.offmax) & ~int64_t(1);
    if (xr + BR <= a.xlen) bulk_prefetch_l2(a.x + xr, 8 * BR);
    if (OP != kSpmv && first + BR <= a.nrows && !(row & 1)) bulk_prefetch_l2(own + row, 8 * BR);
    if (first + BR <= a.nrows && !(row & 15)) bulk_prefetch_l2(a.pid + row, BR);
}

// One thread per row (32-bit indices: a Sell holds < 2^31 rows); rows past
// nrows recompute the last row and do not store (every lane reaches the
// warp vote).  The clamp test is per block (uniform).
template <int OP, bool ROWS, int LL, bool HALO = false, typename PT = StenParam>
__device__ __forceinline__ void sten1_block(const StenArgs& a, const PT& p, int blk) {
    const int i = blk * 256 + static_cast<int>(threadIdx.x);
    const bool valid = i < a.nrows;
    const int ic = valid ? i : a.nrows - 1;
    const int row = ROWS ? a.rows[ic] : a.row0 + ic;
    const bool edge = ROWS || blk < a.safe_lo || blk >= a.safe_hi;
    if (!ROWS) sten_prefetch<OP>(a, a.r, blk);
    const int q = a.pid[row];
    double ri = 0.0, xi = 0.0;
    if (OP != kSpmv) ri = a.r[row];
    if (OP == kJacobi && LL == 0) xi = a.x[row];
    const double sum = sten_sum<LL, HALO>(a, p, row, p.pmask[q], edge, xi);
    if (!valid) return;
    if (OP == kSpmv) {
        a.y[row] = sum;
    } else if (OP == kResid) {
        a.y[row] = dsub(ri, sum);
    } else {
        const double t = dsub(ri, sum);  // omega = 1 (the paper's setting) multiplies exactly: skip it
        a.y[row] = dadd(xi, ddiv_recip(dmul(a.omega, t), p.pdiag[q], p.pinv[q]));  // 1.0 * t == t exactly
    }
}

// Grid-stride over the logical blocks: a capped grid leaves SM slots free for
// concurrent communication kernels (halo levels).
// GS: grid-stride over the logical blocks (a capped grid leaves SM slots to
// concurrent kernels); the one-block-per-CTA form keeps fewer registers.
template <int OP, bool ROWS, int LL, bool GS = false>
__global__ void __launch_bounds__(256) k_sten(StenArgs a, const __grid_constant__ StenParam p) {
    pdl_begin();
    if constexpr (GS) {
        for (int blk = static_cast<int>(blockIdx.x); blk < a.nblk; blk += static_cast<int>(gridDim.x))
            sten1_block<OP, ROWS, LL>(a, p, blk);
    } else {
        sten1_block<OP, ROWS, LL>(a, p, static_cast<int>(blockIdx.x));
    }
}

// Two rows per thread (rows t and t + 256 of a 512-row block), every load of
// both rows issued before the first multiply: twice the gathers in flight
// per warp at a register cost that still leaves 40+ warps per SM (LL = 7).
template <int LL, bool EDGE>
__device__ __forceinline__ void sten_load(const StenArgs& a, const StenParam& p, int row, double (&xv)[LL]) {
#pragma unroll
    for (int k = 0; k < LL; ++k) {
        int c = row + p.off[k];
        if (EDGE) c = min(max(c, 0), a.xlen - 1);
        xv[k] = a.x[c];  // coherent load: this kernel may start before x's producer completes (PDL)
    }
}

// x * -1.0 is exactly -x, so sum + (-1.0 * x) is bitwise sum - x: with
// p.neg1 (a uniform branch) the off-centre records skip their multiply.
template <int LL>
__device__ __forceinline__ double sten_fold_neg1(const StenParam& p, const double (&xv)[LL], uint32_t m) {
    double sum = 0.0;
    if (__all_sync(0xffffffffu, m == 0u)) {
#pragma unroll
        for (int k = 0; k < LL; ++k) sum = k == LL / 2 ? dadd(sum, dmul(p.val[k], xv[k])) : dsub(sum, xv[k]);
    } else {
#pragma unroll
        for (int k = 0; k < LL; ++k)
            if (!((m >> k) & 1u)) sum = k == LL / 2 ? dadd(sum, dmul(p.val[k], xv[k])) : dsub(sum, xv[k]);
    }
    return sum;
}

template <int LL>
__device__ __forceinline__ double sten_fold(const StenParam& p, const double (&xv)[LL], uint32_t m) {
    if (p.neg1) return sten_fold_neg1<LL>(p, xv, m);
    double sum = 0.0;
    if (__all_sync(0xffffffffu, m == 0u)) {
#pragma unroll
        for (int k = 0; k < LL; ++k) sum = dadd(sum, dmul(p.val[k], xv[k]));
    } else {
#pragma unroll
        for (int k = 0; k < LL; ++k) {
            const double pr = dmul(p.val[k], xv[k]);
            if (!((m >> k) & 1u)) sum = dadd(sum, pr);
        }
    }
    return sum;
}

template <int OP, int LL>
__device__ __forceinline__ void sten_store(const StenArgs& a, const StenParam& p, int row, int q, double ri,
                                           double xi, double sum) {
    if (OP == kSpmv) {
        a.y[row] = sum;
    } else if (OP == kResid) {
        a.y[row] = dsub(ri, sum);
    } else {
        const double t = dsub(ri, sum);
        a.y[row] = dadd(xi, ddiv_recip(dmul(a.omega, t), p.pdiag[q], p.pinv[q]));  // 1.0 * t == t exactly
    }
}

template <int OP, bool ROWS, int LL, bool EDGE>
__device__ __forceinline__ void sten2_body(const StenArgs& a, const StenParam& p, int ia, int ib) {
    const bool va = ia < a.nrows, vb = ib < a.nrows;
    const int ra = ROWS ? a.rows[va ? ia : a.nrows - 1] : a.row0 + (va ? ia : a.nrows - 1);
    const int rb = ROWS ? a.rows[vb ? ib : a.nrows - 1] : a.row0 + (vb ? ib : a.nrows - 1);
    const int qa = a.pid[ra], qb = a.pid[rb];
    double ria = 0.0, rib = 0.0;
    if (OP != kSpmv) {
        ria = a.r[ra];
        rib = a.r[rb];
    }
    double xa[LL], xb[LL];
    sten_load<LL, EDGE>(a, p, ra, xa);
    sten_load<LL, EDGE>(a, p, rb, xb);
    const double sa = sten_fold<LL>(p, xa, p.pmask[qa]);
    const double sb = sten_fold<LL>(p, xb, p.pmask[qb]);
    if (va) sten_store<OP, LL>(a, p, ra, qa, ria, xa[LL / 2], sa);
    if (vb) sten_store<OP, LL>(a, p, rb, qb, rib, xb[LL / 2], sb);
}

template <int OP, bool ROWS, int LL>
__device__ __forceinline__ void sten2_block(const StenArgs& a, const StenParam& p, int blk) {
    const int ia = blk * 512 + static_cast<int>(threadIdx.x);
    const bool edge = ROWS || blk < a.safe_lo || blk >= a.safe_hi;
    if (!ROWS) sten_prefetch<OP, 512>(a, a.r, blk);
    if (edge)
        sten2_body<OP, ROWS, LL, true>(a, p, ia, ia + 256);
    else
        sten2_body<OP, ROWS, LL, false>(a, p, ia, ia + 256);
}

template <int OP, bool ROWS, int LL, bool GS = false>
__global__ void __launch_bounds__(256) k_sten2(StenArgs a, const __grid_constant__ StenParam p) {
    pdl_begin();
    if constexpr (GS) {
        for (int blk = static_cast<int>(blockIdx.x); blk < a.nblk; blk += static_cast<int>(gridDim.x))
            sten2_block<OP, ROWS, LL>(a, p, blk);
    } else {
        sten2_block<OP, ROWS, LL>(a, p, static_cast<int>(blockIdx.x));
    }
}

// v = A w + block partials of (w.r, w.v, w.q) (fixed order -> deterministic).
template <bool ROWS, int LL, bool HALO = false, typename PT = StenParam>
__device__ __forceinline__ void sten1_dots_block(const StenArgs& a, const PT& p, int blk, double& sa, double& sb,
                                                 double& sg) {
    const int i = blk * 256 + static_cast<int>(threadIdx.x);
    const bool valid = i < a.nrows;
    const int ic = valid ? i : a.nrows - 1;
    const int row = ROWS ? a.rows[ic] : a.row0 + ic;
    const bool edge = ROWS || blk < a.safe_lo || blk >= a.safe_hi;
    if (!ROWS) sten_prefetch<-1>(a, a.r, blk);
    const int q = a.pid[row];
    double wi = LL == 0 ? a.x[row] : 0.0;
    const double rr = a.r[row], qq = a.q[row];
    const double sum = sten_sum<LL, HALO>(a, p, row, p.pmask[q], edge, wi);
    if (valid) {
        a.y[row] = sum;
        sa = dadd(sa, dmul(wi, rr));
        sb = dadd(sb, dmul(wi, sum));
        sg = dadd(sg, dmul(wi, qq));
    }
}

// Block sum of the dot triple in a fixed order -> partials[blockIdx.x] (3 doubles).
__device__ __forceinline__ void dots_block_store(double sa, double sb, double sg, double* partials) {
    for (int o = 16; o; o >>= 1) {
        sa = dadd(sa, __shfl_down_sync(0xffffffffu, sa, o));
        sb = dadd(sb, __shfl_down_sync(0xffffffffu, sb, o));
        sg = dadd(sg, __shfl_down_sync(0xffffffffu, sg, o));
    }
    __shared__ double red[3][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][warp] = sa;
        red[1][warp] = sb;
        red[2][warp] = sg;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double acc = 0.0;
        for (int k = 0; k < 8; ++k) acc = dadd(acc, red[threadIdx.x][k]);
        partials[blockIdx.x * 3 + threadIdx.x] = acc;
    }
}

// v = A w + per-CTA partials of (w.r, w.v, w.q) (fixed order -> deterministic).
template <bool ROWS, int LL, bool GS = false>
__global__ void __launch_bounds__(256) k_sten_dots(StenArgs a, const __grid_constant__ StenParam p) {
    pdl_begin();
    double sa = 0.0, sb = 0.0, sg = 0.0;
    if constexpr (GS) {
        for (int blk = static_cast<int>(blockIdx.x); blk < a.nblk; blk += static_cast<int>(gridDim.x))
            sten1_dots_block<ROWS, LL>(a, p, blk, sa, sb, sg);
    } else {
        sten1_dots_block<ROWS, LL>(a, p, static_cast<int>(blockIdx.x), sa, sb, sg);
    }
    dots_block_store(sa, sb, sg, a.partials);
}

// Two rows per thread (rows t and t + 256 of a 512-row block), as k_sten2.
template <bool ROWS, int LL, bool EDGE>
__device__ __forceinline__ void sten2_dots_body(const StenArgs& a, const StenParam& p, int ia, int ib, double& sa,
                                                double& sb, double& sg) {
    const bool va = ia < a.nrows, vb = ib < a.nrows;
    const int ra = ROWS ? a.rows[va ? ia : a.nrows - 1] : a.row0 + (va ? ia : a.nrows - 1);
    const int rb = ROWS ? a.rows[vb ? ib : a.nrows - 1] : a.row0 + (vb ? ib : a.nrows - 1);
    const int qa = a.pid[ra], qb = a.pid[rb];
    const double rra = a.r[ra], rrb = a.r[rb], qqa = a.q[ra], qqb = a.q[rb];
    double xa[LL], xb[LL];
    sten_load<LL, EDGE>(a, p, ra, xa);
    sten_load<LL, EDGE>(a, p, rb, xb);
    const double va_ = sten_fold<LL>(p, xa, p.pmask[qa]);
    const double vb_ = sten_fold<LL>(p, xb, p.pmask[qb]);
    const double wa = xa[LL / 2], wb = xb[LL / 2];
    if (va) {
        a.y[ra] = va_;
        sa = dadd(sa, dmul(wa, rra));
        sb = dadd(sb, dmul(wa, va_));
        sg = dadd(sg, dmul(wa, qqa));
    }
    if (vb) {
        a.y[rb] = vb_;
        sa = dadd(sa, dmul(wb, rrb));
        sb = dadd(sb, dmul(wb, vb_));
        sg = dadd(sg, dmul(wb, qqb));
    }
}

template <bool ROWS, int LL>
__device__ __forceinline__ void sten2_dots_block(const StenArgs& a, const StenParam& p, int blk, double& sa, double& sb,
                                                 double& sg) {
    const int ia = blk * 512 + static_cast<int>(threadIdx.x);
    const bool edge = ROWS || blk < a.safe_lo || blk >= a.safe_hi;
    if (!ROWS) sten_prefetch<-1, 512>(a, a.r, blk);
    if (edge)
        sten2_dots_body<ROWS, LL, true>(a, p, ia, ia + 256, sa, sb, sg);
    else
        sten2_dots_body<ROWS, LL, false>(a, p, ia, ia + 256, sa, sb, sg);
}

// Per-WARP partial triples (partials[(block * 8 + warp) * 3 + k]): no block
// barrier at the end of the row work (ncu: 1.5 of ~15 stall cycles per issue
// were that barrier); the fixed-order reduction takes 8x the partials.
__device__ __forceinline__ void dots_warp_store(double sa, double sb, double sg, double* partials) {
    for (int o = 16; o; o >>= 1) {
        sa = dadd(sa, __shfl_down_sync(0xffffffffu, sa, o));
        sb = dadd(sb, __shfl_down_sync(0xffffffffu, sb, o));
        sg = dadd(sg, __shfl_down_sync(0xffffffffu, sg, o));
    }
    if ((threadIdx.x & 31) == 0) {
        double* out = partials + (static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5)) * 3;
        out[0] = sa;
        out[1] = sb;
        out[2] = sg;
    }
}

template <bool ROWS, int LL, bool GS = false>
__global__ void __launch_bounds__(256) k_sten2_dots(StenArgs a, const __grid_constant__ StenParam p) {
    pdl_begin();
    double sa = 0.0, sb = 0.0, sg = 0.0;
    if constexpr (GS) {
        for (int blk = static_cast<int>(blockIdx.x); blk < a.nblk; blk += static_cast<int>(gridDim.x))
            sten2_dots_block<ROWS, LL>(a, p, blk, sa, sb, sg);
        dots_block_store(sa, sb, sg, a.partials);
    } else {
        sten2_dots_block<ROWS, LL>(a, p, static_cast<int>(blockIdx.x), sa, sb, sg);
        dots_warp_store(sa, sb, sg, a.partials);
    }
}


// ---------------------------------------------------------------------------
// 27-point STEN on a contiguous row set, 2.5-D blocked ("marching" form).
// Applies when the main pattern is the full 3x3x3 box: record
// 9*(dk+1) + 3*(dj+1) + (di+1) at offset di + nx*dj + nxy*dk (levels of the
// 27-point hierarchies; nx, nxy read off the pattern).  Row r is split as
// r = i + nx*j + nxy*k (a bijection; the split only organises the work): a
// CTA owns a 32 x 8 (i, j) tile and marches over kz consecutive k.  Every
// haloed x-plane (34 x 10) is copied ONCE into shared memory by cp.async
// (four buffers, two planes in flight, one barrier per plane) and each
// thread reads its 3x3 neighbourhood of it; that plane feeds three rows of
// the thread's column (records 18..26 of row k-1, 9..17 of row k, 0..8 of
// row k+1), so only one plane of values and two running sums live in
// registers.  Per row: ~1.3 global + 9 shared loads instead of 27 gathers.
// The k_sten<27> gather kernel was latency-bound (47 M instructions per
// 192^3 sweep, 31 % occupancy at 68 registers, 96 us); this form runs at
// 4 CTAs per SM (<= 64 registers): 72 us.  The value used for record
// (dk, dj, di) of row r is x[r + di + nx*dj + nxy*dk] = x[r + off] exactly
// as in k_sten, halo cells included (the index is linear in (i, j, k));
// records absent from a row's pattern are skipped by its mask; each row's
// sum runs in record order: bitwise k_sten.
constexpr int kMarchTX = 32, kMarchTY = 8;
constexpr int kMarchMinBlocks = 4;  // CTAs per SM (<= 64 registers; 4 beat 3 and 2: 72 vs 86 vs 119 us)
constexpr int kMarchWaves = 2;      // grid ~ two waves: planes per CTA = columns * planes / (2 * 4 * 148)
constexpr int kMarchHX = kMarchTX + 2, kMarchHY = kMarchTY + 2, kMarchPlane = kMarchHX * kMarchHY;

struct MarchGeom {
    int nx, nxy, ny;           // row split r = i + nx*j + nxy*k (rows < 2^31)
    int tiles_x, tiles_y;      // (i, j) tiles per plane
    int k0, nk;                // planes [k0, k0 + nk) hold the row set
    int kz, chunks;            // planes per CTA, ceil(nk / kz)
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kMarchBuf = 4;  // planes in shared memory: 2 being read, 2 in flight (cp.async)

// Fold N values into a row sum as records BASE .. BASE+N-1 (record order;
// masked records skipped; records other than the diagonal DIAG subtract
// when neg1).  The uniform branches (neg1, every row of the warp complete)
// are hoisted out of the record loop.
template <int BASE, int N, int DIAG>
__device__ __forceinline__ double march_fold(const StenParam& p, const double* v, double sum, uint32_t m, bool full) {
    if (p.neg1) {
        if (full) {
#pragma unroll
            for (int t = 0; t < N; ++t) sum = (BASE + t == DIAG) ? dadd(sum, dmul(p.val[DIAG], v[t])) : dsub(sum, v[t]);
        } else {
#pragma unroll
            for (int t = 0; t < N; ++t)
                if (!((m >> (BASE + t)) & 1u))
                    sum = (BASE + t == DIAG) ? dadd(sum, dmul(p.val[DIAG], v[t])) : dsub(sum, v[t]);
        }
    } else {
#pragma unroll
        for (int t = 0; t < N; ++t)
            if (full || !((m >> (BASE + t)) & 1u)) sum = dadd(sum, dmul(p.val[BASE + t], v[t]));
    }
    return sum;
}

// The 3x3 neighbourhood of a plane (9 shared loads): records 0-8 of the row
// above, 9-17 (diagonal 13) of the row in the plane, 18-26 of the row below.
struct MarchPlane {
    double v[9];
    __device__ __forceinline__ void load(const double* buf, int lx, int ly) {
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) v[3 * dy + dx] = buf[(ly + dy) * kMarchHX + lx + dx];
    }
    __device__ __forceinline__ double centre() const { return v[4]; }
    __device__ __forceinline__ double first(const StenParam& p, uint32_t m, bool f) const {
        return march_fold<0, 9, 13>(p, v, 0.0, m, f);
    }
    __device__ __forceinline__ double mid(const StenParam& p, double s, uint32_t m, bool f) const {
        return march_fold<9, 9, 13>(p, v, s, m, f);
    }
    __device__ __forceinline__ double last(const StenParam& p, double s, uint32_t m, bool f) const {
        return march_fold<18, 9, 13>(p, v, s, m, f);
    }
};

// Streaming form: plane P, read once from shared memory, feeds three rows of
// the thread's column -- the last records of row P-1 (which then completes),
// the middle records of row P and the first of row P+1 -- so one plane of
// values and two running sums (each in record order: bitwise k_sten) live in
// registers, and a row's pattern byte / r / q load two planes before use.
template <int OP, bool DOTS>
__device__ __forceinline__ void march_body(const StenArgs& a, const StenParam& p, const MarchGeom& g, int blk,
                                           double& sa, double& sb, double& sg) {
    __shared__ double pl[kMarchBuf][kMarchPlane];
    const int tx = blk % g.tiles_x;
    blk /= g.tiles_x;
    const int ty = blk % g.tiles_y;
    const int kc = blk / g.tiles_y;
    const int i0 = tx * kMarchTX, j0 = ty * kMarchTY;
    const int kb = g.k0 + kc * g.kz;
    const int kend = min(kb + g.kz, g.k0 + g.nk);
    const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
    const bool h1ok = threadIdx.x + 256 < kMarchPlane;
    const int h0 = threadIdx.x, h1 = threadIdx.x + 256;
    const int c0 = (i0 - 1 + h0 % kMarchHX) + g.nx * (j0 - 1 + h0 / kMarchHX);
    const int c1 = (i0 - 1 + h1 % kMarchHX) + g.nx * (j0 - 1 + h1 / kMarchHX);
    const int st = g.nxy, hi = a.xlen - 1;
    const int i = i0 + lx, j = j0 + ly;
    const bool col_ok = i < g.nx && j < g.ny;
    const int colrow = i + g.nx * j;
    const int row_lo = a.row0, row_hi = a.row0 + a.nrows;
    // plane P -> buffer (P - kb + 1) % kMarchBuf, copied asynchronously
    auto issue = [&](int P) {
        if (P <= kend) {
            const int bf = (P - kb + 1) & (kMarchBuf - 1);
            cp_async8(&pl[bf][h0], a.x + min(max(c0 + st * P, 0), hi));
            if (h1ok) cp_async8(&pl[bf][h1], a.x + min(max(c1 + st * P, 0), hi));
        }
        cp_async_commit();  // one group per plane slot, empty past the chunk: uniform counting
    };
    issue(kb - 1);
    issue(kb);
    issue(kb + 1);
    // rows of this CTA: k in [kb, kend); row (i, j, k) = colrow + st*k
    double s_old = 0.0, s_mid = 0.0;  // rows P-1 and P, their records before plane P folded
    uint32_t m_old = 0u, m_mid = 0u;
    bool f_old = true, f_mid = true, ok_old = false, ok_mid = false;
    int q_old = 0, q_mid = 0, r_old = 0, r_mid = 0;
    double ri_old = 0.0, ri_mid = 0.0, qq_old = 0.0, qq_mid = 0.0;
    double x_old = 0.0;  // own x of row P-1 (centre of plane P-1)
    for (int P = kb - 1; P <= kend; ++P) {
        // row P+1 starts at this plane: its operands now, used two planes later
        const int r64 = colrow + st * (P + 1);
        const bool ok_new = col_ok && P + 1 >= kb && P + 1 < kend && r64 >= row_lo && r64 < row_hi;
        const int r_new = ok_new ? r64 : row_lo;
        const int q_new = a.pid[r_new];
        const double ri_new = (OP != kSpmv || DOTS) ? a.r[r_new] : 0.0;
        const double qq_new = DOTS ? a.q[r_new] : 0.0;
        cp_async_wait<1>();  // plane P landed; P+1 may still fly
        __syncthreads();     // ... for every thread; the buffer of plane P-2 is free
        issue(P + 2);
        MarchPlane v;
        v.load(pl[(P - kb + 1) & (kMarchBuf - 1)], lx, ly);
        if (P - 1 >= kb) {  // row P-1 completes
            const double sum = v.last(p, s_old, m_old, f_old);
            if (ok_old) {
                if (DOTS) {
                    a.y[r_old] = sum;
                    sa = dadd(sa, dmul(x_old, ri_old));
                    sb = dadd(sb, dmul(x_old, sum));
                    sg = dadd(sg, dmul(x_old, qq_old));
                } else {
                    sten_store<OP, 27>(a, p, r_old, q_old, ri_old, x_old, sum);
                }
            }
        }
        s_old = v.mid(p, s_mid, m_mid, f_mid);  // row P
        m_old = m_mid, f_old = f_mid, ok_old = ok_mid, q_old = q_mid, r_old = r_mid, ri_old = ri_mid, qq_old = qq_mid;
        x_old = v.centre();
        const uint32_t m_new = p.pmask[q_new];
        const bool f_new = __all_sync(0xffffffffu, !ok_new || m_new == 0u);
        s_mid = v.first(p, m_new, f_new);  // row P+1
        m_mid = m_new, f_mid = f_new, ok_mid = ok_new, q_mid = q_new, r_mid = r_new, ri_mid = ri_new, qq_mid = qq_new;
    }
    cp_async_wait<0>();
}

template <int OP>
__global__ void __launch_bounds__(256, kMarchMinBlocks) k_sten_march(StenArgs a, const __grid_constant__ StenParam p, MarchGeom g) {
    pdl_begin();
    double sa = 0.0, sb = 0.0, sg = 0.0;
    march_body<OP, false>(a, p, g, static_cast<int>(blockIdx.x), sa, sb, sg);
}

// v = A w + per-CTA partials of (w.r, w.v, w.q), marching form.
__global__ void __launch_bounds__(256, kMarchMinBlocks) k_sten_march_dots(StenArgs a, const __grid_constant__ StenParam p, MarchGeom g) {
    pdl_begin();
    double sa = 0.0, sb = 0.0, sg = 0.0;
    march_body<kSpmv, true>(a, p, g, static_cast<int>(blockIdx.x), sa, sb, sg);
    dots_block_store(sa, sb, sg, a.partials);
}

// ---------------------------------------------------------------------------
// The coarsest level's whole smoothing (zero start + nu-1 l1-Jacobi sweeps,
// cycle.cpp:86-93) in ONE launch of one thread-block cluster: every CTA
// owns R consecutive rows, keeps its slice of the iterate in shared memory
// (ping-pong), gathers neighbours from the owning CTA's shared memory
// (distributed shared memory) and the cluster barrier separates the sweeps.
// Replaces nu launch-bound kernels (19 x ~3.7 us at 256^3) by one.  Row sums
// in CSR order with the same dadd/dmul chain: bitwise the sweep kernels.
constexpr int kCoarseCta = 8;          // portable cluster size
constexpr int kCoarseThreads = 1024;
constexpr int kCoarseRows = 2048;      // rows per CTA (2 per thread)

template <int LL>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_solve(StenArgs a, const __grid_constant__ StenParam p,
                                                                 double* out, int nu, int R) {
    namespace cg = cooperative_groups;
    pdl_begin();
    __shared__ double xs[2][kCoarseRows];
    cg::cluster_group cl = cg::this_cluster();
    const int me = static_cast<int>(cl.block_rank());
    const int n = a.nrows;
    const int L = LL ? LL : a.L;
    int rowv[2];
    double rv[2], dv[2], yv[2];
    uint32_t mv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int t = static_cast<int>(threadIdx.x) + h * kCoarseThreads;
        const int row = me * R + t;
        rowv[h] = (t < R && row < n) ? row : -1;
        if (rowv[h] >= 0) {
            const int q = a.pid[row];
            rv[h] = a.r[row];
            dv[h] = p.pdiag[q];
            yv[h] = p.pinv[q];
            mv[h] = p.pmask[q];
            xs[0][t] = ddiv_recip(a.omega == 1.0 ? rv[h] : dmul(a.omega, rv[h]), dv[h], yv[h]);  // zero start
        }
    }
    cl.sync();
    for (int sweep = 1; sweep < nu; ++sweep) {
        const int cur = (sweep - 1) & 1, nxt = sweep & 1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (rowv[h] < 0) continue;
            const int row = rowv[h];
            double sum = 0.0;
            for (int k0 = 0; k0 < L; k0 += 8) {  // 8 independent DSMEM loads in flight, then the CSR-order sum
                double xv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int k = k0 + j;
                    int c = row + (k < L ? p.off[k] : 0);
                    c = min(max(c, 0), n - 1);
                    const int owner = c / R, loc = c - owner * R;
                    xv[j] = *cl.map_shared_rank(&xs[cur][loc], owner);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int k = k0 + j;
                    if (k < L && !((mv[h] >> k) & 1u)) sum = dadd(sum, dmul(p.val[k], xv[j]));
                }
            }
            const int t = row - me * R;
            const double t1 = dsub(rv[h], sum);
            xs[nxt][t] = dadd(xs[cur][t], ddiv_recip(a.omega == 1.0 ? t1 : dmul(a.omega, t1), dv[h], yv[h]));
        }
        cl.sync();
    }
    const int fin = (nu - 1) & 1;
#pragma unroll
    for (int h = 0; h < 2; ++h)
        if (rowv[h] >= 0) out[rowv[h]] = xs[fin][rowv[h] - me * R];
}

// ---------------------------------------------------------------------------
// Interior + halo-boundary rows of a halo level in ONE launch, with the halo
// delivered by NVLink direct stores (p2p.cu).  Block order: push |
// interior[0, bnd_at) | boundary | interior[bnd_at, nblk_a), bnd_at = two
// resident waves before the end of the interior.  The push blocks (lowest
// ids, dispatched first) store this rank's boundary values into the
// neighbours' staging and raise their flags; they never wait.  The interior
// blocks never wait either.  Only the boundary blocks wait, for every
// neighbour's flag of this exchange, then gather halo columns straight from
// the staging slot of its parity; dispatched late in the grid their halo has
// normally arrived, and the last interior waves overlap them instead of a
// serial boundary tail.  No circular wait: a neighbour's push for exchange k
// sits in the first blocks of its own launch k, which depends only on its
// exchange k-1 having completed (its boundary blocks of k-1 waited for OUR
// push k-1, already done); the blocks of this grid that a waiting boundary
// block could delay never wait themselves, and the neighbour's GPU is a
// different device.  (Ranks sharing one GPU -- LOCAL
// runtime -- do not use this launch: Solver::split_launch.)  The last
// boundary block advances the exchange counter (read by the next push).
struct HaloSplit {
    StenParam pa;              // interior main pattern
    StenParamW pb;             // boundary main pattern (<= 64 records)
    StenArgs b;                // boundary rows (list, or range on an end rank)
    int nblk_a, nblk_b;
    const unsigned long long* flags;  // this rank's flag slots (indexed by sender)
    int nfrom;
    int from[8];
    const double* staging;     // this rank's staging, parity stride nhalo
    int64_t nhalo;
    unsigned long long* ctr;   // [0] exchanges done, [3] boundary blocks done, [4]/[5] pushes / push blocks
    // fused push: blocks [0, npush) store this rank's boundary values into
    // the neighbours' staging, then [npush, npush + nblk_b) are the boundary
    // rows and the rest the interior
    int npush, npeers;
    int bnd_at;                // interior blocks before the boundary blocks (block order
                               // push | interior[0, bnd_at) | boundary | interior[bnd_at, nblk_a))
    int64_t off[9];
    double* dst[8];
    int64_t stride[8];
    unsigned long long* pflag[8];
    const int32_t* send_idx;
};

// One push block: a grid-stride share of x[send_idx] into the peers' staging
// slots of parity (pushes done & 1); the last push block advances the push
// count and raises the peers' flags (system-scope release after a system
// fence, as k_p2p_push).  Runs after the launch's griddepcontrol.wait, so x
// is the previous kernel's complete output.
__device__ __forceinline__ void halo_push_block(const HaloSplit& h, const double* x, int blk) {
    const unsigned long long e = h.ctr[4];
    const int64_t par = static_cast<int64_t>(e & 1ull);
    const int64_t nsend = h.off[h.npeers];
    for (int64_t i = blk * int64_t(256) + threadIdx.x; i < nsend; i += int64_t(h.npush) * 256) {
        int p = 0;
        while (p + 1 < h.npeers && i >= h.off[p + 1]) ++p;
        h.dst[p][par * h.stride[p] + (i - h.off[p])] = x[h.send_idx[i]];
    }
    __threadfence_system();
    __syncthreads();
    // every push block's stores are system-visible (its fence) before its
    // count; the last block's acq_rel count therefore follows all of them,
    // and its flag store needs no second system fence (~3 us of the level-1
    // launch's critical path under the interior's HBM load)
    if (threadIdx.x == 0) {
        unsigned long long prev;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(prev) : "l"(h.ctr + 5) : "memory");
        if (prev == static_cast<unsigned long long>(h.npush) - 1) {
            h.ctr[5] = 0;
            h.ctr[4] = e + 1;
            for (int p = 0; p < h.npeers; ++p)
                asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(h.pflag[p]), "l"(e + 1) : "memory");
        }
    }
}

// Block rel (past the push blocks) -> boundary block index, or -1 with the
// interior block index in blk.
__device__ __forceinline__ int split_bnd_index(const HaloSplit& h, int rel, int& blk) {
    blk = rel;
    if (rel < h.bnd_at) return -1;
    const int bb = rel - h.bnd_at;
    if (bb < h.nblk_b) return bb;
    blk = rel - h.nblk_b;
    return -1;
}

__device__ __forceinline__ const double* halo_wait_p2p(const HaloSplit& h) {
    const unsigned long long e = h.ctr[0];
    if (threadIdx.x == 0) {
        for (int k = 0; k < h.nfrom; ++k) {
            long long spins = 0;
            unsigned long long v;
            do {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(h.flags + h.from[k]) : "memory");
                if (v < e + 1) __nanosleep(64);
                if (++spins == (1ll << 28)) {
                    printf("pairamg: halo flag wait timed out\n");
                    __trap();
                }
            } while (v < e + 1);
        }
    }
    __syncthreads();
    return h.staging + static_cast<int64_t>(e & 1ull) * h.nhalo;
}

__device__ __forceinline__ void halo_done_p2p(const HaloSplit& h) {
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&h.ctr[3], 1ull) == static_cast<unsigned long long>(h.nblk_b) - 1) {
        h.ctr[3] = 0;
        h.ctr[0] = h.ctr[0] + 1;
    }
}

// 7 records: hold the interior at k_sten2's 5 CTAs/SM (<= 51 registers); the
// push / generic boundary paths otherwise raise the whole kernel to 54 and
// cost the interior a fifth of its warps.
template <int OP, int LLA, bool R2, bool BROWS>
__global__ void __launch_bounds__(256, LLA == 7 ? 5 : 1) k_sten_split(StenArgs a, const __grid_constant__ HaloSplit h) {
    pdl_wait_only();  // no early dependents (measured: an early trigger gains nothing here)
    // push blocks first; then most of the interior rows, whose pass covers
    // the neighbours' pushes, and the boundary rows once their halo has
    // arrived -- boundary blocks dispatched first would hold SM slots while
    // they wait (measured +25-30 us per level-0 sweep at 4 GPUs)
    if (static_cast<int>(blockIdx.x) < h.npush) {
        halo_push_block(h, a.x, static_cast<int>(blockIdx.x));
        return;
    }
    int blk;
    const int bb = split_bnd_index(h, static_cast<int>(blockIdx.x) - h.npush, blk);
    if (bb < 0) {
        if constexpr (R2) {
            const int ia = blk * 512 + static_cast<int>(threadIdx.x);
            const bool edge = blk < a.safe_lo || blk >= a.safe_hi;
            sten_prefetch<OP, 512>(a, a.r, blk);
            if (edge)
                sten2_body<OP, false, LLA, true>(a, h.pa, ia, ia + 256);
            else
                sten2_body<OP, false, LLA, false>(a, h.pa, ia, ia + 256);
        } else {
            sten1_block<OP, false, LLA>(a, h.pa, blk);
        }
        return;
    }
    StenArgs b = h.b;
    b.hsrc = halo_wait_p2p(h);
    sten1_block<OP, BROWS, 0, true>(b, h.pb, bb);
    halo_done_p2p(h);
}

template <int LLA, bool R2, bool BROWS>
__global__ void __launch_bounds__(256, LLA == 7 ? 5 : 2) k_sten_split_dots(StenArgs a, const __grid_constant__ HaloSplit h) {
    pdl_wait_only();
    double sa = 0.0, sb = 0.0, sg = 0.0;
    if (static_cast<int>(blockIdx.x) < h.npush) {  // push blocks first (zero partials)
        halo_push_block(h, a.x, static_cast<int>(blockIdx.x));
        dots_block_store(sa, sb, sg, a.partials);
        return;
    }
    int blk;  // then interior / boundary as k_sten_split
    const int bb = split_bnd_index(h, static_cast<int>(blockIdx.x) - h.npush, blk);
    if (bb < 0) {
        if constexpr (R2) {
            const int ia = blk * 512 + static_cast<int>(threadIdx.x);
            const bool edge = blk < a.safe_lo || blk >= a.safe_hi;
            sten_prefetch<-1, 512>(a, a.r, blk);
            if (edge)
                sten2_dots_body<false, LLA, true>(a, h.pa, ia, ia + 256, sa, sb, sg);
            else
                sten2_dots_body<false, LLA, false>(a, h.pa, ia, ia + 256, sa, sb, sg);
        } else {
            sten1_dots_block<false, LLA>(a, h.pa, blk, sa, sb, sg);
        }
        dots_block_store(sa, sb, sg, a.partials);
        return;
    }
    StenArgs b = h.b;
    b.hsrc = halo_wait_p2p(h);
    sten1_dots_block<BROWS, 0, true>(b, h.pb, bb, sa, sb, sg);
    dots_block_store(sa, sb, sg, a.partials);
    halo_done_p2p(h);
}

// The split launch with marching interior blocks (27-point levels whose
// interior is a contiguous plane range, sten_march): push | marching tiles |
// boundary rows, so a halo level keeps the 72-us marching sweep and still
// needs no communication stream, pull kernel or cross-stream join.  The
// boundary rows stay on the generic per-row path (their halo records read
// the staging buffer).  Same 4-CTA/SM bound as k_sten_march.
template <int OP, bool BROWS>
__global__ void __launch_bounds__(256, kMarchMinBlocks) k_sten_march_split(StenArgs a, const __grid_constant__ HaloSplit h,
                                                                            MarchGeom g) {
    pdl_wait_only();
    double sa = 0.0, sb = 0.0, sg = 0.0;
    if (static_cast<int>(blockIdx.x) < h.npush) {
        halo_push_block(h, a.x, static_cast<int>(blockIdx.x));
        return;
    }
    int blk;
    const int bb = split_bnd_index(h, static_cast<int>(blockIdx.x) - h.npush, blk);
    if (bb < 0) {
        march_body<OP, false>(a, h.pa, g, blk, sa, sb, sg);
        return;
    }
    StenArgs b = h.b;
    b.hsrc = halo_wait_p2p(h);
    sten1_block<OP, BROWS, 0, true>(b, h.pb, bb);
    halo_done_p2p(h);
}

template <bool BROWS>
__global__ void __launch_bounds__(256, kMarchMinBlocks) k_sten_march_split_dots(StenArgs a, const __grid_constant__ HaloSplit h,
                                                                                 MarchGeom g) {
    pdl_wait_only();
    double sa = 0.0, sb = 0.0, sg = 0.0;
    if (static_cast<int>(blockIdx.x) < h.npush) {
        halo_push_block(h, a.x, static_cast<int>(blockIdx.x));
        dots_block_store(sa, sb, sg, a.partials);
        return;
    }
    int blk;
    const int bb = split_bnd_index(h, static_cast<int>(blockIdx.x) - h.npush, blk);
    if (bb < 0) {
        march_body<kSpmv, true>(a, h.pa, g, blk, sa, sb, sg);
        dots_block_store(sa, sb, sg, a.partials);
        return;
    }
    StenArgs b = h.b;
    b.hsrc = halo_wait_p2p(h);
    sten1_dots_block<BROWS, 0, true>(b, h.pb, bb, sa, sb, sg);
    dots_block_store(sa, sb, sg, a.partials);
    halo_done_p2p(h);
}


