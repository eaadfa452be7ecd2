// sell.cu -- SELL-32 storage and the row-sum kernels of the solve path.
//
// Two lossless encodings of the same rows (matrix.cuh):
//  * PLAIN : per-slice width, int32 column + f64 value per entry (12 B),
//            pad column -1, slice offsets in `slice_off`.
//  * DICT  : one byte per entry indexing a per-matrix dictionary of distinct
//            (column - row, value) pairs (<= 255 pairs; code 0xFF = pad),
//            packed 4 per 32-bit word; every row padded to the same W words
//            so a lane's words sit at code[(slice*W + w)*32 + lane] (no offset
//            table on the critical path).  Chosen automatically when the rows
//            have <= 255 distinct pairs (every level of the slab-aligned
//            Poisson hierarchies has 7 or 27).  The dictionary travels in the
//            constant bank (kernel parameter), with the distinct l1 diagonal
//            values when a level has <= 256 of them (then a 1-byte code per
//            row replaces the 8-byte diagonal stream).  Columns and values
//            are reproduced exactly, so every row sum is bit-identical to
//            PLAIN and to spmv_local.
//
// Operators (one warp per slice, one lane per row, CSR-order sums with
// separately rounded multiply/add; the row's own operands are loaded before
// the gather chain so their latency overlaps it):
//   kSpmv        y = A x                                  (spmv_dist, dist.cpp:164-187)
//   kJacobi      y = x + (omega*(r - A x))/d              (cycle.cpp:56-60)
//   kResid       y = r - A x                              (cycle.cpp:101-103)
//   spmv+dots    v = A w with the FCG dot triple (w.r, w.v, w.q) (Alg. 1 l.10-13)
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "matrix.cuh"

namespace pb {

namespace {

using ull = unsigned long long;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kDictMax = 255;
constexpr int kTableCap = 1024;
constexpr ull kEmptyLo = 0x8000000000000000ULL;

// STEN sweeps divide by the pattern's l1 diagonal through ddiv_recip
// (common.cuh) with a host-computed reciprocal (bitwise the IEEE quotient).
constexpr bool fast_div() { return true; }

struct SellArgs {
    const int64_t* soff;  // PLAIN
    const int32_t* col;
    const double* val;
    const uint32_t* code;  // DICT
    int words;             // DICT: words per row
    const ulonglong2* dict;  // DICT: 256 records {value bits, column offset}
    const int32_t* rows;
    int row0;  // first row when the row set is a contiguous range (rows == nullptr)
    int64_t nslices, nrows;
    const double* x;
    double* y;
    const double* r;
    const double* d;
    double omega;
    const double* q;
    double* partials;
};

template <int OP>
__device__ __forceinline__ double xval(const SellArgs& a, int c) {
    return __ldg(a.x + c);
}

template <int OP>
__device__ __forceinline__ double row_sum_plain(const SellArgs& a, int64_t slice, int lane) {
    const int64_t beg = a.soff[slice];
    const int width = static_cast<int>((a.soff[slice + 1] - beg) >> 5);
    const int32_t* cp = a.col + beg + lane;
    const double* vp = a.val + beg + lane;
    double sum = 0.0;
    for (int k = 0; k < width; k += 8) {
        int c[8];
        double av[8], xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const bool in = k + j < width;
            c[j] = in ? __ldg(cp + (k + j) * 32) : -1;
            av[j] = in ? __ldg(vp + (k + j) * 32) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = c[j] >= 0 ? xval<OP>(a, c[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (c[j] >= 0) sum = dadd(sum, dmul(av[j], xv[j]));
    }
    return sum;
}

// The dictionary (256 records {value bits, column offset}; slot 255 = pad =
// {0, 0}) travels as a 4 KB __grid_constant__ kernel parameter: lookups are
// indexed constant-bank loads (LDC), served by the constant cache --
// broadcast when a warp's lanes share a code (interior slices) -- instead
// of competing with the gathers for L1TEX bandwidth.
// F: kFPlain / kFDict / kFCoded (the row-sum flavour of k_sell).  CODED
// uses only the value half of each record.
constexpr int kFPlain = 0, kFDict = 1, kFCoded = 2;
template <int F>
struct DictParam {
    ulonglong2 e[256];
};
template <>
struct DictParam<kFPlain> {
    int unused;
};

__device__ __forceinline__ void dict_entry(const DictParam<kFDict>& dp, uint32_t e, double& v, int& dc) {
    const ulonglong2 r = dp.e[e];
    v = __longlong_as_double(static_cast<long long>(r.x));
    dc = static_cast<int>(r.y);
}

// DICT row sum: the lane's words are code[(slice*W + w)*32 + lane]; 32-bit
// index math throughout (the encoded matrix is < 2^31 words).
//
// Pads are not predicated away: code 0xFF is the record {+0.0, 0}, so a pad
// gathers the row's own x and adds +0.0 * x = +-0.  The sum starts at +0.0
// and a round-to-nearest sum that starts at +0 never becomes -0, so adding
// +-0 leaves every bit of it unchanged (for finite x): the CSR-order sum is
// reproduced exactly with 5 fewer instructions per entry (predicate, two
// selects, zeroing) on this issue-bound loop.
template <int OP>
__device__ __forceinline__ double row_sum_dict(const SellArgs& a, const DictParam<kFDict>& dp, int slice, int lane,
                                               int row) {
    const int W = a.words;
    const uint32_t* cp = a.code + (slice * W) * 32 + lane;
    double sum = 0.0;
    for (int w0 = 0; w0 < W; w0 += 2) {
        const uint32_t wa = __ldg(cp + w0 * 32);
        const uint32_t wb = w0 + 1 < W ? __ldg(cp + (w0 + 1) * 32) : 0xFFFFFFFFu;
        uint32_t e[8];
        double av[8], xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = ((j < 4 ? wa : wb) >> (8 * (j & 3))) & 0xFFu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int dc;
            dict_entry(dp, e[j], av[j], dc);
            xv[j] = xval<OP>(a, row + dc);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) sum = dadd(sum, dmul(av[j], xv[j]));
    }
    return sum;
}

// CODED row sum: one 32-bit word per entry, (column - row) in the high 24
// bits (signed) and a value code in the low 8 (SELL-32 slices of the row
// set's own widths, as PLAIN).  Pad word 0x000000FF = {+0.0, own row}: not
// predicated, bit-neutral for the same reason as the DICT pads.
template <int OP>
__device__ __forceinline__ double row_sum_coded(const SellArgs& a, const DictParam<kFCoded>& dp, int slice, int lane,
                                                int row) {
    const int beg = static_cast<int>(a.soff[slice]);
    const int width = (static_cast<int>(a.soff[slice + 1]) - beg) >> 5;
    const uint32_t* cp = a.code + beg + lane;
    double sum = 0.0;
    for (int k = 0; k < width; k += 8) {
        uint32_t w[8];
        double av[8], xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = k + j < width ? __ldg(cp + (k + j) * 32) : 0xFFu;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            av[j] = __longlong_as_double(static_cast<long long>(dp.e[w[j] & 0xFFu].x));
            xv[j] = xval<OP>(a, row + (static_cast<int32_t>(w[j]) >> 8));
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) sum = dadd(sum, dmul(av[j], xv[j]));
    }
    return sum;
}

template <int OP, int F>
__device__ __forceinline__ double row_sum(const SellArgs& a, const DictParam<F>& dp, int slice, int lane, int row) {
    if constexpr (F == kFDict)
        return row_sum_dict<OP>(a, dp, slice, lane, row);
    else if constexpr (F == kFCoded)
        return row_sum_coded<OP>(a, dp, slice, lane, row);
    else
        return row_sum_plain<OP>(a, slice, lane);
}

template <int OP, bool ROWS, int F>
__global__ void __launch_bounds__(kThreads) k_sell(SellArgs a, const __grid_constant__ DictParam<F> dp) {
    const int lane = threadIdx.x & 31;
    const int slice = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (slice >= a.nslices) return;
    const int sr = slice * 32 + lane;
    const bool valid = sr < a.nrows;
    const int row = !valid ? 0 : (ROWS ? a.rows[sr] : a.row0 + sr);
    // own-row operands first: their latency overlaps the gather chain
    double xi = 0.0, ri = 0.0, di = 1.0;
    if (valid) {
        if (OP == kJacobi) {
            ri = a.r[row];
            di = a.d[row];
        }
        if (OP == kResid) ri = a.r[row];
        if (OP == kJacobi) xi = a.x[row];
    }
    const double sum = row_sum<OP, F>(a, dp, slice, lane, row);
    if (!valid) return;
    if (OP == kSpmv) {
        a.y[row] = sum;
    } else if (OP == kResid) {
        a.y[row] = dsub(ri, sum);
    } else {
        a.y[row] = dadd(xi, ddiv(dmul(a.omega, dsub(ri, sum)), di));
    }
}

// v = A w with block partials of (w.r, w.v, w.q) (fixed order ->
// deterministic).  Launched with one warp per slice like the sweeps; the
// grid-stride loop only matters for capped grids.
template <int F, bool ROWS>
__global__ void __launch_bounds__(kThreads, 8) k_sell_spmv_dots(SellArgs a, const __grid_constant__ DictParam<F> dp) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    double sa = 0.0, sb = 0.0, sg = 0.0;
    for (int slice = blockIdx.x * kWarps + warp; slice < a.nslices; slice += gridDim.x * kWarps) {
        const int sr = slice * 32 + lane;
        const bool valid = sr < a.nrows;
        const int row = !valid ? 0 : (ROWS ? a.rows[sr] : a.row0 + sr);
        double wi = 0.0, rr = 0.0, qq = 0.0;
        if (valid) {
            wi = a.x[row];
            rr = a.r[row];
            qq = a.q[row];
        }
        const double sum = row_sum<kSpmv, F>(a, dp, slice, lane, row);
        if (valid) {
            a.y[row] = sum;
            sa = dadd(sa, dmul(wi, rr));
            sb = dadd(sb, dmul(wi, sum));
            sg = dadd(sg, dmul(wi, qq));
        }
    }
    for (int o = 16; o; o >>= 1) {
        sa = dadd(sa, __shfl_down_sync(0xffffffffu, sa, o));
        sb = dadd(sb, __shfl_down_sync(0xffffffffu, sb, o));
        sg = dadd(sg, __shfl_down_sync(0xffffffffu, sg, o));
    }
    __shared__ double red[3][kWarps];
    if (lane == 0) {
        red[0][warp] = sa;
        red[1][warp] = sb;
        red[2][warp] = sg;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double acc = 0.0;
        for (int i = 0; i < kWarps; ++i) acc = dadd(acc, red[threadIdx.x][i]);
        a.partials[blockIdx.x * 3 + threadIdx.x] = acc;
    }
}

#include "sell_sten.cuh"

// ------------------------------------------------------------------ PAT ---
//
// One thread per row: pid -> {first record, length} -> records {value,
// column - row} in CSR order.  Rows of a warp are consecutive, so on the
// interior of a stencil operator all lanes read the same records (L1
// broadcast) and run the same trip count; the row's l1 diagonal comes from
// the pattern (no per-row d stream).

#ifndef PB_PAT_BLOCKS
#define PB_PAT_BLOCKS 4
#endif
constexpr int kPatBlocks = PB_PAT_BLOCKS;  // resident blocks/SM the register budget targets

struct PatArgs {
    const uint8_t* pid;
    const ulonglong2* ptab;
    const int2* pmeta;
    const double* pdiag;
    int maxlen;
    int xlen;  // length of the gathered vector (owned + halo slots)
    const int32_t* rows;
    int row0;  // first row when the row set is a contiguous range (rows == nullptr)
    int64_t nrows;
    const double* x;
    double* y;
    const double* r;
    double omega;
    const double* q;
    double* partials;
};

// All record and gather loads are unconditional so they issue back to back
// before the first multiply: the table is padded with 8 records past its end
// and out-of-pattern gathers are clamped into x (their values are never
// accumulated -- the add itself is predicated, keeping the CSR-order sum exact).
// Empty asm statements that consume all eight values of a load batch: ptxas
// must issue the whole batch before them, so a batch costs one memory
// latency instead of eight (without them it interleaves each multiply with
// the next load to save registers, serialising the gathers).
__device__ __forceinline__ void batch_fence(const double (&v)[8]) {
    asm volatile("" ::"d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]), "d"(v[4]), "d"(v[5]), "d"(v[6]), "d"(v[7]));
}
__device__ __forceinline__ void batch_fence(const ulonglong2 (&v)[8]) {
    asm volatile("" ::"l"(v[0].y), "l"(v[1].y), "l"(v[2].y), "l"(v[3].y), "l"(v[4].y), "l"(v[5].y), "l"(v[6].y),
                 "l"(v[7].y));
}

__device__ __forceinline__ double pat_row_sum(const PatArgs& a, int row, int2 m) {
    double sum = 0.0;
    for (int k0 = 0; k0 < a.maxlen; k0 += 8) {
        ulonglong2 rec[8];
        double xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) rec[j] = __ldg(a.ptab + m.x + k0 + j);
        batch_fence(rec);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = min(max(row + static_cast<int>(rec[j].y), 0), a.xlen - 1);
            xv[j] = __ldg(a.x + c);
        }
        batch_fence(xv);
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (k0 + j < m.y) sum = dadd(sum, dmul(__longlong_as_double(static_cast<long long>(rec[j].x)), xv[j]));
    }
    return sum;
}

template <int OP, bool ROWS>
__global__ void __launch_bounds__(kThreads, kPatBlocks) k_pat(PatArgs a) {
    const int i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= a.nrows) return;
    const int row = ROWS ? a.rows[i] : a.row0 + i;
    const int p = a.pid[row];
    const int2 m = __ldg(a.pmeta + p);
    double xi = 0.0, ri = 0.0, di = 1.0;
    if (OP != kSpmv) ri = a.r[row];
    if (OP == kJacobi) {
        xi = a.x[row];
        di = __ldg(a.pdiag + p);
    }
    const double sum = pat_row_sum(a, row, m);
    if (OP == kSpmv)
        a.y[row] = sum;
    else if (OP == kResid)
        a.y[row] = dsub(ri, sum);
    else
        a.y[row] = dadd(xi, ddiv(dmul(a.omega, dsub(ri, sum)), di));
}

// v = A w + block partials of (w.r, w.v, w.q), grid-stride (fixed order).
template <bool ROWS>
__global__ void __launch_bounds__(kThreads) k_pat_spmv_dots(PatArgs a) {
    double sa = 0.0, sb = 0.0, sg = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < a.nrows;
         i += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int row = ROWS ? a.rows[i] : a.row0 + static_cast<int>(i);
        const int p = a.pid[row];
        const int2 m = __ldg(a.pmeta + p);
        const double wi = a.x[row], rr = a.r[row], qq = a.q[row];
        const double sum = pat_row_sum(a, row, m);
        a.y[row] = sum;
        sa = dadd(sa, dmul(wi, rr));
        sb = dadd(sb, dmul(wi, sum));
        sg = dadd(sg, dmul(wi, qq));
    }
    for (int o = 16; o; o >>= 1) {
        sa = dadd(sa, __shfl_down_sync(0xffffffffu, sa, o));
        sb = dadd(sb, __shfl_down_sync(0xffffffffu, sb, o));
        sg = dadd(sg, __shfl_down_sync(0xffffffffu, sg, o));
    }
    __shared__ double red[3][kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][warp] = sa;
        red[1][warp] = sb;
        red[2][warp] = sg;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double acc = 0.0;
        for (int k = 0; k < kWarps; ++k) acc = dadd(acc, red[threadIdx.x][k]);
        a.partials[blockIdx.x * 3 + threadIdx.x] = acc;
    }
}

// --- PAT building: hash every row's entry sequence, collect <= 255 patterns
// (representative = smallest row), then assign + verify exactly on device.

__device__ __forceinline__ ull mix64(ull h, ull v) {
    h ^= v + 0x9E3779B97F4A7C15ULL + (h << 6) + (h >> 2);
    h *= 0xBF58476D1CE4E5B9ULL;
    return h ^ (h >> 31);
}

__device__ ull row_hash(const int64_t* rp, const int32_t* col, const double* val, int64_t row) {
    ull h = mix64(0x243F6A8885A308D3ULL, static_cast<ull>(rp[row + 1] - rp[row]));
    for (int64_t t = rp[row]; t < rp[row + 1]; ++t) {
        h = mix64(h, static_cast<ull>(static_cast<int64_t>(col[t]) - row));
        h = mix64(h, static_cast<ull>(__double_as_longlong(val[t])));
    }
    return h | 1ULL;  // 0 marks an empty slot
}

__global__ void k_pat_insert(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const double* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                             ull* keys, unsigned long long* rep, unsigned* count, int* overflow) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    if (*reinterpret_cast<volatile int*>(overflow)) return;
    const int64_t row = rows ? rows[i] : i;
    const ull h = row_hash(rp, col, val, row);
    unsigned s = static_cast<unsigned>(h >> 20) & (kTableCap - 1);
    for (int probe = 0; probe < kTableCap; ++probe, s = (s + 1) & (kTableCap - 1)) {
        const ull old = atomicCAS(keys + s, 0ULL, h);
        if (old == 0ULL || old == h) {
            atomicMin(rep + s, static_cast<unsigned long long>(row));
            if (old == 0ULL && atomicAdd(count, 1u) >= static_cast<unsigned>(kDictMax)) atomicExch(overflow, 1);
            return;
        }
    }
    atomicExch(overflow, 1);
}

__global__ void k_pat_assign(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const double* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                             const ull* __restrict__ keys, const int* __restrict__ slot_pid,
                             const ulonglong2* __restrict__ ptab, const int2* __restrict__ pmeta,
                             const double* __restrict__ pdiag, const double* __restrict__ l1, uint8_t* __restrict__ pid,
                             int* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    const int64_t row = rows ? rows[i] : i;
    const ull h = row_hash(rp, col, val, row);
    unsigned s = static_cast<unsigned>(h >> 20) & (kTableCap - 1);
    int p = -1;
    for (int probe = 0; probe < kTableCap; ++probe, s = (s + 1) & (kTableCap - 1)) {
        if (keys[s] == h) {
            p = slot_pid[s];
            break;
        }
        if (keys[s] == 0ULL) break;
    }
    bool ok = p >= 0;
    if (ok) {
        const int2 m = pmeta[p];
        ok = m.y == rp[row + 1] - rp[row];
        for (int k = 0; ok && k < m.y; ++k) {
            const int64_t t = rp[row] + k;
            ok = ptab[m.x + k].x == static_cast<ull>(__double_as_longlong(val[t])) &&
                 static_cast<int64_t>(static_cast<long long>(ptab[m.x + k].y)) == static_cast<int64_t>(col[t]) - row;
        }
        ok = ok && __double_as_longlong(pdiag[p]) == __double_as_longlong(l1[row]);
    }
    if (!ok) {
        atomicExch(bad, 1);
        return;
    }
    pid[row] = static_cast<uint8_t>(p);
}

// ------------------------------------------------------------- building ---

__global__ void k_sell_width(const int64_t* __restrict__ rp, const int32_t* __restrict__ rows, int64_t nrows,
                             int64_t nslices, int64_t* __restrict__ width) {
    const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= nslices) return;
    const int64_t sr = s * 32 + lane;
    int len = 0;
    if (sr < nrows) {
        const int64_t row = rows ? rows[sr] : sr;
        len = static_cast<int>(rp[row + 1] - rp[row]);
    }
    for (int o = 16; o; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if (lane == 0) width[s] = 32LL * len;
}

__global__ void k_sell_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                            const int64_t* __restrict__ soff, int32_t* __restrict__ scol, double* __restrict__ sval) {
    const int64_t sr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sr >= nrows) return;
    const int64_t row = rows ? rows[sr] : sr;
    const int64_t base = soff[sr >> 5] + (sr & 31);
    const int64_t b = rp[row], e = rp[row + 1];
    for (int64_t t = b; t < e; ++t) {
        scol[base + (t - b) * 32] = col[t];
        sval[base + (t - b) * 32] = val[t];
    }
}

__global__ void k_fill_u32(uint32_t* __restrict__ p, int64_t n, uint32_t v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// CODED words: ((column - row) << 8) | value code; bad = a delta outside 24 bits.
__global__ void k_sell_fill_coded(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                  const uint8_t* __restrict__ vcode, const int32_t* __restrict__ rows, int64_t nrows,
                                  const int64_t* __restrict__ soff, uint32_t* __restrict__ code, int* bad) {
    const int64_t sr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sr >= nrows) return;
    const int64_t row = rows ? rows[sr] : sr;
    const int64_t base = soff[sr >> 5] + (sr & 31);
    const int64_t b = rp[row], e = rp[row + 1];
    for (int64_t t = b; t < e; ++t) {
        const int64_t d = static_cast<int64_t>(col[t]) - row;
        if (d < -(int64_t(1) << 23) || d >= (int64_t(1) << 23) || vcode[t] == 0xFF) {
            atomicExch(bad, 1);
            return;
        }
        code[base + (t - b) * 32] = (static_cast<uint32_t>(static_cast<int32_t>(d)) << 8) | vcode[t];
    }
}

__device__ __forceinline__ void ld_slot(const ull* p, ull& lo, ull& hi) {
    asm volatile(
        "{\n\t.reg .b128 v;\n\t"
        "ld.relaxed.gpu.global.b128 v, [%2];\n\t"
        "mov.b128 {%0, %1}, v;\n\t}"
        : "=l"(lo), "=l"(hi)
        : "l"(p)
        : "memory");
}

__device__ __forceinline__ bool cas_slot(ull* p, ull cmp_lo, ull cmp_hi, ull new_lo, ull new_hi) {
    ull old_lo, old_hi;
    asm volatile(
        "{\n\t.reg .b128 c, n, o;\n\t"
        "mov.b128 c, {%3, %4};\n\t"
        "mov.b128 n, {%5, %6};\n\t"
        "atom.relaxed.gpu.global.cas.b128 o, [%2], c, n;\n\t"
        "mov.b128 {%0, %1}, o;\n\t}"
        : "=l"(old_lo), "=l"(old_hi)
        : "l"(p), "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi)
        : "memory");
    return old_lo == cmp_lo && old_hi == cmp_hi;
}

__device__ __forceinline__ unsigned slot_hash(ull lo, ull hi) {
    ull h = lo * 0x9E3779B97F4A7C15ULL ^ (hi + 0x632BE59BD9B4E019ULL) * 0xC2B2AE3D27D4EB4FULL;
    return static_cast<unsigned>(h >> 40) & (kTableCap - 1);
}

// Find (or insert) key (delta, value bits) in the open-addressing table;
// returns the slot, or -1 on overflow / absence.  Slots go empty -> key once
// (128-bit CAS) and are read with single-copy-atomic 128-bit loads.
__device__ int table_find(ull* table, ull lo, ull hi, bool insert, unsigned* count, int* overflow) {
    unsigned h = slot_hash(lo, hi);
    for (int probe = 0; probe < kTableCap; ++probe, h = (h + 1) & (kTableCap - 1)) {
        ull slo, shi;
        ld_slot(table + 2 * h, slo, shi);
        if (slo == lo && shi == hi) return static_cast<int>(h);
        if (slo == kEmptyLo && shi == 0) {
            if (!insert) return -1;
            if (*reinterpret_cast<volatile int*>(overflow)) return -1;
            if (cas_slot(table + 2 * h, kEmptyLo, 0, lo, hi)) {
                if (atomicAdd(count, 1u) >= static_cast<unsigned>(kDictMax)) atomicExch(overflow, 1);
                return static_cast<int>(h);
            }
            ld_slot(table + 2 * h, slo, shi);  // lost the race: the winner's key is there now
            if (slo == lo && shi == hi) return static_cast<int>(h);
        }
    }
    if (overflow) atomicExch(overflow, 1);
    return -1;
}

__global__ void k_table_init(ull* table) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < kTableCap) {
        table[2 * i] = kEmptyLo;
        table[2 * i + 1] = 0;
    }
}

__global__ void k_dict_insert(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const double* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                              ull* table, unsigned* count, int* overflow, unsigned* maxlen) {
    const int64_t sr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sr >= nrows) return;
    const int64_t row = rows ? rows[sr] : sr;
    atomicMax(maxlen, static_cast<unsigned>(rp[row + 1] - rp[row]));
    for (int64_t t = rp[row]; t < rp[row + 1]; ++t) {
        if (*reinterpret_cast<volatile int*>(overflow)) return;
        const ull lo = static_cast<ull>(static_cast<int64_t>(col[t]) - row);
        const ull hi = static_cast<ull>(__double_as_longlong(val[t]));
        if (table_find(table, lo, hi, true, count, overflow) < 0) return;
    }
}

__global__ void k_sell_fill_dict(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const double* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                                 int W, ull* table, const int* __restrict__ slot_code, uint32_t* __restrict__ code,
                                 int* bad) {
    const int64_t sr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (sr >= nrows) return;
    const int64_t row = rows ? rows[sr] : sr;
    const int64_t base = (sr >> 5) * W * 32 + (sr & 31);
    const int64_t b = rp[row], e = rp[row + 1];
    for (int w = 0; w < W; ++w) {
        uint32_t word = 0xFFFFFFFFu;
        for (int j = 0; j < 4; ++j) {
            const int64_t t = b + 4 * w + j;
            if (t >= e) break;
            const ull lo = static_cast<ull>(static_cast<int64_t>(col[t]) - row);
            const ull hi = static_cast<ull>(__double_as_longlong(val[t]));
            const int slot = table_find(table, lo, hi, false, nullptr, nullptr);
            const int c = slot < 0 ? -1 : slot_code[slot];
            if (c < 0) {
                atomicExch(bad, 1);
                continue;
            }
            word = (word & ~(0xFFu << (8 * j))) | (static_cast<uint32_t>(c) << (8 * j));
        }
        code[base + static_cast<int64_t>(w) * 32] = word;
    }
}

// Generic value codes (transfer operators): key (0, value bits).
__global__ void k_val_insert(const double* __restrict__ v, int64_t n, ull* table, unsigned* count, int* overflow) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || *reinterpret_cast<volatile int*>(overflow)) return;
    table_find(table, 0, static_cast<ull>(__double_as_longlong(v[i])), true, count, overflow);
}

__global__ void k_val_fill(const double* __restrict__ v, int64_t n, ull* table, const int* __restrict__ slot_code,
                           uint8_t* __restrict__ code, int* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int slot = table_find(table, 0, static_cast<ull>(__double_as_longlong(v[i])), false, nullptr, nullptr);
    const int c = slot < 0 ? -1 : slot_code[slot];
    if (c < 0) {
        atomicExch(bad, 1);
        return;
    }
    code[i] = static_cast<uint8_t>(c);
}

template <typename F>
void cub_call(F&& f, cudaStream_t s) {
    size_t bytes = 0;
    PB_CUDA(f(nullptr, bytes));
    DBuf<uint8_t> tmp(bytes ? bytes : 1, s);
    PB_CUDA(f(tmp.get(), bytes));
}

bool try_dict(const DevMatrix& M, const int32_t* rows, Sell& S, const double* l1, cudaStream_t s) {
    if (S.nrows == 0) return false;
    if (S.nslices * 32 >= (int64_t(1) << 31) / 8) return false;  // 32-bit code index range
    DBuf<ull> table(2 * kTableCap, s);
    DBuf<unsigned> cnt(2, s);  // [0] distinct pairs, [1] longest row
    DBuf<int> flags(2, s);
    cnt.zero(s);
    flags.zero(s);
    k_table_init<<<kTableCap / 256, 256, 0, s>>>(table.get());
    k_dict_insert<<<blocks_for(S.nrows, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), M.val.get(), rows, S.nrows,
                                                            table.get(), cnt.get(), flags.get(), cnt.get() + 1);
    PB_CHECK_LAUNCH();
    int over = 0;
    unsigned hc[2] = {0, 0};
    PB_CUDA(cudaMemcpyAsync(&over, flags.get(), 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaMemcpyAsync(hc, cnt.get(), 8, cudaMemcpyDeviceToHost, s));
    std::vector<ull> h(2 * kTableCap);
    PB_CUDA(cudaMemcpyAsync(h.data(), table.get(), 16 * kTableCap, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (over) return false;
    // deterministic code order: ascending (delta, value bits)
    std::vector<std::pair<std::pair<int64_t, int64_t>, int>> keys;
    for (int i = 0; i < kTableCap; ++i)
        if (!(h[2 * i] == kEmptyLo && h[2 * i + 1] == 0))
            keys.push_back({{static_cast<int64_t>(h[2 * i]), static_cast<int64_t>(h[2 * i + 1])}, i});
    if (keys.empty() || keys.size() > static_cast<size_t>(kDictMax)) return false;
    std::sort(keys.begin(), keys.end());
    std::vector<int> slot_code(kTableCap, -1);
    std::vector<int32_t> dcol(keys.size());
    std::vector<double> dval(keys.size());
    for (size_t c = 0; c < keys.size(); ++c) {
        slot_code[keys[c].second] = static_cast<int>(c);
        dcol[c] = static_cast<int32_t>(keys[c].first.first);
        const int64_t bitsv = keys[c].first.second;
        std::memcpy(&dval[c], &bitsv, 8);
    }
    S.ndict = static_cast<int>(keys.size());
    S.words = static_cast<int>((hc[1] + 3) / 4);
    if (S.words == 0) S.words = 1;
    std::vector<ulonglong2> rec(256, make_ulonglong2(0ULL, 0ULL));  // slot 255 = pad
    for (size_t c = 0; c < keys.size(); ++c) {
        ull vb;
        std::memcpy(&vb, &dval[c], 8);
        rec[c] = make_ulonglong2(vb, static_cast<ull>(static_cast<int64_t>(dcol[c])));
    }
    S.dict.alloc(256, s);
    PB_CUDA(cudaMemcpyAsync(S.dict.get(), rec.data(), 16 * 256, cudaMemcpyHostToDevice, s));
    S.hdict = rec;  // host copy: passed by value to the kernels (constant bank)
    DBuf<int> dsc(kTableCap, s);
    PB_CUDA(cudaMemcpyAsync(dsc.get(), slot_code.data(), 4 * kTableCap, cudaMemcpyHostToDevice, s));
    S.padded_nnz = S.nslices * 32 * S.words;  // in words
    S.code.alloc(static_cast<size_t>(S.padded_nnz), s);
    PB_CUDA(cudaMemsetAsync(S.code.get(), 0xff, 4 * S.padded_nnz, s));
    k_sell_fill_dict<<<blocks_for(S.nrows, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), M.val.get(), rows, S.nrows,
                                                              S.words, table.get(), dsc.get(), S.code.get(),
                                                              flags.get() + 1);
    PB_CHECK_LAUNCH();
    int bad = 0;
    PB_CUDA(cudaMemcpyAsync(&bad, flags.get() + 1, 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (bad) fail(PAIRAMG_INTERNAL, "sell: dictionary encoding lost an entry");
    S.format = Sell::kDict;
    return true;
}

__global__ void k_max_len(const int64_t* __restrict__ rp, const int32_t* __restrict__ rows, int64_t nrows,
                          unsigned long long* mx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    const int64_t row = rows ? rows[i] : i;
    atomicMax(mx, static_cast<unsigned long long>(rp[row + 1] - rp[row]));
}

void max_row_len(const DevMatrix& M, const int32_t* rows, int64_t nrows, int64_t* d_out, cudaStream_t s) {
    if (!nrows) return;
    k_max_len<<<blocks_for(nrows, 256), 256, 0, s>>>(M.rp.get(), rows, nrows,
                                                     reinterpret_cast<unsigned long long*>(d_out));
    PB_CHECK_LAUNCH();
}

void reset_pat(Sell& S) {
    S.pid.reset();
    S.ptab.reset();
    S.pmeta.reset();
    S.pdiag.reset();
    S.pinv.reset();
    S.npat = 0;
    S.maxlen = 0;
    S.hptab.clear();
    S.hpmeta.clear();
    S.hpdiag.clear();
    S.format = Sell::kPlain;
}

// PAT -> STEN: the main pattern is a common supersequence of all row patterns
// (records compared bitwise), built from the longest pattern by merging in
// every pattern that is not already a subsequence (shortest common
// supersequence of the two, LCS dynamic programme); <= kStenMax records.
// Slab-partition boundary rows, whose halo neighbour sits at a different
// local offset on each face, nest this way.
bool try_sten(Sell& S, int max_len = kStenMax) {
    if (S.npat < 1) return false;
    auto eq = [](const ulonglong2& a, const ulonglong2& b) { return a.x == b.x && a.y == b.y; };
    auto pat = [&](int p) {
        return std::vector<ulonglong2>(S.hptab.begin() + S.hpmeta[p].x, S.hptab.begin() + S.hpmeta[p].x + S.hpmeta[p].y);
    };
    auto subseq = [&](const std::vector<ulonglong2>& P, const std::vector<ulonglong2>& M, unsigned long long* present) {
        size_t j = 0;
        unsigned long long pr = 0;
        for (const auto& r : P) {
            while (j < M.size() && !eq(M[j], r)) ++j;
            if (j == M.size()) return false;
            pr |= 1ull << j;
            ++j;
        }
        if (present) *present = pr;
        return true;
    };
    std::vector<int> order(S.npat);
    for (int p = 0; p < S.npat; ++p) order[p] = p;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return S.hpmeta[a].y > S.hpmeta[b].y; });
    std::vector<ulonglong2> M = pat(order[0]);
    for (int p : order) {
        const std::vector<ulonglong2> P = pat(p);
        if (subseq(P, M, nullptr)) continue;
        const size_t a = M.size(), b = P.size();
        std::vector<std::vector<int>> lcs(a + 1, std::vector<int>(b + 1, 0));
        for (size_t i = a; i-- > 0;)
            for (size_t j = b; j-- > 0;)
                lcs[i][j] = eq(M[i], P[j]) ? lcs[i + 1][j + 1] + 1 : std::max(lcs[i + 1][j], lcs[i][j + 1]);
        std::vector<ulonglong2> U;
        size_t i = 0, j = 0;
        while (i < a && j < b) {
            if (eq(M[i], P[j])) {
                U.push_back(M[i++]);
                ++j;
            } else if (lcs[i + 1][j] >= lcs[i][j + 1]) {
                U.push_back(M[i++]);
            } else {
                U.push_back(P[j++]);
            }
        }
        while (i < a) U.push_back(M[i++]);
        while (j < b) U.push_back(P[j++]);
        if (U.size() > static_cast<size_t>(max_len)) return false;
        M.swap(U);
    }
    const int L = static_cast<int>(M.size());
    if (L < 1 || L > max_len) return false;
    const ulonglong2* mr = M.data();
    std::vector<unsigned long long> mask(S.npat, 0ull);
    for (int p = 0; p < S.npat; ++p) {
        unsigned long long present = 0;
        if (!subseq(pat(p), M, &present)) return false;
        mask[p] = ~present & (L == 64 ? ~0ull : ((1ull << L) - 1ull));
    }
    S.sten_L = L;
    S.sten_off.assign(L, 0);
    S.sten_val.assign(L, 0.0);
    int64_t omin = 0, omax = 0;
    for (int k = 0; k < L; ++k) {
        const int64_t o = static_cast<int64_t>(mr[k].y);
        S.sten_off[k] = static_cast<int>(o);
        std::memcpy(&S.sten_val[k], &mr[k].x, 8);
        omin = std::min(omin, o);
        omax = std::max(omax, o);
    }
    S.sten_offmin = static_cast<int>(omin);
    S.sten_offmax = static_cast<int>(omax);
    S.sten_mask64 = mask;
    S.sten_mask.assign(mask.size(), 0u);
    for (size_t p = 0; p < mask.size(); ++p) S.sten_mask[p] = static_cast<uint32_t>(mask[p]);  // used iff L <= 32
    S.ptab.reset();
    S.pmeta.reset();  // pdiag stays: the FCG update reads it (fused zero-start)
    S.format = Sell::kSten;
    return true;
}

bool try_pattern(const DevMatrix& M, const int32_t* rows, Sell& S, const double* l1, cudaStream_t s) {
    if (S.nrows == 0 || !l1) return false;
    DBuf<ull> keys(kTableCap, s), rep(kTableCap, s);
    DBuf<unsigned> cnt(1, s);
    DBuf<int> flags(2, s);
    keys.zero(s);
    cnt.zero(s);
    flags.zero(s);
    PB_CUDA(cudaMemsetAsync(rep.get(), 0xff, 8 * kTableCap, s));
    k_pat_insert<<<blocks_for(S.nrows, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), M.val.get(), rows, S.nrows,
                                                           keys.get(), rep.get(), cnt.get(), flags.get());
    PB_CHECK_LAUNCH();
    int over = 0;
    std::vector<ull> hk(kTableCap), hr(kTableCap);
    PB_CUDA(cudaMemcpyAsync(&over, flags.get(), 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaMemcpyAsync(hk.data(), keys.get(), 8 * kTableCap, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaMemcpyAsync(hr.data(), rep.get(), 8 * kTableCap, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (over) return false;
    std::vector<std::pair<ull, int>> pats;  // (representative row, slot)
    for (int i = 0; i < kTableCap; ++i)
        if (hk[i]) pats.push_back({hr[i], i});
    if (pats.empty() || pats.size() > static_cast<size_t>(kDictMax)) return false;
    std::sort(pats.begin(), pats.end());
    std::vector<int> slot_pid(kTableCap, -1);
    std::vector<ulonglong2> rec;
    std::vector<int2> meta;
    std::vector<double> pd;
    int maxlen = 0;
    for (size_t p = 0; p < pats.size(); ++p) {
        const int64_t row = static_cast<int64_t>(pats[p].first);
        slot_pid[pats[p].second] = static_cast<int>(p);
        int64_t b_e[2];
        PB_CUDA(cudaMemcpyAsync(b_e, M.rp.get() + row, 16, cudaMemcpyDeviceToHost, s));
        PB_CUDA(cudaStreamSynchronize(s));
        const int64_t len = b_e[1] - b_e[0];
        std::vector<int32_t> c(static_cast<size_t>(len));
        std::vector<double> v(static_cast<size_t>(len));
        if (len) {
            PB_CUDA(cudaMemcpyAsync(c.data(), M.col.get() + b_e[0], 4 * len, cudaMemcpyDeviceToHost, s));
            PB_CUDA(cudaMemcpyAsync(v.data(), M.val.get() + b_e[0], 8 * len, cudaMemcpyDeviceToHost, s));
            PB_CUDA(cudaStreamSynchronize(s));
        }
        meta.push_back(make_int2(static_cast<int>(rec.size()), static_cast<int>(len)));
        // l1 diagonal of the pattern in CSR order (cycle.cpp:20-27): a_ii + sum |a_ij|
        double acc = 0.0;
        for (int64_t k = 0; k < len; ++k) {
            const int64_t delta = static_cast<int64_t>(c[k]) - row;
            ull vb;
            std::memcpy(&vb, &v[k], 8);
            rec.push_back(make_ulonglong2(vb, static_cast<ull>(delta)));
            acc += delta == 0 ? v[k] : std::fabs(v[k]);
        }
        pd.push_back(acc);
        maxlen = std::max<int>(maxlen, static_cast<int>(len));
    }
    S.npat = static_cast<int>(pats.size());
    S.maxlen = maxlen;
    S.hptab = rec;
    S.hpmeta = meta;
    S.hpdiag = pd;
    rec.resize(rec.size() + static_cast<size_t>((maxlen + 7) / 8) * 8, make_ulonglong2(0ULL, 0ULL));  // load padding
    S.ptab.alloc(std::max<size_t>(rec.size(), 1), s);
    S.pmeta.alloc(meta.size(), s);
    S.pdiag.alloc(pd.size(), s);
    if (!rec.empty()) PB_CUDA(cudaMemcpyAsync(S.ptab.get(), rec.data(), 16 * rec.size(), cudaMemcpyHostToDevice, s));
    PB_CUDA(cudaMemcpyAsync(S.pmeta.get(), meta.data(), 8 * meta.size(), cudaMemcpyHostToDevice, s));
    PB_CUDA(cudaMemcpyAsync(S.pdiag.get(), pd.data(), 8 * pd.size(), cudaMemcpyHostToDevice, s));
    {
        std::vector<double> inv(pd.size());
        for (size_t i = 0; i < pd.size(); ++i) inv[i] = fast_div() && pd[i] != 0.0 ? 1.0 / pd[i] : 0.0;
        S.pinv.alloc(inv.size(), s);
        PB_CUDA(cudaMemcpyAsync(S.pinv.get(), inv.data(), 8 * inv.size(), cudaMemcpyHostToDevice, s));
        PB_CUDA(cudaStreamSynchronize(s));  // inv is a host temporary
    }
    DBuf<int> dsp(kTableCap, s);
    PB_CUDA(cudaMemcpyAsync(dsp.get(), slot_pid.data(), 4 * kTableCap, cudaMemcpyHostToDevice, s));
    S.pid.alloc(static_cast<size_t>(M.n), s);
    k_pat_assign<<<blocks_for(S.nrows, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), M.val.get(), rows, S.nrows,
                                                           keys.get(), dsp.get(), S.ptab.get(), S.pmeta.get(),
                                                           S.pdiag.get(), l1, S.pid.get(), flags.get() + 1);
    PB_CHECK_LAUNCH();
    int bad = 0;
    PB_CUDA(cudaMemcpyAsync(&bad, flags.get() + 1, 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (bad) {  // hash collision or l1 mismatch: keep an exact format instead
        reset_pat(S);
        return false;
    }
    S.format = Sell::kPat;
    return true;
}

StenArgs sten_args_of(const Sell& S, int block_rows = 256) {
    StenArgs a{};
    a.pid = S.pid.get();
    a.rows = S.rows.empty() ? nullptr : S.rows.get();
    a.row0 = static_cast<int>(S.row0);
    a.nrows = static_cast<int>(S.nrows);
    a.xlen = static_cast<int>(S.xlen);
    a.L = S.sten_L;
    // blocks whose rows r all satisfy r + offmin >= 0 and r + offmax < xlen
    // (first and last row grow with the block index: both tests are monotone)
    const int64_t B = block_rows, nb = (S.nrows + B - 1) / B;
    int64_t lo = 0, hi = 0;
    if (S.rows.empty() && nb > 0) {
        auto last = [&](int64_t b) { return S.row0 + std::min<int64_t>(B * b + B - 1, S.nrows - 1); };
        while (lo < nb && S.row0 + B * lo + S.sten_offmin < 0) ++lo;
        hi = nb;
        while (hi > lo && last(hi - 1) + S.sten_offmax > S.xlen - 1) --hi;
    }
    a.safe_lo = static_cast<int>(lo);
    a.safe_hi = static_cast<int>(hi);
    a.nblk = static_cast<int>((S.nrows + block_rows - 1) / block_rows);
    a.pf_blocks = 16 * kSmCount * 256 / block_rows;
    a.offmax = S.sten_offmax;
    return a;
}

// The fixed-length kernels take the row's own x from record L/2.
bool sten_center(const Sell& S) { return S.sten_L > 0 && S.sten_off[static_cast<size_t>(S.sten_L / 2)] == 0; }

// Every main record but the centre (L/2, the fixed-length kernels' diagonal)
// is exactly -1.0: the row sums subtract instead of multiplying (bitwise equal).
int sten_neg1(const Sell& S) {
    if (S.sten_L <= 0) return 0;
    for (int k = 0; k < S.sten_L; ++k)
        if (k != S.sten_L / 2 && S.sten_val[k] != -1.0) return 0;
    return 1;
}

StenParam sten_param(const Sell& S) {
    StenParam p{};
    for (int k = 0; k < S.sten_L; ++k) {
        p.off[k] = S.sten_off[k];
        p.val[k] = S.sten_val[k];
    }
    for (int q = 0; q < 256; ++q) {
        p.pmask[q] = q < S.npat ? S.sten_mask[q] : 0u;
        p.pdiag[q] = q < S.npat ? S.hpdiag[q] : 1.0;
        p.pinv[q] = fast_div() ? 1.0 / p.pdiag[q] : 0.0;
    }
    p.neg1 = sten_neg1(S);
    return p;
}

StenParamW sten_param_w(const Sell& S) {
    StenParamW p{};
    for (int k = 0; k < S.sten_L; ++k) {
        p.off[k] = S.sten_off[k];
        p.val[k] = S.sten_val[k];
    }
    for (int q = 0; q < 256; ++q) {
        p.pmask[q] = q < S.npat ? S.sten_mask64[q] : 0ull;
        p.pdiag[q] = q < S.npat ? S.hpdiag[q] : 1.0;
        p.pinv[q] = fast_div() ? 1.0 / p.pdiag[q] : 0.0;
    }
    p.neg1 = sten_neg1(S);
    return p;
}

// Two rows per thread for the 7-record main pattern (k_sten2): +10% bandwidth.
// 27 records: only the SpMV+dots kernel gains (122 vs 132 us; sweeps lose).
bool sten_rpt2(const Sell& S, bool dots = false) {
    if (!sten_center(S)) return false;
    return S.sten_L == 7 || (S.sten_L == 27 && dots);
}

inline int capped(int nblk, int cap) { return cap > 0 ? std::min(nblk, cap) : nblk; }

// The 27-record main pattern as the full 3x3x3 box (record 9(dk+1) + 3(dj+1)
// + (di+1) at offset di + nx dj + nxy dk) on contiguous rows: the marching
// kernels apply (sell_sten.cuh).  Fills the geometry of the row set.
bool sten_march(const Sell& S, MarchGeom* out = nullptr) {
    if (S.sten_L != 27 || !S.rows.empty() || !sten_center(S) || S.nrows == 0) return false;
    const auto& o = S.sten_off;
    const int nx = o[16] - o[13], nxy = o[22] - o[13];
    if (nx < 2 || nxy < 2 * nx || nxy % nx) return false;
    for (int dk = -1; dk <= 1; ++dk)
        for (int dj = -1; dj <= 1; ++dj)
            for (int di = -1; di <= 1; ++di)
                if (o[static_cast<size_t>(9 * (dk + 1) + 3 * (dj + 1) + di + 1)] != di + nx * dj + nxy * dk) return false;
    MarchGeom g{};
    g.nx = nx;
    g.nxy = nxy;
    g.ny = nxy / nx;
    g.tiles_x = (nx + kMarchTX - 1) / kMarchTX;
    g.tiles_y = (g.ny + kMarchTY - 1) / kMarchTY;
    g.k0 = static_cast<int>(S.row0 / nxy);
    g.nk = static_cast<int>((S.row0 + S.nrows - 1) / nxy) - g.k0 + 1;
    // planes per CTA: about two waves of 4 CTAs per SM (measured at 192^3:
    // 2 waves 72 us per sweep, 1 wave 83, 4 waves 77, 8 waves 84; the two
    // halo planes per chunk are the re-read cost); small levels keep k_sten
    const int64_t cols = int64_t(g.tiles_x) * g.tiles_y;
    g.kz = static_cast<int>(std::min<int64_t>(32, cols * g.nk / (int64_t(kMarchWaves) * kMarchMinBlocks * kSmCount)));
    if (g.kz < 4) return false;
    g.chunks = (g.nk + g.kz - 1) / g.kz;
    if (out) *out = g;
    return true;
}

int march_grid(const MarchGeom& g) { return g.tiles_x * g.tiles_y * g.chunks; }

template <int OP, bool ROWS>
void launch_sten(const Sell& S, const StenArgs& a0, int cap, cudaStream_t s) {
    const StenParam p = sten_param(S);
    MarchGeom g;
    if (!ROWS && cap == 0 && sten_march(S, &g)) {
        launch_k<2>(k_sten_march<OP>, march_grid(g), 256, 0, s, a0, p, g);
        return;
    }
    if (sten_rpt2(S)) {
        StenArgs a = sten_args_of(S, 512);
        a.x = a0.x;
        a.y = a0.y;
        a.r = a0.r;
        a.omega = a0.omega;
        const int grid = capped(a.nblk, cap);
        const bool gs = grid < a.nblk;
        if (S.sten_L == 7)
            launch_k<2>(gs ? k_sten2<OP, ROWS, 7, true> : k_sten2<OP, ROWS, 7, false>, grid, 256, 0, s, a, p);
        else
            launch_k<2>(gs ? k_sten2<OP, ROWS, 27, true> : k_sten2<OP, ROWS, 27, false>, grid, 256, 0, s, a, p);
        return;
    }
    const StenArgs& a = a0;
    const int grid = capped(a.nblk, cap);
    const bool gs = grid < a.nblk;
    if (S.sten_L == 7 && sten_center(S))
        launch_k<2>(gs ? k_sten<OP, ROWS, 7, true> : k_sten<OP, ROWS, 7, false>, grid, 256, 0, s, a, p);
    else if (S.sten_L == 27 && sten_center(S))
        launch_k<2>(gs ? k_sten<OP, ROWS, 27, true> : k_sten<OP, ROWS, 27, false>, grid, 256, 0, s, a, p);
    else
        launch_k<2>(gs ? k_sten<OP, ROWS, 0, true> : k_sten<OP, ROWS, 0, false>, grid, 256, 0, s, a, p);
}

template <bool ROWS>
int launch_sten_dots(const Sell& S, const StenArgs& a0, int cap, cudaStream_t s) {
    const StenParam p = sten_param(S);
    MarchGeom g;
    if (!ROWS && cap == 0 && sten_march(S, &g)) {
        launch_k<2>(k_sten_march_dots, march_grid(g), 256, 0, s, a0, p, g);
        return march_grid(g);
    }
    if (sten_rpt2(S, true)) {
        StenArgs a = sten_args_of(S, 512);
        a.x = a0.x;
        a.y = a0.y;
        a.r = a0.r;
        a.q = a0.q;
        a.partials = a0.partials;
        const int grid = capped(a.nblk, cap);
        const bool gs = grid < a.nblk;
        if (S.sten_L == 7)
            launch_k<2>(gs ? k_sten2_dots<ROWS, 7, true> : k_sten2_dots<ROWS, 7, false>, grid, 256, 0, s, a, p);
        else
            launch_k<2>(gs ? k_sten2_dots<ROWS, 27, true> : k_sten2_dots<ROWS, 27, false>, grid, 256, 0, s, a, p);
        return gs ? grid : 8 * grid;  // partial triples: per warp unless grid-striding
    }
    const StenArgs& a = a0;
    const int grid = capped(a.nblk, cap);
    const bool gs = grid < a.nblk;
    if (S.sten_L == 7 && sten_center(S))
        launch_k<2>(gs ? k_sten_dots<ROWS, 7, true> : k_sten_dots<ROWS, 7, false>, grid, 256, 0, s, a, p);
    else if (S.sten_L == 27 && sten_center(S))
        launch_k<2>(gs ? k_sten_dots<ROWS, 27, true> : k_sten_dots<ROWS, 27, false>, grid, 256, 0, s, a, p);
    else
        launch_k<2>(gs ? k_sten_dots<ROWS, 0, true> : k_sten_dots<ROWS, 0, false>, grid, 256, 0, s, a, p);
    return grid;
}

PatArgs pat_args_of(const Sell& S) {
    PatArgs a{};
    a.pid = S.pid.get();
    a.ptab = S.ptab.get();
    a.pmeta = S.pmeta.get();
    a.pdiag = S.pdiag.get();
    a.maxlen = S.maxlen;
    a.xlen = static_cast<int>(S.xlen);
    a.rows = S.rows.empty() ? nullptr : S.rows.get();
    a.row0 = static_cast<int>(S.row0);
    a.nrows = S.nrows;
    return a;
}

SellArgs args_of(const Sell& S) {
    SellArgs a{};
    a.soff = S.slice_off.get();
    a.col = S.col.get();
    a.val = S.val.get();
    a.code = S.code.get();
    a.words = S.words;
    a.dict = S.dict.get();
    a.rows = S.rows.empty() ? nullptr : S.rows.get();
    a.row0 = static_cast<int>(S.row0);
    a.nslices = S.nslices;
    a.nrows = S.nrows;
    return a;
}

template <int F = kFDict>
DictParam<F> dict_param(const Sell& S) {
    DictParam<F> dp;
    for (int i = 0; i < 256; ++i) dp.e[i] = i < static_cast<int>(S.hdict.size()) ? S.hdict[i] : make_ulonglong2(0ULL, 0ULL);
    return dp;
}
DictParam<kFCoded> coded_param(const Sell& S) { return dict_param<kFCoded>(S); }

template <int OP>
void launch_op(const Sell& S, const SellArgs& a, cudaStream_t s) {
    const int grid = blocks_for(S.nslices, kWarps);
    const bool rows = a.rows != nullptr;
    if (S.format == Sell::kDict) {
        const DictParam<kFDict> dp = dict_param(S);
        if (rows)
            k_sell<OP, true, kFDict><<<grid, kThreads, 0, s>>>(a, dp);
        else
            k_sell<OP, false, kFDict><<<grid, kThreads, 0, s>>>(a, dp);
    } else if (S.format == Sell::kCoded) {
        const DictParam<kFCoded> dp = coded_param(S);
        if (rows)
            k_sell<OP, true, kFCoded><<<grid, kThreads, 0, s>>>(a, dp);
        else
            k_sell<OP, false, kFCoded><<<grid, kThreads, 0, s>>>(a, dp);
    } else {
        const DictParam<kFPlain> dp{0};
        if (rows)
            k_sell<OP, true, kFPlain><<<grid, kThreads, 0, s>>>(a, dp);
        else
            k_sell<OP, false, kFPlain><<<grid, kThreads, 0, s>>>(a, dp);
    }
    PB_CHECK_LAUNCH();
}

}  // namespace

bool build_value_codes(const double* v, int64_t n, DBuf<uint8_t>& code, std::vector<double>& table, cudaStream_t s) {
    code.reset();
    table.clear();
    if (n <= 0) return false;
    DBuf<ull> tab(2 * kTableCap, s);
    DBuf<unsigned> cnt(1, s);
    DBuf<int> flags(2, s);
    cnt.zero(s);
    flags.zero(s);
    k_table_init<<<kTableCap / 256, 256, 0, s>>>(tab.get());
    k_val_insert<<<blocks_for(n, 256), 256, 0, s>>>(v, n, tab.get(), cnt.get(), flags.get());
    PB_CHECK_LAUNCH();
    int over = 0;
    std::vector<ull> h(2 * kTableCap);
    PB_CUDA(cudaMemcpyAsync(&over, flags.get(), 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaMemcpyAsync(h.data(), tab.get(), 16 * kTableCap, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (over) return false;
    std::vector<std::pair<ull, int>> vals;
    for (int i = 0; i < kTableCap; ++i)
        if (!(h[2 * i] == kEmptyLo && h[2 * i + 1] == 0)) vals.push_back({h[2 * i + 1], i});
    if (vals.empty() || vals.size() > 256) return false;
    std::sort(vals.begin(), vals.end());
    std::vector<int> slot_code(kTableCap, -1);
    table.assign(vals.size(), 0.0);
    for (size_t c = 0; c < vals.size(); ++c) {
        slot_code[vals[c].second] = static_cast<int>(c);
        std::memcpy(&table[c], &vals[c].first, 8);
    }
    DBuf<int> dsc(kTableCap, s);
    PB_CUDA(cudaMemcpyAsync(dsc.get(), slot_code.data(), 4 * kTableCap, cudaMemcpyHostToDevice, s));
    code.alloc(static_cast<size_t>(n), s);
    k_val_fill<<<blocks_for(n, 256), 256, 0, s>>>(v, n, tab.get(), dsc.get(), code.get(), flags.get() + 1);
    PB_CHECK_LAUNCH();
    int bad = 0;
    PB_CUDA(cudaMemcpyAsync(&bad, flags.get() + 1, 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (bad) {
        code.reset();
        table.clear();
        return false;
    }
    return true;
}

namespace {

void sell_prologue(const DevMatrix& M, const int32_t* rows, int64_t nrows, Sell& S, cudaStream_t s) {
    S = Sell();
    S.nrows = nrows;
    S.nslices = (nrows + 31) / 32;
    S.xlen = M.n + M.halo.n_halo;
    if (S.nslices * 32 >= (int64_t(1) << 31))
        fail(PAIRAMG_INVALID_ARGUMENT, "sell: more than 2^31 rows per rank");
    if (rows && nrows) {
        // An ascending row set that is one contiguous range (the interior of a
        // slab partition) is addressed by offset: no row-id load per row.
        int32_t ends[2] = {0, 0};
        PB_CUDA(cudaMemcpyAsync(&ends[0], rows, 4, cudaMemcpyDeviceToHost, s));
        PB_CUDA(cudaMemcpyAsync(&ends[1], rows + nrows - 1, 4, cudaMemcpyDeviceToHost, s));
        PB_CUDA(cudaStreamSynchronize(s));
        if (static_cast<int64_t>(ends[1]) - ends[0] == nrows - 1) {
            S.row0 = ends[0];
        } else {
            S.rows.alloc(static_cast<size_t>(nrows), s);
            PB_CUDA(cudaMemcpyAsync(S.rows.get(), rows, 4 * nrows, cudaMemcpyDeviceToDevice, s));
        }
    }
}

// SELL-32 slice offsets (elements, multiples of 32) from the rows' lengths.
void slice_widths(const DevMatrix& M, const int32_t* rows, Sell& S, cudaStream_t s) {
    S.slice_off.alloc(static_cast<size_t>(S.nslices + 1), s);
    PB_CUDA(cudaMemsetAsync(S.slice_off.get(), 0, 8 * (S.nslices + 1), s));
    if (S.nslices) {
        k_sell_width<<<blocks_for(S.nslices * 32, 256), 256, 0, s>>>(M.rp.get(), rows, S.nrows, S.nslices,
                                                                     S.slice_off.get());
        PB_CHECK_LAUNCH();
        cub_call([&](void* t, size_t& bytes) {
            return cub::DeviceScan::ExclusiveSum(t, bytes, S.slice_off.get(), S.slice_off.get(), S.nslices + 1, s);
        }, s);
    }
    PB_CUDA(cudaMemcpyAsync(&S.padded_nnz, S.slice_off.get() + S.nslices, 8, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
}

// CODED: <= 255 distinct values over the matrix and every |column - row| <
// 2^23 (the irregular coarse levels of odd grids and general matrices: tens
// of values, thousands of distinct offsets -> neither DICT nor PAT fits).
bool try_coded(const DevMatrix& M, const int32_t* rows, Sell& S, cudaStream_t s) {
    if (S.nrows == 0 || M.nnz == 0) return false;
    DBuf<uint8_t> vcode;
    std::vector<double> table;
    if (!build_value_codes(M.val.get(), M.nnz, vcode, table, s) || table.size() > 255) return false;
    slice_widths(M, rows, S, s);
    if (S.padded_nnz >= (int64_t(1) << 31)) return false;
    S.code.alloc(static_cast<size_t>(S.padded_nnz), s);
    if (S.padded_nnz)
        k_fill_u32<<<blocks_for(S.padded_nnz, 256), 256, 0, s>>>(S.code.get(), S.padded_nnz, 0xFFu);
    DBuf<int> bad(1, s);
    bad.zero(s);
    k_sell_fill_coded<<<blocks_for(S.nrows, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), vcode.get(), rows, S.nrows,
                                                                S.slice_off.get(), S.code.get(), bad.get());
    PB_CHECK_LAUNCH();
    int hb = 0;
    PB_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (hb) {
        S.code.reset();
        S.slice_off.reset();
        S.padded_nnz = 0;
        return false;
    }
    S.hdict.assign(256, make_ulonglong2(0ULL, 0ULL));  // code 255 = pad {+0.0}
    for (size_t c = 0; c < table.size(); ++c) {
        ull vb;
        std::memcpy(&vb, &table[c], 8);
        S.hdict[c] = make_ulonglong2(vb, 0ULL);
    }
    S.ndict = static_cast<int>(table.size());
    S.format = Sell::kCoded;
    return true;
}

}  // namespace

namespace {
void sell_prologue(const DevMatrix& M, const int32_t* rows, int64_t nrows, Sell& S, cudaStream_t s);
}

bool build_sten_wide(const DevMatrix& M, const int32_t* rows, int64_t nrows, Sell& S, cudaStream_t s,
                     const double* l1) {
    sell_prologue(M, rows, nrows, S, s);
    if (nrows && try_pattern(M, rows, S, l1, s) && try_sten(S, kStenWide)) return true;
    S = Sell();
    return false;
}

void build_sell(const DevMatrix& M, const int32_t* rows, int64_t nrows, Sell& S, cudaStream_t s, int storage,
                const double* l1) {
    NvtxRange nv("setup/solve-time storage");
    sell_prologue(M, rows, nrows, S, s);

    // Format choice (measured on B200): STEN whenever the rows
    // nest into one main pattern; else DICT keeps 32 registers and full
    // occupancy, best for short rows; PAT removes the per-entry code stream,
    // best once rows are long (27-point: 187 vs 198 us per L0 sweep); CODED
    // for few distinct values with irregular offsets; PLAIN otherwise.  A
    // forced format (pairamg_setup_config::storage) falls back to PLAIN.
    if (storage != Sell::kPlain) {
        int maxlen = 0;
        {
            DBuf<int64_t> mx(1, s);
            mx.zero(s);
            max_row_len(M, rows, nrows, mx.get(), s);
            int64_t h = 0;
            PB_CUDA(cudaMemcpyAsync(&h, mx.get(), 8, cudaMemcpyDeviceToHost, s));
            PB_CUDA(cudaStreamSynchronize(s));
            maxlen = static_cast<int>(h);
        }
        if (storage < 0) {
            const bool want_pat = maxlen > 16;
            if (maxlen <= kStenMax && try_pattern(M, rows, S, l1, s)) {
                if (try_sten(S) || want_pat) return;
                reset_pat(S);
            }
            if (want_pat && try_pattern(M, rows, S, l1, s)) return;
            if (!want_pat && try_pattern(M, rows, S, l1, s)) return;
            // CODED before DICT: with per-entry values DICT's lookups diverge
            // (varcoef 256^3 level-0 sweep: CODED 202 us, DICT 258 us)
            if (try_coded(M, rows, S, s)) return;
            if (try_dict(M, rows, S, l1, s)) return;
        } else if (storage == Sell::kSten) {
            if (maxlen <= kStenMax && try_pattern(M, rows, S, l1, s)) {
                if (try_sten(S)) return;
                reset_pat(S);
            }
        } else if (storage == Sell::kPat) {
            if (try_pattern(M, rows, S, l1, s)) return;
        } else if (storage == Sell::kDict) {
            if (try_dict(M, rows, S, l1, s)) return;
        } else if (storage == Sell::kCoded) {
            if (try_coded(M, rows, S, s)) return;
        }
        sell_prologue(M, rows, nrows, S, s);
    }
    S.format = Sell::kPlain;
    slice_widths(M, rows, S, s);
    S.col.alloc(static_cast<size_t>(S.padded_nnz), s);
    S.val.alloc(static_cast<size_t>(S.padded_nnz), s);
    if (S.padded_nnz) {
        PB_CUDA(cudaMemsetAsync(S.col.get(), 0xff, 4 * S.padded_nnz, s));
        PB_CUDA(cudaMemsetAsync(S.val.get(), 0, 8 * S.padded_nnz, s));
    }
    if (nrows) {
        k_sell_fill<<<blocks_for(nrows, 256), 256, 0, s>>>(M.rp.get(), M.col.get(), M.val.get(), rows, nrows,
                                                           S.slice_off.get(), S.col.get(), S.val.get());
        PB_CHECK_LAUNCH();
    }
}

double sell_bytes(const Sell& S) {
    if (S.format == Sell::kSten) return 1.0 * S.nrows + 12.0 * S.sten_L + 12.0 * S.npat;
    if (S.format == Sell::kPat) return 1.0 * S.nrows + 16.0 * S.ptab.size() + 16.0 * S.npat;
    if (S.format == Sell::kDict) return 4.0 * S.padded_nnz + 16.0 * S.ndict;
    if (S.format == Sell::kCoded) return 4.0 * S.padded_nnz + 8.0 * (S.nslices + 1) + 8.0 * S.ndict;
    return 12.0 * S.padded_nnz + 8.0 * (S.nslices + 1);
}

double sell_op_bytes(const Sell& S, int op) {
    const double n = static_cast<double>(S.nrows), mat = sell_bytes(S);
    switch (op) {
        case kSpmv: return mat + 16.0 * n;                                             // x, y
        case kJacobi: return mat + (S.format == Sell::kPat || S.format == Sell::kSten ? 24.0 : 32.0) * n;  // x, r, (d), y
        case kResid: return mat + 24.0 * n;                                            // x, r, y
        default: return mat + 32.0 * n;                                                // spmv+dots: w, r, q, v
    }
}

void sell_apply(const Sell& S, const SellOpArgs& o, cudaStream_t s) {
    if (!S.nslices) return;
    if (S.format == Sell::kSten) {
        StenArgs a = sten_args_of(S);
        a.x = o.x;
        a.y = o.y;
        a.r = o.r;
        a.omega = o.omega;
        const bool rows = a.rows != nullptr;
#define PB_STEN(OP)                          \
    if (rows)                                \
        launch_sten<OP, true>(S, a, o.max_grid, s);  \
    else                                     \
        launch_sten<OP, false>(S, a, o.max_grid, s);
        switch (o.op) {
            case kSpmv: PB_STEN(kSpmv) break;
            case kJacobi: PB_STEN(kJacobi) break;
            case kResid: PB_STEN(kResid) break;
            default: fail(PAIRAMG_INTERNAL, "sell_apply: bad op");
        }
#undef PB_STEN
        PB_CHECK_LAUNCH();
        return;
    }
    if (S.format == Sell::kPat) {
        PatArgs a = pat_args_of(S);
        a.x = o.x;
        a.y = o.y;
        a.r = o.r;
        a.omega = o.omega;
        const int grid = blocks_for(S.nrows, kThreads);
        const bool rows = a.rows != nullptr;
#define PB_PAT(OP)                                             \
    if (rows)                                                  \
        k_pat<OP, true><<<grid, kThreads, 0, s>>>(a);          \
    else                                                       \
        k_pat<OP, false><<<grid, kThreads, 0, s>>>(a);
        switch (o.op) {
            case kSpmv: PB_PAT(kSpmv) break;
            case kJacobi: PB_PAT(kJacobi) break;
            case kResid: PB_PAT(kResid) break;
            default: fail(PAIRAMG_INTERNAL, "sell_apply: bad op");
        }
#undef PB_PAT
        PB_CHECK_LAUNCH();
        return;
    }
    SellArgs a = args_of(S);
    a.x = o.x;
    a.y = o.y;
    a.r = o.r;
    a.d = o.d;
    a.omega = o.omega;
    switch (o.op) {
        case kSpmv: launch_op<kSpmv>(S, a, s); break;
        case kJacobi: launch_op<kJacobi>(S, a, s); break;
        case kResid: launch_op<kResid>(S, a, s); break;
        default: fail(PAIRAMG_INTERNAL, "sell_apply: bad op");
    }
}

bool sell_coarse_solve(const Sell& S, const double* rhs, double* x, int nu, double omega, cudaStream_t s) {
    // <= 8 records: with 27 the remote (DSMEM) gathers outweigh the saved
    // launches (measured 1.28 vs 1.25 ms/iter at 27-point 192^3)
    if (S.format != Sell::kSten || !S.rows.empty() || S.row0 != 0 || S.nrows != S.xlen || nu < 1 ||
        S.nrows > int64_t(kCoarseCta) * kCoarseRows || S.sten_L > 8)
        return false;
    const int R = static_cast<int>((S.nrows + kCoarseCta - 1) / kCoarseCta);
    StenArgs a = sten_args_of(S);
    a.r = rhs;
    a.omega = omega;
    const StenParam p = sten_param(S);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kCoarseCta);
    cfg.blockDim = dim3(kCoarseThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCoarseCta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl_mask() & 2) ? 2 : 1;
    if (S.sten_L == 7)
        PB_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_solve<7>, a, p, x, nu, R));
    else if (S.sten_L == 27)
        PB_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_solve<27>, a, p, x, nu, R));
    else
        PB_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_solve<0>, a, p, x, nu, R));
    return true;
}

bool sell_march_ok(const Sell& S) { return S.format == Sell::kSten && sten_march(S); }

bool sell_split_ok(const Sell& I, const Sell& B) {
    return I.format == Sell::kSten && B.format == Sell::kSten && I.rows.empty() && I.nrows > 0 && B.nrows > 0;
}

namespace {
struct SplitPlan {
    StenArgs a;
    HaloSplit h;
    int la;
    bool r2;
    bool march;  // interior blocks are marching tiles (k_sten_march_split)
    MarchGeom g;
    int grid;
};

// Push blocks: kPushVals values each (2 per thread: the push is on the
// neighbour's critical path -- the 2.1 M-row level 1 at N = 2 runs its V-cycle
// share in 181 vs 199 us/iter with 512 vs 2048 per block), at most kMaxPush
// (more push blocks at level 0 took SM slots from the interior: 7-point
// level 0 807-836 vs 800 us/iter uncapped).
constexpr int kPushVals = 512;
constexpr int kMaxPush = 32;

SplitPlan split_plan(const Sell& I, const Sell& B, bool dots, const HaloSrc* hs) {
    SplitPlan P{};
    P.march = sten_march(I, &P.g);
    P.la = (I.sten_L == 7 || I.sten_L == 27) && sten_center(I) ? I.sten_L : 0;
    P.r2 = !P.march && P.la != 0 && sten_rpt2(I, dots);
    P.a = sten_args_of(I, P.r2 ? 512 : 256);
    P.h.pa = sten_param(I);
    P.h.pb = sten_param_w(B);
    P.h.b = sten_args_of(B);
    P.h.nblk_a = P.march ? march_grid(P.g) : P.a.nblk;
    P.h.nblk_b = P.h.b.nblk;
    P.grid = P.h.nblk_a + P.h.nblk_b;
    if (hs) {
        P.h.flags = hs->flags;
        P.h.nfrom = hs->nfrom;
        for (int i = 0; i < 8; ++i) P.h.from[i] = hs->from[i];
        P.h.staging = hs->staging;
        P.h.nhalo = hs->nhalo;
        P.h.ctr = hs->ctr;
        P.h.b.nown = static_cast<int>(I.xlen - hs->nhalo);
        if (hs->fused) {  // push blocks ahead of the boundary blocks
            const int64_t nsend = hs->off[hs->npeers];
            P.h.npush = static_cast<int>(
                std::min<int64_t>(kMaxPush, std::max<int64_t>(1, (nsend + kPushVals - 1) / kPushVals)));
            P.h.npeers = hs->npeers;
            for (int i = 0; i <= hs->npeers; ++i) P.h.off[i] = hs->off[i];
            for (int i = 0; i < hs->npeers; ++i) {
                P.h.dst[i] = hs->dst[i];
                P.h.stride[i] = hs->stride[i];
                P.h.pflag[i] = hs->pflag[i];
            }
            P.h.send_idx = hs->send_idx;
        }
    }
    // gather interiors: boundary blocks dispatched two resident waves before
    // the end of the interior -- their halo has long arrived at level 0 (the
    // neighbours push at their launch start) and they no longer form a
    // serial tail after the last interior wave (7-point N = 2: 72.3 -> 71.5
    // ms).  Marching interiors keep the boundary last (two waves early:
    // 42.6 -> 46.6 ms, 27-point).
    const int resident = kSmCount * (P.la == 7 ? 5 : 2);
    P.h.bnd_at = P.march ? P.h.nblk_a : std::max(0, P.h.nblk_a - 2 * resident);
    P.grid = P.h.npush + P.h.nblk_a + P.h.nblk_b;
    return P;
}
}  // namespace

void sell_apply_split(const Sell& I, const Sell& B, const SellOpArgs& o, const HaloSrc& hs, cudaStream_t s) {
    SplitPlan P = split_plan(I, B, false, &hs);
    for (StenArgs* a : {&P.a, &P.h.b}) {
        a->x = o.x;
        a->y = o.y;
        a->r = o.r;
        a->omega = o.omega;
    }
    const bool br = !B.rows.empty();
#define PB_SPLIT2(OP, BR)                                                                                 \
    if (P.march) launch_k<2>(k_sten_march_split<OP, BR>, P.grid, 256, 0, s, P.a, P.h, P.g);              \
    else if (P.la == 7 && P.r2) launch_k<2>(k_sten_split<OP, 7, true, BR>, P.grid, 256, 0, s, P.a, P.h);        \
    else if (P.la == 7) launch_k<2>(k_sten_split<OP, 7, false, BR>, P.grid, 256, 0, s, P.a, P.h);         \
    else if (P.la == 27 && P.r2) launch_k<2>(k_sten_split<OP, 27, true, BR>, P.grid, 256, 0, s, P.a, P.h);  \
    else if (P.la == 27) launch_k<2>(k_sten_split<OP, 27, false, BR>, P.grid, 256, 0, s, P.a, P.h);       \
    else launch_k<2>(k_sten_split<OP, 0, false, BR>, P.grid, 256, 0, s, P.a, P.h);
#define PB_SPLIT(OP)      \
    if (br) {             \
        PB_SPLIT2(OP, true)  \
    } else {              \
        PB_SPLIT2(OP, false) \
    }
    switch (o.op) {
        case kSpmv: PB_SPLIT(kSpmv) break;
        case kJacobi: PB_SPLIT(kJacobi) break;
        case kResid: PB_SPLIT(kResid) break;
        default: fail(PAIRAMG_INTERNAL, "sell_apply_split: bad op");
    }
#undef PB_SPLIT
#undef PB_SPLIT2
}

// upper bound: the fused push adds <= kMaxPush blocks
int sell_split_dots_grid(const Sell& I, const Sell& B) { return split_plan(I, B, true, nullptr).grid + kMaxPush; }

int sell_spmv_dots_split(const Sell& I, const Sell& B, const double* w, double* v, const double* r, const double* q,
                         double* partials, int max_blocks, const HaloSrc& hs, cudaStream_t s) {
    SplitPlan P = split_plan(I, B, true, &hs);
    if (P.grid > max_blocks) fail(PAIRAMG_INTERNAL, "sell_spmv_dots_split: partial buffer too small");
    for (StenArgs* a : {&P.a, &P.h.b}) {
        a->x = w;
        a->y = v;
        a->r = r;
        a->q = q;
        a->partials = partials;
    }
    const bool br = !B.rows.empty();
    auto go = [&](auto kt, auto kf) {
        if (br)
            launch_k<2>(kt, P.grid, 256, 0, s, P.a, P.h);
        else
            launch_k<2>(kf, P.grid, 256, 0, s, P.a, P.h);
    };
    if (P.march) {
        if (br)
            launch_k<2>(k_sten_march_split_dots<true>, P.grid, 256, 0, s, P.a, P.h, P.g);
        else
            launch_k<2>(k_sten_march_split_dots<false>, P.grid, 256, 0, s, P.a, P.h, P.g);
    } else if (P.la == 7 && P.r2)
        go(k_sten_split_dots<7, true, true>, k_sten_split_dots<7, true, false>);
    else if (P.la == 7)
        go(k_sten_split_dots<7, false, true>, k_sten_split_dots<7, false, false>);
    else if (P.la == 27 && P.r2)
        go(k_sten_split_dots<27, true, true>, k_sten_split_dots<27, true, false>);
    else if (P.la == 27)
        go(k_sten_split_dots<27, false, true>, k_sten_split_dots<27, false, false>);
    else
        go(k_sten_split_dots<0, false, true>, k_sten_split_dots<0, false, false>);
    return P.grid;
}

int sell_dots_grid(const Sell& S, int cap) {
    MarchGeom g;
    if (S.format == Sell::kSten && cap == 0 && S.rows.empty() && sten_march(S, &g)) return march_grid(g);
    if (S.format == Sell::kSten && sten_rpt2(S, true)) {  // k_sten2_dots: per-warp partials unless capped
        const int nb = blocks_for(S.nrows, 512), grid = capped(nb, cap);
        return grid < nb ? grid : 8 * grid;
    }
    if (S.format == Sell::kSten) return capped(blocks_for(S.nrows, 256), cap);
    if (S.format != Sell::kPat) return blocks_for(S.nslices, kWarps);  // one warp per slice
    const int64_t want = (S.nrows + kThreads - 1) / kThreads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(kSmCount) * 8)));
}

int sell_spmv_dots(const Sell& S, const double* w, double* v, const double* r, const double* q, double* partials,
                   int max_blocks, cudaStream_t s, int cap) {
    if (!S.nrows) return 0;
    const int grid = sell_dots_grid(S, cap);
    if (grid > max_blocks) fail(PAIRAMG_INTERNAL, "sell_spmv_dots: partial buffer too small");
    const bool rows = !S.rows.empty();
    if (S.format == Sell::kSten) {
        StenArgs a = sten_args_of(S);
        a.x = w;
        a.y = v;
        a.r = r;
        a.q = q;
        a.partials = partials;
        const int g = rows ? launch_sten_dots<true>(S, a, cap, s) : launch_sten_dots<false>(S, a, cap, s);
        PB_CHECK_LAUNCH();
        if (g != grid) fail(PAIRAMG_INTERNAL, "sell_spmv_dots: grid mismatch");
        return grid;
    }
    if (S.format == Sell::kPat) {
        PatArgs p = pat_args_of(S);
        p.x = w;
        p.y = v;
        p.r = r;
        p.q = q;
        p.partials = partials;
        if (rows)
            k_pat_spmv_dots<true><<<grid, kThreads, 0, s>>>(p);
        else
            k_pat_spmv_dots<false><<<grid, kThreads, 0, s>>>(p);
        PB_CHECK_LAUNCH();
        return grid;
    }
    SellArgs a = args_of(S);
    a.x = w;
    a.y = v;
    a.r = r;
    a.q = q;
    a.partials = partials;
    if (S.format == Sell::kDict) {
        const DictParam<kFDict> dp = dict_param(S);
        if (rows)
            k_sell_spmv_dots<kFDict, true><<<grid, kThreads, 0, s>>>(a, dp);
        else
            k_sell_spmv_dots<kFDict, false><<<grid, kThreads, 0, s>>>(a, dp);
    } else if (S.format == Sell::kCoded) {
        const DictParam<kFCoded> dp = coded_param(S);
        if (rows)
            k_sell_spmv_dots<kFCoded, true><<<grid, kThreads, 0, s>>>(a, dp);
        else
            k_sell_spmv_dots<kFCoded, false><<<grid, kThreads, 0, s>>>(a, dp);
    } else {
        const DictParam<kFPlain> dp{0};
        if (rows)
            k_sell_spmv_dots<kFPlain, true><<<grid, kThreads, 0, s>>>(a, dp);
        else
            k_sell_spmv_dots<kFPlain, false><<<grid, kThreads, 0, s>>>(a, dp);
    }
    PB_CHECK_LAUNCH();
    return grid;
}

}  // namespace pb
