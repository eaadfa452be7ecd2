// setup.cu -- decoupled-aggregation AMG setup on the device (amg.cpp:144-295):
//   per pairwise step:
//     k_diag + k_weights   extract_diagonal_block + build_weights (matching.cpp:8-60)
//     k_suitor + k_mate    parallel Suitor matching (matching.cpp:62-100) under the
//                          total order key(e) = (w, -min, -max): lock-free proposals
//                          with 128-bit compare-and-swap on (weight, proposer) slots;
//                          equals the sequential total-order Suitor / greedy matching
//     k_leader + scan +    build_pairwise_prolongator (amg.cpp:38-77)
//     k_aggregate
//     k_galerkin_*         galerkin_product R*(A*P) (amg.cpp:110-142) as ONE fused
//                          kernel per coarse row: the A*P row products and the R*C
//                          accumulation in the reference's exact summation order
//                          (csr.cpp:206-272), two-phase (symbolic count, numeric fill)
//     k_wnext              w_{k+1} = R w_k (amg.cpp:244-247)
//   per level: k_compose (compose_prolongators, amg.cpp:79-85), composed Galerkin,
//   R = P^T (transpose_block, amg.cpp:87-108), l1 diagonal, halo plan, SELL copy.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cmath>

#include "amg.cuh"

namespace pb {

namespace {

using ull = unsigned long long;
using Clock = std::chrono::steady_clock;

double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// PAIRAMG_VERBOSE: per-phase setup times on stderr (development aid)
void trace(const Runtime& rt, const char* what, double secs) {
    static const bool on = env_flag("PAIRAMG_VERBOSE", false);
    if (on) std::fprintf(stderr, "rank %d setup %-28s %.4f s\n", rt.rank(), what, secs);
}

template <typename F>
void cub_call(F&& f, cudaStream_t s) {
    size_t bytes = 0;
    PB_CUDA(f(nullptr, bytes));
    DBuf<uint8_t> tmp(bytes ? bytes : 1, s);
    PB_CUDA(f(tmp.get(), bytes));
}

template <typename T>
T read_one(const T* d, cudaStream_t s) {
    T h{};
    PB_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    return h;
}

// ------------------------------------------------------------ weights ---

__global__ void k_diag(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                       const double* __restrict__ val, int64_t n, double* __restrict__ diag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = 0.0;
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t)
        if (col[t] == i) d = val[t];
    diag[i] = d;
}

// build_weights (matching.cpp:28-60), exact operation order:
//   num = ((2*a_ij)*w_i)*w_j ; den = (a_ii*w_i)*w_i + (a_jj*w_j)*w_j ;
//   weight = 1 - num/den, non-finite -> -1e300 (matching.hpp:29).
__global__ void k_weights(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                          const double* __restrict__ val, int64_t n, const double* __restrict__ w,
                          const double* __restrict__ diag, double* __restrict__ gw,
                          ull* __restrict__ clamped) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double wi = w[i], di = diag[i];
    ull nclamp = 0;
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
        const int32_t j = col[t];
        if (j >= n || j == i) continue;
        const double wj = w[j];
        const double num = dmul(dmul(dmul(2.0, val[t]), wi), wj);
        const double den = dadd(dmul(dmul(di, wi), wi), dmul(dmul(diag[j], wj), wj));
        double weight = dsub(1.0, ddiv(num, den));
        if (!isfinite(weight)) {
            weight = -1e300;
            ++nclamp;
        }
        gw[t] = weight;
    }
    if (nclamp) atomicAdd(clamped, nclamp);
}

// ------------------------------------------------------------ suitor ---

// Monotone map double -> uint64 (larger double -> larger integer).
__device__ __forceinline__ ull ordered(double x) {
    if (x == 0.0) x = 0.0;  // canonical +0
    const long long b = __double_as_longlong(x);
    return b < 0 ? ~static_cast<ull>(b) : (static_cast<ull>(b) | 0x8000000000000000ULL);
}

// Strong (relaxed, gpu scope) single-copy-atomic 128-bit load of a slot.
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

__device__ __forceinline__ bool key_gt(ull ahi, ull alo, ull bhi, ull blo) {
    return ahi > bhi || (ahi == bhi && alo > blo);
}

// Parallel Suitor (Manne & Halappanavar) on the owned diagonal block.  Slot
// v holds (lo = ~proposer, hi = ordered(weight)); a proposer u beats the
// holder s of v iff key(u,v) > key(s,v), i.e. heavier, or equally heavy and
// u < s -- exactly key(e) = (w, -min, -max) restricted to edges at v.  A
// proposer picks its heaviest acceptable neighbour, smallest index on ties
// (the reference's ascending strict scan, matching.cpp:79-86); a displaced
// holder re-proposes (matching.cpp:88-91).  With a strict total order on
// edges the result is unique (the greedy matching) whatever the schedule.
__global__ void k_suitor(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                         const double* __restrict__ gw, int64_t n, ull* __restrict__ slot) {
    const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u >= n) return;
    int64_t cur = u;
    while (cur >= 0) {
        const ull mylo = ~static_cast<ull>(cur);
        int64_t partner = -1;
        ull bhi = 0;
        for (int64_t t = rp[cur]; t < rp[cur + 1]; ++t) {
            const int32_t j = col[t];
            if (j >= n || j == cur) continue;
            const ull hi = ordered(gw[t]);
            if (partner >= 0 && hi <= bhi) continue;
            ull slo, shi;
            ld_slot(slot + 2 * j, slo, shi);
            if (key_gt(hi, mylo, shi, slo)) {
                partner = j;
                bhi = hi;
            }
        }
        if (partner < 0) break;
        while (true) {
            ull slo, shi;
            ld_slot(slot + 2 * partner, slo, shi);
            if (!key_gt(bhi, mylo, shi, slo)) break;  // lost the slot: rescan
            if (cas_slot(slot + 2 * partner, slo, shi, mylo, bhi)) {
                cur = (slo == 0 && shi == 0) ? -1 : static_cast<int64_t>(~slo);
                break;
            }
        }
    }
}

// mate = mutual suitors (matching.cpp:95-98)
__global__ void k_mate(const ull* __restrict__ slot, int64_t n, int64_t* __restrict__ mate) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const ull lo = slot[2 * v], hi = slot[2 * v + 1];
    int64_t m = -1;
    if (lo || hi) {
        const int64_t s = static_cast<int64_t>(~lo);
        const ull slo = slot[2 * s], shi = slot[2 * s + 1];
        if ((slo || shi) && static_cast<int64_t>(~slo) == v) m = s;
    }
    mate[v] = m;
}

// ------------------------------------------------------- aggregation ---

__global__ void k_leader(const int64_t* __restrict__ mate, int64_t n, int64_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (mate[i] < 0 || mate[i] > i) ? 1 : 0;
    if (i == n) flag[n] = 0;
}

// build_pairwise_prolongator (amg.cpp:38-77): aggregate id = rank of the
// smallest member; P value w_i/sqrt(w_i^2 + w_j^2) (1/sqrt(2) if the norm is
// 0) or w_i/|w_i| (1 if w_i == 0).
__global__ void k_aggregate(const int64_t* __restrict__ mate, const int64_t* __restrict__ pos,
                            const double* __restrict__ w, int64_t n, int32_t* __restrict__ agg,
                            double* __restrict__ pv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t j = mate[i];
    const int64_t leader = (j < 0 || j > i) ? i : j;
    agg[i] = static_cast<int32_t>(pos[leader]);
    const double wi = w[i];
    if (j < 0) {
        pv[i] = wi == 0.0 ? 1.0 : ddiv(wi, fabs(wi));
    } else {
        const double wj = w[j];
        const double norm = __dsqrt_rn(dadd(dmul(wi, wi), dmul(wj, wj)));
        pv[i] = norm == 0.0 ? ddiv(1.0, __dsqrt_rn(2.0)) : ddiv(wi, norm);
    }
}

__global__ void k_global_mate(const int64_t* __restrict__ mate, int64_t n, int64_t base,
                              int64_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = mate[i] < 0 ? -1 : mate[i] + base;
}

// ------------------------------------------------------------ R = P^T ---

__global__ void k_count(const int32_t* __restrict__ pcol, int64_t nf, int64_t* __restrict__ cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nf) atomicAdd(reinterpret_cast<ull*>(cnt + pcol[i]), 1ULL);
}

__global__ void k_rfill(const int32_t* __restrict__ pcol, int64_t nf, const int64_t* __restrict__ rrp,
                        ull* __restrict__ cursor, int32_t* __restrict__ rcol) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int32_t c = pcol[i];
    const ull slot = atomicAdd(cursor + c, 1ULL);
    rcol[rrp[c] + static_cast<int64_t>(slot)] = static_cast<int32_t>(i);
}

// transpose_block order (amg.cpp:99-106): fine rows ascending within a row.
__global__ void k_rsort(const int64_t* __restrict__ rrp, int64_t nc, int32_t* __restrict__ rcol,
                        const double* __restrict__ pval, double* __restrict__ rval) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const int64_t b = rrp[c], e = rrp[c + 1];
    for (int64_t a = b + 1; a < e; ++a) {
        const int32_t k = rcol[a];
        int64_t q = a - 1;
        while (q >= b && rcol[q] > k) {
            rcol[q + 1] = rcol[q];
            --q;
        }
        rcol[q + 1] = k;
    }
    for (int64_t a = b; a < e; ++a) rval[a] = pval[rcol[a]];
}

// w_{k+1} = R w_k (amg.cpp:244-247): 0.0 + sum over fine rows ascending.
__global__ void k_wnext(const int64_t* __restrict__ rrp, const int32_t* __restrict__ rcol,
                        const double* __restrict__ rval, const double* __restrict__ w, int64_t nc,
                        double* __restrict__ wn) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    double s = 0.0;
    for (int64_t t = rrp[c]; t < rrp[c + 1]; ++t) s = dadd(s, dmul(rval[t], w[rcol[t]]));
    wn[c] = s;
}

// compose_prolongators (amg.cpp:79-85): left to right, value (v1*p2)*p3.
__global__ void k_compose(int32_t* __restrict__ ccol, double* __restrict__ cval, int64_t nf,
                          const int32_t* __restrict__ agg, const double* __restrict__ pv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int32_t c = ccol[i];
    cval[i] = dmul(cval[i], pv[c]);
    ccol[i] = agg[c];
}

__global__ void k_pext(const int32_t* __restrict__ pcol, const double* __restrict__ pval, int64_t n,
                       int64_t cbase, int64_t* __restrict__ gc, double* __restrict__ gv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    gc[i] = cbase + pcol[i];
    gv[i] = pval[i];
}

// ----------------------------------------------------------- Galerkin ---

// One team (a warp, or a whole block for dense rows) owns coarse row c of
// A_c = R*(A*P).  Contributions are gathered in the reference's encounter
// order (fine row t of R's row ascending, then A's row in CSR order), each
// (gc = P column of a_ij's column, v = a_ij * p_j, r_t).  Per distinct coarse
// column:  C_t = first v, then + later v of fine row t (A*P entry,
// csr.cpp:145-160);  A_c = first r_t*C_t, then + later ones (R*C entry).
struct GalerkinArgs {
    const int64_t* rp;
    const int32_t* col;
    const double* val;
    const int64_t* pc;  // P column (global coarse id) per local column slot
    const double* pv;
    const int64_t* rrp;
    const int32_t* rcol;
    const double* rval;
    int64_t nc;
    int64_t* cnt;        // symbolic: distinct columns per row (-1 = needs the big kernel)
    const int64_t* orp;  // numeric: output row pointer
    int64_t* ocol;
    double* oval;
};

template <bool NUMERIC>
__device__ void galerkin_team(const GalerkinArgs& a, int64_t c, int lane, int team, int cap,
                              int64_t* sgc, double* sv, double* sr, int* st, bool block_sync) {
    auto sync = [&] {
        if (block_sync)
            __syncthreads();
        else
            __syncwarp();
    };
    // gather
    int m = 0;
    const int64_t rb = a.rrp[c], re = a.rrp[c + 1];
    bool overflow = false;
    for (int64_t t = rb; t < re; ++t) {
        const int32_t i = a.rcol[t];
        const double rv = a.rval[t];
        const int64_t b = a.rp[i], e = a.rp[i + 1];
        const int len = static_cast<int>(e - b);
        if (m + len > cap) {
            overflow = true;
            break;
        }
        for (int u = lane; u < len; u += team) {
            const int32_t j = a.col[b + u];
            sgc[m + u] = a.pc[j];
            if (NUMERIC) {
                sv[m + u] = dmul(a.val[b + u], a.pv[j]);
                sr[m + u] = rv;
                st[m + u] = static_cast<int>(t - rb);
            }
        }
        m += len;
    }
    sync();
    if (overflow) {
        if (!NUMERIC && lane == 0) a.cnt[c] = -1;
        return;
    }
    // Sort keys (coarse column << 16 | encounter position) with a team-wide
    // bitonic network: equal columns become contiguous segments whose
    // elements stay in encounter order (t ascending, then CSR order).
    uint64_t* key = reinterpret_cast<uint64_t*>(sgc);  // in place over the gathered columns
    int p2 = 2;
    while (p2 < m) p2 <<= 1;
    for (int q = lane; q < p2; q += team)
        key[q] = q < m ? (static_cast<uint64_t>(sgc[q]) << 16) | static_cast<uint64_t>(q) : ~0ULL;
    sync();
    for (int k = 2; k <= p2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < p2; i += team) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t x = key[i], y = key[ixj];
                    if ((x > y) == ((i & k) == 0)) {
                        key[i] = y;
                        key[ixj] = x;
                    }
                }
            }
            sync();
        }
    // segment starts -> distinct count and output rank (team exclusive scan
    // over contiguous per-thread chunks)
    const int chunk = (p2 + team - 1) / team;
    const int c0 = lane * chunk, c1 = min(c0 + chunk, m);
    int mine = 0;
    for (int i = c0; i < c1; ++i) mine += (i == 0 || (key[i] >> 16) != (key[i - 1] >> 16)) ? 1 : 0;
    int incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((lane & 31) >= o) incl += v;
    }
    int total = __shfl_sync(0xffffffffu, incl, 31);
    int base = incl - mine;
    if (block_sync) {
        __shared__ int wsum[32];
        if ((lane & 31) == 31) wsum[lane >> 5] = incl;
        __syncthreads();
        int before = 0;
        total = 0;
        for (int w = 0; w < (team + 31) / 32; ++w) {
            if (w < (lane >> 5)) before += wsum[w];
            total += wsum[w];
        }
        base += before;
        __syncthreads();
    }
    if (!NUMERIC) {
        if (lane == 0) a.cnt[c] = total;
        return;
    }
    const int64_t ob = a.orp[c];
    int rank = base;
    for (int i = c0; i < c1; ++i) {
        const uint64_t g = key[i] >> 16;
        if (!(i == 0 || g != (key[i - 1] >> 16))) continue;
        // reference-order accumulation over the segment
        bool acc_set = false, ct_set = false;
        double acc = 0.0, ct = 0.0, rt = 0.0;
        int cur_t = -1;
        for (int j = i; j < m && (key[j] >> 16) == g; ++j) {
            const int q = static_cast<int>(key[j] & 0xFFFFu);
            const int t2 = st[q];
            if (t2 != cur_t) {
                if (ct_set) {
                    const double contrib = dmul(rt, ct);
                    acc = acc_set ? dadd(acc, contrib) : contrib;
                    acc_set = true;
                }
                ct_set = false;
                cur_t = t2;
                rt = sr[q];
            }
            ct = ct_set ? dadd(ct, sv[q]) : sv[q];
            ct_set = true;
        }
        if (ct_set) {
            const double contrib = dmul(rt, ct);
            acc = acc_set ? dadd(acc, contrib) : contrib;
        }
        a.ocol[ob + rank] = static_cast<int64_t>(g);
        a.oval[ob + rank] = acc;
        ++rank;
    }
}

constexpr int kGalWarps = 4;
constexpr int kGalCap = 256;      // contributions per coarse row (warp kernel)
constexpr int kGalBigCap = 4096;  // block kernel
constexpr int kGalBigThreads = 256;

template <bool NUMERIC>
__global__ void __launch_bounds__(kGalWarps * 32) k_galerkin_warp(GalerkinArgs a) {
    __shared__ int64_t sgc[kGalWarps][kGalCap];
    __shared__ double sv[NUMERIC ? kGalWarps : 1][NUMERIC ? kGalCap : 1];
    __shared__ double sr[NUMERIC ? kGalWarps : 1][NUMERIC ? kGalCap : 1];
    __shared__ int st[NUMERIC ? kGalWarps : 1][NUMERIC ? kGalCap : 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kGalWarps + warp;
    if (c >= a.nc) return;
    if (NUMERIC && a.cnt[c] < 0) return;  // handled by the block kernel
    galerkin_team<NUMERIC>(a, c, lane, 32, kGalCap, sgc[warp], NUMERIC ? sv[warp] : nullptr,
                           NUMERIC ? sr[warp] : nullptr, NUMERIC ? st[warp] : nullptr, false);
}

template <bool NUMERIC>
__global__ void __launch_bounds__(kGalBigThreads) k_galerkin_block(GalerkinArgs a, const int64_t* rows,
                                                                   int64_t nrows) {
    extern __shared__ __align__(16) unsigned char smem[];
    int64_t* sgc = reinterpret_cast<int64_t*>(smem);
    double* sv = reinterpret_cast<double*>(sgc + kGalBigCap);
    double* sr = sv + kGalBigCap;
    int* st = reinterpret_cast<int*>(sr + kGalBigCap);
    for (int64_t k = blockIdx.x; k < nrows; k += gridDim.x) {
        const int64_t c = rows[k];
        galerkin_team<NUMERIC>(a, c, threadIdx.x, blockDim.x, kGalBigCap, sgc, sv, sr, st, true);
        __syncthreads();
    }
}

// ---- coarse rows beyond the block kernel's shared-memory capacity ----
// Contributions of each such row go to global memory in encounter order
// (key = row << 40 | coarse column), a stable radix sort makes equal columns
// contiguous without reordering them, and one thread per segment folds it in
// the reference's order -- the same arithmetic as galerkin_team.
constexpr int kHugeColBits = 40;

__global__ void k_huge_len(GalerkinArgs a, const int64_t* __restrict__ rows, int64_t nh, int64_t* __restrict__ len) {
    const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h > nh) return;
    if (h == nh) {
        len[nh] = 0;
        return;
    }
    const int64_t c = rows[h];
    int64_t m = 0;
    for (int64_t t = a.rrp[c]; t < a.rrp[c + 1]; ++t) {
        const int32_t i = a.rcol[t];
        m += a.rp[i + 1] - a.rp[i];
    }
    len[h] = m;
}

__global__ void k_huge_fill(GalerkinArgs a, const int64_t* __restrict__ rows, int64_t nh, const int64_t* __restrict__ off,
                            uint64_t* __restrict__ key, int64_t* __restrict__ pos, double* __restrict__ hv,
                            double* __restrict__ hr, int32_t* __restrict__ ht) {
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t c = rows[h];
        int64_t m = off[h];
        const int64_t rb = a.rrp[c], re = a.rrp[c + 1];
        for (int64_t t = rb; t < re; ++t) {
            const int32_t i = a.rcol[t];
            const double rv = a.rval[t];
            const int64_t b = a.rp[i], e = a.rp[i + 1];
            for (int64_t u = threadIdx.x; u < e - b; u += blockDim.x) {
                const int32_t j = a.col[b + u];
                key[m + u] = (static_cast<uint64_t>(h) << kHugeColBits) | static_cast<uint64_t>(a.pc[j]);
                pos[m + u] = m + u;
                hv[m + u] = dmul(a.val[b + u], a.pv[j]);
                hr[m + u] = rv;
                ht[m + u] = static_cast<int32_t>(t - rb);
            }
            m += e - b;
        }
    }
}

__global__ void k_huge_heads(const uint64_t* __restrict__ key, int64_t M, int64_t* __restrict__ head) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < M) head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// distinct columns of huge row h = segments starting in [off[h], off[h+1])
__global__ void k_huge_count(const int64_t* __restrict__ rows, int64_t nh, const int64_t* __restrict__ off,
                             const int64_t* __restrict__ segx, int64_t M, int64_t nseg, int64_t* __restrict__ cnt) {
    const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h >= nh) return;
    const int64_t a0 = off[h] < M ? segx[off[h]] : nseg;
    const int64_t a1 = off[h + 1] < M ? segx[off[h + 1]] : nseg;
    cnt[rows[h]] = a1 - a0;
}

__global__ void k_huge_fold(GalerkinArgs a, const int64_t* __restrict__ rows, const int64_t* __restrict__ off,
                            const uint64_t* __restrict__ key, const int64_t* __restrict__ pos,
                            const double* __restrict__ hv, const double* __restrict__ hr,
                            const int32_t* __restrict__ ht, const int64_t* __restrict__ segx, int64_t M) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M || !(i == 0 || key[i] != key[i - 1])) return;
    const int64_t h = static_cast<int64_t>(key[i] >> kHugeColBits);
    const int64_t c = rows[h];
    bool acc_set = false, ct_set = false;
    double acc = 0.0, ct = 0.0, rt = 0.0;
    int cur_t = -1;
    for (int64_t j = i; j < M && key[j] == key[i]; ++j) {
        const int64_t q = pos[j];
        const int t2 = ht[q];
        if (t2 != cur_t) {
            if (ct_set) {
                const double contrib = dmul(rt, ct);
                acc = acc_set ? dadd(acc, contrib) : contrib;
                acc_set = true;
            }
            ct_set = false;
            cur_t = t2;
            rt = hr[q];
        }
        ct = ct_set ? dadd(ct, hv[q]) : hv[q];
        ct_set = true;
    }
    if (ct_set) {
        const double contrib = dmul(rt, ct);
        acc = acc_set ? dadd(acc, contrib) : contrib;
    }
    const int64_t o = a.orp[c] + (segx[i] - segx[off[h]]);
    a.ocol[o] = static_cast<int64_t>(key[i] & ((uint64_t(1) << kHugeColBits) - 1));
    a.oval[o] = acc;
}

__global__ void k_flag_big(const int64_t* __restrict__ cnt, int64_t nc, int64_t* __restrict__ flag) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < nc) flag[c] = cnt[c] < 0 ? 1 : 0;
}

__global__ void k_fill_l(double* __restrict__ x, int64_t n, double v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

#define LAUNCH(kernel, n, ...)                                                          \
    do {                                                                                \
        if ((n) > 0) kernel<<<blocks_for((n), 256), 256, 0, s>>>(__VA_ARGS__);          \
        PB_CHECK_LAUNCH();                                                              \
    } while (0)

// R = P^T from a local prolongator (pcol over nf fine rows into nc coarse).
void build_R(const int32_t* pcol, const double* pval, int64_t nf, int64_t nc, DBuf<int64_t>& rrp,
             DBuf<int32_t>& rcol, DBuf<double>& rval, cudaStream_t s) {
    rrp.alloc(static_cast<size_t>(nc + 1), s);
    rrp.zero(s);
    LAUNCH(k_count, nf, pcol, nf, rrp.get());
    cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, rrp.get(), rrp.get(), nc + 1, s);
    }, s);
    DBuf<ull> cursor(static_cast<size_t>(nc), s);
    cursor.zero(s);
    rcol.alloc(static_cast<size_t>(nf), s);
    rval.alloc(static_cast<size_t>(nf), s);
    LAUNCH(k_rfill, nf, pcol, nf, rrp.get(), cursor.get(), rcol.get());
    LAUNCH(k_rsort, nc, rrp.get(), nc, rcol.get(), pval, rval.get());
}

// Galerkin product A_c = R*(A*P) (galerkin_product, amg.cpp:110-142).
// pc/pv cover the owned + halo column slots of A.  Returns the global-column
// CSR of the owned coarse rows.
int64_t galerkin(const DevMatrix& A, const int64_t* pc, const double* pv, const int64_t* rrp,
                 const int32_t* rcol, const double* rval, int64_t nc, DBuf<int64_t>& orp,
                 DBuf<int64_t>& ocol, DBuf<double>& oval, cudaStream_t s) {
    NvtxRange nv("setup/galerkin R*(A*P)");
    GalerkinArgs a{};
    a.rp = A.rp.get();
    a.col = A.col.get();
    a.val = A.val.get();
    a.pc = pc;
    a.pv = pv;
    a.rrp = rrp;
    a.rcol = rcol;
    a.rval = rval;
    a.nc = nc;
    DBuf<int64_t> cnt(static_cast<size_t>(nc + 1), s);
    PB_CUDA(cudaMemsetAsync(cnt.get() + nc, 0, 8, s));
    a.cnt = cnt.get();
    const int gw = blocks_for(nc, kGalWarps);
    if (nc) k_galerkin_warp<false><<<gw, kGalWarps * 32, 0, s>>>(a);
    PB_CHECK_LAUNCH();
    // rows that overflowed the warp capacity
    DBuf<int64_t> big;
    int64_t nbig = 0;
    {
        DBuf<int64_t> flag(static_cast<size_t>(nc), s), sel(static_cast<size_t>(nc), s), num(1, s);
        LAUNCH(k_flag_big, nc, cnt.get(), nc, flag.get());
        thrust::counting_iterator<int64_t> it(0);
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, it, flag.get(), sel.get(), num.get(), nc, s);
        }, s);
        nbig = read_one(num.get(), s);
        if (nbig) {
            big.alloc(static_cast<size_t>(nbig), s);
            PB_CUDA(cudaMemcpyAsync(big.get(), sel.get(), 8 * nbig, cudaMemcpyDeviceToDevice, s));
        }
    }
    const size_t big_smem = kGalBigCap * (8 + 8 + 8 + 4);
    int64_t nhuge = 0;
    if (nbig) {
        PB_CUDA(cudaFuncSetAttribute(k_galerkin_block<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(big_smem)));
        PB_CUDA(cudaFuncSetAttribute(k_galerkin_block<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(big_smem)));
        k_galerkin_block<false><<<static_cast<int>(std::min<int64_t>(nbig, 4 * kSmCount)), kGalBigThreads,
                                  big_smem, s>>>(a, big.get(), nbig);
        PB_CHECK_LAUNCH();
        // still negative -> too dense
        DBuf<int64_t> flag(static_cast<size_t>(nc), s), num(1, s);
        LAUNCH(k_flag_big, nc, cnt.get(), nc, flag.get());
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceReduce::Sum(t, b, flag.get(), num.get(), nc, s);
        }, s);
        nhuge = read_one(num.get(), s);
    }
    // rows beyond kGalBigCap: global-memory contributions + stable radix sort
    DBuf<int64_t> hrows, hoff, hpos, hsegx;
    DBuf<uint64_t> hkey;
    DBuf<double> hv, hr;
    DBuf<int32_t> ht;
    int64_t M = 0;
    if (nhuge) {
        DBuf<int64_t> flag(static_cast<size_t>(nc), s), num(1, s);
        LAUNCH(k_flag_big, nc, cnt.get(), nc, flag.get());
        hrows.alloc(static_cast<size_t>(nhuge), s);
        thrust::counting_iterator<int64_t> it(0);
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, it, flag.get(), hrows.get(), num.get(), nc, s);
        }, s);
        if (a.nc >= (int64_t(1) << (64 - kHugeColBits)) || nhuge >= (int64_t(1) << (64 - kHugeColBits)))
            fail(PAIRAMG_INTERNAL, "galerkin: too many dense coarse rows");
        hoff.alloc(static_cast<size_t>(nhuge + 1), s);
        LAUNCH(k_huge_len, nhuge + 1, a, hrows.get(), nhuge, hoff.get());
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, hoff.get(), hoff.get(), nhuge + 1, s);
        }, s);
        M = read_one(hoff.get() + nhuge, s);
        DBuf<uint64_t> key0(static_cast<size_t>(M), s);
        DBuf<int64_t> pos0(static_cast<size_t>(M), s);
        hv.alloc(static_cast<size_t>(M), s);
        hr.alloc(static_cast<size_t>(M), s);
        ht.alloc(static_cast<size_t>(M), s);
        k_huge_fill<<<static_cast<int>(std::min<int64_t>(nhuge, 8 * kSmCount)), 256, 0, s>>>(
            a, hrows.get(), nhuge, hoff.get(), key0.get(), pos0.get(), hv.get(), hr.get(), ht.get());
        PB_CHECK_LAUNCH();
        hkey.alloc(static_cast<size_t>(M), s);
        hpos.alloc(static_cast<size_t>(M), s);
        int hb = 0;
        while ((int64_t(1) << hb) <= nhuge) ++hb;
        const int end_bit = kHugeColBits + hb;
        cub_call([&](void* t, size_t& b) {  // stable: equal keys keep encounter order
            return cub::DeviceRadixSort::SortPairs(t, b, key0.get(), hkey.get(), pos0.get(), hpos.get(), M, 0,
                                                   end_bit, s);
        }, s);
        hsegx.alloc(static_cast<size_t>(M), s);
        LAUNCH(k_huge_heads, M, hkey.get(), M, hsegx.get());
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, hsegx.get(), hsegx.get(), M, s);
        }, s);
        int64_t nseg = 0;
        {
            int64_t last = 0;
            uint64_t k1 = 0, k0 = 0;
            PB_CUDA(cudaMemcpyAsync(&last, hsegx.get() + M - 1, 8, cudaMemcpyDeviceToHost, s));
            PB_CUDA(cudaMemcpyAsync(&k1, hkey.get() + M - 1, 8, cudaMemcpyDeviceToHost, s));
            if (M > 1) PB_CUDA(cudaMemcpyAsync(&k0, hkey.get() + M - 2, 8, cudaMemcpyDeviceToHost, s));
            PB_CUDA(cudaStreamSynchronize(s));
            nseg = last + ((M == 1 || k1 != k0) ? 1 : 0);
        }
        LAUNCH(k_huge_count, nhuge, hrows.get(), nhuge, hoff.get(), hsegx.get(), M, nseg, cnt.get());
    }
    orp.alloc(static_cast<size_t>(nc + 1), s);
    cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, cnt.get(), orp.get(), nc + 1, s);
    }, s);
    const int64_t nnz = read_one(orp.get() + nc, s);
    ocol.alloc(static_cast<size_t>(nnz), s);
    oval.alloc(static_cast<size_t>(nnz), s);
    a.orp = orp.get();
    a.ocol = ocol.get();
    a.oval = oval.get();
    if (nc) k_galerkin_warp<true><<<gw, kGalWarps * 32, 0, s>>>(a);
    PB_CHECK_LAUNCH();
    if (nbig) {
        k_galerkin_block<true><<<static_cast<int>(std::min<int64_t>(nbig, 4 * kSmCount)), kGalBigThreads,
                                 big_smem, s>>>(a, big.get(), nbig);
        PB_CHECK_LAUNCH();
    }
    if (M) {  // the huge rows' numeric pass (the warp / block kernels skipped them: overflow)
        LAUNCH(k_huge_fold, M, a, hrows.get(), hoff.get(), hkey.get(), hpos.get(), hv.get(), hr.get(), ht.get(),
               hsegx.get(), M);
    }
    return nnz;
}

// P over A's column slots, overlapped: the owned part and
// the halo exchange of P run on the communication stream as soon as the
// matching is done, while the compute stream builds R, w_next and the
// composed prolongator; extend_p_join makes the compute stream wait and
// books only the exposed wait as spmm_comm.
struct PExt {
    cudaEvent_t done = nullptr;
    bool pending = false;
};

void extend_p_begin(Runtime& rt, DevMatrix& A, const int32_t* pcol, const double* pval, int64_t cbase,
                    DBuf<int64_t>& pc, DBuf<double>& pv, PExt& x) {
    cudaStream_t s = rt.stream(), c = rt.comm_stream();
    const int64_t next = A.n + A.halo.n_halo;
    pc.alloc(static_cast<size_t>(next), s);
    pv.alloc(static_cast<size_t>(next), s);
    cudaEvent_t ready;
    PB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    PB_CUDA(cudaEventRecord(ready, s));  // pcol / pval and the buffers are ready
    PB_CUDA(cudaStreamWaitEvent(c, ready, 0));
    PB_CUDA(cudaEventDestroy(ready));
    if (A.n) {
        k_pext<<<blocks_for(A.n, 256), 256, 0, c>>>(pcol, pval, A.n, cbase, pc.get(), pv.get());
        PB_CHECK_LAUNCH();
    }
    if (A.halo.has_traffic())
        halo_exchange_pair(rt, A.halo, pc.get(), pc.get() + A.n, pv.get(), pv.get() + A.n, c);
    PB_CUDA(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming));
    PB_CUDA(cudaEventRecord(x.done, c));
    x.pending = true;
}

void extend_p_join(Runtime& rt, PExt& x, SetupStats& st) {
    if (!x.pending) return;
    const auto t0 = Clock::now();
    PB_CUDA(cudaEventSynchronize(x.done));
    st.t_spmm_comm += since(t0);
    PB_CUDA(cudaStreamWaitEvent(rt.stream(), x.done, 0));
    PB_CUDA(cudaEventDestroy(x.done));
    x.done = nullptr;
    x.pending = false;
}

// P over A's column slots: owned from (pcol + cbase, pval), halo by exchange.
[[maybe_unused]] void extend_p(Runtime& rt, DevMatrix& A, const int32_t* pcol, const double* pval, int64_t cbase,
                               DBuf<int64_t>& pc, DBuf<double>& pv, SetupStats& st) {
    cudaStream_t s = rt.stream();
    const int64_t next = A.n + A.halo.n_halo;
    pc.alloc(static_cast<size_t>(next), s);
    pv.alloc(static_cast<size_t>(next), s);
    LAUNCH(k_pext, A.n, pcol, pval, A.n, cbase, pc.get(), pv.get());
    if (A.halo.has_traffic()) {
        PB_CUDA(cudaStreamSynchronize(s));
        const auto t0 = Clock::now();
        halo_exchange_pair(rt, A.halo, pc.get(), pc.get() + A.n, pv.get(), pv.get() + A.n, s);
        PB_CUDA(cudaStreamSynchronize(s));
        st.t_spmm_comm += since(t0);
        trace(rt, "P halo exchange", since(t0));
    }
}

}  // namespace

// ------------------------------------------------- coarse replication ---

namespace {

constexpr int kMaxRanks = 64;

struct SegInfo {
    int64_t off[kMaxRanks];
    int64_t cnt[kMaxRanks];
    int64_t max;
    int p;
};

template <typename T>
__global__ void k_unpad(const T* __restrict__ recv, SegInfo si, T* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= si.max * si.p) return;
    const int r = static_cast<int>(t / si.max);
    const int64_t i = t - r * si.max;
    if (i < si.cnt[r]) out[si.off[r] + i] = recv[t];
}

__global__ void k_rowlen(const int64_t* __restrict__ rp, int64_t n, int64_t* __restrict__ len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) len[i] = rp[i + 1] - rp[i];
    if (i == n) len[n] = 0;
}

__global__ void k_to_i32(const int64_t* __restrict__ a, int64_t n, int32_t* __restrict__ b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = static_cast<int32_t>(a[i]);
}

__global__ void k_shift_i32(const int32_t* __restrict__ a, int64_t n, int64_t shift, int32_t* __restrict__ b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = static_cast<int32_t>(a[i] + shift);
}

SegInfo seg_info(const std::vector<int64_t>& counts) {
    if (counts.size() > static_cast<size_t>(kMaxRanks)) fail(PAIRAMG_INVALID_ARGUMENT, "more than 64 ranks");
    SegInfo si{};
    si.p = static_cast<int>(counts.size());
    int64_t off = 0;
    for (int r = 0; r < si.p; ++r) {
        si.off[r] = off;
        si.cnt[r] = counts[r];
        off += counts[r];
        si.max = std::max(si.max, counts[r]);
    }
    return si;
}

// Setup-time allgatherv of a device array (padded allgather + unpad).
template <typename T>
int64_t allgatherv(Runtime& rt, const T* d_local, int64_t count, DBuf<T>& out) {
    cudaStream_t s = rt.stream();
    const std::vector<int64_t> counts = rt.allgather_i64(count);
    const SegInfo si = seg_info(counts);
    const int64_t total = si.off[si.p - 1] + si.cnt[si.p - 1];
    DBuf<T> send(static_cast<size_t>(std::max<int64_t>(si.max, 1)), s), recv(static_cast<size_t>(std::max<int64_t>(si.max * si.p, 1)), s);
    if (count) PB_CUDA(cudaMemcpyAsync(send.get(), d_local, sizeof(T) * count, cudaMemcpyDeviceToDevice, s));
    rt.allgather_dev(send.get(), recv.get(), sizeof(T) * si.max);
    out.alloc(static_cast<size_t>(total), s);
    if (si.max) k_unpad<T><<<blocks_for(si.max * si.p, 256), 256, 0, s>>>(recv.get(), si, out.get());
    PB_CHECK_LAUNCH();
    PB_CUDA(cudaStreamSynchronize(s));
    return total;
}

}  // namespace

void gather_segments(Runtime& rt, const double* d_local, int64_t count, double* sendbuf, double* recvbuf,
                     int64_t maxcount, const std::vector<int64_t>& offsets, const std::vector<int64_t>& counts,
                     double* d_out, cudaStream_t s) {
    SegInfo si = seg_info(counts);
    (void)offsets;
    if (count) PB_CUDA(cudaMemcpyAsync(sendbuf, d_local, 8 * count, cudaMemcpyDeviceToDevice, s));
    rt.allgather_f64(sendbuf, recvbuf, static_cast<size_t>(maxcount), s);
    if (maxcount) k_unpad<double><<<blocks_for(maxcount * si.p, 256), 256, 0, s>>>(recvbuf, si, d_out);
    PB_CHECK_LAUNCH();
}

void replicate_coarse_levels(Runtime& rt, Hierarchy& h, int64_t max_rows, int storage) {
    NvtxRange nv("setup/replicate coarse levels");
    h.rep_level = -1;
    h.rep.clear();
    if (rt.nranks() == 1) return;
    cudaStream_t s = rt.stream();
    // replicate from the first level small in rows AND in nonzeros: a
    // replicated level costs every rank the whole level's sweep, a
    // distributed one a halo exchange per launch (measured at N = 2: the
    // 27-point level 1, 1.8 M rows / 47 M nonzeros, ran 2.3x slower
    // replicated than distributed; 7-point levels of <= 1 M rows, ~7 M
    // nonzeros, are faster replicated)
    int kr = -1;
    for (int k = 1; k < h.nl(); ++k)
        if (h.levels[k]->A.n_global <= max_rows && h.level_nnz[static_cast<size_t>(k)] <= 8 * max_rows) {
            kr = k;
            break;
        }
    if (kr < 0) return;
    for (int k = kr; k < h.nl(); ++k) {
        Level& D = *h.levels[k];
        auto R = std::make_unique<Level>();
        // global CSR (rows in rank order = global order)
        DBuf<int64_t> len(static_cast<size_t>(D.A.n + 1), s), glen;
        LAUNCH(k_rowlen, D.A.n + 1, D.A.rp.get(), D.A.n, len.get());
        const int64_t ng = allgatherv(rt, len.get(), D.A.n, glen);
        DBuf<int64_t> rp(static_cast<size_t>(ng + 1), s);
        PB_CUDA(cudaMemsetAsync(rp.get() + ng, 0, 8, s));
        if (ng) PB_CUDA(cudaMemcpyAsync(rp.get(), glen.get(), 8 * ng, cudaMemcpyDeviceToDevice, s));
        cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, rp.get(), rp.get(), ng + 1, s); }, s);
        DBuf<int64_t> gcol_local(static_cast<size_t>(std::max<int64_t>(D.A.nnz, 1)), s), gcol;
        global_columns(D.A, gcol_local.get(), s);
        DBuf<double> gval;
        const int64_t nnz = allgatherv(rt, gcol_local.get(), D.A.nnz, gcol);
        allgatherv(rt, D.A.val.get(), D.A.nnz, gval);
        R->A.starts = {0, ng};
        R->A.n = ng;
        R->A.n_global = ng;
        R->A.row_begin = 0;
        R->A.nnz = nnz;
        R->A.rp = std::move(rp);
        R->A.col.alloc(static_cast<size_t>(nnz), s);
        LAUNCH(k_to_i32, nnz, gcol.get(), nnz, R->A.col.get());
        R->A.val = std::move(gval);
        R->l1.alloc(static_cast<size_t>(ng), s);
        l1_diagonal(R->A, R->l1.get(), s);
        build_sell(R->A, nullptr, ng, R->sell_all, s, storage, R->l1.get());
        R->x.alloc(static_cast<size_t>(ng), s);
        R->xt.alloc(static_cast<size_t>(ng), s);
        R->x.zero(s);
        R->xt.zero(s);
        R->rhs.alloc(static_cast<size_t>(ng), s);
        R->res.alloc(static_cast<size_t>(ng), s);
        if (k > kr) {  // replicated transfer from the (replicated) finer level
            const Level& Df = *h.levels[k - 1];
            DBuf<int32_t> pg(static_cast<size_t>(std::max<int64_t>(Df.A.n, 1)), s);
            LAUNCH(k_shift_i32, Df.A.n, D.pcol.get(), Df.A.n, D.A.row_begin, pg.get());
            const int64_t nf = allgatherv(rt, pg.get(), Df.A.n, R->pcol);
            allgatherv(rt, D.pval.get(), Df.A.n, R->pval);
            build_R(R->pcol.get(), R->pval.get(), nf, ng, R->rrp, R->rcol, R->rval, s);
        }
        h.rep.push_back(std::move(R));
    }
    h.rep_counts = rt.allgather_i64(h.levels[kr]->A.n);
    h.rep_offsets.assign(h.rep_counts.size(), 0);
    h.rep_max = 0;
    for (size_t r = 0; r < h.rep_counts.size(); ++r) {
        h.rep_offsets[r] = r ? h.rep_offsets[r - 1] + h.rep_counts[r - 1] : 0;
        h.rep_max = std::max(h.rep_max, h.rep_counts[r]);
    }
    h.rep_send.alloc(static_cast<size_t>(std::max<int64_t>(h.rep_max, 1)), s);
    h.rep_recv.alloc(static_cast<size_t>(std::max<int64_t>(h.rep_max * rt.nranks(), 1)), s);
    h.rep_level = kr;
    PB_CUDA(cudaStreamSynchronize(s));
}

// SetupConfig::replay (amg.cpp:182-197): the owned block of a recorded
// global matching, checked as the reference checks it -- a mate outside
// [h_own, k_own) crosses the partition (amg.cpp:187-189), a non-mutual or
// self mate is an invalid matching (build_pairwise_prolongator, amg.cpp:54-57).
static __global__ void k_replay_local(const int64_t* __restrict__ gm, int64_t n, int64_t h_own,
                               int64_t* __restrict__ mate, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t g = gm[i];
    if (g == -1) {
        mate[i] = -1;
    } else if (g < h_own || g >= h_own + n) {
        atomicOr(bad, 1);
        mate[i] = -1;
    } else {
        mate[i] = g - h_own;
    }
}

static __global__ void k_replay_check(const int64_t* __restrict__ mate, int64_t n, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t j = mate[i];
    if (j != -1 && (j == i || mate[j] != i)) atomicOr(bad, 2);
}

static void replay_matching(const SetupConfig& cfg, size_t step, int64_t fine_n, int64_t h_own, int64_t n, int64_t* mate,
                     cudaStream_t s) {
    if (step >= cfg.replay.size()) fail(PAIRAMG_CONTRACT_VIOLATION, "setup: matching trace exhausted");
    if (!cfg.replay[step] || cfg.replay_sizes[step] != fine_n)
        fail(PAIRAMG_CONTRACT_VIOLATION, "setup: replayed matching of step " + std::to_string(step) + " has " +
                                             std::to_string(cfg.replay_sizes[step]) + " entries, the level has " +
                                             std::to_string(fine_n) + " rows");
    if (!n) return;
    DBuf<int64_t> gm(static_cast<size_t>(n), s);
    DBuf<int> bad(1, s);
    bad.zero(s);
    PB_CUDA(cudaMemcpyAsync(gm.get(), cfg.replay[step] + h_own, 8 * n, cudaMemcpyHostToDevice, s));
    LAUNCH(k_replay_local, n, gm.get(), n, h_own, mate, bad.get());
    int hb = 0;
    PB_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (hb & 1) fail(PAIRAMG_CONTRACT_VIOLATION, "setup: replayed matching crosses the rank partition");
    LAUNCH(k_replay_check, n, mate, n, bad.get());
    PB_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, s));
    PB_CUDA(cudaStreamSynchronize(s));
    if (hb & 2) fail(PAIRAMG_CONTRACT_VIOLATION, "build_pairwise_prolongator: invalid matching");
}

void suitor_match_device(const int64_t* rp, const int32_t* col, const double* w, int64_t n, int64_t* mate,
                         cudaStream_t s) {
    DBuf<ull> slot(static_cast<size_t>(2 * n), s);
    slot.zero(s);
    LAUNCH(k_suitor, n, rp, col, w, n, slot.get());
    LAUNCH(k_mate, n, slot.get(), n, mate);
    PB_CUDA(cudaStreamSynchronize(s));
}

void setup_hierarchy(Runtime& rt, Hierarchy& h, std::vector<int64_t> starts, DBuf<int64_t>&& rp,
                     DBuf<int64_t>&& gcol, DBuf<double>&& val, int64_t nnz, const double* d_w0,
                     const SetupConfig& cfg) {
    if (cfg.aggregation_exponent < 1)
        fail(PAIRAMG_INVALID_ARGUMENT, "setup: aggregation exponent must be >= 1");
    if (cfg.max_levels < 1) fail(PAIRAMG_INVALID_ARGUMENT, "setup: max_levels must be >= 1");
    cudaStream_t s = rt.stream();
    const int rank = rt.rank();
    const auto t_start = Clock::now();
    NvtxRange nv_setup("pairamg/setup_hierarchy");
    h = Hierarchy();

    auto L0 = std::make_unique<Level>();
    L0->A.starts = std::move(starts);
    {
        const auto tc = Clock::now();
        localize(rt, L0->A, std::move(rp), std::move(gcol), std::move(val), nnz);
        h.stats.t_spmm_comm += since(tc);
        trace(rt, "localize level 0", since(tc));
    }
    L0->w.alloc(static_cast<size_t>(L0->A.n), s);
    if (d_w0) {
        if (L0->A.n)
            PB_CUDA(cudaMemcpyAsync(L0->w.get(), d_w0, 8 * L0->A.n, cudaMemcpyDeviceToDevice, s));
    } else {
        LAUNCH(k_fill_l, L0->A.n, L0->w.get(), L0->A.n, 1.0);
    }
    h.levels.push_back(std::move(L0));

    size_t trace_step = 0;
    while (h.nl() < cfg.max_levels && h.levels.back()->A.n_global > cfg.coarse_size_target) {
        Level& Lf = *h.levels.back();
        const int level_index = h.nl();
        // A_pair: level matrix for step 0, then owned pairwise products.
        DevMatrix* A_pair = &Lf.A;
        std::unique_ptr<DevMatrix> A_pair_own;
        DBuf<double> w_pair(static_cast<size_t>(Lf.A.n), s);
        if (Lf.A.n) PB_CUDA(cudaMemcpyAsync(w_pair.get(), Lf.w.get(), 8 * Lf.A.n, cudaMemcpyDeviceToDevice, s));
        std::vector<int64_t> part = Lf.A.starts;
        DBuf<int32_t> comp_col;
        DBuf<double> comp_val;
        int nsteps = 0;

        for (int step = 0; step < cfg.aggregation_exponent; ++step) {
            const int64_t fine_n = part.back();
            if (fine_n <= cfg.coarse_size_target) break;
            const int64_t n = A_pair->n;

            // ---- decoupled matching (no communication) ----
            PB_CUDA(cudaStreamSynchronize(s));
            const auto tm = Clock::now();
            nvtxRangePushA("setup/matching");
            const int64_t msg0 = rt.stats().total_messages();
            DBuf<int64_t> mate(static_cast<size_t>(n), s);
            if (!cfg.replay.empty()) {
                replay_matching(cfg, trace_step, fine_n, part[rank], n, mate.get(), s);
            } else {
                DBuf<double> diag(static_cast<size_t>(n), s), gw(static_cast<size_t>(A_pair->nnz), s);
                DBuf<ull> clamped(1, s);
                clamped.zero(s);
                LAUNCH(k_diag, n, A_pair->rp.get(), A_pair->col.get(), A_pair->val.get(), n, diag.get());
                LAUNCH(k_weights, n, A_pair->rp.get(), A_pair->col.get(), A_pair->val.get(), n, w_pair.get(),
                       diag.get(), gw.get(), clamped.get());
                DBuf<ull> slot(static_cast<size_t>(2 * n), s);
                slot.zero(s);
                LAUNCH(k_suitor, n, A_pair->rp.get(), A_pair->col.get(), gw.get(), n, slot.get());
                LAUNCH(k_mate, n, slot.get(), n, mate.get());
            }
            ++trace_step;
            DBuf<int64_t> pos(static_cast<size_t>(n + 1), s);
            LAUNCH(k_leader, n + 1, mate.get(), n, pos.get());
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceScan::ExclusiveSum(t, b, pos.get(), pos.get(), n + 1, s);
            }, s);
            DBuf<int32_t> agg(static_cast<size_t>(n), s);
            DBuf<double> pval(static_cast<size_t>(n), s);
            LAUNCH(k_aggregate, n, mate.get(), pos.get(), w_pair.get(), n, agg.get(), pval.get());
            const int64_t local_aggs = read_one(pos.get() + n, s);
            h.stats.matching_messages += rt.stats().total_messages() - msg0;
            h.stats.t_matching += since(tm);
            nvtxRangePop();
            {
                DBuf<int64_t> gm(static_cast<size_t>(n), s);
                LAUNCH(k_global_mate, n, mate.get(), n, part[rank], gm.get());
                h.matchings.push_back(std::move(gm));
            }

            // ---- coarse partition (allgather_partition, amg.cpp:19-27) ----
            std::vector<int64_t> counts = rt.allgather_i64(local_aggs);
            std::vector<int64_t> cpart(counts.size() + 1, 0);
            for (size_t r = 0; r < counts.size(); ++r) cpart[r + 1] = cpart[r] + counts[r];
            const int64_t coarse_n = cpart.back();
            if (coarse_n == fine_n)
                fail(PAIRAMG_STAGNATION, "setup: coarsening stagnated at level " + std::to_string(level_index) +
                                             " (empty matching)");
            if (static_cast<double>(coarse_n) > 0.9 * static_cast<double>(fine_n))
                h.warnings.push_back("level " + std::to_string(level_index) + " pairwise step " +
                                     std::to_string(step) + " shrank only " +
                                     std::to_string(fine_n - coarse_n) + " of " + std::to_string(fine_n) +
                                     " rows");

            // P's halo exchange in flight (comm stream) during R / w_next / composition
            const bool more = step + 1 < cfg.aggregation_exponent && coarse_n > cfg.coarse_size_target;
            const bool pair_galerkin = more || nsteps == 0;
            DBuf<int64_t> pc;
            DBuf<double> pv;
            PExt px;
            if (pair_galerkin && cfg.setup_overlap)
                extend_p_begin(rt, *A_pair, agg.get(), pval.get(), cpart[rank], pc, pv, px);

            // ---- R, w_next, composition ----
            const auto tg = Clock::now();
            DBuf<int64_t> rrp;
            DBuf<int32_t> rcol;
            DBuf<double> rval;
            build_R(agg.get(), pval.get(), n, local_aggs, rrp, rcol, rval, s);
            DBuf<double> wn(static_cast<size_t>(local_aggs), s);
            LAUNCH(k_wnext, local_aggs, rrp.get(), rcol.get(), rval.get(), w_pair.get(), local_aggs, wn.get());
            if (step == 0) {
                comp_col.alloc(static_cast<size_t>(n), s);
                comp_val.alloc(static_cast<size_t>(n), s);
                if (n) {
                    PB_CUDA(cudaMemcpyAsync(comp_col.get(), agg.get(), 4 * n, cudaMemcpyDeviceToDevice, s));
                    PB_CUDA(cudaMemcpyAsync(comp_val.get(), pval.get(), 8 * n, cudaMemcpyDeviceToDevice, s));
                }
            } else {
                LAUNCH(k_compose, Lf.A.n, comp_col.get(), comp_val.get(), Lf.A.n, agg.get(), pval.get());
            }
            ++nsteps;
            PB_CUDA(cudaStreamSynchronize(s));
            h.stats.t_spmm += since(tg);

            // ---- pairwise Galerkin, only when the next step (or a
            // single-step level) consumes it; the reference discards the
            // last pairwise product of a multi-step level (amg.cpp:261-264).
            if (pair_galerkin) {
                if (px.pending)
                    extend_p_join(rt, px, h.stats);
                else
                    extend_p(rt, *A_pair, agg.get(), pval.get(), cpart[rank], pc, pv, h.stats);
                const auto tp = Clock::now();
                const int64_t msg1 = rt.stats().total_messages();
                DBuf<int64_t> orp, ocol;
                DBuf<double> oval;
                const int64_t onnz = galerkin(*A_pair, pc.get(), pv.get(), rrp.get(), rcol.get(), rval.get(),
                                              local_aggs, orp, ocol, oval, s);
                h.stats.rc_messages += rt.stats().total_messages() - msg1;
                PB_CUDA(cudaStreamSynchronize(s));
                h.stats.t_spmm += since(tp);
                auto An = std::make_unique<DevMatrix>();
                An->starts = cpart;
                const auto tc = Clock::now();
                localize(rt, *An, std::move(orp), std::move(ocol), std::move(oval), onnz);
                h.stats.t_spmm_comm += since(tc);
                trace(rt, "localize pairwise", since(tc));
                A_pair_own = std::move(An);
                A_pair = A_pair_own.get();
            }
            part = cpart;
            w_pair = std::move(wn);
        }
        if (nsteps == 0) break;

        auto Lc = std::make_unique<Level>();
        const int64_t nc_local = part[rank + 1] - part[rank];
        if (nsteps == 1) {
            Lc->A = std::move(*A_pair_own);
        } else {
            DBuf<int64_t> pc;
            DBuf<double> pv;
            PExt px;
            const bool ov = cfg.setup_overlap;
            if (ov) extend_p_begin(rt, Lf.A, comp_col.get(), comp_val.get(), part[rank], pc, pv, px);
            DBuf<int64_t> rrp;
            DBuf<int32_t> rcol;
            DBuf<double> rval;
            build_R(comp_col.get(), comp_val.get(), Lf.A.n, nc_local, rrp, rcol, rval, s);
            if (ov)
                extend_p_join(rt, px, h.stats);
            else
                extend_p(rt, Lf.A, comp_col.get(), comp_val.get(), part[rank], pc, pv, h.stats);
            const auto tp = Clock::now();
            DBuf<int64_t> orp, ocol;
            DBuf<double> oval;
            const int64_t onnz = galerkin(Lf.A, pc.get(), pv.get(), rrp.get(), rcol.get(), rval.get(), nc_local,
                                          orp, ocol, oval, s);
            PB_CUDA(cudaStreamSynchronize(s));
            h.stats.t_spmm += since(tp);
            Lc->A.starts = part;
            const auto tc = Clock::now();
            localize(rt, Lc->A, std::move(orp), std::move(ocol), std::move(oval), onnz);
            h.stats.t_spmm_comm += since(tc);
            trace(rt, "localize composed", since(tc));
        }
        A_pair_own.reset();
        Lc->w = std::move(w_pair);
        Lc->pcol = std::move(comp_col);
        Lc->pval = std::move(comp_val);
        build_R(Lc->pcol.get(), Lc->pval.get(), Lf.A.n, nc_local, Lc->rrp, Lc->rcol, Lc->rval, s);
        h.levels.push_back(std::move(Lc));
    }

    // Smoother data, SELL copies, work vectors (amg.cpp:279-289).
    for (auto& lp : h.levels) {
        Level& L = *lp;
        const int64_t n = L.A.n, next = L.A.n + L.A.halo.n_halo;
        L.l1.alloc(static_cast<size_t>(n), s);
        l1_diagonal(L.A, L.l1.get(), s);
        if (L.A.halo.n_halo > 0) {
            build_sell(L.A, L.A.interior_rows.get(), n - L.A.n_boundary, L.sell_int, s, cfg.storage, L.l1.get());
            // boundary rows: STEN too when the faces' halo offsets nest into
            // one main pattern (slab partitions), else PAT/DICT/PLAIN
            build_sell(L.A, L.A.boundary_rows.get(), L.A.n_boundary, L.sell_bnd, s, cfg.storage, L.l1.get());
            // an interior rank's two faces reach different halo slots: with
            // 27 points their merged pattern has 36 records -> wide STEN for
            // the split launch (boundary blocks take up to 64)
            if (L.sell_bnd.format != Sell::kSten && (cfg.storage < 0 || cfg.storage == Sell::kSten))
                build_sten_wide(L.A, L.A.boundary_rows.get(), L.A.n_boundary, L.sell_bndw, s, L.l1.get());
            // whole level incl. halo columns, for the exchange-then-compute
            // schedule (slab partitions keep constant halo column offsets,
            // so DICT/PAT usually still apply)
            build_sell(L.A, nullptr, n, L.sell_all, s, cfg.storage, L.l1.get());
        } else {
            build_sell(L.A, nullptr, n, L.sell_all, s, cfg.storage, L.l1.get());
        }
        L.x.alloc(static_cast<size_t>(next), s);
        L.xt.alloc(static_cast<size_t>(next), s);
        L.x.zero(s);
        L.xt.zero(s);
        L.rhs.alloc(static_cast<size_t>(n), s);
        L.res.alloc(static_cast<size_t>(n), s);
        h.level_sizes.push_back(L.A.n_global);
        h.level_nnz.push_back(rt.allreduce_sum_i64(L.A.nnz));
    }
    double opc = 0.0;
    for (int64_t z : h.level_nnz) opc += static_cast<double>(z) / static_cast<double>(h.level_nnz[0]);
    h.opc = opc;
    {
        const auto tc = Clock::now();
        replicate_coarse_levels(rt, h, cfg.replicate_rows, cfg.storage);
        h.stats.t_spmm_comm += since(tc);
        trace(rt, "replicate coarse levels", since(tc));
    }
    PB_CUDA(cudaStreamSynchronize(s));
    h.stats.t_total = since(t_start);
}

}  // namespace pb
