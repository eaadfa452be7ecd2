// sell_stenwin.cuh -- STEN row operators with the gathered vector staged in
// shared memory (included by sell.cu after sell_win.cuh / sell_sten.cuh).
//
// Why: the one-row-per-lane STEN kernels reach 0.78-0.80 of HBM bandwidth;
// what is left is memory-level parallelism -- every warp issues its gathers,
// then waits a full DRAM latency.  Here a tile of T consecutive rows needs x
// only in a few contiguous windows (x[tile + lo_k, tile + T + hi_k): 7-point
// 256^3 -> {-65536}, {-256..256}, {+65536}), so one thread streams the
// windows and the tile's r into shared memory with cp.async.bulk (completion
// on an mbarrier), two tiles ahead of the CTA computing from the other stage:
// tens of KB in flight per SM, and the gathers become shared-memory loads.
//
// Arithmetic is unchanged (same main records, masks, CSR-order dadd/dmul
// chain, ddiv_recip epilogue), so every result is bitwise k_sten's.

struct StenWinArgs {
    int row0, nrows, ntiles, T;
    int64_t xlen;
    int nwin;
    int lo[kWinMax], len[kWinMax], soff[kWinMax];
    int r_soff, stage, al_r;
    int base[kStenMax];  // shared-memory index of record k's x for tile row 0
    const uint8_t* pid;
    const double* x;
    double* y;
    const double* r;
    double omega;
};

template <int OP>
__device__ __forceinline__ void stenwin_issue(const StenWinArgs& a, int t, double* st, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int64_t tr0 = static_cast<int64_t>(a.row0) + static_cast<int64_t>(t) * a.T;
    uint32_t bytes = 0;
    for (int k = 0; k < a.nwin; ++k) {
        const int64_t g = tr0 + a.lo[k];
        bytes += win_copy(st + a.soff[k], a.x, g - (g & 1), a.len[k], a.xlen, bar);
    }
    if (OP != kSpmv)
        bytes += win_copy(st + a.r_soff, a.r, tr0 - a.al_r, a.T + 2, static_cast<int64_t>(a.row0) + a.nrows, bar);
    mbar_arrive_tx(bar, bytes);
}

template <int OP, int LL>  // LL = 7 or 27 with the diagonal as record LL/2
__global__ void __launch_bounds__(256) k_stenwin(StenWinArgs a, const __grid_constant__ StenParam p) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t bar[2];
    pdl_begin();  // the copies read x / r written by the predecessor
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockIdx.x < a.ntiles) stenwin_issue<OP>(a, blockIdx.x, smem, &bar[0]);
        if (blockIdx.x + gridDim.x < a.ntiles) stenwin_issue<OP>(a, blockIdx.x + gridDim.x, smem + a.stage, &bar[1]);
    }
    int it = 0;
    for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
        const int s = it & 1;
        mbar_wait(&bar[s], (it >> 1) & 1);
        const double* st = smem + s * a.stage;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = static_cast<int>(threadIdx.x) + h * 256;
            const int sr = t * a.T + i;
            const bool valid = i < a.T && sr < a.nrows;
            const int row = a.row0 + (valid ? sr : 0);
            const int q = valid ? a.pid[row] : 0;
            const uint32_t m = p.pmask[q];
            double sum = 0.0, own = 0.0;
            {
                double xv[LL];
#pragma unroll
                for (int k = 0; k < LL; ++k) xv[k] = st[a.base[k] + i];
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
                own = xv[LL / 2];
            }
            if (!valid) continue;
            if (OP == kSpmv) {
                a.y[row] = sum;
            } else {
                const double ri = st[a.r_soff + a.al_r + i];
                if (OP == kResid) {
                    a.y[row] = dsub(ri, sum);
                } else {
                    const double tt = dsub(ri, sum);
                    a.y[row] = dadd(own, ddiv_recip(a.omega == 1.0 ? tt : dmul(a.omega, tt), p.pdiag[q], p.pinv[q]));
                }
            }
        }
        __syncthreads();  // stage s fully consumed
        if (threadIdx.x == 0 && t + 2 * static_cast<int>(gridDim.x) < a.ntiles)
            stenwin_issue<OP>(a, t + 2 * gridDim.x, smem + s * a.stage, &bar[s]);
    }
}
