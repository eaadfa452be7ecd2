// solve.cu -- the solve path: the symmetric V-cycle (vcycle_apply,
// cycle.cpp:86-112) with l1-Jacobi sweeps (cycle.cpp:37-62), local
// restriction / prolongation (cycle.cpp:64-84), and Notay's flexible CG
// (Alg. 1) with one fused dot-triple reduction and one
// fused four-vector update per iteration.  One whole FCG iteration (all
// levels, halos, reductions) is captured once into a CUDA graph and
// replayed; the host reads 80 bytes of device scalars per iteration for the
// stopping test.
#include <cmath>
#include <cstring>
#include <string>

#include <cstdio>

#include "solver.cuh"

namespace pb {

namespace {

constexpr int kRedThreads = 256;

// x = (omega*r)/d : the zero-start sweep (cycle.cpp:49-53)
__global__ void k_zero_start(const double* r, const double* d,
                             double* x, int64_t n, double omega) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = ddiv(dmul(omega, r[i]), d[i]);
}

// restrict_to_coarse (cycle.cpp:64-75): rc_c = 0.0 + sum R_ci res_i, fine ascending
// The coarse level's zero-start sweep x1 = (omega*rc)/d (cycle.cpp:49-53),
// formed by the restriction that produced rc (one launch and one pass over
// rc and d fewer per level and V-cycle; the same operations, bitwise).
struct RestrictZs {
    double* x = nullptr;  // null: no fused zero start
    const double* d = nullptr;
    double omega = 1.0;
};

__device__ __forceinline__ void restrict_store(double* rc, int64_t c, double s, const RestrictZs& z) {
    rc[c] = s;
    if (z.x) z.x[c] = ddiv(dmul(z.omega, s), z.d[c]);
}

__global__ void k_restrict(const int64_t* rrp, const int32_t* rcol,
                           const double* rval, const double* res,
                           double* rc, int64_t nc, RestrictZs z) {
    pdl_begin();
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    double s = 0.0;
    for (int64_t t = rrp[c]; t < rrp[c + 1]; ++t) s = dadd(s, dmul(rval[t], res[rcol[t]]));
    restrict_store(rc, c, s, z);
}

// prolongate_add (cycle.cpp:77-84): x_i = x_i + p_i * e_agg(i)
__global__ void k_prolong(const int32_t* pcol, const double* pval,
                          const double* e, double* x, int64_t n) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = dadd(x[i], dmul(pval[i], e[pcol[i]]));
}

// Same two operators with the transfer values as byte codes into a table of
// <= 256 distinct values (kernel parameter): 7 fewer bytes per fine row.
struct CodeTab {
    double v[256];
};

__global__ void k_restrict_c(const int64_t* rrp, const int32_t* rcol,
                             const uint8_t* rcode, const __grid_constant__ CodeTab t,
                             const double* res, double* rc, int64_t nc, RestrictZs z) {
    pdl_begin();
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    double s = 0.0;
    for (int64_t k = rrp[c]; k < rrp[c + 1]; ++k) s = dadd(s, dmul(t.v[rcode[k]], res[rcol[k]]));
    restrict_store(rc, c, s, z);
}

__global__ void k_prolong_c(const int32_t* pcol, const uint8_t* pcode,
                            const __grid_constant__ CodeTab t, const double* e, double* x,
                            int64_t n) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = dadd(x[i], dmul(t.v[pcode[i]], e[pcol[i]]));
}

// Four rows per thread with 16-byte loads/stores (x, pcol) and one 4-byte
// pattern load: the four coarse gathers are independent and in flight
// together (the one-row kernel is a load -> gather -> store latency chain).
__global__ void __launch_bounds__(256) k_prolong_c4(const int4* pcol, const uint32_t* pcode,
                                                     const __grid_constant__ CodeTab t, const double* e, double2* x,
                                                     int64_t n4) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n4) return;
    const int4 c = pcol[i];
    const uint32_t k = pcode[i];
    const double e0 = e[c.x], e1 = e[c.y], e2 = e[c.z], e3 = e[c.w];
    double2 a = x[2 * i], b = x[2 * i + 1];
    a.x = dadd(a.x, dmul(t.v[k & 0xFF], e0));
    a.y = dadd(a.y, dmul(t.v[(k >> 8) & 0xFF], e1));
    b.x = dadd(b.x, dmul(t.v[(k >> 16) & 0xFF], e2));
    b.y = dadd(b.y, dmul(t.v[k >> 24], e3));
    x[2 * i] = a;
    x[2 * i + 1] = b;
}

CodeTab code_tab(const std::vector<double>& v) {
    CodeTab t{};
    for (size_t i = 0; i < v.size() && i < 256; ++i) t.v[i] = v[i];
    return t;
}

// FCG vector updates (Alg. 1 lines 16-19), op order shared with the oracle:
//   d = w - c d ; q = v - c q ; u = u + a d ; r = r - a q ;  plus |r|^2 partials.
// ZS: also forms the next V-cycle's level-0 zero-start sweep from the new
// residual, x1 = (omega*r)/d (cycle.cpp:49-53), while r is in registers; d
// is the pattern's l1 diagonal (STEN level 0: one byte per row) or the l1
// array.
template <bool ZS>
__device__ __forceinline__ void zs_store(const ZeroStart& z, int64_t i, double rn) {
    if (!ZS) return;
    if (z.pid) {
        const int q = z.pid[i];
        z.x[i] = ddiv_recip(dmul(z.omega, rn), z.ptab[q], z.pinv[q]);
    } else {
        z.x[i] = ddiv(dmul(z.omega, rn), z.l1[i]);
    }
}

template <bool ZS>
__global__ void __launch_bounds__(kRedThreads)
    k_update(const double* w, double* d, double* u,
             const double* v, double* q, double* r, int64_t n,
             const FcgState* st, double* partials, ZeroStart z) {
    pdl_begin();
    if (st->stop) return;  // multi-rank: r_k already met the stopping test (k_fcg_scalars4)
    const double c = st->c, a = st->a;
    double rr = 0.0;
    // 16-byte vector accesses (all vectors are 256-byte aligned), scalar tail
    const int64_t n2 = n >> 1;
    const double2* w2 = reinterpret_cast<const double2*>(w);
    const double2* v2 = reinterpret_cast<const double2*>(v);
    double2* d2 = reinterpret_cast<double2*>(d);
    double2* q2 = reinterpret_cast<double2*>(q);
    double2* u2 = reinterpret_cast<double2*>(u);
    double2* r2 = reinterpret_cast<double2*>(r);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 wi = __ldcs(w2 + i), vi = __ldcs(v2 + i), di = d2[i], qi = q2[i], ui = u2[i], ri = r2[i];
        double2 dn, qn, un, rn;
        dn.x = dsub(wi.x, dmul(c, di.x));
        dn.y = dsub(wi.y, dmul(c, di.y));
        qn.x = dsub(vi.x, dmul(c, qi.x));
        qn.y = dsub(vi.y, dmul(c, qi.y));
        un.x = dadd(ui.x, dmul(a, dn.x));
        un.y = dadd(ui.y, dmul(a, dn.y));
        rn.x = dsub(ri.x, dmul(a, qn.x));
        rn.y = dsub(ri.y, dmul(a, qn.y));
        d2[i] = dn;
        q2[i] = qn;
        u2[i] = un;
        r2[i] = rn;
        zs_store<ZS>(z, 2 * i, rn.x);
        zs_store<ZS>(z, 2 * i + 1, rn.y);
        rr = dadd(rr, dmul(rn.x, rn.x));
        rr = dadd(rr, dmul(rn.y, rn.y));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t i = n - 1;
        const double dn = dsub(w[i], dmul(c, d[i]));
        const double qn = dsub(v[i], dmul(c, q[i]));
        d[i] = dn;
        q[i] = qn;
        u[i] = dadd(u[i], dmul(a, dn));
        const double rn = dsub(r[i], dmul(a, qn));
        r[i] = rn;
        zs_store<ZS>(z, i, rn);
        rr = dadd(rr, dmul(rn, rn));
    }
    for (int o = 16; o; o >>= 1) rr = dadd(rr, __shfl_down_sync(0xffffffffu, rr, o));
    __shared__ double red[kRedThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = rr;
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int k = 0; k < kRedThreads / 32; ++k) acc = dadd(acc, red[k]);
        partials[blockIdx.x] = acc;
    }
}

__global__ void __launch_bounds__(kRedThreads)
    k_norm_partials(const double* r, int64_t n, double* partials) {
    pdl_begin();
    double rr = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        rr = dadd(rr, dmul(r[i], r[i]));
    for (int o = 16; o; o >>= 1) rr = dadd(rr, __shfl_down_sync(0xffffffffu, rr, o));
    __shared__ double red[kRedThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = rr;
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int k = 0; k < kRedThreads / 32; ++k) acc = dadd(acc, red[k]);
        partials[blockIdx.x] = acc;
    }
}

// Fixed-order reduction of G partial K-tuples into out[K] (one block).
__global__ void __launch_bounds__(kRedThreads)
    k_reduce(const double* partials, int G, int K, double* out) {
    pdl_begin();
    __shared__ double red[kRedThreads];
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int g = threadIdx.x; g < G; g += kRedThreads) s = dadd(s, partials[g * K + k]);
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = kRedThreads / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] = dadd(red[threadIdx.x], red[threadIdx.x + w]);
            __syncthreads();
        }
        if (threadIdx.x == 0) out[k] = red[0];
        __syncthreads();
    }
}

constexpr int kStage = 256;

// First stage for large partial counts: block b reduces the contiguous chunk
// [b*G/gridDim, (b+1)*G/gridDim) of K-tuples in a fixed order.
__global__ void __launch_bounds__(kRedThreads)
    k_reduce_chunks(const double* partials, int G, int K, double* out) {
    pdl_begin();
    __shared__ double red[kRedThreads];
    const int64_t g0 = static_cast<int64_t>(G) * blockIdx.x / gridDim.x;
    const int64_t g1 = static_cast<int64_t>(G) * (blockIdx.x + 1) / gridDim.x;
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int64_t g = g0 + threadIdx.x; g < g1; g += kRedThreads) s = dadd(s, partials[g * K + k]);
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = kRedThreads / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] = dadd(red[threadIdx.x], red[threadIdx.x + w]);
            __syncthreads();
        }
        if (threadIdx.x == 0) out[blockIdx.x * K + k] = red[0];
        __syncthreads();
    }
}

// Cross-rank sums in rank order (runtime.cpp:250-258), then the FCG scalar
// recurrences (Alg. 1 lines 4-5, 14; breakdown check SPEC.md:478).
__global__ void k_fcg_scalars(const double* g, int p, FcgState* st) {
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double al = 0.0, be = 0.0, ga = 0.0;
    for (int r = 0; r < p; ++r) {
        al = dadd(al, g[3 * r + 0]);
        be = dadd(be, g[3 * r + 1]);
        ga = dadd(ga, g[3 * r + 2]);
    }
    st->alpha = al;
    st->beta = be;
    st->gamma = ga;
    double rho_new, c;
    if (st->it == 0) {
        rho_new = be;  // rho_0 = w_0^T v_0
        c = 0.0;       // d_0 = w_0, q_0 = v_0 (d, q start at zero)
    } else {
        rho_new = dsub(be, ddiv(dmul(ga, ga), st->rho));
        c = ddiv(ga, st->rho);
    }
    if (rho_new == 0.0 || !isfinite(rho_new)) st->status = 1;
    st->c = c;
    st->a = ddiv(al, rho_new);
    st->rho = rho_new;
}

// Multi-rank form with ONE cross-rank exchange per iteration (
// SURVEY.md 8c item 2): g holds every rank's (w.r, w.v, w.q, |r_k|^2_local)
// where r_k is the residual this iteration's V-cycle was applied to.  The
// stopping test of r_k is evaluated here, one V-cycle late: when it holds
// (or k = max_iters) the update is skipped (st->stop) and the solve ends with
// u_k -- the same iterate and count as testing right after update k.
__global__ void k_fcg_scalars4(const double* g, int p, FcgState* st, double rtol, int max_iters, double* hist) {
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double al = 0.0, be = 0.0, ga = 0.0, rr = 0.0;
    for (int r = 0; r < p; ++r) {
        al = dadd(al, g[4 * r + 0]);
        be = dadd(be, g[4 * r + 1]);
        ga = dadd(ga, g[4 * r + 2]);
        rr = dadd(rr, g[4 * r + 3]);
    }
    st->rr = rr;
    const double rel = ddiv(__dsqrt_rn(rr), __dsqrt_rn(st->rr0));
    if (hist && st->it <= max_iters) hist[st->it] = rel;
    if (rel < rtol || st->it >= max_iters) {
        st->stop = 1;
        return;
    }
    st->stop = 0;
    st->alpha = al;
    st->beta = be;
    st->gamma = ga;
    double rho_new, c;
    if (st->it == 0) {
        rho_new = be;
        c = 0.0;
    } else {
        rho_new = dsub(be, ddiv(dmul(ga, ga), st->rho));
        c = ddiv(ga, st->rho);
    }
    if (rho_new == 0.0 || !isfinite(rho_new)) st->status = 1;
    st->c = c;
    st->a = ddiv(al, rho_new);
    st->rho = rho_new;
    st->it += 1;  // the update of this iteration runs
}

// Local |r_{k+1}|^2 of the update's block partials into out (no exchange:
// it travels with the next iteration's dot triple).
__global__ void __launch_bounds__(kRedThreads) k_rr_local(const double* partials, int G, double* out) {
    pdl_begin();
    __shared__ double red[kRedThreads];
    double s = 0.0;
    for (int g = threadIdx.x; g < G; g += kRedThreads) s = dadd(s, partials[g]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = dadd(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// Device-side stopping test of the graph loop (same operations as the host
// loop: rel = sqrt(rr)/sqrt(rr0); stop on rel < rtol, max_iters or breakdown).
// Multi-rank loop: k_fcg_scalars4 (same allgathered sums in the same order on
// every rank, so every rank stops after the same iteration) already decided.
__global__ void k_loop_ctl_mr(const FcgState* st, cudaGraphConditionalHandle h) {
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    cudaGraphSetConditional(h, (st->stop || st->status) ? 0u : 1u);
}

__global__ void k_loop_ctl(const FcgState* st, double rtol, int max_iters, double* hist,
                           cudaGraphConditionalHandle h) {
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double rel = ddiv(__dsqrt_rn(st->rr), __dsqrt_rn(st->rr0));
    if (st->it <= max_iters) hist[st->it] = rel;
    const bool stop = st->status != 0 || rel < rtol || st->it >= max_iters;
    cudaGraphSetConditional(h, stop ? 0u : 1u);
}

__global__ void k_norm_final(const double* g, int p, FcgState* st, int init) {
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double rr = 0.0;
    for (int r = 0; r < p; ++r) rr = dadd(rr, g[r]);
    st->rr = rr;
    if (init) {
        st->rr0 = rr;
        st->it = 0;
        st->status = 0;
        st->stop = 0;
        st->rho = 0.0;
    } else {
        st->it += 1;
    }
}

// validate_cycle_config (cycle.cpp:7-13): negative sweep counts are an
// error, pre != post a warning (the preconditioner is then not symmetric).
std::string check_cycle(const CycleConfig& cc) {
    if (cc.pre_sweeps < 0 || cc.post_sweeps < 0 || cc.coarsest_sweeps < 0)
        fail(PAIRAMG_INVALID_ARGUMENT, "cycle config: sweep counts must be >= 0");
    if (cc.pre_sweeps != cc.post_sweeps) return "pre_sweeps != post_sweeps: the V-cycle preconditioner is not symmetric";
    return {};
}

int red_grid(int64_t n) {
    const int64_t want = (n + kRedThreads - 1) / kRedThreads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(kSmCount) * 8)));
}

}  // namespace

Solver::Solver(Runtime& r) : rt(r), s_(r.stream()) {
    // spmv_dist's overlap flag (dist.cpp:128-199): interior rows while the
    // halo is in flight (default, as every reference call site) or exchange first
    overlap = env_flag("PAIRAMG_OVERLAP", true);
    // LOCAL runtimes (thread ranks) exchange solve-path data by P2P stores only
    p2p_ = rt.local() || env_flag("PAIRAMG_P2P", true);
    halo_grid_ = kSmCount * 4;
    PB_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    PB_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    PB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_state_), sizeof(FcgState)));
}

Solver::~Solver() {
    cudaSetDevice(rt.device());
    cudaStreamSynchronize(s_);
    destroy_graph();
    for (auto& v : tev_)
        for (auto& pr : v) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (h_state_) cudaFreeHost(h_state_);
}

void Solver::destroy_graph() {
    if (graph_) cudaGraphExecDestroy(graph_);
    graph_ = nullptr;
    if (loop_graph_) cudaGraphExecDestroy(loop_graph_);
    loop_graph_ = nullptr;
}

// The multi-rank iteration can loop on the device when nothing in it needs
// the host: the dot allgather, every halo exchange and the replicated-level
// gather are P2P kernels (no NCCL call), and the ranks own their GPUs (LOCAL
// ranks sharing one keep the per-iteration launches).
bool Solver::mr_device_loop_ok() const {
    if (rt.shared_device() || !dots_gather_.ok) return false;
    if (h.rep_level >= 0 && !rep_gather_.ok) return false;
    const int nd = h.rep_level >= 0 ? h.rep_level : h.nl();
    for (int k = 0; k < nd; ++k) {
        const Level& L = *h.levels[static_cast<size_t>(k)];
        if (L.A.halo.has_traffic() && !L.p2p.ok) return false;
    }
    return true;
}

void Solver::ensure_loop_graph(const CycleConfig& cc, bool precflag, double rtol, int max_iters) {
    if (loop_graph_ && loop_cc_.pre_sweeps == cc.pre_sweeps && loop_cc_.post_sweeps == cc.post_sweeps &&
        loop_cc_.coarsest_sweeps == cc.coarsest_sweeps && loop_cc_.relax_weight == cc.relax_weight &&
        loop_prec_ == precflag && loop_rtol_ == rtol && loop_maxit_ == max_iters)
        return;
    if (loop_graph_) cudaGraphExecDestroy(loop_graph_);
    loop_graph_ = nullptr;
    // (multi-rank: preallocated by solve(); the per-iteration graph writes it too)
    if (hist_.size() < static_cast<size_t>(max_iters) + 1) hist_.alloc(static_cast<size_t>(max_iters) + 1, s_);
    cudaGraph_t g;
    PB_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle handle;
    PB_CUDA(cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    PB_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    const int64_t l0 = launches_;
    PB_CUDA(cudaStreamBeginCaptureToGraph(s_, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    iteration_enqueue(cc, precflag);
    if (rt.nranks() > 1)
        launch_k(k_loop_ctl_mr, 1, 32, 0, s_, state_.get(), handle);
    else
        launch_k(k_loop_ctl, 1, 32, 0, s_, state_.get(), rtol, max_iters, hist_.get(), handle);
    PB_CHECK_LAUNCH();
    PB_CUDA(cudaStreamEndCapture(s_, &body));
    launches_ = l0;
    PB_CUDA(cudaGraphInstantiate(&loop_graph_, g, 0));
    PB_CUDA(cudaGraphDestroy(g));
    loop_cc_ = cc;
    loop_prec_ = precflag;
    loop_rtol_ = rtol;
    loop_maxit_ = max_iters;
}

void Solver::setup(std::vector<int64_t> starts, DBuf<int64_t>&& rp, DBuf<int64_t>&& col, DBuf<double>&& val,
                   int64_t nnz, const double* d_w0, const SetupConfig& cfg) {
    destroy_graph();
    ready = false;
    if (rt.nranks() > 1 && h.nl() > 0) {
        // collective teardown of the previous hierarchy's peer mappings: every
        // rank closes what it imported, then (barrier) the exporters free
        PB_CUDA(cudaStreamSynchronize(s_));
        for (auto& L : h.levels) p2p_close_imports(L->p2p);
        p2p_seg_close_imports(rep_gather_);
        rt.barrier();
        p2p_seg_destroy(rep_gather_);
    }
    setup_hierarchy(rt, h, std::move(starts), std::move(rp), std::move(col), std::move(val), nnz, d_w0, cfg);

    if (rt.nranks() > 1 && p2p_)
        p2p_gather_setup(rt, dots_gather_, 4, s_);  // collective
    if (rt.nranks() > 1 && p2p_) {  // collective: every rank, every distributed level
        const int nd = h.rep_level >= 0 ? h.rep_level : h.nl();
        for (int k = 0; k < nd; ++k) p2p_setup(rt, h.levels[static_cast<size_t>(k)]->A.halo, h.levels[static_cast<size_t>(k)]->p2p, s_);
    }
    p2p_seg_destroy(rep_gather_);
    if (rt.nranks() > 1 && h.rep_level >= 0 && p2p_)
        p2p_seg_setup(rt, rep_gather_, h.rep[0]->A.n, s_);  // collective
    {  // byte codes of the transfer values (<= 256 distinct per level)
        auto codes = [&](Level& L) {
            if (L.pval.empty()) return;
            build_value_codes(L.pval.get(), static_cast<int64_t>(L.pval.size()), L.pcode, L.ptab, s_);
            build_value_codes(L.rval.get(), static_cast<int64_t>(L.rval.size()), L.rcode, L.rtab, s_);
        };
        for (int k = 1; k < h.nl(); ++k) codes(*h.levels[k]);
        for (auto& R : h.rep) codes(*R);
    }
    ensure_vectors();
    ready = true;
    if (env_flag("PAIRAMG_VERBOSE", false)) {  // per-level solve storage (stderr)
        static const char* fmt[] = {"plain", "dict", "pat", "sten", "coded", "?", "?", "?"};
        auto desc = [&](const Sell& S) {
            char b[96];
            std::snprintf(b, sizeof b, "%s(rows %lld, L %d, pat %d)", fmt[S.format & 7],
                          static_cast<long long>(S.nrows), S.sten_L, S.npat);
            return std::string(b);
        };
        for (int k = 0; k < h.nl(); ++k) {
            Level& L = lvl(k);
            const bool rep = h.rep_level >= 0 && k >= h.rep_level;
            std::fprintf(stderr, "rank %d level %d %s rows %lld halo %lld p2p %d: %s%s%s\n", rt.rank(), k,
                         rep ? "replicated" : "distributed", static_cast<long long>(L.A.n),
                         static_cast<long long>(L.A.halo.n_halo), L.p2p.ok ? 1 : 0,
                         L.A.halo.n_halo > 0 ? ("int " + desc(L.sell_int) + " bnd " + desc(L.sell_bnd) +
                                                (L.sell_bndw.format == Sell::kSten ? " bnd-wide " + desc(L.sell_bndw) : "") + " all ").c_str() : "",
                         desc(L.sell_all).c_str(), L.pcode.empty() ? "" : " pcode");
        }
    }
}

void Solver::ensure_vectors() {
    Level& L0 = *h.levels[0];
    n_ = L0.A.n;
    next_ = L0.A.n + L0.A.halo.n_halo;
    u_.alloc(static_cast<size_t>(next_), s_);
    r_.alloc(static_cast<size_t>(n_), s_);
    w_.alloc(static_cast<size_t>(next_), s_);
    v_.alloc(static_cast<size_t>(n_), s_);
    d_.alloc(static_cast<size_t>(n_), s_);
    q_.alloc(static_cast<size_t>(n_), s_);
    // partial triples of the SpMV+dots launches (interior + boundary, one
    // block per 8 slices) and of the grid-stride reductions
    // (overlapped schedule: interior + boundary partials; exchange-then-compute: sell_all)
    int64_t dots_blocks = sell_dots_grid(L0.sell_all);
    if (L0.A.halo.n_halo > 0) {
        dots_blocks = std::max<int64_t>(dots_blocks, int64_t(sell_dots_grid(L0.sell_int)) + sell_dots_grid(L0.sell_bnd));
        if (sell_split_ok(L0.sell_int, L0.split_bnd()))
            dots_blocks = std::max<int64_t>(dots_blocks, sell_split_dots_grid(L0.sell_int, L0.split_bnd()));
    }
    max_blocks_ = static_cast<int>(std::max<int64_t>(dots_blocks, kSmCount * 8));
    partials_.alloc(static_cast<size_t>(3 * max_blocks_), s_);
    stage_.alloc(static_cast<size_t>(3 * kStage), s_);
    local_.alloc(8, s_);
    gathered_.alloc(static_cast<size_t>(4 * rt.nranks()), s_);
    state_.alloc(1, s_);
    u_.zero(s_);
    w_.zero(s_);
}

void Solver::ensure_events(int kc, int idx) {
    while (static_cast<int>(tev_[kc].size()) <= idx) {
        cudaEvent_t a, b;
        PB_CUDA(cudaEventCreate(&a));
        PB_CUDA(cudaEventCreate(&b));
        tev_[kc].push_back({a, b});
    }
}

static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st;
    PB_CUDA(cudaStreamIsCapturing(s, &st));
    return st == cudaStreamCaptureStatusActive;
}

void Solver::begin_time(int kc) {
    if (!timing || kc < 0) return;
    const int idx = tcount_[kc];
    ensure_events(kc, idx);
    topen_[kc] = idx;
    if (capturing(s_))
        PB_CUDA(cudaEventRecordWithFlags(tev_[kc][idx].first, s_, cudaEventRecordExternal));
    else
        PB_CUDA(cudaEventRecord(tev_[kc][idx].first, s_));
}

void Solver::end_time(int kc) {
    if (!timing || kc < 0) return;
    const int idx = topen_[kc];
    if (capturing(s_))
        PB_CUDA(cudaEventRecordWithFlags(tev_[kc][idx].second, s_, cudaEventRecordExternal));
    else
        PB_CUDA(cudaEventRecord(tev_[kc][idx].second, s_));
    tcount_[kc] = idx + 1;
}

void Solver::collect_times() {
    if (!timing) return;
    for (int kc = 0; kc < kNumClasses; ++kc)
        for (int i = 0; i < tcount_[kc]; ++i) {
            float ms = 0.f;
            PB_CUDA(cudaEventElapsedTime(&ms, tev_[kc][i].first, tev_[kc][i].second));
            ktime[kc].ms += ms;
            ktime[kc].launches += 1;
        }
}

Level& Solver::lvl(int k) {
    return (h.rep_level >= 0 && k >= h.rep_level) ? *h.rep[static_cast<size_t>(k - h.rep_level)] : *h.levels[k];
}

void Solver::apply(int k, const SellOpArgs& o, int kc) { apply_on(lvl(k), o, kc); }

// Halo of x (owned -> slots [n, n + n_halo)): NVLink direct stores when the
// level's P2P plan is up, else NCCL send/recv.
void Solver::exchange(Level& L, const double* x, cudaStream_t st) {
    double* halo = const_cast<double*>(x) + L.A.n;
    if (L.p2p.ok) {
        p2p_exchange(L.A.halo, L.p2p, x, halo, st);
        rt.stats().halo_exchanges += 1;
        rt.stats().halo_bytes += 8 * L.A.halo.n_halo;
    }
    else
        halo_exchange(rt, L.A.halo, x, halo, st);
}

// One launch for interior + boundary rows whose boundary blocks wait for the
// neighbours' pushes.  Not when ranks share a GPU (LOCAL runtime): a grid
// whose last blocks wait on a peer's kernel could hold every SM slot.
// Interior rows that run the 27-point marching kernels keep them inside the
// split launch (k_sten_march_split; the level-0 sweep at N = 2: 74 us vs
// 81.9 with the exchange on the communication stream).
bool Solver::split_launch(const Level& L) const {
    return L.p2p.ok && L.A.halo.n_halo > 0 && sell_split_ok(L.sell_int, L.split_bnd()) && !rt.shared_device();
}

int Solver::interior_cap(const Level& L) const { return sell_march_ok(L.sell_int) ? 0 : halo_grid_; }

void Solver::apply_on(Level& L, const SellOpArgs& o, int kc) {
    begin_time(kc);
    if (L.A.halo.has_traffic() && !overlap) {
        // exchange first (on the compute stream), then one kernel over all rows
        exchange(L, o.x, s_);
        sell_apply(L.sell_all, o, s_);
        launches_ += 1 + (L.A.halo.send_off.back() ? 1 : 0);
        end_time(kc);
        return;
    }
    if (split_launch(L)) {
        // push this rank's boundary values into the neighbours, then one
        // launch whose boundary blocks wait for theirs (no comm stream)
        const HaloSrc hs = p2p_halo_src(L.A.halo, L.p2p);
        rt.stats().halo_exchanges += 1;
        rt.stats().halo_bytes += 8 * L.A.halo.n_halo;
        if (!hs.fused) p2p_push(L.A.halo, L.p2p, o.x, s_);
        sell_apply_split(L.sell_int, L.split_bnd(), o, hs, s_);
        launches_ += hs.fused ? 1 : 2;
        end_time(kc);
        return;
    }
    if (L.A.halo.has_traffic()) {
        // The boundary rows run on the (high-priority) communication stream
        // right behind the halo receive, concurrently with the interior rows:
        // the compute stream only joins at the end, no second launch on it.
        PB_CUDA(cudaEventRecord(ev_fork_, s_));
        PB_CUDA(cudaStreamWaitEvent(rt.comm_stream(), ev_fork_, 0));
        exchange(L, o.x, rt.comm_stream());
        if (L.A.halo.n_halo > 0) {
            sell_apply(L.sell_bnd, o, rt.comm_stream());
            launches_ += 1;
        }
        PB_CUDA(cudaEventRecord(ev_join_, rt.comm_stream()));
        launches_ += L.A.halo.send_off.back() ? 1 : 0;
    }
    if (L.A.halo.n_halo > 0) {
        // capped grid: the interior kernel leaves SM slots to the pack/NCCL/
        // boundary kernels (else they only run once every interior CTA has
        // been dispatched; measured: halo done at 91 us of an 89 us interior)
        SellOpArgs oi = o;
        oi.max_grid = interior_cap(L);
        sell_apply(L.sell_int, oi, s_);
        PB_CUDA(cudaStreamWaitEvent(s_, ev_join_, 0));
        launches_ += 1;
    } else {
        if (L.A.halo.has_traffic()) PB_CUDA(cudaStreamWaitEvent(s_, ev_join_, 0));
        sell_apply(L.sell_all, o, s_);
        launches_ += 1;
    }
    end_time(kc);
}

static SellOpArgs jacobi_args(int op, const double* x, double* y, const double* rhs, const double* d, double omega) {
    SellOpArgs o;
    o.op = op;
    o.x = x;
    o.y = y;
    o.r = rhs;
    o.d = d;
    o.omega = omega;
    return o;
}

void Solver::smooth(int k, bool zero_start, int nu, const double* rhs, double*& xc, double*& xo, double omega,
                    bool l0) {
    Level& L = lvl(k);
    const int64_t n = L.A.n;
    if (nu == 0) {
        if (zero_start && n) PB_CUDA(cudaMemsetAsync(xc, 0, 8 * n, s_));
        return;
    }
    int sweep = 0;
    if (zero_start && k == 0 && zs_pending_) {  // x1 already formed by the previous update / the solve prologue
        zs_pending_ = false;
        sweep = 1;
    } else if (zero_start && k == zs_level_) {  // x1 formed by the restriction into this level
        zs_level_ = -1;
        sweep = 1;
    } else if (zero_start) {
        begin_time(-1);
        if (n) launch_k<4>(k_zero_start, blocks_for(n, 256), 256, 0, s_, rhs, L.l1.get(), xc, n, omega);
        PB_CHECK_LAUNCH();
        launches_ += 1;
        sweep = 1;
    }
    for (; sweep < nu; ++sweep) {
        apply(k, jacobi_args(kJacobi, xc, xo, rhs, L.l1.get(), omega), l0 ? 0 : -1);
        std::swap(xc, xo);
    }
}

void Solver::vcycle_enqueue(int k, const double* rhs, double*& out, const CycleConfig& cc) {
    Level& L = lvl(k);
    double* xc = L.x.get();
    double* xo = L.xt.get();
    const bool l0 = k == 0;
    const int lc = k < kTimedLevels ? kLevelClass + k : -1;
    begin_time(lc);
    if (k == h.nl() - 1) {
        if (!L.A.halo.has_traffic() && !(k == 0 && zs_pending_) &&
            sell_coarse_solve(L.sell_all, rhs, xc, cc.coarsest_sweeps, cc.relax_weight, s_)) {
            launches_ += 1;
        } else {
            smooth(k, true, cc.coarsest_sweeps, rhs, xc, xo, cc.relax_weight, l0);
        }
        end_time(lc);
        out = xc;
        return;
    }
    smooth(k, true, cc.pre_sweeps, rhs, xc, xo, cc.relax_weight, l0);
    {
        SellOpArgs o;
        o.op = kResid;
        o.x = xc;
        o.y = L.res.get();
        o.r = rhs;
        apply(k, o, l0 ? 1 : -1);
    }
    // T holds the transfer operators into level k+1 (the distributed owned
    // blocks when level k+1 is the first replicated level), C its vectors.
    const bool gather = h.rep_level >= 0 && k + 1 == h.rep_level;
    Level& T = gather ? *h.levels[k + 1] : lvl(k + 1);
    Level& C = lvl(k + 1);
    RestrictZs zs;
    if (!gather && k + 1 < h.nl() - 1 && cc.pre_sweeps >= 1) {  // level k+1 starts with a zero-start sweep
        zs.x = C.x.get();
        zs.d = C.l1.get();
        zs.omega = cc.relax_weight;
        zs_level_ = k + 1;
    }
    if (T.A.n && !T.rcode.empty())
        launch_k<4>(k_restrict_c, blocks_for(T.A.n, 256), 256, 0, s_, T.rrp.get(), T.rcol.get(), T.rcode.get(),
                                                             code_tab(T.rtab), L.res.get(), T.rhs.get(), T.A.n, zs);
    else if (T.A.n)
        launch_k<4>(k_restrict, blocks_for(T.A.n, 256), 256, 0, s_, T.rrp.get(), T.rcol.get(), T.rval.get(), L.res.get(),
                                                           T.rhs.get(), T.A.n, zs);
    PB_CHECK_LAUNCH();
    launches_ += 1;
    const double* crhs = C.rhs.get();
    if (gather) {  // the replicated level's right-hand side: every rank's segment to every rank
        rt.stats().halo_exchanges += 1;
        rt.stats().halo_bytes += 8 * (C.A.n - T.A.n);
    }
    if (gather && rep_gather_.ok) {  // NVLink stores of the restricted rhs into every rank's copy
        p2p_seg_gather(rep_gather_, T.rhs.get(), T.A.n, h.rep_offsets[static_cast<size_t>(rt.rank())], s_);
        crhs = rep_gather_.buf;
        launches_ += 1;
    } else if (gather) {  // one padded allgather of the restricted rhs, then redundant coarse levels
        gather_segments(rt, T.rhs.get(), T.A.n, h.rep_send.get(), h.rep_recv.get(), h.rep_max, h.rep_offsets,
                        h.rep_counts, C.rhs.get(), s_);
        launches_ += 2;
    }
    double* e = nullptr;
    end_time(lc);
    vcycle_enqueue(k + 1, crhs, e, cc);
    begin_time(lc);
    if (gather) e += h.rep_offsets[static_cast<size_t>(rt.rank())];
    {
        const bool v4 = L.A.n >= 4 && (reinterpret_cast<uintptr_t>(xc) & 15) == 0;  // 16-byte aligned buffers
        if (L.A.n && !T.pcode.empty() && v4) {
            const int64_t n4 = L.A.n / 4;  // the < 4 tail rows by the scalar kernel
            launch_k<4>(k_prolong_c4, blocks_for(n4, 256), 256, 0, s_, reinterpret_cast<const int4*>(T.pcol.get()),
                        reinterpret_cast<const uint32_t*>(T.pcode.get()), code_tab(T.ptab), e,
                        reinterpret_cast<double2*>(xc), n4);
            if (L.A.n % 4) {
                launch_k<4>(k_prolong_c, 1, 32, 0, s_, T.pcol.get() + 4 * n4, T.pcode.get() + 4 * n4, code_tab(T.ptab),
                            e, xc + 4 * n4, L.A.n - 4 * n4);
                launches_ += 1;
            }
        } else if (L.A.n && !T.pcode.empty())
            launch_k<4>(k_prolong_c, blocks_for(L.A.n, 256), 256, 0, s_, T.pcol.get(), T.pcode.get(), code_tab(T.ptab), e, xc,
                                                                L.A.n);
        else if (L.A.n)
            launch_k<4>(k_prolong, blocks_for(L.A.n, 256), 256, 0, s_, T.pcol.get(), T.pval.get(), e, xc, L.A.n);
        PB_CHECK_LAUNCH();
        launches_ += 1;
    }
    smooth(k, false, cc.post_sweeps, rhs, xc, xo, cc.relax_weight, l0);
    end_time(lc);
    out = xc;
}

void Solver::reduce_dots_enqueue(bool fused_norm) {
    const int p = rt.nranks();
    // partial count G is encoded by the producer; it is fixed for the level
    const int G = dots_grid_;  // partial triples written by the SpMV+dots launches
    if (G > kStage) {  // two fixed-order stages: kStage blocks over contiguous chunks, then one block
        launch_k(k_reduce_chunks, kStage, kRedThreads, 0, s_, partials_.get(), G, 3, stage_.get());
        PB_CHECK_LAUNCH();
        launch_k(k_reduce, 1, kRedThreads, 0, s_, stage_.get(), kStage, 3, local_.get());
        launches_ += 1;
    } else {
        launch_k(k_reduce, 1, kRedThreads, 0, s_, partials_.get(), G, 3, local_.get());
    }
    PB_CHECK_LAUNCH();
    const double* g = local_.get();
    const int K = fused_norm ? 4 : 3;  // local_[3] = |r_k|^2 of this rank (k_rr_local / prologue)
    if (p > 1) {
        rt.stats().device_reductions += 1;
        if (dots_gather_.ok)
            p2p_allgather(dots_gather_, local_.get(), gathered_.get(), K, s_);
        else
            rt.allgather_f64(local_.get(), gathered_.get(), static_cast<size_t>(K), s_);
        g = gathered_.get();
        launches_ += 1;
    }
    if (fused_norm)
        launch_k(k_fcg_scalars4, 1, 32, 0, s_, g, p, state_.get(), cap_rtol_, cap_maxit_, hist_.get());
    else
        launch_k(k_fcg_scalars, 1, 32, 0, s_, g, p, state_.get());
    PB_CHECK_LAUNCH();
    launches_ += 2;
}

void Solver::reduce_norm_enqueue(bool init) {
    const int p = rt.nranks();
    launch_k(k_reduce, 1, kRedThreads, 0, s_, partials_.get(), red_grid(n_), 1, local_.get() + 3);
    PB_CHECK_LAUNCH();
    const double* g = local_.get() + 3;
    if (p > 1) {
        rt.stats().device_reductions += 1;
        if (dots_gather_.ok)
            p2p_allgather(dots_gather_, local_.get() + 3, gathered_.get() + 3 * p, 1, s_);
        else
            rt.allgather_f64(local_.get() + 3, gathered_.get() + 3 * p, 1, s_);
        g = gathered_.get() + 3 * p;
    }
    launch_k(k_norm_final, 1, 32, 0, s_, g, p, state_.get(), init ? 1 : 0);
    PB_CHECK_LAUNCH();
    launches_ += 2;
}

// The level-0 zero-start sweep of every V-cycle is formed by the FCG update
// that produced its right-hand side (and by the solve prologue for the first).
bool Solver::zs_fused(const CycleConfig& cc, bool precflag) {
    const int nu0 = h.nl() == 1 ? cc.coarsest_sweeps : cc.pre_sweeps;
    return precflag && nu0 >= 1;
}

ZeroStart Solver::zero_start_args(const CycleConfig& cc) {
    Level& L0 = *h.levels[0];
    ZeroStart z{};
    z.x = L0.x.get();
    z.omega = cc.relax_weight;
    const Sell& S = L0.sell_all;
    // the pattern id of every owned row names its l1 diagonal (pdiag), halo
    // or not: 1 B per row instead of the 8 B l1 stream
    if (S.format == Sell::kSten && S.nrows == L0.A.n && S.rows.empty() && S.row0 == 0) {
        z.pid = S.pid.get();
        z.ptab = S.pdiag.get();
        z.pinv = S.pinv.get();
    } else {
        z.l1 = L0.l1.get();
    }
    return z;
}

void Solver::iteration_enqueue(const CycleConfig& cc, bool precflag) {
    Level& L0 = *h.levels[0];
    double* w = nullptr;
    const bool zs = zs_fused(cc, precflag);
    zs_pending_ = zs;
    if (precflag) {
        vcycle_enqueue(0, r_.get(), w, cc);
    } else {
        if (n_) PB_CUDA(cudaMemcpyAsync(w_.get(), r_.get(), 8 * n_, cudaMemcpyDeviceToDevice, s_));
        w = w_.get();
    }
    w_out_ = w;
    // v = A w and the dot triple (Alg. 1 lines 10-13)
    begin_time(2);
    if (L0.A.halo.has_traffic() && !overlap) {
        exchange(L0, w, s_);
        dots_grid_ = sell_spmv_dots(L0.sell_all, w, v_.get(), r_.get(), q_.get(), partials_.get(), max_blocks_, s_);
        launches_ += 2;
    } else if (split_launch(L0)) {
        const HaloSrc hs = p2p_halo_src(L0.A.halo, L0.p2p);
        rt.stats().halo_exchanges += 1;
        rt.stats().halo_bytes += 8 * L0.A.halo.n_halo;
        if (!hs.fused) p2p_push(L0.A.halo, L0.p2p, w, s_);
        dots_grid_ = sell_spmv_dots_split(L0.sell_int, L0.split_bnd(), w, v_.get(), r_.get(), q_.get(), partials_.get(),
                                          max_blocks_, hs, s_);
        launches_ += hs.fused ? 1 : 2;
    } else if (L0.A.halo.n_halo > 0) {  // boundary rows behind the halo, on the comm stream
        const int g1 = sell_dots_grid(L0.sell_int, interior_cap(L0));
        PB_CUDA(cudaEventRecord(ev_fork_, s_));
        PB_CUDA(cudaStreamWaitEvent(rt.comm_stream(), ev_fork_, 0));
        exchange(L0, w, rt.comm_stream());
        const int g2 = sell_spmv_dots(L0.sell_bnd, w, v_.get(), r_.get(), q_.get(), partials_.get() + 3 * g1,
                                      max_blocks_ - g1, rt.comm_stream());
        PB_CUDA(cudaEventRecord(ev_join_, rt.comm_stream()));
        const int g1b = sell_spmv_dots(L0.sell_int, w, v_.get(), r_.get(), q_.get(), partials_.get(), g1, s_,
                                       interior_cap(L0));
        if (g1b != g1) fail(PAIRAMG_INTERNAL, "spmv+dots: interior partial count changed");
        PB_CUDA(cudaStreamWaitEvent(s_, ev_join_, 0));
        dots_grid_ = g1 + g2;
        launches_ += 3;
    } else if (L0.A.halo.has_traffic()) {  // halo of w in flight while the interior rows run
        PB_CUDA(cudaEventRecord(ev_fork_, s_));
        PB_CUDA(cudaStreamWaitEvent(rt.comm_stream(), ev_fork_, 0));
        exchange(L0, w, rt.comm_stream());
        PB_CUDA(cudaEventRecord(ev_join_, rt.comm_stream()));
        launches_ += 1;
    }
    if ((L0.A.halo.has_traffic() && !overlap) || L0.A.halo.n_halo > 0) {
        // done above
    } else {
        if (L0.A.halo.has_traffic()) PB_CUDA(cudaStreamWaitEvent(s_, ev_join_, 0));
        dots_grid_ = sell_spmv_dots(L0.sell_all, w, v_.get(), r_.get(), q_.get(), partials_.get(), max_blocks_, s_);
        launches_ += 1;
    }
    end_time(2);
    const bool fused_norm = rt.nranks() > 1;
    reduce_dots_enqueue(fused_norm);
    begin_time(3);
    zs_pending_ = false;
    if (zs)
        launch_k<8>(k_update<true>, red_grid(n_), kRedThreads, 0, s_, w, d_.get(), u_.get(), v_.get(), q_.get(), r_.get(),
                                                              n_, state_.get(), partials_.get(), zero_start_args(cc));
    else
        launch_k<8>(k_update<false>, red_grid(n_), kRedThreads, 0, s_, w, d_.get(), u_.get(), v_.get(), q_.get(), r_.get(),
                                                               n_, state_.get(), partials_.get(), ZeroStart{});
    PB_CHECK_LAUNCH();
    end_time(3);
    launches_ += 1;
    if (fused_norm) {
        launch_k(k_rr_local, 1, kRedThreads, 0, s_, partials_.get(), red_grid(n_), local_.get() + 3);
        PB_CHECK_LAUNCH();
        launches_ += 1;
    } else {
        reduce_norm_enqueue(false);
    }
}

void Solver::solve(const double* d_b, double* d_u, const CycleConfig& cc, double rtol, int max_iters,
                   bool precflag, pairamg_solve_stats* st) {
    NvtxRange nv("pairamg/solve");
    if (!ready) fail(PAIRAMG_CONTRACT_VIOLATION, "solve: setup not run");
    if (rtol <= 0.0 || max_iters < 1) fail(PAIRAMG_INVALID_ARGUMENT, "solve: need rtol > 0 and max_iters >= 1");
    cycle_warning = check_cycle(cc);
    if (rt.nranks() > 1 && hist_.size() < static_cast<size_t>(max_iters) + 1) {
        destroy_graph();  // the multi-rank iteration graph writes the history (k_fcg_scalars4)
        hist_.alloc(static_cast<size_t>(max_iters) + 1, s_);
    }
    shared_gpu_fence();
    Level& L0 = *h.levels[0];
    for (auto& kt : ktime) kt = KernelClassTiming{};
    // Algorithmic bytes per level-0 launch of the stored format (matrix
    // entries once + every vector once; gathers counted once).
    const double n0 = static_cast<double>(n_);
    const double mat = L0.A.halo.n_halo > 0 ? sell_bytes(L0.sell_int) + sell_bytes(L0.sell_bnd)
                                            : sell_bytes(L0.sell_all);
    auto op_bytes = [&](int op) {
        return L0.A.halo.n_halo > 0 ? sell_op_bytes(L0.sell_int, op) + sell_op_bytes(L0.sell_bnd, op)
                                    : sell_op_bytes(L0.sell_all, op);
    };
    ktime[0].bytes_per_launch = op_bytes(kJacobi);            // x, r, (d) read; y written
    ktime[1].bytes_per_launch = op_bytes(kResid);             // x, r read; y written
    ktime[2].bytes_per_launch = op_bytes(-1);                 // w, r, q read; v written
    // 6 vectors read, 4 written; + the fused zero-start: pattern byte (or l1) read, x1 written
    const bool zs = zs_fused(cc, precflag);
    ktime[3].bytes_per_launch = (80.0 + (zs ? (zero_start_args(cc).pid ? 9.0 : 16.0) : 0.0)) * n0;

    cudaEvent_t e0, e1;
    PB_CUDA(cudaEventCreate(&e0));
    PB_CUDA(cudaEventCreate(&e1));
    PB_CUDA(cudaEventRecord(e0, s_));
    launches_ = 0;
    // u0, d = q = 0, r0 = b - A u0, |r0|^2
    if (n_) {
        PB_CUDA(cudaMemcpyAsync(u_.get(), d_u, 8 * n_, cudaMemcpyDeviceToDevice, s_));
        PB_CUDA(cudaMemsetAsync(d_.get(), 0, 8 * n_, s_));
        PB_CUDA(cudaMemsetAsync(q_.get(), 0, 8 * n_, s_));
    }
    const bool timing_save = timing;
    timing = false;
    {
        SellOpArgs o;
        o.op = kResid;
        o.x = u_.get();
        o.y = r_.get();
        o.r = d_b;
        apply(0, o, -1);
    }
    launch_k(k_norm_partials, red_grid(n_), kRedThreads, 0, s_, r_.get(), n_, partials_.get());
    PB_CHECK_LAUNCH();
    launches_ += 1;
    reduce_norm_enqueue(true);
    if (zs_fused(cc, precflag) && n_) {
        launch_k<4>(k_zero_start, blocks_for(n_, 256), 256, 0, s_, r_.get(), L0.l1.get(), L0.x.get(), n_, cc.relax_weight);
        PB_CHECK_LAUNCH();
        launches_ += 1;
    }
    timing = timing_save;
    PB_CUDA(cudaMemcpyAsync(h_state_, state_.get(), sizeof(FcgState), cudaMemcpyDeviceToHost, s_));
    PB_CUDA(cudaStreamSynchronize(s_));
    const double rr0 = h_state_->rr0;
    const double rnorm0 = std::sqrt(rr0);
    int it = 0;
    double rel = 1.0;
    std::vector<double> hist{1.0};
    if (rnorm0 != 0.0) {
        // (re)capture the iteration graph
        const bool mr = rt.nranks() > 1;  // stopping test inside the graph (k_fcg_scalars4)
        if (!graph_ || graph_cc_.pre_sweeps != cc.pre_sweeps || graph_cc_.post_sweeps != cc.post_sweeps ||
            graph_cc_.coarsest_sweeps != cc.coarsest_sweeps || graph_cc_.relax_weight != cc.relax_weight ||
            graph_prec_ != precflag || graph_timing_ != timing ||
            (mr && (cap_rtol_ != rtol || cap_maxit_ != max_iters))) {
            destroy_graph();
            cap_rtol_ = rtol;
            cap_maxit_ = max_iters;
            tcount_.fill(0);
            cudaGraph_t g;
            const int64_t l0 = launches_;
            const CommStats c0 = rt.stats();
            PB_CUDA(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal));
            iteration_enqueue(cc, precflag);
            PB_CUDA(cudaStreamEndCapture(s_, &g));
            per_iter_launches_ = launches_ - l0;
            reductions_per_iter_ = static_cast<int>(rt.stats().device_reductions - c0.device_reductions);
            halos_per_iter_ = static_cast<int>(rt.stats().halo_exchanges - c0.halo_exchanges);
            halo_bytes_per_iter_ = static_cast<double>(rt.stats().halo_bytes - c0.halo_bytes);
            launches_ = l0;
            PB_CUDA(cudaGraphInstantiate(&graph_, g, 0));
            PB_CUDA(cudaGraphDestroy(g));
            graph_cc_ = cc;
            graph_prec_ = precflag;
            graph_timing_ = timing;
            // ranks sharing a GPU: nobody launches a graph whose halo waits
            // spin while a peer is still instantiating its own (instantiation
            // may synchronise the device)
            if (rt.shared_device()) rt.barrier();
        }
        const bool device_loop = loop_ok && !timing && (!mr || mr_device_loop_ok()) &&
                                 env_flag("PAIRAMG_GRAPH_LOOP", true);
        if (device_loop) {
            // the whole iteration loop as ONE graph launch: a conditional WHILE
            // node re-runs the captured iteration until k_loop_ctl clears it
            // (multi-rank: every exchange in it is a P2P kernel, no host step)
            ensure_loop_graph(cc, precflag, rtol, max_iters);
            PB_CUDA(cudaGraphLaunch(loop_graph_, s_));
            PB_CUDA(cudaMemcpyAsync(h_state_, state_.get(), sizeof(FcgState), cudaMemcpyDeviceToHost, s_));
            if (mr)
                rt.wait(s_);  // NCCL error / deadlock polling while the loop runs
            else
                PB_CUDA(cudaStreamSynchronize(s_));
            it = h_state_->it;
            launches_ += (per_iter_launches_ + 1) * (mr ? it + 1 : it);
            if (h_state_->status) fail(PAIRAMG_BREAKDOWN, "fcg: breakdown at iteration " + std::to_string(it));
            std::vector<double> dh(static_cast<size_t>(it) + 1);
            PB_CUDA(cudaMemcpy(dh.data(), hist_.get(), 8 * (it + 1), cudaMemcpyDeviceToHost));
            for (int i = 1; i <= it; ++i) hist.push_back(dh[static_cast<size_t>(i)]);
            rel = dh[static_cast<size_t>(it)];
        } else if (mr) {
            // one launch per iteration; launch j tests r_j (k_fcg_scalars4) and
            // updates to r_{j+1} unless that test already stopped the solve
            while (true) {
                PB_CUDA(cudaGraphLaunch(graph_, s_));
                launches_ += per_iter_launches_;
                PB_CUDA(cudaMemcpyAsync(h_state_, state_.get(), sizeof(FcgState), cudaMemcpyDeviceToHost, s_));
                rt.wait(s_);  // NCCL error / deadlock polling while the iteration runs
                collect_times();
                if (h_state_->status)
                    fail(PAIRAMG_BREAKDOWN, "fcg: breakdown at iteration " + std::to_string(h_state_->it));
                const int j = h_state_->stop ? h_state_->it : h_state_->it - 1;
                rel = std::sqrt(h_state_->rr) / rnorm0;
                if (j >= 1) hist.push_back(rel);
                it = j;
                if (h_state_->stop) break;
            }
        } else {
            while (true) {
                PB_CUDA(cudaGraphLaunch(graph_, s_));
                launches_ += per_iter_launches_;
                PB_CUDA(cudaMemcpyAsync(h_state_, state_.get(), sizeof(FcgState), cudaMemcpyDeviceToHost, s_));
                PB_CUDA(cudaStreamSynchronize(s_));
                collect_times();
                if (h_state_->status)
                    fail(PAIRAMG_BREAKDOWN, "fcg: breakdown at iteration " + std::to_string(h_state_->it));
                it = h_state_->it;
                rel = std::sqrt(h_state_->rr) / rnorm0;
                hist.push_back(rel);
                if (rel < rtol || it >= max_iters) break;
            }
        }
    }
    if (n_) PB_CUDA(cudaMemcpyAsync(d_u, u_.get(), 8 * n_, cudaMemcpyDeviceToDevice, s_));
    PB_CUDA(cudaEventRecord(e1, s_));
    PB_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    last_launches = launches_;
    if (st) {
        st->iterations = it;
        st->converged = rel < rtol ? 1 : 0;
        st->final_relres = rel;
        st->rnorm0 = rnorm0;
        st->t_solve_s = ms * 1e-3;
        st->t_h2d_s = 0.0;
        st->t_d2h_s = 0.0;
        st->reductions_per_iter = reductions_per_iter_;
        st->halo_exchanges_per_iter = halos_per_iter_;
        st->halo_bytes_per_iter = halo_bytes_per_iter_;
        if (st->history)
            for (int i = 0; i < st->history_cap && i < static_cast<int>(hist.size()); ++i) st->history[i] = hist[i];
    }
}

std::vector<std::string> Solver::warnings() const {
    std::vector<std::string> w = h.warnings;
    if (!cycle_warning.empty()) w.push_back(cycle_warning);
    return w;
}

// Ranks sharing one GPU (LOCAL runtime): every rank has made this call's
// allocations (the C ABI's staging buffers, pool growth -- which may
// synchronise the device) before any rank enqueues a kernel that spins on a
// peer's halo flag.  Collective, like the call itself.
void Solver::shared_gpu_fence() {
    if (rt.shared_device()) rt.barrier();
}

void Solver::vcycle(const double* d_r, double* d_x, const CycleConfig& cc) {
    if (!ready) fail(PAIRAMG_CONTRACT_VIOLATION, "vcycle: setup not run");
    cycle_warning = check_cycle(cc);
    shared_gpu_fence();
    if (n_) PB_CUDA(cudaMemcpyAsync(r_.get(), d_r, 8 * n_, cudaMemcpyDeviceToDevice, s_));
    double* out = nullptr;
    const bool t = timing;
    timing = false;
    vcycle_enqueue(0, r_.get(), out, cc);
    timing = t;
    if (n_) PB_CUDA(cudaMemcpyAsync(d_x, out, 8 * n_, cudaMemcpyDeviceToDevice, s_));
    PB_CUDA(cudaStreamSynchronize(s_));
    // the single-buffered replicated-rhs gather needs a collective step between
    // two V-cycles (inside FCG the dot allgather is one)
    if (rep_gather_.ok) rt.allreduce_sum_i64(0);
}

void Solver::spmv(int level, const double* d_x, double* d_y) {
    if (!ready) fail(PAIRAMG_CONTRACT_VIOLATION, "spmv: setup not run");
    if (level < 0 || level >= h.nl()) fail(PAIRAMG_INVALID_ARGUMENT, "spmv: level out of range");
    shared_gpu_fence();
    Level& L = *h.levels[level];
    if (L.A.n) PB_CUDA(cudaMemcpyAsync(L.xt.get(), d_x, 8 * L.A.n, cudaMemcpyDeviceToDevice, s_));
    const bool t = timing;
    timing = false;
    SellOpArgs o;
    o.op = kSpmv;
    o.x = L.xt.get();
    o.y = L.res.get();
    apply_on(L, o, -1);  // the distributed level (spmv_dist semantics), never the replicated copy
    timing = t;
    if (L.A.n) PB_CUDA(cudaMemcpyAsync(d_y, L.res.get(), 8 * L.A.n, cudaMemcpyDeviceToDevice, s_));
    PB_CUDA(cudaStreamSynchronize(s_));
}

}  // namespace pb
