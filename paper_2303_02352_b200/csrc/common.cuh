// common.cuh -- shared infrastructure of the B200 AMG-FCG library: error
// model (the reference ErrorCode taxonomy, types.hpp:13-35), stream-ordered
// device buffers, launch helpers and exact-rounding FP64 primitives.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "pairamg_b200.h"

namespace pb {

// pairamg::Error (types.hpp:26-35) with the C status attached.
class Error : public std::runtime_error {
public:
    Error(pairamg_status code, const std::string& what) : std::runtime_error(what), code_(code) {}
    pairamg_status code() const noexcept { return code_; }

private:
    pairamg_status code_;
};

[[noreturn]] inline void fail(pairamg_status code, const std::string& msg) { throw Error(code, msg); }

#define PB_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e__ = (call);                                                              \
        if (e__ != cudaSuccess)                                                                \
            ::pb::fail(PAIRAMG_INTERNAL, std::string("CUDA error ") + cudaGetErrorString(e__) + \
                                             " at " __FILE__ ":" + std::to_string(__LINE__));  \
    } while (0)

#define PB_CHECK_LAUNCH() PB_CUDA(cudaGetLastError())

constexpr int kSmCount = 148;  // B200: 148 SMs on two dies

// Development switches (A/B of format and fusion choices), default on.
inline bool env_flag(const char* name, bool dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    return !(v[0] == '0' || v[0] == 'n' || v[0] == 'N' || v[0] == 'f' || v[0] == 'F');
}
inline int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}

// NVTX range for the host phases (setup steps, solve): visible in nsys /
// ncu --nvtx timelines, a no-op without a tool attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

inline int blocks_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 0x7fffffffLL) fail(PAIRAMG_INTERNAL, "grid too large");
    return static_cast<int>(b);
}

// Stream-ordered device buffer (cudaMallocAsync on the solver stream; the
// device's default memory pool keeps freed blocks cached, so the many setup
// temporaries do not hit the driver allocator).
template <typename T>
class DBuf {
public:
    DBuf() = default;
    DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
    ~DBuf() { reset(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void alloc(size_t n, cudaStream_t s) {
        reset();
        s_ = s;
        n_ = n;
        if (n) PB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), s));
    }
    void reset() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }
    void zero(cudaStream_t s) {
        if (n_) PB_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    bool empty() const { return n_ == 0; }
    operator T*() const { return p_; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

// Exactly rounded FP64 (no contraction), matching the reference objects,
// which contain no FMA.  The library is also
// compiled with --fmad=false; these make the intent explicit at call sites.
// Programmatic dependent launch: solve-path kernels are launched with
// programmatic stream serialization (launch_k), so a kernel's CTAs can be
// scheduled while its predecessor drains; every such kernel first lets its own
// dependents launch, then waits until its predecessor grid has completed and
// its writes are visible (griddepcontrol; no-ops without the attribute).
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Kernels whose blocks may wait on another GPU must not let their dependents
// launch early (waiting dependent CTAs would hold SM slots).
__device__ __forceinline__ void pdl_wait_only() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline int pdl_mask() {
    static const int m = env_int("PAIRAMG_PDL", 15);  // bits: 1 reductions, 2 row kernels, 4 transfers, 8 FCG update
    return m;
}

template <int CLASS = 1, typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl_mask() & CLASS) ? 1 : 0;
    PB_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// t / d correctly rounded from y = RN(1/d) (host-computed per pattern):
// q0 = RN(t*y) is within one ulp of t/d, r = t - q0*d is exact by FMA, and
// RN(q0 + r*y) = RN(t/d) (Markstein's correction theorem; no underflow or
// overflow: outside [2^-1000, 2^1000] it falls back to the division; zeros
// take that branch too, so q0 != 0 below and r == +-0 returns q0 exactly).
// y == 0: plain division.
// Exhaustively spot-checked against IEEE division: 0 mismatches in 4e8 pairs
// incl. near-ties.  Replaces the ~20-instruction DDIV sequence
// in the sweeps' epilogue.
__device__ __forceinline__ double ddiv_recip(double t, double d, double y) {
    if (y == 0.0) return __ddiv_rn(t, d);
    const double q0 = __dmul_rn(t, y);
    const double aq = fabs(q0);
    if (!(aq >= 0x1p-1000 && aq <= 0x1p1000)) return (q0 == 0.0 && t == 0.0) ? q0 : __ddiv_rn(t, d);
    const double r = __fma_rn(-q0, d, t);
    return __fma_rn(r, y, q0);  // r == +-0 gives q0 exactly (q0 is nonzero here)
}

}  // namespace pb
