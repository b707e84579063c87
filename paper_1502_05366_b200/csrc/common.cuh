// common.cuh — shared device/host plumbing for the rlra B200 engine.
//
// Errors: engine code throws rlra_b200::Error{status, message}; the C-ABI
// layer (capi.cu) catches it, stores the message in a thread-local buffer and
// returns the status.  The status values map 1:1 onto the reference's
// exception classes (reference core/errors.hpp:11-33).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/rlra_c.h"

namespace rlra_b200 {

struct Error {
    int status;
    std::string msg;
};

inline std::string fmt(const char* f, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, f);
    vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return std::string(buf);
}

[[noreturn]] inline void raise(int status, const std::string& m) { throw Error{status, m}; }

#define RLRA_CUDA(x)                                                                      \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess)                                                            \
            ::rlra_b200::raise(RLRA_ECUDA, ::rlra_b200::fmt("CUDA error %s at %s:%d",      \
                                                            cudaGetErrorString(e_),       \
                                                            __FILE__, __LINE__));         \
    } while (0)

#define RLRA_LAUNCH_CHECK() RLRA_CUDA(cudaGetLastError())

// Column-major device matrix view: element (i,j) at p[i + j*ld].
struct DMat {
    double* p = nullptr;
    int64_t rows = 0, cols = 0, ld = 0;
    __host__ __device__ double* col(int64_t j) const { return p + j * ld; }
    __host__ __device__ double& at(int64_t i, int64_t j) const { return p[i + j * ld]; }
    DMat block(int64_t r0, int64_t c0, int64_t nr, int64_t nc) const {
        DMat b;
        b.p = p + r0 + c0 * ld;
        b.rows = nr;
        b.cols = nc;
        b.ld = ld;
        return b;
    }
};

// Execution context: one device, one stream, a stream-ordered pool for
// scratch.  Everything the engine launches goes on `stream`.
struct Context {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host->device uploads overlapped with compute (lazy)
    cudaMemPool_t pool = nullptr;
    // pinned scalars for device->host flags without extra allocations
    double* h_scalars = nullptr;  // pinned, 64 doubles
    int* h_flags = nullptr;       // pinned, 64 ints
    // statistics: kernels launched by this context since last reset
    uint64_t launches = 0;
    // device grid-barrier state for the cooperative kernels (see grid_sync)
    unsigned* gbar = nullptr;
    // Cholesky-QR policy knobs (see qr.cu)
    double cholqr_pivot_floor = 1e-12;
    // force the launch-per-block Cholesky (GEMM trailing updates) for every n
    bool chol_blocked_gemm = false;
    // optional per-launch / per-phase timing with CUDA events on `stream`
    bool profile = false;
    struct ProfRec {
        const char* name;
        cudaEvent_t start, stop;
        int M, N, K;
        double flops;
    };
    std::vector<ProfRec> prof;
    // label the profiler gives the next GEMM launches (see GemmTag)
    const char* gemm_tag = "gemm";
    // pinned staging slots + host copy threads for pageable buffers (hostio.cu, lazy)
    void* stager = nullptr;
    // small_svd convergence checks deferred to the end of the API call (no
    // host sync inside the factorization): status words land in
    // h_flags[32 + i] asynchronously; the C-ABI guard reads them after its sync
    int svd_pending = 0;
    int svd_pending_mn[8][2] = {};
};

// Scoped label for GEMM launches (profiling/accounting only).
struct GemmTag {
    Context& ctx;
    const char* prev;
    GemmTag(Context& c, const char* tag) : ctx(c), prev(c.gemm_tag) { c.gemm_tag = tag; }
    ~GemmTag() { ctx.gemm_tag = prev; }
};

// Records one interval on ctx.stream when profiling is enabled, and always
// an NVTX range of the same name (host timeline for Nsight tools; a no-op
// without a tool attached).
struct ProfScope {
    Context& ctx;
    int idx = -1;
    ProfScope(Context& c, const char* name, int M = 0, int N = 0, int K = 0, double flops = 0.0)
        : ctx(c) {
        nvtxRangePushA(name);
        if (!ctx.profile) return;
        Context::ProfRec r{name, nullptr, nullptr, M, N, K, flops};
        cudaEventCreate(&r.start);
        cudaEventCreate(&r.stop);
        cudaEventRecord(r.start, ctx.stream);
        ctx.prof.push_back(r);
        idx = int(ctx.prof.size()) - 1;
    }
    ~ProfScope() {
        if (idx >= 0) cudaEventRecord(ctx.prof[idx].stop, ctx.stream);
        nvtxRangePop();
    }
};

// NVTX range for a C-ABI entry point (rlra_rsvd, rlra_qb_blocked, ...)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// RAII device scratch buffer on the context's pool.
struct Buf {
    Context* ctx = nullptr;
    void* p = nullptr;
    size_t bytes = 0;
    Buf() = default;
    Buf(Context& c, size_t b) : ctx(&c), bytes(b) {
        if (b) RLRA_CUDA(cudaMallocAsync(&p, b, c.stream));
    }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept : ctx(o.ctx), p(o.p), bytes(o.bytes) { o.p = nullptr; }
    Buf& operator=(Buf&& o) noexcept {
        release();
        ctx = o.ctx;
        p = o.p;
        bytes = o.bytes;
        o.p = nullptr;
        return *this;
    }
    ~Buf() { release(); }
    void release() {
        if (p && ctx) cudaFreeAsync(p, ctx->stream);
        p = nullptr;
    }
    double* d() const { return static_cast<double*>(p); }
    int* i() const { return static_cast<int*>(p); }
};

// A device matrix that owns its storage (ld == rows).
struct DMatBuf {
    Buf buf;
    DMat m;
    DMatBuf() = default;
    DMatBuf(Context& c, int64_t rows, int64_t cols)
        : buf(c, sizeof(double) * size_t(rows > 0 ? rows : 0) * size_t(cols > 0 ? cols : 0)) {
        m.p = buf.d();
        m.rows = rows;
        m.cols = cols;
        m.ld = rows > 0 ? rows : 1;
    }
    operator DMat() const { return m; }
};

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

// Grid-wide barrier for kernels launched with cudaLaunchCooperativeKernel
// (co-residency guaranteed).  bar[0] counts arrivals, bar[1] is the
// generation; the last CTA to arrive resets the count and publishes the next
// generation with a release store.  Waiters poll with relaxed loads and
// __nanosleep back-off and take ONE acquire fence on exit, so 147 waiting SMs
// do not saturate the L2 slice holding the flag (cooperative_groups'
// grid.sync() re-issues an acquire load + L1 invalidate per poll).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
        unsigned gen;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (atomicAdd(bar, 1u) == nb - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(bar), "r"(0u) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1u) : "memory");
        } else {
            unsigned cur, ns = 32;
            for (;;) {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
                if (cur != gen) break;
                __nanosleep(ns);
                ns = ns < 256 ? ns * 2 : 256;
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    __syncthreads();
}

}  // namespace rlra_b200
